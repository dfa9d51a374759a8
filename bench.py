#!/usr/bin/env python
"""Benchmark of the GPU-UMAP hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--knn-mode exact|tensor] [--sgd-mode deterministic|hogwild]

A step = one pass of the whole hot path over the config's synthetic input: umap_fit
(a1 validate, a2 kNN, a3/a4 rho-sigma-membership, a5 fuzzy union, a6/a7 schedule +
init, a8 SGD epochs) followed by umap_trustworthiness (a10) of the result.
N = 1: configs[1] (C2, MNIST-shaped 70,000 x 784, k=15, 2-D, 500 epochs).
N > 1: the kNN index rows and the trust rows are sharded across ranks (NCCL
all-gather / all-reduce), graph + SGD replicated (strong scaling, dist.py).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fit wall-s & SGD edge-updates/s at MNIST-70k shape; trustworthiness"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--knn-mode", default="tensor", choices=["exact", "tensor"])
    ap.add_argument("--sgd-mode", default="deterministic", choices=["deterministic", "hogwild"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], None, set()
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax = float(s[1])
            except ValueError:
                continue
            for nm, v in zip(names, s[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if smax and x > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, \
            "fallback"


def profile_traffic(name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("kernels", {}).get(name, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cfg_of(name):
    import synth
    c = dict(synth.CONFIGS[name])
    return c


# ----------------------------------------------------------------------------- cpu oracle timing
def oracle_step_estimate(X, k, n_epochs, knn_rows=32, graph_rows=2000, sgd_epochs=6, trust_rows=32, trust_k=15):
    """Time the CPU oracle (1 thread, as it stands) on bounded samples of one step and
    extrapolate to the full step: kNN and trust rows are independent (linear in rows);
    the graph stages and SGD are timed on a `graph_rows` sub-problem and scaled by
    n / graph_rows (nnz per row is constant) and by the epoch count."""
    import numpy as np
    from oracle import oracle as O
    O.build()
    n = X.shape[0]
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n, knn_rows, replace=False))
    t0 = time.perf_counter()
    for r in rows:
        O.knn(X[r:r + 1], X, k, self_offset=int(r))
    t_knn = (time.perf_counter() - t0) * n / knn_rows
    Xs = X[:graph_rows]
    idx, dist = O.knn(Xs, Xs, k, self_offset=0)  # untimed: input of the graph stages
    t0 = time.perf_counter()
    rho, sigma = O.smooth_knn(dist)
    w = O.membership(dist, rho, sigma)
    indptr, col, val = O.fuzzy_union(idx, w)
    t_graph = (time.perf_counter() - t0) * n / graph_rows
    Y0 = O.random_init(graph_rows, 2, 0)
    a, b = 1.5769434603, 0.8950608779
    t0 = time.perf_counter()
    O.optimize(indptr, col, val, Y0, a, b, n_epochs, e_begin=1, e_end=1 + sgd_epochs, m=5, seed=0)
    t_sgd = (time.perf_counter() - t0) * (n / graph_rows) * (n_epochs - 1) / sgd_epochs
    Y = O.random_init(n, 2, 1)
    trows = np.sort(rng.choice(n, trust_rows, replace=False))
    t0 = time.perf_counter()
    for r in trows:
        O.trust_penalty(X, Y, trust_k, int(r), int(r) + 1)
    t_trust = (time.perf_counter() - t0) * n / trust_rows
    total = t_knn + t_graph + t_sgd + t_trust
    sample = (f"oracle 1 thread: kNN {knn_rows} query rows x {n} refs (x{n / knn_rows:.0f}); graph+union on "
              f"{graph_rows} rows (x{n / graph_rows:.0f}); SGD {sgd_epochs} epochs on that graph "
              f"(x{(n / graph_rows) * (n_epochs - 1) / sgd_epochs:.0f}); trust {trust_rows} rows x {n} (x{n / trust_rows:.0f}); "
              f"extrapolated linearly to one full step")
    return total, {"knn_s": t_knn, "graph_s": t_graph, "sgd_s": t_sgd, "trust_s": t_trust}, sample


def run_reference(args):
    """--impl reference: the oracle (this task's reference arm) timed on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    c = cfg_of(args.config)
    X = synth.lowrank(c["n"], c["d"], c["blobs"], c["seed"])
    times = []
    parts = None
    for i in range(args.warmup + args.steps):
        t, parts, sample = oracle_step_estimate(X, c["k"], c["n_epochs"], knn_rows=8, graph_rows=1000, sgd_epochs=3,
                                                trust_rows=8)
        if i >= args.warmup:
            times.append(t)
    v = sum(times) / len(times)
    line = {"metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} lowrank {c['n']}x{c['d']} k={c['k']} 2-D {c['n_epochs']} epochs"
                                   f" fit + trust(k=15)", "l2": "n/a (CPU)"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "oracle", "sample": sample,
                             "stages_s": parts},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2008_00325_b200 as U
    from paper_2008_00325_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = cfg_of(args.config)
    n, d, k, N = c["n"], c["d"], c["k"], c["n_epochs"]
    trust_k = 15
    X_host = torch.from_numpy(synth.lowrank(n, d, c["blobs"], c["seed"])).pin_memory()
    X = X_host.to("cuda", non_blocking=False)
    torch.cuda.synchronize()
    kw = dict(n_neighbors=k, n_epochs=N, seed=0, sgd_mode=args.sgd_mode, knn_mode=args.knn_mode)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def step(Xd):
        if world == 1:
            Y, st = U.fit(Xd, **kw)
            T, S = U.trustworthiness(Xd, Y, trust_k, knn_mode=args.knn_mode)
        else:
            Y, st = D.sharded_fit(Xd, **kw)
            T, S = D.sharded_trustworthiness(Xd, Y, trust_k, knn_mode=args.knn_mode)
        return Y, st, T

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(X)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = U.kernel_launch_count()
    stats = []
    T = None
    barrier()
    for i in range(args.steps):
        flush.fill_(float(i))  # L2 flush between timed steps (untimed)
        ev[i][0].record()
        Y, st, T = step(X)
        ev[i][1].record()
        stats.append(st)
    barrier()
    launches = U.kernel_launch_count() - launches0
    clk = clocks.stop()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms = sum(ms_steps) / len(ms_steps)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- e2e through the public API with host buffers: H2D of X, fit, trust, D2H of Y and T
    e2e = None
    if not args.no_e2e:
        e2e_ms = []
        for i in range(max(1, min(args.steps, 3))):
            flush.fill_(float(i))
            barrier()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            Xd = X_host.to("cuda", non_blocking=True)
            Y, st, Te = step(Xd)
            Yh = Y.to("cpu")
            e1.record()
            torch.cuda.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
            del Xd
        em = sum(e2e_ms) / len(e2e_ms)
        if world > 1:
            t = torch.tensor([em], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em = float(t.item())
        e2e = {"value": em / 1e3, "unit": "s", "h2d_bytes_per_step": int(X_host.numel() * 4),
               "d2h_bytes_per_step": int(Yh.numel() * 4 + 8)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    st = stats[-1]
    pk, pk_kind = peaks()
    positives = st["positives"]
    sgd_s = st["ms_sgd"] / 1e3
    # dominant kernel: the distance-tile kernel of the kNN stage (exact mode: fp32 SIMT ALU-bound)
    if args.knn_mode == "exact":
        # 2 fp32 lane-instructions (FADD + FFMA) per (query, reference, feature); peak = 148 SMs x
        # 128 FP32 lanes x sm_max clock
        work = 2.0 * n * n * d
        sm_hz = (pk.get("sm_max_mhz") or 1965.0) * 1e6
        peak = 148 * 128 * sm_hz / 1e12
        achieved = work / (st["ms_knn"] / 1e3) / 1e12
        roof = {"kernel": "dist_tile_kernel<16,0> (kNN, exact fp32)", "bound": "alu", "achieved": achieved,
                "peak": peak, "unit": "Tinst/s (fp32 FADD+FFMA lane-ops)", "frac": achieved / peak,
                "traffic": profile_traffic("dist_tile_kernel"), "peak_source": "derived: 148 SM x 128 lanes x sm_max",
                "duration_ms": st["ms_knn"]}
    else:
        flops = 2.0 * n * n * d
        peak = pk.get("bf16_tflops", 1590.0)
        achieved = flops / (st["ms_knn"] / 1e3) / 1e12
        roof = {"kernel": "knn_tc_kernel (tcgen05 BF16 + re-rank)", "bound": "tensor", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": profile_traffic("knn_tc"),
                "peak_source": pk_kind + " bf16 burst", "duration_ms": st["ms_knn"]}
    # SGD against the HBM byte model: 8 B/edge/epoch + 4*dim*(m+1) B/positive + 8*dim*n B/epoch
    sgd_bytes = 8.0 * st["nnz"] * (N - 1) + 4 * 2 * 6 * positives + 8 * 2 * n * (N - 1)
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if world > 1 else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.config} lowrank {n}x{d} k={k} 2-D {N} epochs fit + trust(k={trust_k})",
                   "knn_mode": args.knn_mode, "sgd_mode": args.sgd_mode,
                   "l2": "flushed (256 MiB write) between timed steps; X = %.0f MB > L2" % (n * d * 4 / 1e6),
                   "parallelism": f"kNN+trust rows sharded x{world}" if world > 1 else "1 GPU"},
        "stages_ms": {"knn": st["ms_knn"], "smooth": st["ms_smooth"], "union": st["ms_union"],
                      "init": st["ms_init"], "sgd": st["ms_sgd"], "fit_total": st["ms_total"],
                      "trust": ms - st["ms_total"]},
        "fit_s": st["ms_total"] / 1e3,
        "sgd_edge_updates_per_s": positives / sgd_s if sgd_s > 0 else None,
        "sgd_hbm_model_frac": (sgd_bytes / sgd_s / 1e9) / pk["hbm_gbs"] if sgd_s > 0 else None,
        "positives": positives, "nnz": st["nnz"], "trustworthiness": T,
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "peaks": {"source": pk_kind, "hbm_gbs": pk.get("hbm_gbs"), "bf16_tflops": pk.get("bf16_tflops")},
    }
    if not args.no_cpu_baseline and world == 1:
        t_cpu, parts, sample = oracle_step_estimate(np.ascontiguousarray(X_host.numpy()), k, N)
        line["cpu_baseline"] = {"value": t_cpu, "unit": "s", "cores": 1, "kind": "oracle", "sample": sample,
                                "stages_s": parts}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
