"""Every BASELINE.json config at full size on one GPU, with its parity check against the
oracle (or the exact GPU path where the oracle would take hours), one JSON line each.

    python tools/run_configs.py [C1 C3 C4 C5]      (C2 is bench.py's workload)
"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_2008_00325_b200 as U
from oracle import oracle as O

A_, B_ = 1.5769434603, 0.8950608779


def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, time.perf_counter() - t


def c1():
    c = synth.CONFIGS["C1"]
    X = synth.make("C1"); Xg = torch.from_numpy(X).cuda()
    out = {"config": "C1 digits-shaped 1797x64 B=10, k=15, 200 epochs"}
    for knn_mode in ["exact", "tensor"]:
        for sgd in ["deterministic", "hogwild"]:
            U.fit(Xg, n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=1, sgd_mode=sgd, knn_mode=knn_mode, trust_k=15)
            (Y, st), t = timed(lambda: U.fit(Xg, n_neighbors=15, n_epochs=200, a=A_, b=B_, seed=1, sgd_mode=sgd,
                                             knn_mode=knn_mode, trust_k=15))
            out[f"{knn_mode}/{sgd}"] = {"fit_trust_s": t, "trust": st["trustworthiness"], "sgd_ms": st["ms_sgd"]}
    t0 = time.perf_counter()
    Yr = O.fit(X, k=15, n_epochs=200, a=A_, b=B_, seed=1, mode="deterministic")
    T_ref = O.trustworthiness(X, Yr, 15)
    out["oracle"] = {"fit_trust_s_1thread": time.perf_counter() - t0, "trust": T_ref}
    out["parity"] = {"max_abs_trust_diff": max(abs(v["trust"] - T_ref) for k, v in out.items() if "/" in k),
                     "bar": 0.005}
    return out


def c3():
    c = synth.CONFIGS["C3"]
    X = synth.make("C3"); Xg = torch.from_numpy(X).cuda()
    out = {"config": "C3 60000x3072 B=20, k=15, 200 epochs, tensor kNN, trust k=5"}
    U.fit(Xg, n_neighbors=15, n_epochs=200, knn_mode="tensor", trust_k=5)
    (Y, st), t = timed(lambda: U.fit(Xg, n_neighbors=15, n_epochs=200, knn_mode="tensor", trust_k=5))
    (Te, Se), te = timed(lambda: U.trustworthiness(Xg, Y, 5, knn_mode="exact"))
    out.update(fit_trust_s=t, stages_ms={k: v for k, v in st.items() if k.startswith("ms_")},
               trust_tensor=st["trustworthiness"], S_tensor=st["trust_penalty"], S_exact=Se, trust_exact_s=te,
               parity={"S_tensor == S_exact": st["trust_penalty"] == Se})
    gi, gd = U.knn(Xg, Xg, 15, exclude_self=True, mode="tensor")
    rows = np.random.default_rng(0).choice(c["n"], 8, replace=False)
    ok = 0
    for r in rows:
        ri, rd = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        ok += int(np.array_equal(gi[r].cpu().numpy(), ri[0]) and np.array_equal(gd[r].cpu().numpy(), rd[0]))
    out["parity"]["sampled_knn_rows_bitexact"] = f"{ok}/{len(rows)}"
    return out


def c4():
    c = synth.CONFIGS["C4"]
    X = synth.make("C4"); Xg = torch.from_numpy(X).cuda()
    out = {"config": "C4 1,000,000x50 B=30, k=15, 200 epochs (1 GPU: the whole index)"}
    (gi, gd), tk = timed(lambda: U.knn(Xg, Xg, 15, exclude_self=True, mode="tensor"))
    (gi, gd), tk = timed(lambda: U.knn(Xg, Xg, 15, exclude_self=True, mode="tensor"))
    rows = np.random.default_rng(0).choice(c["n"], 8, replace=False)
    ok = 0
    gin, gdn = gi.cpu().numpy(), gd.cpu().numpy()
    for r in rows:
        ri, rd = O.knn(X[r:r + 1], X, 15, self_offset=int(r))
        ok += int(np.array_equal(gin[r], ri[0]) and np.array_equal(gdn[r], rd[0]))
    (Y, st), t = timed(lambda: U.fit(Xg, n_neighbors=15, n_epochs=200, knn_mode="tensor"))
    out.update(knn_tensor_s=tk, fit_s=t, stages_ms={k: v for k, v in st.items() if k.startswith("ms_")},
               nnz=st["nnz"], positives=st["positives"],
               sgd_edge_updates_per_s=st["positives"] / (st["ms_sgd"] / 1e3),
               parity={"sampled_knn_rows_bitexact": f"{ok}/{len(rows)}"})
    return out


def c5():
    model = synth.lowrank_model(784, 10, 4)
    Xtr = synth.lowrank_sample(model, 100000, 40)
    Xg = torch.from_numpy(Xtr).cuda()
    out = {"config": "C5 fit 100,000x784 then umap_transform of 8,000,000x784 (8 chunks of 1M, on device)"}
    (Ytr, st), tf = timed(lambda: U.fit(Xg, n_neighbors=15, n_epochs=200, knn_mode="tensor", a=A_, b=B_))
    t_tr = 0.0
    checks = []
    for ch in range(8):
        Xq = synth.lowrank_sample_device(model, 1000000, 41 + ch)
        Yq, t = timed(lambda: U.transform(Xg, Ytr, Xq, q_offset=ch * 1000000, n_neighbors=15, n_epochs=200,
                                          knn_mode="tensor", a=A_, b=B_))
        t_tr += t
        if ch in (0, 7):
            for r in (0, 999999):
                xr = Xq[r:r + 1].cpu().numpy()
                yo = O.transform(Xtr, Ytr.cpu().numpy(), xr, k=15, n_epochs=200, a=A_, b=B_, seed=0,
                                 q_offset=ch * 1000000 + r)
                checks.append(float(np.abs(Yq[r].cpu().numpy() - yo[0]).max()))
        del Xq, Yq
    out.update(fit_s=tf, transform_s=t_tr, transform_rows_per_s=8e6 / t_tr,
               parity={"sampled_rows_max_abs_diff_vs_oracle": checks,
                       "note": "end-to-end (67 epochs of per-row fp32 SGD vs fp64 oracle); per-epoch parity is in tests"})
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C3", "C4", "C5"]
    for w in which:
        r = {"C1": c1, "C3": c3, "C4": c4, "C5": c5}[w]()
        print(json.dumps(r), flush=True)
