"""Summarise an ncu --set full report into profiles/: per kernel duration, DRAM bytes,
L2 sectors, SM / tensor / DRAM throughput.  usage: python tools/ncu_summary.py <rep> <out.json> [<launches.csv>]"""
import csv, io, json, subprocess, sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",  # tcgen05 tensor pipe busy
     "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
     "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
     "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
rep, out = sys.argv[1], sys.argv[2]
if rep.endswith(".csv") or rep.endswith(".csv.gz"):  # a raw-page CSV exported on the GPU box
    import gzip
    raw = (gzip.open(rep, "rt") if rep.endswith(".gz") else open(rep)).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = dict(zip(h, rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "second": 1e9, "sector": 1, "Ksector": 1e3, "Msector": 1e6, "Gsector": 1e9,
         "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}
res = {"source": rep, "kernels": {}}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("umapb200::", "").replace("<unnamed>::", "")
    rec = {}
    for m in M:
        col = m if m in d else next((c for c in d if c.endswith("." + m)), None)  # section-prefixed names
        if col is not None:
            try:
                rec[m] = float(d[col].replace(",", "")) * SCALE.get(units.get(col, ""), 1)
            except ValueError:
                rec[m] = d[col]
    if "dram__bytes_read.sum" in rec:
        rec["dram_bytes_per_launch"] = rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
    key = name
    i = 2
    while key in res["kernels"]:
        key = f"{name}#{i}"; i += 1
    res["kernels"][key] = rec
json.dump(res, open(out, "w"), indent=1)
for k, v in res["kernels"].items():
    print(f"{k[:48]:48s} {v.get('gpu__time_duration.sum', 0) / 1e6:9.3f} ms  dram {v.get('dram_bytes_per_launch', 0) / 1e6:9.1f} MB"
          f"  L2 {v.get('lts__t_sectors.sum', 0) * 32 / 1e9:7.2f} GB  sm {v.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%"
          f"  tensor pipe {v.get('sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', '-')}%")
