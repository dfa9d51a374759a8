#!/bin/bash
# per-kernel device time (ncu launch list) of one C2 fit + trust, for the kernels matching $1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$1" --csv \
    python tools/profile_step.py --knn-mode tensor 2>/dev/null > /tmp/lt.csv
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("/tmp/lt.csv")))
h = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r)); k = d["Kernel Name"].split("(")[0][-60:]
        agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += float(d["Metric Value"].replace(",", ""))
for k, (c, t) in agg.items(): print(f"{k:60s} {c:4d} {t / 1e6:8.3f} ms")
PY
