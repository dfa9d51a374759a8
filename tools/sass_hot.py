"""Summarise an ncu source-page SASS CSV (gz): instructions by executed count and by stall
samples, with the dominant stall reasons.   python tools/sass_hot.py file.csv.gz [top]"""
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), encoding="utf-8")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
tot_samples = sum(int(r[ix["# Samples"]] or 0) for r in body)
tot_exec = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
print("instructions executed (warp):", tot_exec, " samples:", tot_samples)
agg = {}
for r in body:
    for h in stall_cols:
        v = r[ix[h]]
        if v and v != "-":
            agg[h] = agg.get(h, 0) + int(float(v))
print("stall reasons:", sorted(((v, k) for k, v in agg.items()), reverse=True)[:10])
print("--- top by samples (addr idx, samples, executed, top stalls, instr)")
order = sorted(range(len(body)), key=lambda i: -int(body[i][ix["# Samples"]] or 0))
for i in order[:top]:
    r = body[i]
    st = sorted(((int(float(r[ix[h]])) if r[ix[h]] not in ("", "-") else 0, h[6:]) for h in stall_cols), reverse=True)[:2]
    print(f"{i:5d} {r[ix['# Samples']]:>7} {r[ix['Instructions Executed']]:>10} {st} {r[ix['Source']].strip()}")
