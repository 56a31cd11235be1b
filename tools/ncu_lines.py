"""Aggregate an ncu source page (--page source --csv --print-source
cuda,sass) per CUDA source line: share of executed instructions and of warp
stall samples.  Usage: ncu -i X.ncu-rep --page source --csv --print-source
cuda,sass --kernel-name regex:K > s.csv; python tools/ncu_lines.py s.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, hdr, agg = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr, r))
    try:
        agg[(cur_file, line, r[1][:70])] = (int(d["Instructions Executed"] or 0),
                                            int(d["Warp Stall Sampling (All Samples)"] or 0))
    except ValueError:
        continue
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
print("total inst", tot, "stall samples", stot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n_top]:
    print(f"{v[0] / tot * 100:5.1f}% inst {v[1] / stot * 100:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
