"""Group an ncu source page (csv, --print-source cuda,sass) of k_replay into
the kernel's phases by replay.cu line ranges found from marker comments.
Usage: python tools/ncu_phases.py s.csv [N top lines]"""
import csv
import pathlib
import re
import sys

SRC = pathlib.Path(__file__).resolve().parents[1] / "paper_2504_15303_b200" / "csrc" / "replay.cu"
lines = SRC.read_text().splitlines()


def find(pat, start=0):
    for i in range(start, len(lines)):
        if re.search(pat, lines[i]):
            return i + 1
    raise SystemExit(f"marker not found: {pat}")


ev0 = find(r"auto event_step = \[&\]")
adv0 = find(r"auto advance = \[&\]")
pure0 = find(r"const bool pure = valid && sched")
pure1 = find(r"n_steps \+= k - k0;")
aerr0 = find(r"const unsigned eb = __ballot_sync")
main0 = find(r"const bool is_static = c_rep.mode == 1;")
price0 = find(r"price \(arrival, class\) pairs")
arr0 = find(r"for \(int al = 0; al < n_in; \+\+al\)")
choose0 = find(r"---- choose")
eval0 = find(r"---- evaluate")
err0 = find(r"const unsigned errb = __ballot_sync")
mm0 = find(r"if \(eval_all\) \{", err0)
com0 = find(r"---- commit")
tail0 = find(r"if \(assign && wsub == 0")
phases = [("heap/okey helpers", 1, ev0 - 150 if ev0 > 150 else 1), ("prologue", 200, ev0 - 1),
          ("event_step", ev0, adv0 - 1), ("advance ctl", adv0, pure0 - 1), ("pure steps", pure0, pure1),
          ("advance ctl", pure1 + 1, aerr0 - 1), ("advance err", aerr0, main0 - 1),
          ("arrivals+price", main0, arr0 - 1), ("adv call+shfl", arr0, choose0 - 1), ("choose nonOS", choose0, eval0 - 1),
          ("evaluate", eval0, err0 - 1), ("err check", err0, mm0 - 1), ("min-max", mm0, com0 - 1),
          ("commit", com0, tail0 - 1), ("tail", tail0, len(lines))]
rows = list(csv.reader(open(sys.argv[1])))
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        ln = int(r[0])
        d = dict(zip(hdr, r))
        agg[(cur, ln)] = (int(d["Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0))
    except ValueError:
        continue
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
ph = {}
for (f, ln), (i, s) in agg.items():
    name = "other:" + f
    if f == "replay.cu":
        name = "heap/okey helpers" if ln < 200 else "?"
        for n, a, b in phases[1:]:
            if a <= ln <= b:
                name = n
                break
    pi, ps = ph.get(name, (0, 0))
    ph[name] = (pi + i, ps + s)
print(f"total warp inst {ti}, stall samples {ts}")
for n, (i, s) in sorted(ph.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:24s} inst {i / ti * 100:5.1f}%  stall {s / ts * 100:5.1f}%")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print()
for (f, ln), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    src = lines[ln - 1].strip()[:70] if f == "replay.cu" else ""
    print(f"{s / ts * 100:5.1f}% stall {i / ti * 100:5.1f}% inst  {f}:{ln}  {src}")
