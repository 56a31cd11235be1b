"""Per-kernel resource usage of the built engine (registers, shared memory,
local-memory spill) from `cuobjdump -res-usage`, plus a static SASS mnemonic
census of the engine's own kernels (FP64 ops, branches, barriers, memory ops)
from `cuobjdump -sass`.  Writes profiles/resources_<tag>.txt.

    python tools/resource_summary.py r02
"""

from __future__ import annotations

import collections
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2504_15303_b200" / "libhetserve_b200.so"
CLASSES = {
    "fp64": ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"),
    "int/logic": ("IADD3", "IMAD", "LOP3", "ISETP", "SHF", "LEA", "SEL", "IMNMX", "FLO", "POPC", "BREV"),
    "convert": ("I2F", "F2I", "F2F", "I2I"),
    "shared": ("LDS", "STS", "ATOMS"),
    "global/local": ("LDG", "STG", "LDL", "STL", "ATOMG", "RED"),
    "sync/shuffle": ("BAR", "SHFL", "VOTE", "MATCH", "REDUX", "WARPSYNC", "BSSY", "BSYNC"),
    "branch": ("BRA", "BRX", "CALL", "RET", "EXIT"),
}


def demangle(names: list[str]) -> list[str]:
    r = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True)
    out = r.stdout.splitlines() if r.returncode == 0 else names
    return out if len(out) == len(names) else names


def short(name: str) -> str:
    depth = 0
    for i, ch in enumerate(name):
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            name = name[:i]
            break
    name = name.removeprefix("void ").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name[:90]


def main(tag: str) -> None:
    res = subprocess.run(["cuobjdump", "-res-usage", str(LIB)], capture_output=True, text=True, check=True).stdout
    rows = re.findall(r"Function (\S+):\n\s+REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", res)
    mangled = [r[0] for r in rows]
    names = demangle(mangled)
    lines = [f"# cuobjdump -res-usage {LIB.name} (sm_100a, -O3 -fmad=false)",
             f"{'kernel':90s} {'REG':>4s} {'STACK':>5s} {'SHARED':>7s} {'LOCAL':>5s}"]
    for n, (_m, reg, stack, shared, local) in sorted(zip(names, rows), key=lambda x: short(x[0])):
        if "cub" in n or "thrust" in n:
            continue
        lines.append(f"{short(n):90s} {reg:>4s} {stack:>5s} {shared:>7s} {local:>5s}")
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    per = collections.defaultdict(collections.Counter)
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m and cur:
            per[cur][m.group(1).split(".")[0]] += 1
    keep = [k for k in per if re.search(r"k_replay|k_search|k_topk|k_build|k_rng|k_exp", k)]
    dn = dict(zip(keep, demangle(keep)))
    lines += ["", "# static SASS census (instruction count in the binary, not executed)",
              f"{'kernel':90s} {'total':>6s} " + " ".join(f"{c:>12s}" for c in CLASSES)]
    for k in sorted(keep, key=lambda k: short(dn[k])):
        c = per[k]
        tot = sum(c.values())
        cls = [sum(c[o] for o in ops) for ops in CLASSES.values()]
        lines.append(f"{short(dn[k]):90s} {tot:>6d} " + " ".join(f"{v:>12d}" for v in cls))
    tc = sum(per[k][o] for k in keep for o in ("UTCMMA", "UTCHMMA", "UTCQMMA", "UBLKCP", "UTMALDG"))
    lines += ["", f"# tcgen05/TMA mnemonics in the engine's kernels: {tc} (none expected: no contraction on the path,"
              " see DESIGN.md 'Why no tensor cores / TMA')"]
    out = ROOT / "profiles" / f"resources_{tag}.txt"
    out.write_text("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
