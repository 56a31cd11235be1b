"""Config-5 latency probe: is the 1024-deployment replay bound by its slowest
trace (latency) or by the whole launch (throughput)?

    python tools/c5_probe.py [q]

Runs the full top-1024 launch, then sub-launches: the traces grouped by warp
count W, the 16 traces with the most steps, and the single slowest one.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2504_15303_b200 as hs  # noqa: E402
from paper_2504_15303_b200 import _native as nat  # noqa: E402
from paper_2504_15303_b200 import planner  # noqa: E402
from paper_2504_15303_b200 import workloads as wl  # noqa: E402


def main():
    q = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 100_000
    eng = nat.engine_for(0)
    cluster, reqs, params, _I, _O = bench.search_inputs(10_000)
    t = planner.build_tables(cluster, reqs, params, engine=eng)
    top, _nf, _ = planner.search_topk(t, 1024, engine=eng)
    idx_all = top["index"]
    I1, O1 = wl.trace_lengths(q, seed=0)
    M = len(t.names)
    nd = np.asarray(t.n_degrees, np.int64)
    x = np.asarray(idx_all, np.int64).copy()
    digs = np.empty((len(x), M), np.int64)
    for m in range(M - 1, -1, -1):
        digs[:, m] = x % nd[m]
        x //= nd[m]
    n_inst = t.entries["instance_count"][np.arange(M)[None, :], digs].sum(axis=1)

    def run(sel, reps=2):
        n = len(sel)
        off = np.arange(n + 1, dtype=np.int64) * q
        ms = []
        for _ in range(reps):
            res = hs.replay_candidates(t, params, idx_all[sel], hs.PolicyConfig(), np.arange(n), off,
                                       np.tile(I1, n), np.tile(O1, n), np.tile(O1, n), engine=eng, want_assign=False)
            ms.append(res.kernel_ms)
        assert (res.result["error"] == 0).all()
        return min(ms), res

    full_ms, res = run(np.arange(1024))
    if hasattr(eng.lib, "hs_debug_timers"):  # diagnostic build (HS_LIB=...timers.so)
        import ctypes
        buf = np.zeros(24, np.uint64)
        eng.lib.hs_debug_timers(buf.ctypes.data_as(ctypes.c_void_p), 1)
        run(np.arange(1024), reps=1)
        eng.lib.hs_debug_timers(buf.ctypes.data_as(ctypes.c_void_p), 0)
        nw = int(((n_inst + 31) // 32).sum())
        names = {0: "advance", 1: "price", 2: "evaluate", 21: "  exp part (lanes that need it)", 16: "minmax",
                 20: "  barrier wait", 17: "commit", 18: "drain", 19: "whole"}
        print("cycles per warp per request:", {v: round(float(buf[k]) / nw / q, 1) for k, v in names.items()})
        print("cycles per warp (whole trace): %.3g" % (float(buf[19]) / nw))
        calls = max(int(buf[7]), 1)
        print("event-step lane calls %d (%.2f per request per trace), cycles per call: retire %.0f admit %.0f price %.0f, "
              "steps with nact>kHS %.3f, mean nact %.1f"
              % (calls, calls / (1024 * q), buf[3] / calls, buf[4] / calls, buf[5] / calls, buf[14] / calls,
                 buf[15] / calls))
        print("rescans per event call %.4f (mean length %.1f)" % (buf[10] / calls, buf[11] / max(int(buf[10]), 1)))
        if "--timers-only" in sys.argv:
            return
    steps = res.result["n_steps"].astype(np.int64)
    W = (n_inst + 31) // 32
    print(f"full: {full_ms:.1f} ms; instances min/med/max {n_inst.min()}/{int(np.median(n_inst))}/{n_inst.max()}; "
          f"W counts {dict(zip(*np.unique(W, return_counts=True)))}")
    print(f"steps per trace: min {steps.min()} med {int(np.median(steps))} max {steps.max()}; "
          f"steps per instance med {np.median(steps / n_inst):.0f} max {(steps / n_inst).max():.0f}")
    for w in np.unique(W):
        sel = np.nonzero(W == w)[0]
        ms, _ = run(sel)
        print(f"W={w}: {len(sel)} traces alone: {ms:.1f} ms")
    order = np.argsort(-steps)
    for k in (1, 16, 148):
        ms, r = run(order[:k])
        print(f"top-{k} by steps alone: {ms:.1f} ms (steps {steps[order[:k]].min()}..{steps[order[0]]}, "
              f"instances {n_inst[order[:k]].min()}..{n_inst[order[:k]].max()})")
    order_n = np.argsort(-n_inst, kind="stable")
    ms, _ = run(order_n[:1])
    print(f"widest trace alone ({n_inst[order_n[0]]} instances, {steps[order_n[0]]} steps): {ms:.1f} ms")
    one = np.nonzero(W == 1)[0][:1]
    if len(one):
        ms, _ = run(one)
        print(f"one W=1 trace alone ({n_inst[one[0]]} instances, {steps[one[0]]} steps): {ms:.1f} ms")


if __name__ == "__main__":
    main()
