"""Small fixed workloads for ncu captures of the engine's kernels.

    python tools/profile_kernels.py replay [traces] [q]
    python tools/profile_kernels.py search
    python tools/profile_kernels.py config5 [deployments] [q]

Runs one warm-up call and one measured call; prints the kernel time.
"""

from __future__ import annotations

import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2504_15303_b200 as hs  # noqa: E402
from paper_2504_15303_b200 import _native as nat  # noqa: E402
from paper_2504_15303_b200 import planner  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "replay"
    eng = nat.engine_for(0)
    if what == "replay":
        T = int(sys.argv[2]) if len(sys.argv) > 2 else 1184
        q = int(sys.argv[3]) if len(sys.argv) > 3 else 20_000
        off, I, O, Tarr = bench.replay_inputs(0, T, q, 140.0)
        rc, config, params = bench.replay_deployment()
        reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
        # device-resident inputs: kernel time only (as bench.py's value)
        from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
        handles = build_instances(rc, config, params)
        pol = hs.PolicyConfig()
        inst = engine_instances(handles, pol)
        ps = _policy_struct(pol, len(handles), hs.kv_bytes_per_token(rc.model))
        d = {}
        for name, arr in (("off", off), ("I", I), ("O", O), ("T", Tarr)):
            d[name] = eng.device_alloc(arr.nbytes)
            eng.h2d(d[name], arr)
        d["a"] = eng.device_alloc(len(I))
        d["m"] = eng.device_alloc(T * len(handles) * nat.METRICS_DTYPE.itemsize)
        d["r"] = eng.device_alloc(T * nat.RESULT_DTYPE.itemsize)
        times = []
        for _ in range(reps):
            eng.replay_device(inst, ps, T, d["off"], d["I"], d["O"], d["O"], d["T"], d["a"], d["m"], d["r"])
            times.append(eng.last_kernel_ms)
        import numpy as np
        res = np.zeros(T, nat.RESULT_DTYPE)
        eng.d2h(res, d["r"])
        assert (res["error"] == 0).all()

        class _R:
            pass
        r = _R()
        r.kernel_ms = min(times[1:]) if len(times) > 1 else times[0]
        r.result = res
        if reps > 2:
            print("kernel ms per rep:", [round(x, 1) for x in times])
        print(f"replay {T} traces x {q}: {r.kernel_ms:.2f} ms, {T * q / r.kernel_ms * 1e3:.3g} req/s, "
              f"{r.result['n_steps'].sum() / (T * q):.1f} steps/request")
        if hasattr(eng.lib, "hs_debug_timers"):
            import ctypes
            import numpy as np
            buf = np.zeros(24, np.uint64)
            eng.lib.hs_debug_timers(buf.ctypes.data_as(ctypes.c_void_p), 1)
            eng.replay_device(inst, ps, T, d["off"], d["I"], d["O"], d["O"], d["T"], d["a"], d["m"], d["r"])
            eng.lib.hs_debug_timers(buf.ctypes.data_as(ctypes.c_void_p), 0)
            names = ["advance", "price", "evaluate", "ev_retire", "ev_admit", "ev_price", "pure_phase"]
            per = buf[:7].astype(float) / (T * q)
            print("cycles per arrival per warp:", {n: round(v, 1) for n, v in zip(names, per)})
            calls = max(int(buf[7]), 1)
            print("event_step calls per arrival:", calls / (T * q), " cycles per call: retire %.0f admit %.0f price %.0f"
                  % (buf[3] / calls, buf[4] / calls, buf[5] / calls))
            n = T * q
            print("per arrival: outer passes %.2f, lanes in event phase per pass %.2f, pure-block passes %.2f, "
                  "lane pure blocks %.2f, rescans %.4f (mean len %.1f), event steps with nact>16: %.3f, mean nact %.1f"
                  % (buf[8] / n, buf[12] / max(buf[8], 1), buf[9] / n, buf[13] / n, buf[10] / n,
                     buf[11] / max(buf[10], 1), buf[14] / calls, buf[15] / calls))
    elif what == "config5":
        import numpy as np
        from paper_2504_15303_b200 import workloads as wl
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
        q = int(sys.argv[3]) if len(sys.argv) > 3 else 100_000
        cluster, reqs, params, _I, _O = bench.search_inputs(10_000)
        t = planner.build_tables(cluster, reqs, params, engine=eng)
        top, _nf, _ = planner.search_topk(t, n, engine=eng)
        I1, O1 = wl.trace_lengths(q, seed=0)
        off = np.arange(n + 1, dtype=np.int64) * q
        I, O = np.tile(I1, n), np.tile(O1, n)
        for _ in range(2):
            res = hs.replay_candidates(t, params, top["index"], hs.PolicyConfig(), np.arange(n), off, I, O, O,
                                       engine=eng, want_assign=False)
        assert (res.result["error"] == 0).all()
        print(f"config5 replay {n} deployments x {q}: {res.kernel_ms:.2f} ms, "
              f"{res.result['n_steps'].sum() / (n * q):.2f} steps/request")
    else:
        cluster, reqs, params, _I, _O = bench.search_inputs(10_000)
        t = planner.build_tables(cluster, reqs, params, engine=eng)
        for _ in range(2):
            total, idx, nf, ms = planner.search_best(t, engine=eng)
        print(f"search {t.space_size} candidates: {ms:.2f} ms, {t.space_size / ms * 1e3:.3g} cand/s; best {idx}")


if __name__ == "__main__":
    main()
