"""Config-5 end-to-end anatomy on the GPU box: build_tables, search_topk and
replay_candidates wall times, the C call inside the last and its kernel time.

    python tools/c5_host_profile.py
"""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path.cwd()))
import numpy as np
import bench
import paper_2504_15303_b200 as hs
from paper_2504_15303_b200 import _native as nat, planner, simulator
from paper_2504_15303_b200 import workloads as wl
eng = nat.engine_for(0)
cluster, reqs, params, _I, _O = bench.search_inputs(10_000)
q = 100_000; n = 1024
I1, O1 = wl.trace_lengths(q, seed=0)
ti = eng.host_array((n * q,), np.int32); to = eng.host_array((n * q,), np.int32)
ti[:] = np.tile(I1, n); to[:] = np.tile(O1, n)
ta = eng.host_array((n * q,), np.uint8)
off = np.arange(n + 1, dtype=np.int64) * q
orig = eng.replay_deployments
acc = {}
def timed(*a, **k):
    t0 = time.perf_counter(); r = orig(*a, **k); acc['c_call'] = (time.perf_counter() - t0) * 1e3; return r
eng.replay_deployments = timed
for it in range(3):
    t0 = time.perf_counter(); t = planner.build_tables(cluster, reqs, params, engine=eng); t1 = time.perf_counter()
    top, nf, ms = planner.search_topk(t, 1024, engine=eng); t2 = time.perf_counter()
    res = hs.replay_candidates(t, params, top["index"], hs.PolicyConfig(), np.arange(n), off, ti, to, to, engine=eng, want_assign=True, assign_out=ta); t3 = time.perf_counter()
    print(f"build_tables {1e3*(t1-t0):.1f} ms  search_topk {1e3*(t2-t1):.1f} ms  replay_candidates {1e3*(t3-t2):.1f} ms (C call {acc['c_call']:.1f}, kernel {res.kernel_ms:.1f})")
