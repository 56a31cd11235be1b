"""Host-side wall time of each phase of bench.py's step (build_tables,
search_best, replay_device), to see where non-kernel time goes.
Usage: python tools/step_host_profile.py [steps]"""
import gc
import pathlib
import sys
import time


ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2504_15303_b200 as hs  # noqa: E402
from paper_2504_15303_b200 import _native as nat, planner, streams  # noqa: E402
from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eng = nat.engine_for(0)
cluster, reqs, params, _sI, _sO = bench.search_inputs(10_000)
rc, config, rparams = bench.replay_deployment()
handles = build_instances(rc, config, rparams)
pol = hs.PolicyConfig()
inst = engine_instances(handles, pol)
ps = _policy_struct(pol, len(handles), hs.kv_bytes_per_token(rc.model))
T, q = 4096, 100_000
lens = streams.gen_trace_lengths_device(list(range(T)), q, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096,
                                        engine=eng)
arrs = streams.arrival_times_device([42 + t for t in range(T)], [q] * T, 140.0, engine=eng)
off = lens.offsets
d_off = eng.device_alloc(off.nbytes)
eng.h2d(d_off, off)
d_a = eng.device_alloc(T * q)
d_m = eng.device_alloc(T * 32 * nat.METRICS_DTYPE.itemsize)
d_r = eng.device_alloc(T * nat.RESULT_DTYPE.itemsize)
for s in range(steps):
    t0 = time.perf_counter()
    tab = planner.build_tables(cluster, reqs, params, engine=eng)
    t1 = time.perf_counter()
    planner.search_best(tab, engine=eng)
    k2 = eng.last_kernel_ms
    t2 = time.perf_counter()
    eng.replay_device(inst, ps, T, d_off, lens.ptrs[0], lens.ptrs[1], lens.ptrs[1], arrs.ptrs[0], d_a, d_m, d_r)
    k3 = eng.last_kernel_ms
    t3 = time.perf_counter()
    print(f"step {s}: build_tables {1e3 * (t1 - t0):.2f} ms, search {1e3 * (t2 - t1):.2f} ms (kernel {k2:.2f}), "
          f"replay {1e3 * (t3 - t2):.2f} ms (kernels {k3:.2f}), gc counts {gc.get_count()}")
