"""Per-request latency of the live scheduler: the native hs_sched_* engine
vs the reference's Python Scheduler (importable only where /root/reference
exists), config-4 deployment (32 instances), OS policy, steady state with
~200 requests in flight.  Usage: python tools/bench_scheduler.py [n]"""
import pathlib
import random
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2504_15303_b200 as hs  # noqa: E402
from paper_2504_15303_b200 import simulator  # noqa: E402
from paper_2504_15303_b200 import workloads as wl  # noqa: E402


def run(mod, build, n):
    prof = wl.config4()
    cluster = mod.ClusterSpec(mod.ModelSpec(**prof.model), mod.EngineOverheads(**prof.engine),
                              tuple(mod.MachineSpec(a, c, m, t) for a, c, m, t in prof.machines),
                              mod.WorkloadLimits(**prof.limits))
    params = {k: mod.LatencyParams(*v) for k, v in prof.params.items()}
    handles = build(cluster, mod.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES}), params)
    sch = mod.Scheduler(handles, cluster.model, mod.PolicyConfig())
    rng = random.Random(1)
    reqs = [mod.Request(f"r{i}", rng.randint(50, 800), 150, rng.randint(50, 400)) for i in range(n)]
    t0 = time.perf_counter()
    for i, r in enumerate(reqs):
        sch.choose(r)
        if i >= 200:
            sch.complete(reqs[i - 200].id)
    return (time.perf_counter() - t0) / n * 1e6


n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
print(f"native: {run(hs, simulator.build_instances, n):.2f} us per choose+complete (32 instances)")
try:
    sys.path.insert(0, "/root/reference/pkg/src")
    import hetserve as ref
    print(f"reference: {run(ref, ref.build_instances, min(n, 3000)):.2f} us per choose+complete")
except ImportError:
    print("reference not importable here")
