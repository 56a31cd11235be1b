"""Batched replay vs the C oracle (run by tests/test_gpu_replay_layouts.py);
prints OK or raises."""

import math
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import helpers as H  # noqa: E402
import paper_2504_15303_b200 as hs  # noqa: E402
from oracle import hs_oracle as orc  # noqa: E402
from paper_2504_15303_b200 import _native as nat  # noqa: E402
from paper_2504_15303_b200 import workloads as wl  # noqa: E402
from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances  # noqa: E402


def main(n_traces: int, qmax: int, n_inst: int):
    prof = wl.config4()
    cluster = H.cluster_from({"model": prof.model, "engine": {"mem_utilization_fraction": (0.9).hex(),
                              "static_overhead_bytes": prof.engine["static_overhead_bytes"]},
                              "limits": prof.limits, "machines": [list(m) for m in prof.machines], "params": []})
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    # n_inst instances: the first machines at t = 1, the rest at the largest degree
    degs = {a: 1 for a in wl.CONFIG4_TYPES}
    if n_inst < 32:
        for a in wl.CONFIG4_TYPES[n_inst // 8:]:
            degs[a] = 8
    config = hs.deployment_for(cluster.machines, degs)
    N = len(build_instances(cluster, config, params))
    rng = np.random.default_rng(7 + n_inst)
    lens = [int(x) for x in rng.integers(0, qmax, n_traces)]
    lens[3] = 0
    Is, Os, Ts = [], [], []
    for t, q in enumerate(lens):
        I, O = wl.trace_lengths(q, seed=2000 + t)
        rate = [8.0, 140.0, 1500.0, math.inf, 60.0][t % 5]
        Is.append(I)
        Os.append(O)
        Ts.append(np.zeros(q) if math.isinf(rate) else wl.arrivals(q, rate, seed=t))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I, O, T = np.concatenate(Is), np.concatenate(Os), np.concatenate(Ts)
    eng = nat.engine_for(0)
    for policy in ("OS", "RR", "WRR", "SI", "MB"):
        wrr = tuple(float(x) for x in rng.integers(1, 5, N)) if policy == "WRR" else None
        pol = hs.PolicyConfig(policy=policy, theta=2.0, wrr_weights=wrr)
        for want_depart in (True, False):
            res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, arrival=T, want_assign=True,
                                   want_depart=want_depart, engine=eng)
            handles = build_instances(cluster, config, params)
            a, d, m, r = orc.replay(engine_instances(handles, pol),
                                    _policy_struct(pol, N, hs.kv_bytes_per_token(cluster.model)), off, I, O, O, T,
                                    nthreads=8)
            assert (res.result["error"] == 0).all() and (r["error"] == 0).all(), policy
            assert np.array_equal(res.result["n_steps"], r["n_steps"]), (policy, "n_steps")
            assert np.array_equal(res.assign, a), policy
            if want_depart:
                assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64)), policy
            for f in ("completion_time", "peak_kv_usage", "residual_load"):
                assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), (policy, f)
            for f in ("request_count", "token_count"):
                assert np.array_equal(res.metrics[f], m[f]), (policy, f)
    print("OK", N, sum(lens))


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]))
