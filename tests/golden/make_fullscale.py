"""Generate tests/golden/fullscale_cases.json: the REFERENCE's own SimMetrics
at the bench's full trace size (100,000 requests) on the config-4 deployment.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_fullscale.py [workers]

The small fixtures of make_golden.py stop at 10k requests; these pin the
1e5-request behaviour of the engine to the reference itself, not to the C
oracle.  Each case is one bench trace (gen-trace lengths seeded t, arrivals
seeded 42 + t, bench.py replay_inputs) under one policy / predictor / mode;
the reference runs unmodified (hetserve.simulator.run_continuous /
run_static, simulator.py:199-363), one process per case.  Outputs are
make_golden.metrics_desc digests (float.hex, sha256 of assignments and
request times), so the fixture stays small.
"""

from __future__ import annotations

import json
import math
import pathlib
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

OUT = pathlib.Path(__file__).resolve().parent / "fullscale_cases.json"
Q = 100_000
RATE = 140.0  # bench.py's config-4 arrival rate

# (trace index t, policy, rate, mode, predictor) -- t indexes the bench's
# 4,096 config-4 traces; 0 and 4095 are the first and last of the bench step
CASES = [
    (0, "OS", RATE, "continuous", None),
    (4095, "OS", RATE, "continuous", None),
    (2, "RR", RATE, "continuous", None),
    (3, "MB", RATE, "continuous", None),
    (6, "WRR", RATE, "continuous", None),
    (9, "OS", RATE, "continuous", {"mode": "normal", "mean": 150.0, "stddev": 60.0, "seed": 9}),
    (7, "OS", math.inf, "static", None),
    (8, "OS", math.inf, "continuous", None),
]


def case_scenario(H, HS, wl, case):
    """The scenario of one case, built from module H (reference or drop-in)."""
    t, pol, rate, mode, pred = case
    prof = wl.config4()
    cluster = H.ClusterSpec(model=H.ModelSpec(**prof.model), engine=H.EngineOverheads(**prof.engine),
                            machines=tuple(H.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                            limits=H.WorkloadLimits(**prof.limits))
    params = {k: H.LatencyParams(*v) for k, v in prof.params.items()}
    config = H.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    I, O = wl.trace_lengths(Q, seed=t)
    trace = tuple(H.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(Q))
    n_inst = sum(p.instance_count for p in config.per_machine)
    wrr = tuple(float(1 + (k % 3)) for k in range(n_inst)) if pol == "WRR" else None
    predictor = H.PredictorConfig(**pred) if pred else H.PredictorConfig()
    policy = H.PolicyConfig(policy=pol, wrr_weights=wrr, predictor=predictor)
    return HS.Scenario(cluster=cluster, config=config, trace=trace, arrival_rate=rate, policy=policy, mode=mode,
                       seed=42 + t, params=params)


def _run(case):
    sys.path.insert(0, "/root/reference/pkg/src")
    import hetserve as H
    import hetserve.simulator as HS
    from make_golden import metrics_desc
    from paper_2504_15303_b200 import workloads as wl

    sc = case_scenario(H, HS, wl, case)
    t0 = time.perf_counter()
    m = HS.run_static(sc) if sc.mode == "static" else HS.run_continuous(sc)
    dt = time.perf_counter() - t0
    t, pol, rate, mode, pred = case
    return {"trace": t, "policy": pol, "rate": "inf" if math.isinf(rate) else rate, "mode": mode,
            "predictor": pred, "q": Q, "ref_seconds": round(dt, 1), "metrics": metrics_desc(m)}


# BASELINE config 5: deployments of the config-3 space's top-1024 (by the
# search over bench.py's 10k-request search trace), each replayed by the
# reference on the 1e5-request trace (lengths seeded 0) at rate = inf with OS
CONFIG5_RANKS = (0, 1, 511, 1023)


def config5_degrees(index: int, machines, enumerate_tp_degrees) -> dict:
    """Mixed-radix candidate index -> {machine: degree} (planner.py:213-226:
    itertools.product order, the last machine varies fastest)."""
    degs = [enumerate_tp_degrees(m) for m in machines]
    dig = [0] * len(degs)
    for i in range(len(degs) - 1, -1, -1):
        index, dig[i] = divmod(index, len(degs[i]))
    return {m.name: degs[i][d] for i, (m, d) in enumerate(zip(machines, dig))}


def config5_top():
    """(rank, index) of the chosen top-1024 positions plus the widest
    deployment among the 1024, from the C oracle's top-k (pinned to the
    reference's rankings by tests/test_oracle_golden.py)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import bench
    import helpers
    from oracle import hs_oracle as orc
    from paper_2504_15303_b200 import domain

    cluster, _reqs, params, I, O = bench.search_inputs(10_000)
    table, nd = orc.tables(*helpers.search_structs(cluster, params), I, O)
    top, _nf = orc.topk(table, nd, 1024)
    width = []
    for idx in top["index"].tolist():
        d = config5_degrees(int(idx), cluster.machines, domain.enumerate_tp_degrees)
        width.append(sum(m.accelerator_count // d[m.name] for m in cluster.machines))
    ranks = sorted(set(CONFIG5_RANKS) | {max(range(len(width)), key=lambda r: (width[r], -r))})
    return [(r, int(top["index"][r])) for r in ranks]


def config5_scenario(H, HS, wl, degrees):
    prof = wl.config3()
    cluster = H.ClusterSpec(model=H.ModelSpec(**prof.model), engine=H.EngineOverheads(**prof.engine),
                            machines=tuple(H.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                            limits=H.WorkloadLimits(**prof.limits))
    params = {k: H.LatencyParams(*v) for k, v in prof.params.items()}
    config = H.deployment_for(cluster.machines, degrees)
    I, O = wl.trace_lengths(Q, seed=0)
    trace = tuple(H.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(Q))
    return HS.Scenario(cluster=cluster, config=config, trace=trace, arrival_rate=math.inf,
                       policy=H.PolicyConfig(), mode="continuous", seed=0, params=params)


def _run5(item):
    rank, index = item
    sys.path.insert(0, "/root/reference/pkg/src")
    import hetserve as H
    import hetserve.simulator as HS
    from make_golden import metrics_desc
    from paper_2504_15303_b200 import workloads as wl

    prof = wl.config3()
    machines = tuple(H.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines)
    degrees = config5_degrees(index, machines, H.enumerate_tp_degrees)
    sc = config5_scenario(H, HS, wl, degrees)
    t0 = time.perf_counter()
    m = HS.run_continuous(sc)
    return {"rank": rank, "index": index, "degrees": degrees, "instances": len(m.per_instance), "q": Q,
            "ref_seconds": round(time.perf_counter() - t0, 1), "metrics": metrics_desc(m)}


def main():
    workers = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 8
    only5 = "--config5" in sys.argv
    with ProcessPoolExecutor(max_workers=workers) as ex:
        if only5:
            out = json.loads(OUT.read_text())["cases"]
        else:
            out = list(ex.map(_run, CASES))
        out5 = list(ex.map(_run5, config5_top()))
    OUT.write_text(json.dumps({"generator": "tests/golden/make_fullscale.py", "cases": out, "config5": out5},
                              indent=1) + "\n")
    print(OUT, [c["ref_seconds"] for c in out], [(c["rank"], c["instances"], c["ref_seconds"]) for c in out5])


if __name__ == "__main__":
    main()
