"""Shared builders: golden-fixture descriptions -> engine objects / C structs."""

from __future__ import annotations

import json
import math
import pathlib
import random

import numpy as np

import paper_2504_15303_b200 as hs
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import workloads as wl
from paper_2504_15303_b200.simulator import engine_instances

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def load(name: str):
    return json.loads((GOLDEN / name).read_text())


def fx(h: str) -> float:
    return float.fromhex(h)


def cluster_from(desc) -> hs.ClusterSpec:
    eng = desc["engine"]
    return hs.ClusterSpec(
        model=hs.ModelSpec(**desc["model"]),
        engine=hs.EngineOverheads(fx(eng["mem_utilization_fraction"]), eng["static_overhead_bytes"]),
        machines=tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in desc["machines"]),
        limits=hs.WorkloadLimits(**desc["limits"]),
    )


def params_from(desc) -> dict:
    return {(n, t): hs.LatencyParams(*(fx(x) for x in v)) for n, t, v in desc["params"]}


def search_trace(case):
    """Rebuild the trace a search fixture was generated on (make_golden.py)."""
    name = case["name"]
    if name == "planner_search_setup":
        rng = random.Random(0)
        I = [rng.randint(8, 64) for _ in range(40)]
        O = [rng.randint(8, 64) for _ in range(40)]
    elif name in ("planner_product_4x3", "ties_identical_machines", "mixed_failures", "zero_division",
                  "duplicate_names", "negative_params"):
        rng = random.Random(4)
        I = [rng.randint(8, 64) for _ in range(30)]
        O = [rng.randint(8, 64) for _ in range(30)]
        if name == "mixed_failures":
            I[7] = 40_000_000
        if name == "zero_division":
            I, O = I[:5], O[:5]
    else:
        I, O = wl.trace_lengths(case["trace"]["q"], seed=case["trace"]["seed"])
        I, O = I.tolist(), O.tolist()
    return [hs.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(len(I))]


def replay_trace(case):
    kind = case["trace"].get("kind")
    q = case["q"]
    if kind == "randint64":
        rng = random.Random(21)
        I = np.array([rng.randint(1, 64) for _ in range(300)], np.int64)
        O = np.array([rng.randint(1, 64) for _ in range(300)], np.int64)
    elif kind == "criterion5":
        rng5 = np.random.default_rng(0)
        I = np.clip(np.round(rng5.lognormal(math.log(200) - 0.405, 0.9, 4000)), 1, 1024).astype(np.int64)
        O = np.clip(np.round(rng5.lognormal(math.log(150) - 0.08, 0.4, 4000)), 1, 1024).astype(np.int64)
    elif kind == "crit3":
        rng3 = random.Random(1000)
        I = np.array([rng3.randint(1, 64) for _ in range(200)], np.int64)
        O = np.array([rng3.randint(1, 64) for _ in range(200)], np.int64)
    elif kind == "fixed":
        if case["name"] == "err_oversized":
            I = np.array([400, 5, 6]); O = np.array([400, 5, 6])
        elif case["name"] == "static_err_oversized":
            I = np.array([5, 400, 6]); O = np.array([5, 400, 6])
        else:
            I = np.full(50, 60); O = np.full(50, 60)
            if case["name"] == "err_nonpositive_cost":
                I, O = I[:5], O[:5]
    else:
        I, O = wl.trace_lengths(q, seed=case["trace"]["seed"])
    assert len(I) == q, (case["name"], len(I), q)
    return [hs.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q)]


def scenario_from(case, policy_name: str) -> hs.Scenario:
    cluster = cluster_from(case["profile"])
    params = params_from(case["profile"])
    pred = case["predictor"]
    pc = hs.PredictorConfig(mode=pred["mode"], mean=pred.get("mean"), stddev=pred.get("stddev"),
                            seed=pred.get("seed"))
    wrr = tuple(case["wrr"]) if case.get("wrr") else None
    policy = hs.PolicyConfig(policy=policy_name, theta=fx(case["theta"]), wrr_weights=wrr, predictor=pc)
    rate = math.inf if case["rate"] == "inf" else fx(case["rate"])
    return hs.Scenario(cluster=cluster, config=hs.deployment_for(cluster.machines, case["degrees"]),
                       trace=tuple(replay_trace(case)), arrival_rate=rate, policy=policy,
                       mode=case.get("mode", "continuous"), seed=case["seed"], params=params)


# ----------------------------------------------------------- C-struct inputs
def search_structs(cluster, params_by):
    """(model, engine, limits, machines, params, present) for hs_search_tables
    / the oracle, with the engine's spec_index convention."""
    M = len(cluster.machines)
    first = {}
    for i, m in enumerate(cluster.machines):
        first.setdefault(m.name, i)
    machines = (nat.hs_machine * M)()
    params = np.zeros((M, nat.HS_MAX_DEGREES, 8))
    present = np.zeros((M, nat.HS_MAX_DEGREES), np.uint8)
    for i, m in enumerate(cluster.machines):
        spec = cluster.machines[first[m.name]]
        machines[i].accelerator_count = m.accelerator_count
        machines[i].accelerator_mem_bytes = spec.accelerator_mem_bytes
        machines[i].spec_index = first[m.name]
        machines[i].fixed_degree = 0
        for d, t in enumerate(hs.enumerate_tp_degrees(m)):
            p = params_by.get((m.name, t))
            if p is not None:
                params[i, d] = p.as_tuple()
                present[i, d] = 1
    mdl = cluster.model
    return (nat.hs_model(mdl.layers, mdl.hidden_dim, mdl.param_count, mdl.bytes_per_param),
            nat.hs_engine(float(cluster.engine.mem_utilization_fraction), cluster.engine.static_overhead_bytes),
            nat.hs_limits(cluster.limits.max_input_len, cluster.limits.max_output_len), machines, params, present)


def replay_structs(scenario):
    """(instances, policy, I, O, P, arrival-or-None) for hs_replay / oracle."""
    static = scenario.mode == "static"
    from paper_2504_15303_b200.simulator import _policy_struct, _predictor, arrival_times, build_instances
    handles = build_instances(scenario.cluster, scenario.config, scenario.params)
    per_token = hs.kv_bytes_per_token(scenario.cluster.model)
    tr = scenario.trace
    I = np.array([r.input_len for r in tr], np.int32)
    O = np.array([r.output_len for r in tr], np.int32)
    P = _predictor(scenario).predict_lengths(O.astype(np.int64)).astype(np.int32)
    T = None if math.isinf(scenario.arrival_rate) else arrival_times(len(tr), scenario.arrival_rate, scenario.seed)
    return (engine_instances(handles, scenario.policy),
            _policy_struct(scenario.policy, len(handles), per_token, 1 if static else 0), handles, I, O, P, T)


ENTRY_STATUS = {"ok": nat.ENTRY_OK, "infeasible_config": nat.ENTRY_INFEASIBLE_CONFIG,
                "infeasible_request": nat.ENTRY_INFEASIBLE_REQUEST, "zero_division": nat.ENTRY_ZERO_DIVISION}


def check_table(case, table, nd, requests):
    """Compare an engine/oracle table against the reference's per-entry rows."""
    cluster = cluster_from(case["profile"])
    rows = iter(case["table"])
    for i, m in enumerate(cluster.machines):
        degs = hs.enumerate_tp_degrees(m)
        assert int(nd[i]) == len(degs)
        for d, t in enumerate(degs):
            row = next(rows)
            assert row["machine"] == i and row["t"] == t
            e = table[i, d]
            st = int(e["status"])
            if row["status"] == "ok":
                assert st == nat.ENTRY_OK, (case["name"], i, t, st)
                assert float(e["contribution"]).hex() == row["contribution"], (case["name"], i, t)
                assert float(e["rate"]).hex() == row["rate"]
                assert float(e["budget"]).hex() == row["budget"]
                assert float(e["slack"]).hex() == row["slack"]
                assert int(e["instance_count"]) == row["instance_count"]
            elif row["status"] == "spec":
                assert st in (nat.ENTRY_MISSING_PARAMS, nat.ENTRY_BAD_DEGREE), (case["name"], i, t, st)
            else:
                assert st == ENTRY_STATUS[row["status"]], (case["name"], i, t, st, row["status"])
            if row["status"] != "ok":
                from paper_2504_15303_b200.planner import _entry_exception
                msg = str(_entry_exception(cluster, requests, m.name, t, e))
                assert msg == row["msg"], (msg, row["msg"])


def metrics_digest(assign, depart, metrics_row, handles, trace, arrival, policy, static=False):
    """The same digest make_golden.metrics_desc computes from a SimMetrics."""
    import hashlib
    H = lambda x: float(x).hex()  # noqa: E731
    completion = metrics_row["completion_time"].tolist()
    tok = metrics_row["token_count"].tolist()
    makespan = max(completion)
    if static:
        order = np.lexsort((np.arange(len(trace)), assign.astype(np.int64)))
    else:
        order = np.lexsort((np.arange(len(trace)), assign.astype(np.int64), depart))
    ids = [r.id for r in trace]
    arr = [0.0] * len(trace) if arrival is None else arrival.tolist()
    times = [(ids[k], arr[k], float(depart[k])) for k in order.tolist()]
    return {
        "policy": policy,
        "makespan": H(makespan),
        "throughput": H(sum(tok) / makespan if makespan > 0 else math.inf),
        "spread": H(max(completion) - min(completion)),
        "per_instance": [[h.id, H(metrics_row["completion_time"][i]), int(metrics_row["request_count"][i]),
                          int(metrics_row["token_count"][i]), H(metrics_row["peak_kv_usage"][i])]
                         for i, h in enumerate(handles)],
        "residual_loads": [H(x) for x in metrics_row["residual_load"].tolist()],
        "assign_sha": hashlib.sha256(bytes(assign.tolist())).hexdigest(),
        "assign_head": assign[:64].tolist(),
        "times_sha": hashlib.sha256(",".join(f"{rid}:{H(d)}" for rid, _a, d in times).encode()).hexdigest(),
        "depart_sha": hashlib.sha256(",".join(H(d) for d in depart.tolist()).encode()).hexdigest(),
        "times_head": [[rid, H(a), H(d)] for rid, a, d in times[:16]],
    }


def sim_digest(m):
    """Digest of a SimMetrics object (same fields as make_golden.metrics_desc)."""
    import hashlib
    H = lambda x: float(x).hex()  # noqa: E731
    return {
        "policy": m.policy,
        "makespan": H(m.makespan),
        "throughput": H(m.system_throughput),
        "spread": H(m.completion_time_spread),
        "per_instance": [[x.id, H(x.completion_time), x.request_count, x.token_count, H(x.peak_kv_usage)]
                         for x in m.per_instance],
        "residual_loads": [H(x) for x in m.residual_loads],
        "assign_sha": hashlib.sha256(bytes(m.assignments)).hexdigest(),
        "assign_head": list(m.assignments[:64]),
        "times_sha": hashlib.sha256(",".join(f"{rid}:{H(d)}" for rid, _a, d in m.request_times).encode()).hexdigest(),
        "depart_sha": hashlib.sha256(",".join(
            H(d) for _k, d in sorted((int(rid[1:]), d) for rid, _a, d in m.request_times)).encode()).hexdigest(),
        "times_head": [[rid, H(a), H(d)] for rid, a, d in m.request_times[:16]],
    }
