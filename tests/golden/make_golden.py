"""Generate tests/golden/*.json by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Every fixture records outputs of the unmodified reference (hetserve) on
inputs described by paper_2504_15303_b200.workloads (seeded numpy), with
floats as float.hex so comparisons are bit-exact.  The oracle tests
(tests/test_oracle_golden.py) pin oracle/hs_oracle.c to these fixtures and
the GPU tests pin the CUDA engine to them.
"""

from __future__ import annotations

import hashlib
import json
import math
import pathlib
import random
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import hetserve as hs  # noqa: E402  (the reference)

from paper_2504_15303_b200 import workloads as wl  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def H(x: float) -> str:
    return float(x).hex()


# ----------------------------------------------------------------- builders
def ref_cluster(p: wl.ClusterProfile) -> hs.ClusterSpec:
    return hs.ClusterSpec(
        model=hs.ModelSpec(**p.model),
        engine=hs.EngineOverheads(**p.engine),
        machines=tuple(
            hs.MachineSpec(name=n, accelerator_count=c, accelerator_mem_bytes=m, accelerator_type=a)
            for n, c, m, a in p.machines
        ),
        limits=hs.WorkloadLimits(**p.limits),
    )


def ref_params(p: wl.ClusterProfile) -> dict:
    return {k: hs.LatencyParams(*(float(x) for x in v)) for k, v in p.params.items()}


def ref_trace(I, O, P=None) -> list:
    P = O if P is None else P
    return [hs.Request(f"r{k}", int(I[k]), int(O[k]), int(P[k])) for k in range(len(I))]


def profile_desc(p: wl.ClusterProfile) -> dict:
    return {
        "model": p.model,
        "engine": {"mem_utilization_fraction": H(p.engine["mem_utilization_fraction"]),
                   "static_overhead_bytes": p.engine["static_overhead_bytes"]},
        "limits": p.limits,
        "machines": [list(m) for m in p.machines],
        "params": [[k[0], k[1], [H(x) for x in v]] for k, v in p.params.items()],
    }


# ------------------------------------------------------------------ search
def table_entries(cluster, trace, params) -> list:
    """Per (machine, degree): the reference's per-machine body of
    estimate_system_throughput (planner.py:152-179), run on a one-machine
    config so the exception it raises (if any) is the entry's status."""
    rows = []
    for i, m in enumerate(cluster.machines):
        for t in hs.enumerate_tp_degrees(m):
            placement = hs.MachinePlacement(machine=m.name, tp_degree=t, instance_count=m.accelerator_count // t)
            cfg = hs.DeploymentConfig(per_machine=(placement,))
            row = {"machine": i, "t": t}
            try:
                est = hs.estimate_system_throughput(cluster, cfg, trace, params)
                me = est.per_machine[0]
                row.update(status="ok", contribution=H(me.machine_tokens_per_sec),
                           rate=H(me.instance_tokens_per_sec), budget=H(me.budget_bytes),
                           slack=H(me.slack_bytes), instance_count=me.instance_count)
            except hs.InfeasibleConfigError as exc:
                row.update(status="infeasible_config", slack=H(exc.slack_bytes), msg=str(exc))
            except hs.InfeasibleRequestError as exc:
                row.update(status="infeasible_request", request_id=exc.request_id, msg=str(exc))
            except hs.SpecError as exc:
                row.update(status="spec", msg=str(exc))
            except ZeroDivisionError as exc:
                row.update(status="zero_division", msg=str(exc))
            rows.append(row)
    return rows


def search_case(name, profile, I, O, full=True, extra=None) -> dict:
    cluster, params = ref_cluster(profile), ref_params(profile)
    trace = ref_trace(I, O)
    case = {"kind": "search", "name": name, "profile": profile_desc(profile), "q": len(I),
            "trace": extra or {}}
    case["table"] = table_entries(cluster, trace, params)
    if full:
        t0 = time.time()
        try:
            out = hs.search_optimal_config(cluster, trace, params)
            case["ranked"] = [
                {"degrees": [p.tp_degree for p in e.config.per_machine], "total": H(e.system_tokens_per_sec),
                 "per_machine": [[H(m.instance_tokens_per_sec), H(m.machine_tokens_per_sec), H(m.budget_bytes),
                                  H(m.slack_bytes), m.instance_count] for m in e.per_machine]}
                for e in out.ranked
            ]
            case["infeasible"] = [[[p.tp_degree for p in c.per_machine], r] for c, r in out.infeasible]
            case["visited"] = out.candidates_visited
        except ZeroDivisionError as exc:
            case["error"] = {"type": "ZeroDivisionError", "msg": str(exc)}
        case["ref_seconds"] = time.time() - t0
    return case


def sampled_candidates(name, profile, I, O, n, seed) -> dict:
    """Large space: the literal reference estimate on sampled indices."""
    cluster, params = ref_cluster(profile), ref_params(profile)
    trace = ref_trace(I, O)
    dl = profile.degree_lists()
    size = profile.space_size()
    rng = random.Random(seed)
    rows = []
    t0 = time.time()
    ok = {}
    for row in table_entries(cluster, trace, params):
        ok.setdefault(row["machine"], []).append(row["status"] == "ok")
    for k in range(n):
        if k % 2 == 0:
            idx = rng.randrange(size)
        else:  # a feasible candidate: every digit drawn from its machine's OK degrees
            idx = 0
            for i, d in enumerate(dl):
                choices = [j for j in range(len(d)) if ok[i][j]] or list(range(len(d)))
                idx = idx * len(d) + rng.choice(choices)
        x, digits = idx, []
        for d in reversed(dl):
            digits.append(d[x % len(d)])
            x //= len(d)
        digits.reverse()
        cfg = hs.deployment_for(cluster.machines, {m.name: t for m, t in zip(cluster.machines, digits)})
        try:
            est = hs.estimate_system_throughput(cluster, cfg, trace, params)
            rows.append([idx, H(est.system_tokens_per_sec), None])
        except (hs.InfeasibleConfigError, hs.InfeasibleRequestError, hs.SpecError) as exc:
            rows.append([idx, None, str(exc)])
    return {"kind": "search_sample", "name": name, "profile": profile_desc(profile), "q": len(I),
            "samples": rows, "ref_seconds_per_candidate": (time.time() - t0) / n}


# ------------------------------------------------------------------ replay
def metrics_desc(m) -> dict:
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
        "times_sha": hashlib.sha256(
            ",".join(f"{rid}:{H(d)}" for rid, _a, d in m.request_times).encode()).hexdigest(),
        "depart_sha": hashlib.sha256(",".join(
            H(d) for _k, d in sorted((int(rid[1:]), d) for rid, _a, d in m.request_times)).encode()).hexdigest(),
        "times_head": [[rid, H(a), H(d)] for rid, a, d in m.request_times[:16]],
    }


def replay_scenario(profile, degrees, trace, rate, policy, seed, mode="continuous"):
    cluster, params = ref_cluster(profile), ref_params(profile)
    cfg = hs.deployment_for(cluster.machines, degrees)
    return hs.Scenario(cluster=cluster, config=cfg, trace=tuple(trace), arrival_rate=rate, policy=policy,
                       mode=mode, seed=seed, params=params)


def replay_case(name, profile, degrees, trace_desc, I, O, rate, seed, policies, predictor=None,
                theta=2.0, wrr=None, mode="continuous") -> dict:
    trace = ref_trace(I, O)
    pred = predictor or {"mode": "oracle"}
    pc = hs.PredictorConfig(mode=pred["mode"], mean=pred.get("mean"), stddev=pred.get("stddev"),
                            seed=pred.get("seed"))
    base = hs.PolicyConfig(policy=policies[0], theta=theta, wrr_weights=wrr, predictor=pc)
    sc = replay_scenario(profile, degrees, trace, rate, base, seed, mode)
    case = {"kind": "replay", "mode": mode, "name": name, "profile": profile_desc(profile), "degrees": degrees,
            "trace": trace_desc, "q": len(I), "rate": "inf" if math.isinf(rate) else H(rate), "seed": seed,
            "predictor": pred, "theta": H(theta), "wrr": wrr, "results": []}
    t0 = time.time()
    for pol in policies:
        scp = replay_scenario(profile, degrees, trace, rate,
                              hs.PolicyConfig(policy=pol, theta=theta, wrr_weights=wrr, predictor=pc), seed, mode)
        try:
            m = hs.run_scenario(scp)
            case["results"].append(metrics_desc(m))
        except (hs.HetserveError, OverflowError) as exc:
            case["results"].append({"policy": pol, "error": type(exc).__name__, "msg": str(exc),
                                    "request_id": getattr(exc, "request_id", None)})
    case["ref_seconds"] = time.time() - t0
    del sc
    return case


# ------------------------------------------------------------------- cases
def tiny_profile(machines, model=None, engine=None, limits=None, params=None) -> wl.ClusterProfile:
    p = wl.ClusterProfile("tiny", model or dict(layers=2, hidden_dim=4, param_count=100, bytes_per_param=2),
                          engine or dict(mem_utilization_fraction=1.0, static_overhead_bytes=0),
                          limits or dict(max_input_len=64, max_output_len=64), machines)
    p.params = params or {}
    return p


def build_search_cases() -> list:
    cases = []
    # reference test_planner.py:204-212 _search_setup shape
    rng = random.Random(0)
    I = np.array([rng.randint(8, 64) for _ in range(40)], np.int32)
    O = np.array([rng.randint(8, 64) for _ in range(40)], np.int32)
    p = tiny_profile([("m0", 8, 10**9, "test")])
    p.params = {("m0", t): wl.scaled_params(wl.RANK_BASE, t**-0.7) for t in (1, 2, 4, 8)}
    cases.append(search_case("planner_search_setup", p, I, O))
    # test_planner.py:249-268 4x3 product
    rng = random.Random(4)
    I = np.array([rng.randint(8, 64) for _ in range(30)], np.int32)
    O = np.array([rng.randint(8, 64) for _ in range(30)], np.int32)
    p = tiny_profile([("m0", 8, 10**9, "test"), ("m1", 4, 10**9, "test")])
    for name, cnt in (("m0", 8), ("m1", 4)):
        for t in wl.enumerate_degrees(cnt):
            p.params[(name, t)] = wl.scaled_params(wl.RANK_BASE, t**-0.6 * (1.5 if name == "m1" else 1.0))
    cases.append(search_case("planner_product_4x3", p, I, O))
    # identical machines: exact ties, lowest-index winner
    p = tiny_profile([("a", 4, 10**9, "x"), ("b", 4, 10**9, "x"), ("c", 4, 10**9, "x")])
    for name in "abc":
        for t in (1, 2, 4):
            p.params[(name, t)] = wl.scaled_params(wl.RANK_BASE, t**-0.5)
    cases.append(search_case("ties_identical_machines", p, I, O))
    # mixed failures: missing params, infeasible config, oversized request
    tight = dict(layers=2, hidden_dim=4, param_count=3 * 10**9 // 2, bytes_per_param=2)
    p = tiny_profile([("m0", 8, 10**9, "x"), ("m1", 2, 4 * 10**9, "x"), ("m2", 4, 2 * 10**9, "x")], model=tight)
    for t in (1, 2, 4, 8):
        if t != 4:
            p.params[("m0", t)] = wl.scaled_params(wl.RANK_BASE, t**-0.6)
    for t in (1, 2):
        p.params[("m1", t)] = wl.scaled_params(wl.RANK_BASE, 2.0 * t**-0.6)
    for t in (1, 2, 4):
        p.params[("m2", t)] = wl.scaled_params(wl.RANK_BASE, 0.5 * t**-0.6)
    I2 = I.copy(); O2 = O.copy()
    I2[7] = 40_000_000  # needs 32*(4e7+O) bytes: only wide instances hold it
    cases.append(search_case("mixed_failures", p, I2, O2))
    # zero time -> ZeroDivisionError aborts the search (planner.py:118)
    p = tiny_profile([("m0", 2, 10**9, "x"), ("m1", 2, 10**9, "x")])
    p.params = {("m0", 1): (0,) * 3 + (1.0,) + (0,) * 4, ("m0", 2): (0.0,) * 8,
                ("m1", 1): (0,) * 3 + (1.0,) + (0,) * 4, ("m1", 2): (0,) * 3 + (2.0,) + (0,) * 4}
    cases.append(search_case("zero_division", p, I[:5], O[:5]))
    # duplicate machine names: cluster.machine(name) resolves to the first
    p = tiny_profile([("dup", 4, 10**9, "x"), ("dup", 8, 3 * 10**9, "x")])
    for t in (1, 2, 4, 8):
        p.params[("dup", t)] = wl.scaled_params(wl.RANK_BASE, t**-0.6)
    cases.append(search_case("duplicate_names", p, I, O))
    # negative coefficients (fitted params may be negative): negative rates
    p = tiny_profile([("m0", 4, 10**9, "x")])
    p.params = {("m0", 1): (1e-5, 1e-4, 1e-5, -5.0, 1e-6, 1e-4, 1e-6, 1e-4),
                ("m0", 2): (1e-5, 1e-4, 1e-5, 1e-3, 1e-6, 1e-4, 1e-6, 1e-4),
                ("m0", 4): (1e-5, 1e-4, 1e-5, -1e-3, 1e-6, 1e-4, 1e-6, -1e-4)}
    cases.append(search_case("negative_params", p, I, O))
    # BASELINE config 1 and 2 (q = 10k)
    I, O = wl.trace_lengths(10_000, seed=1)
    cases.append(search_case("config1", wl.config1(), I, O, extra={"seed": 1, "q": 10_000}))
    I, O = wl.trace_lengths(10_000, seed=2)
    cases.append(search_case("config2", wl.config2(), I, O, extra={"seed": 2, "q": 10_000}))
    # config 3: table + sampled literal candidates (space is 5^16)
    I, O = wl.trace_lengths(10_000, seed=3)
    c3 = search_case("config3_table", wl.config3(), I, O, full=False, extra={"seed": 3, "q": 10_000})
    cases.append(c3)
    cases.append(sampled_candidates("config3_samples", wl.config3(), I, O, 60, seed=33))
    return cases


POSITIVE = (1e-4, 2e-3, 5e-5, 8e-3, 2e-5, 5e-4, 1e-5, 2e-4)  # test_simulator.py:34


def two_instance_profile(strong=POSITIVE, weak_scale=4.0, strong_tokens=20_000, weak_tokens=5_000, max_len=512):
    weights = 100 * 2
    p = tiny_profile([("strong", 1, 32 * strong_tokens + weights, "x"), ("weak", 1, 32 * weak_tokens + weights, "x")],
                     limits=dict(max_input_len=max_len, max_output_len=max_len))
    p.params = {("strong", 1): tuple(strong), ("weak", 1): wl.scaled_params(strong, weak_scale)}
    return p


def build_replay_cases() -> list:
    cases = []
    pols = ["OS", "RR", "WRR", "SI", "MB"]
    rng = random.Random(21)
    n = 300
    I = np.array([rng.randint(1, 64) for _ in range(n)], np.int32)
    O = np.array([rng.randint(1, 64) for _ in range(n)], np.int32)
    p = two_instance_profile()
    for rate, seed in ((math.inf, 0), (8.0, 4), (40.0, 13)):
        cases.append(replay_case(f"two_instance_rate{rate}", p, {"strong": 1, "weak": 1}, {"kind": "randint64"},
                                 I, O, rate, seed, pols, wrr=(4.0, 1.0)))
    # normal predictor (test_simulator.py:603-617 shape)
    cases.append(replay_case("two_instance_normal_pred", p, {"strong": 1, "weak": 1}, {"kind": "randint64"},
                             I, O, 12.0, 77, ["OS", "RR", "MB"],
                             predictor={"mode": "normal", "mean": 30, "stddev": 10, "seed": None}))
    # criterion-5 analogue: 4:1 pair, normal(150, 60, seed 7) predictor
    rng5 = np.random.default_rng(0)
    n5 = 4000
    I5 = np.clip(np.round(rng5.lognormal(math.log(200) - 0.405, 0.9, n5)), 1, 1024).astype(np.int32)
    O5 = np.clip(np.round(rng5.lognormal(math.log(150) - 0.08, 0.4, n5)), 1, 1024).astype(np.int32)
    p5 = two_instance_profile(strong=wl.RANK_BASE, max_len=1024)
    for rate in (3.7, 11.0, math.inf):
        cases.append(replay_case(f"criterion5_rate{rate}", p5, {"strong": 1, "weak": 1}, {"kind": "criterion5"},
                                 I5, O5, rate, 42, pols, predictor={"mode": "normal", "mean": 150, "stddev": 60,
                                                                    "seed": 7}, wrr=(4.0, 1.0)))
    # config 1 / 2 replays on their search winners (10k requests)
    I, O = wl.trace_lengths(10_000, seed=1)
    cases.append(replay_case("config1_replay", wl.config1(), {"v100": 1, "a800": 1}, {"seed": 1}, I, O, 60.0, 42,
                             ["OS", "RR"]))
    I, O = wl.trace_lengths(10_000, seed=2)
    cases.append(replay_case("config2_replay", wl.config2(), {"v100": 2, "a800": 1, "h100": 1}, {"seed": 2},
                             I, O, 150.0, 42, ["OS", "RR"]))
    # config 4 shape: 32 instances, 3k requests near capacity and overloaded
    for tseed, rate in ((0, wl.CONFIG4_RATE), (1, math.inf)):
        I, O = wl.trace_lengths(3000, seed=tseed)
        cases.append(replay_case(f"config4_small_seed{tseed}", wl.config4(),
                                 {a: 1 for a in wl.CONFIG4_TYPES}, {"seed": tseed}, I, O, rate, 42 + tseed,
                                 ["OS", "MB", "RR"]))
    # errors: oversized request, exp overflow, non-positive cost
    big = np.array([400, 5, 6], np.int32)
    pb = tiny_profile([("m0", 1, 32 * 100 + 200, "x")], limits=dict(max_input_len=32, max_output_len=32))
    pb.params = {("m0", 1): POSITIVE}
    cases.append(replay_case("err_oversized", pb, {"m0": 1}, {"kind": "fixed"}, big, np.array([400, 5, 6], np.int32),
                             math.inf, 0, ["OS"]))
    I, O = np.full(50, 60, np.int32), np.full(50, 60, np.int32)
    po = tiny_profile([("m0", 1, 32 * 1000 + 200, "x"), ("m1", 1, 32 * 900 + 200, "x")],
                      limits=dict(max_input_len=64, max_output_len=64))
    po.params = {("m0", 1): POSITIVE, ("m1", 1): POSITIVE}
    cases.append(replay_case("err_exp_overflow", po, {"m0": 1, "m1": 1}, {"kind": "fixed"}, I, O, math.inf, 0,
                             ["OS", "RR"], theta=300.0))
    pn = tiny_profile([("m0", 1, 32 * 1000 + 200, "x"), ("m1", 1, 32 * 1000 + 200, "x")],
                      limits=dict(max_input_len=64, max_output_len=64))
    pn.params = {("m0", 1): POSITIVE, ("m1", 1): (0, 0, 0, -1.0, 0, 0, 0, 0)}
    cases.append(replay_case("err_nonpositive_cost", pn, {"m0": 1, "m1": 1}, {"kind": "fixed"}, I[:5], O[:5],
                             math.inf, 0, ["OS", "RR", "SI", "MB"]))
    return cases


def build_static_cases() -> list:
    """run_static (simulator.py:206-250), the first 'next' row of SURVEY 8f."""
    cases = []
    pols = ["OS", "RR", "WRR", "SI", "MB"]
    rng = random.Random(21)
    I = np.array([rng.randint(1, 64) for _ in range(300)], np.int32)
    O = np.array([rng.randint(1, 64) for _ in range(300)], np.int32)
    cases.append(replay_case("static_two_instance", two_instance_profile(), {"strong": 1, "weak": 1},
                             {"kind": "randint64"}, I, O, math.inf, 0, pols, wrr=(4.0, 1.0), mode="static"))
    cases.append(replay_case("static_two_instance_normal", two_instance_profile(), {"strong": 1, "weak": 1},
                             {"kind": "randint64"}, I, O, math.inf, 5, ["OS", "MB"],
                             predictor={"mode": "normal", "mean": 30, "stddev": 10, "seed": None}, mode="static"))
    # criterion-3 shape: one machine x4 at tp 4, SI, 2000-token budget (test_acceptance.py:170-219)
    p3 = tiny_profile([("m0", 4, (32 * 2000 + 200) // 4 + 1, "x")], limits=dict(max_input_len=512, max_output_len=512))
    p3.params = {("m0", 4): POSITIVE}
    rng3 = random.Random(1000)
    I3 = np.array([rng3.randint(1, 64) for _ in range(200)], np.int32)
    O3 = np.array([rng3.randint(1, 64) for _ in range(200)], np.int32)
    cases.append(replay_case("static_criterion3", p3, {"m0": 4}, {"kind": "crit3"}, I3, O3, math.inf, 0, ["SI", "OS"],
                             mode="static"))
    I, O = wl.trace_lengths(3000, seed=7)
    cases.append(replay_case("static_config4_small", wl.config4(), {a: 1 for a in wl.CONFIG4_TYPES}, {"seed": 7},
                             I, O, math.inf, 0, ["OS", "RR", "MB"], mode="static"))
    pb = tiny_profile([("m0", 1, 32 * 100 + 200, "x")], limits=dict(max_input_len=32, max_output_len=32))
    pb.params = {("m0", 1): POSITIVE}
    cases.append(replay_case("static_err_oversized", pb, {"m0": 1}, {"kind": "fixed"}, np.array([5, 400, 6], np.int32),
                             np.array([5, 400, 6], np.int32), math.inf, 0, ["OS"], mode="static"))
    return cases


def build_wide_cases() -> list:
    """Deployments with more than 32 instances (config-5 shapes): the
    config-3 cluster at 70B with several per-machine degrees."""
    cases = []
    p3 = wl.config3()
    # 72 instances: b200/h200 at t=2 (8 each x 4 machines), the rest t=4 / t=8
    deg72 = {}
    for name, count, _mem, acc in p3.machines:
        deg72[name] = 2 if acc in ("b200", "h200") else (8 if acc in ("v100", "a10") else 4)
    I, O = wl.trace_lengths(1500, seed=11)
    cases.append(replay_case("wide72", p3, deg72, {"seed": 11}, I, O, 400.0, 3, ["OS", "RR", "MB"]))
    deg40 = {n: (4 if acc in ("b200", "h200") else (16 if acc in ("v100", "a10", "l40s") else 8))
             for n, c, m, acc in p3.machines}
    I, O = wl.trace_lengths(1500, seed=12)
    cases.append(replay_case("wide40_inf", p3, deg40, {"seed": 12}, I, O, math.inf, 0, ["OS", "SI"]))
    cases.append(replay_case("wide40_static", p3, deg40, {"seed": 12}, I, O, math.inf, 0, ["OS"], mode="static"))
    return cases


def build_exp_vectors() -> dict:
    rng = np.random.default_rng(5)
    xs = np.concatenate([rng.uniform(0, 1, 3000), rng.uniform(0, 20, 3000), rng.uniform(0, 709.7, 3000),
                         rng.uniform(-745, 0, 1000), np.array([0.0, 1e-300, 5e-324, 511.99, 512.0, 700.0, 709.78,
                                                               -1e-18, 1e-18, 2.0, 0.5])])
    return {"x": [H(x) for x in xs], "y": [H(math.exp(x)) for x in xs],
            "overflow": [H(x) for x in (709.8, 710.0, 1e5)]}


STREAM_TRACES = [  # (seed, count, input_dist, output_dist, max_in, max_out)
    (0, 2001, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096),
    (7, 1001, "uniform:1:4096", "lognormal:300:1.0", 4096, 2048),
    (9, 999, "uniform:5:77", "uniform:1:9", 64, 8),
    (3, 777, "lognormal:1000:2.5", "uniform:1:4294967296", 4096, 4096),
    (11, 1, "uniform:3:3", "lognormal:50:0.1", 4096, 4096),
    (12, 0, "lognormal:50:0.1", "lognormal:50:0.1", 4096, 4096),
    (13, 300, "lognormal:1.7e308:0.5", "lognormal:10:0.5", 4096, 4096),  # overflows: round(inf)
]
STREAM_ARRIVALS = [(3000, 140.0, 42), (1000, 0.5, 1), (257, 1e6, 77), (5, float("inf"), 3)]
STREAM_PREDICTORS = [(2000, 150.0, 60.0, 5, 4096), (999, 3.0, 40.0, 8, 16), (300, 1e4, 1.0, 2, 4096)]


def build_stream_cases() -> dict:
    """The reference's own seeded draws: cmd_gen_trace (cli.py:183-197),
    generate_arrivals (simulator.py:112-124), OutputLengthPredictor.predict
    (scheduling.py:87-95), one call per request in trace order."""
    import argparse
    import tempfile

    from hetserve import cli as ref_cli

    traces = []
    for seed, count, di, do, mi, mo in STREAM_TRACES:
        with tempfile.TemporaryDirectory() as tmp:
            out = pathlib.Path(tmp) / "t.jsonl"
            ns = argparse.Namespace(seed=seed, count=count, input_dist=di, output_dist=do, max_input_len=mi,
                                    max_output_len=mo, out=str(out))
            try:
                ref_cli.cmd_gen_trace(ns)
                reqs = hs.parse_trace(out.read_text())
                traces.append(dict(seed=seed, count=count, input_dist=di, output_dist=do, max_in=mi, max_out=mo,
                                   I=[r.input_len for r in reqs], O=[r.output_len for r in reqs], error=None))
            except Exception as exc:  # noqa: BLE001
                traces.append(dict(seed=seed, count=count, input_dist=di, output_dist=do, max_in=mi, max_out=mo,
                                   I=None, O=None, error=f"{type(exc).__name__}: {exc}"))
    arrivals = []
    for n, rate, seed in STREAM_ARRIVALS:
        trace = [hs.Request(f"r{k}", 1, 1, 1) for k in range(n)]
        arrivals.append(dict(n=n, rate=H(rate), seed=seed, t=[H(t) for _, t in hs.generate_arrivals(trace, rate, seed)]))
    preds = []
    for n, mean, sd, seed, cap in STREAM_PREDICTORS:
        pr = hs.OutputLengthPredictor(hs.PredictorConfig(mode="normal", mean=mean, stddev=sd, seed=seed), cap)
        preds.append(dict(n=n, mean=H(mean), stddev=H(sd), seed=seed, cap=cap,
                          p=[pr.predict(hs.Request(f"r{k}", 1, 7, 7)) for k in range(n)]))
    return dict(traces=traces, arrivals=arrivals, predictors=preds)


def _sched_snapshot(sch) -> dict:
    snap = sch.snapshot()
    return {"loads": [H(v) for v in snap["loads"].values()], "kv_usage": [H(v) for v in snap["kv_usage"].values()],
            "running": list(snap["running_tokens"].values()), "oversized": list(snap["oversized"].values()),
            "in_flight": snap["in_flight"]}


def sched_case(name, profile, degrees, policy, n_ops, seed, max_len=2000, allowed_p=0.3, complete_p=0.3,
               evaluate_p=0.1, dup_p=0.03, bogus_p=0.03) -> dict:
    """A seeded sequence of Scheduler.choose / complete / evaluate calls on
    the reference's live scheduler (scheduling.py:175-346), recording every
    result or exception and the snapshot after each call."""
    cluster, params = ref_cluster(profile), ref_params(profile)
    cfg = hs.deployment_for(cluster.machines, degrees)
    handles = hs.build_instances(cluster, cfg, params)
    n = len(handles)
    if policy.get("wrr") == "auto":
        policy = dict(policy, wrr=[1 + (7 * j) % 5 for j in range(n)])
    pol = hs.PolicyConfig(policy=policy["policy"], theta=policy.get("theta", 2.0),
                          wrr_weights=tuple(policy["wrr"]) if policy.get("wrr") else None)
    sch = hs.Scheduler(handles, cluster.model, pol)
    rng = random.Random(seed)
    ops, live, next_id = [], [], 0
    for _ in range(n_ops):
        u = rng.random()
        allowed = None
        if rng.random() < allowed_p:
            allowed = sorted(rng.sample(range(n + 2), rng.randint(0, min(n + 2, 4))))
        if u < complete_p and (live or rng.random() < bogus_p * 10):
            if live and rng.random() > bogus_p:
                rid = live.pop(rng.randrange(len(live)))
            else:
                rid = f"ghost{next_id}"
            op = {"op": "complete", "id": rid}
            try:
                sch.complete(rid)
            except (hs.HetserveError, OverflowError, ZeroDivisionError) as exc:
                op["error"], op["msg"] = type(exc).__name__, str(exc)
        else:
            if rng.random() < dup_p and live:
                rid = rng.choice(live)
            else:
                rid = f"r{next_id}"
                next_id += 1
            I = rng.randint(1, max_len)
            P = rng.randint(1, max_len)
            req = hs.Request(rid, I, P, P)
            kind = "evaluate" if u > 1.0 - evaluate_p else "choose"
            op = {"op": kind, "id": rid, "I": I, "P": P, "allowed": allowed}
            try:
                if kind == "choose":
                    op["chosen"] = sch.choose(req, set(allowed) if allowed is not None else None)
                    live.append(rid)
                else:
                    op["weights"] = [H(w) for w in sch.evaluate(req, set(allowed) if allowed is not None else None)]
            except (hs.HetserveError, OverflowError, ZeroDivisionError) as exc:
                op["error"], op["msg"] = type(exc).__name__, str(exc)
        op["snap"] = _sched_snapshot(sch)
        ops.append(op)
    return {"name": name, "profile": profile_desc(profile), "degrees": degrees, "policy": policy, "ops": ops}


def build_sched_cases() -> list:
    cases = []
    p2 = wl.config2()
    deg2 = {"v100": 2, "a800": 1, "h100": 1}
    for pol in ({"policy": "OS"}, {"policy": "MB"}, {"policy": "RR"}, {"policy": "SI"},
                {"policy": "WRR", "wrr": "auto"}, {"policy": "OS", "theta": 0.7}):
        cases.append(sched_case(f"config2-{pol['policy']}-{pol.get('theta', 2.0)}", p2, deg2, pol, 400,
                                seed=len(cases)))
    p4 = wl.config4()
    cases.append(sched_case("config4-OS", p4, {a: 1 for a in wl.CONFIG4_TYPES}, {"policy": "OS"}, 600, seed=77,
                            max_len=4000))
    # tiny budgets: oversized requests, exp overflow at high KV pressure, negative decode prices
    tiny = tiny_profile([("a", 2, 30_000, "x"), ("b", 1, 40_000, "y")],
                        params={("a", 1): (1e-5, 1e-4, 1e-5, 1e-3, 1e-6, 1e-4, 1e-7, 1e-4),
                                ("a", 2): (1e-5, 1e-4, 1e-5, 1e-3, 1e-6, 1e-4, 1e-7, 1e-4),
                                ("b", 1): (2e-5, 2e-4, 2e-5, 2e-3, 2e-6, 2e-4, 2e-7, 2e-4)})
    cases.append(sched_case("tiny-OS-theta40", tiny, {"a": 1, "b": 1}, {"policy": "OS", "theta": 40.0}, 200, seed=5,
                            max_len=900, complete_p=0.15))
    cases.append(sched_case("tiny-MB-theta40", tiny, {"a": 1, "b": 1}, {"policy": "MB", "theta": 40.0}, 200, seed=8,
                            max_len=900, complete_p=0.15))
    neg = tiny_profile([("a", 1, 2_000_000, "x"), ("b", 1, 3_000_000, "y")],
                       params={("a", 1): (1e-5, 1e-4, 1e-5, 1e-3, 1e-6, 1e-4, 1e-7, 1e-4),
                               ("b", 1): (-1e-3, -1e-2, -1e-3, -1e-1, 1e-6, 1e-4, 1e-7, 1e-4)})
    cases.append(sched_case("tiny-negative-RR", neg, {"a": 1, "b": 1}, {"policy": "RR"}, 60, seed=6, max_len=50))
    cases.append(sched_case("tiny-negative-OS", neg, {"a": 1, "b": 1}, {"policy": "OS"}, 60, seed=7, max_len=50))
    return cases


PLAN_CASES = [  # (name, seed, n, lo, hi, budget bytes, params scale) on a 7B model
    ("typical", 1, 3000, 20, 900, 8.0e9, 1.0),
    ("tight", 2, 500, 100, 4000, 4.5e9, 0.5),
    ("one_batch", 3, 64, 1, 30, 1e13, 2.0),
    ("empty", 4, 0, 1, 2, 1e9, 1.0),
    ("infeasible", 5, 200, 10, 3300, 3.0e9, 1.0),
    ("zero_time", 6, 40, 5, 50, 5e9, 0.0),
    ("negative_budget", 7, 10, 5, 50, -1.0, 1.0),
    ("ragged_budget", 8, 2000, 1, 2000, 1234567.89 * 4096, 1.7),
]


def build_plan_cases() -> list:
    """planner.py:51-118 single-instance functions of the reference:
    plan_static_batches, time_batches, estimate_instance_throughput."""
    model = hs.ModelSpec(**wl.MODEL_7B)
    out = []
    for name, seed, n, lo, hi, budget, scale in PLAN_CASES:
        rng = random.Random(seed)
        reqs = [hs.Request(f"q{k}", rng.randint(lo, hi), rng.randint(lo, hi), 1) for k in range(n)]
        params = hs.LatencyParams(*(scale * x for x in wl.RANK_BASE))
        kb = hs.KvBudget(total_bytes=budget)
        case = {"name": name, "seed": seed, "n": n, "lo": lo, "hi": hi, "budget": H(budget), "scale": H(scale)}
        try:
            plan = hs.plan_static_batches(reqs, kb, model)
            case["batches"] = [list(b) for b in plan.batches]
            case["times"] = [H(t) for t in hs.time_batches(plan, reqs, params).per_batch_time]
        except (hs.HetserveError, ZeroDivisionError) as exc:
            case["plan_error"] = [type(exc).__name__, str(exc)]
        try:
            case["rate"] = H(hs.estimate_instance_throughput(reqs, kb, model, params))
        except (hs.HetserveError, ZeroDivisionError) as exc:
            case["rate_error"] = [type(exc).__name__, str(exc)]
        out.append(case)
    return out


def main() -> None:
    which = sys.argv[1:] or ["exp", "search", "replay", "static", "wide", "streams", "sched", "plan"]
    if "exp" in which:
        (OUT / "exp_vectors.json").write_text(json.dumps(build_exp_vectors()))
    if "search" in which:
        (OUT / "search_cases.json").write_text(json.dumps(build_search_cases()))
    if "replay" in which:
        (OUT / "replay_cases.json").write_text(json.dumps(build_replay_cases()))
    if "static" in which:
        (OUT / "static_cases.json").write_text(json.dumps(build_static_cases()))
    if "wide" in which:
        (OUT / "wide_cases.json").write_text(json.dumps(build_wide_cases()))
    if "streams" in which:
        (OUT / "stream_cases.json").write_text(json.dumps(build_stream_cases()))
    if "sched" in which:
        (OUT / "sched_cases.json").write_text(json.dumps(build_sched_cases()))
    if "plan" in which:
        (OUT / "plan_cases.json").write_text(json.dumps(build_plan_cases()))


if __name__ == "__main__":
    main()
