"""CUDA engine vs the reference (golden fixtures) and vs the C oracle.

Every assertion is bit-exact (float.hex / integer equality): the path is
integer and fp64 work evaluated in the reference's operation order.
"""

import math

import numpy as np
import pytest

import helpers as H
import paper_2504_15303_b200 as hs
from oracle import hs_oracle as orc
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import planner
from paper_2504_15303_b200 import workloads as wl

pytestmark = pytest.mark.gpu

SEARCH = H.load("search_cases.json")
REPLAY = H.load("replay_cases.json") + H.load("static_cases.json") + H.load("wide_cases.json")


@pytest.fixture(scope="module")
def eng():
    e = nat.engine_for(0)
    yield e


@pytest.mark.parametrize("case", [c for c in SEARCH if c["kind"] == "search"], ids=lambda c: c["name"])
def test_search_tables_match_reference(eng, case):
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    requests = H.search_trace(case)
    t = planner.build_tables(cluster, requests, params_by, engine=eng)
    H.check_table(case, t.entries, t.n_degrees, requests)


@pytest.mark.parametrize("case", [c for c in SEARCH if c["kind"] == "search" and ("ranked" in c or "error" in c)],
                         ids=lambda c: c["name"])
def test_search_optimal_config_matches_reference(eng, case):
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    requests = H.search_trace(case)
    if "error" in case:
        with pytest.raises(ZeroDivisionError, match=case["error"]["msg"]):
            hs.search_optimal_config(cluster, requests, params_by, engine=eng)
        return
    out = hs.search_optimal_config(cluster, requests, params_by, engine=eng)
    assert out.candidates_visited == case["visited"]
    assert len(out.ranked) == len(case["ranked"])
    for got, want in zip(out.ranked, case["ranked"]):
        assert [p.tp_degree for p in got.config.per_machine] == want["degrees"]
        assert got.system_tokens_per_sec.hex() == want["total"]
        pm = [[m.instance_tokens_per_sec.hex(), m.machine_tokens_per_sec.hex(), m.budget_bytes.hex(),
               m.slack_bytes.hex(), m.instance_count] for m in got.per_machine]
        assert pm == want["per_machine"]
    assert [[[p.tp_degree for p in c.per_machine], r] for c, r in out.infeasible] == case["infeasible"]
    if out.ranked:
        best = out.best
        est = hs.estimate_system_throughput(cluster, best.config, requests, params_by, engine=eng)
        assert est.system_tokens_per_sec == best.system_tokens_per_sec
        assert est.per_machine == best.per_machine


def test_estimate_system_throughput_errors_in_config_order(eng):
    case = next(c for c in SEARCH if c["name"] == "mixed_failures")
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    requests = H.search_trace(case)
    for degrees, reason in case["infeasible"][:12]:
        cfg = hs.deployment_for(cluster.machines, {m.name: t for m, t in zip(cluster.machines, degrees)})
        with pytest.raises((hs.InfeasibleConfigError, hs.InfeasibleRequestError, hs.SpecError)) as ei:
            hs.estimate_system_throughput(cluster, cfg, requests, params_by, engine=eng)
        assert str(ei.value) == reason


def _config3_tables(eng):
    case = next(c for c in SEARCH if c["name"] == "config3_table")
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    requests = H.search_trace(case)
    return case, requests, planner.build_tables(cluster, requests, params_by, engine=eng)


def test_config3_full_space_argmax(eng):
    """5^16 = 1.5e11 candidates: every one evaluated on the GPU; the winner,
    its total and the feasible count checked against the exact oracle."""
    case, requests, t = _config3_tables(eng)
    H.check_table(case, t.entries, t.n_degrees, requests)
    P = t.space_size
    assert P == 5**16
    total, idx, nfeas, _ms = planner.search_best(t, engine=eng)
    V, vidx, vfeas = orc.best_monotone(t.entries, t.n_degrees)
    assert (total.hex(), idx, nfeas) == (V.hex(), vidx, vfeas)
    # the winner re-scored through the table equals the reported total
    assert planner.best_config(t, idx).system_tokens_per_sec == total


def test_config3_sharded_ranges_combine(eng):
    _case, _req, t = _config3_tables(eng)
    P = t.space_size
    cuts = [0, P // 7, P // 3, P // 3 + 12345, (2 * P) // 3, P]
    parts = [planner.search_best(t, a, b, engine=eng) for a, b in zip(cuts, cuts[1:])]
    best = max(((p[0], -p[1]) for p in parts if p[1] >= 0))
    total, idx, nfeas, _ = planner.search_best(t, engine=eng)
    assert (best[0], -best[1]) == (total, idx)
    assert sum(p[2] for p in parts) == nfeas


def test_search_best_random_ranges_vs_bruteforce_oracle(eng):
    _case, _req, t = _config3_tables(eng)
    P = t.space_size
    rng = np.random.default_rng(7)
    for _ in range(6):
        a = int(rng.integers(0, P - 3_000_000))
        b = a + int(rng.integers(1, 3_000_000))
        got = planner.search_best(t, a, b, engine=eng)
        want = orc.best(t.entries, t.n_degrees, a, b, nthreads=4)
        assert (got[0], got[1], got[2]) == want or (got[1] == -1 and want[1] == -1 and got[2] == want[2])


def test_search_best_small_spaces_vs_rank(eng):
    """Every search fixture: argmax == head of the full ranking."""
    for case in SEARCH:
        if case["kind"] != "search" or not case.get("ranked"):
            continue
        cluster = H.cluster_from(case["profile"])
        t = planner.build_tables(cluster, H.search_trace(case), H.params_from(case["profile"]), engine=eng)
        total, idx, nfeas, _ = planner.search_best(t, engine=eng)
        assert total.hex() == case["ranked"][0]["total"]
        assert nfeas == len(case["ranked"])


REPLAY_PARAMS = [(c, k) for c in REPLAY for k in range(len(c["results"]))]


@pytest.mark.parametrize("case,k", REPLAY_PARAMS, ids=lambda v: v["name"] if isinstance(v, dict) else str(v))
def test_run_scenario_matches_reference(eng, case, k):
    want = case["results"][k]
    sc = H.scenario_from(case, want["policy"])
    if "error" in want:
        exc = {"InfeasibleRequestError": hs.InfeasibleRequestError, "OverflowError": OverflowError,
               "SpecError": hs.SpecError, "SchedulingError": hs.SchedulingError}[want["error"]]
        with pytest.raises(exc) as ei:
            hs.run_scenario(sc, engine=eng)
        assert str(ei.value) == want["msg"]
        return
    got = H.sim_digest(hs.run_scenario(sc, engine=eng))
    for key, val in want.items():
        assert got[key] == val, (case["name"], want["policy"], key)


@pytest.mark.parametrize("policy", ["OS", "RR", "WRR", "SI", "MB"])
def test_batched_replay_vs_oracle(eng, policy):
    """64 ragged config-4-shaped traces (incl. an empty one) at mixed rates."""
    prof = wl.config4()
    cluster = H.cluster_from({"model": prof.model, "engine": {"mem_utilization_fraction": (0.9).hex(),
                              "static_overhead_bytes": prof.engine["static_overhead_bytes"]},
                              "limits": prof.limits, "machines": [list(m) for m in prof.machines], "params": []})
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    rng = np.random.default_rng(99)
    lens = [int(x) for x in rng.integers(0, 1500, 64)]
    lens[5] = 0
    Is, Os, Ts = [], [], []
    for t, q in enumerate(lens):
        I, O = wl.trace_lengths(q, seed=1000 + t)
        rate = [20.0, 140.0, 1500.0, math.inf][t % 4]
        Is.append(I)
        Os.append(O)
        Ts.append(np.zeros(q) if math.isinf(rate) else wl.arrivals(q, rate, seed=t))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I, O, T = np.concatenate(Is), np.concatenate(Os), np.concatenate(Ts)
    wrr = tuple(float(x) for x in rng.integers(1, 5, 32)) if policy == "WRR" else None
    pol = hs.PolicyConfig(policy=policy, theta=2.0, wrr_weights=wrr)
    res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, arrival=T, want_assign=True,
                           want_depart=True, engine=eng)
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    handles = build_instances(cluster, config, params)
    a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, 32, hs.kv_bytes_per_token(cluster.model)),
                            off, I, O, O, T, nthreads=8)
    assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
    assert np.array_equal(res.assign, a)
    assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64))
    for f in ("completion_time", "peak_kv_usage", "residual_load"):
        assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), f
    for f in ("request_count", "token_count"):
        assert np.array_equal(res.metrics[f], m[f]), f


@pytest.mark.parametrize("policy", ["OS", "RR", "MB"])
def test_batched_static_replay_vs_oracle(eng, policy):
    """run_static on 48 ragged config-4-shaped traces vs the oracle."""
    prof = wl.config4()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(1, 4000, 48)]
    Is, Os = zip(*(wl.trace_lengths(q, seed=500 + t) for t, q in enumerate(lens)))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I, O = np.concatenate(Is), np.concatenate(Os)
    pol = hs.PolicyConfig(policy=policy)
    res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, want_depart=True,
                           engine=eng, static=True)
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    handles = build_instances(cluster, config, params)
    a, d, m, r = orc.replay(engine_instances(handles, pol),
                            _policy_struct(pol, 32, hs.kv_bytes_per_token(cluster.model), 1), off, I, O, O, None,
                            nthreads=8)
    assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
    assert np.array_equal(res.assign, a)
    assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64))
    for f in ("completion_time", "peak_kv_usage", "residual_load"):
        assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), f


def test_config4_full_size_static_vs_oracle(eng):
    """run_static at bench scale: 4 full config-4 traces (1e5 requests each,
    OS) vs the oracle -- every assignment, batch completion time and metric."""
    from paper_2504_15303_b200 import streams
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    prof = wl.config4()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    nT, q = 4, wl.CONFIG4_Q
    I, O = streams.gen_trace_lengths(list(range(200, 200 + nT)), q, "lognormal:200:0.6", "lognormal:150:0.6",
                                     4096, 4096, engine=eng)
    off = np.arange(nT + 1, dtype=np.int64) * q
    pol = hs.PolicyConfig()
    res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, want_depart=True,
                           engine=eng, static=True)
    handles = build_instances(cluster, config, params)
    a, d, m, r = orc.replay(engine_instances(handles, pol),
                            _policy_struct(pol, 32, hs.kv_bytes_per_token(cluster.model), 1), off, I, O, O, None,
                            nthreads=8)
    assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
    assert np.array_equal(res.assign, a)
    assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64))
    for f in ("completion_time", "peak_kv_usage", "residual_load"):
        assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), f


def test_config3_top1024_vs_oracle(eng):
    """BASELINE config 5's first stage: top-1024 of the 5^16 space."""
    _case, _req, t = _config3_tables(eng)
    top, nf, _ms = planner.search_topk(t, 1024, engine=eng)
    want, wnf = orc.topk(t.entries, t.n_degrees, 1024)
    assert nf == wnf == 5184 ** 2
    assert top["index"].tolist() == want["index"].tolist()
    assert top["total"].view(np.uint64).tolist() == want["total"].view(np.uint64).tolist()
    # head agrees with the exhaustive argmax
    total, idx, _n, _ = planner.search_best(t, engine=eng)
    assert (float(top["total"][0]), int(top["index"][0])) == (total, idx)
    parts = [planner.search_topk(t, 1024, s, 4, engine=eng)[0] for s in range(4)]
    merged = planner.merge_topk(parts, 1024)
    assert merged["index"].tolist() == want["index"].tolist()


@pytest.mark.parametrize("case", [c for c in SEARCH if c["kind"] == "search" and c.get("ranked")],
                         ids=lambda c: c["name"])
def test_topk_is_head_of_reference_ranking(eng, case):
    cluster = H.cluster_from(case["profile"])
    t = planner.build_tables(cluster, H.search_trace(case), H.params_from(case["profile"]), engine=eng)
    k = len(case["ranked"])
    top, nf, _ = planner.search_topk(t, k + 5, engine=eng)
    assert nf == k
    assert [float(x).hex() for x in top["total"]] == [r["total"] for r in case["ranked"]]


def test_replay_deployments_mixed_widths_vs_oracle(eng):
    """Config-5 shape: each trace on its own deployment (9 to 100 instances,
    1 to 4 warps per trace) in one launch, vs the oracle trace by trace."""
    p3 = wl.config3()
    cluster = hs.ClusterSpec(hs.ModelSpec(**p3.model), hs.EngineOverheads(**p3.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in p3.machines),
                             hs.WorkloadLimits(**p3.limits))
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    rng = np.random.default_rng(17)
    feas = {"b200": [2, 4, 8, 16], "h200": [2, 4, 8, 16], "h100": [4, 8, 16], "a100": [4, 8, 16],
            "a800": [4, 8, 16], "l40s": [4, 8, 16], "v100": [8, 16], "a10": [8, 16]}
    configs = []
    for _ in range(6):
        deg = {n: int(rng.choice(feas[acc])) for n, c, m, acc in p3.machines}
        configs.append(hs.deployment_for(cluster.machines, deg))
    configs.append(hs.deployment_for(cluster.machines, {n: feas[acc][0] for n, c, m, acc in p3.machines}))
    configs.append(hs.deployment_for(cluster.machines, {n: 16 for n, c, m, acc in p3.machines}))
    sizes = [len(hs.build_instances(cluster, c, params)) for c in configs]
    assert max(sizes) > 64 and min(sizes) <= 32
    T = 28
    tdep = np.arange(T) % len(configs)
    lens = [int(x) for x in rng.integers(200, 1500, T)]
    Is, Os, Ts = [], [], []
    for t, q in enumerate(lens):
        I, O = wl.trace_lengths(q, seed=900 + t)
        Is.append(I); Os.append(O); Ts.append(wl.arrivals(q, [200.0, 2000.0][t % 2], seed=t))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I, O, Tm = np.concatenate(Is), np.concatenate(Os), np.concatenate(Ts)
    pol = hs.PolicyConfig(policy="OS")
    res = hs.replay_deployments(cluster, configs, params, pol, tdep, off, I, O, O, arrival=Tm, want_depart=True,
                                engine=eng)
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    per_token = hs.kv_bytes_per_token(cluster.model)
    for t in range(T):
        handles = build_instances(cluster, configs[tdep[t]], params)
        n = len(handles)
        sl = slice(off[t], off[t + 1])
        a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, n, per_token),
                                np.array([0, lens[t]], np.int64), I[sl], O[sl], O[sl], Tm[sl])
        assert int(res.result[t]["error"]) == 0 == int(r[0]["error"])
        assert np.array_equal(res.assign[sl], a), t
        assert np.array_equal(res.depart[sl].view(np.uint64), d.view(np.uint64)), t
        for f in ("completion_time", "residual_load", "peak_kv_usage"):
            assert np.array_equal(res.metrics[t, :n][f].view(np.uint64), m[0][f].view(np.uint64)), (t, f)


def test_config5_shape_topk_then_rescore(eng):
    """Top-12 deployments of the config-3 space, each replayed (rate=inf, OS)
    on the same 3000-request trace in one launch, vs the oracle."""
    _case, _req, t = _config3_tables(eng)
    top, _nf, _ = planner.search_topk(t, 12, engine=eng)
    configs = [planner.deployment_of(t, int(i)) for i in top["index"]]
    p3 = wl.config3()
    cluster = t.cluster
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    I1, O1 = wl.trace_lengths(3000, seed=0)
    n = len(configs)
    off = np.arange(n + 1, dtype=np.int64) * 3000
    I, O = np.tile(I1, n), np.tile(O1, n)
    res = hs.replay_deployments(cluster, configs, params, hs.PolicyConfig(), np.arange(n), off, I, O, O,
                                want_depart=True, engine=eng)
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    per_token = hs.kv_bytes_per_token(cluster.model)
    for d in range(n):
        handles = build_instances(cluster, configs[d], params)
        sl = slice(off[d], off[d + 1])
        a, dep, m, r = orc.replay(engine_instances(handles, hs.PolicyConfig()),
                                  _policy_struct(hs.PolicyConfig(), len(handles), per_token),
                                  np.array([0, 3000], np.int64), I1, O1, O1, None)
        assert int(res.result[d]["error"]) == 0 == int(r[0]["error"])
        assert np.array_equal(res.assign[sl], a)
        assert np.array_equal(res.depart[sl].view(np.uint64), dep.view(np.uint64))


def test_config4_full_size_traces_vs_oracle(eng):
    """Bench-scale parity: 48 full config-4 traces (1e5 requests each, 140
    req/s, OS, 32 instances) -- the bench's exact inputs for traces 0..47,
    drawn on the device -- vs the literal C oracle, every assignment and
    departure time bit for bit."""
    from paper_2504_15303_b200 import streams
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    prof = wl.config4()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    nT, q = 48, wl.CONFIG4_Q
    seeds = list(range(nT))
    I, O = streams.gen_trace_lengths(seeds, q, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096, engine=eng)
    T = streams.arrival_times([42 + s for s in seeds], [q] * nT, wl.CONFIG4_RATE, engine=eng)
    off = np.arange(nT + 1, dtype=np.int64) * q
    pol = hs.PolicyConfig()
    res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, arrival=T, want_assign=True,
                           want_depart=True, engine=eng)
    handles = build_instances(cluster, config, params)
    a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, 32, hs.kv_bytes_per_token(cluster.model)),
                            off, I, O, O, T, nthreads=16)
    assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
    assert np.array_equal(res.result["n_steps"], r["n_steps"])
    assert np.array_equal(res.assign, a)
    assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64))
    for f in ("completion_time", "peak_kv_usage", "residual_load"):
        assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), f


@pytest.mark.parametrize("policy,pred", [("RR", "oracle"), ("WRR", "oracle"), ("SI", "oracle"), ("MB", "oracle"),
                                         ("OS", "normal")])
def test_config4_full_size_policies_vs_oracle(eng, policy, pred):
    """Bench-scale parity for the baselines and the normal predictor: 8 full
    config-4 traces (1e5 requests each, 140 req/s, 32 instances) per policy,
    inputs drawn on the device (lengths, arrivals, normal predictions), vs the
    literal C oracle bit for bit."""
    from paper_2504_15303_b200 import streams
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    prof = wl.config4()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    nT, q = 8, wl.CONFIG4_Q
    seeds = list(range(100, 100 + nT))
    I, O = streams.gen_trace_lengths(seeds, q, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096, engine=eng)
    T = streams.arrival_times([42 + s for s in seeds], [q] * nT, wl.CONFIG4_RATE, engine=eng)
    if pred == "normal":
        P = streams.predict_lengths([7 + s for s in seeds], [q] * nT, 150.0, 60.0, 4096, engine=eng)
        pc = hs.PredictorConfig(mode="normal", mean=150.0, stddev=60.0, seed=7)
    else:
        P = O
        pc = hs.PredictorConfig()
    off = np.arange(nT + 1, dtype=np.int64) * q
    # WRR weights: proportional to the instance's capacity class (b200 > h100 = a800 > v100)
    wrr = tuple(float(w) for w in np.repeat([4.0, 2.0, 2.0, 1.0], 8)) if policy == "WRR" else None
    pol = hs.PolicyConfig(policy=policy, theta=2.0, predictor=pc, wrr_weights=wrr)
    res = hs.replay_traces(cluster, config, params, pol, off, I, O, P, arrival=T, want_assign=True,
                           want_depart=True, engine=eng)
    handles = build_instances(cluster, config, params)
    a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, 32, hs.kv_bytes_per_token(cluster.model)),
                            off, I, O, P, T, nthreads=16)
    assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
    assert np.array_equal(res.result["n_steps"], r["n_steps"])
    assert np.array_equal(res.assign, a)
    assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64))
    for f in ("completion_time", "peak_kv_usage", "residual_load"):
        assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), f


def test_config5_full_size_rescore_vs_oracle(eng):
    """BASELINE config 5 at full size for a slice: the top-1024 deployments of
    the config-3 space, the first 128 of them each replayed on the 1e5-request
    trace (rate = inf, OS; up to 72 instances = 3 warps per trace, the
    warp-0 dispatch phase) in one launch, vs the oracle."""
    from concurrent.futures import ThreadPoolExecutor
    _case, _req, t = _config3_tables(eng)
    top, _nf, _ = planner.search_topk(t, 1024, engine=eng)
    assert len(top) == 1024
    n = 128
    configs = [planner.deployment_of(t, int(i)) for i in top["index"][:n]]
    p3 = wl.config3()
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    q = wl.CONFIG4_Q
    I1, O1 = wl.trace_lengths(q, seed=0)
    off = np.arange(n + 1, dtype=np.int64) * q
    res = hs.replay_deployments(t.cluster, configs, params, hs.PolicyConfig(), np.arange(n), off, np.tile(I1, n),
                                np.tile(O1, n), np.tile(O1, n), want_depart=True, engine=eng)
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    per_token = hs.kv_bytes_per_token(t.cluster.model)

    def oracle(d):
        handles = build_instances(t.cluster, configs[d], params)
        return orc.replay(engine_instances(handles, hs.PolicyConfig()),
                          _policy_struct(hs.PolicyConfig(), len(handles), per_token),
                          np.array([0, q], np.int64), I1, O1, O1, None)

    widths = set()
    with ThreadPoolExecutor(max_workers=16) as ex:
        for d, (a, dep, m, r) in enumerate(ex.map(oracle, range(n))):
            sl = slice(off[d], off[d + 1])
            assert int(res.result[d]["error"]) == 0 == int(r[0]["error"])
            assert res.result[d]["n_steps"] == r[0]["n_steps"]
            assert np.array_equal(res.assign[sl], a)
            assert np.array_equal(res.depart[sl].view(np.uint64), dep.view(np.uint64))
            nd = m.shape[1]
            for f in ("completion_time", "peak_kv_usage", "residual_load"):
                assert np.array_equal(res.metrics[d][:nd][f].view(np.uint64), m[0][f].view(np.uint64)), (d, f)
            widths.add((nd + 31) // 32)
    assert 3 in widths


def test_replay_candidates_equals_object_path(eng):
    """replay_candidates (instance arrays assembled from the K1 table with
    numpy) == replay_deployments on deployment_of(...) objects, bit for bit."""
    _case, _req, t = _config3_tables(eng)
    top, _nf, _ = planner.search_topk(t, 40, engine=eng)
    idx = top["index"]
    p3 = wl.config3()
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    q = 2048
    I1, O1 = wl.trace_lengths(q, seed=5)
    n = len(idx)
    off = np.arange(n + 1, dtype=np.int64) * q
    I, O = np.tile(I1, n), np.tile(O1, n)
    for pol in (hs.PolicyConfig(), hs.PolicyConfig(policy="MB"), hs.PolicyConfig(policy="RR")):
        a = hs.replay_candidates(t, params, idx, pol, np.arange(n), off, I, O, O, want_depart=True, engine=eng)
        b = hs.replay_deployments(t.cluster, [planner.deployment_of(t, int(i)) for i in idx], params, pol,
                                  np.arange(n), off, I, O, O, want_depart=True, engine=eng)
        assert (b.result["error"] == 0).all()
        assert np.array_equal(a.assign, b.assign)
        assert np.array_equal(a.depart.view(np.uint64), b.depart.view(np.uint64))
        assert a.metrics.tobytes() == b.metrics.tobytes()
        assert a.result.tobytes() == b.result.tobytes()


def test_replay_candidates_assign_out_in_place(eng):
    """A page-locked assign_out is written by the kernel in place (no copy
    back) and equals the default (device buffer copied back) path."""
    _case, _req, t = _config3_tables(eng)
    top, _nf, _ = planner.search_topk(t, 24, engine=eng)
    p3 = wl.config3()
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    q = 3000
    I1, O1 = wl.trace_lengths(q, seed=11)
    n = len(top)
    off = np.arange(n + 1, dtype=np.int64) * q
    I, O = np.tile(I1, n), np.tile(O1, n)
    a = hs.replay_candidates(t, params, top["index"], hs.PolicyConfig(), np.arange(n), off, I, O, O, engine=eng)
    buf = eng.host_array((n * q + 5,), np.uint8)
    buf[:] = 0xAB
    b = hs.replay_candidates(t, params, top["index"], hs.PolicyConfig(), np.arange(n), off, I, O, O, engine=eng,
                             assign_out=buf)
    assert np.array_equal(a.assign, b.assign) and np.array_equal(buf[: n * q], a.assign)
    assert (buf[n * q:] == 0xAB).all()
    assert a.metrics.tobytes() == b.metrics.tobytes() and a.result.tobytes() == b.result.tobytes()
    with pytest.raises(ValueError):
        hs.replay_candidates(t, params, top["index"], hs.PolicyConfig(), np.arange(n), off, I, O, O, engine=eng,
                             assign_out=np.zeros(5, np.uint8))


def _twin_cluster():
    """Two machines of one accelerator type: equal degrees make one instance
    class, different degrees two."""
    prof = wl.config4()
    base = prof.machines[1]  # h100
    machines = (hs.MachineSpec("h100-0", 8, base[2], "h100"), hs.MachineSpec("h100-1", 8, base[2], "h100"),
                hs.MachineSpec("b200-0", 4, prof.machines[0][2], "b200"))
    cluster = hs.ClusterSpec(model=hs.ModelSpec(**prof.model), engine=hs.EngineOverheads(**prof.engine),
                             machines=machines, limits=hs.WorkloadLimits(**prof.limits))
    params = {}
    for m in machines:
        for t in wl.enumerate_degrees(m.accelerator_count):
            params[(m.name, t)] = hs.LatencyParams(*wl.scaled_params(wl.RANK_BASE, t ** -wl.TP_ALPHA *
                                                                     wl.TYPE_SCALE[m.accelerator_type]))
    return cluster, params


def test_replay_deployments_mixed_class_counts_small_deployments(eng):
    """deployments of <= 32 instances share a block (4 traces
    per block) while having different instance-class counts (1, 2, 3); the
    shared-memory price / class regions must not overlap.  Finite rate, OS
    and MB, each trace vs the oracle."""
    cluster, params = _twin_cluster()
    degs = [(1, 1, 1), (1, 2, 4), (2, 2, 2), (4, 8, 1), (1, 1, 4), (8, 8, 2), (2, 4, 1), (1, 8, 2)]
    configs = [hs.deployment_for(cluster.machines, dict(zip(("h100-0", "h100-1", "b200-0"), d))) for d in degs]
    q = 4000
    T = 16
    trace_dep = np.arange(T) % len(configs)
    I = np.concatenate([wl.trace_lengths(q, seed=100 + t)[0] for t in range(T)])
    O = np.concatenate([wl.trace_lengths(q, seed=100 + t)[1] for t in range(T)])
    A = np.concatenate([wl.arrivals(q, 60.0, 7 + t) for t in range(T)])
    off = np.arange(T + 1, dtype=np.int64) * q
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    per_token = hs.kv_bytes_per_token(cluster.model)
    for pol in (hs.PolicyConfig(), hs.PolicyConfig(policy="MB")):
        res = hs.replay_deployments(cluster, configs, params, pol, trace_dep, off, I, O, O, arrival=A,
                                    want_depart=True, engine=eng)
        for t in range(T):
            handles = build_instances(cluster, configs[trace_dep[t]], params)
            sl = slice(off[t], off[t + 1])
            a, dep, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, len(handles), per_token),
                                      np.array([0, q], np.int64), I[sl], O[sl], O[sl], A[sl])
            assert int(res.result[t]["error"]) == 0 == int(r[0]["error"])
            assert np.array_equal(res.assign[sl], a), (pol.policy, t)
            assert np.array_equal(res.depart[sl].view(np.uint64), dep.view(np.uint64)), (pol.policy, t)
            n = len(handles)
            for f in ("completion_time", "peak_kv_usage", "residual_load"):
                assert np.array_equal(res.metrics[t][:n][f].view(np.uint64), m[0][f].view(np.uint64)), f


@pytest.mark.parametrize("policy", ["OS", "RR", "WRR", "SI", "MB"])
def test_multiwarp_rate_inf_dispatch_phase_vs_oracle(eng, policy):
    """W = 2-3 warps per trace at rate = inf: warp 0 makes the whole dispatch
    sequence, then every warp steps its own instances (replay.cu inf_multi);
    each policy, continuous and static mode, vs the oracle."""
    _case, _req, t = _config3_tables(eng)
    top, _nf, _ = planner.search_topk(t, 64, engine=eng)
    p3 = wl.config3()
    params = {k: hs.LatencyParams(*v) for k, v in p3.params.items()}
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    per_token = hs.kv_bytes_per_token(t.cluster.model)
    seen = set()
    for idx in top["index"][::16]:
        config = planner.deployment_of(t, int(idx))
        handles = build_instances(t.cluster, config, params)
        N = len(handles)
        seen.add((N + 31) // 32)
        wrr = tuple(float(1 + k % 4) for k in range(N)) if policy == "WRR" else None
        pol = hs.PolicyConfig(policy=policy, wrr_weights=wrr)
        q, T = 6000, 3
        Is, Os = zip(*[wl.trace_lengths(q, seed=300 + k) for k in range(T)])
        I, O = np.concatenate(Is), np.concatenate(Os)
        off = np.arange(T + 1, dtype=np.int64) * q
        for static in (False, True):
            res = hs.replay_traces(t.cluster, config, params, pol, off, I, O, O, want_depart=True, engine=eng,
                                   static=static)
            a, d, m, r = orc.replay(engine_instances(handles, pol),
                                    _policy_struct(pol, N, per_token, 1 if static else 0), off, I, O, O, None,
                                    nthreads=4)
            assert (res.result["error"] == 0).all() and (r["error"] == 0).all()
            assert np.array_equal(res.assign, a), (policy, N, static)
            assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64)), (policy, N, static)
            for f in ("completion_time", "peak_kv_usage", "residual_load"):
                assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), (policy, N, f)
            for f in ("request_count", "token_count"):
                assert np.array_equal(res.metrics[f], m[f]), (policy, N, f)
    assert seen & {2, 3}


@pytest.mark.parametrize("n_machines", [17, 31])
def test_wide_deployments_over_128_instances_vs_oracle(eng, n_machines):
    """Deployments of 136 and 248 instances (6 and 8 warps per trace, four
    heap entries per lane in shared memory), every policy, finite rate and
    rate = inf, vs the oracle (the reference has no instance limit;
    simulator.py:127-158)."""
    prof = wl.config4()
    types = list(wl.CONFIG4_TYPES)
    machines = tuple(hs.MachineSpec(f"m{k}", 8, wl.TYPE_MEM_GB[types[k % 4]] * 1_000_000_000, types[k % 4])
                     for k in range(n_machines))
    cluster = hs.ClusterSpec(model=hs.ModelSpec(**prof.model), engine=hs.EngineOverheads(**prof.engine),
                             machines=machines, limits=hs.WorkloadLimits(**prof.limits))
    params = {(m.name, t): hs.LatencyParams(*wl.scaled_params(wl.RANK_BASE, t ** -wl.TP_ALPHA *
                                                               wl.TYPE_SCALE[m.accelerator_type]))
              for m in machines for t in wl.enumerate_degrees(8)}
    config = hs.deployment_for(machines, {m.name: 1 for m in machines})
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    handles = build_instances(cluster, config, params)
    N = len(handles)
    assert N > 128
    q, T = 5000, 3
    Is, Os = zip(*[wl.trace_lengths(q, seed=700 + k) for k in range(T)])
    I, O = np.concatenate(Is), np.concatenate(Os)
    off = np.arange(T + 1, dtype=np.int64) * q
    per_token = hs.kv_bytes_per_token(cluster.model)
    for policy in ("OS", "RR", "WRR", "SI", "MB"):
        wrr = tuple(float(1 + k % 3) for k in range(N)) if policy == "WRR" else None
        pol = hs.PolicyConfig(policy=policy, wrr_weights=wrr)
        for rate in (600.0, math.inf):
            A = None if math.isinf(rate) else np.concatenate([wl.arrivals(q, rate, seed=k) for k in range(T)])
            res = hs.replay_traces(cluster, config, params, pol, off, I, O, O, arrival=A, want_depart=True,
                                   engine=eng)
            a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, N, per_token), off, I, O, O,
                                    A, nthreads=3)
            assert (res.result["error"] == 0).all() and (r["error"] == 0).all(), (policy, rate)
            assert np.array_equal(res.assign, a), (policy, rate)
            assert np.array_equal(res.depart.view(np.uint64), d.view(np.uint64)), (policy, rate)
            assert np.array_equal(res.result["n_steps"], r["n_steps"]), (policy, rate)
            for f in ("completion_time", "peak_kv_usage", "residual_load"):
                assert np.array_equal(res.metrics[f].view(np.uint64), m[f].view(np.uint64)), (policy, rate, f)


@pytest.mark.parametrize("max_out", [60, 5000, 12000, 20000])
def test_retirement_calendar_ring_sizes_vs_oracle(eng, max_out):
    """Multi-warp multi-deployment replays size the retirement calendar from the
    launch's largest output length: 2^6 .. 2^14 buckets (one to four summary
    words per lane), and beyond 2^14 - 1 the heap again.  48- and 27-instance
    deployments (2 and 1 warps), OS / RR, finite rate and rate = inf, with a
    few outputs as long as max_out, vs the oracle."""
    prof = wl.config4()
    types = list(wl.CONFIG4_TYPES)
    machines = tuple(hs.MachineSpec(f"m{k}", 8, wl.TYPE_MEM_GB[types[k % 4]] * 1_000_000_000, types[k % 4])
                     for k in range(6))
    cluster = hs.ClusterSpec(model=hs.ModelSpec(**prof.model), engine=hs.EngineOverheads(**prof.engine),
                             machines=machines, limits=hs.WorkloadLimits(**prof.limits))
    params = {(m.name, t): hs.LatencyParams(*wl.scaled_params(wl.RANK_BASE, t ** -wl.TP_ALPHA *
                                                               wl.TYPE_SCALE[m.accelerator_type]))
              for m in machines for t in wl.enumerate_degrees(8)}
    configs = [hs.deployment_for(machines, {m.name: 1 for m in machines}),
               hs.deployment_for(machines, {m.name: (1 if k % 2 else 8) for k, m in enumerate(machines)})]
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    sizes = [len(build_instances(cluster, c, params)) for c in configs]
    assert sizes[0] == 48 and sizes[1] < 32
    q, T = 1500, 4
    Is, Os = [], []
    for t in range(T):
        I, O = wl.trace_lengths(q, seed=40 + t)
        O = np.minimum(O, max_out).astype(np.int32)
        O[np.random.default_rng(t).choice(q, 3, replace=False)] = max_out  # the longest retirements
        Is.append(I)
        Os.append(O)
    I, O = np.concatenate(Is), np.concatenate(Os)
    off = np.arange(T + 1, dtype=np.int64) * q
    tdep = np.arange(T) % 2
    per_token = hs.kv_bytes_per_token(cluster.model)
    for policy in ("OS", "RR"):
        pol = hs.PolicyConfig(policy=policy)
        for rate in (400.0, math.inf):
            A = None if math.isinf(rate) else np.concatenate([wl.arrivals(q, rate, seed=t) for t in range(T)])
            res = hs.replay_deployments(cluster, configs, params, pol, tdep, off, I, O, O, arrival=A,
                                        want_depart=True, engine=eng)
            for t in range(T):
                handles = build_instances(cluster, configs[tdep[t]], params)
                n = len(handles)
                sl = slice(off[t], off[t + 1])
                a, d, m, r = orc.replay(engine_instances(handles, pol), _policy_struct(pol, n, per_token),
                                        np.array([0, q], np.int64), I[sl], O[sl], O[sl],
                                        None if A is None else A[sl])
                assert int(res.result[t]["error"]) == int(r[0]["error"]), (policy, rate, t)
                assert res.result[t]["n_steps"] == r[0]["n_steps"], (policy, rate, t)
                assert np.array_equal(res.assign[sl], a), (policy, rate, t)
                assert np.array_equal(res.depart[sl].view(np.uint64), d.view(np.uint64)), (policy, rate, t)
                for f in ("completion_time", "peak_kv_usage", "residual_load"):
                    assert np.array_equal(res.metrics[t, :n][f].view(np.uint64), m[0][f].view(np.uint64)), f
