"""Pin the C oracle (oracle/hs_oracle.c) to outputs of the reference itself.

tests/golden/*.json were produced by tests/golden/make_golden.py running the
unmodified reference package; every float is compared bit for bit.
"""

import json
import math
import pathlib
import random
import sys

import numpy as np
import pytest

import helpers as H
import paper_2504_15303_b200 as hs
from oracle import hs_oracle as orc
from paper_2504_15303_b200 import _native as nat


def test_exp_matches_math_exp_bitwise():
    g = H.load("exp_vectors.json")
    for xs, ys in zip(g["x"], g["y"]):
        y, of = orc.exp(float.fromhex(xs))
        assert not of
        assert y.hex() == ys, (xs, y.hex(), ys)
    for xs in g["overflow"]:
        _y, of = orc.exp(float.fromhex(xs))
        assert of


def test_exp_matches_live_math_exp():
    rng = np.random.default_rng(11)
    for x in rng.uniform(0, 709.0, 20000).tolist() + rng.uniform(0, 3, 20000).tolist():
        y, of = orc.exp(x)
        assert y == math.exp(x) and not of


def test_floordiv_and_sum_match_cpython():
    rng = random.Random(3)
    for _ in range(20000):
        a = rng.uniform(1.0, 1e13)
        b = float(rng.randint(1, 10**10))
        assert orc.floordiv(a, b) == a // b
    for _ in range(2000):
        xs = [rng.uniform(-1, 1) * 10 ** rng.randint(-5, 16) for _ in range(rng.randint(1, 40))]
        assert orc.pysum(xs) == sum(xs)
    assert orc.pysum([1e16, 1.0, -1e16]) == 1.0


SEARCH = H.load("search_cases.json")


@pytest.mark.parametrize("case", [c for c in SEARCH if c["kind"] == "search"], ids=lambda c: c["name"])
def test_oracle_search_matches_reference(case):
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    requests = H.search_trace(case)
    model, engine, limits, machines, params, present = H.search_structs(cluster, params_by)
    I = np.array([r.input_len for r in requests], np.int32)
    O = np.array([r.output_len for r in requests], np.int32)
    table, nd = orc.tables(model, engine, limits, machines, params, present, I, O)
    H.check_table(case, table, nd, requests)
    if "ranked" not in case and "error" not in case:
        return
    if "error" in case:
        zd = (table["status"] == nat.ENTRY_ZERO_DIVISION).any()
        assert zd and case["error"]["type"] == "ZeroDivisionError"
        return
    ranked, first_bad = orc.rank(table, nd)
    assert len(ranked) == len(case["ranked"])
    degs = [hs.enumerate_tp_degrees(m) for m in cluster.machines]
    for got, want in zip(ranked, case["ranked"]):
        x, digits = int(got["index"]), []
        for d in reversed(nd.tolist()):
            digits.append(x % d)
            x //= d
        digits.reverse()
        assert [degs[i][d] for i, d in enumerate(digits)] == want["degrees"]
        assert float(got["total"]).hex() == want["total"]
    bad = np.nonzero(first_bad >= 0)[0]
    assert len(bad) == len(case["infeasible"])
    b_total, b_idx, n_feas = orc.best(table, nd, 0, int(np.prod(nd.astype(np.int64))), nthreads=2)
    if case["ranked"]:
        assert b_idx == int(ranked[0]["index"]) and b_total == float(ranked[0]["total"])
    assert n_feas == len(case["ranked"])


def test_oracle_literal_candidates_match_reference_samples():
    case = next(c for c in SEARCH if c["name"] == "config3_samples")
    cluster = H.cluster_from(case["profile"])
    params_by = H.params_from(case["profile"])
    I, O = hs.workloads.trace_lengths(10_000, seed=3) if hasattr(hs, "workloads") else (None, None)
    from paper_2504_15303_b200 import workloads as wl
    I, O = wl.trace_lengths(10_000, seed=3)
    model, engine, limits, machines, params, present = H.search_structs(cluster, params_by)
    table, nd = orc.tables(model, engine, limits, machines, params, present, I, O)
    n_ok = 0
    for idx, total_hex, reason in case["samples"]:
        t, fb, st = orc.candidate_literal(model, engine, limits, machines, params, present, I, O, idx)
        if total_hex is None:
            assert fb >= 0
        else:
            n_ok += 1
            assert fb < 0 and t.hex() == total_hex
            # the table decomposition gives the same total
            x, acc = idx, []
            for d in reversed(nd.tolist()):
                acc.append(x % d)
                x //= d
            acc.reverse()
            s = 0.0
            for i, d in enumerate(acc):
                s = s + float(table[i, d]["contribution"])
            assert s.hex() == total_hex
    assert n_ok >= 20


REPLAY = H.load("replay_cases.json") + H.load("static_cases.json") + H.load("wide_cases.json")
REPLAY_PARAMS = [(c, k) for c in REPLAY for k in range(len(c["results"]))]


@pytest.mark.parametrize("case,k", REPLAY_PARAMS, ids=lambda v: v["name"] if isinstance(v, dict) else str(v))
def test_oracle_replay_matches_reference(case, k):
    want = case["results"][k]
    sc = H.scenario_from(case, want["policy"])
    inst, pol, handles, I, O, P, T = H.replay_structs(sc)
    offsets = np.array([0, len(I)], np.int64)
    assign, depart, metrics, result = orc.replay(inst, pol, offsets, I, O, P, T)
    if "error" in want:
        assert int(result[0]["error"]) != nat.TRACE_OK, want
        exp_err = {"InfeasibleRequestError": nat.TRACE_INFEASIBLE_REQUEST, "OverflowError": nat.TRACE_EXP_OVERFLOW,
                   "SpecError": nat.TRACE_NONPOSITIVE_COST, "SchedulingError": nat.TRACE_NO_INSTANCE}[want["error"]]
        assert int(result[0]["error"]) == exp_err
        return
    assert int(result[0]["error"]) == nat.TRACE_OK
    got = H.metrics_digest(assign, depart, metrics[0], handles, sc.trace, T, want["policy"],
                           static=sc.mode == "static")
    for key in ("assign_head", "assign_sha", "makespan", "per_instance", "residual_loads", "depart_sha",
                "times_sha", "times_head", "throughput", "spread"):
        assert got[key] == want[key], (case["name"], want["policy"], key)


@pytest.mark.parametrize("case", [c for c in SEARCH if c["kind"] == "search" and c.get("ranked")],
                         ids=lambda c: c["name"])
def test_oracle_topk_is_head_of_reference_ranking(case):
    cluster = H.cluster_from(case["profile"])
    requests = H.search_trace(case)
    model, engine, limits, machines, params, present = H.search_structs(cluster, H.params_from(case["profile"]))
    I = np.array([r.input_len for r in requests], np.int32)
    O = np.array([r.output_len for r in requests], np.int32)
    table, nd = orc.tables(model, engine, limits, machines, params, present, I, O)
    k = max(1, len(case["ranked"]) // 2)
    top, nf = orc.topk(table, nd, k)
    assert nf == len(case["ranked"])
    assert [float(x).hex() for x in top["total"]] == [r["total"] for r in case["ranked"][:k]]
    # shards merge to the same head
    parts = [orc.topk(table, nd, k, s, 3)[0] for s in range(3)]
    from paper_2504_15303_b200.planner import merge_topk
    merged = merge_topk(parts, k)
    assert merged["index"].tolist() == top["index"].tolist()


FULLSCALE = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "fullscale_cases.json").read_text())["cases"]


@pytest.mark.parametrize("case", FULLSCALE, ids=lambda c: f"t{c['trace']}-{c['policy']}-{c['mode']}-{c['rate']}")
def test_oracle_fullscale_matches_reference(case):
    """The C oracle on the bench's own 1e5-request traces against the
    reference's outputs (tests/golden/make_fullscale.py): the bench-scale GPU
    parity tests that use the oracle as checker rest on this pin."""
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent / "golden"))
    from make_fullscale import case_scenario
    from paper_2504_15303_b200 import simulator as S
    from paper_2504_15303_b200 import workloads as wl

    rate = math.inf if case["rate"] == "inf" else float(case["rate"])
    sc = case_scenario(hs, S, wl, (case["trace"], case["policy"], rate, case["mode"], case["predictor"]))
    inst, pol, handles, I, O, P, T = H.replay_structs(sc)
    assign, depart, metrics, result = orc.replay(inst, pol, np.array([0, len(I)], np.int64), I, O, P, T)
    assert int(result[0]["error"]) == nat.TRACE_OK
    want = case["metrics"]
    got = H.metrics_digest(assign, depart, metrics[0], handles, sc.trace, T, want["policy"],
                           static=sc.mode == "static")
    for key in ("assign_head", "assign_sha", "makespan", "per_instance", "residual_loads", "depart_sha",
                "times_sha", "times_head", "throughput", "spread"):
        assert got[key] == want[key], key


C5 = json.loads((pathlib.Path(__file__).resolve().parent / "golden" / "fullscale_cases.json").read_text())["config5"]


@pytest.mark.parametrize("c", C5, ids=lambda c: f"rank{c['rank']}")
def test_oracle_config5_fullscale_matches_reference(c):
    """Config-5 deployments (66-72 instances) on the 1e5-request trace at
    rate = inf: the C oracle against the reference's run_continuous."""
    import bench
    from paper_2504_15303_b200 import workloads as wl
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances

    cluster, _reqs, params, _I, _O = bench.search_inputs(16)
    config = hs.deployment_for(cluster.machines, c["degrees"])
    handles = build_instances(cluster, config, params)
    assert len(handles) == c["instances"]
    I1, O1 = wl.trace_lengths(c["q"], seed=0)
    pol = hs.PolicyConfig()
    assign, depart, metrics, result = orc.replay(
        engine_instances(handles, pol), _policy_struct(pol, len(handles), hs.kv_bytes_per_token(cluster.model)),
        np.array([0, c["q"]], np.int64), I1, O1, O1, None)
    assert int(result[0]["error"]) == nat.TRACE_OK
    trace = [hs.Request(f"r{k}", int(I1[k]), int(O1[k]), int(O1[k])) for k in range(c["q"])]
    got = H.metrics_digest(assign, depart, metrics[0], handles, trace, None, "OS")
    for key, want in c["metrics"].items():
        assert got[key] == want, key
