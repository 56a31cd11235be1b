"""Host-side logic of the drop-in (no GPU): C-ABI exports, domain types,
error messages, sharding helpers, predictor semantics."""

import math
import pathlib
import re
import sys

import numpy as np
import pytest

import paper_2504_15303_b200 as hs
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import planner
from paper_2504_15303_b200.simulator import engine_instances

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = pathlib.Path("/root/reference/pkg/src")


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "hetserve_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(hs_\w+)\(", header, re.M))
    assert {"hs_search_tables", "hs_search_best", "hs_replay"} <= declared
    lib = nat.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(nat.EXPORTS) == declared
    assert lib.hs_abi_version() == 4


def test_no_cuda_means_engine_unavailable_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nat.EngineUnavailable):
        nat.Engine(0)
    # the product never imports the oracle
    for f in (ROOT / "paper_2504_15303_b200").rglob("*.py"):
        src = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(nat.hs_entry) == nat.ENTRY_DTYPE.itemsize == 72
    assert C.sizeof(nat.hs_inst_metrics) == nat.METRICS_DTYPE.itemsize == 40
    assert C.sizeof(nat.hs_trace_result) == nat.RESULT_DTYPE.itemsize == 32
    assert C.sizeof(nat.hs_instance) == 88
    assert C.sizeof(nat.hs_machine) == 24
    assert C.sizeof(nat.hs_pcg64_state) == nat.PCG64_DTYPE.itemsize == 40
    assert C.sizeof(nat.hs_dist) == 40
    assert C.sizeof(nat.hs_replay_seeds) == 48


def test_domain_known_answers():
    m = hs.MachineSpec("m", 8, 32_000_000_000)
    assert hs.enumerate_tp_degrees(m) == [1, 2, 4, 8]
    assert hs.enumerate_tp_degrees(hs.MachineSpec("a", 6, 1)) == [1, 2]
    assert hs.enumerate_tp_degrees(hs.MachineSpec("a", 12, 1)) == [1, 2, 4]
    model = hs.ModelSpec(32, 4096, 8_000_000_000, 2)
    ovh = hs.EngineOverheads(0.9, 2_000_000_000)
    assert hs.kv_budget(m, 2, model, ovh).total_bytes == pytest.approx(39.6e9, rel=1e-12)
    assert hs.kv_bytes_per_token(model) == 524288
    v = hs.check_memory_constraint(hs.kv_budget(m, 1, model, ovh), hs.WorkloadLimits(4096, 4096), model)
    assert v.feasible and v.required_bytes == 524288 * 8192
    v = hs.check_memory_constraint(hs.kv_budget(hs.MachineSpec("s", 1, 16_000_000_000), 1, model, ovh),
                                   hs.WorkloadLimits(4096, 4096), model)
    assert not v.feasible and v.slack_bytes < 0
    with pytest.raises(hs.SpecError):
        hs.ModelSpec(0, 1, 1, 1)
    with pytest.raises(hs.SpecError):
        hs.EngineOverheads(1.5, 0)
    with pytest.raises(hs.SpecError, match="does not divide"):
        hs.deployment_for((m,), {"m": 3})
    with pytest.raises(hs.SpecError):
        hs.PolicyConfig(policy="WRR")
    with pytest.raises(hs.SpecError):
        hs.Scenario(hs.ClusterSpec(model, ovh, (m,), hs.WorkloadLimits(1, 1)), None, (), 1.0, hs.PolicyConfig(),
                    "continuous", 0, {})


def test_latency_model_expression_order():
    p = hs.LatencyParams(1e-5, 1e-3, 2e-5, 5e-3, 1e-6, 1e-4, 1e-7, 1e-5)
    assert hs.prefill_time(p, 3, 17) == ((((1e-5 * 3) * 17) + (1e-3 * 3)) + (2e-5 * 17)) + 5e-3
    assert hs.decode_time(p, 2, 10, 4) == ((1e-6 * 2 + 1e-7) * (4 * 10 + 4 * 5 / 2.0)) + ((1e-4 * 2 + 1e-5) * 4)


def _table(rows):
    """rows: list per machine of (status, contribution)."""
    M = len(rows)
    t = np.zeros((M, nat.HS_MAX_DEGREES), nat.ENTRY_DTYPE)
    nd = np.zeros(M, np.int32)
    for i, row in enumerate(rows):
        nd[i] = len(row)
        for d, (st, c) in enumerate(row):
            t[i, d]["status"] = st
            t[i, d]["contribution"] = c
    return t, nd


def test_fatal_zero_division_rule():
    ok, zd, bad = nat.ENTRY_OK, nat.ENTRY_ZERO_DIVISION, nat.ENTRY_INFEASIBLE_CONFIG
    cluster = hs.ClusterSpec(hs.ModelSpec(1, 1, 1, 1), hs.EngineOverheads(1.0, 0),
                             (hs.MachineSpec("a", 2, 1), hs.MachineSpec("b", 2, 1)), hs.WorkloadLimits(1, 1))

    def tables(rows):
        t, nd = _table(rows)
        return planner.SearchTables(cluster, [], ["a", "b"], [[1, 2], [1, 2]], t, nd)

    assert isinstance(planner._fatal_zero_division(tables([[(ok, 1.0), (zd, 0)], [(ok, 1.0), (ok, 2.0)]])),
                      ZeroDivisionError)
    # machine 0 has no OK degree: every candidate fails on machine 0 first
    assert planner._fatal_zero_division(tables([[(bad, 0), (bad, 0)], [(zd, 0), (ok, 2.0)]])) is None
    assert isinstance(planner._fatal_zero_division(tables([[(ok, 1.0), (bad, 0)], [(zd, 0), (ok, 2.0)]])),
                      ZeroDivisionError)


def test_instance_classes_dedupe_bit_identical():
    p = hs.LatencyParams(*([1e-4] * 8))
    q = hs.LatencyParams(*([1e-4] * 7 + [2e-4]))
    hh = [hs.InstanceHandle(f"i{k}", "m", 1, p if k % 2 else q, hs.KvBudget(1e9 if k < 4 else 2e9))
          for k in range(8)]
    arr = engine_instances(hh, hs.PolicyConfig())
    types = [arr[k].type for k in range(8)]
    assert types == [0, 1, 0, 1, 2, 3, 2, 3]


def test_predictor_modes():
    O = np.array([5, 7, 9], np.int64)
    o = hs.OutputLengthPredictor(hs.PredictorConfig(), 100).predict_lengths(O)
    assert o.tolist() == [5, 7, 9]
    m = hs.OutputLengthPredictor(hs.PredictorConfig(mode="mean", mean=99.5), 100).predict_lengths(O)
    assert m.tolist() == [100, 100, 100]  # round half to even
    n = hs.OutputLengthPredictor(hs.PredictorConfig(mode="normal", mean=10, stddev=50, seed=3), 40)
    d = n.predict_lengths(np.zeros(400, np.int64))
    assert d.min() == 1 and d.max() <= 40


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_predictor_stream_equals_reference_per_call():
    sys.path.insert(0, str(REF))
    import hetserve as ref
    cfg = ref.PredictorConfig(mode="normal", mean=150, stddev=60, seed=7)
    rp = ref.OutputLengthPredictor(cfg, 1024)
    r = ref.Request("x", 1, 1, 1)
    want = [rp.predict(r) for _ in range(5000)]
    got = hs.OutputLengthPredictor(hs.PredictorConfig("normal", 150, 60, 7), 1024).predict_lengths(
        np.zeros(5000, np.int64))
    assert got.tolist() == want


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_workload_generators_match_reference_semantics():
    sys.path.insert(0, str(REF))
    import hetserve as ref
    from paper_2504_15303_b200 import workloads as wl
    trace = [ref.Request(f"r{k}", 1, 1, 1) for k in range(3000)]
    want = [t for _r, t in ref.generate_arrivals(trace, 37.5, 11)]
    assert wl.arrivals(3000, 37.5, 11).tolist() == want
    assert hs.simulator.arrival_times(3000, math.inf, 0).tolist() == [0.0] * 3000


def test_scalar_helpers_match_reference():
    """capacity.py / scheduling.py scalar helpers (host), against the
    reference itself where it is importable."""
    if not REF.exists():
        pytest.skip("reference not present")
    import sys
    sys.path.insert(0, str(REF))
    import hetserve as ref
    import random
    from paper_2504_15303_b200 import workloads as wl
    rng = random.Random(3)
    for mod in (hs, ref):
        assert mod.ideal_batch_size and mod.per_request_cost and mod.workload and mod.kv_usage
    for _ in range(300):
        I, P = rng.randint(1, 5000), rng.randint(1, 5000)
        budget = rng.uniform(-1e9, 1e11)
        params = tuple(rng.uniform(-1e-4, 1e-3) for _ in range(8))
        ours, theirs = [], []
        for mod, out in ((hs, ours), (ref, theirs)):
            model = mod.ModelSpec(**wl.MODEL_7B)
            kb = mod.KvBudget(total_bytes=budget)
            req = mod.Request("x", I, P, P)
            lp = mod.LatencyParams(*params)
            for fn in (lambda: mod.ideal_batch_size(req, kb, model),
                       lambda: mod.request_oversized(req, kb, model),
                       lambda: mod.per_request_cost(lp, req, rng_b),
                       lambda: mod.workload(abs(params[0]) * 1e3, I / 5000, 2.0 + params[1]),
                       lambda: mod.kv_usage(_running(mod, I, P), model, kb)):
                try:
                    v = fn()
                    out.append(("ok", v.hex() if isinstance(v, float) else v))
                except Exception as exc:  # noqa: BLE001
                    out.append((type(exc).__name__, str(exc)))
        assert ours == theirs
    rt = hs.RunningTokens()
    rt.add(3, 4)
    rt.remove(3, 4)
    with pytest.raises(hs.SpecError, match="completion applied twice"):
        rt.remove(1, 0)


rng_b = 7


def _running(mod, i, p):
    r = mod.RunningTokens()
    r.add(i, p)
    return r
