"""Single-instance planning on the GPU (hs_plan_instance: K1's scan with an
explicit KV budget) vs the reference's own plan_static_batches /
time_batches / estimate_instance_throughput (tests/golden/plan_cases.json)."""

import json
import pathlib
import random

import pytest

import paper_2504_15303_b200 as hs
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import workloads as wl

pytestmark = pytest.mark.gpu

CASES = json.loads((pathlib.Path(__file__).parent / "golden" / "plan_cases.json").read_text())


def _inputs(case):
    rng = random.Random(case["seed"])
    reqs = [hs.Request(f"q{k}", rng.randint(case["lo"], case["hi"]), rng.randint(case["lo"], case["hi"]), 1)
            for k in range(case["n"])]
    scale = float.fromhex(case["scale"])
    params = hs.LatencyParams(*(scale * x for x in wl.RANK_BASE))
    return reqs, hs.KvBudget(total_bytes=float.fromhex(case["budget"])), hs.ModelSpec(**wl.MODEL_7B), params


@pytest.fixture(scope="module")
def eng():
    return nat.engine_for(0)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_planning_matches_reference(eng, case):
    reqs, budget, model, params = _inputs(case)
    if "plan_error" in case:
        with pytest.raises(getattr(hs, case["plan_error"][0]), match=case["plan_error"][1].replace("'", ".")):
            hs.plan_static_batches(reqs, budget, model, engine=eng)
    else:
        plan = hs.plan_static_batches(reqs, budget, model, engine=eng)
        assert [list(b) for b in plan.batches] == case["batches"]
        assert [t.hex() for t in hs.time_batches(plan, reqs, params).per_batch_time] == case["times"]
    if "rate_error" in case:
        etype = ZeroDivisionError if case["rate_error"][0] == "ZeroDivisionError" else getattr(hs, case["rate_error"][0])
        with pytest.raises(etype) as ei:
            hs.estimate_instance_throughput(reqs, budget, model, params, engine=eng)
        assert str(ei.value) == case["rate_error"][1]
    else:
        assert hs.estimate_instance_throughput(reqs, budget, model, params, engine=eng).hex() == case["rate"]


def test_device_times_equal_host_time_batches(eng):
    """hs_plan_instance's per-batch seconds equal time_batches on its plan."""
    reqs, budget, model, params = _inputs(CASES[0])
    stops, times, e = eng.plan_instance(budget.total_bytes, hs.kv_bytes_per_token(model),
                                        [getattr(params, f"p{k}") for k in range(1, 9)],
                                        [r.input_len for r in reqs], [r.output_len for r in reqs])
    plan = hs.plan_static_batches(reqs, budget, model, engine=eng)
    assert [b[1] for b in plan.batches] == stops.tolist()
    assert [t.hex() for t in hs.time_batches(plan, reqs, params).per_batch_time] == [t.hex() for t in times]
