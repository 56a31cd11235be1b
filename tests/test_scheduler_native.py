"""The native live scheduler (csrc/scheduler.cpp, hs_sched_*) vs the
reference's own Scheduler (scheduling.py:175-346): every recorded choose /
complete / evaluate call of tests/golden/sched_cases.json is replayed and its
result or exception (type and message) and the snapshot after it are
compared exactly (float.hex).  Host code: runs without a GPU."""

from __future__ import annotations

import json
import pathlib
import threading

import pytest

import helpers as H
import paper_2504_15303_b200 as hs
from paper_2504_15303_b200 import simulator

CASES = json.loads((pathlib.Path(__file__).parent / "golden" / "sched_cases.json").read_text())


def _scheduler(case):
    cluster = H.cluster_from(case["profile"])
    params = H.params_from(case["profile"])
    cfg = hs.deployment_for(cluster.machines, case["degrees"])
    handles = simulator.build_instances(cluster, cfg, params)
    pol = case["policy"]
    wrr = pol.get("wrr")
    if wrr == "auto":
        wrr = [1 + (7 * j) % 5 for j in range(len(handles))]
    policy = hs.PolicyConfig(policy=pol["policy"], theta=pol.get("theta", 2.0),
                             wrr_weights=tuple(wrr) if wrr else None)
    return hs.Scheduler(handles, cluster.model, policy)


def _snap(sch) -> dict:
    s = sch.snapshot()
    return {"loads": [v.hex() for v in s["loads"].values()], "kv_usage": [v.hex() for v in s["kv_usage"].values()],
            "running": list(s["running_tokens"].values()), "oversized": list(s["oversized"].values()),
            "in_flight": s["in_flight"]}


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_scheduler_matches_reference(case):
    sch = _scheduler(case)
    for k, op in enumerate(case["ops"]):
        allowed = set(op["allowed"]) if op.get("allowed") is not None else None
        got = {}
        try:
            if op["op"] == "complete":
                sch.complete(op["id"])
            else:
                req = hs.Request(op["id"], op["I"], op["P"], op["P"])
                if op["op"] == "choose":
                    got["chosen"] = sch.choose(req, allowed)
                else:
                    got["weights"] = [w.hex() for w in sch.evaluate(req, allowed)]
        except (hs.HetserveError, OverflowError, ZeroDivisionError) as exc:
            got["error"], got["msg"] = type(exc).__name__, str(exc)
        want = {key: op[key] for key in ("chosen", "weights", "error", "msg") if key in op}
        assert got == want, (case["name"], k, op)
        assert _snap(sch) == op["snap"], (case["name"], k, op)


def test_constructor_checks_match_reference():
    case = CASES[0]
    cluster = H.cluster_from(case["profile"])
    params = H.params_from(case["profile"])
    handles = simulator.build_instances(cluster, hs.deployment_for(cluster.machines, case["degrees"]), params)
    with pytest.raises(hs.SchedulingError, match="scheduler needs at least one instance"):
        hs.Scheduler([], cluster.model)
    with pytest.raises(hs.SpecError, match=r"WRR needs one weight per instance \(16\), got 2"):
        hs.Scheduler(handles, cluster.model, hs.PolicyConfig(policy="WRR", wrr_weights=(1.0, 2.0)))
    sch = hs.Scheduler(handles, cluster.model)
    assert sch.policy.policy == "OS" and len(sch.instances) == 16 and sch.in_flight_count() == 0


def test_concurrent_choose_complete_is_consistent():
    """choose/complete from many threads (the gateway's use): bookkeeping
    returns exactly to zero load and zero running tokens."""
    sch = _scheduler(CASES[0])

    def worker(t):
        for i in range(300):
            rid = f"t{t}-{i}"
            sch.choose(hs.Request(rid, 10 + i % 50, 20, 20 + i % 7))
            if i % 3 == 2:
                sch.complete(rid)
        for i in range(300):
            if i % 3 != 2:
                sch.complete(f"t{t}-{i}")

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert sch.in_flight_count() == 0
    assert all(v == 0 for v in sch.running_totals())
