"""Full-scale parity against the reference itself: the drop-in's
run_continuous / run_static on the bench's own 100,000-request config-4
traces must reproduce the SimMetrics the unmodified reference produced
(tests/golden/fullscale_cases.json, made by tests/golden/make_fullscale.py
in the build container).  The smaller golden fixtures stop at 10k requests
and the bench-scale tests in test_gpu_parity.py compare with the C oracle;
these pin the 1e5-request behaviour (event loop simulator.py:272-363, the
normal predictor scheduling.py:87-95, run_static simulator.py:199-247) to
the reference's own outputs, bit for bit (float.hex digests)."""

import json
import math
import pathlib
import sys

import pytest

from helpers import sim_digest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests" / "golden"))

pytestmark = pytest.mark.gpu

CASES = json.loads((ROOT / "tests" / "golden" / "fullscale_cases.json").read_text())["cases"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"t{c['trace']}-{c['policy']}-{c['mode']}-{c['rate']}"
                         + ("-normal" if c["predictor"] else ""))
def test_fullscale_matches_reference(case):
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import simulator as S
    from paper_2504_15303_b200 import workloads as wl
    from make_fullscale import case_scenario

    rate = math.inf if case["rate"] == "inf" else float(case["rate"])
    sc = case_scenario(hs, S, wl, (case["trace"], case["policy"], rate, case["mode"], case["predictor"]))
    assert len(sc.trace) == case["q"] == 100_000
    m = S.run_static(sc) if sc.mode == "static" else S.run_continuous(sc)
    got, want = sim_digest(m), case["metrics"]
    for key in want:  # field by field, so a failure names what differs
        assert got[key] == want[key], key


C5 = json.loads((ROOT / "tests" / "golden" / "fullscale_cases.json").read_text())["config5"]


def test_config5_fullscale_matches_reference():
    """BASELINE config 5 through its own API: search_topk over the config-3
    space, then replay_candidates of top-k deployments (66-72 instances: three
    warps per trace, the retirement calendar) on the 1e5-request trace at
    rate = inf, against the reference's run_continuous of the same
    deployments (planner.py:213-228 + simulator.py:272-363)."""
    import numpy as np

    import bench
    import helpers as H
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import planner
    from paper_2504_15303_b200 import workloads as wl
    from paper_2504_15303_b200.simulator import build_instances

    cluster, _reqs, params, I3, O3 = bench.search_inputs(10_000)
    t = planner.build_tables(cluster, _reqs, params)
    top, _nf, _ms = planner.search_topk(t, 1024)
    assert [int(top["index"][c["rank"]]) for c in C5] == [c["index"] for c in C5]
    idx = np.array([c["index"] for c in C5], np.int64)
    q = C5[0]["q"]
    I1, O1 = wl.trace_lengths(q, seed=0)
    n = len(C5)
    off = np.arange(n + 1, dtype=np.int64) * q
    res = hs.replay_candidates(t, params, idx, hs.PolicyConfig(), np.arange(n), off, np.tile(I1, n), np.tile(O1, n),
                               np.tile(O1, n), want_depart=True)
    trace = [hs.Request(f"r{k}", int(I1[k]), int(O1[k]), int(O1[k])) for k in range(q)]
    for d, c in enumerate(C5):
        config = planner.deployment_of(t, int(c["index"]))
        assert {p.machine: p.tp_degree for p in config.per_machine} == c["degrees"]
        handles = build_instances(cluster, config, params)
        assert len(handles) == c["instances"]
        assert int(res.result[d]["error"]) == 0
        sl = slice(off[d], off[d + 1])
        got = H.metrics_digest(res.assign[sl], res.depart[sl], res.metrics[d][:len(handles)], handles, trace, None,
                               "OS")
        for key, want in c["metrics"].items():
            assert got[key] == want, (c["rank"], key)
