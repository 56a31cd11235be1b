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
