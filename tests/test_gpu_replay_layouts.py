"""The replay kernel vs the C oracle, bit for bit, on 40 ragged
config-4-shaped traces at five arrival rates (incl. rate = inf and an empty
trace), all five policies, with and without departure times, at 32 and 9
instances (one warp per trace, lanes left idle): assignments, departures,
metrics and step-event counts.  Runs in its own process (tests/replay_check.py)."""

import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pipe", ["0", "1"])
@pytest.mark.parametrize("n_inst", [32, 9])
def test_replay_vs_oracle_all_policies(n_inst, pipe):
    """pipe: HS_REPLAY_PIPE forces either one-warp pure-step loop (the launch
    picks by traces per SM: the pipelined one below 8 per SM)."""
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "replay_check.py"), "40", "3000", str(n_inst)],
                       env=dict(os.environ, HS_REPLAY_PIPE=pipe), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
