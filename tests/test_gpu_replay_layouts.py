"""K3 kernel configurations vs the oracle, bit for bit: the default
one-warp-per-trace kernel (replay.cu) and the opt-in interval-bound kernel
(replay_mt.cu, HS_REPLAY_MT=1) at 8 / 16 / 32 lanes per trace, with its
bounds as built and artificially widened (HS_REPLAY_WIDEN: many event orders
and admission steps are then settled by the exact clock chain instead of
the bounds).
Each configuration runs in its own process (the library reads the
environment once)."""

import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

MT = {"HS_REPLAY_MT": "1"}
CONFIGS = [
    ({**MT, "HS_REPLAY_LANES": "8"}, 32),
    ({**MT, "HS_REPLAY_LANES": "16"}, 32),
    ({**MT, "HS_REPLAY_LANES": "32"}, 32),
    ({**MT, "HS_REPLAY_LANES": "8"}, 9),
    ({**MT, "HS_REPLAY_LANES": "16"}, 17),
    ({**MT, "HS_REPLAY_LANES": "8", "HS_REPLAY_WIDEN": "1e6"}, 32),
    ({**MT, "HS_REPLAY_LANES": "32", "HS_REPLAY_WIDEN": "1e7"}, 24),
    ({}, 32),
]


@pytest.mark.parametrize("env,n_inst", CONFIGS, ids=lambda x: str(x))
def test_replay_configuration_vs_oracle(env, n_inst):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "replay_check.py"), "40", "3000", str(n_inst)], env=e,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
