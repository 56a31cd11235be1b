"""The reference's own test-suite, unmodified, against the engine.

SURVEY.md section 4 item 5: run /root/reference/pkg/tests with the reference's
hot-path entry points routed through the engine (paper_2504_15303_b200.refbind,
INTEGRATION.md section 2): search_optimal_config, estimate_system_throughput,
plan_static_batches, estimate_instance_throughput (planner.py), run_continuous
and run_static -- and through them run_scenario / run_policy_comparison --
(simulator.py), plus the native Scheduler (scheduling.py:175-346) for the
scheduler / gateway files.  The vendored copy lives in baseline/_ref
(tools/vendor_reference.py; git-ignored, shipped to the GPU box by gpurun).
"""

import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.skipif(not (REF / "tests" / "conftest.py").exists(),
                                reason="baseline/_ref not vendored (python tools/vendor_reference.py)")


def _run(files, scheduler: bool):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests"), str(ROOT), env.get("PYTHONPATH", "")])
    env["HS_REFBIND_SCHEDULER"] = "1" if scheduler else "0"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "refsuite_plugin", *files]
    r = subprocess.run(cmd, cwd=REF / "tests", env=env, capture_output=True, text=True, timeout=1800)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_planner_simulator_acceptance_through_engine():
    """test_planner.py, test_simulator.py, test_acceptance.py (criteria 1-8)
    and test_cli.py (hetserve plan / simulate / compare, incl. the plan
    report's byte stability) with the search and both simulator modes on the
    GPU."""
    rc, out = _run(["test_planner.py", "test_simulator.py", "test_acceptance.py", "test_cli.py"], scheduler=False)
    assert rc == 0, out[-6000:]
    assert " failed" not in out and "[criterion 8] PASS" in out, out[-3000:]


@pytest.mark.gpu
def test_reference_scheduler_and_gateway_through_native_scheduler():
    """test_scheduling.py and test_gateway.py with hetserve.scheduling.Scheduler
    replaced by the native one (its _states view included), plus the
    acceptance suite again (criterion 7 drives the gateway)."""
    rc, out = _run(["test_scheduling.py", "test_gateway.py", "test_acceptance.py", "test_simulator.py",
                    "test_planner.py"], scheduler=True)
    assert rc == 0, out[-6000:]


def test_reference_suite_collects_with_binding():
    """CPU: the binding installs and every reference test module imports."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests"), str(ROOT), env.get("PYTHONPATH", "")])
    env["HS_REFBIND_SCHEDULER"] = "1"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "--collect-only", "-p", "no:cacheprovider", "-p",
                        "refsuite_plugin", "."], cwd=REF / "tests", env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "167 tests collected" in r.stdout, r.stdout[-1000:]
