"""Fuzzed drop-in parity against the live reference (baseline/_ref, the
unmodified package, run on the host) for the edge cases the golden fixtures
do not cover: repeated request ids (in flight -> SchedulingError at the
repeat, scheduling.py:239-240; completed -> the request_times dict keeps the
first position and the last value, simulator.py:275, 337), negative and zero
step costs (the event heap's pop order, simulator.py:285-355), every policy,
rate inf and finite, continuous and static mode.  Whole SimMetrics objects are
compared with == (fp64 bit equality), exceptions by type name and message."""

import math
from dataclasses import replace
import pathlib
import random
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "hetserve" / "__init__.py").exists(),
                                 reason="baseline/_ref not vendored (python tools/vendor_reference.py)")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import hetserve
    import hetserve.simulator

    yield hetserve
    sys.path.remove(str(REF))


def _scenario(ref, rng: random.Random, case: int, wide: bool = False):
    # wide: 5-12 machines of 4 or 8 GPUs, so deployments of 33-96 instances
    # (2-3 warps per trace) exercise the multi-warp dispatch and its errors
    n_mach = rng.randint(5, 12) if wide else rng.randint(1, 3)
    # wide: small memories too (6,000 B holds ~180 tokens: instances fill up)
    mems = [6_000, 20_000, 200_000] if wide else [200_000, 400_000, 900_000]
    machines = tuple(ref.MachineSpec(f"m{i}", rng.choice([4, 8] if wide else [1, 2, 4]), rng.choice(mems), "t")
                     for i in range(n_mach))
    model = ref.ModelSpec(layers=2, hidden_dim=4, param_count=100, bytes_per_param=2)  # 32 B/token
    cluster = ref.ClusterSpec(model=model, engine=ref.EngineOverheads(1.0, 0), machines=machines,
                              limits=ref.WorkloadLimits(max_input_len=64, max_output_len=64))
    kind = case % 4
    params = {}
    for m in machines:
        for t in ref.enumerate_tp_degrees(m):
            p = [rng.uniform(1e-5, 1e-3), rng.uniform(1e-4, 1e-2), rng.uniform(1e-6, 1e-4), rng.uniform(1e-3, 1e-2),
                 rng.uniform(1e-7, 1e-5), rng.uniform(1e-5, 1e-3), rng.uniform(1e-7, 1e-5), rng.uniform(1e-4, 1e-3)]
            if kind == 1:  # negative decode terms: step costs can go negative
                p[7] = -rng.uniform(1e-3, 2e-2)  # short steps of small batches cost < 0
                if wide and rng.random() < 0.3:  # per-request costs <= 0 for some classes
                    p[1], p[7] = 0.0, -rng.uniform(0.05, 0.5)
            elif kind == 2:  # constant-only prefill, zero decode: many steps at one time
                p = [0.0, rng.choice([1.0, 0.5]), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0]
            params[(m.name, t)] = ref.LatencyParams(*p)
    degrees = {m.name: (1 if wide and rng.random() < 0.7 else rng.choice(ref.enumerate_tp_degrees(m)))
               for m in machines}
    config = ref.deployment_for(machines, degrees)
    q = rng.randint(20, 250)
    ids = [f"r{k}" for k in range(q)]
    if kind == 3 or rng.random() < 0.2:  # repeated ids
        for _ in range(rng.randint(1, 4)):
            a, b = sorted(rng.sample(range(q), 2))
            ids[b] = ids[a]
    trace = tuple(ref.Request(ids[k], rng.randint(1, 64), o, o) for k, o in
                  ((k, rng.randint(1, 64)) for k in range(q)))
    policy_name = rng.choice(["OS", "OS", "RR", "WRR", "SI", "MB"])
    n_inst = sum(p.instance_count for p in config.per_machine)
    wrr = tuple(float(rng.randint(1, 4)) for _ in range(n_inst)) if policy_name == "WRR" else None
    # theta 2000: exp(theta * usage) overflows once an instance is ~36 % full
    policy = ref.PolicyConfig(policy=policy_name, theta=rng.choice([0.5, 2.0, 2000.0] if wide else [0.5, 2.0]),
                              wrr_weights=wrr)
    mode = "static" if rng.random() < 0.2 else "continuous"
    rate = math.inf if (mode == "static" or rng.random() < 0.3) else rng.choice([5.0, 40.0, 400.0])
    return ref.simulator.Scenario(cluster=cluster, config=config, trace=trace, arrival_rate=rate, policy=policy,
                                  mode=mode, seed=rng.randint(0, 99), params=params)


def _outcome(fn, scenario):
    try:
        return "ok", fn(scenario)
    except Exception as exc:  # noqa: BLE001 -- compared by type name and message
        return "err", (type(exc).__name__, str(exc))


def test_fuzzed_scenarios_match_live_reference(ref):
    from paper_2504_15303_b200 import refbind

    binding = refbind.bindings(ref)
    S = sys.modules["hetserve.simulator"]
    ours = {name: fn for (mod, name), fn in binding.items() if mod is S}
    n_dup = n_err = n_neg = 0
    for case in range(240):
        rng = random.Random(case)
        sc = _scenario(ref, rng, case)
        run_ref = S.run_static if sc.mode == "static" else S.run_continuous
        run_gpu = ours["run_static"] if sc.mode == "static" else ours["run_continuous"]
        want = _outcome(run_ref, sc)
        got = _outcome(run_gpu, sc)
        assert got == want, (case, sc.mode, sc.policy.policy, sc.arrival_rate, want[1] if want[0] == "err" else "",
                             got[1] if got[0] == "err" else "")
        n_dup += len({r.id for r in sc.trace}) < len(sc.trace)
        n_err += want[0] == "err"
        n_neg += case % 4 == 1 and want[0] == "ok"
    assert n_dup > 40 and n_err > 10 and n_neg > 20, (n_dup, n_err, n_neg)


def test_fuzzed_wide_scenarios_match_live_reference(ref):
    """As above on deployments of 33-96 instances (multi-warp traces: the
    fused one-barrier OS / MB dispatch, the exchanged SI / RR / WRR choice,
    and their error paths)."""
    from paper_2504_15303_b200 import refbind

    binding = refbind.bindings(ref)
    S = sys.modules["hetserve.simulator"]
    ours = {name: fn for (mod, name), fn in binding.items() if mod is S}
    n_err = n_wide = 0
    kinds = set()
    for case in range(1000, 1160):
        rng = random.Random(case)
        sc = _scenario(ref, rng, case, wide=True)
        n_inst = sum(p.instance_count for p in sc.config.per_machine)
        run_ref = S.run_static if sc.mode == "static" else S.run_continuous
        run_gpu = ours["run_static"] if sc.mode == "static" else ours["run_continuous"]
        want = _outcome(run_ref, sc)
        got = _outcome(run_gpu, sc)
        assert got == want, (case, n_inst, sc.mode, sc.policy.policy, sc.arrival_rate,
                             want[1] if want[0] == "err" else "", got[1] if got[0] == "err" else "")
        n_wide += n_inst > 32
        if want[0] == "err":
            n_err += 1
            kinds.add(want[1][0])
    assert n_wide > 100 and n_err > 10, (n_wide, n_err, kinds)


def test_run_policy_comparison_matches_live_reference(ref):
    """run_policy_comparison (simulator.py:372-380): every policy on the
    identical arrival / prediction realisation, the reference's own function
    routed through the engine vs the unmodified one, normal predictor
    included (scheduling.py:87-95)."""
    from paper_2504_15303_b200 import refbind

    S = sys.modules["hetserve.simulator"]
    ours = {name: fn for (mod, name), fn in refbind.bindings(ref).items() if mod is S}
    n = 0
    for case in range(400, 430):
        rng = random.Random(case)
        sc = _scenario(ref, rng, 4 * case)  # kind 0: plain coefficients
        ids = [f"r{k}" for k in range(len(sc.trace))]  # unique ids: compare metrics, not errors
        trace = tuple(ref.Request(i, r.input_len, r.output_len, r.predicted_output_len) for i, r in zip(ids, sc.trace))
        n_inst = sum(p.instance_count for p in sc.config.per_machine)
        pred = ref.PredictorConfig(mode="normal", mean=30.0, stddev=12.0, seed=case) if case % 2 else \
            ref.PredictorConfig()
        pol = ref.PolicyConfig(policy="OS", theta=2.0, wrr_weights=tuple(float(1 + k % 3) for k in range(n_inst)),
                               predictor=pred)
        sc = replace(sc, trace=trace, policy=pol)
        names = ["OS", "RR", "WRR", "SI", "MB"]
        want = _outcome(lambda s: S.run_policy_comparison(s, names), sc)
        # the reference's own run_policy_comparison, with run_continuous / run_static routed to the engine
        saved = (S.run_continuous, S.run_static)
        S.run_continuous, S.run_static = ours["run_continuous"], ours["run_static"]
        try:
            got = _outcome(lambda s: S.run_policy_comparison(s, names), sc)
        finally:
            S.run_continuous, S.run_static = saved
        assert got == want, case
        n += want[0] == "ok"
    assert n >= 20
