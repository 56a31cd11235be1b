"""hetserve plan --out byte-identity (reference
cli.py:70-109 _plan_records + cmd_plan, tests/test_cli.py:166-188): the
reference's own report writer applied to the engine's SearchOutcome
(through refbind) produces the same bytes as applied to the unmodified
reference's search, on BASELINE configs 1 and 2 and on a 16,384-candidate
synthetic space with mixed feasibility (a short trace keeps the reference's
own search to seconds)."""

import json
import pathlib
import sys

import pytest

import paper_2504_15303_b200.workloads as wl

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "hetserve" / "__init__.py").exists(),
                                 reason="baseline/_ref not vendored (python tools/vendor_reference.py)")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import hetserve
    import hetserve.cli
    yield hetserve
    sys.path.remove(str(REF))


def _inputs(ref, prof, q, seed):
    cluster = ref.ClusterSpec(model=ref.ModelSpec(**prof.model), engine=ref.EngineOverheads(**prof.engine),
                              machines=tuple(ref.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                              limits=ref.WorkloadLimits(**prof.limits))
    params = {k: ref.LatencyParams(*v) for k, v in prof.params.items()}
    I, O = wl.trace_lengths(q, seed=seed)
    trace = [ref.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q)]
    return cluster, trace, params


def _synthetic():
    """7 machines x 8 GPUs (4 degrees each: 4^7 = 16384 candidates), memory
    sizes that make some degrees infeasible, one machine without params at t=8."""
    mems = {"a": 24, "b": 32, "c": 40, "d": 48, "e": 80, "f": 24, "g": 141}
    prof = wl.ClusterProfile("synthetic", dict(wl.MODEL_13B), dict(wl.ENGINE), dict(wl.LIMITS),
                             [(f"m{n}", 8, gb * 1_000_000_000, "v100") for n, gb in mems.items()])
    for k, (name, count, _m, _a) in enumerate(prof.machines):
        for t in wl.enumerate_degrees(count):
            if name == "mc" and t == 8:
                continue
            prof.params[(name, t)] = wl.scaled_params(wl.RANK_BASE, t ** -wl.TP_ALPHA * (1.0 + 0.1 * k))
    return prof


@pytest.mark.parametrize("which", ["config1", "config2", "synthetic"])
def test_plan_report_bytes_match_reference(ref, which):
    from paper_2504_15303_b200 import refbind

    P = sys.modules["hetserve.planner"]
    cli = sys.modules["hetserve.cli"]
    if which == "config1":
        prof, q = wl.config1(), 2000
    elif which == "config2":
        prof, q = wl.config2(), 1000
    else:
        prof, q = _synthetic(), 24
    cluster, trace, params = _inputs(ref, prof, q, seed=5)
    want = P.search_optimal_config(cluster, trace, params)
    ours = {name: fn for (mod, name), fn in refbind.bindings(ref).items() if mod is P}["search_optimal_config"]
    got = ours(cluster, trace, params)
    text = lambda o: "\n".join(json.dumps(r, sort_keys=True) for r in cli._plan_records(o)) + "\n"  # noqa: E731
    assert text(got).encode() == text(want).encode()
    assert got == want
    assert len(want.ranked) > 0 and (which == "config1" or len(want.infeasible) > 0)


def test_streamed_plan_report_equals_materialised_1m_candidates(ref, tmp_path):
    """The streamed report writer (planner.write_plan_report: device ranking in
    chunks through hs_search_topk_after, infeasible list in product order) over
    a 4^10 = 1,048,576-candidate space with many exact ties (identical
    machines) gives the bytes of the reference's own report writer
    (cli._plan_records) over the materialised SearchOutcome."""
    from paper_2504_15303_b200 import planner, refbind

    cli = sys.modules["hetserve.cli"]
    P = sys.modules["hetserve.planner"]
    mems = [24, 32, 24, 32, 80, 24, 32, 24, 80, 32]  # repeated machines: exact ties in the ranking
    prof = wl.ClusterProfile("ties", dict(wl.MODEL_13B), dict(wl.ENGINE), dict(wl.LIMITS),
                             [(f"m{k}", 8, gb * 1_000_000_000, "v100") for k, gb in enumerate(mems)])
    for k, (name, count, gb, _a) in enumerate(prof.machines):
        for t in wl.enumerate_degrees(count):
            prof.params[(name, t)] = wl.scaled_params(wl.RANK_BASE, t ** -wl.TP_ALPHA * (1.0 + 0.1 * (gb // 10**9 % 7)))
    cluster, trace, params = _inputs(ref, prof, 16, seed=9)
    ours = {name: fn for (mod, name), fn in refbind.bindings(ref).items() if mod is P}["search_optimal_config"]
    outcome = ours(cluster, trace, params)
    want = ("\n".join(json.dumps(r, sort_keys=True) for r in cli._plan_records(outcome)) + "\n").encode()
    tables = planner.build_tables(cluster, trace, params)
    path = tmp_path / "plan.jsonl"
    with open(path, "wb") as fh:
        n = planner.write_plan_report(tables, fh, chunk=4096)
    assert n == outcome.candidates_visited == 4 ** 10
    assert len(outcome.ranked) > 10_000 and len(outcome.infeasible) > 10_000
    assert path.read_bytes() == want
