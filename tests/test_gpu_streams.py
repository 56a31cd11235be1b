"""Device-drawn numpy streams (rng.cu) vs the reference's own draws
(tests/golden/stream_cases.json) and vs the C oracle, bit-exact; and the
seeded replay (hs_replay_seeded) vs the replay of host-drawn inputs."""

import json
import math
import pathlib

import numpy as np
import pytest

import paper_2504_15303_b200 as hs
from oracle import hs_oracle as orc
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import streams
from paper_2504_15303_b200 import workloads as wl

pytestmark = pytest.mark.gpu

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "stream_cases.json").read_text())


@pytest.fixture(scope="module")
def eng():
    return nat.engine_for(0)


@pytest.mark.parametrize("case", GOLD["traces"], ids=lambda c: f"seed{c['seed']}-{c['input_dist']}")
def test_gen_trace_golden(eng, case):
    args = (case["count"], case["input_dist"], case["output_dist"], case["max_in"], case["max_out"])
    if case["error"]:
        with pytest.raises(OverflowError, match="cannot convert float infinity to integer"):
            streams.gen_trace_lengths([case["seed"]], *args, engine=eng)
        return
    I, O = streams.gen_trace_lengths([case["seed"]], *args, engine=eng)
    assert I.tolist() == case["I"] and O.tolist() == case["O"]


@pytest.mark.parametrize("case", GOLD["arrivals"], ids=lambda c: f"n{c['n']}")
def test_arrivals_golden(eng, case):
    T = streams.arrival_times([case["seed"]], [case["n"]], float.fromhex(case["rate"]), engine=eng)
    assert [t.hex() for t in T.tolist()] == case["t"]


@pytest.mark.parametrize("case", GOLD["predictors"], ids=lambda c: f"n{c['n']}")
def test_predictor_golden(eng, case):
    P = streams.predict_lengths([case["seed"]], [case["n"]], float.fromhex(case["mean"]),
                                float.fromhex(case["stddev"]), case["cap"], engine=eng)
    assert P.tolist() == case["p"]


def _oracle(seeds, counts, dists):
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    st = np.concatenate([orc.numpy_state(s) for s in seeds])
    outs, bad = orc.rng_generate(st, off, dists)
    return outs, bad, st


@pytest.mark.parametrize("kinds", ["lognormal", "uniform32", "uniform64", "normal", "expsum", "mixed"])
def test_ragged_batch_vs_oracle(eng, kinds):
    """200 ragged streams (incl. empty and length-1 ones) with the final
    generator states compared too (continuation semantics)."""
    rng = np.random.default_rng(17)
    counts = [int(x) for x in rng.integers(0, 6000, 200)]
    counts[3], counts[4], counts[5] = 0, 1, 33
    seeds = [int(s) for s in rng.integers(0, 2**40, 200)]
    mu = math.log(200) - 0.18
    D = {
        "lognormal": [nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 4096, 0, 0, mu, 0.6),
                      nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 2048, 0, 0, math.log(1000) - 2.0, 2.0)],
        "uniform32": [nat.hs_dist(nat.DIST_UNIFORM_LEN, 4096, 1, 4096, 0, 0),
                      nat.hs_dist(nat.DIST_UNIFORM_LEN, 50, 3, 2**31 + 5, 0, 0)],
        "uniform64": [nat.hs_dist(nat.DIST_UNIFORM_LEN, 2**31 - 1, 1, 2**32, 0, 0),
                      nat.hs_dist(nat.DIST_UNIFORM_LEN, 2**31 - 1, 9, 2**50 + 3, 0, 0)],
        "normal": [nat.hs_dist(nat.DIST_NORMAL_LEN, 4096, 0, 0, 150.0, 60.0),
                   nat.hs_dist(nat.DIST_NORMAL_LEN, 16, 0, 0, 3.0, 40.0)],
        "expsum": [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0 / 140.0, 0),
                   nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 2.0, 0)],
        "mixed": [nat.hs_dist(nat.DIST_UNIFORM_LEN, 4096, 1, 77, 0, 0),
                  nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 4096, 0, 0, mu, 0.6),
                  nat.hs_dist(nat.DIST_UNIFORM_LEN, 4096, 1, 5, 0, 0),
                  nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 0.01, 0)],
    }[kinds]
    want, wbad, wst = _oracle(seeds, counts, D)
    st = nat.pcg64_states(seeds)
    out = streams._generate(seeds, counts, D, engine=eng, states=st)
    try:
        got = out.to_host()
    finally:
        out.close()
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and np.array_equal(g.view(np.uint8), w.view(np.uint8))
    assert st.tobytes() == wst.tobytes()
    assert np.array_equal(out.bad, wbad)


def test_config4_scale_streams_vs_numpy(eng):
    """Full-size streams (1e5 requests) for a few traces of the bench
    workload, straight against numpy (workloads.py helpers)."""
    q = wl.CONFIG4_Q
    seeds = [0, 1, 4095]
    I, O = streams.gen_trace_lengths(seeds, q, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096, engine=eng)
    T = streams.arrival_times([42 + s for s in seeds], [q] * 3, wl.CONFIG4_RATE, engine=eng)
    for k, s in enumerate(seeds):
        i, o = wl.trace_lengths(q, seed=s)
        assert np.array_equal(I[k * q:(k + 1) * q], i) and np.array_equal(O[k * q:(k + 1) * q], o)
        assert np.array_equal(T[k * q:(k + 1) * q], wl.arrivals(q, wl.CONFIG4_RATE, seed=42 + s))


def _config4():
    prof = wl.config4()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    return cluster, params, config


@pytest.mark.parametrize("policy", ["OS", "MB"])
def test_seeded_replay_equals_host_drawn_replay(eng, policy):
    """hs_replay_seeded (arrivals + normal predictions drawn on the device,
    per chunk) gives exactly the replay of the same draws made by numpy."""
    cluster, params, config = _config4()
    rng = np.random.default_rng(3)
    lens = [int(x) for x in rng.integers(0, 3000, 40)]
    lens[7] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I = np.concatenate([wl.trace_lengths(q, seed=50 + t)[0] for t, q in enumerate(lens)])
    O = np.concatenate([wl.trace_lengths(q, seed=50 + t)[1] for t, q in enumerate(lens)])
    aseeds = [900 + t for t in range(len(lens))]
    pseeds = [700 + t for t in range(len(lens))]
    pc = hs.PredictorConfig(mode="normal", mean=150.0, stddev=60.0, seed=0)
    pol = hs.PolicyConfig(policy=policy, theta=2.0, predictor=pc)
    T = np.concatenate([wl.arrivals(q, 140.0, seed=s) for q, s in zip(lens, aseeds)])
    P = np.concatenate([wl.predictions(O[off[t]:off[t + 1]], "normal", 150.0, 60.0, seed=s) for t, s in
                        enumerate(pseeds)])
    want = hs.replay_traces(cluster, config, params, pol, off, I, O, P, arrival=T, want_assign=True,
                            want_depart=True, engine=eng)
    got = hs.replay_traces(cluster, config, params, pol, off, I, O, None, want_assign=True, want_depart=True,
                           engine=eng, rate=140.0, arrival_seeds=aseeds, predictor_seeds=pseeds)
    assert (want.result["error"] == 0).all()
    assert np.array_equal(got.assign, want.assign)
    assert np.array_equal(got.depart.view(np.uint64), want.depart.view(np.uint64))
    assert got.metrics.tobytes() == want.metrics.tobytes()
    assert got.result.tobytes() == want.result.tobytes()


def test_seeded_replay_rate_inf_draws_nothing(eng):
    cluster, params, config = _config4()
    I, O = wl.trace_lengths(500, seed=1)
    off = np.array([0, 500], np.int64)
    pol = hs.PolicyConfig()
    a = hs.replay_traces(cluster, config, params, pol, off, I, O, O, arrival=None, want_depart=True, engine=eng)
    b = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_depart=True, engine=eng, rate=math.inf,
                         arrival_seeds=[5])
    assert np.array_equal(a.depart, b.depart) and np.array_equal(a.assign, b.assign)


def test_device_stream_launches_counted(eng):
    n0 = eng.launch_count
    streams.arrival_times([1, 2, 3], [10, 0, 5], 3.0, engine=eng)
    assert eng.launch_count == n0 + 1


def test_rng_argument_validation(eng):
    st = nat.pcg64_states([1])
    off = np.array([0, 10], np.int64)
    ptr = eng.device_alloc(80)
    try:
        bad_kind = nat.hs_dist(9, 10, 0, 0, 0.0, 0.0)
        with pytest.raises(nat.EngineError, match="unknown distribution"):
            eng.rng_generate(st, off, [bad_kind], [ptr])
        with pytest.raises(nat.EngineError, match="lo <= hi"):
            eng.rng_generate(st, off, [nat.hs_dist(nat.DIST_UNIFORM_LEN, 10, 5, 4, 0, 0)], [ptr])
        with pytest.raises(nat.EngineError, match="cap must be >= 1"):
            eng.rng_generate(st, off, [nat.hs_dist(nat.DIST_NORMAL_LEN, 0, 0, 0, 1.0, 1.0)], [ptr])
        with pytest.raises(nat.EngineError, match="n_dists"):
            eng.rng_generate(st, off, [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0, 0)] * 5, [ptr] * 5)
        with pytest.raises(nat.EngineError, match="non-decreasing"):
            eng.rng_generate(nat.pcg64_states([1, 2]), np.array([0, 5, 3], np.int64),
                             [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0, 0)], [ptr])
        # the state is untouched by a rejected call
        assert st.tobytes() == nat.pcg64_states([1]).tobytes()
    finally:
        eng.device_free(ptr)


def test_seeded_replay_rejects_arrivals_and_seeds_together(eng):
    cluster, params, config = _config4()
    I, O = wl.trace_lengths(50, seed=1)
    off = np.array([0, 50], np.int64)
    with pytest.raises(hs.SpecError, match="either arrival times or arrival seeds"):
        hs.replay_traces(cluster, config, params, hs.PolicyConfig(), off, I, O, O, arrival=np.zeros(50),
                         rate=3.0, arrival_seeds=[1], engine=eng)
    with pytest.raises(hs.SpecError, match="arrival rate must be positive"):
        hs.replay_traces(cluster, config, params, hs.PolicyConfig(), off, I, O, O, rate=-1.0, arrival_seeds=[1],
                         engine=eng)


@pytest.mark.parametrize("seeded", [False, True])
def test_streamed_replay_equals_chunked(eng, seeded, monkeypatch):
    """Equal-length traces take the streamed host path (phase-wise 2-D copies
    published through a progress word the kernel waits on); it must give
    exactly what the chunked path (HS_NO_STREAM) gives."""
    cluster, params, config = _config4()
    nT, q = 96, 4096
    I = np.concatenate([wl.trace_lengths(q, seed=300 + t)[0] for t in range(nT)])
    O = np.concatenate([wl.trace_lengths(q, seed=300 + t)[1] for t in range(nT)])
    off = np.arange(nT + 1, dtype=np.int64) * q
    pc = hs.PredictorConfig(mode="normal", mean=150.0, stddev=60.0, seed=0)
    pol = hs.PolicyConfig(policy="OS", predictor=pc if seeded else hs.PredictorConfig())
    if seeded:
        kw = dict(rate=140.0, arrival_seeds=[7 + t for t in range(nT)], predictor_seeds=[9 + t for t in range(nT)])
        P = None
    else:
        kw = dict(arrival=np.concatenate([wl.arrivals(q, 140.0, seed=7 + t) for t in range(nT)]))
        P = O
    got = hs.replay_traces(cluster, config, params, pol, off, I, O, P, want_assign=True, want_depart=True,
                           engine=eng, **kw)
    launches = eng.launch_count
    monkeypatch.setenv("HS_NO_STREAM", "1")
    want = hs.replay_traces(cluster, config, params, pol, off, I, O, P, want_assign=True, want_depart=True,
                            engine=eng, **kw)
    assert eng.launch_count - launches >= 8  # the chunked path: one replay launch per chunk
    assert (want.result["error"] == 0).all()
    assert np.array_equal(got.assign, want.assign)
    assert np.array_equal(got.depart.view(np.uint64), want.depart.view(np.uint64))
    assert got.metrics.tobytes() == want.metrics.tobytes()
    assert got.result.tobytes() == want.result.tobytes()


def test_streamed_replay_redoes_when_phase0_sizing_is_too_small(eng, monkeypatch):
    """Phase 0 of every trace holds only huge requests, so min(I + O) over
    phase 0 (which sizes the streamed heaps) is far above the rest; at rate
    inf the later tiny requests pile up beyond that capacity, the kernel
    reports CAPACITY and the call is redone on the exactly sized chunked path.
    The result must equal the chunked path's."""
    prof = wl.config1()
    cluster = hs.ClusterSpec(hs.ModelSpec(**prof.model), hs.EngineOverheads(**prof.engine),
                             tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                             hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {"v100": 1, "a800": 1})
    nT, q = 4, 512
    I = np.ones((nT, q), np.int32)
    O = np.ones((nT, q), np.int32)
    I[:, :32], O[:, :32] = 2000, 2000
    I, O = I.reshape(-1), O.reshape(-1)
    off = np.arange(nT + 1, dtype=np.int64) * q
    pol = hs.PolicyConfig()
    n0 = eng.launch_count
    got = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, want_depart=True,
                           engine=eng)
    n1 = eng.launch_count
    monkeypatch.setenv("HS_NO_STREAM", "1")
    want = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, want_depart=True,
                            engine=eng)
    # streamed attempt (phase-0 sizing + replay) then the chunked redo's launches
    assert n1 - n0 == 2 + (eng.launch_count - n1)
    assert (want.result["error"] == 0).all() and (got.result["error"] == 0).all()
    assert np.array_equal(got.assign, want.assign)
    assert np.array_equal(got.depart.view(np.uint64), want.depart.view(np.uint64))
    assert got.metrics.tobytes() == want.metrics.tobytes()


@pytest.mark.parametrize("ragged", [False, True])
def test_pinned_assign_written_in_place(eng, ragged):
    """A page-locked `assign_out` is written by the replay kernel itself while
    it runs (zero-copy, no copy back after the kernel); the assignments equal
    those of the pageable-buffer replay on the streamed (equal lengths) and the
    chunked (ragged) host paths."""
    cluster, params, config = _config4()
    lens = [1500 + (53 * t if ragged else 0) for t in range(24)]
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    I = np.concatenate([wl.trace_lengths(q, seed=300 + t)[0] for t, q in enumerate(lens)])
    O = np.concatenate([wl.trace_lengths(q, seed=300 + t)[1] for t, q in enumerate(lens)])
    aseeds = [42 + t for t in range(len(lens))]
    pol = hs.PolicyConfig()
    want = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, engine=eng, rate=140.0,
                            arrival_seeds=aseeds)
    hA = eng.host_array((len(I),), np.uint8)
    hA[:] = 255
    got = hs.replay_traces(cluster, config, params, pol, off, I, O, O, want_assign=True, assign_out=hA,
                           engine=eng, rate=140.0, arrival_seeds=aseeds)
    assert (want.result["error"] == 0).all() and (got.result["error"] == 0).all()
    assert np.array_equal(hA, want.assign[:len(I)])
    assert got.metrics.tobytes() == want.metrics.tobytes()
