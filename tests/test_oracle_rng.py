"""The numpy-stream oracle (oracle/hs_oracle_rng.c) pinned to the
reference's own draws (tests/golden/stream_cases.json, made by running
hetserve's cmd_gen_trace / generate_arrivals / OutputLengthPredictor) and to
numpy itself; plus the host-side pieces of the product's stream API that run
without a GPU (seeding, spec parsing)."""

from __future__ import annotations

import json
import math
import pathlib
import struct

import numpy as np
import pytest

from oracle import hs_oracle as orc
from paper_2504_15303_b200 import _native as nat
from paper_2504_15303_b200 import streams
from paper_2504_15303_b200.domain import SpecError

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "stream_cases.json").read_text())


def bits(x: float) -> bytes:
    return struct.pack("<d", x)


def test_log1p_matches_libm():
    rng = np.random.default_rng(5)
    xs = np.concatenate([-rng.random(100_000), rng.random(20_000) * 10, -rng.random(5_000) * 1e-8,
                         -rng.random(5_000) * 1e-17, rng.standard_normal(5_000) * 1e3,
                         np.exp(rng.uniform(-700, 700, 5_000)),
                         [-0.0, 0.0, 1e-300, 5e-324, -0.2929, -0.29289321881345254, 0.41421356, 2.0**-29,
                          -(2.0**-29), 2.0**-54, 1e300, math.inf]])
    xs = xs[xs > -1]
    bad = [x for x in xs if bits(orc.log1p(float(x))) != bits(math.log1p(float(x)))]
    assert not bad, bad[:5]


@pytest.mark.parametrize("seed", [0, 1, 7, 42, 2**32 - 1, 2**32, 2**64 + 5, 12345678901234567890123])
def test_pcg64_seed_matches_numpy(seed):
    """hs_pcg64_seed (numpy SeedSequence + pcg64_set_seed, host code)."""
    assert nat.pcg64_state(seed).tobytes() == orc.numpy_state(seed).tobytes()


def test_raw_draws_match_numpy():
    st = orc.numpy_state(3)
    g = np.random.default_rng(3).bit_generator
    ours = [orc.lib().hs_oracle_pcg64_next64(orc._p(st)) for _ in range(1000)]
    assert ours == [int(v) for v in g.random_raw(1000)]


def _trace_dists(case):
    return [streams.parse_length_dist(case["input_dist"], case["max_in"]),
            streams.parse_length_dist(case["output_dist"], case["max_out"])]


@pytest.mark.parametrize("case", GOLD["traces"], ids=lambda c: f"seed{c['seed']}-{c['input_dist']}")
def test_gen_trace_golden(case):
    st = orc.numpy_state(case["seed"])
    (I, O), bad = orc.rng_generate(st, np.array([0, case["count"]]), _trace_dists(case))
    if case["error"]:
        assert case["error"].startswith("OverflowError") and bad[0] >= 0
        return
    assert bad[0] == -1
    assert I.tolist() == case["I"] and O.tolist() == case["O"]


@pytest.mark.parametrize("case", GOLD["arrivals"], ids=lambda c: f"n{c['n']}")
def test_arrivals_golden(case):
    rate = float.fromhex(case["rate"])
    if math.isinf(rate):
        assert all(float.fromhex(t) == 0.0 for t in case["t"])
        return
    st = orc.numpy_state(case["seed"])
    (T,), _ = orc.rng_generate(st, np.array([0, case["n"]]), [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0 / rate, 0)])
    assert [t.hex() for t in T.tolist()] == case["t"]


@pytest.mark.parametrize("case", GOLD["predictors"], ids=lambda c: f"n{c['n']}")
def test_predictor_golden(case):
    st = orc.numpy_state(case["seed"])
    d = nat.hs_dist(nat.DIST_NORMAL_LEN, case["cap"], 0, 0, float.fromhex(case["mean"]), float.fromhex(case["stddev"]))
    (P,), _ = orc.rng_generate(st, np.array([0, case["n"]]), [d])
    assert P.tolist() == case["p"]


def test_multi_stream_batch_and_final_state():
    """Ragged batch of streams; each stream's final state equals numpy's."""
    seeds = [5, 6, 7, 8]
    counts = [0, 1, 4097, 333]
    off = np.concatenate([[0], np.cumsum(counts)])
    st = np.concatenate([orc.numpy_state(s) for s in seeds])
    mu = math.log(200) - 0.18
    dists = [nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 4096, 0, 0, mu, 0.6),
             nat.hs_dist(nat.DIST_UNIFORM_LEN, 4096, 1, 4096, 0, 0),
             nat.hs_dist(nat.DIST_NORMAL_LEN, 100, 0, 0, 50.0, 30.0),
             nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 0.25, 0)]
    (A, B, Cn, D), bad = orc.rng_generate(st, off, dists)
    for t, s in enumerate(seeds):
        g = np.random.default_rng(s)
        n = counts[t]
        sl = slice(off[t], off[t + 1])
        assert A[sl].tolist() == np.clip(np.rint(g.lognormal(mu, 0.6, n)), 1, 4096).astype(int).tolist()
        assert B[sl].tolist() == g.integers(1, 4097, size=n).tolist()
        assert Cn[sl].tolist() == np.clip(np.rint(g.normal(50.0, 30.0, n)), 1, 100).astype(int).tolist()
        assert np.array_equal(D[sl], np.cumsum(g.exponential(0.25, n)))
        ref = g.bit_generator.state
        assert (int(st["state_hi"][t]) << 64 | int(st["state_lo"][t])) == ref["state"]["state"]
        assert int(st["has_uint32"][t]) == ref["has_uint32"] and int(st["uinteger"][t]) == ref["uinteger"]
    assert (bad == -1).all()


@pytest.mark.parametrize("lo,hi", [(1, 1), (1, 2), (3, 2**31), (1, 2**32 - 1), (1, 2**32), (7, 2**40), (1, 2**62)])
def test_uniform_ranges_match_numpy(lo, hi):
    st = orc.numpy_state(99)
    g = np.random.default_rng(99)
    outs = []
    for n in (1, 31, 64, 1000):  # odd counts leave a buffered half behind
        (v,), _ = orc.rng_generate(st, np.array([0, n]), [nat.hs_dist(nat.DIST_UNIFORM_LEN, 2**31 - 1, lo, hi, 0, 0)])
        outs.append(v.tolist() == np.minimum(g.integers(lo, hi + 1, size=n), 2**31 - 1).tolist())
    assert all(outs)


def test_spec_parsing_messages():
    """cli.py:160-180 errors, same text."""
    with pytest.raises(SpecError, match="lognormal needs positive mean and sigma, got 'lognormal:0:1'"):
        streams.parse_length_dist("lognormal:0:1", 10)
    with pytest.raises(SpecError, match="uniform needs 1 <= lo <= hi, got 'uniform:5:4'"):
        streams.parse_length_dist("uniform:5:4", 10)
    with pytest.raises(SpecError, match="unknown distribution 'zipf'"):
        streams.parse_length_dist("zipf:1:2", 10)
    with pytest.raises(SpecError, match="cannot parse distribution 'lognormal:1'"):
        streams.parse_length_dist("lognormal:1", 10)
    with pytest.raises(SpecError, match="cannot parse distribution 'uniform:a:b'"):
        streams.parse_length_dist("uniform:a:b", 10)
    d = streams.parse_length_dist("LogNormal:200:0.6", 4096)
    assert d.kind == nat.DIST_LOGNORMAL_LEN and d.p0 == math.log(200.0) - 0.6 * 0.6 / 2.0 and d.cap == 4096


def test_pcg64_states_batch_matches_numpy():
    seeds = [0, 1, 5, 2**32 - 1, 2**32, 2**64 - 1, 2**70 + 3]
    assert nat.pcg64_states(seeds).tobytes() == b"".join(orc.numpy_state(s).tobytes() for s in seeds)
