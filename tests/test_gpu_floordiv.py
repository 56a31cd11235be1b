"""The device floor division the replay uses for ideal_batch_size
(scheduling.py:128: budget // (per_token * tokens), CPython float `//`;
hs_device.cuh py_floordiv with the exact FMA remainder) vs CPython itself:
adversarial pairs (exact multiples and their neighbours, quotients up to and
beyond 2^52, subnormals, x < w, zero) and 2e7 random pairs over the replay's
range, plus the library-fmod fallback (negative, infinite operands)."""

import math

import numpy as np
import pytest

from paper_2504_15303_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return nat.engine_for(0)


def _same(got, x, w):
    want = [a // b for a, b in zip(x.tolist(), w.tolist())]
    bad = [(a, b, g, e) for a, b, g, e in zip(x.tolist(), w.tolist(), got.tolist(), want)
           if not (g == e and math.copysign(1.0, g) == math.copysign(1.0, e)) and not (math.isnan(g) and math.isnan(e))]
    return bad


def test_floordiv_adversarial_pairs(eng):
    rng = np.random.default_rng(11)
    w = np.concatenate([rng.uniform(1.0, 1e9, 4000), rng.uniform(1e-300, 1e-290, 500), [5e-324, 1e-310, 3.0, 0.1]])
    k = np.floor(rng.uniform(0, 2.0 ** 53, len(w)))
    base = k * w
    xs, ws = [], []
    for d in (-2, -1, 0, 1, 2):  # exact multiples and their float neighbours
        x = base.copy()
        for _ in range(abs(d)):
            x = np.nextafter(x, np.inf if d > 0 else -np.inf)
        xs.append(np.abs(x))
        ws.append(w)
    q = rng.uniform(0, 2.0 ** 60, 2000)  # quotients around and beyond 2^52
    wq = rng.uniform(1.0, 1e3, 2000)
    xs += [q * wq, rng.uniform(0, 1, 1000) * wq[:1000], np.zeros(10)]
    ws += [wq, wq[:1000], np.ones(10)]
    x, w = np.concatenate(xs), np.concatenate(ws)
    x = np.where(np.isfinite(x), x, 1.0)
    got = eng.floordiv_batch(x, w)
    assert _same(got, x, w) == []


def test_floordiv_library_fallback(eng):
    x = np.array([-7.5, -1e300, 7.5, math.inf, -math.inf, 3.0, 1e308, -0.0, 5.0])
    w = np.array([2.0, 3.0, -2.0, 1.0, 2.0, math.inf, 1e-10, 1.0, -math.inf])
    got = eng.floordiv_batch(x, w)
    assert _same(got, x, w) == []


def test_floordiv_2e7_random_pairs_replay_range(eng):
    # budgets up to ~1e12 bytes over per-token bytes (1e5..1e7) x tokens (1..1e4)
    rng = np.random.default_rng(2026)
    x = np.floor(rng.uniform(1e8, 1e12, 20_000_000)) * rng.choice([1.0, 0.9, 0.123456789], 20_000_000)
    w = np.floor(rng.uniform(1e5, 1e7, 20_000_000)) * np.floor(rng.uniform(1, 1e4, 20_000_000))
    got = eng.floordiv_batch(x, w)
    want = np.floor_divide(x, w)  # numpy's float floor division restates CPython's (checked below)
    sub = slice(0, 200_000)
    assert _same(got[sub], x[sub], w[sub]) == []
    assert np.array_equal(want[sub], np.array([a // b for a, b in zip(x[sub].tolist(), w[sub].tolist())]))
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


# ---- kv_usage's division (capacity.py:98-106): x / budget from RN(1 / budget)
def _div_bits_equal(eng, x, b):
    got = eng.div_batch(x, b)
    want = x / b  # IEEE round-to-nearest quotient, the same as CPython's float `/`
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    return bad, got, want


def test_div_replay_range_1e8(eng):
    """1e8 random (x, budget) pairs over the replay's range: x = per_token *
    running tokens (integers to 2^50), budgets from 1e6 to 1e13 bytes,
    fractional and integral, in chunks of 1e7."""
    rng = np.random.default_rng(77)
    for c in range(10):
        n = 10_000_000
        x = np.floor(rng.uniform(0, 2.0 ** rng.integers(10, 51), n))
        b = rng.uniform(1e6, 1e13, n)
        b = np.where(rng.random(n) < 0.5, np.floor(b), b)
        bad, got, want = _div_bits_equal(eng, x, b)
        assert len(bad) == 0, (c, x[bad[:5]].tolist(), b[bad[:5]].tolist())


def test_div_adversarial(eng):
    """Divisors with all-ones and near-one mantissas, powers of two, exact
    quotients and their neighbours, quotients at rounding ties of nearby
    precision, full-range random doubles."""
    rng = np.random.default_rng(5)
    k = rng.integers(-40, 40, 20000)
    ones = np.ldexp((2.0 ** 53 - 1) / 2.0 ** 52, k)  # 1.111...1 * 2^k
    near1 = np.ldexp(1.0 + rng.integers(1, 1000, 20000) * 2.0 ** -52, k)
    pow2 = np.ldexp(1.0, k)
    b = np.concatenate([ones, near1, pow2, np.nextafter(ones, 0), np.nextafter(near1, np.inf)])
    q = np.floor(rng.uniform(0, 2.0 ** 52, len(b)))
    xs, bs = [], []
    for d in (-1, 0, 1):
        x = q * b
        x = np.nextafter(x, np.inf) if d > 0 else (np.nextafter(x, 0) if d < 0 else x)
        xs.append(x)
        bs.append(b)
    xs.append(np.floor(rng.uniform(0, 2.0 ** 50, len(b))))
    bs.append(b)
    xs.append(np.abs(rng.standard_normal(200000)) * 10.0 ** rng.integers(-100, 100, 200000))
    bs.append(np.abs(rng.standard_normal(200000)) * 10.0 ** rng.integers(-100, 100, 200000) + 1e-300)
    x, b = np.concatenate(xs), np.concatenate(bs)
    ok = np.isfinite(x) & np.isfinite(b) & (b > 0) & np.isfinite(x / b) & (np.abs(x / b) > 1e-290) | (x == 0)
    x, b = x[ok], b[ok]
    bad, got, want = _div_bits_equal(eng, x, b)
    assert len(bad) == 0, (x[bad[:5]].tolist(), b[bad[:5]].tolist(), got[bad[:5]].tolist(), want[bad[:5]].tolist())
