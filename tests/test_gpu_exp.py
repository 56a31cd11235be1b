"""The device exp the replay uses for workload() (scheduling.py:154,
math.exp -> glibc 2.39 exp, FMA ifunc body; hs_device.cuh py_exp) vs the
reference's own values: the golden vectors CPython produced
(tests/golden/exp_vectors.json, incl. the OverflowError arguments), and 1e8
random arguments over the domain the replay uses, [0, 709.78], plus the
overflow edge, against glibc's exp itself on this host (the function
math.exp calls) and the C port."""

import math

import numpy as np
import pytest

import helpers as H
from oracle import hs_oracle as orc
from paper_2504_15303_b200 import _native as nat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return nat.engine_for(0)


def test_device_exp_golden_vectors(eng):
    g = H.load("exp_vectors.json")
    x = np.array([float.fromhex(v) for v in g["x"]])
    y, of = eng.exp_batch(x)
    assert not of.any()
    assert [v.hex() for v in y.tolist()] == g["y"]
    xo = np.array([float.fromhex(v) for v in g["overflow"]])
    _y, of = eng.exp_batch(xo)
    assert of.all()


def test_device_exp_1e8_random_points_vs_glibc(eng):
    rng = np.random.default_rng(2025)
    n_chunk, chunks = 20_000_000, 5
    mism = 0
    for c in range(chunks):
        x = rng.uniform(0.0, 709.78, n_chunk)
        if c == 0:  # dense near 0 (small usages) and at the overflow edge
            x[:1_000_000] = rng.uniform(0.0, 1e-3, 1_000_000)
            x[1_000_000:1_100_000] = rng.uniform(709.7, 709.79, 100_000)
        y, of = eng.exp_batch(x)
        ref = orc.libm_exp_batch(x)  # glibc exp: math.exp's own function
        ofr = np.isinf(ref)
        assert np.array_equal(of, ofr), c
        ok = ~ofr
        mism += int((y[ok].view(np.uint64) != ref[ok].view(np.uint64)).sum())
        if c == 0:
            yp, ofp = orc.exp_batch(x[:2_000_000])  # the C port agrees too
            assert np.array_equal(yp.view(np.uint64), y[:2_000_000].view(np.uint64))
            assert np.array_equal(ofp, of[:2_000_000])
    assert mism == 0
    # spot check against CPython itself
    for v in rng.uniform(0, 709.78, 2000).tolist():
        y, _ = eng.exp_batch(np.array([v]))
        assert y[0] == math.exp(v)
