"""Seeded synthetic workload streams drawn on the GPU (SURVEY.md section 8f,
rank 3), bit-identical to the reference's numpy draws.

The reference builds every synthetic input from numpy.random.default_rng(seed)
(numpy Generator over PCG64):

* ``gen_trace_lengths`` -- cli.py:160-197 ``cmd_gen_trace`` /
  ``_sample_lengths``: inputs then outputs from ONE generator, each
  ``lognormal:MEAN:SIGMA`` (mu = ln(mean) - sigma^2 / 2) or ``uniform:LO:HI``
  (``integers(lo, hi + 1)``), then ``int(min(max(round(v), 1), upper))``;
* ``arrival_times_device`` -- simulator.py:112-124 ``generate_arrivals``:
  ``np.cumsum(rng.exponential(1 / rate, n))`` (all 0.0 for rate = inf);
* ``predict_lengths_device`` -- scheduling.py:87-95 normal predictor:
  ``int(min(max(round(rng.normal(mean, sd)), 1), max_output_len))`` per
  request in trace order.

One warp per stream (kernel rng.cu); a batch of streams (one per trace) is a
single launch.  Seeds map to generator states with ``hs_pcg64_seed`` (numpy's
SeedSequence), so stream t of a batch equals ``default_rng(seeds[t])``.
Outputs land in device memory (``*_device`` pointers, for hs_replay_device)
or are copied back as numpy arrays.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .domain import SpecError


def parse_length_dist(spec: str, upper: int) -> nat.hs_dist:
    """cli.py:160-180 ``_sample_lengths`` argument handling, same messages."""
    parts = spec.split(":")
    kind = parts[0].lower()
    try:
        if kind == "lognormal":
            mean, sigma = float(parts[1]), float(parts[2])
            if mean <= 0 or sigma <= 0:
                raise SpecError(f"lognormal needs positive mean and sigma, got {spec!r}")
            mu = math.log(mean) - sigma * sigma / 2.0
            return nat.hs_dist(nat.DIST_LOGNORMAL_LEN, int(upper), 0, 0, mu, sigma)
        if kind == "uniform":
            lo, hi = int(parts[1]), int(parts[2])
            if lo < 1 or hi < lo:
                raise SpecError(f"uniform needs 1 <= lo <= hi, got {spec!r}")
            if hi >= 2**63:
                raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, "uniform bounds beyond int64")
            return nat.hs_dist(nat.DIST_UNIFORM_LEN, int(upper), lo, hi, 0.0, 0.0)
        raise SpecError(f"unknown distribution {kind!r}; use lognormal:MEAN:SIGMA or uniform:LO:HI")
    except (IndexError, ValueError) as exc:
        raise SpecError(f"cannot parse distribution {spec!r}: {exc}") from exc


def _upper(v: int) -> int:
    if not 1 <= int(v) <= 2**31 - 1:
        raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, "length caps must lie in [1, 2^31 - 1]")
    return int(v)


def _offsets(counts) -> np.ndarray:
    c = np.asarray(counts, np.int64)
    if (c < 0).any():
        raise SpecError("stream lengths must be non-negative")
    return np.concatenate([[0], np.cumsum(c)]).astype(np.int64)


class DeviceStreams:
    """Device buffers produced by one generation call (freed on close())."""

    def __init__(self, engine: nat.Engine, offsets: np.ndarray, ptrs: list, dtypes: list):
        self.engine, self.offsets, self.ptrs, self.dtypes = engine, offsets, ptrs, dtypes

    def to_host(self) -> list:
        total = int(self.offsets[-1])
        outs = []
        for p, dt in zip(self.ptrs, self.dtypes):
            a = np.empty(total, dt)
            if total:
                self.engine.d2h(a, p)
            outs.append(a)
        return outs

    def close(self) -> None:
        for p in self.ptrs:
            if p:
                self.engine.device_free(p)
        self.ptrs = []


def _generate(seeds, counts, dists, engine=None, states=None) -> DeviceStreams:
    eng = engine or nat.engine_for()
    off = _offsets(counts)
    if len(off) - 1 != len(seeds):
        raise SpecError("one seed per stream")
    st = nat.pcg64_states(seeds) if states is None else states
    total = int(off[-1])
    dtypes = [np.float64 if d.kind == nat.DIST_EXP_CUMSUM else np.int32 for d in dists]
    ptrs = [eng.device_alloc(max(total, 1) * np.dtype(dt).itemsize) for dt in dtypes]
    out = DeviceStreams(eng, off, ptrs, dtypes)
    try:
        bad = eng.rng_generate(st, off, dists, ptrs)
    except Exception:
        out.close()
        raise
    out.bad = bad
    return out


def gen_trace_lengths_device(seeds, count: int, input_dist: str, output_dist: str, max_input_len: int,
                             max_output_len: int, engine=None) -> DeviceStreams:
    """``cmd_gen_trace`` for each seed (count requests each), on the device.
    Raises OverflowError like round(inf) when a lognormal draw overflows."""
    di = parse_length_dist(input_dist, _upper(max_input_len))
    do = parse_length_dist(output_dist, _upper(max_output_len))
    out = _generate(list(seeds), [int(count)] * len(seeds), [di, do], engine)
    if (out.bad >= 0).any():
        out.close()
        raise OverflowError("cannot convert float infinity to integer")
    return out


def gen_trace_lengths(seeds, count: int, input_dist: str, output_dist: str, max_input_len: int,
                      max_output_len: int, engine=None):
    """Host copies of gen_trace_lengths_device: (I, O) int32, stream-major."""
    d = gen_trace_lengths_device(seeds, count, input_dist, output_dist, max_input_len, max_output_len, engine)
    try:
        I, O = d.to_host()
    finally:
        d.close()
    return I, O


def arrival_times_device(seeds, counts, rate: float, engine=None) -> DeviceStreams | None:
    """generate_arrivals for each (seed, count); None means rate = inf
    (every arrival at 0.0, no draws)."""
    if math.isinf(rate):
        return None
    if rate <= 0:
        raise SpecError(f"arrival rate must be positive, got {rate}")
    return _generate(list(seeds), counts, [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0 / rate, 0.0)], engine)


def arrival_times(seeds, counts, rate: float, engine=None) -> np.ndarray:
    d = arrival_times_device(seeds, counts, rate, engine)
    if d is None:
        return np.zeros(int(np.sum(counts)), np.float64)
    try:
        return d.to_host()[0]
    finally:
        d.close()


def _check_finite_normal(seed, mean: float, stddev: float) -> None:
    """A non-finite mean / stddev makes the predictor's first draw non-finite,
    and the reference's round() raises on it (scheduling.py:94: ValueError for
    NaN, OverflowError for inf): raise exactly that, from the same draw."""
    if math.isfinite(float(mean)) and math.isfinite(float(stddev)):
        return
    round(float(np.random.default_rng(seed).normal(float(mean), float(stddev))))


def predict_lengths_device(seeds, counts, mean: float, stddev: float, max_output_len: int,
                           engine=None) -> DeviceStreams:
    """The normal-mode OutputLengthPredictor for each (seed, count)."""
    seeds = list(seeds)
    for sd, n in zip(seeds, counts):
        if int(n) > 0:
            _check_finite_normal(sd, mean, stddev)
            break
    return _generate(list(seeds), counts,
                     [nat.hs_dist(nat.DIST_NORMAL_LEN, _upper(max_output_len), 0, 0, float(mean), float(stddev))],
                     engine)


def predict_lengths(seeds, counts, mean: float, stddev: float, max_output_len: int, engine=None) -> np.ndarray:
    d = predict_lengths_device(seeds, counts, mean, stddev, max_output_len, engine)
    try:
        return d.to_host()[0]
    finally:
        d.close()


def replay_seeds(arrival_seeds=None, rate: float = math.inf, predictor=None, predictor_seeds=None,
                 max_output_len: int = 0):
    """hs_replay_seeds for hs_replay_seeded: device-drawn arrivals (finite
    rate) and/or normal-mode predictions.  Returns (struct, keep-alive)."""
    keep = []
    s = nat.hs_replay_seeds()
    if arrival_seeds is not None and not math.isinf(rate):
        if rate <= 0:
            raise SpecError(f"arrival rate must be positive, got {rate}")
        st = nat.pcg64_states(list(arrival_seeds))
        keep.append(st)
        s.arrival_state = st.ctypes.data
        s.arrival_scale = 1.0 / rate
    if predictor is not None and predictor.mode == "normal":
        if len(predictor_seeds):
            _check_finite_normal(list(predictor_seeds)[0], predictor.mean, predictor.stddev)
        st = nat.pcg64_states(list(predictor_seeds))
        keep.append(st)
        s.predictor_state = st.ctypes.data
        s.pred_mean = float(predictor.mean)
        s.pred_stddev = float(predictor.stddev)
        s.pred_cap = _upper(max_output_len)
    return s, keep
