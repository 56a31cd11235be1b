"""Synthetic cluster profiles and request traces for BASELINE.json configs 1-5.

Plain numbers only (no engine types), so the golden-fixture generator can
build reference objects and the tests / bench can build engine objects from
the same description.  Shapes follow SURVEY.md section 8(d):

* trace lengths as ``hetserve gen-trace`` draws them (cli.py:160-193):
  lognormal with the given mean and sigma, ``mu = ln(mean) - sigma^2 / 2``,
  rounded half-even, clamped to [1, limit]; inputs then outputs from one
  ``default_rng(seed)``;
* arrivals as simulator.py:112-124 generate_arrivals: cumulative sum of
  ``default_rng(seed).exponential(1 / rate, q)`` (all 0.0 for rate = inf);
* latency parameters = RANK_BASE (test_acceptance.py:225) scaled by a
  per-accelerator-type factor times t ** -0.6, the sublinear TP speed-up the
  reference's own tests use (test_planner.py:255-259).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

from .domain import enumerate_tp_degrees
from .scheduling import OutputLengthPredictor, PredictorConfig
from .simulator import arrival_times

RANK_BASE = (2e-5, 4e-4, 1e-5, 3e-3, 1.5e-6, 2e-4, 5e-7, 1e-4)
TP_ALPHA = 0.6

# relative slowness per accelerator type (V100 = 1.0)
TYPE_SCALE = {
    "b200": 0.25,
    "h200": 0.28,
    "h100": 0.30,
    "a100": 0.40,
    "a800": 0.38,
    "l40s": 0.60,
    "v100": 1.00,
    "a10": 1.20,
}
TYPE_MEM_GB = {
    "b200": 180,
    "h200": 141,
    "h100": 80,
    "a100": 80,
    "a800": 80,
    "l40s": 48,
    "v100": 32,
    "a10": 24,
}

MODEL_7B = dict(layers=32, hidden_dim=4096, param_count=7_000_000_000, bytes_per_param=2)
MODEL_13B = dict(layers=40, hidden_dim=5120, param_count=13_000_000_000, bytes_per_param=2)
MODEL_70B = dict(layers=80, hidden_dim=8192, param_count=70_000_000_000, bytes_per_param=2)
ENGINE = dict(mem_utilization_fraction=0.9, static_overhead_bytes=2_000_000_000)
LIMITS = dict(max_input_len=4096, max_output_len=4096)


def enumerate_degrees(count: int) -> list[int]:
    """core.py:363-371 enumerate_tp_degrees for an accelerator count
    (domain.enumerate_tp_degrees on a bare count)."""
    return enumerate_tp_degrees(SimpleNamespace(accelerator_count=count))


def scaled_params(base: tuple, alpha: float) -> tuple:
    """latency.py:56-58 LatencyParams.scaled: alpha * p for each p."""
    return tuple(alpha * p for p in base)


@dataclass
class ClusterProfile:
    """A cluster spec plus its fitted-parameter table, as plain values."""

    name: str
    model: dict
    engine: dict
    limits: dict
    machines: list  # [(name, accelerator_count, accelerator_mem_bytes, type)]
    params: dict = field(default_factory=dict)  # {(machine, t): 8-tuple}

    def degree_lists(self) -> list[list[int]]:
        return [enumerate_degrees(m[1]) for m in self.machines]

    def space_size(self) -> int:
        n = 1
        for d in self.degree_lists():
            n *= len(d)
        return n


def _machine(name: str, acc_type: str, count: int) -> tuple:
    return (name, count, TYPE_MEM_GB[acc_type] * 1_000_000_000, acc_type)


def _fill_params(profile: ClusterProfile) -> ClusterProfile:
    for name, count, _mem, acc_type in profile.machines:
        for t in enumerate_degrees(count):
            profile.params[(name, t)] = scaled_params(RANK_BASE, t**-TP_ALPHA * TYPE_SCALE[acc_type])
    return profile


def config1() -> ClusterProfile:
    """Paper section 5.3 pair: 8x V100-32G + 1x A800-80G, 7B-class."""
    return _fill_params(
        ClusterProfile(
            "config1", dict(MODEL_7B), dict(ENGINE), dict(LIMITS),
            [_machine("v100", "v100", 8), _machine("a800", "a800", 1)],
        )
    )


def config2() -> ClusterProfile:
    """Three machine types, 13B-class: V100x8, A800x4, H100x8 (48 candidates)."""
    return _fill_params(
        ClusterProfile(
            "config2", dict(MODEL_13B), dict(ENGINE), dict(LIMITS),
            [_machine("v100", "v100", 8), _machine("a800", "a800", 4), _machine("h100", "h100", 8)],
        )
    )


CONFIG3_TYPES = ("b200", "h200", "h100", "a100", "a800", "l40s", "v100", "a10")


def config3() -> ClusterProfile:
    """8 accelerator types x 2 machines x 16 GPUs, 70B-class: 5^16 candidates."""
    machines = []
    for acc in CONFIG3_TYPES:
        for k in range(2):
            machines.append(_machine(f"{acc}-{k}", acc, 16))
    return _fill_params(ClusterProfile("config3", dict(MODEL_70B), dict(ENGINE), dict(LIMITS), machines))


CONFIG4_TYPES = ("b200", "h100", "a800", "v100")


def config4() -> ClusterProfile:
    """32 instances: 4 types x 8 GPUs deployed at t = 1, 7B-class."""
    return _fill_params(
        ClusterProfile(
            "config4", dict(MODEL_7B), dict(ENGINE), dict(LIMITS),
            [_machine(acc, acc, 8) for acc in CONFIG4_TYPES],
        )
    )


CONFIG4_RATE = 140.0
CONFIG4_TRACES = 4096
CONFIG4_Q = 100_000


def trace_lengths(q: int, seed: int, in_mean: float = 200.0, out_mean: float = 150.0,
                  sigma: float = 0.6, max_in: int = 4096, max_out: int = 4096):
    """gen-trace lognormal lengths (cli.py:160-193) as int32 arrays."""
    rng = np.random.default_rng(seed)
    mu_i = math.log(in_mean) - sigma * sigma / 2.0
    vi = rng.lognormal(mu_i, sigma, size=q)
    mu_o = math.log(out_mean) - sigma * sigma / 2.0
    vo = rng.lognormal(mu_o, sigma, size=q)
    I = np.clip(np.rint(vi), 1, max_in).astype(np.int32)
    O = np.clip(np.rint(vo), 1, max_out).astype(np.int32)
    return I, O


def arrivals(q: int, rate: float, seed: int) -> np.ndarray:
    """simulator.py:112-124 generate_arrivals as an fp64 array (simulator.arrival_times)."""
    return arrival_times(q, rate, seed)


def predictions(O: np.ndarray, mode: str = "oracle", mean=None, stddev=None, seed=None,
                max_output_len: int = 4096) -> np.ndarray:
    """scheduling.py:65-95 OutputLengthPredictor, one draw per request in
    trace order (the dispatch order): OutputLengthPredictor.predict_lengths."""
    cfg = PredictorConfig(mode=mode, mean=mean, stddev=stddev, seed=seed)
    return OutputLengthPredictor(cfg, max_output_len).predict_lengths(O).astype(np.int32)


def deployment_instances(profile: ClusterProfile, degrees: dict) -> list:
    """simulator.py:127-158 build_instances order: machines in config order,
    k = 0..count/t-1.  Returns [(instance id, machine, t)]."""
    out = []
    for name, count, _mem, _acc in profile.machines:
        t = degrees[name]
        for k in range(count // t):
            out.append((f"{name}/{k}", name, t))
    return out
