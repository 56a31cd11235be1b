"""Scheduler configuration types of the drop-in API.

The scheduling decisions themselves run on the GPU inside the replay kernel
(csrc/replay.cu).  This module keeps the reference's configuration surface
(/root/reference/pkg/src/hetserve/scheduling.py:41-116): the policy record,
the output-length predictor and the instance handle.  The predictor is
evaluated host-side for a whole trace at once; its draws equal the
reference's one-draw-per-dispatch stream because dispatch order is trace
order and numpy's Generator produces the same sequence in bulk.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .domain import KvBudget, LatencyParams, SpecError

POLICIES = ("OS", "RR", "WRR", "SI", "MB")


@dataclass(frozen=True)
class InstanceHandle:
    id: str
    machine: str
    tp_degree: int
    params: LatencyParams
    budget: KvBudget


@dataclass(frozen=True)
class PredictorConfig:
    mode: str = "oracle"
    mean: float | None = None
    stddev: float | None = None
    seed: int | None = None


@dataclass(frozen=True)
class PolicyConfig:
    policy: str = "OS"
    theta: float = 2.0
    wrr_weights: tuple | None = None
    predictor: PredictorConfig = field(default_factory=PredictorConfig)

    def __post_init__(self):
        if self.policy not in POLICIES:
            raise SpecError(f"unknown policy {self.policy!r}; expected one of {POLICIES}")
        if self.theta <= 0:
            raise SpecError(f"theta must be > 0, got {self.theta}")
        if self.policy == "WRR":
            if not self.wrr_weights:
                raise SpecError("WRR requires wrr_weights")
            if any(w <= 0 for w in self.wrr_weights):
                raise SpecError("wrr_weights must all be positive")


class OutputLengthPredictor:
    """oracle -> true length; mean -> round(mean); normal -> round(N(mean, sd))
    clamped to [1, max_output_len], one draw per request in dispatch order."""

    def __init__(self, config: PredictorConfig, max_output_len: int):
        if config.mode not in ("oracle", "mean", "normal"):
            raise SpecError(f"unknown predictor mode {config.mode!r}")
        if config.mode in ("mean", "normal") and config.mean is None:
            raise SpecError(f"predictor mode {config.mode!r} requires a mean")
        if config.mode == "normal" and config.stddev is None:
            raise SpecError("normal predictor requires a stddev")
        self._config = config
        self._max_output_len = max_output_len
        self._rng = np.random.default_rng(config.seed)

    @classmethod
    def from_config(cls, config: PredictorConfig, limits) -> "OutputLengthPredictor":
        return cls(config, limits.max_output_len)

    def predict(self, request) -> int:
        return int(self.predict_lengths(np.array([request.output_len], np.int64))[0])

    def predict_lengths(self, output_len: np.ndarray) -> np.ndarray:
        """Predictions for consecutive dispatches (int64 array)."""
        mode = self._config.mode
        if mode == "oracle":
            return np.asarray(output_len, np.int64).copy()
        n = len(output_len)
        if mode == "mean":
            v = np.full(n, float(round(self._config.mean)))
        else:
            v = np.rint(self._rng.normal(self._config.mean, self._config.stddev, size=n))
        return np.clip(v, 1, self._max_output_len).astype(np.int64)
