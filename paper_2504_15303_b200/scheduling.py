"""Scheduler types of the drop-in API, and the live scheduler.

Replayed traces are scheduled on the GPU inside the replay kernel
(csrc/replay.cu).  This module keeps the reference's configuration surface
(/root/reference/pkg/src/hetserve/scheduling.py:41-116): the policy record,
the output-length predictor and the instance handle.  The predictor is
evaluated host-side for a whole trace at once; its draws equal the
reference's one-draw-per-dispatch stream because dispatch order is trace
order and numpy's Generator produces the same sequence in bulk.

``Scheduler`` (scheduling.py:175-346) is the live, per-request scheduler the
reference's gateway calls; it runs natively (csrc/scheduler.cpp, hs_sched_*
in include/hetserve_b200.h) with the reference's checks, messages and
arithmetic and an O(N) min-max.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from .domain import KvBudget, LatencyParams, SchedulingError, SpecError, kv_bytes_per_token

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


def ideal_batch_size(request, budget, model) -> int:
    """scheduling.py:119-128."""
    if budget.total_bytes <= 0:
        raise SpecError(f"ideal_batch_size needs a positive budget, got {budget.total_bytes}")
    per_request = kv_bytes_per_token(model) * (request.input_len + request.predicted_output_len)
    return max(1, int(budget.total_bytes // per_request))


def request_oversized(request, budget, model) -> bool:
    """scheduling.py:131-133."""
    per_request = kv_bytes_per_token(model) * (request.input_len + request.predicted_output_len)
    return per_request > budget.total_bytes


def per_request_cost(params, request, batch_size: int) -> float:
    """scheduling.py:136-147."""
    from .domain import decode_time, prefill_time
    if batch_size < 1:
        raise SpecError(f"batch_size must be >= 1, got {batch_size}")
    total = prefill_time(params, batch_size, request.input_len) + decode_time(
        params, batch_size, request.input_len, request.predicted_output_len
    )
    if total <= 0:
        raise SpecError(
            f"non-positive batch time {total} for request {request.id!r}; latency parameters are corrupt"
        )
    return total / batch_size


def workload(cost: float, usage: float, theta: float) -> float:
    """scheduling.py:150-154."""
    if theta <= 0:
        raise SpecError(f"theta must be > 0, got {theta}")
    return cost * math.exp(theta * usage)


class _RunningView:
    """RunningTokens (capacity.py:33-55) of one native scheduler instance."""

    def __init__(self, sched, j: int):
        self._s, self._j = sched, j

    @property
    def input_sum(self) -> int:
        return self._s._get_state(self._j)[1]

    @input_sum.setter
    def input_sum(self, v: int) -> None:
        self._s._set_state(self._j, input_sum=int(v))

    @property
    def predicted_output_sum(self) -> int:
        return self._s._get_state(self._j)[2]

    @predicted_output_sum.setter
    def predicted_output_sum(self, v: int) -> None:
        self._s._set_state(self._j, pred_sum=int(v))

    def add(self, input_len: int, predicted_output_len: int) -> None:
        _l, i, p, _o = self._s._get_state(self._j)
        self._s._set_state(self._j, input_sum=i + input_len, pred_sum=p + predicted_output_len)

    def remove(self, input_len: int, predicted_output_len: int) -> None:
        _l, i, p, _o = self._s._get_state(self._j)
        i, p = i - input_len, p - predicted_output_len
        self._s._set_state(self._j, input_sum=i, pred_sum=p)
        if i < 0 or p < 0:
            raise SpecError("running token sums went negative; completion applied twice?")

    def total(self) -> int:
        _l, i, p, _o = self._s._get_state(self._j)
        return i + p


class _StateView:
    """scheduling.py:157-164 InstanceState of one native scheduler instance:
    reads and writes go to the native state (hs_sched_get/set_state,
    hs_sched_set_instance), so code that pokes Scheduler._states works."""

    def __init__(self, sched, j: int):
        self._s, self._j = sched, j

    @property
    def load(self) -> float:
        return self._s._get_state(self._j)[0]

    @load.setter
    def load(self, v: float) -> None:
        self._s._set_state(self._j, load=float(v))

    @property
    def running(self) -> _RunningView:
        return _RunningView(self._s, self._j)

    @property
    def oversized_count(self) -> int:
        return self._s._get_state(self._j)[3]

    @oversized_count.setter
    def oversized_count(self, v: int) -> None:
        self._s._set_state(self._j, oversized=int(v))

    @property
    def handle(self):
        return self._s._handles[self._j]

    @handle.setter
    def handle(self, h) -> None:
        self._s._set_handle(self._j, h)


class Scheduler:
    """scheduling.py:175-346 Scheduler over the native hs_sched_* engine:
    choose() / complete() / evaluate() / snapshot() with the reference's
    semantics; thread-safe (one native mutex, as the reference's _lock)."""

    def __init__(self, instances: list, model, policy: PolicyConfig | None = None):
        from . import _native as nat
        if not instances:
            raise SchedulingError("scheduler needs at least one instance")
        policy = policy or PolicyConfig()
        if policy.policy == "WRR" and len(policy.wrr_weights) != len(instances):
            raise SpecError(
                f"WRR needs one weight per instance ({len(instances)}), got {len(policy.wrr_weights)}"
            )
        for handle in instances:
            if handle.budget.total_bytes <= 0:
                raise SpecError(f"instance {handle.id!r} has a non-positive KV budget")
        self._nat = nat
        self._lib = nat.load_library()
        self._handles = list(instances)
        self._model = model
        self._policy = policy
        self._n = len(instances)
        arr = (nat.hs_instance * self._n)()
        for j, h in enumerate(instances):
            p = h.params
            for k, name in enumerate(("p1", "p2", "p3", "p4", "p5", "p6", "p7", "p8")):
                arr[j].p[k] = float(getattr(p, name))
            arr[j].budget = float(h.budget.total_bytes)
            arr[j].wrr_weight = float(policy.wrr_weights[j]) if policy.policy == "WRR" else 0.0
        pol = nat.hs_policy(nat.POLICY_CODE[policy.policy], self._n, float(policy.theta),
                            int(kv_bytes_per_token(model)), 0, 0)
        h = C.c_void_p()
        rc = self._lib.hs_sched_create(C.cast(arr, C.c_void_p), self._n, C.byref(pol), C.byref(h))
        if rc != nat.HS_OK:
            raise nat.EngineError(rc, "hs_sched_create: " + (self._lib.hs_last_error() or b"").decode())
        self._h = h
        self._st = nat.hs_sched_status()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.hs_sched_destroy(h)
            self._h = None

    @property
    def instances(self) -> list:
        return list(self._handles)

    @property
    def _states(self) -> list:
        """InstanceState views (scheduling.py:202), backed by the native state."""
        return [_StateView(self, j) for j in range(self._n)]

    def _get_state(self, j: int):
        load, i, p, o = C.c_double(), C.c_int64(), C.c_int64(), C.c_int64()
        rc = self._lib.hs_sched_get_state(self._h, j, C.byref(load), C.byref(i), C.byref(p), C.byref(o))
        if rc != self._nat.HS_OK:
            raise self._nat.EngineError(rc, "hs_sched_get_state: " + (self._lib.hs_last_error() or b"").decode())
        return load.value, i.value, p.value, o.value

    def _set_state(self, j: int, load=None, input_sum=None, pred_sum=None, oversized=None) -> None:
        cur = self._get_state(j)
        new = [cur[k] if v is None else v for k, v in enumerate((load, input_sum, pred_sum, oversized))]
        rc = self._lib.hs_sched_set_state(self._h, j, float(new[0]), int(new[1]), int(new[2]), int(new[3]))
        if rc != self._nat.HS_OK:
            raise self._nat.EngineError(rc, "hs_sched_set_state: " + (self._lib.hs_last_error() or b"").decode())

    def _set_handle(self, j: int, h) -> None:
        nat = self._nat
        rec = nat.hs_instance()
        for k, name in enumerate(("p1", "p2", "p3", "p4", "p5", "p6", "p7", "p8")):
            rec.p[k] = float(getattr(h.params, name))
        rec.budget = float(h.budget.total_bytes)
        rec.wrr_weight = float(self._policy.wrr_weights[j]) if self._policy.policy == "WRR" else 0.0
        rc = self._lib.hs_sched_set_instance(self._h, j, C.byref(rec))
        if rc != nat.HS_OK:
            raise nat.EngineError(rc, "hs_sched_set_instance: " + (self._lib.hs_last_error() or b"").decode())
        self._handles[j] = h

    @property
    def policy(self) -> PolicyConfig:
        return self._policy

    # ------------------------------------------------------------ internals
    def _allowed(self, allowed):
        if allowed is None:
            return None
        a = (C.c_uint8 * self._n)()
        for i in allowed:
            if isinstance(i, int) and 0 <= i < self._n:
                a[i] = 1
        return a

    def _raise(self, st, request=None, request_id=None):
        nat = self._nat
        code = st.error
        if code == nat.SCHED_OK:
            return
        if code == nat.SCHED_NO_INSTANCE:
            raise SchedulingError("no instance available for scheduling")
        if code == nat.SCHED_ALREADY_IN_FLIGHT:
            raise SchedulingError(f"request {request.id!r} is already in flight")
        if code == nat.SCHED_NOT_IN_FLIGHT:
            raise SchedulingError(f"request {request_id!r} is not in flight (double completion?)")
        if code == nat.SCHED_NONPOSITIVE_COST:
            raise SpecError(
                f"non-positive batch time {st.value} for request {request.id!r}; latency parameters are corrupt"
            )
        if code == nat.SCHED_EXP_OVERFLOW:
            raise OverflowError("math range error")
        if code == nat.SCHED_NEGATIVE_RUNNING:
            raise SpecError("running token sums went negative; completion applied twice?")
        if code == nat.SCHED_ZERO_DIVISION:
            raise ZeroDivisionError("float floor division by zero")
        raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, f"scheduler status {code}")

    # ------------------------------------------------------------------ API
    def evaluate(self, request, allowed: set | None = None) -> list:
        """Per-instance workload of this request (no state change)."""
        w = (C.c_double * self._n)()
        st = self._nat.hs_sched_status()
        rc = self._lib.hs_sched_evaluate(self._h, int(request.input_len), int(request.predicted_output_len),
                                         self._allowed(allowed), w, C.byref(st))
        if rc != self._nat.HS_OK:
            raise self._nat.EngineError(rc, "hs_sched_evaluate: " + (self._lib.hs_last_error() or b"").decode())
        self._raise(st, request=request)
        return list(w)

    def choose(self, request, allowed: set | None = None) -> int:
        """Pick an instance for the request and commit the dispatch bookkeeping."""
        rid = str(request.id).encode("utf-8", "surrogatepass")
        out = C.c_int32()
        st = self._nat.hs_sched_status()
        rc = self._lib.hs_sched_choose(self._h, rid, len(rid), int(request.input_len),
                                       int(request.predicted_output_len), self._allowed(allowed), C.byref(out),
                                       C.byref(st))
        if rc != self._nat.HS_OK:
            raise self._nat.EngineError(rc, "hs_sched_choose: " + (self._lib.hs_last_error() or b"").decode())
        self._raise(st, request=request)
        return int(out.value)

    def complete(self, request_id: str) -> None:
        """Fire the completion hook: subtract exactly what dispatch recorded."""
        rid = str(request_id).encode("utf-8", "surrogatepass")
        st = self._nat.hs_sched_status()
        rc = self._lib.hs_sched_complete(self._h, rid, len(rid), C.byref(st))
        if rc != self._nat.HS_OK:
            raise self._nat.EngineError(rc, "hs_sched_complete: " + (self._lib.hs_last_error() or b"").decode())
        self._raise(st, request_id=request_id)

    def _snap(self):
        n = self._n
        loads, usage = (C.c_double * n)(), (C.c_double * n)()
        running, over = (C.c_int64 * n)(), (C.c_int64 * n)()
        inflight = C.c_int64()
        self._lib.hs_sched_snapshot(self._h, loads, running, usage, over, C.byref(inflight))
        return list(loads), list(running), list(usage), list(over), int(inflight.value)

    def in_flight_count(self) -> int:
        return self._snap()[4]

    def snapshot(self) -> dict:
        """Consistent view of loads, KV usage, and in-flight work per instance."""
        loads, running, usage, over, inflight = self._snap()
        ids = [h.id for h in self._handles]
        return {
            "loads": dict(zip(ids, loads)),
            "kv_usage": dict(zip(ids, usage)),
            "running_tokens": dict(zip(ids, running)),
            "oversized": dict(zip(ids, over)),
            "in_flight": inflight,
        }

    def loads(self) -> list:
        return self._snap()[0]

    def running_totals(self) -> list:
        return self._snap()[1]
