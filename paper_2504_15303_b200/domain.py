"""Domain model of the hot path: exception types, cluster / request types,
KV accounting and the latency model, as one module.

Public names, fields, validation and messages match the reference so the
engine is a drop-in (reference /root/reference/pkg/src/hetserve:
errors.py:8-62, core.py:45-165 and 363-390, capacity.py:58-106,
latency.py:36-109).  Out of scope here: file parsers
and latency fitting -- build these objects directly, or pass the reference's
own objects; every engine entry point reads them by attribute.

The search's per-(machine, degree) budget / feasibility is computed on the
GPU (csrc/search.cu K1).  The host helpers below serve instance setup (the
reference also computes instance budgets on the host, simulator.py:127-158)
and error messages, and evaluate the same expressions in the same order.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

# ----------------------------------------------------------------------
# errors
class HetserveError(Exception):
    """Root of every domain error raised by this package."""


class SpecError(HetserveError):
    """Malformed or invariant-violating spec / scenario / config input."""


class TraceError(HetserveError):
    """Malformed trace or parameter file (1-based line number in the text)."""


class FitError(HetserveError):
    """Latency-model fitting failed."""


class RankDeficientError(FitError):
    """Profiling design cannot identify every coefficient."""

    def __init__(self, message: str, dimension: str | None = None):
        super().__init__(message)
        self.dimension = dimension


class InfeasibleError(HetserveError):
    """Something cannot satisfy the KV-memory constraint."""


class InfeasibleRequestError(InfeasibleError):
    """One request cannot fit an instance's KV budget even alone."""

    def __init__(self, message: str, request_id: str):
        super().__init__(message)
        self.request_id = request_id


class InfeasibleConfigError(InfeasibleError):
    """A placement fails the per-instance memory constraint; slack_bytes < 0."""

    def __init__(self, message: str, machine: str, slack_bytes: float):
        super().__init__(message)
        self.machine = machine
        self.slack_bytes = slack_bytes


class SchedulingError(HetserveError):
    """Invalid scheduler operation (no candidate instance, ...)."""


# ----------------------------------------------------------------------
# core
def _positive_int(value, what: str) -> int:
    if isinstance(value, bool) or not isinstance(value, int):
        raise SpecError(f"{what} must be an integer, got {value!r}")
    if value <= 0:
        raise SpecError(f"{what} must be strictly positive, got {value}")
    return value


@dataclass(frozen=True)
class ModelSpec:
    layers: int
    hidden_dim: int
    param_count: int
    bytes_per_param: int

    def __post_init__(self):
        for name in ("layers", "hidden_dim", "param_count", "bytes_per_param"):
            _positive_int(getattr(self, name), f"model.{name}")


@dataclass(frozen=True)
class MachineSpec:
    name: str
    accelerator_count: int
    accelerator_mem_bytes: int
    accelerator_type: str = "generic"

    def __post_init__(self):
        if not self.name:
            raise SpecError("machine.name must be a non-empty string")
        _positive_int(self.accelerator_count, f"machine[{self.name}].accelerator_count")
        _positive_int(self.accelerator_mem_bytes, f"machine[{self.name}].accelerator_mem_bytes")


@dataclass(frozen=True)
class EngineOverheads:
    mem_utilization_fraction: float
    static_overhead_bytes: int

    def __post_init__(self):
        f = self.mem_utilization_fraction
        if not (isinstance(f, (int, float)) and 0.0 < float(f) <= 1.0):
            raise SpecError(f"engine.mem_utilization_fraction must be in (0, 1], got {f!r}")
        o = self.static_overhead_bytes
        if isinstance(o, bool) or not isinstance(o, int) or o < 0:
            raise SpecError(f"engine.static_overhead_bytes must be a non-negative integer, got {o!r}")


@dataclass(frozen=True)
class WorkloadLimits:
    max_input_len: int
    max_output_len: int

    def __post_init__(self):
        _positive_int(self.max_input_len, "limits.max_input_len")
        _positive_int(self.max_output_len, "limits.max_output_len")


@dataclass(frozen=True)
class Request:
    """Lengths of one request; the scheduler sees only predicted_output_len."""

    id: str
    input_len: int
    output_len: int
    predicted_output_len: int

    def __post_init__(self):
        if not self.id:
            raise SpecError("request.id must be a non-empty string")
        _positive_int(self.input_len, f"request[{self.id}].input_len")
        _positive_int(self.output_len, f"request[{self.id}].output_len")
        _positive_int(self.predicted_output_len, f"request[{self.id}].predicted_output_len")

    def with_prediction(self, predicted: int) -> "Request":
        return replace(self, predicted_output_len=predicted)


@dataclass(frozen=True)
class MachinePlacement:
    machine: str
    tp_degree: int
    instance_count: int


@dataclass(frozen=True)
class DeploymentConfig:
    per_machine: tuple

    def degree_for(self, machine: str) -> int:
        for p in self.per_machine:
            if p.machine == machine:
                return p.tp_degree
        raise SpecError(f"deployment config has no entry for machine {machine!r}")

    def describe(self) -> str:
        return ", ".join(f"{p.machine}:t{p.tp_degree}x{p.instance_count}" for p in self.per_machine)


@dataclass(frozen=True)
class ClusterSpec:
    model: ModelSpec
    engine: EngineOverheads
    machines: tuple
    limits: WorkloadLimits

    def machine(self, name: str) -> MachineSpec:
        for m in self.machines:
            if m.name == name:
                return m
        raise SpecError(f"unknown machine {name!r}")


def enumerate_tp_degrees(machine) -> list:
    """Powers of two t <= count with count % t == 0, ascending (core.py:363-371)."""
    count = machine.accelerator_count
    out, t = [], 1
    while t <= count:
        if count % t == 0:
            out.append(t)
        t <<= 1
    return out


def deployment_for(machines, degrees: dict) -> DeploymentConfig:
    """DeploymentConfig from {machine name: tp degree} (core.py:374-390)."""
    known = {m.name for m in machines}
    for name in degrees:
        if name not in known:
            raise SpecError(f"deployment names unknown machine {name!r}")
    out = []
    for m in machines:
        if m.name not in degrees:
            raise SpecError(f"deployment is missing a tensor-parallel degree for machine {m.name!r}")
        t = degrees[m.name]
        if t < 1 or m.accelerator_count % t != 0:
            raise SpecError(
                f"machine {m.name!r}: tp degree {t} does not divide accelerator count {m.accelerator_count}"
            )
        out.append(MachinePlacement(machine=m.name, tp_degree=t, instance_count=m.accelerator_count // t))
    return DeploymentConfig(per_machine=tuple(out))


# ----------------------------------------------------------------------
# capacity
@dataclass(frozen=True)
class KvBudget:
    total_bytes: float


@dataclass(frozen=True)
class FeasibilityVerdict:
    feasible: bool
    required_bytes: float
    slack_bytes: float


def kv_bytes_per_token(model) -> int:
    """2 (K and V) x layers x hidden x bytes per element."""
    return 2 * model.layers * model.hidden_dim * model.bytes_per_param


def kv_budget(machine, tp_degree: int, model, overheads) -> KvBudget:
    if tp_degree < 1 or machine.accelerator_count % tp_degree != 0:
        raise SpecError(
            f"tp degree {tp_degree} does not divide machine {machine.name!r}'s "
            f"accelerator count {machine.accelerator_count}"
        )
    usable = tp_degree * machine.accelerator_mem_bytes * overheads.mem_utilization_fraction
    return KvBudget(total_bytes=usable - overheads.static_overhead_bytes - model.param_count * model.bytes_per_param)


def check_memory_constraint(budget: KvBudget, limits, model) -> FeasibilityVerdict:
    need = kv_bytes_per_token(model) * (limits.max_input_len + limits.max_output_len)
    slack = budget.total_bytes - need
    return FeasibilityVerdict(feasible=slack >= 0, required_bytes=need, slack_bytes=slack)


# ----------------------------------------------------------------------
# latency
@dataclass(frozen=True)
class LatencyParams:
    """p1..p4 prefill (p1*b*I + p2*b + p3*I + p4); p5..p8 one decode step
    (p5*b*c + p6*b + p7*c + p8), seconds."""

    p1: float
    p2: float
    p3: float
    p4: float
    p5: float
    p6: float
    p7: float
    p8: float

    def as_tuple(self) -> tuple:
        return (self.p1, self.p2, self.p3, self.p4, self.p5, self.p6, self.p7, self.p8)

    def scaled(self, alpha: float) -> "LatencyParams":
        return LatencyParams(*(alpha * v for v in self.as_tuple()))


def prefill_time(params, batch_size: int, input_len: int) -> float:
    return params.p1 * batch_size * input_len + params.p2 * batch_size + params.p3 * input_len + params.p4


def decode_iteration_time(params, cached_len: int, batch_size: int) -> float:
    return params.p5 * batch_size * cached_len + params.p6 * batch_size + params.p7 * cached_len + params.p8


def decode_time(params, batch_size: int, input_len: int, output_len: int) -> float:
    """Closed form of sum_{k=1..O} decode_iteration_time(I + k, b)."""
    s = output_len * input_len + output_len * (output_len + 1) / 2.0
    return (params.p5 * batch_size + params.p7) * s + (params.p6 * batch_size + params.p8) * output_len


# ------------------------------------------------------ capacity.py helpers
@dataclass
class RunningTokens:
    """capacity.py:34-55: live token sums of an instance's unfinished requests."""

    input_sum: int = 0
    predicted_output_sum: int = 0

    def add(self, input_len: int, predicted_output_len: int) -> None:
        self.input_sum += input_len
        self.predicted_output_sum += predicted_output_len

    def remove(self, input_len: int, predicted_output_len: int) -> None:
        self.input_sum -= input_len
        self.predicted_output_sum -= predicted_output_len
        if self.input_sum < 0 or self.predicted_output_sum < 0:
            raise SpecError("running token sums went negative; completion applied twice?")

    def total(self) -> int:
        return self.input_sum + self.predicted_output_sum


def kv_usage(running, model, budget) -> float:
    """capacity.py:98-106 (unclamped)."""
    if budget.total_bytes <= 0:
        raise SpecError(f"kv_usage needs a positive budget, got {budget.total_bytes}")
    return kv_bytes_per_token(model) * running.total() / budget.total_bytes
