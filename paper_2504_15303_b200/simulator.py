"""Cluster replay on the GPU, behind the reference's simulator API.

Drop-in entry points (reference /root/reference/pkg/src/hetserve/simulator.py):

* ``run_continuous(scenario)`` (simulator.py:272-363) -> SimMetrics, with
  assignments, departure times, per-instance metrics and residual loads
  bit-identical to the reference;
* ``run_scenario`` / ``run_policy_comparison`` (simulator.py:366-380);
* ``generate_arrivals`` / ``build_instances`` (simulator.py:112-158): host
  setup, same arithmetic as the reference.

Engine-level API: ``replay_traces(...)`` replays a batch of traces (one warp
each) on one deployment and returns arrays, for the batched-replay configs.

``run_static`` (simulator.py:206-250), the first "next" row of SURVEY.md
section 8f, runs on the same kernel in static mode.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import _native as nat
from . import streams
from .domain import (
    InfeasibleConfigError,
    InfeasibleRequestError,
    SchedulingError,
    SpecError,
    check_memory_constraint,
    kv_budget,
    kv_bytes_per_token,
)
from .scheduling import InstanceHandle, OutputLengthPredictor, PolicyConfig


@dataclass(frozen=True)
class Scenario:
    cluster: object
    config: object
    trace: tuple
    arrival_rate: float
    policy: PolicyConfig
    mode: str
    seed: int
    params: dict

    def __post_init__(self):
        if not self.trace:
            raise SpecError("scenario trace must be non-empty")
        if self.mode not in ("static", "continuous"):
            raise SpecError(f"mode must be 'static' or 'continuous', got {self.mode!r}")
        if not (self.arrival_rate > 0):
            raise SpecError(f"arrival rate must be positive or inf, got {self.arrival_rate}")


@dataclass(frozen=True)
class InstanceMetrics:
    id: str
    completion_time: float
    request_count: int
    token_count: int
    peak_kv_usage: float


@dataclass(frozen=True)
class SimMetrics:
    policy: str
    mode: str
    rate: float
    system_throughput: float
    makespan: float
    completion_time_spread: float
    per_instance: tuple
    assignments: tuple
    request_times: tuple
    residual_loads: tuple


def arrival_times(n: int, rate: float, seed: int) -> np.ndarray:
    """simulator.py:112-124 as an fp64 array: all 0.0 at rate=inf, else the
    running sum of seeded exponential gaps (np.cumsum is sequential)."""
    if math.isinf(rate):
        return np.zeros(n, np.float64)
    if rate <= 0:
        raise SpecError(f"arrival rate must be positive, got {rate}")
    rng = np.random.default_rng(seed)
    return np.cumsum(rng.exponential(1.0 / rate, size=n))


def generate_arrivals(trace, rate: float, seed: int) -> list:
    return [(r, float(t)) for r, t in zip(trace, arrival_times(len(trace), rate, seed))]


def build_instances(cluster, config, params) -> list:
    """Every deployed instance in config order (simulator.py:127-158)."""
    out = []
    for placement in config.per_machine:
        machine = cluster.machine(placement.machine)
        budget = kv_budget(machine, placement.tp_degree, cluster.model, cluster.engine)
        verdict = check_memory_constraint(budget, cluster.limits, cluster.model)
        if not verdict.feasible:
            raise InfeasibleConfigError(
                f"machine {machine.name!r} at tp={placement.tp_degree} cannot hold one maximal "
                f"request (slack {verdict.slack_bytes:.0f} bytes)",
                machine=machine.name,
                slack_bytes=verdict.slack_bytes,
            )
        key = (machine.name, placement.tp_degree)
        if key not in params:
            raise SpecError(f"no fitted parameters for machine {machine.name!r} at tp={placement.tp_degree}")
        for k in range(placement.instance_count):
            out.append(InstanceHandle(id=f"{machine.name}/{k}", machine=machine.name,
                                      tp_degree=placement.tp_degree, params=params[key], budget=budget))
    return out


def _params_tuple(p) -> tuple:
    return tuple(float(x) for x in (p.p1, p.p2, p.p3, p.p4, p.p5, p.p6, p.p7, p.p8))


def engine_instances(handles, policy: PolicyConfig):
    """hs_instance array: classes = bit-identical (params, budget), numbered in
    order of first appearance (the key is the bit pattern, so -0.0 and 0.0
    stay distinct classes)."""
    n = len(handles)
    arr = (nat.hs_instance * max(n, 1))()
    if n == 0:
        return arr
    pb = np.empty((n, 9), np.float64)
    for j, h in enumerate(handles):
        pb[j, :8] = _params_tuple(h.params)
        pb[j, 8] = float(h.budget.total_bytes)
    keys = np.ascontiguousarray(pb).view(np.uint64)
    _, first, inverse = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    rank = np.empty(len(first), np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(first))
    view = np.frombuffer(arr, dtype=nat.INSTANCE_DTYPE, count=n)
    view["p"] = pb[:, :8]
    view["budget"] = pb[:, 8]
    view["type"] = rank[np.asarray(inverse).reshape(-1)]
    if policy.policy == "WRR":
        view["wrr_weight"] = [float(policy.wrr_weights[j]) for j in range(n)]
    return arr


def _check_scheduler(handles, policy: PolicyConfig) -> None:
    """Scheduler.__init__ validation (scheduling.py:184-199)."""
    if not handles:
        raise SchedulingError("scheduler needs at least one instance")
    if policy.policy == "WRR" and len(policy.wrr_weights) != len(handles):
        raise SpecError(f"WRR needs one weight per instance ({len(handles)}), got {len(policy.wrr_weights)}")
    for h in handles:
        if h.budget.total_bytes <= 0:
            raise SpecError(f"instance {h.id!r} has a non-positive KV budget")


def _predictor(scenario) -> OutputLengthPredictor:
    cfg = scenario.policy.predictor
    if cfg.seed is None:
        cfg = replace(cfg, seed=scenario.seed)
    return OutputLengthPredictor(cfg, scenario.cluster.limits.max_output_len)


def _raise_trace_error(res, handles, trace, per_token, static=False) -> None:
    err = int(res["error"])
    if err == nat.TRACE_OK:
        return
    inst = int(res["err_instance"])
    ridx = int(res["err_request"])
    if err == nat.TRACE_INFEASIBLE_REQUEST:
        r = trace[ridx]
        need = r.input_len + r.output_len
        budget = handles[inst].budget.total_bytes
        if static:  # raised by plan_static_batches (planner.py:80-83)
            raise InfeasibleRequestError(
                f"request {r.id!r} needs {per_token * need:.0f} KV bytes alone, budget is {budget:.0f}",
                request_id=r.id,
            )
        raise InfeasibleRequestError(
            f"request {r.id!r} needs {per_token * need:.0f} KV bytes alone, budget of "
            f"instance {handles[inst].id!r} is {budget:.0f}",
            request_id=r.id,
        )
    if err == nat.TRACE_NONPOSITIVE_COST:
        total = float(res["err_value"])
        raise SpecError(
            f"non-positive batch time {total} for request {trace[ridx].id!r}; latency parameters are corrupt"
        )
    if err == nat.TRACE_EXP_OVERFLOW:
        raise OverflowError("math range error")
    if err == nat.TRACE_NO_INSTANCE:
        raise SchedulingError("no instance available for scheduling")
    if err == nat.TRACE_NEGATIVE_RUNNING:
        raise SpecError("running token sums went negative; completion applied twice?")
    raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, f"replay hit an engine limit (code {err})")


def _policy_struct(policy: PolicyConfig, n: int, per_token: int, mode: int = 0, flags: int = 0) -> nat.hs_policy:
    return nat.hs_policy(nat.POLICY_CODE[policy.policy], n, float(policy.theta), per_token, mode, flags)


def _first_duplicate_in_flight(ids, arr, key, static: bool):
    """Index of the first arrival whose request id is still in flight
    (Scheduler.choose raises before anything else, scheduling.py:239-240), or
    None.  An earlier request with the same id is in flight unless its
    retirement step popped before this arrival: the step's heap key (its
    time, or with negative step costs the running max of its busy period's
    step times) < the arrival time (arrivals pop first at equal times,
    simulator.py:285-290).  In static mode every dispatch precedes every
    completion (simulator.py:216-220)."""
    seen: dict = {}
    first = None
    for k, rid in enumerate(ids):
        prev = seen.get(rid)
        seen[rid] = k
        if prev is None:
            continue
        if static or not (key[prev] < arr[k]):  # NaN: never retired
            if first is None or k < first:
                first = k
    return first


def _duplicate_wins(a: int, res, arr, static: bool) -> bool:
    """Does the in-flight error at arrival `a` happen before the kernel's
    own failure (if any) in the reference's event order?"""
    err = int(res["error"])
    if err == nat.TRACE_OK:
        return True
    if err in (nat.TRACE_NONPOSITIVE_COST, nat.TRACE_EXP_OVERFLOW, nat.TRACE_NO_INSTANCE):
        return a <= int(res["err_request"])  # both at arrivals: the in-flight check runs first
    if static:
        return True  # planning failures come after every dispatch
    if err in (nat.TRACE_INFEASIBLE_REQUEST, nat.TRACE_NEGATIVE_RUNNING):
        return arr[a] <= float(res["err_value"])  # a step at the arrival's own time pops after it
    return True


def _run(scenario, static: bool, engine=None) -> SimMetrics:
    handles = build_instances(scenario.cluster, scenario.config, scenario.params)
    policy = scenario.policy
    _check_scheduler(handles, policy)
    N = len(handles)
    if N > nat.HS_MAX_INSTANCES:
        raise nat.EngineError(nat.HS_ERR_UNSUPPORTED,
                              f"{N} instances: the replay kernel handles up to {nat.HS_MAX_INSTANCES}")
    trace = scenario.trace
    ids = [r.id for r in trace]
    per_token = kv_bytes_per_token(scenario.cluster.model)
    I = np.fromiter((r.input_len for r in trace), np.int64, len(trace))
    O = np.fromiter((r.output_len for r in trace), np.int64, len(trace))
    for a in (I, O):
        if len(a) and a.max() > 2**31 - 1:
            raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, "request lengths above 2^31 - 1")
    eng = engine or nat.engine_for()
    # seeded draws on the device (rng.cu), bit-identical to the reference's
    # numpy streams: predictor (scheduling.py:87-95), arrivals (simulator.py:112-124)
    pred = _predictor(scenario)
    cfg = pred._config
    if cfg.mode == "normal":
        P = streams.predict_lengths([cfg.seed], [len(trace)], cfg.mean, cfg.stddev,
                                    scenario.cluster.limits.max_output_len, engine=eng).astype(np.int64)
    else:
        P = pred.predict_lengths(O)
    if not math.isinf(scenario.arrival_rate) and scenario.arrival_rate <= 0:
        raise SpecError(f"arrival rate must be positive, got {scenario.arrival_rate}")
    T = streams.arrival_times([scenario.seed], [len(trace)], scenario.arrival_rate, engine=eng)
    offsets = np.array([0, len(trace)], np.int64)
    # (time, heap key, per-instance sequence) per request; NaN = never retired
    dep_out = np.full(3 * len(trace), np.nan)
    assign, dep3, metrics, result = eng.replay(
        engine_instances(handles, policy),
        _policy_struct(policy, N, per_token, 1 if static else 0, nat.REPLAY_ORDER_KEYS), offsets,
        I.astype(np.int32), O.astype(np.int32), P.astype(np.int32),
        None if math.isinf(scenario.arrival_rate) else T, depart_out=dep_out)
    depart = dep3[:, 0]
    arr = T.tolist()
    dup = _first_duplicate_in_flight(ids, arr, dep3[:, 1].tolist(), static)
    if dup is not None and _duplicate_wins(dup, result[0], arr, static):
        raise SchedulingError(f"request {ids[dup]!r} is already in flight")
    _raise_trace_error(result[0], handles, trace, per_token, static=static)
    m = metrics[0]
    completion = m["completion_time"].tolist()
    req_count = m["request_count"].tolist()
    tok_count = m["token_count"].tolist()
    peak = m["peak_kv_usage"].tolist()
    if static:
        # simulator.py:229-245: times filled instance by instance, batch by batch
        order = np.lexsort((dep3[:, 2], assign.astype(np.int64)))
    else:
        # the reference's heap pop order of the retiring steps (simulator.py:285-355):
        # (heap key, instance index, per-instance retirement sequence)
        order = np.lexsort((dep3[:, 2], assign.astype(np.int64), dep3[:, 1]))
    dep = depart.tolist()
    # `times` is a dict keyed by request id (simulator.py:275, 337): a repeated
    # id keeps its first position and its last value
    times: dict = {}
    for k in order.tolist():
        times[ids[k]] = (0.0 if static else arr[k], dep[k])
    request_times = tuple((rid, a, d) for rid, (a, d) in times.items())
    makespan = max(completion) if completion else 0.0
    total_tokens = sum(tok_count)
    return SimMetrics(
        policy=policy.policy,
        mode=scenario.mode,
        rate=scenario.arrival_rate,
        system_throughput=total_tokens / makespan if makespan > 0 else math.inf,
        makespan=makespan,
        completion_time_spread=max(completion) - min(completion) if completion else 0.0,
        per_instance=tuple(
            InstanceMetrics(id=h.id, completion_time=completion[i], request_count=req_count[i],
                            token_count=tok_count[i], peak_kv_usage=peak[i])
            for i, h in enumerate(handles)
        ),
        assignments=tuple(assign.tolist()),
        request_times=request_times,
        residual_loads=tuple(m["residual_load"].tolist()),
    )


def run_continuous(scenario, engine=None) -> SimMetrics:
    """simulator.py:272-363 on the GPU (one trace, one warp)."""
    return _run(scenario, static=False, engine=engine)


def run_static(scenario, engine=None) -> SimMetrics:
    """simulator.py:206-250 on the GPU: the rate=inf dispatch sequence, then
    per-instance greedy static batches (planner.py:51-101)."""
    if not math.isinf(scenario.arrival_rate):
        raise SpecError("static mode needs arrival_rate=inf (a fully known queue)")
    return _run(scenario, static=True, engine=engine)


def run_scenario(scenario, engine=None) -> SimMetrics:
    if scenario.mode == "static":
        return run_static(scenario, engine=engine)
    return run_continuous(scenario, engine=engine)


def run_policy_comparison(scenario, policies, engine=None) -> list:
    """Each policy on the identical arrival / prediction realisation."""
    if not policies:
        raise SpecError("policy comparison needs at least one policy")
    return [run_scenario(replace(scenario, policy=replace(scenario.policy, policy=p)), engine=engine)
            for p in policies]


# ------------------------------------------------------------ batched API
@dataclass
class ReplayBatchResult:
    assign: np.ndarray | None      # [total requests] uint8
    depart: np.ndarray | None      # [total requests] float64
    metrics: np.ndarray            # [T, N] METRICS_DTYPE
    result: np.ndarray             # [T] RESULT_DTYPE
    kernel_ms: float


def replay_traces(cluster, config, params, policy: PolicyConfig, offsets, input_len, output_len, pred_output_len,
                  arrival=None, want_assign=True, want_depart=False, engine=None, static=False, rate=None,
                  arrival_seeds=None, predictor_seeds=None, assign_out=None, depart_out=None) -> ReplayBatchResult:
    """Replay T traces (offsets [T+1]) on one deployment in one launch.

    Arrivals are either given (``arrival``, fp64 per request; None = rate
    inf) or drawn on the device as generate_arrivals(trace_t, rate,
    arrival_seeds[t]) (simulator.py:112-124).  With policy.predictor in
    "normal" mode and ``predictor_seeds``, predictions are drawn on the
    device as OutputLengthPredictor (scheduling.py:87-95) seeded per trace,
    and pred_output_len may be None.  assign_out / depart_out: optional
    caller-owned result buffers (e.g. Engine.host_array, page-locked)."""
    handles = build_instances(cluster, config, params)
    _check_scheduler(handles, policy)
    N = len(handles)
    if N > nat.HS_MAX_INSTANCES:
        raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, f"{N} instances (max {nat.HS_MAX_INSTANCES})")
    per_token = kv_bytes_per_token(cluster.model)
    eng = engine or nat.engine_for()
    seeds = keep = None
    pred = policy.predictor
    dev_pred = predictor_seeds is not None and pred.mode == "normal"
    if dev_pred:
        OutputLengthPredictor(pred, cluster.limits.max_output_len)  # the reference's argument checks
    if (arrival_seeds is not None and rate is not None and not math.isinf(rate)) or dev_pred:
        if arrival is not None and arrival_seeds is not None:
            raise SpecError("give either arrival times or arrival seeds, not both")
        seeds, keep = streams.replay_seeds(arrival_seeds, math.inf if rate is None else rate,
                                           pred if dev_pred else None, predictor_seeds,
                                           cluster.limits.max_output_len)
    elif rate is not None and not math.isinf(rate) and arrival is None:
        raise SpecError("a finite rate needs arrival times or arrival seeds")
    P = None if dev_pred else np.ascontiguousarray(pred_output_len, np.int32)
    a, d, m, r = eng.replay(engine_instances(handles, policy), _policy_struct(policy, N, per_token, 1 if static else 0),
                            np.ascontiguousarray(offsets, np.int64), np.ascontiguousarray(input_len, np.int32),
                            np.ascontiguousarray(output_len, np.int32), P,
                            None if arrival is None else np.ascontiguousarray(arrival, np.float64),
                            want_assign=want_assign, want_depart=want_depart, seeds=seeds, assign_out=assign_out,
                            depart_out=depart_out)
    del keep
    return ReplayBatchResult(a, d, m, r, eng.last_kernel_ms)


def replay_deployments(cluster, configs, params, policy: PolicyConfig, trace_deployment, offsets, input_len,
                       output_len, pred_output_len, arrival=None, want_assign=True, want_depart=False, engine=None,
                       static=False, assign_out=None, depart_out=None) -> ReplayBatchResult:
    """Replay trace t on deployment configs[trace_deployment[t]] (BASELINE
    config 5: every top-k deployment re-scored by a full simulation), all
    traces in one launch.  metrics is [T, max instances].  assign_out /
    depart_out: caller buffers, as for replay_traces."""
    per_token = kv_bytes_per_token(cluster.model)
    inst_all, offs = [], [0]
    for cfg in configs:
        handles = build_instances(cluster, cfg, params)
        _check_scheduler(handles, policy)
        if len(handles) > nat.HS_MAX_INSTANCES:
            raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, f"{len(handles)} instances (max {nat.HS_MAX_INSTANCES})")
        inst_all.append(engine_instances(handles, policy))
        offs.append(offs[-1] + len(handles))
    arr = (nat.hs_instance * max(offs[-1], 1))()
    k = 0
    for part, n in zip(inst_all, np.diff(offs)):
        for j in range(n):
            arr[k] = part[j]
            k += 1
    eng = engine or nat.engine_for()
    pol = _policy_struct(policy, 0, per_token, 1 if static else 0)
    a, d, m, r = eng.replay_deployments(arr, np.array(offs, np.int32), pol, np.asarray(trace_deployment, np.int32),
                                        np.ascontiguousarray(offsets, np.int64),
                                        np.ascontiguousarray(input_len, np.int32),
                                        np.ascontiguousarray(output_len, np.int32),
                                        np.ascontiguousarray(pred_output_len, np.int32),
                                        None if arrival is None else np.ascontiguousarray(arrival, np.float64),
                                        want_assign=want_assign, want_depart=want_depart, assign_out=assign_out,
                                        depart_out=depart_out)
    return ReplayBatchResult(a, d, m, r, eng.last_kernel_ms)


def replay_candidates(tables, params_by_machine_tp, indices, policy: PolicyConfig, trace_deployment, offsets,
                      input_len, output_len, pred_output_len, arrival=None, want_assign=True, want_depart=False,
                      engine=None, assign_out=None, depart_out=None) -> ReplayBatchResult:
    """BASELINE config 5 (search -> re-score): replay trace t on
    candidate indices[trace_deployment[t]] of a search's tables, every
    deployment in one launch.  The instance arrays are assembled straight from
    the K1 table (budgets, instance counts per (machine, degree)) with numpy,
    instead of DeploymentConfig / InstanceHandle objects per candidate; the
    results equal replay_deployments on [deployment_of(tables, i) ...]."""
    if policy.policy == "WRR":
        raise SpecError("WRR weights are per instance: use replay_deployments")
    idx = np.asarray(indices, np.int64)
    M = len(tables.names)
    nd = np.asarray(tables.n_degrees, np.int64)
    ent = tables.entries
    digs = np.empty((len(idx), M), np.int64)
    x = idx.copy()
    for m in range(M - 1, -1, -1):
        digs[:, m] = x % nd[m]
        x //= nd[m]
    rows = np.arange(M)[None, :]
    if M > nat.HS_MAX_CLASSES or (ent["status"][rows, digs] != nat.ENTRY_OK).any():
        # not a set of feasible candidates: the object path raises the reference's errors
        from .planner import deployment_of
        configs = [deployment_of(tables, int(i)) for i in idx]
        return replay_deployments(tables.cluster, configs, params_by_machine_tp, policy, trace_deployment, offsets,
                                  input_len, output_len, pred_output_len, arrival, want_assign, want_depart, engine)
    p8 = np.zeros((M, nat.HS_MAX_DEGREES, 8), np.float64)
    for m, name in enumerate(tables.names):
        for d, t in enumerate(tables.degrees[m]):
            pr = params_by_machine_tp.get((name, t))
            if pr is not None:
                p8[m, d] = _params_tuple(pr)
    counts = ent["instance_count"][rows, digs].astype(np.int64)  # [K, M]
    n_per = counts.sum(axis=1)
    if len(n_per) and n_per.max() > nat.HS_MAX_INSTANCES:
        raise nat.EngineError(nat.HS_ERR_UNSUPPORTED, f"{int(n_per.max())} instances (max {nat.HS_MAX_INSTANCES})")
    inst_off = np.concatenate([[0], np.cumsum(n_per)]).astype(np.int32)
    flat = counts.reshape(-1)
    total = int(flat.sum())
    arr = (nat.hs_instance * max(total, 1))()
    view = np.frombuffer(arr, dtype=nat.INSTANCE_DTYPE, count=max(total, 1))[:total]
    view["p"] = np.repeat(p8[rows, digs].reshape(-1, 8), flat, axis=0)
    view["budget"] = np.repeat(ent["budget"][rows, digs].reshape(-1), flat)
    # instance classes = bit-identical (params, budget) within each deployment,
    # numbered densely per deployment (as engine_instances does)
    key = np.concatenate([p8, ent["budget"][:, :, None].astype(np.float64)], axis=2)  # [M, D, 9]
    _, gid = np.unique(np.ascontiguousarray(key).view(np.uint64).reshape(-1, 9), axis=0, return_inverse=True)
    g = np.asarray(gid).reshape(M, nat.HS_MAX_DEGREES)[rows, digs]  # [K, M] global class ids
    order = np.argsort(g, axis=1, kind="stable")
    gs = np.take_along_axis(g, order, axis=1)
    dense_sorted = np.concatenate([np.zeros((len(idx), 1), np.int64),
                                   np.cumsum(gs[:, 1:] != gs[:, :-1], axis=1)], axis=1)
    dense = np.empty_like(dense_sorted)
    np.put_along_axis(dense, order, dense_sorted, axis=1)
    view["type"] = np.repeat(dense.reshape(-1).astype(np.int32), flat)
    per_token = kv_bytes_per_token(tables.cluster.model)
    eng = engine or nat.engine_for()
    pol = _policy_struct(policy, 0, per_token, 0)
    a, d, m, r = eng.replay_deployments(arr, inst_off, pol, np.asarray(trace_deployment, np.int32),
                                        np.ascontiguousarray(offsets, np.int64),
                                        np.ascontiguousarray(input_len, np.int32),
                                        np.ascontiguousarray(output_len, np.int32),
                                        np.ascontiguousarray(pred_output_len, np.int32),
                                        None if arrival is None else np.ascontiguousarray(arrival, np.float64),
                                        want_assign=want_assign, want_depart=want_depart, assign_out=assign_out,
                                        depart_out=depart_out)
    return ReplayBatchResult(a, d, m, r, eng.last_kernel_ms)
