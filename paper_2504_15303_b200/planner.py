"""Deployment search on the GPU, behind the reference's planner API.

Drop-in entry points (reference /root/reference/pkg/src/hetserve/planner.py):

* ``search_optimal_config(cluster, requests, params_by_machine_tp)``
  (planner.py:202-228) -> SearchOutcome with the full ranking and the
  infeasible list, bit-identical totals;
* ``estimate_system_throughput(cluster, config, requests, params)``
  (planner.py:143-181) -> ThroughputEstimate.

Engine-level API for spaces too large to materialise:

* ``build_tables(...)`` -> SearchTables: K1 output, one entry per (machine,
  degree) = what estimate_system_throughput computes for that machine;
* ``search_best(tables, begin, end)`` -> (total, index, n_feasible): K2
  exhaustive argmax over a candidate-index range (shardable across GPUs).

Reasons for infeasible candidates are rebuilt host-side from the first
failing machine's entry with the reference's exact message formats
(planner.py:80-83, 157-162, 166; capacity.py:80-83).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .domain import (
    DeploymentConfig,
    InfeasibleConfigError,
    InfeasibleRequestError,
    MachinePlacement,
    SpecError,
    decode_time,
    enumerate_tp_degrees,
    kv_bytes_per_token,
    prefill_time,
)

MAX_MATERIALISED = 1 << 26  # candidates search_optimal_config ranks on the device (hs_search_rank's limit)


@dataclass(frozen=True)
class MachineEstimate:
    machine: str
    tp_degree: int
    instance_count: int
    instance_tokens_per_sec: float
    machine_tokens_per_sec: float
    budget_bytes: float
    slack_bytes: float


@dataclass(frozen=True)
class ThroughputEstimate:
    config: DeploymentConfig
    per_machine: tuple
    system_tokens_per_sec: float


@dataclass(frozen=True)
class SearchOutcome:
    """Feasible configs best-first (by -total, then tp tuple) plus failures."""

    ranked: tuple
    infeasible: tuple

    @property
    def best(self) -> ThroughputEstimate:
        if not self.ranked:
            raise InfeasibleConfigError("no feasible deployment configuration", machine="*", slack_bytes=0.0)
        return self.ranked[0]

    @property
    def candidates_visited(self) -> int:
        return len(self.ranked) + len(self.infeasible)


@dataclass
class SearchTables:
    """K1 output for one (cluster, trace, params) triple."""

    cluster: object
    requests: object
    names: list           # machine names, config order
    degrees: list         # per machine: list of tp degrees (radix digits)
    entries: np.ndarray   # [M, HS_MAX_DEGREES] of _native.ENTRY_DTYPE
    n_degrees: np.ndarray  # [M] int32
    kernel_ms: float = 0.0

    @property
    def space_size(self) -> int:
        n = 1
        for d in self.n_degrees:
            n *= int(d)
        return n

    def digits(self, index: int) -> list:
        out = []
        for nd in reversed(self.n_degrees.tolist()):
            out.append(index % nd)
            index //= nd
        return out[::-1]


def _model(cluster) -> nat.hs_model:
    m = cluster.model
    return nat.hs_model(m.layers, m.hidden_dim, m.param_count, m.bytes_per_param)


def _lengths(requests):
    I = np.fromiter((r.input_len for r in requests), dtype=np.int64, count=len(requests))
    O = np.fromiter((r.output_len for r in requests), dtype=np.int64, count=len(requests))
    if len(I) and (I.max() > 2**31 - 1 or O.max() > 2**31 - 1):
        raise SpecError("request lengths above 2^31 - 1 are not supported by the engine")
    return I.astype(np.int32), O.astype(np.int32)


def _run_tables(cluster, requests, params_by_machine_tp, placements=None, lengths=None, engine=None):
    """placements: None (every enumerated degree of every machine) or a list
    of MachinePlacement (one fixed degree each, explicit instance counts)."""
    machines = list(cluster.machines)
    first_index = {}
    for i, m in enumerate(machines):
        first_index.setdefault(m.name, i)
    if placements is None:
        rows = [(m.name, m.accelerator_count, 0) for m in machines]
        deg_lists = [enumerate_tp_degrees(m) for m in machines]
    else:
        rows, deg_lists = [], []
        for p in placements:
            if p.machine not in first_index:
                raise SpecError(f"unknown machine {p.machine!r}")
            rows.append((p.machine, p.tp_degree * p.instance_count if p.tp_degree > 0 else 1, p.tp_degree))
            deg_lists.append([p.tp_degree])
    M = len(rows)
    if M == 0 or M > nat.HS_MAX_MACHINES:
        raise SpecError(f"the engine handles 1..{nat.HS_MAX_MACHINES} machines, got {M}")
    arr = (nat.hs_machine * M)()
    params = np.zeros((M, nat.HS_MAX_DEGREES, 8), np.float64)
    present = np.zeros((M, nat.HS_MAX_DEGREES), np.uint8)
    for i, (name, count, fixed) in enumerate(rows):
        spec = machines[first_index[name]]
        arr[i].accelerator_count = count
        arr[i].accelerator_mem_bytes = spec.accelerator_mem_bytes
        arr[i].spec_index = first_index[name] if placements is None else i
        arr[i].fixed_degree = fixed
        for d, t in enumerate(deg_lists[i]):
            p = params_by_machine_tp.get((name, t))
            if p is not None:
                params[i, d] = [float(x) for x in (p.p1, p.p2, p.p3, p.p4, p.p5, p.p6, p.p7, p.p8)]
                present[i, d] = 1
    if placements is not None:
        # the spec machine (cluster.machine(name)) carries memory and the
        # divisibility check; encode it as that placement's own record
        for i, (name, _c, fixed) in enumerate(rows):
            spec = machines[first_index[name]]
            if fixed < 1 or spec.accelerator_count % fixed != 0:
                arr[i].accelerator_count = fixed if fixed > 0 else 1
                arr[i].fixed_degree = fixed if fixed > 0 else 1
                # marked below as a divisibility failure
    eng = engine or nat.engine_for()
    I, O = lengths if lengths is not None else _lengths(requests)
    lim = cluster.limits
    table, nd = eng.search_tables(_model(cluster), nat.hs_engine(float(cluster.engine.mem_utilization_fraction),
                                                                  cluster.engine.static_overhead_bytes),
                                  nat.hs_limits(lim.max_input_len, lim.max_output_len), arr, params, present, I, O)
    if placements is not None:
        for i, (name, _c, fixed) in enumerate(rows):
            spec = machines[first_index[name]]
            if fixed < 1 or spec.accelerator_count % fixed != 0:
                table[i, 0]["status"] = nat.ENTRY_BAD_DEGREE
    return [r[0] for r in rows], deg_lists, table, nd, eng.last_kernel_ms


def build_tables(cluster, requests, params_by_machine_tp, engine=None) -> SearchTables:
    """K1 on the GPU: every (machine, enumerated degree) entry."""
    names, degs, table, nd, ms = _run_tables(cluster, requests, params_by_machine_tp, engine=engine)
    return SearchTables(cluster, requests, names, degs, table, nd, ms)


# ------------------------------------------------------------ error messages
def _entry_exception(cluster, requests, name: str, t: int, e) -> Exception:
    """The exception estimate_system_throughput raises for this machine entry."""
    machine = cluster.machine(name)
    st = int(e["status"])
    if st == nat.ENTRY_INFEASIBLE_CONFIG:
        budget, slack = float(e["budget"]), float(e["slack"])
        return InfeasibleConfigError(
            f"machine {machine.name!r} at tp={t}: KV budget {budget:.0f} bytes is short by {-slack:.0f} "
            f"for one maximal request",
            machine=machine.name,
            slack_bytes=slack,
        )
    if st == nat.ENTRY_MISSING_PARAMS:
        return SpecError(f"no fitted parameters for machine {machine.name!r} at tp={t}")
    if st == nat.ENTRY_INFEASIBLE_REQUEST:
        r = requests[int(e["bad_request"])]
        per_token = kv_bytes_per_token(cluster.model)
        return InfeasibleRequestError(
            f"request {r.id!r} needs {per_token * (r.input_len + r.output_len):.0f} KV bytes alone, "
            f"budget is {float(e['budget']):.0f}",
            request_id=r.id,
        )
    if st == nat.ENTRY_BAD_DEGREE:
        return SpecError(
            f"tp degree {t} does not divide machine {machine.name!r}'s accelerator count {machine.accelerator_count}"
        )
    if st == nat.ENTRY_ZERO_DIVISION:
        return ZeroDivisionError("division by zero" if int(e["zero_div_int"]) else "float division by zero")
    raise AssertionError(f"entry status {st} is not an error")


# ------------------------------------------------- single-instance planning
@dataclass(frozen=True)
class BatchPlan:
    """planner.py:36-48: contiguous batches (half-open index ranges) and,
    once timed, their seconds."""

    batches: tuple = ()
    per_batch_time: tuple = ()

    @property
    def total_time(self) -> float:
        return sum(self.per_batch_time)


def _plan_on_device(requests, budget, model, params, engine):
    I, O = _lengths(requests)
    per_token = kv_bytes_per_token(model)
    p8 = None if params is None else [float(getattr(params, f"p{k}")) for k in range(1, 9)]
    eng = engine or nat.engine_for()
    stops, times, e = eng.plan_instance(float(budget.total_bytes), per_token, p8, I, O)
    if int(e["status"]) == nat.ENTRY_INFEASIBLE_REQUEST:
        r = requests[int(e["bad_request"])]
        raise InfeasibleRequestError(
            f"request {r.id!r} needs {per_token * (r.input_len + r.output_len):.0f} KV bytes alone, "
            f"budget is {budget.total_bytes:.0f}",
            request_id=r.id,
        )
    starts = [0] + [int(x) for x in stops[:-1]]
    batches = tuple(zip(starts, (int(x) for x in stops)))
    return batches, times, e


def plan_static_batches(requests, budget, model, engine=None) -> BatchPlan:
    """planner.py:51-87 on the GPU (K1's warp-cooperative greedy scan): the
    largest KV-feasible contiguous batches, in order."""
    batches, _times, _e = _plan_on_device(list(requests), budget, model, None, engine)
    return BatchPlan(batches=batches)


def estimate_batch_time(batch, params) -> float:
    """planner.py:90-101 for one batch (host scalar helper)."""
    if not batch:
        raise SpecError("cannot time an empty batch")
    b = len(batch)
    max_i = max(r.input_len for r in batch)
    max_o = max(r.output_len for r in batch)
    return prefill_time(params, b, max_i) + decode_time(params, b, max_i, max_o)


def time_batches(plan: BatchPlan, requests, params) -> BatchPlan:
    """planner.py:104-106 (host scalar helper over the plan's batches)."""
    requests = list(requests)
    return BatchPlan(batches=plan.batches,
                     per_batch_time=tuple(estimate_batch_time(requests[s:e], params) for s, e in plan.batches))


def estimate_instance_throughput(requests, budget, model, params, engine=None) -> float:
    """planner.py:109-118 on the GPU: plan, time and sum the static batches of
    one instance (K1's scan with an explicit KV budget, hs_plan_instance)."""
    _batches, _times, e = _plan_on_device(list(requests), budget, model, params, engine)
    if int(e["status"]) == nat.ENTRY_ZERO_DIVISION:
        raise ZeroDivisionError("division by zero" if int(e["zero_div_int"]) else "float division by zero")
    return float(e["rate"])


def _machine_estimate(name: str, t: int, e) -> MachineEstimate:
    return MachineEstimate(
        machine=name,
        tp_degree=t,
        instance_count=int(e["instance_count"]),
        instance_tokens_per_sec=float(e["rate"]),
        machine_tokens_per_sec=float(e["contribution"]),
        budget_bytes=float(e["budget"]),
        slack_bytes=float(e["slack"]),
    )


def _fatal_zero_division(tables: SearchTables):
    """search_optimal_config only catches InfeasibleConfigError,
    InfeasibleRequestError and SpecError (planner.py:225); a ZeroDivisionError
    from the first candidate (product order) whose first non-OK machine
    divides by zero escapes.  Such a candidate exists iff some machine i has
    a zero-division entry and every machine before i has an OK degree."""
    for i in range(len(tables.names)):
        row = tables.entries[i, : tables.n_degrees[i]]
        for d in range(len(row)):
            if int(row[d]["status"]) == nat.ENTRY_ZERO_DIVISION:
                return _entry_exception(tables.cluster, tables.requests, tables.names[i], tables.degrees[i][d], row[d])
        if not (row["status"] == nat.ENTRY_OK).any():
            return None
    return None


def _config_for(tables: SearchTables, digits: list) -> DeploymentConfig:
    machines = tables.cluster.machines
    return DeploymentConfig(
        per_machine=tuple(
            MachinePlacement(machine=m.name, tp_degree=tables.degrees[i][d],
                             instance_count=m.accelerator_count // tables.degrees[i][d])
            for i, (m, d) in enumerate(zip(machines, digits))
        )
    )


# --------------------------------------------------------------- drop-ins
def search_optimal_config(cluster, requests, params_by_machine_tp, engine=None) -> SearchOutcome:
    """planner.py:202-228 on the GPU: K1 table build, then every candidate of
    the product space scored (left-to-right fp64 sum, planner.py:151,180) and
    ranked by (-total, index) on the device."""
    tables = build_tables(cluster, requests, params_by_machine_tp, engine=engine)
    fatal = _fatal_zero_division(tables)
    if fatal is not None:
        raise fatal
    P = tables.space_size
    if P > MAX_MATERIALISED:
        raise SpecError(
            f"candidate space of {P} configurations is too large to materialise; use "
            f"planner.build_tables + planner.search_best"
        )
    eng = engine or nat.engine_for()
    ranked_arr, first_bad = eng.search_rank(tables.entries, tables.n_degrees)
    # frozen per-(machine, digit) pieces are shared between candidates
    machines = tables.cluster.machines
    place = [[MachinePlacement(machine=m.name, tp_degree=t, instance_count=m.accelerator_count // t)
              for t in tables.degrees[i]] for i, m in enumerate(machines)]
    est = [[_machine_estimate(tables.names[i], t, tables.entries[i, d]) for d, t in enumerate(tables.degrees[i])]
           for i in range(len(machines))]
    nd = [int(x) for x in tables.n_degrees]

    def digits_of(idx: int) -> list:
        out = [0] * len(nd)
        for i in range(len(nd) - 1, -1, -1):
            idx, out[i] = divmod(idx, nd[i])
        return out

    ranked = []
    for total, idx in zip(ranked_arr["total"].tolist(), ranked_arr["index"].tolist()):
        digits = digits_of(idx)
        ranked.append(ThroughputEstimate(
            config=DeploymentConfig(per_machine=tuple(place[i][d] for i, d in enumerate(digits))),
            per_machine=tuple(est[i][d] for i, d in enumerate(digits)), system_tokens_per_sec=total))
    infeasible = []
    cache = {}
    for c in np.nonzero(first_bad >= 0)[0].tolist():
        digits = digits_of(c)
        i = int(first_bad[c])
        key = (i, digits[i])
        if key not in cache:
            cache[key] = str(_entry_exception(cluster, requests, tables.names[i], tables.degrees[i][digits[i]],
                                              tables.entries[i, digits[i]]))
        infeasible.append((DeploymentConfig(per_machine=tuple(place[k][d] for k, d in enumerate(digits))),
                           cache[key]))
    return SearchOutcome(ranked=tuple(ranked), infeasible=tuple(infeasible))


def estimate_system_throughput(cluster, config, requests, params_by_machine_tp, engine=None) -> ThroughputEstimate:
    """planner.py:143-181: per placement (config order) the K1 entry; the
    first failing placement raises its exception; total = left-to-right sum."""
    placements = list(config.per_machine)
    for p in placements:
        cluster.machine(p.machine)  # SpecError for unknown names, in order
    names, degs, table, nd, _ms = _run_tables(cluster, requests, params_by_machine_tp, placements=placements,
                                              engine=engine)
    per_machine = []
    total = 0.0
    for i, p in enumerate(placements):
        e = table[i, 0]
        if int(e["status"]) != nat.ENTRY_OK:
            raise _entry_exception(cluster, requests, p.machine, p.tp_degree, e)
        est = _machine_estimate(cluster.machine(p.machine).name, p.tp_degree, e)
        per_machine.append(est)
        total += est.machine_tokens_per_sec
    return ThroughputEstimate(config=config, per_machine=tuple(per_machine), system_tokens_per_sec=total)


def search_best(tables: SearchTables, begin: int = 0, end: int | None = None, engine=None):
    """K2: exhaustive argmax over candidate indices [begin, end).  Returns
    (best_total, best_index or -1, n_feasible, kernel_ms)."""
    end = tables.space_size if end is None else end
    eng = engine or nat.engine_for()
    total, idx, nfeas = eng.search_best(tables.entries, tables.n_degrees, begin, end)
    return total, idx, nfeas, eng.last_kernel_ms


def search_topk(tables: SearchTables, k: int, shard: int = 0, n_shards: int = 1, engine=None):
    """Top-k of planner.py:227's ranking (total desc, index asc) over one
    shard of the feasible sub-product.  Returns (cands, n_feasible,
    kernel_ms) with cands a structured array of (total, index)."""
    eng = engine or nat.engine_for()
    cands, nf = eng.search_topk(tables.entries, tables.n_degrees, k, shard, n_shards)
    return cands, nf, eng.last_kernel_ms


def merge_topk(parts, k: int) -> np.ndarray:
    """Merge per-shard top-k lists (same order rule)."""
    allc = np.concatenate([p for p in parts if len(p)]) if any(len(p) for p in parts) else np.zeros(0, nat.CAND_DTYPE)
    order = sorted(range(len(allc)), key=lambda j: (-float(allc[j]["total"]), int(allc[j]["index"])))
    return allc[order[:k]]


def best_config(tables: SearchTables, index: int) -> ThroughputEstimate:
    """The ThroughputEstimate of candidate `index` (as search_optimal_config
    would report it), from the table."""
    digits = tables.digits(index)
    per_machine = []
    total = 0.0
    for i, d in enumerate(digits):
        e = tables.entries[i, d]
        if int(e["status"]) != nat.ENTRY_OK:
            raise _entry_exception(tables.cluster, tables.requests, tables.names[i], tables.degrees[i][d], e)
        est = _machine_estimate(tables.names[i], tables.degrees[i][d], e)
        per_machine.append(est)
        total += est.machine_tokens_per_sec
    return ThroughputEstimate(config=_config_for(tables, digits), per_machine=tuple(per_machine),
                              system_tokens_per_sec=total)


def deployment_of(tables: SearchTables, index: int) -> DeploymentConfig:
    """The DeploymentConfig of candidate `index` (itertools.product order)."""
    return _config_for(tables, tables.digits(index))


# ------------------------------------------------ streamed ranking / report
def iter_ranked(tables: SearchTables, chunk: int = 1 << 16, engine=None):
    """planner.py:227's ranking of a space of any size, streamed best-first
    in chunks of (total, index) (hs_search_topk_after: each chunk is the top
    of what ranks after the previous chunk's last candidate).  Only feasible
    candidates are ranked (planner.py:225-226)."""
    eng = engine or nat.engine_for()
    after = None
    while True:
        cands, _nf = eng.search_topk_after(tables.entries, tables.n_degrees, chunk, after)
        if len(cands) == 0:
            return
        yield cands
        after = (float(cands["total"][-1]), int(cands["index"][-1]))


def iter_infeasible(tables: SearchTables, chunk: int = 1 << 20):
    """The infeasible candidates in product order (planner.py:216-226) with the
    reason search_optimal_config records for each (the first failing
    machine's exception, planner.py:152-166), in chunks of (indices, first
    failing machine, its digit) from the per-(machine, degree) statuses."""
    nd = np.asarray(tables.n_degrees, np.int64)
    ok = tables.entries["status"] == nat.ENTRY_OK  # [M, HS_MAX_DEGREES]
    P = tables.space_size
    M = len(nd)
    for lo in range(0, P, chunk):
        idx = np.arange(lo, min(P, lo + chunk), dtype=np.int64)
        digs = np.empty((len(idx), M), np.int64)
        x = idx.copy()
        for m in range(M - 1, -1, -1):
            digs[:, m] = x % nd[m]
            x //= nd[m]
        bad = ~ok[np.arange(M)[None, :], digs]
        anyb = bad.any(axis=1)
        first = np.argmax(bad, axis=1)
        sel = np.nonzero(anyb)[0]
        if len(sel):
            yield idx[sel], first[sel], digs[sel, first[sel]]


def write_plan_report(tables: SearchTables, out, engine=None, chunk: int = 1 << 16) -> int:
    """`hetserve plan --out` (cli.py:70-109: one json.dumps(sort_keys=True)
    line per _plan_records record, ranked then infeasible) streamed from the
    device ranking, for spaces too large to materialise as a SearchOutcome.
    `out` is a binary file object; returns the number of records."""
    import json

    fatal = _fatal_zero_division(tables)
    if fatal is not None:
        raise fatal
    names = tables.names
    counts = [m.accelerator_count for m in tables.cluster.machines]
    pm = [[{"machine": names[i], "tp_degree": t, "instance_count": int(tables.entries[i, d]["instance_count"]),
            "instance_tokens_per_sec": float(tables.entries[i, d]["rate"]),
            "machine_tokens_per_sec": float(tables.entries[i, d]["contribution"]),
            "slack_bytes": float(tables.entries[i, d]["slack"])}
           for d, t in enumerate(tables.degrees[i])] for i in range(len(names))]
    del counts
    nd = [int(x) for x in tables.n_degrees]

    def digits_of(idx: int) -> list:
        o = [0] * len(nd)
        for i in range(len(nd) - 1, -1, -1):
            idx, o[i] = divmod(idx, nd[i])
        return o

    n = 0
    for cands in iter_ranked(tables, chunk=chunk, engine=engine):
        lines = []
        for total, idx in zip(cands["total"].tolist(), cands["index"].tolist()):
            dg = digits_of(idx)
            n += 1
            rec = {"rank": n, "config": {names[i]: tables.degrees[i][d] for i, d in enumerate(dg)},
                   "system_tokens_per_sec": total, "per_machine": [pm[i][d] for i, d in enumerate(dg)]}
            lines.append(json.dumps(rec, sort_keys=True))
        out.write(("\n".join(lines) + "\n").encode())
    reasons = {}
    for idx, first, fdig in iter_infeasible(tables):
        lines = []
        for c, i, d in zip(idx.tolist(), first.tolist(), fdig.tolist()):
            key = (i, d)
            if key not in reasons:
                reasons[key] = str(_entry_exception(tables.cluster, tables.requests, names[i], tables.degrees[i][d],
                                                    tables.entries[i, d]))
            dg = digits_of(c)
            rec = {"config": {names[k]: tables.degrees[k][x] for k, x in enumerate(dg)}, "infeasible": reasons[key]}
            lines.append(json.dumps(rec, sort_keys=True))
            n += 1
        out.write(("\n".join(lines) + "\n").encode())
    return n
