"""Route the reference package's hot-path entry points through the engine.

This is INTEGRATION.md section 2's binding as code: ``install()`` rebinds, in
the reference package ``hetserve`` (/root/reference/pkg/src/hetserve), the
functions this engine replaces, so the reference's parsers, CLI, tests and
gateway keep working while the hot path runs on the GPU:

* ``planner.search_optimal_config`` (planner.py:202-228),
  ``planner.estimate_system_throughput`` (planner.py:143-181),
  ``planner.plan_static_batches`` (planner.py:51-87),
  ``planner.estimate_instance_throughput`` (planner.py:109-118);
* ``simulator.run_continuous`` (simulator.py:272-363) and
  ``simulator.run_static`` (simulator.py:206-250) -- the reference's own
  ``run_scenario`` / ``run_policy_comparison`` (simulator.py:366-380) call them
  through the module globals, so they route too;
* optionally ``scheduling.Scheduler`` (scheduling.py:175-346) -> the native
  host scheduler (``scheduler=True``).

Results come back as the reference's own dataclasses and failures as the
reference's own exception classes (same message and fields), so code written
against ``hetserve`` -- including its test-suite -- cannot tell the difference
except by speed.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import functools
import importlib
import sys

from . import domain as _dom

_PLANNER = ("search_optimal_config", "estimate_system_throughput", "plan_static_batches",
            "estimate_instance_throughput")
_SIMULATOR = ("run_continuous", "run_static")
_saved: dict = {}


def _ref_exception(exc: BaseException, E) -> BaseException:
    """The reference's exception for one of ours (errors.py:8-62)."""
    if isinstance(exc, _dom.InfeasibleConfigError):
        return E.InfeasibleConfigError(str(exc), machine=exc.machine, slack_bytes=exc.slack_bytes)
    if isinstance(exc, _dom.InfeasibleRequestError):
        return E.InfeasibleRequestError(str(exc), request_id=exc.request_id)
    if isinstance(exc, _dom.RankDeficientError):
        return E.RankDeficientError(str(exc), dimension=exc.dimension)
    for name in ("SchedulingError", "SpecError", "TraceError", "FitError", "InfeasibleError", "HetserveError"):
        if isinstance(exc, getattr(_dom, name)):
            return getattr(E, name)(str(exc))
    return exc


def _translated(fn, E):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except _dom.HetserveError as exc:
            raise _ref_exception(exc, E) from None
    return wrapper


def _ref_config(cfg, C):
    return C.DeploymentConfig(per_machine=tuple(
        C.MachinePlacement(machine=p.machine, tp_degree=p.tp_degree, instance_count=p.instance_count)
        for p in cfg.per_machine))


def _ref_estimate(est, P, C, config=None):
    return P.ThroughputEstimate(
        config=config if config is not None else _ref_config(est.config, C),
        per_machine=tuple(P.MachineEstimate(machine=m.machine, tp_degree=m.tp_degree, instance_count=m.instance_count,
                                            instance_tokens_per_sec=m.instance_tokens_per_sec,
                                            machine_tokens_per_sec=m.machine_tokens_per_sec,
                                            budget_bytes=m.budget_bytes, slack_bytes=m.slack_bytes)
                          for m in est.per_machine),
        system_tokens_per_sec=est.system_tokens_per_sec)


def _ref_metrics(m, S):
    return S.SimMetrics(
        policy=m.policy, mode=m.mode, rate=m.rate, system_throughput=m.system_throughput, makespan=m.makespan,
        completion_time_spread=m.completion_time_spread,
        per_instance=tuple(S.InstanceMetrics(id=i.id, completion_time=i.completion_time,
                                             request_count=i.request_count, token_count=i.token_count,
                                             peak_kv_usage=i.peak_kv_usage) for i in m.per_instance),
        assignments=m.assignments, request_times=m.request_times, residual_loads=m.residual_loads)


def bindings(hetserve, scheduler: bool = False) -> dict:
    """{(module, name): replacement} for the reference package `hetserve`."""
    from . import planner as gp
    from . import scheduling as gsch
    from . import simulator as gs
    P = importlib.import_module(hetserve.__name__ + ".planner")
    S = importlib.import_module(hetserve.__name__ + ".simulator")
    C = importlib.import_module(hetserve.__name__ + ".core")
    E = importlib.import_module(hetserve.__name__ + ".errors")

    def search_optimal_config(cluster, requests, params_by_machine_tp):
        out = gp.search_optimal_config(cluster, requests, params_by_machine_tp)
        return P.SearchOutcome(ranked=tuple(_ref_estimate(e, P, C) for e in out.ranked),
                               infeasible=tuple((_ref_config(c, C), reason) for c, reason in out.infeasible))

    def estimate_system_throughput(cluster, config, requests, params_by_machine_tp):
        # the caller's own config object is returned, as the reference does (planner.py:181)
        return _ref_estimate(gp.estimate_system_throughput(cluster, config, requests, params_by_machine_tp), P, C,
                             config=config)

    def plan_static_batches(requests, budget, model):
        return P.BatchPlan(batches=gp.plan_static_batches(requests, budget, model).batches)

    def estimate_instance_throughput(requests, budget, model, params):
        return gp.estimate_instance_throughput(requests, budget, model, params)

    def run_continuous(scenario):
        return _ref_metrics(gs.run_continuous(scenario), S)

    def run_static(scenario):
        return _ref_metrics(gs.run_static(scenario), S)

    out = {}
    for name, fn in (("search_optimal_config", search_optimal_config),
                     ("estimate_system_throughput", estimate_system_throughput),
                     ("plan_static_batches", plan_static_batches),
                     ("estimate_instance_throughput", estimate_instance_throughput)):
        out[(P, name)] = _translated(fn, E)
    for name, fn in (("run_continuous", run_continuous), ("run_static", run_static)):
        out[(S, name)] = _translated(fn, E)
    if scheduler:
        Sch = importlib.import_module(hetserve.__name__ + ".scheduling")

        class Scheduler(gsch.Scheduler):
            __doc__ = gsch.Scheduler.__doc__

        for meth in ("__init__", "evaluate", "choose", "complete", "snapshot", "loads", "running_totals",
                     "in_flight_count"):
            setattr(Scheduler, meth, _translated(getattr(gsch.Scheduler, meth), E))
        out[(Sch, "Scheduler")] = Scheduler
    return out


def install(hetserve=None, scheduler: bool = False) -> None:
    """Rebind the reference's hot-path functions (and, with scheduler=True,
    its Scheduler class) to the engine, in the defining modules, in the
    package namespace and in every already-imported hetserve module that
    imported the name (e.g. simulator's ``plan_static_batches``)."""
    if hetserve is None:
        hetserve = importlib.import_module("hetserve")
    prefix = hetserve.__name__
    for (mod, name), fn in bindings(hetserve, scheduler=scheduler).items():
        orig = getattr(mod, name)
        for m in [sys.modules[k] for k in list(sys.modules) if k == prefix or k.startswith(prefix + ".")]:
            if getattr(m, name, None) is orig:
                _saved.setdefault((m, name), orig)
                setattr(m, name, fn)


def uninstall() -> None:
    for (m, name), orig in list(_saved.items()):
        setattr(m, name, orig)
    _saved.clear()
