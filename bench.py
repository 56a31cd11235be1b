#!/usr/bin/env python
"""Benchmark: deployment configs evaluated/sec + simulated requests/sec.

One step = one pass of the hot path over one batch of synthetic input:
  * search   -- BASELINE config 3 (8 accelerator types x 2 machines x 16
                GPUs, 70B-class, 10k-request trace): K1 table build and K2
                exhaustive argmax over all 5^16 = 1.53e11 candidates;
  * replay   -- BASELINE config 4 (4096 Poisson traces x 100k requests at
                140 req/s on 32 heterogeneous instances, OS policy): K3;
  * combine  -- per-GPU search winners reduced with one NCCL all-reduce.
Units per step = candidates evaluated + requests simulated (dispatched and
run to completion); value = units / step time (max over ranks).  N GPUs
split the candidate range and the trace batch (strong scaling: the total
work is fixed).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "deployment configs evaluated/sec + simulated requests/sec at 1/2/4/8 B200"
UNIT = "(configs + requests)/s"
BYTES_PER_DISPATCH = 21  # I, O, Opred int32 + arrival fp64 + assignment u8


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--traces", type=int, default=4096)
    ap.add_argument("--q", type=int, default=100_000)
    ap.add_argument("--rate", type=float, default=140.0)
    ap.add_argument("--search-q", type=int, default=10_000)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample duration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--topk", type=int, default=1024)
    ap.add_argument("--no-config5", action="store_true", help="skip the config-5 sub-record of the default line")
    return ap.parse_args()


# ----------------------------------------------------------------- inputs
def search_inputs(q: int):
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import workloads as wl
    prof = wl.config3()
    cluster = hs.ClusterSpec(
        model=hs.ModelSpec(**prof.model), engine=hs.EngineOverheads(**prof.engine),
        machines=tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
        limits=hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    I, O = wl.trace_lengths(q, seed=3)
    reqs = [hs.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q)]
    return cluster, reqs, params, I, O


def replay_deployment():
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import workloads as wl
    prof = wl.config4()
    cluster = hs.ClusterSpec(
        model=hs.ModelSpec(**prof.model), engine=hs.EngineOverheads(**prof.engine),
        machines=tuple(hs.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
        limits=hs.WorkloadLimits(**prof.limits))
    params = {k: hs.LatencyParams(*v) for k, v in prof.params.items()}
    config = hs.deployment_for(cluster.machines, {a: 1 for a in wl.CONFIG4_TYPES})
    return cluster, config, params


def replay_inputs(t_lo: int, t_hi: int, q: int, rate: float, out=None):
    """Traces t_lo..t_hi-1: lengths seeded by trace index, arrivals by 42+t."""
    from paper_2504_15303_b200 import workloads as wl
    n = t_hi - t_lo
    if out is None:
        out = (np.empty(n * q, np.int32), np.empty(n * q, np.int32), np.empty(n * q, np.float64))
    I, O, T = out

    def one(k):
        t = t_lo + k
        i, o = wl.trace_lengths(q, seed=t)
        I[k * q:(k + 1) * q] = i
        O[k * q:(k + 1) * q] = o
        T[k * q:(k + 1) * q] = wl.arrivals(q, rate, seed=42 + t)

    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        list(ex.map(one, range(n)))
    offsets = np.arange(n + 1, dtype=np.int64) * q
    return offsets, I, O, T


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU baselines
# (1) the reference itself: the unmodified Python package vendored in
#     baseline/_ref (tools/vendor_reference.py), on every host core through a
#     process pool -- kind "reference";
# (2) the reference's algorithm restated in C (oracle/, test infrastructure)
#     on every host core -- kind "port".
# Both run outside the timed regions of the engine.
REF_DIR = ROOT / "baseline" / "_ref"
_REF: dict = {}


def _ref_cluster(H, prof):
    return H.ClusterSpec(model=H.ModelSpec(**prof.model), engine=H.EngineOverheads(**prof.engine),
                         machines=tuple(H.MachineSpec(n, c, m, a) for n, c, m, a in prof.machines),
                         limits=H.WorkloadLimits(**prof.limits))


def _ref_init(q_search: int, rate: float):
    """Pool worker setup: the reference's own objects for config 3 (search)
    and config 4 (replay), built once per worker."""
    sys.path.insert(0, str(REF_DIR))
    import hetserve as H
    import hetserve.simulator as HS
    from paper_2504_15303_b200 import workloads as wl
    p3 = wl.config3()
    c3 = _ref_cluster(H, p3)
    I, O = wl.trace_lengths(q_search, seed=3)
    p4 = wl.config4()
    c4 = _ref_cluster(H, p4)
    _REF.update(H=H, HS=HS, wl=wl, c3=c3, params3={k: H.LatencyParams(*v) for k, v in p3.params.items()},
                reqs3=[H.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q_search)],
                degs3=[H.enumerate_tp_degrees(m) for m in c3.machines], c4=c4,
                cfg4=H.deployment_for(c4.machines, {a: 1 for a in wl.CONFIG4_TYPES}),
                params4={k: H.LatencyParams(*v) for k, v in p4.params.items()}, rate=rate)


def _ref_candidates(indices) -> float:
    """The body of the reference's search loop (planner.py:216-226) for the
    given mixed-radix indices: deployment_for -> estimate_system_throughput,
    infeasibility exceptions caught and turned into their message."""
    H, c3, degs = _REF["H"], _REF["c3"], _REF["degs3"]
    names = [m.name for m in c3.machines]
    t0 = time.perf_counter()
    for idx in indices:
        idx = int(idx)
        dig = [0] * len(degs)
        for i in range(len(degs) - 1, -1, -1):
            idx, dig[i] = divmod(idx, len(degs[i]))
        config = H.deployment_for(c3.machines, {n: degs[i][d] for i, (n, d) in enumerate(zip(names, dig))})
        try:
            H.estimate_system_throughput(c3, config, _REF["reqs3"], _REF["params3"])
        except (H.InfeasibleConfigError, H.InfeasibleRequestError, H.SpecError) as exc:
            str(exc)
    return time.perf_counter() - t0


def _ref_replay(task) -> float:
    """The reference's run_continuous on config-4 trace t (gen-trace lengths
    seeded t, arrivals seeded 42 + t), truncated to q requests."""
    t, q = task
    H, HS, wl = _REF["H"], _REF["HS"], _REF["wl"]
    I, O = wl.trace_lengths(100_000, seed=t)
    trace = tuple(H.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q))
    sc = HS.Scenario(cluster=_REF["c4"], config=_REF["cfg4"], trace=trace, arrival_rate=_REF["rate"],
                     policy=H.PolicyConfig(), mode="continuous", seed=42 + t, params=_REF["params4"])
    t0 = time.perf_counter()
    HS.run_continuous(sc)
    return time.perf_counter() - t0


class RefPool:
    """A fork pool of reference workers on every host core."""

    def __init__(self, rate: float, q_search: int = 10_000):
        import multiprocessing as mp
        self.cores = len(os.sched_getaffinity(0))
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_ref_init, initargs=(q_search, rate))

    def close(self):
        self.pool.terminate()

    def sample(self, P: int, feasible_digits, f_feasible: float, n_uniform: int, n_feasible: int, n_traces: int,
               q_trace: int, rng) -> dict:
        """Per-candidate cost of the reference's search loop, stratified: a
        uniform sample of candidate indices (the infeasible ~all of the space)
        plus a sample of feasible candidates, weighted by the exact feasible
        fraction; and run_continuous throughput on n_traces traces of
        q_trace requests.  Wall-clock over all cores."""
        cores = self.cores
        uni = rng.integers(0, P, n_uniform)
        t0 = time.perf_counter()
        self.pool.map(_ref_candidates, np.array_split(uni, cores))
        w_uni = time.perf_counter() - t0
        fea = feasible_digits(rng, n_feasible)
        t0 = time.perf_counter()
        self.pool.map(_ref_candidates, np.array_split(fea, cores))
        w_fea = time.perf_counter() - t0
        # wall seconds per candidate on all cores, stratified by feasibility
        per_cand = (1.0 - f_feasible) * (w_uni / n_uniform) + f_feasible * (w_fea / max(n_feasible, 1))
        t0 = time.perf_counter()
        self.pool.map(_ref_replay, [(t, q_trace) for t in range(n_traces)], chunksize=1)
        w_rep = time.perf_counter() - t0
        return {"configs_per_s": 1.0 / per_cand, "requests_per_s": n_traces * q_trace / w_rep,
                "desc": (f"the unmodified reference (baseline/_ref, Python {sys.version.split()[0]}) in a {cores}-process "
                         f"pool: search loop body (planner.py:216-226) on {n_uniform} uniform + {n_feasible} feasible "
                         f"config-3 candidates, stratified by the exact feasible fraction {f_feasible:.3g} "
                         f"({w_uni:.1f}s + {w_fea:.1f}s); run_continuous on {n_traces} config-4 traces x {q_trace} "
                         f"requests ({w_rep:.1f}s)")}


def feasible_sampler(tables):
    """Random candidates of the feasible sub-product (original mixed-radix indices)."""
    from paper_2504_15303_b200 import _native as nat
    ok = [np.nonzero(tables.entries[i, : tables.n_degrees[i]]["status"] == nat.ENTRY_OK)[0]
          for i in range(len(tables.names))]
    nd = [int(x) for x in tables.n_degrees]

    def draw(rng, n):
        out = np.zeros(n, np.int64)
        for i, digs in enumerate(ok):
            out = out * nd[i] + rng.choice(digs, n)
        return out
    n_feas = 1
    for d in ok:
        n_feas *= len(d)
    return draw, n_feas


def port_baseline(target_s: float, P: int, R_total: int, q: int, rate: float):
    """The reference's algorithm, restated in C (oracle/, kind "port"), on the
    host cores: the literal per-candidate estimate_system_throughput on
    random candidates of config 3 and literal run_continuous on full-length
    config-4 traces; extrapolated to the full step workload."""
    from oracle import hs_oracle as orc
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances
    sys.path.insert(0, str(ROOT / "tests"))
    cores = len(os.sched_getaffinity(0))
    cluster, reqs, params, I, O = search_inputs(10_000)
    from helpers import search_structs
    model, engine, limits, machines, pr, present = search_structs(cluster, params)
    rng = np.random.default_rng(1)
    # calibrate the candidate sample to ~half of the budget
    n_c = cores * 64
    t0 = time.perf_counter()
    orc.candidates_literal(model, engine, limits, machines, pr, present, I, O, rng.integers(0, P, n_c), cores)
    dt = time.perf_counter() - t0
    n_c = max(cores, int(n_c * (0.45 * target_s) / max(dt, 1e-6)))
    idx = rng.integers(0, P, n_c)
    t0 = time.perf_counter()
    orc.candidates_literal(model, engine, limits, machines, pr, present, I, O, idx, cores)
    t_search = time.perf_counter() - t0
    cand_rate = n_c / t_search
    # replay sample: `cores` full-length traces in parallel
    rc, config, rparams = replay_deployment()
    handles = build_instances(rc, config, rparams)
    pol = hs.PolicyConfig()
    inst = engine_instances(handles, pol)
    ps = _policy_struct(pol, len(handles), hs.kv_bytes_per_token(rc.model))
    off, Ir, Or, Tr = replay_inputs(0, cores, q, rate)
    t0 = time.perf_counter()
    orc.replay(inst, ps, off, Ir, Or, Or, Tr, nthreads=cores, want_depart=False)
    t_rep = time.perf_counter() - t0
    req_rate = (cores * q) / t_rep
    value = (P + R_total) / (P / cand_rate + R_total / req_rate)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"oracle/hs_oracle.c on {cores} threads: literal estimate_system_throughput on {n_c} random "
                       f"config-3 candidates ({t_search:.1f}s, {cand_rate:.3g} cand/s) + literal run_continuous on "
                       f"{cores} config-4 traces x {q} requests ({t_rep:.1f}s, {req_rate:.3g} req/s); "
                       f"extrapolated to the step's {P:.3g} candidates + {R_total:.3g} requests"),
            "configs_per_s": cand_rate, "requests_per_s": req_rate}


def reference_baseline(pool: RefPool, P: int, R_total: int, tables, q_trace: int, n_traces: int, n_uniform: int,
                       n_feasible: int, seed: int = 1):
    draw, n_feas = feasible_sampler(tables)
    r = pool.sample(P, draw, n_feas / P, n_uniform, n_feasible, n_traces, q_trace, np.random.default_rng(seed))
    value = (P + R_total) / (P / r["configs_per_s"] + R_total / r["requests_per_s"])
    return {"value": value, "unit": UNIT, "cores": pool.cores, "kind": "reference",
            "sample": r["desc"] + f"; extrapolated to the step's {P:.3g} candidates + {R_total:.3g} requests",
            "configs_per_s": r["configs_per_s"], "requests_per_s": r["requests_per_s"]}


def reference_arm(args, rank, world):
    """bench.py --impl reference: the unmodified Python reference on the host
    cores, each step a bounded sample of the step workload (~5 s)."""
    if rank != 0:
        return
    import paper_2504_15303_b200  # noqa: F401 (workloads for the inputs; no engine call)
    P = 5**16
    R = args.traces * args.q
    if not (REF_DIR / "hetserve" / "__init__.py").exists():
        return port_reference_arm(args, P, R)  # the reference was not vendored: its C restatement
    tables = reference_tables(args.search_q)
    pool = RefPool(args.rate, args.search_q)
    cores = pool.cores
    vals = []
    try:
        for k in range(args.warmup + args.steps):
            v = reference_baseline(pool, P, R, tables, q_trace=4000, n_traces=cores, n_uniform=cores * 100,
                                   n_feasible=cores, seed=k)
            if k >= args.warmup:
                vals.append(v)
    finally:
        pool.close()
    v = statistics.median(x["value"] for x in vals)
    last = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": (P + R) / v * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64+int64", "data": "synthetic",
        "config": bench_config(args), "parallelism": f"{cores} host processes",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": last["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "breakdown": {"configs_per_s": statistics.median(x["configs_per_s"] for x in vals),
                      "requests_per_s": statistics.median(x["requests_per_s"] for x in vals)},
    }
    print(json.dumps(line), flush=True)


def port_reference_arm(args, P: int, R: int):
    """--impl reference without baseline/_ref: the C restatement (kind "port")."""
    vals = [port_baseline(args.cpu_seconds, P, R, args.q, args.rate) for _ in range(args.warmup + args.steps)]
    vals = vals[args.warmup:]
    v = statistics.median(x["value"] for x in vals)
    last = vals[-1]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": (P + R) / v * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64+int64", "data": "synthetic",
        "config": bench_config(args), "parallelism": "host threads",
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": last["cores"], "kind": "port", "sample": last["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "breakdown": {"configs_per_s": last["configs_per_s"], "requests_per_s": last["requests_per_s"]},
        "note": "baseline/_ref absent (python tools/vendor_reference.py): the reference's C restatement instead"}),
        flush=True)


def reference_tables(q_search: int):
    """The config-3 (machine, degree) feasibility table for the stratified
    sample, from the C oracle's table build (host only: no GPU on this arm)."""
    from oracle import hs_oracle as orc
    sys.path.insert(0, str(ROOT / "tests"))
    from helpers import search_structs
    from paper_2504_15303_b200 import _native as nat
    from paper_2504_15303_b200.planner import SearchTables
    cluster, reqs, params, I, O = search_inputs(q_search)
    model, engine, limits, machines, pr, present = search_structs(cluster, params)
    table, nd = orc.tables(model, engine, limits, machines, pr, present, I, O)
    names = [m.name for m in cluster.machines]
    from paper_2504_15303_b200.domain import enumerate_tp_degrees
    return SearchTables(cluster, reqs, names, [enumerate_tp_degrees(m) for m in cluster.machines],
                        np.asarray(table).reshape(len(names), nat.HS_MAX_DEGREES), np.asarray(nd, np.int32))


WORKLOAD = ("config3 search (5^16 candidates, 70B, 10k trace) + config4 replay ({traces} traces x {q} requests, "
            "32 instances, {rate} req/s, OS)")


def bench_config(args) -> dict:
    """The workload description both arms print (identical dicts)."""
    return {"workload": WORKLOAD.format(traces=args.traces, q=args.q, rate=args.rate), "candidates": 5**16,
            "requests": args.traces * args.q,
            "l2": "inputs larger than L2 (replay inputs %.1f GB)" % (args.traces * args.q * 4 * 5 / 1e9)}


# ------------------------------------------------------------------ engine
def engine_arm(args, rank, world, local_rank):
    import torch

    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import _native as nat
    from paper_2504_15303_b200 import planner
    from paper_2504_15303_b200.simulator import _policy_struct, build_instances, engine_instances

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    eng = nat.engine_for(local_rank)
    ext = torch.cuda.ExternalStream(eng.stream, device=dev)

    def barrier():
        if dist:
            tdist.barrier(device_ids=[local_rank])

    # ---- search inputs (every rank builds the same table; shards the index range)
    cluster, reqs, params, sI, sO = search_inputs(args.search_q)
    tables = planner.build_tables(cluster, reqs, params, engine=eng)
    P = tables.space_size
    from paper_2504_15303_b200.distributed import shard_range
    lo, hi = shard_range(P, rank, world)
    # ---- replay inputs (trace shard)
    T_lo, T_hi = shard_range(args.traces, rank, world)
    nT = T_hi - T_lo
    # inputs drawn on the device (rng.cu), bit-identical to the numpy streams
    # of gen-trace (lengths seeded by trace index) and generate_arrivals
    # (seed 42 + trace index); host copies for the e2e leg
    from paper_2504_15303_b200 import streams
    t0 = time.time()
    tseeds = list(range(T_lo, T_hi))
    lens = streams.gen_trace_lengths_device(tseeds, args.q, "lognormal:200:0.6", "lognormal:150:0.6", 4096, 4096,
                                            engine=eng)
    gen_lens_ms = eng.last_kernel_ms
    arrs = streams.arrival_times_device([42 + t for t in tseeds], [args.q] * nT, args.rate, engine=eng)
    gen_arr_ms = eng.last_kernel_ms if arrs is not None else 0.0
    gen_s = time.time() - t0
    off = lens.offsets
    I, O = lens.to_host()
    rc, config, rparams = replay_deployment()
    handles = build_instances(rc, config, rparams)
    N = len(handles)
    pol = hs.PolicyConfig()
    inst = engine_instances(handles, pol)
    ps = _policy_struct(pol, N, hs.kv_bytes_per_token(rc.model))
    nreq = int(off[-1])
    d = {"I": lens.ptrs[0], "O": lens.ptrs[1], "T": None if arrs is None else arrs.ptrs[0]}
    d["off"] = eng.device_alloc(off.nbytes)
    eng.h2d(d["off"], off)
    d["assign"] = eng.device_alloc(max(nreq, 1))
    d["metrics"] = eng.device_alloc(max(nT * N, 1) * nat.METRICS_DTYPE.itemsize)
    d["result"] = eng.device_alloc(max(nT, 1) * nat.RESULT_DTYPE.itemsize)

    from paper_2504_15303_b200 import distributed as hsd

    def combine(total, idx, nfeas):
        """One NCCL all-reduce of a per-rank slot buffer, then a local
        lexicographic reduce (max total, then lowest index)."""
        if not dist:
            return total, idx, nfeas
        return hsd.combine_best(total, idx, nfeas, device=dev, stream=ext)

    kms = {"k1": [], "k2": [], "k3": []}

    def step():
        t = planner.build_tables(cluster, reqs, params, engine=eng)
        kms["k1"].append(eng.last_kernel_ms)
        total, idx, nfeas, k2 = planner.search_best(t, lo, hi, engine=eng)
        kms["k2"].append(k2)
        eng.replay_device(inst, ps, nT, d["off"], d["I"], d["O"], d["O"], d["T"], d["assign"], d["metrics"],
                          d["result"])
        kms["k3"].append(eng.last_kernel_ms)
        return combine(total, idx, nfeas)

    def timed(fn, k):
        barrier()
        torch.cuda.synchronize(dev)
        eng.lib.hs_device_synchronize(eng.handle)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        out = None
        for _ in range(k):
            out = fn()
        e1.record(ext)
        e1.synchronize()
        eng.lib.hs_device_synchronize(eng.handle)
        torch.cuda.synchronize(dev)
        barrier()
        ms = e0.elapsed_time(e1) / k
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    for _ in range(args.warmup):
        best = step()
    for k in kms:
        kms[k].clear()
    launches0 = eng.launch_count
    with ClockSampler(local_rank) as clk:
        ms, best = timed(step, args.steps)
    launches = (eng.launch_count - launches0) // args.steps
    res = np.zeros(nT, nat.RESULT_DTYPE)
    eng.d2h(res, d["result"])
    assert (res["error"] == 0).all(), "replay reported an error"
    n_steps_ev = int(res["n_steps"].sum())
    R_total = args.traces * args.q
    units = P + R_total
    value = units / (ms / 1e3)

    # ---- e2e: the public API with host (pinned) buffers, copies inside
    e2e = None
    if not args.no_e2e:
        hI = eng.host_array(I.shape, np.int32); hI[:] = I
        hO = eng.host_array(O.shape, np.int32); hO[:] = O
        rc_, config_, rparams_ = rc, config, rparams
        aseeds = [42 + t for t in tseeds]
        hA = eng.host_array((max(nreq, 1),), np.uint8)  # page-locked result buffer, reused every step
        e2e_parts = {"search_call_ms": [], "replay_call_ms": [], "replay_pipeline_ms": []}

        def e2e_step():
            w0 = time.perf_counter()
            t = planner.build_tables(cluster, reqs, params, engine=eng)
            total, idx, nfeas, _ = planner.search_best(t, lo, hi, engine=eng)
            w1 = time.perf_counter()
            e2e_parts["search_call_ms"].append((w1 - w0) * 1e3)
            # arrivals drawn on the device from the seeds, inside the call, as
            # run_continuous draws them (simulator.py:112-124)
            r = hs.replay_traces(rc_, config_, rparams_, pol, off, hI, hO, hO, rate=args.rate,
                                 arrival_seeds=aseeds, want_assign=True, assign_out=hA,
                                 want_depart=False, engine=eng)
            e2e_parts["replay_call_ms"].append((time.perf_counter() - w1) * 1e3)
            e2e_parts["replay_pipeline_ms"].append(eng.last_kernel_ms)
            assert (r.result["error"] == 0).all()
            return combine(total, idx, nfeas)

        for _ in range(max(1, args.warmup - 1)):
            e2e_step()
        e2e_ms, _ = timed(e2e_step, args.steps)
        M = len(tables.names)
        # predictions are the outputs (oracle predictor): the library copies that buffer once
        h2d = sI.nbytes + sO.nbytes + off.nbytes + hI.nbytes + hO.nbytes + nT * nat.PCG64_DTYPE.itemsize
        d2h = nreq + nT * N * nat.METRICS_DTYPE.itemsize + nT * nat.RESULT_DTYPE.itemsize + \
            M * nat.HS_MAX_DEGREES * nat.ENTRY_DTYPE.itemsize + 16
        if dist:
            d2h += world * 24
        sc_ms = statistics.median(e2e_parts["search_call_ms"][-args.steps:])
        rc_ms = statistics.median(e2e_parts["replay_call_ms"][-args.steps:])
        e2e = {"value": units / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d * world),
               "d2h_bytes_per_step": int(d2h * world), "ms_per_step": e2e_ms,
               # the two halves of the metric, each through its own public call (rank 0's wall clock)
               "configs_per_s": P / (sc_ms / 1e3), "requests_per_s": R_total / (rc_ms / 1e3),
               "inputs": "host I/O lengths copied in; arrivals drawn on the device from per-trace seeds",
               "search_call_ms": sc_ms, "replay_call_ms": rc_ms,
               "replay_pipeline_ms": statistics.median(e2e_parts["replay_pipeline_ms"][-args.steps:])}

    # ---- roofline of the dominant kernel (K3 replay)
    peaks = {}
    pf = ROOT / "MEASURED_PEAKS.json"
    if pf.exists():
        peaks = json.loads(pf.read_text())
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    k3 = statistics.median(kms["k3"])
    k2 = statistics.median(kms["k2"])
    k1 = statistics.median(kms["k1"])
    achieved = BYTES_PER_DISPATCH * nreq / (k3 / 1e3) / 1e9
    traffic = None
    inst_per_dispatch = None
    prof = ROOT / "profiles" / "k3_replay_ncu.json"
    if prof.exists():
        pj = json.loads(prof.read_text())
        if pj.get("dram_bytes_per_dispatch"):
            traffic = pj["dram_bytes_per_dispatch"] * BYTES_PER_DISPATCH / BYTES_PER_DISPATCH * nreq
        inst_per_dispatch = pj.get("warp_inst_per_dispatch")
    fp64_peak = eng.probe_fp64()
    # K2 scores the feasible sub-product only (every infeasible candidate is
    # decided by its non-OK (machine, degree) entry): 1 DADD + 1 compare per
    # feasible candidate of this rank's range
    _t, _i, nfeas_local, _ms = planner.search_best(tables, lo, hi, engine=eng)
    if dist:  # the search half's time is its slowest shard's
        t2 = torch.tensor([k2], dtype=torch.float64, device=dev)
        tdist.all_reduce(t2, op=tdist.ReduceOp.MAX)
        k2 = float(t2.item())
    k2s = max(k2, 1e-6) / 1e3  # (a shard without feasible candidates launches nothing)
    k2_fp64 = 2.0 * best[2] / k2s
    # K3 against the FP64 pipe with the reference-literal op count of SURVEY
    # section 8(d): OS scoring ~67 FP64 ops per instance per dispatch
    # (divides, floordiv, prefill, decode, exp, min-max) + ~15 per step event
    steps_per_req = n_steps_ev / max(nreq, 1)
    k3_ops_per_dispatch = N * 67 + 15 * steps_per_req
    k3_fp64 = k3_ops_per_dispatch * nreq / (k3 / 1e3)
    clocks = clk.summary()
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    issue_peak = 4.0 * n_sm * (clocks.get("sm_mhz") or 1965.0) * 1e6
    roof_issue = None
    if inst_per_dispatch:
        ach = inst_per_dispatch * nreq / (k3 / 1e3)
        roof_issue = {"bound": "issue", "achieved": ach, "peak": issue_peak, "unit": "warp-instructions/s",
                      "frac": ach / issue_peak, "kernel": "k_replay", "inst_per_dispatch": inst_per_dispatch,
                      "note": "instructions per dispatch from ncu at this workload (profiles/k3_replay_ncu.json, "
                              "smsp__inst_executed.sum / dispatches); peak = 4 schedulers x SMs x SM clock"}

    c5 = None
    if not args.no_config5:
        c5 = config5_measure(args, rank, world, local_rank, eng, ext, cluster, reqs, params)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not (REF_DIR / "hetserve" / "__init__.py").exists():
        cpu = port_baseline(args.cpu_seconds, P, R_total, args.q, args.rate)  # reference not vendored
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        pool = RefPool(args.rate, args.search_q)
        try:
            cpu = reference_baseline(pool, P, R_total, tables, q_trace=args.q, n_traces=8,
                                     n_uniform=pool.cores * 200, n_feasible=pool.cores * 2)
            if c5 is not None:
                c5["cpu_baseline"] = config5_reference_baseline(pool, args, cpu["configs_per_s"], c5)
        finally:
            pool.close()
        cpu["port"] = port_baseline(args.cpu_seconds, P, R_total, args.q, args.rate)

    if c5 is not None:
        for key in ("_units", "_P", "_nreq", "top_indices"):
            c5.pop(key, None)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+int64", "data": "synthetic (gen-trace lognormal lengths + Poisson arrivals, numpy PCG64 streams drawn on the GPU)",
            "config": bench_config(args), "parallelism": f"shard{world}",
            "search": {"candidates_visited": P, "feasible_scored": best[2],
                       "note": "every candidate is decided; K2 sums and compares only the feasible sub-product "
                               "(an infeasible candidate holds a non-OK (machine, degree) entry and cannot win)"},
            "breakdown": {"k1_table_ms": k1, "k2_search_ms": k2, "k3_replay_ms": k3,
                          "configs_per_s": P / k2s,
                          "feasible_scored_per_s": best[2] / k2s,
                          "requests_per_s_kernel": nreq / (k3 / 1e3) * world,
                          "step_events_per_request": n_steps_ev / max(nreq, 1),
                          "best_total": best[0], "best_index": best[1], "n_feasible": best[2],
                          "trace_gen_s": gen_s, "gen_lengths_kernel_ms": gen_lens_ms,
                          "gen_arrivals_kernel_ms": gen_arr_ms},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "kernel": "k_replay",
                         "note": "replay is bound by dependent FP64 event chains, not bytes: see roofline_k3_fp64 "
                                 "and DESIGN.md"},
            "roofline_k2": {"bound": "fp64", "achieved": k2_fp64, "peak": fp64_peak * world, "unit": "FP64 op/s",
                            "frac": k2_fp64 / (fp64_peak * world), "kernel": "k_search_best",
                            "peak_source": "hs_probe_fp64 DADD throughput measured in this run",
                            "note": "2 FP64 ops (the left-to-right add and the compare, SURVEY.md 8d) per FEASIBLE "
                                    "candidate scored; a launch of a few microseconds is bound by launch latency"},
            "roofline_k3_fp64": {"bound": "fp64", "achieved": k3_fp64, "peak": fp64_peak, "unit": "FP64 op/s",
                                 "frac": k3_fp64 / fp64_peak, "kernel": "k_replay",
                                 "ops_per_dispatch": k3_ops_per_dispatch,
                                 "note": "reference-literal FP64 op count (SURVEY.md 8d: N*67 per dispatch + 15 per "
                                         "step event); the kernel executes fewer (per-class pricing, O(N) min-max)"},
            "gpu_launches": int(launches),
            "roofline_k3_issue": roof_issue,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "config5": c5,
        }
        print(json.dumps(line), flush=True)
    if dist:
        tdist.barrier(device_ids=[local_rank])


def config5_measure(args, rank, world, local_rank, eng, ext, cluster, reqs, params) -> dict | None:
    """BASELINE config 5: the top-k deployments of the config-3
    space (planner.py:227 order), each re-scored by a full continuous-batching
    simulation of one 1e5-request trace (rate = inf, OS; simulator.py:60-80 +
    run_continuous).  Units = feasible candidates ranked + requests replayed.
    value: device time of the top-k and replay kernels; e2e: the same step
    through the public calls with host buffers (search_topk, replay_candidates)."""
    import torch
    import paper_2504_15303_b200 as hs
    from paper_2504_15303_b200 import _native as nat
    from paper_2504_15303_b200 import planner
    from paper_2504_15303_b200.distributed import shard_range
    from paper_2504_15303_b200 import workloads as wl
    dist = world > 1
    if dist:
        import torch.distributed as tdist
    dev = torch.device("cuda", local_rank)
    I1, O1 = wl.trace_lengths(args.q, seed=0)
    tiles = {}
    kk = args.topk

    def tiled(n):
        # every deployment replays the same trace: tiled once into page-locked buffers
        if n not in tiles:
            ti = eng.host_array((max(n * args.q, 1),), np.int32)
            to = eng.host_array((max(n * args.q, 1),), np.int32)
            ta = eng.host_array((max(n * args.q, 1),), np.uint8)  # assignments, written in place by the kernel
            ti[: n * args.q] = np.tile(I1, n)
            to[: n * args.q] = np.tile(O1, n)
            tiles[n] = (ti[: n * args.q], to[: n * args.q], ta)
        return tiles[n]

    def step():
        t = planner.build_tables(cluster, reqs, params, engine=eng)
        k1 = eng.last_kernel_ms
        cands, nf, ms_topk = planner.search_topk(t, kk, rank, world, engine=eng)
        if dist:  # one all-gather of the per-rank top-k lists
            buf = torch.zeros(kk, 2, dtype=torch.int64, device=dev)
            loc = np.zeros((kk, 2), np.int64)
            loc[:, 1] = -1
            loc[:len(cands), 0] = cands["total"].view(np.int64)
            loc[:len(cands), 1] = cands["index"]
            buf.copy_(torch.from_numpy(loc))
            outs = [torch.zeros_like(buf) for _ in range(world)]
            tdist.all_gather(outs, buf)  # on the stream that wrote buf
            parts = []
            for o in outs:
                h = o.cpu().numpy()
                h = h[h[:, 1] >= 0]
                p = np.zeros(len(h), nat.CAND_DTYPE)
                p["total"] = h[:, 0].view(np.float64)
                p["index"] = h[:, 1]
                parts.append(p)
            top = planner.merge_topk(parts, kk)
            nf_all = torch.tensor([nf], dtype=torch.int64, device=dev)
            tdist.all_reduce(nf_all)
            nf = int(nf_all.item())
        else:
            top = cands
        lo, hi = shard_range(len(top), rank, world)
        n = hi - lo
        off = np.arange(n + 1, dtype=np.int64) * args.q
        I, O, A = tiled(n)
        res = hs.replay_candidates(t, params, top["index"][lo:hi], hs.PolicyConfig(), np.arange(n), off, I, O, O,
                                   engine=eng, want_assign=True, assign_out=A)
        assert (res.result["error"] == 0).all()
        return nf, k1, ms_topk, res.kernel_ms, n, top, res, t, lo, hi

    for _ in range(max(1, args.warmup - 1)):
        step()
    if dist:
        tdist.barrier(device_ids=[local_rank])
    torch.cuda.synchronize(dev)
    kern, walls = [], []
    for _ in range(args.steps):
        w0 = time.perf_counter()
        nf, k1, ms_topk, ms_rep, n, top, res, t, lo, hi = step()
        walls.append((time.perf_counter() - w0) * 1e3)
        kern.append(k1 + ms_topk + ms_rep)
    ms_k = statistics.median(kern)
    ms_w = statistics.median(walls)
    if dist:
        tt = torch.tensor([ms_k, ms_w], dtype=torch.float64, device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        ms_k, ms_w = (float(x) for x in tt.tolist())
    units = nf + kk * args.q
    nreq = n * args.q
    steps_per_req = float(res.result["n_steps"].sum()) / max(nreq, 1)
    # instances per replayed deployment (SURVEY.md 8d's reference-literal FP64 count: N * 67 per
    # dispatch + 15 per step event)
    ent = t.entries
    M = len(t.names)
    nd_ = np.asarray(t.n_degrees, np.int64)
    x = np.asarray(top["index"][lo:hi], np.int64).copy()
    n_inst = np.zeros(len(x), np.int64)
    for m in range(M - 1, -1, -1):
        n_inst += ent["instance_count"][m, x % nd_[m]]
        x //= nd_[m]
    ops = float(n_inst.mean()) * 67 + 15 * steps_per_req if len(n_inst) else 0.0
    fp64_peak = eng.probe_fp64()
    traffic = None
    pj = ROOT / "profiles" / "k3_config5_ncu.json"
    if pj.exists():
        traffic = json.loads(pj.read_text()).get("dram_bytes_per_request", 0.0) * nreq or None
    h2d = 2 * nreq * 4 + (n + 1) * 8
    d2h = nreq + n * res.metrics.shape[1] * nat.METRICS_DTYPE.itemsize + n * nat.RESULT_DTYPE.itemsize
    return {
        "metric": METRIC, "value": units / (ms_k / 1e3), "unit": UNIT, "ms_per_step": ms_k,
        "config": {"workload": f"config5: top-{kk} of the config-3 space (70B), each deployment replayed on "
                               f"{args.q} requests (rate=inf, OS)",
                   "feasible_candidates_ranked": nf, "requests": kk * args.q},
        "breakdown": {"k1_table_ms": k1, "topk_ms": ms_topk, "replay_ms": ms_rep, "deployments_rank0": n,
                      "step_events_per_request": steps_per_req, "requests_per_s_kernel": nreq / (ms_rep / 1e3)},
        "roofline": {"bound": "hbm", "achieved": BYTES_PER_DISPATCH * nreq / (ms_rep / 1e3) / 1e9,
                     "peak": json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0)
                     if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0,
                     "unit": "GB/s", "kernel": "k_replay (multi-deployment)", "traffic": traffic,
                     "traffic_source": "profiles/k3_config5_ncu.json (ncu --set full, DRAM bytes per request)"},
        "roofline_fp64": {"bound": "fp64", "achieved": ops * nreq / (ms_rep / 1e3), "peak": fp64_peak,
                          "unit": "FP64 op/s", "frac": ops * nreq / (ms_rep / 1e3) / fp64_peak,
                          "ops_per_dispatch": ops, "mean_instances": float(n_inst.mean()) if len(n_inst) else 0.0,
                          "kernel": "k_replay (multi-deployment)"},
        "e2e": {"value": units / (ms_w / 1e3), "unit": UNIT, "ms_per_step": ms_w, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": "search_topk + replay_candidates with page-locked host traces (copies inside the call) and a page-locked assignment buffer the kernel writes in place"},
        "top_indices": [int(x) for x in top["index"][:8]],
        "_units": units, "_P": 5**16, "_nreq": kk * args.q,
    }


def _ref_replay5(task) -> float:
    """The reference's run_continuous of config-3 candidate `index` at rate =
    inf (OS) on the first q requests of the config-5 trace (seed 0)."""
    index, q = task
    H, HS, wl, c3, degs = _REF["H"], _REF["HS"], _REF["wl"], _REF["c3"], _REF["degs3"]
    idx = int(index)
    dig = [0] * len(degs)
    for i in range(len(degs) - 1, -1, -1):
        idx, dig[i] = divmod(idx, len(degs[i]))
    config = H.deployment_for(c3.machines, {m.name: degs[i][d] for i, (m, d) in enumerate(zip(c3.machines, dig))})
    I, O = wl.trace_lengths(100_000, seed=0)
    trace = tuple(H.Request(f"r{k}", int(I[k]), int(O[k]), int(O[k])) for k in range(q))
    sc = HS.Scenario(cluster=c3, config=config, trace=trace, arrival_rate=float("inf"), policy=H.PolicyConfig(),
                     mode="continuous", seed=0, params=_REF["params3"])
    t0 = time.perf_counter()
    HS.run_continuous(sc)
    return time.perf_counter() - t0


def config5_reference_baseline(pool: RefPool, args, cand_per_s: float, c5: dict, q_s: int = 1500) -> dict:
    """The unmodified reference on config 5's work: its search visits all 5^16
    candidates (per-candidate cost from the main line's sample) before it can
    rank; each top-k deployment is then a run_continuous at rate = inf,
    sampled on the first q_s requests of the trace for `cores` of the top
    deployments and extrapolated per request."""
    idx = c5["top_indices"]
    tasks = [(idx[k % len(idx)], q_s) for k in range(pool.cores)]
    t0 = time.perf_counter()
    pool.pool.map(_ref_replay5, tasks, chunksize=1)
    w = time.perf_counter() - t0
    req_rate = len(tasks) * q_s / w
    P, nreq, units = c5["_P"], c5["_nreq"], c5["_units"]
    value = units / (P / cand_per_s + nreq / req_rate)
    return {"value": value, "unit": UNIT, "cores": pool.cores, "kind": "reference",
            "sample": (f"the unmodified reference (baseline/_ref) in a {pool.cores}-process pool: run_continuous "
                       f"(rate=inf, OS) of {len(tasks)} of the top deployments on the first {q_s} requests "
                       f"({w:.1f}s, {req_rate:.3g} req/s) + the search loop at the main line's "
                       f"{cand_per_s:.3g} candidates/s over all {P:.3g} candidates; extrapolated"),
            "configs_per_s": cand_per_s, "requests_per_s": req_rate}


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    engine_arm(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as tdist
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
