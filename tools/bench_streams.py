"""Time the device stream generator (rng.cu) on the config-4 workload:
4096 traces x 1e5 requests -- gen-trace lengths (two lognormal streams per
trace) and arrivals (exponential running sum), vs numpy on the host.

    python tools/bench_streams.py [--traces 4096] [--q 100000] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2504_15303_b200 import _native as nat  # noqa: E402
from paper_2504_15303_b200 import streams  # noqa: E402
from paper_2504_15303_b200 import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=4096)
    ap.add_argument("--q", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    eng = nat.engine_for(0)
    T, q = a.traces, a.q
    seeds = list(range(T))
    counts = [q] * T
    mu_i = np.log(200.0) - 0.18
    mu_o = np.log(150.0) - 0.18
    d_len = [nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 4096, 0, 0, mu_i, 0.6),
             nat.hs_dist(nat.DIST_LOGNORMAL_LEN, 4096, 0, 0, mu_o, 0.6)]
    d_arr = [nat.hs_dist(nat.DIST_EXP_CUMSUM, 0, 0, 0, 1.0 / wl.CONFIG4_RATE, 0)]
    res = {}
    for name, dists, sd in (("lengths", d_len, seeds), ("arrivals", d_arr, [42 + s for s in seeds])):
        ms = []
        for _ in range(a.reps):
            out = streams._generate(sd, counts, dists, engine=eng)
            ms.append(eng.last_kernel_ms)
            out.close()
        bytes_out = T * q * (8 if name == "lengths" else 8)
        best = min(ms)
        res[name] = {"kernel_ms": best, "values_per_s": T * q * len(dists) / (best / 1e3),
                     "write_GBps": bytes_out / (best / 1e3) / 1e9, "all_ms": ms}
    # numpy on the host: a sample of traces on all cores
    cores = len(os.sched_getaffinity(0))
    n_s = min(T, cores * 2)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        list(ex.map(lambda t: (wl.trace_lengths(q, seed=t), wl.arrivals(q, wl.CONFIG4_RATE, seed=42 + t)),
                    range(n_s)))
    dt = time.perf_counter() - t0
    res["numpy_host"] = {"cores": cores, "sample_traces": n_s, "s": dt,
                         "extrapolated_full_s": dt * T / n_s}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
