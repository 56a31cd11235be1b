"""ctypes binding of oracle/build/libhs_oracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module.  See hs_oracle.h.
"""

from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB = HERE / "build" / "libhs_oracle.so"


def build() -> pathlib.Path:
    gcc = "/usr/bin/gcc" if pathlib.Path("/usr/bin/gcc").exists() else "gcc"
    subprocess.run(["make", "-s", "-C", str(HERE), f"CC={gcc}"], check=True)
    return LIB


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    srcs = list(HERE.glob("*.c")) + list(HERE.glob("*.h")) + [HERE.parent / "include" / "hetserve_b200.h"]
    return any(f.exists() and f.stat().st_mtime > t for f in srcs)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if _stale():
            build()
        L = C.CDLL(str(LIB))
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.hs_oracle_exp.argtypes = [dbl, C.POINTER(C.c_int)]
        L.hs_oracle_exp.restype = dbl
        L.hs_oracle_floordiv.argtypes = [dbl, dbl]
        L.hs_oracle_floordiv.restype = dbl
        L.hs_oracle_pysum.argtypes = [vp, i64]
        L.hs_oracle_pysum.restype = dbl
        L.hs_oracle_tables.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, vp, vp]
        L.hs_oracle_tables.restype = C.c_int
        L.hs_oracle_candidate_literal.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, i64,
                                                  C.POINTER(i32), C.POINTER(i32)]
        L.hs_oracle_candidate_literal.restype = dbl
        L.hs_oracle_candidates_literal.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, vp, i64, C.c_int, vp, vp]
        L.hs_oracle_candidates_literal.restype = C.c_int
        L.hs_oracle_best.argtypes = [vp, vp, i32, i64, i64, C.c_int, vp, vp]
        L.hs_oracle_best.restype = C.c_int
        L.hs_oracle_topk.argtypes = [vp, vp, i32, i64, i32, i32, vp, vp, vp]
        L.hs_oracle_topk.restype = C.c_int
        L.hs_oracle_rank.argtypes = [vp, vp, i32, vp, vp, vp]
        L.hs_oracle_rank.restype = C.c_int
        L.hs_oracle_replay.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp, vp]
        L.hs_oracle_replay.restype = C.c_int
        L.hs_oracle_log1p.argtypes = [dbl]
        L.hs_oracle_log1p.restype = dbl
        L.hs_oracle_pcg64_next64.argtypes = [vp]
        L.hs_oracle_pcg64_next64.restype = C.c_uint64
        L.hs_oracle_std_normal.argtypes = [vp]
        L.hs_oracle_std_normal.restype = dbl
        L.hs_oracle_std_exp.argtypes = [vp]
        L.hs_oracle_std_exp.restype = dbl
        L.hs_oracle_rng_fill.argtypes = [vp, vp, i64, vp]
        L.hs_oracle_rng_fill.restype = i64
        L.hs_oracle_rng_generate.argtypes = [vp, i32, vp, vp, i32, vp, vp]
        L.hs_oracle_rng_generate.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def exp(x: float):
    of = C.c_int()
    y = lib().hs_oracle_exp(float(x), C.byref(of))
    return y, bool(of.value)


def exp_batch(x):
    """The C port over an array: (values, overflow flags)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    of = np.empty(len(x), np.uint8)
    lib().hs_oracle_exp_batch(_p(x), C.c_int64(len(x)), _p(y), _p(of))
    return y, of.astype(bool)


def libm_exp_batch(x):
    """glibc's exp itself (what CPython's math.exp calls) over an array."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().hs_libm_exp_batch(_p(x), C.c_int64(len(x)), _p(y))
    return y


def floordiv(a: float, b: float) -> float:
    return lib().hs_oracle_floordiv(float(a), float(b))


def pysum(xs) -> float:
    a = np.ascontiguousarray(xs, np.float64)
    return lib().hs_oracle_pysum(_p(a), len(a))


def tables(model, engine, limits, machines, params, present, I, O):
    """Same layout as hs_search_tables; structs from paper_2504_15303_b200._native."""
    from paper_2504_15303_b200 import _native as nat
    M = len(machines)
    table = np.zeros(M * nat.HS_MAX_DEGREES, nat.ENTRY_DTYPE)
    nd = np.zeros(M, np.int32)
    I = np.ascontiguousarray(I, np.int32)
    O = np.ascontiguousarray(O, np.int32)
    rc = lib().hs_oracle_tables(C.byref(model), C.byref(engine), C.byref(limits), C.cast(machines, C.c_void_p), M,
                                _p(params), _p(present), _p(I), _p(O), len(I), _p(table), _p(nd))
    assert rc == 0
    return table.reshape(M, nat.HS_MAX_DEGREES), nd


def candidate_literal(model, engine, limits, machines, params, present, I, O, index: int):
    fb, st = C.c_int32(), C.c_int32()
    I = np.ascontiguousarray(I, np.int32)
    O = np.ascontiguousarray(O, np.int32)
    t = lib().hs_oracle_candidate_literal(C.byref(model), C.byref(engine), C.byref(limits),
                                          C.cast(machines, C.c_void_p), len(machines), _p(params), _p(present),
                                          _p(I), _p(O), len(I), int(index), C.byref(fb), C.byref(st))
    return t, fb.value, st.value


def candidates_literal(model, engine, limits, machines, params, present, I, O, indices, nthreads=1):
    idx = np.ascontiguousarray(indices, np.int64)
    totals = np.zeros(max(len(idx), 1), np.float64)
    fb = np.zeros(max(len(idx), 1), np.int32)
    I = np.ascontiguousarray(I, np.int32)
    O = np.ascontiguousarray(O, np.int32)
    rc = lib().hs_oracle_candidates_literal(C.byref(model), C.byref(engine), C.byref(limits),
                                            C.cast(machines, C.c_void_p), len(machines), _p(params), _p(present),
                                            _p(I), _p(O), len(I), _p(idx), len(idx), int(nthreads), _p(totals),
                                            _p(fb))
    assert rc == 0
    return totals[: len(idx)], fb[: len(idx)]


def best(table, nd, begin, end, nthreads=1):
    from paper_2504_15303_b200 import _native as nat
    out = np.zeros(1, nat.CAND_DTYPE)
    nf = np.zeros(1, np.int64)
    t = np.ascontiguousarray(table.reshape(-1))
    rc = lib().hs_oracle_best(_p(t), _p(np.ascontiguousarray(nd, np.int32)), len(nd), int(begin), int(end),
                              int(nthreads), _p(out), _p(nf))
    assert rc == 0
    return float(out["total"][0]), int(out["index"][0]), int(nf[0])


def topk(table, nd, k, shard=0, n_shards=1):
    from paper_2504_15303_b200 import _native as nat
    out = np.zeros(max(k, 1), nat.CAND_DTYPE)
    n = np.zeros(1, np.int64)
    nf = np.zeros(1, np.int64)
    t = np.ascontiguousarray(table.reshape(-1))
    rc = lib().hs_oracle_topk(_p(t), _p(np.ascontiguousarray(nd, np.int32)), len(nd), int(k), int(shard),
                              int(n_shards), _p(out), _p(n), _p(nf))
    assert rc == 0
    return out[: n[0]], int(nf[0])


def rank(table, nd):
    from paper_2504_15303_b200 import _native as nat
    P = int(np.prod(np.asarray(nd, np.int64)))
    ranked = np.zeros(max(P, 1), nat.CAND_DTYPE)
    fb = np.zeros(max(P, 1), np.int8)
    n = np.zeros(1, np.int64)
    t = np.ascontiguousarray(table.reshape(-1))
    rc = lib().hs_oracle_rank(_p(t), _p(np.ascontiguousarray(nd, np.int32)), len(nd), _p(ranked), _p(n), _p(fb))
    assert rc == 0
    return ranked[: n[0]], fb[:P]


def replay(instances, policy, offsets, I, O, P, arrival=None, nthreads=1, want_depart=True):
    from paper_2504_15303_b200 import _native as nat
    T = len(offsets) - 1
    N = policy.n_instances
    total = int(offsets[-1])
    offsets = np.ascontiguousarray(offsets, np.int64)
    I = np.ascontiguousarray(I, np.int32)
    O = np.ascontiguousarray(O, np.int32)
    P = np.ascontiguousarray(P, np.int32)
    arrival = None if arrival is None else np.ascontiguousarray(arrival, np.float64)
    batch = nat.hs_trace_batch(T, offsets.ctypes.data, I.ctypes.data, O.ctypes.data, P.ctypes.data,
                               None if arrival is None else arrival.ctypes.data)
    assign = np.zeros(max(total, 1), np.uint8)
    depart = np.zeros(max(total, 1), np.float64) if want_depart else None
    metrics = np.zeros(max(T * N, 1), nat.METRICS_DTYPE)
    result = np.zeros(max(T, 1), nat.RESULT_DTYPE)
    rc = lib().hs_oracle_replay(C.cast(instances, C.c_void_p), C.byref(policy), C.byref(batch), int(nthreads),
                                _p(assign), _p(depart), _p(metrics), _p(result))
    assert rc == 0
    return assign[:total], (None if depart is None else depart[:total]), metrics[: T * N].reshape(T, N), result[:T]


def best_monotone(table, nd):
    """Exact argmax of the left-to-right fp64 sum over the full product space
    in O(M^2 * D), for tables whose OK contributions are all finite.

    Rounded addition is monotone in each argument, so from a prefix sum s the
    largest reachable total is the greedy completion g(s) = (((s + m_k) +
    m_{k+1}) ...) with m_j the largest OK contribution of machine j.  The
    global maximum V is g from the empty prefix; the lowest index reaching V
    is found digit by digit: at each machine take the smallest OK digit whose
    greedy completion still equals V (planner.py:227's tie rule).  Returns
    (V, index, n_feasible) with n_feasible = prod(#OK degrees)."""
    from paper_2504_15303_b200 import _native as nat
    M = len(nd)
    C = [[float(table[i, d]["contribution"]) if int(table[i, d]["status"]) == nat.ENTRY_OK else None
          for d in range(int(nd[i]))] for i in range(M)]
    mx = []
    nfeas = 1
    for row in C:
        ok = [v for v in row if v is not None]
        nfeas *= len(ok)
        mx.append(max(ok) if ok else None)
    if nfeas == 0:
        return 0.0, -1, 0

    def greedy(s, k):
        for j in range(k, M):
            s = s + mx[j]
        return s

    V = greedy(0.0, 0)
    s, index = 0.0, 0
    for i in range(M):
        for d, v in enumerate(C[i]):
            if v is not None and greedy(s + v, i + 1) == V:
                s = s + v
                index = index * int(nd[i]) + d
                break
        else:
            raise AssertionError("monotone search lost the maximum")
    return V, index, nfeas


# ------------------------------------------------------- numpy PCG64 streams
def log1p(x: float) -> float:
    return lib().hs_oracle_log1p(float(x))


def numpy_state(seed: int) -> np.ndarray:
    """The initial state numpy itself computes for default_rng(seed)."""
    from paper_2504_15303_b200._native import PCG64_DTYPE
    st = np.random.PCG64(seed).state
    out = np.zeros(1, PCG64_DTYPE)
    s, inc = st["state"]["state"], st["state"]["inc"]
    out["state_hi"], out["state_lo"] = s >> 64, s & (2**64 - 1)
    out["inc_hi"], out["inc_lo"] = inc >> 64, inc & (2**64 - 1)
    out["has_uint32"], out["uinteger"] = st["has_uint32"], st["uinteger"]
    return out


def rng_generate(states: np.ndarray, offsets: np.ndarray, dists):
    """hs_oracle_rng_generate with host outputs; returns (outs, bad)."""
    from paper_2504_15303_b200._native import DIST_EXP_CUMSUM, hs_dist
    n = len(offsets) - 1
    total = int(offsets[-1])
    outs = [np.zeros(max(total, 1), np.float64 if d.kind == DIST_EXP_CUMSUM else np.int32) for d in dists]
    darr = (hs_dist * len(dists))(*dists)
    oarr = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    bad = np.full(max(n, 1), -1, np.int64)
    off = np.ascontiguousarray(offsets, np.int64)
    rc = lib().hs_oracle_rng_generate(_p(states), n, _p(off), C.cast(darr, C.c_void_p), len(dists),
                                      C.cast(oarr, C.c_void_p), _p(bad))
    assert rc == 0, rc
    return [o[:total] for o in outs], bad[:n]
