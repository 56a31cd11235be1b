"""ctypes binding of libhetserve_b200.so (include/hetserve_b200.h).

The engine has no CPU fallback: if the library cannot be loaded, or no CUDA
device is present, every call raises EngineUnavailable.
"""

from __future__ import annotations

import ctypes as C
import os
import pathlib
import threading

import numpy as np

HS_MAX_DEGREES = 32
HS_MAX_MACHINES = 64
HS_MAX_INSTANCES = 255
HS_MAX_CLASSES = 32

# enums (hetserve_b200.h)
HS_OK, HS_ERR_ARG, HS_ERR_CUDA, HS_ERR_UNSUPPORTED, HS_ERR_NOMEM = 0, 1, 2, 3, 4
ENTRY_OK, ENTRY_INFEASIBLE_CONFIG, ENTRY_MISSING_PARAMS, ENTRY_INFEASIBLE_REQUEST, ENTRY_ZERO_DIVISION, \
    ENTRY_BAD_DEGREE = range(6)
POLICY_CODE = {"OS": 0, "RR": 1, "WRR": 2, "SI": 3, "MB": 4}
TRACE_OK, TRACE_INFEASIBLE_REQUEST, TRACE_NONPOSITIVE_COST, TRACE_EXP_OVERFLOW, TRACE_NO_INSTANCE, \
    TRACE_NEGATIVE_RUNNING, TRACE_CAPACITY, TRACE_STALLED = range(8)

LIB_PATH = pathlib.Path(os.environ.get("HS_LIB", pathlib.Path(__file__).resolve().parent / "libhetserve_b200.so"))


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library missing or no GPU)."""


class EngineError(RuntimeError):
    """A call into the engine failed (CUDA error, unsupported input, ...)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[hs status {code}] {message}")
        self.code = code


class hs_model(C.Structure):
    _fields_ = [("layers", C.c_int64), ("hidden_dim", C.c_int64), ("param_count", C.c_int64),
                ("bytes_per_param", C.c_int64)]


class hs_engine(C.Structure):
    _fields_ = [("mem_utilization_fraction", C.c_double), ("static_overhead_bytes", C.c_int64)]


class hs_limits(C.Structure):
    _fields_ = [("max_input_len", C.c_int64), ("max_output_len", C.c_int64)]


class hs_machine(C.Structure):
    _fields_ = [("accelerator_count", C.c_int64), ("accelerator_mem_bytes", C.c_int64), ("spec_index", C.c_int32),
                ("fixed_degree", C.c_int32)]


class hs_entry(C.Structure):
    _fields_ = [("contribution", C.c_double), ("rate", C.c_double), ("budget", C.c_double), ("slack", C.c_double),
                ("instance_count", C.c_int64), ("bad_request", C.c_int64), ("token_count", C.c_int64),
                ("tp_degree", C.c_int32), ("status", C.c_int32), ("zero_div_int", C.c_int32), ("_pad", C.c_int32)]


class hs_cand(C.Structure):
    _fields_ = [("total", C.c_double), ("index", C.c_int64)]


class hs_instance(C.Structure):
    _fields_ = [("p", C.c_double * 8), ("budget", C.c_double), ("wrr_weight", C.c_double), ("type", C.c_int32),
                ("_pad", C.c_int32)]


class hs_policy(C.Structure):
    _fields_ = [("policy", C.c_int32), ("n_instances", C.c_int32), ("theta", C.c_double), ("per_token", C.c_int64),
                ("mode", C.c_int32), ("flags", C.c_int32)]


REPLAY_ORDER_KEYS = 1  # hs_policy.flags: depart = (time, heap key, per-instance sequence) per request


class hs_inst_metrics(C.Structure):
    _fields_ = [("completion_time", C.c_double), ("peak_kv_usage", C.c_double), ("residual_load", C.c_double),
                ("request_count", C.c_int64), ("token_count", C.c_int64)]


class hs_trace_result(C.Structure):
    _fields_ = [("error", C.c_int32), ("err_instance", C.c_int32), ("err_request", C.c_int64),
                ("err_value", C.c_double), ("n_steps", C.c_int64)]


class hs_trace_batch(C.Structure):
    _fields_ = [("n_traces", C.c_int64), ("offsets", C.c_void_p), ("input_len", C.c_void_p),
                ("output_len", C.c_void_p), ("pred_output_len", C.c_void_p), ("arrival", C.c_void_p)]


class hs_pcg64_state(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64),
                ("has_uint32", C.c_uint32), ("uinteger", C.c_uint32)]


class hs_dist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("cap", C.c_int32), ("lo", C.c_int64), ("hi", C.c_int64), ("p0", C.c_double),
                ("p1", C.c_double)]


class hs_replay_seeds(C.Structure):
    _fields_ = [("arrival_state", C.c_void_p), ("arrival_scale", C.c_double), ("predictor_state", C.c_void_p),
                ("pred_mean", C.c_double), ("pred_stddev", C.c_double), ("pred_cap", C.c_int32), ("_pad", C.c_int32)]


DIST_LOGNORMAL_LEN, DIST_UNIFORM_LEN, DIST_EXP_CUMSUM, DIST_NORMAL_LEN = 0, 1, 2, 3


class hs_sched_status(C.Structure):
    _fields_ = [("error", C.c_int32), ("instance", C.c_int32), ("value", C.c_double)]


(SCHED_OK, SCHED_NO_INSTANCE, SCHED_ALREADY_IN_FLIGHT, SCHED_NOT_IN_FLIGHT, SCHED_NONPOSITIVE_COST,
 SCHED_EXP_OVERFLOW, SCHED_NEGATIVE_RUNNING, SCHED_ZERO_DIVISION) = range(8)

# numpy views of the structs (same layout) for bulk results
ENTRY_DTYPE = np.dtype([("contribution", "<f8"), ("rate", "<f8"), ("budget", "<f8"), ("slack", "<f8"),
                        ("instance_count", "<i8"), ("bad_request", "<i8"), ("token_count", "<i8"),
                        ("tp_degree", "<i4"), ("status", "<i4"), ("zero_div_int", "<i4"), ("_pad", "<i4")])
CAND_DTYPE = np.dtype([("total", "<f8"), ("index", "<i8")])
METRICS_DTYPE = np.dtype([("completion_time", "<f8"), ("peak_kv_usage", "<f8"), ("residual_load", "<f8"),
                          ("request_count", "<i8"), ("token_count", "<i8")])
INSTANCE_DTYPE = np.dtype([("p", "<f8", (8,)), ("budget", "<f8"), ("wrr_weight", "<f8"), ("type", "<i4"),
                           ("_pad", "<i4")])
PCG64_DTYPE = np.dtype([("state_hi", "<u8"), ("state_lo", "<u8"), ("inc_hi", "<u8"), ("inc_lo", "<u8"),
                        ("has_uint32", "<u4"), ("uinteger", "<u4")])
RESULT_DTYPE = np.dtype([("error", "<i4"), ("err_instance", "<i4"), ("err_request", "<i8"), ("err_value", "<f8"),
                         ("n_steps", "<i8")])

# every symbol include/hetserve_b200.h declares
EXPORTS = (
    "hs_abi_version", "hs_ctx_create", "hs_ctx_destroy", "hs_last_error", "hs_ctx_launch_count",
    "hs_ctx_last_kernel_ms", "hs_search_tables", "hs_search_best", "hs_search_rank", "hs_search_topk", "hs_replay",
    "hs_replay_deployments",
    "hs_replay_device", "hs_device_alloc", "hs_device_free", "hs_memcpy_h2d", "hs_memcpy_d2h",
    "hs_device_synchronize", "hs_host_alloc", "hs_host_free", "hs_ctx_stream", "hs_probe_fp64",
    "hs_replay_seeded", "hs_pcg64_seed", "hs_pcg64_seed_u64", "hs_rng_generate",
    "hs_sched_create", "hs_sched_destroy", "hs_sched_evaluate", "hs_sched_choose", "hs_sched_complete",
    "hs_sched_snapshot", "hs_plan_instance", "hs_sched_get_state", "hs_sched_set_state", "hs_sched_set_instance", "hs_exp_batch", "hs_floordiv_batch", "hs_div_batch", "hs_search_topk_after",
)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load the engine library (no GPU needed to load it)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path else LIB_PATH
        if not p.exists():
            raise EngineUnavailable(f"{p} is missing: run `python -m paper_2504_15303_b200.build`")
        lib = C.CDLL(str(p))
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        sig = {
            "hs_abi_version": ([], C.c_int),
            "hs_ctx_create": ([C.c_int, C.POINTER(vp)], C.c_int),
            "hs_ctx_destroy": ([vp], C.c_int),
            "hs_last_error": ([], C.c_char_p),
            "hs_ctx_launch_count": ([vp], i64),
            "hs_ctx_last_kernel_ms": ([vp], dbl),
            "hs_search_tables": ([vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, i64, vp, vp], C.c_int),
            "hs_search_best": ([vp, vp, vp, i32, i64, i64, vp, vp], C.c_int),
            "hs_search_rank": ([vp, vp, vp, i32, vp, vp, vp], C.c_int),
            "hs_search_topk": ([vp, vp, vp, i32, i64, i32, i32, vp, vp, vp], C.c_int),
            "hs_replay": ([vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
            "hs_replay_device": ([vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
            "hs_replay_deployments": ([vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp], C.c_int),
            "hs_device_alloc": ([vp, i64, C.POINTER(vp)], C.c_int),
            "hs_device_free": ([vp, vp], C.c_int),
            "hs_memcpy_h2d": ([vp, vp, vp, i64], C.c_int),
            "hs_memcpy_d2h": ([vp, vp, vp, i64], C.c_int),
            "hs_device_synchronize": ([vp], C.c_int),
            "hs_host_alloc": ([vp, i64, C.POINTER(vp)], C.c_int),
            "hs_host_free": ([vp, vp], C.c_int),
            "hs_ctx_stream": ([vp], vp),
            "hs_probe_fp64": ([vp, C.POINTER(dbl)], C.c_int),
            "hs_replay_seeded": ([vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
            "hs_pcg64_seed": ([vp, i32, vp], C.c_int),
            "hs_pcg64_seed_u64": ([vp, i64, vp], C.c_int),
            "hs_sched_create": ([vp, i32, vp, vp], C.c_int),
            "hs_sched_destroy": ([vp], C.c_int),
            "hs_sched_evaluate": ([vp, i64, i64, vp, vp, vp], C.c_int),
            "hs_sched_choose": ([vp, C.c_char_p, i32, i64, i64, vp, vp, vp], C.c_int),
            "hs_sched_complete": ([vp, C.c_char_p, i32, vp], C.c_int),
            "hs_sched_snapshot": ([vp, vp, vp, vp, vp, vp], C.c_int),
            "hs_sched_get_state": ([vp, i32, vp, vp, vp, vp], C.c_int),
            "hs_sched_set_state": ([vp, i32, dbl, i64, i64, i64], C.c_int),
            "hs_sched_set_instance": ([vp, i32, vp], C.c_int),
            "hs_exp_batch": ([vp, vp, i64, vp, vp], C.c_int),
            "hs_floordiv_batch": ([vp, vp, vp, i64, vp], C.c_int),
            "hs_div_batch": ([vp, vp, vp, i64, vp], C.c_int),
            "hs_search_topk_after": ([vp, vp, vp, i32, i64, dbl, i64, vp, vp, vp], C.c_int),
            "hs_plan_instance": ([vp, dbl, i64, vp, vp, vp, i64, vp, vp, vp, vp], C.c_int),
            "hs_rng_generate": ([vp, vp, i32, vp, vp, i32, vp, vp], C.c_int),
        }
        for name, (args, res) in sig.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:  # an older diagnostic build (HS_LIB); the tests check the real one
                continue
            fn.argtypes = args
            fn.restype = res
        if path is None:
            _lib = lib
        return lib


def _out_buf(out: np.ndarray | None, n: int, dtype) -> np.ndarray:
    if out is None:
        return np.zeros(max(n, 1), dtype)
    if out.dtype != np.dtype(dtype) or not out.flags.c_contiguous or len(out) < n or not out.flags.writeable:
        raise ValueError(f"output buffer must be a writable contiguous {np.dtype(dtype)} array of >= {n} elements")
    return out


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Engine:
    """One engine context (device, stream, device buffers).  Not thread-safe:
    use one Engine per thread (engine_for() keeps one per (thread, device))."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.hs_ctx_create(int(device), C.byref(h))
        if rc != HS_OK:
            raise EngineUnavailable(f"hs_ctx_create(device={device}) failed: {self._err()}")
        self.handle = h
        self.device = device

    def _err(self) -> str:
        msg = self.lib.hs_last_error()
        return msg.decode() if msg else ""

    def check(self, rc: int, what: str) -> None:
        if rc != HS_OK:
            raise EngineError(rc, f"{what}: {self._err()}")

    def close(self) -> None:
        for p in getattr(self, "_pinned", []):
            self.lib.hs_host_free(self.handle, C.c_void_p(p))
        self._pinned = []
        if getattr(self, "handle", None):
            self.lib.hs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(self.lib.hs_ctx_launch_count(self.handle))

    @property
    def last_kernel_ms(self) -> float:
        return float(self.lib.hs_ctx_last_kernel_ms(self.handle))

    @property
    def stream(self) -> int:
        """cudaStream_t of this context (for torch.cuda.ExternalStream)."""
        return int(self.lib.hs_ctx_stream(self.handle) or 0)

    def probe_fp64(self) -> float:
        v = C.c_double()
        self.check(self.lib.hs_probe_fp64(self.handle, C.byref(v)), "hs_probe_fp64")
        return float(v.value)

    # ------------------------------------------------------- raw buffers
    def device_alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        self.check(self.lib.hs_device_alloc(self.handle, int(nbytes), C.byref(p)), "hs_device_alloc")
        return int(p.value)

    def device_free(self, ptr: int) -> None:
        self.check(self.lib.hs_device_free(self.handle, C.c_void_p(ptr)), "hs_device_free")

    def h2d(self, dst: int, src: np.ndarray) -> None:
        self.check(self.lib.hs_memcpy_h2d(self.handle, C.c_void_p(dst), _ptr(src), src.nbytes), "hs_memcpy_h2d")

    def d2h(self, dst: np.ndarray, src: int) -> None:
        self.check(self.lib.hs_memcpy_d2h(self.handle, _ptr(dst), C.c_void_p(src), dst.nbytes), "hs_memcpy_d2h")

    def host_array(self, shape, dtype) -> np.ndarray:
        """A numpy array over page-locked host memory (freed with the engine)."""
        dt = np.dtype(dtype)
        n = int(np.prod(shape)) * dt.itemsize
        p = C.c_void_p()
        self.check(self.lib.hs_host_alloc(self.handle, n, C.byref(p)), "hs_host_alloc")
        buf = (C.c_byte * max(n, 1)).from_address(p.value)
        self._pinned = getattr(self, "_pinned", [])
        self._pinned.append(p.value)
        return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)

    def replay_deployments(self, instances, inst_offsets: np.ndarray, policy: hs_policy, trace_dep: np.ndarray,
                           offsets: np.ndarray, I: np.ndarray, O: np.ndarray, P: np.ndarray,
                           arrival: np.ndarray | None, want_assign: bool = True, want_depart: bool = False,
                           assign_out: np.ndarray | None = None, depart_out: np.ndarray | None = None):
        """assign_out / depart_out: caller buffers (a page-locked assign_out,
        e.g. host_array, is written by the kernel in place)."""
        T = len(offsets) - 1
        nd = len(inst_offsets) - 1
        n_max = int(np.max(np.diff(inst_offsets))) if nd else 0
        total = int(offsets[-1])
        batch = hs_trace_batch(T, offsets.ctypes.data, I.ctypes.data, O.ctypes.data, P.ctypes.data,
                               None if arrival is None else arrival.ctypes.data)
        assign = _out_buf(assign_out, total, np.uint8) if want_assign else None
        depart = _out_buf(depart_out, total, np.float64) if want_depart else None
        metrics = np.zeros(max(T * n_max, 1), METRICS_DTYPE)
        result = np.zeros(max(T, 1), RESULT_DTYPE)
        io = np.ascontiguousarray(inst_offsets, np.int32)
        td = np.ascontiguousarray(trace_dep, np.int32)
        rc = self.lib.hs_replay_deployments(self.handle, C.cast(instances, C.c_void_p), _ptr(io), nd, C.byref(policy),
                                            _ptr(td), C.byref(batch), _ptr(assign), _ptr(depart), _ptr(metrics),
                                            _ptr(result))
        self.check(rc, "hs_replay_deployments")
        return (None if assign is None else assign[:total], None if depart is None else depart[:total],
                metrics[: T * n_max].reshape(T, n_max), result[:T])

    def replay_device(self, instances, policy, n_traces: int, d_off: int, d_I: int, d_O: int, d_P: int,
                      d_T: int | None, d_assign: int | None, d_metrics: int, d_result: int) -> None:
        batch = hs_trace_batch(n_traces, d_off, d_I, d_O, d_P, d_T)
        rc = self.lib.hs_replay_device(self.handle, C.cast(instances, C.c_void_p), C.byref(policy), C.byref(batch),
                                       None if d_assign is None else C.c_void_p(d_assign), None,
                                       C.c_void_p(d_metrics), C.c_void_p(d_result))
        self.check(rc, "hs_replay_device")

    def exp_batch(self, x: np.ndarray):
        """hs_exp_batch: (math.exp(x) as the replay kernels compute it, overflow flags)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        of = np.empty(len(x), np.uint8)
        self.check(self.lib.hs_exp_batch(self.handle, _ptr(x), len(x), _ptr(y), _ptr(of)), "hs_exp_batch")
        return y, of.astype(bool)

    def floordiv_batch(self, x: np.ndarray, w: np.ndarray):
        """hs_floordiv_batch: CPython x // w as the replay kernels compute it."""
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        y = np.empty_like(x)
        self.check(self.lib.hs_floordiv_batch(self.handle, _ptr(x), _ptr(w), len(x), _ptr(y)), "hs_floordiv_batch")
        return y

    def div_batch(self, x: np.ndarray, b: np.ndarray):
        """hs_div_batch: the IEEE quotient x / b as the replay kernels compute kv_usage."""
        x = np.ascontiguousarray(x, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        y = np.empty_like(x)
        self.check(self.lib.hs_div_batch(self.handle, _ptr(x), _ptr(b), len(x), _ptr(y)), "hs_div_batch")
        return y

    # --------------------------------------------------------------- streams
    def rng_generate(self, states: np.ndarray, offsets: np.ndarray, dists, outs) -> np.ndarray:
        """hs_rng_generate: states (PCG64_DTYPE, advanced in place), device
        output pointers one per hs_dist; returns the per-stream bad index."""
        n = len(offsets) - 1
        assert states.dtype == PCG64_DTYPE and states.flags.c_contiguous and len(states) >= n
        off = np.ascontiguousarray(offsets, np.int64)
        darr = (hs_dist * len(dists))(*dists)
        oarr = (C.c_void_p * len(outs))(*[C.c_void_p(int(o)) if o else None for o in outs])
        bad = np.full(max(n, 1), -1, np.int64)
        rc = self.lib.hs_rng_generate(self.handle, _ptr(states), n, _ptr(off), C.cast(darr, C.c_void_p), len(dists),
                                      C.cast(oarr, C.c_void_p), _ptr(bad))
        self.check(rc, "hs_rng_generate")
        return bad[:n]

    def plan_instance(self, budget: float, per_token: int, params8, I: np.ndarray, O: np.ndarray):
        """hs_plan_instance: (stops int64[nb], times float64[nb] or None, entry)."""
        I = np.ascontiguousarray(I, np.int32)
        O = np.ascontiguousarray(O, np.int32)
        q = len(I)
        stops = np.zeros(max(q, 1), np.int64)
        times = np.zeros(max(q, 1), np.float64) if params8 is not None else None
        pr = None if params8 is None else np.ascontiguousarray(params8, np.float64)
        nb = C.c_int64()
        entry = np.zeros(1, ENTRY_DTYPE)
        rc = self.lib.hs_plan_instance(self.handle, float(budget), int(per_token), _ptr(pr), _ptr(I), _ptr(O), q,
                                       _ptr(stops), _ptr(times), C.byref(nb), _ptr(entry))
        self.check(rc, "hs_plan_instance")
        n = int(nb.value)
        return stops[:n], None if times is None else times[:n], entry[0]

    # ---------------------------------------------------------------- search
    def search_tables(self, model: hs_model, engine: hs_engine, limits: hs_limits, machines: np.ndarray,
                      params: np.ndarray, present: np.ndarray, I: np.ndarray, O: np.ndarray):
        M = len(machines)
        table = np.zeros(M * HS_MAX_DEGREES, dtype=ENTRY_DTYPE)
        nd = np.zeros(M, dtype=np.int32)
        I = np.ascontiguousarray(I, dtype=np.int32)
        O = np.ascontiguousarray(O, dtype=np.int32)
        rc = self.lib.hs_search_tables(self.handle, C.byref(model), C.byref(engine), C.byref(limits),
                                       C.cast(machines, C.c_void_p), M, _ptr(params), _ptr(present), _ptr(I),
                                       _ptr(O), len(I), _ptr(table), _ptr(nd))
        self.check(rc, "hs_search_tables")
        return table.reshape(M, HS_MAX_DEGREES), nd

    def search_best(self, table: np.ndarray, nd: np.ndarray, begin: int, end: int):
        best = hs_cand()
        nfeas = C.c_int64()
        t = np.ascontiguousarray(table.reshape(-1))
        rc = self.lib.hs_search_best(self.handle, _ptr(t), _ptr(np.ascontiguousarray(nd, np.int32)), len(nd),
                                     int(begin), int(end), C.byref(best), C.byref(nfeas))
        self.check(rc, "hs_search_best")
        return float(best.total), int(best.index), int(nfeas.value)

    def search_rank(self, table: np.ndarray, nd: np.ndarray):
        P = int(np.prod(nd.astype(np.int64)))
        ranked = np.zeros(max(P, 1), dtype=CAND_DTYPE)
        first_bad = np.zeros(max(P, 1), dtype=np.int8)
        n = C.c_int64()
        t = np.ascontiguousarray(table.reshape(-1))
        rc = self.lib.hs_search_rank(self.handle, _ptr(t), _ptr(np.ascontiguousarray(nd, np.int32)), len(nd),
                                     _ptr(ranked), C.byref(n), _ptr(first_bad))
        self.check(rc, "hs_search_rank")
        return ranked[: n.value], first_bad[:P]

    def search_topk(self, table: np.ndarray, nd: np.ndarray, k: int, shard: int = 0, n_shards: int = 1):
        out = np.zeros(max(k, 1), dtype=CAND_DTYPE)
        n = C.c_int64()
        nf = C.c_int64()
        t = np.ascontiguousarray(table.reshape(-1))
        rc = self.lib.hs_search_topk(self.handle, _ptr(t), _ptr(np.ascontiguousarray(nd, np.int32)), len(nd), int(k),
                                     int(shard), int(n_shards), _ptr(out), C.byref(n), C.byref(nf))
        self.check(rc, "hs_search_topk")
        return out[: n.value], int(nf.value)

    def search_topk_after(self, table: np.ndarray, nd: np.ndarray, k: int, after=None):
        """hs_search_topk_after: the k best candidates ranked after `after` = (total, index)."""
        out = np.zeros(max(k, 1), dtype=CAND_DTYPE)
        n = C.c_int64()
        nf = C.c_int64()
        t = np.ascontiguousarray(table.reshape(-1))
        at, ai = (0.0, -1) if after is None else (float(after[0]), int(after[1]))
        rc = self.lib.hs_search_topk_after(self.handle, _ptr(t), _ptr(np.ascontiguousarray(nd, np.int32)), len(nd),
                                           int(k), at, ai, _ptr(out), C.byref(n), C.byref(nf))
        self.check(rc, "hs_search_topk_after")
        return out[: n.value], int(nf.value)

    # ---------------------------------------------------------------- replay
    def replay(self, instances, policy: hs_policy, offsets: np.ndarray, I: np.ndarray, O: np.ndarray,
               P: np.ndarray | None, arrival: np.ndarray | None, want_assign: bool = True, want_depart: bool = True,
               seeds: hs_replay_seeds | None = None, assign_out: np.ndarray | None = None,
               depart_out: np.ndarray | None = None):
        """hs_replay, or hs_replay_seeded when `seeds` asks for device-drawn
        arrivals / predictions (P may then be None).  assign_out / depart_out:
        optional caller-owned (e.g. page-locked) result buffers."""
        T = len(offsets) - 1
        N = policy.n_instances
        total = int(offsets[-1])
        batch = hs_trace_batch(T, offsets.ctypes.data, I.ctypes.data, O.ctypes.data,
                               None if P is None else P.ctypes.data, None if arrival is None else arrival.ctypes.data)
        assign = _out_buf(assign_out, total, np.uint8) if want_assign else None
        dw = 3 if policy.flags & REPLAY_ORDER_KEYS else 1
        depart = _out_buf(depart_out, total * dw, np.float64) if want_depart else None
        metrics = np.zeros(max(T * N, 1), METRICS_DTYPE)
        result = np.zeros(max(T, 1), RESULT_DTYPE)
        if seeds is None:
            rc = self.lib.hs_replay(self.handle, C.cast(instances, C.c_void_p), C.byref(policy), C.byref(batch),
                                    _ptr(assign), _ptr(depart), _ptr(metrics), _ptr(result))
            self.check(rc, "hs_replay")
        else:
            rc = self.lib.hs_replay_seeded(self.handle, C.cast(instances, C.c_void_p), C.byref(policy),
                                           C.byref(batch), C.byref(seeds), _ptr(assign), _ptr(depart),
                                           _ptr(metrics), _ptr(result))
            self.check(rc, "hs_replay_seeded")
        return (None if assign is None else assign[:total],
                None if depart is None else (depart[:total] if dw == 1 else depart[: 3 * total].reshape(total, 3)),
                metrics[: T * N].reshape(T, N), result[:T])


def pcg64_state(seed: int) -> np.ndarray:
    """numpy.random.PCG64(seed) initial state (SeedSequence(seed) entropy =
    the seed's little-endian 32-bit words) via hs_pcg64_seed; host only."""
    seed = int(seed)
    if seed < 0:
        raise ValueError("expected non-negative integer")
    words = [(seed >> (32 * i)) & 0xFFFFFFFF for i in range(max(1, (seed.bit_length() + 31) // 32))]
    ent = np.array(words, np.uint32)
    out = np.zeros(1, PCG64_DTYPE)
    lib = load_library()
    rc = lib.hs_pcg64_seed(_ptr(ent), len(ent), _ptr(out))
    if rc != HS_OK:
        raise EngineError(rc, "hs_pcg64_seed: " + (lib.hs_last_error() or b"").decode())
    return out


def pcg64_states(seeds) -> np.ndarray:
    """One PCG64 state per seed (PCG64_DTYPE array); one C call for seeds
    below 2^64."""
    seeds = [int(s) for s in seeds]
    if any(s < 0 for s in seeds):
        raise ValueError("expected non-negative integer")
    if not all(s < 2**64 for s in seeds):
        return np.concatenate([pcg64_state(s) for s in seeds])
    arr = np.array(seeds, np.uint64)
    out = np.zeros(len(seeds), PCG64_DTYPE)
    lib = load_library()
    rc = lib.hs_pcg64_seed_u64(_ptr(arr), len(arr), _ptr(out))
    if rc != HS_OK:
        raise EngineError(rc, "hs_pcg64_seed_u64: " + (lib.hs_last_error() or b"").decode())
    return out


_engines: dict = {}
_engines_lock = threading.Lock()


def default_device() -> int:
    env = os.environ.get("HS_DEVICE", os.environ.get("LOCAL_RANK"))
    return int(env) if env else 0


def engine_for(device: int | None = None) -> Engine:
    """The calling thread's engine on `device` (created on first use)."""
    dev = default_device() if device is None else device
    key = (threading.get_ident(), dev)
    with _engines_lock:
        eng = _engines.get(key)
        if eng is None:
            eng = Engine(dev)
            _engines[key] = eng
        return eng
