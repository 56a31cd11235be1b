// capi.cu -- the C ABI (include/hetserve_b200.h): context, device memory,
// argument validation, and the host side of each entry point.  No torch
// types cross this boundary; the Python shim binds it with ctypes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>


#include "hs_device.cuh"
#include "hs_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define HS_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(HS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));          \
  } while (0)

enum Slot {
  S_I, S_O, S_P, S_T, S_OFF, S_DESC, S_TABLE, S_BLK_BEST, S_BLK_IDX, S_BLK_CNT, S_CAND, S_CNT,
  S_TOTAL, S_FIRSTBAD, S_FLAG, S_SELIDX, S_NSEL, S_KEYS, S_KEYS2, S_IDX2, S_CUBTMP, S_RANKED,
  S_ASSIGN, S_DEPART, S_METRICS, S_RESULT, S_WREC, S_HEAP, S_MINNEED, S_TK_HIST, S_TK_CNT, S_TK_KEY,
  S_TK_IDX, S_TK_KEY2, S_TK_IDX2, S_DEPS, S_TDEP, S_THEAP, S_RNG_ST, S_RNG_ST2, S_RNG_OFF, S_RNG_BAD,
  S_PROGRESS, S_STOPS, S_TIMES, S_NB, S_PENTRY, N_SLOTS
};

}  // namespace

constexpr int kPipe = 8;  // replay chunks in flight on the host path

struct hs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;          // copies + search kernels
  cudaStream_t aux = nullptr;             // per-chunk sizing reductions
  cudaStream_t ks[kPipe] = {};            // replay kernels of the pipelined host path
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_copy[kPipe] = {}, ev_min[kPipe] = {}, ev_done[kPipe] = {};
  int32_t* pinned_min = nullptr;          // page-locked per-chunk min(I+O)
  int64_t launches = 0;
  double last_ms = 0.0;
  void* buf[N_SLOTS] = {};
  size_t cap[N_SLOTS] = {};
};

namespace hs {
int set_error(int code, const char* msg) { return fail(code, msg); }

int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
}  // namespace hs

namespace {

int ensure(hs_ctx* c, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  if (c->cap[slot] < bytes) {
    if (c->buf[slot]) cudaFree(c->buf[slot]);
    c->buf[slot] = nullptr;
    c->cap[slot] = 0;
    size_t want = bytes + bytes / 8;
    cudaError_t e = cudaMalloc(&c->buf[slot], want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HS_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(want) + "): " + cudaGetErrorString(e));
    }
    c->cap[slot] = want;
  }
  *out = c->buf[slot];
  return HS_OK;
}

template <typename T>
int ensure_t(hs_ctx* c, int slot, size_t count, T** out) {
  void* p = nullptr;
  int rc = ensure(c, slot, count * sizeof(T), &p);
  *out = static_cast<T*>(p);
  return rc;
}

int use_device(hs_ctx* c) {
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(HS_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return HS_OK;
}

int begin_timing(hs_ctx* c) {
  HS_CUDA(cudaEventRecord(c->ev0, c->stream));
  return HS_OK;
}
int end_timing(hs_ctx* c) {
  HS_CUDA(cudaEventRecord(c->ev1, c->stream));
  HS_CUDA(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  HS_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  c->last_ms = ms;
  return HS_OK;
}

// core.py:363-371 enumerate_tp_degrees
int degrees_of(int64_t count, int32_t* out) {
  int n = 0;
  for (int64_t t = 1; t <= count && n < HS_MAX_DEGREES; t *= 2)
    if (count % t == 0) out[n++] = (int32_t)t;
  return n;
}

// Build the K2 product-space description from a table.
int build_space(const hs_entry* table, const int32_t* nd, int32_t M, hs::SpaceDesc* sd, int32_t* m_off,
                int64_t* P) {
  if (M < 1 || M > HS_MAX_MACHINES) return fail(HS_ERR_ARG, "n_machines out of range");
  std::memset(sd, 0, sizeof(*sd));
  const int off = M >= 4 ? 0 : 4 - M;
  sd->M = M + off;
  for (int v = 0; v < off; ++v) {
    sd->D[v] = 1;
    sd->okcnt[v] = 1;
    sd->C[v * HS_MAX_DEGREES] = 0.0;
  }
  long double size = 1;
  double abs_sum = 0.0;
  int64_t p = 1;
  for (int32_t i = 0; i < M; ++i) {
    if (nd[i] < 1 || nd[i] > HS_MAX_DEGREES) return fail(HS_ERR_ARG, "n_degrees out of range");
    sd->D[i + off] = nd[i];
    size *= nd[i];
    if (size > 4.6e18L) return fail(HS_ERR_ARG, "candidate space exceeds 2^62");
    p *= nd[i];
    double mx = 0.0;
    int64_t ok = 0;
    for (int32_t d = 0; d < nd[i]; ++d) {
      const hs_entry& e = table[i * HS_MAX_DEGREES + d];
      double v = -INFINITY;
      if (e.status == HS_ENTRY_OK) {
        v = e.contribution;
        if (std::isnan(v) || v == -INFINITY)
          return fail(HS_ERR_UNSUPPORTED, "a feasible contribution is NaN or -inf");
        if (std::isfinite(v) && std::fabs(v) > mx) mx = std::fabs(v);
        ++ok;
      }
      sd->C[(i + off) * HS_MAX_DEGREES + d] = v;
    }
    sd->okcnt[i + off] = ok;
    abs_sum += mx;
  }
  if (!(abs_sum < 1e300)) return fail(HS_ERR_UNSUPPORTED, "contributions large enough to overflow a total");
  *m_off = off;
  *P = p;
  return HS_OK;
}

// Largest integer X with per_token * X <= budget (budget > 0): an integer
// product exceeds a float B exactly when it exceeds floor(B)
// (simulator.py:303, planner.py:73).
int64_t cap_tokens(double budget, int64_t per_token) {
  if (!(budget >= 0)) return -1;
  if (budget >= 9.2e18) return INT64_MAX;
  const int64_t fb = (int64_t)std::floor(budget);
  return fb / per_token;
}

// Python sum() semantics for the WRR total (scheduling.py:326)
double pysum(const double* x, int n) {
  double f = 0.0, c = 0.0;
  for (int i = 0; i < n; ++i) {
    if (i == 0) {
      f = 0.0 + x[0];
      continue;
    }
    double t = f + x[i];
    if (std::fabs(f) >= std::fabs(x[i])) c += (f - t) + x[i];
    else c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && std::isfinite(c)) f += c;
  return f;
}

__global__ void k_orderable_keys(const double* total, const int64_t* sel, const int64_t* nsel, uint64_t* keys) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *nsel) return;
  double x = -total[sel[k]];
  if (x == 0.0) x = 0.0;  // -0.0 and 0.0 tie in Python's sort
  uint64_t u = (uint64_t)__double_as_longlong(x);
  keys[k] = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_gather_ranked(const double* total, const int64_t* idx, const int64_t* nsel, hs_cand* out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *nsel) return;
  out[k].total = total[idx[k]];
  out[k].index = idx[k];
}

// Per-launch constants shared by every chunk (instance classes, policy).
int make_const(const hs_instance* inst, const hs_policy* pol, bool has_arrival, hs::ReplayConst* out) {
  const int N = pol->n_instances;
  if (N < 1) return fail(HS_ERR_ARG, "n_instances must be >= 1");
  if (N > HS_MAX_INSTANCES) return fail(HS_ERR_UNSUPPORTED, "more than 255 instances per deployment");
  if (pol->policy < HS_POLICY_OS || pol->policy > HS_POLICY_MB) return fail(HS_ERR_ARG, "unknown policy");
  if (pol->per_token <= 0) return fail(HS_ERR_ARG, "per_token must be positive");
  if (pol->mode != 0 && pol->mode != 1) return fail(HS_ERR_ARG, "mode must be 0 (continuous) or 1 (static)");
  if (pol->mode == 1 && has_arrival) return fail(HS_ERR_ARG, "static mode needs arrival = NULL (rate = inf)");
  hs::ReplayConst& rc = *out;
  std::memset(&rc, 0, sizeof(rc));
  rc.N = N;
  rc.policy = pol->policy;
  rc.theta = pol->theta;
  rc.per_token = pol->per_token;
  rc.has_arrival = has_arrival;
  rc.mode = pol->mode;
  if (pol->flags & ~HS_REPLAY_ORDER_KEYS) return fail(HS_ERR_ARG, "unknown hs_policy.flags bits");
  bool negative = false;  // a negative coefficient can make a step cost negative
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < 8; ++k) negative |= inst[j].p[k] < 0.0;
  rc.flags = (pol->flags & HS_REPLAY_ORDER_KEYS) ? (1 | (negative ? 2 : 0)) : 0;
  bool mono = std::getenv("HS_REPLAY_NO_MONO") == nullptr;  // (diagnostic A/B switch)
  for (int j = 0; j < N; ++j)
    for (int k = 4; k < 8; ++k) mono &= inst[j].p[k] >= 0.0;
  if (mono) rc.flags |= 4;  // replay.cu kMono
  int nt = 0;
  std::vector<double> wts(N);
  for (int j = 0; j < N; ++j) {
    const int ty = inst[j].type;
    if (ty < 0 || ty >= N) return fail(HS_ERR_ARG, "instance type out of range");
    if (ty >= hs::kMaxTypes) return fail(HS_ERR_UNSUPPORTED, "more than 32 distinct instance classes");
    if (!(inst[j].budget > 0)) return fail(HS_ERR_ARG, "instance budget must be positive");
    rc.inst_type[j] = (int8_t)ty;
    bool seen = false;  // every instance of a class must carry the class's exact params and budget
    for (int i = 0; i < j && !seen; ++i) seen = inst[i].type == ty;
    if (seen && (std::memcmp(rc.type_p[ty], inst[j].p, sizeof(double) * 8) != 0 ||
                 std::memcmp(&rc.type_budget[ty], &inst[j].budget, sizeof(double)) != 0))
      return fail(HS_ERR_ARG, "instances sharing a type id differ in params or budget");
    if (ty >= nt) nt = ty + 1;
    std::memcpy(rc.type_p[ty], inst[j].p, sizeof(double) * 8);
    rc.type_budget[ty] = inst[j].budget;
    rc.type_cap_tokens[ty] = cap_tokens(inst[j].budget, pol->per_token);
    rc.wrr_weight[j] = inst[j].wrr_weight;
    wts[j] = inst[j].wrr_weight;
  }
  rc.n_types = nt;
  rc.wrr_total = pysum(wts.data(), N);
  return HS_OK;
}

// Heap overflow regions from the exact active-set bound: at most
// floor(budget / (per_token * min(I+O))) requests fit an instance at once.
// n_max: the widest deployment of the launch (it picks the kernel's warps per
// trace, hence how many heap entries per lane live in shared memory).
//
// Multi-warp traces whose launch knows every output length (max_out >= 0)
// get a retirement calendar instead: 2^cal_bits buckets (> max O, so the
// active retirement steps never share a bucket) of 8 B plus the bucket
// bitmap, per instance, whatever the active-set bound.
int cal_bits_for(int n_max, int32_t max_out) {
  if ((n_max + 31) / 32 < 2 || max_out < 0) return 0;
  int b = 6;
  while (b <= hs::kMaxCalBits && (1 << b) <= max_out) ++b;  // 2^b > max(O, 1)
  return b <= hs::kMaxCalBits ? b : 0;
}

void size_heaps(hs::ReplayConst& rc, const hs_instance* inst, int32_t min_need, int64_t max_q, int n_max = 0,
                int cal_bits = 0) {
  rc.cal_bits = cal_bits;
  if (cal_bits > 0) {
    const int64_t B = int64_t(1) << cal_bits;
    const int64_t per = (B * 8 + (B / 64) * 8 + hs::kHEntBytes - 1) / hs::kHEntBytes;  // in heap entries
    for (int j = 0; j <= rc.N; ++j) rc.heap_off[j] = j * per;
    rc.heap_stride = (rc.N * per + 15) / 16 * 16;
    return;
  }
  const int shared = hs::replay_heap_prefix(((n_max > 0 ? n_max : rc.N) + 31) / 32);
  if (min_need < 1) min_need = 1;
  int64_t acc = 0;
  for (int j = 0; j < rc.N; ++j) {
    const double tokens = std::floor(inst[j].budget / (double)rc.per_token);
    const double capd = std::floor(tokens / (double)min_need) + 1.0;
    int64_t capj = capd > (double)max_q ? max_q : (int64_t)capd;
    capj -= shared;  // the first entries live in shared memory
    if (capj < 1) capj = 1;
    rc.heap_off[j] = acc;
    acc += capj;
  }
  rc.heap_off[rc.N] = acc;
  rc.heap_stride = (acc + 15) / 16 * 16;
}

int check_offsets(const int64_t* h_off, int64_t T, int64_t* max_q) {
  *max_q = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int64_t qt = h_off[t + 1] - h_off[t];
    if (qt < 0) return fail(HS_ERR_ARG, "offsets must be non-decreasing");
    if (qt > INT32_MAX) return fail(HS_ERR_UNSUPPORTED, "trace longer than 2^31 requests");
    if (qt > *max_q) *max_q = qt;
  }
  return HS_OK;
}

// Device-resident inputs: one sizing reduction, then the traces in as few
// launches as the heap memory allows.
int replay_impl(hs_ctx* c, const hs_instance* inst, const hs_policy* pol, int64_t T, const int64_t* d_off,
                const int64_t* h_off, const int32_t* d_I, const int32_t* d_O, const int32_t* d_P, const double* d_arr,
                uint8_t* d_assign, double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result) {
  hs::ReplayConst rc;
  int rcode;
  if ((rcode = make_const(inst, pol, d_arr != nullptr, &rc))) return rcode;
  const int N = rc.N;
  int64_t max_q;
  if ((rcode = check_offsets(h_off, T, &max_q))) return rcode;
  const int64_t total_q = h_off[T] - h_off[0];
  int32_t* d_min = nullptr;
  if ((rcode = ensure_t(c, S_MINNEED, 2, &d_min))) return rcode;
  HS_CUDA(cudaMemsetAsync(d_min, 0x7f, sizeof(int32_t), c->stream));
  HS_CUDA(cudaMemsetAsync(d_min + 1, 0, sizeof(int32_t), c->stream));
  if (total_q > 0) {
    HS_CUDA(hs::launch_min_need(d_I + h_off[0], d_O + h_off[0], total_q, d_min, c->stream, d_min + 1));
    c->launches += 1;
  }
  int32_t need_stats[2] = {0, 0};  // min(I + O), max(O)
  HS_CUDA(cudaMemcpyAsync(need_stats, d_min, sizeof(need_stats), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  const int32_t min_need = need_stats[0];
  size_heaps(rc, inst, min_need, max_q, 0, cal_bits_for(rc.N, need_stats[1]));
  void* d_qrec;
  if ((rcode = ensure(c, S_WREC, (size_t)(h_off[T] > 0 ? h_off[T] : 1) * hs::kQRecBytes, &d_qrec))) return rcode;
  const size_t per_trace = (size_t)rc.heap_stride * hs::kHEntBytes;
  int64_t chunk = T;
  if ((size_t)T * per_trace > c->cap[S_HEAP]) {  // query free memory only when the heap buffer must grow
    size_t free_b = 0, tot_b = 0;
    HS_CUDA(cudaMemGetInfo(&free_b, &tot_b));
    const size_t budget_b = (size_t)((double)(free_b + c->cap[S_HEAP]) * 0.6);
    chunk = per_trace ? (int64_t)(budget_b / per_trace) : T;
  }
  if (chunk < 1) chunk = 1;
  if (chunk > T) chunk = T;
  if (chunk > 16384) chunk = 16384;
  uint64_t* d_heap = nullptr;
  if ((rcode = ensure_t(c, S_HEAP, (size_t)(chunk > 0 ? chunk : 1) * rc.heap_stride * 2, &d_heap))) return rcode;
  if ((rcode = begin_timing(c))) return rcode;
  for (int64_t t0 = 0; t0 < T; t0 += chunk) {
    const int64_t nt_ = (T - t0) < chunk ? (T - t0) : chunk;
    HS_CUDA(hs::launch_replay(rc, nt_, d_off + t0, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics + t0 * N,
                              d_result + t0, d_qrec, d_heap, c->stream));
    c->launches += 1;
  }
  return end_timing(c);
}

int ensure_pipeline(hs_ctx* c) {
  if (c->aux) return HS_OK;
  HS_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  for (int i = 0; i < kPipe; ++i) {
    HS_CUDA(cudaStreamCreateWithFlags(&c->ks[i], cudaStreamNonBlocking));
    HS_CUDA(cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming));
    HS_CUDA(cudaEventCreateWithFlags(&c->ev_min[i], cudaEventDisableTiming));
    HS_CUDA(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
  }
  HS_CUDA(cudaHostAlloc((void**)&c->pinned_min, sizeof(int32_t) * kPipe, cudaHostAllocDefault));
  cudaMemPool_t pool;
  HS_CUDA(cudaDeviceGetDefaultMemPool(&pool, c->device));
  uint64_t keep = UINT64_MAX;  // keep freed chunk heaps in the pool between calls
  HS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  return HS_OK;
}

__global__ void k_probe_fp64(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 1e-12;
  for (int i = 0; i < iters; ++i) {
    a0 = __dadd_rn(a0, b); a1 = __dadd_rn(a1, b); a2 = __dadd_rn(a2, b); a3 = __dadd_rn(a3, b);
    a4 = __dadd_rn(a4, b); a5 = __dadd_rn(a5, b); a6 = __dadd_rn(a6, b); a7 = __dadd_rn(a7, b);
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 42.0) out[0] = s;
}

}  // namespace

extern "C" {

int hs_abi_version(void) { return HS_ABI_VERSION; }

const char* hs_last_error(void) { return g_err.c_str(); }

int hs_ctx_create(int device, hs_ctx** out) {
  if (!out) return fail(HS_ERR_ARG, "out is null");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(HS_ERR_CUDA, "no CUDA device available");
  if (device < 0 || device >= n) return fail(HS_ERR_ARG, "device index out of range");
  hs_ctx* c = new hs_ctx();
  c->device = device;
  if (use_device(c)) {
    delete c;
    return HS_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
    delete c;
    return fail(HS_ERR_CUDA, "stream/event creation failed");
  }
  *out = c;
  return HS_OK;
}

int hs_ctx_destroy(hs_ctx* c) {
  if (!c) return HS_OK;
  cudaSetDevice(c->device);
  for (int s = 0; s < N_SLOTS; ++s)
    if (c->buf[s]) cudaFree(c->buf[s]);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->aux) {
    for (int i = 0; i < kPipe; ++i) {
      cudaStreamDestroy(c->ks[i]);
      cudaEventDestroy(c->ev_copy[i]);
      cudaEventDestroy(c->ev_min[i]);
      cudaEventDestroy(c->ev_done[i]);
    }
    cudaStreamDestroy(c->aux);
    cudaFreeHost(c->pinned_min);
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return HS_OK;
}

int64_t hs_ctx_launch_count(const hs_ctx* c) { return c ? c->launches : 0; }
void* hs_ctx_stream(const hs_ctx* c) { return c ? (void*)c->stream : nullptr; }

int hs_probe_fp64(hs_ctx* c, double* out) {
  if (!c || !out) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  double* d;
  if ((rc = ensure_t(c, S_CAND, 2, &d))) return rc;
  const int blocks = hs::sm_count() * 8, threads = 256, iters = 1 << 14;
  k_probe_fp64<<<blocks, threads, 0, c->stream>>>(d, 256);  // warm-up
  HS_CUDA(cudaGetLastError());
  if ((rc = begin_timing(c))) return rc;
  k_probe_fp64<<<blocks, threads, 0, c->stream>>>(d, iters);
  HS_CUDA(cudaGetLastError());
  if ((rc = end_timing(c))) return rc;
  c->launches += 2;
  *out = (double)blocks * threads * iters * 8.0 / (c->last_ms * 1e-3);
  return HS_OK;
}
double hs_ctx_last_kernel_ms(const hs_ctx* c) { return c ? c->last_ms : 0.0; }
// CPython math.exp (glibc 2.39, FMA variant) as the replay evaluates it
// (scheduling.py:154 via hs_device.cuh py_exp), over an array.
__global__ void k_exp_batch(const double* __restrict__ x, int64_t n, double* __restrict__ y,
                            uint8_t* __restrict__ of) {
  __shared__ uint64_t tab[256];
  for (int k = threadIdx.x; k < 256; k += blockDim.x) tab[k] = kExpTab[k];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool o;
    y[i] = hs::py_exp(x[i], tab, &o);
    of[i] = o ? 1 : 0;
  }
}

__global__ void k_floordiv_batch(const double* __restrict__ x, const double* __restrict__ w, int64_t n,
                                 double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = hs::py_floordiv(x[i], w[i]);
}

int hs_floordiv_batch(hs_ctx* c, const double* x, const double* w, int64_t n, double* y) {
  if (!c || n < 0 || (n > 0 && (!x || !w || !y))) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  if (n == 0) return HS_OK;
  double *dx, *dw, *dy;
  if ((rc = ensure_t(c, S_TOTAL, (size_t)n, &dx)) || (rc = ensure_t(c, S_KEYS2, (size_t)n, &dw)) ||
      (rc = ensure_t(c, S_KEYS, (size_t)n, &dy)))
    return rc;
  HS_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemcpyAsync(dw, w, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  if ((rc = begin_timing(c))) return rc;
  int64_t blocks = (n + 255) / 256;
  if (blocks > hs::sm_count() * 16) blocks = hs::sm_count() * 16;
  k_floordiv_batch<<<(unsigned)blocks, 256, 0, c->stream>>>(dx, dw, n, dy);
  HS_CUDA(cudaGetLastError());
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  HS_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}

__global__ void k_div_batch(const double* __restrict__ x, const double* __restrict__ b, int64_t n,
                            double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = hs::div_rn_by(x[i], b[i], __ddiv_rn(1.0, b[i]));
}

int hs_div_batch(hs_ctx* c, const double* x, const double* b, int64_t n, double* y) {
  if (!c || n < 0 || (n > 0 && (!x || !b || !y))) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  if (n == 0) return HS_OK;
  double *dx, *db, *dy;
  if ((rc = ensure_t(c, S_TOTAL, (size_t)n, &dx)) || (rc = ensure_t(c, S_KEYS2, (size_t)n, &db)) ||
      (rc = ensure_t(c, S_KEYS, (size_t)n, &dy)))
    return rc;
  HS_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  int64_t blocks = (n + 255) / 256;
  if (blocks > hs::sm_count() * 16) blocks = hs::sm_count() * 16;
  k_div_batch<<<(unsigned)blocks, 256, 0, c->stream>>>(dx, db, n, dy);
  HS_CUDA(cudaGetLastError());
  c->launches += 1;
  HS_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}

int hs_exp_batch(hs_ctx* c, const double* x, int64_t n, double* y, uint8_t* overflow) {
  if (!c || n < 0 || (n > 0 && (!x || !y || !overflow))) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  if (n == 0) return HS_OK;
  double *dx, *dy;
  uint8_t* dof;
  if ((rc = ensure_t(c, S_TOTAL, (size_t)n, &dx)) || (rc = ensure_t(c, S_KEYS, (size_t)n, &dy)) ||
      (rc = ensure_t(c, S_FLAG, (size_t)n, &dof)))
    return rc;
  HS_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  if ((rc = begin_timing(c))) return rc;
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > hs::sm_count() * 16) blocks = hs::sm_count() * 16;
  k_exp_batch<<<(unsigned)blocks, threads, 0, c->stream>>>(dx, n, dy, dof);
  HS_CUDA(cudaGetLastError());
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  HS_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaMemcpyAsync(overflow, dof, (size_t)n, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}


int hs_search_tables(hs_ctx* c, const hs_model* model, const hs_engine* engine, const hs_limits* limits,
                     const hs_machine* machines, int32_t M, const double* params, const uint8_t* present,
                     const int32_t* I, const int32_t* O, int64_t q, hs_entry* table, int32_t* n_degrees) {
  if (!c || !model || !engine || !limits || !machines || !params || !present || !table || !n_degrees)
    return fail(HS_ERR_ARG, "null argument");
  if (M < 1 || M > HS_MAX_MACHINES) return fail(HS_ERR_ARG, "n_machines out of range");
  if (q < 0 || (q > 0 && (!I || !O))) return fail(HS_ERR_ARG, "bad trace arguments");
  int rc;
  if ((rc = use_device(c))) return rc;
  std::vector<hs::EntryDesc> desc;
  std::vector<int> slot;
  for (int32_t i = 0; i < M; ++i) {
    const hs_machine& own = machines[i];
    if (own.spec_index < 0 || own.spec_index >= M) return fail(HS_ERR_ARG, "spec_index out of range");
    const hs_machine& spec = machines[own.spec_index];
    int32_t deg[HS_MAX_DEGREES];
    int nd;
    if (own.fixed_degree > 0) {
      deg[0] = own.fixed_degree;
      nd = 1;
    } else {
      nd = degrees_of(own.accelerator_count, deg);
    }
    n_degrees[i] = nd;
    for (int d = 0; d < nd; ++d) {
      hs::EntryDesc e;
      std::memcpy(e.p, params + ((size_t)i * HS_MAX_DEGREES + d) * 8, sizeof(double) * 8);
      e.own_count = own.accelerator_count;
      e.spec_count = spec.accelerator_count;
      e.spec_mem = spec.accelerator_mem_bytes;
      e.tp = deg[d];
      e.present = present[i * HS_MAX_DEGREES + d] ? 1 : 0;
      desc.push_back(e);
      slot.push_back(i * HS_MAX_DEGREES + d);
    }
  }
  hs::SearchConst sc;
  sc.per_token = 2 * model->layers * model->hidden_dim * model->bytes_per_param;
  sc.required = sc.per_token * (limits->max_input_len + limits->max_output_len);
  sc.weights = model->param_count * model->bytes_per_param;
  sc.static_overhead = engine->static_overhead_bytes;
  sc.phi = engine->mem_utilization_fraction;
  sc.q = q;
  const int n = (int)desc.size();
  int32_t *dI, *dO;
  hs::EntryDesc* dD;
  hs_entry* dT;
  if ((rc = ensure_t(c, S_I, (size_t)(q > 0 ? q : 1), &dI)) || (rc = ensure_t(c, S_O, (size_t)(q > 0 ? q : 1), &dO)) ||
      (rc = ensure_t(c, S_DESC, (size_t)n, &dD)) || (rc = ensure_t(c, S_TABLE, (size_t)n, &dT)))
    return rc;
  if (q > 0) {
    HS_CUDA(cudaMemcpyAsync(dI, I, sizeof(int32_t) * q, cudaMemcpyHostToDevice, c->stream));
    HS_CUDA(cudaMemcpyAsync(dO, O, sizeof(int32_t) * q, cudaMemcpyHostToDevice, c->stream));
  }
  HS_CUDA(cudaMemcpyAsync(dD, desc.data(), sizeof(hs::EntryDesc) * n, cudaMemcpyHostToDevice, c->stream));
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_table_build(dD, n, sc, dI, dO, dT, c->stream));
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  std::vector<hs_entry> out(n);
  HS_CUDA(cudaMemcpyAsync(out.data(), dT, sizeof(hs_entry) * n, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < n; ++k) table[slot[k]] = out[k];
  return HS_OK;
}

int hs_plan_instance(hs_ctx* c, double budget, int64_t per_token, const double* params, const int32_t* I,
                     const int32_t* O, int64_t q, int64_t* stops, double* times, int64_t* n_batches,
                     hs_entry* entry) {
  if (!c || !entry || !n_batches || (q > 0 && (!I || !O || !stops))) return fail(HS_ERR_ARG, "null argument");
  if (q < 0) return fail(HS_ERR_ARG, "q < 0");
  if (per_token <= 0) return fail(HS_ERR_ARG, "per_token must be positive");
  if (params && q > 0 && !times) return fail(HS_ERR_ARG, "times is null");
  int rc;
  if ((rc = use_device(c))) return rc;
  const size_t qq = (size_t)(q > 0 ? q : 1);
  int32_t *dI, *dO;
  int64_t *dS, *dNb;
  double* dTm;
  hs_entry* dE;
  if ((rc = ensure_t(c, S_I, qq, &dI)) || (rc = ensure_t(c, S_O, qq, &dO)) || (rc = ensure_t(c, S_STOPS, qq, &dS)) ||
      (rc = ensure_t(c, S_TIMES, qq, &dTm)) || (rc = ensure_t(c, S_NB, 1, &dNb)) || (rc = ensure_t(c, S_PENTRY, 1, &dE)))
    return rc;
  if (q > 0) {
    HS_CUDA(cudaMemcpyAsync(dI, I, sizeof(int32_t) * q, cudaMemcpyHostToDevice, c->stream));
    HS_CUDA(cudaMemcpyAsync(dO, O, sizeof(int32_t) * q, cudaMemcpyHostToDevice, c->stream));
  }
  hs::PlanParams pp{};
  pp.has = params != nullptr;
  if (params) std::memcpy(pp.p, params, sizeof(pp.p));
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_plan_instance(budget, per_token, pp, dI, dO, q, dS, dTm, dNb, dE, c->stream));
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  HS_CUDA(cudaMemcpyAsync(n_batches, dNb, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaMemcpyAsync(entry, dE, sizeof(hs_entry), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t nb = *n_batches;
  if (nb > 0) {
    HS_CUDA(cudaMemcpyAsync(stops, dS, sizeof(int64_t) * nb, cudaMemcpyDeviceToHost, c->stream));
    if (params) HS_CUDA(cudaMemcpyAsync(times, dTm, sizeof(double) * nb, cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
  }
  return HS_OK;
}

// The feasible sub-product of a space: per machine its OK degrees only, in
// degree order.  The map is monotone in every digit, so it preserves the
// mixed-radix order (itertools.product order, planner.py:216): the argmax
// with the lowest-index tie rule (planner.py:227) over the feasible
// sub-product is the argmax over the whole space, and the feasible
// candidates of an index range [b, e) are the compressed range
// [rank(b), rank(e)).  Infeasible candidates (-inf contributions) can never
// win, so the kernel need not visit them: every one of them is decided by
// the per-machine factorisation (hs_entry.status), not by a sum.
struct Compressed {
  hs::SpaceDesc cs;
  int32_t orig[hs::kMaxM][HS_MAX_DEGREES];
  int64_t suffix_ok[hs::kMaxM + 1];  // prod of okcnt over machines > i
  int64_t feasible;
};

void compress_space(const hs::SpaceDesc& sd, Compressed* c) {
  std::memset(&c->cs, 0, sizeof(c->cs));
  c->cs.M = sd.M;
  for (int i = 0; i < sd.M; ++i) {
    int k = 0;
    for (int d = 0; d < sd.D[i]; ++d) {
      const double v = sd.C[i * HS_MAX_DEGREES + d];
      if (v == -INFINITY) continue;
      c->cs.C[i * HS_MAX_DEGREES + k] = v;
      c->orig[i][k] = d;
      ++k;
    }
    c->cs.D[i] = k;
    c->cs.okcnt[i] = k;
  }
  c->suffix_ok[sd.M] = 1;
  for (int i = sd.M - 1; i >= 0; --i) c->suffix_ok[i] = c->suffix_ok[i + 1] * sd.okcnt[i];
  c->feasible = c->suffix_ok[0];
}

// number of feasible candidates with original index < x
int64_t feasible_rank(const hs::SpaceDesc& sd, const Compressed& c, int64_t x, int64_t P) {
  if (x >= P) return c.feasible;
  int32_t dig[hs::kMaxM];
  for (int i = sd.M - 1; i >= 0; --i) {
    dig[i] = (int32_t)(x % sd.D[i]);
    x /= sd.D[i];
  }
  int64_t r = 0;
  for (int i = 0; i < sd.M; ++i) {
    int less = 0;
    for (int d = 0; d < dig[i]; ++d) less += sd.C[i * HS_MAX_DEGREES + d] != -INFINITY;
    r += (int64_t)less * c.suffix_ok[i + 1];
    if (sd.C[i * HS_MAX_DEGREES + dig[i]] == -INFINITY) break;
  }
  return r;
}

int64_t original_index(const hs::SpaceDesc& sd, const Compressed& c, int64_t ci) {
  int32_t dig[hs::kMaxM];
  for (int i = sd.M - 1; i >= 0; --i) {
    dig[i] = c.orig[i][ci % c.cs.D[i]];
    ci /= c.cs.D[i];
  }
  int64_t x = 0;
  for (int i = 0; i < sd.M; ++i) x = x * sd.D[i] + dig[i];
  return x;
}

int hs_search_best(hs_ctx* c, const hs_entry* table, const int32_t* n_degrees, int32_t M, int64_t begin, int64_t end,
                   hs_cand* best, int64_t* n_feasible) {
  if (!c || !table || !n_degrees || !best || !n_feasible) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  hs::SpaceDesc sd;
  int32_t m_off;
  int64_t P;
  if ((rc = build_space(table, n_degrees, M, &sd, &m_off, &P))) return rc;
  if (begin < 0 || end > P || begin > end) return fail(HS_ERR_ARG, "index range outside the candidate space");
  // default: the feasible sub-product (HS_SEARCH_EXHAUSTIVE=1: every candidate)
  const bool exhaustive = std::getenv("HS_SEARCH_EXHAUSTIVE") != nullptr;
  static thread_local Compressed cmp;
  const hs::SpaceDesc* space = &sd;
  int64_t b = begin, e = end;
  if (!exhaustive) {
    compress_space(sd, &cmp);
    b = feasible_rank(sd, cmp, begin, P);
    e = feasible_rank(sd, cmp, end, P);
    space = &cmp.cs;
    if (e <= b) {  // nothing feasible in the range
      best->total = 0.0;
      best->index = -1;
      *n_feasible = 0;
      c->last_ms = 0.0;
      return HS_OK;
    }
  }
  const int64_t Din = (int64_t)space->D[space->M - 4] * space->D[space->M - 3] * space->D[space->M - 2] *
                      space->D[space->M - 1];
  const int64_t items = (e - b) / Din + 2;
  int blocks = hs::sm_count() * 8;
  const int64_t need_blocks = (items + 255) / 256;
  if (need_blocks < blocks) blocks = (int)(need_blocks > 0 ? need_blocks : 1);
  double* bb;
  int64_t *bi, *bc, *cnt;
  hs_cand* cand;
  if ((rc = ensure_t(c, S_BLK_BEST, (size_t)blocks, &bb)) || (rc = ensure_t(c, S_BLK_IDX, (size_t)blocks, &bi)) ||
      (rc = ensure_t(c, S_BLK_CNT, (size_t)blocks, &bc)) || (rc = ensure_t(c, S_CAND, 1, &cand)) ||
      (rc = ensure_t(c, S_CNT, 1, &cnt)))
    return rc;
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_search_best(*space, b, e, blocks, bb, bi, bc, cand, cnt, c->stream));
  c->launches += 2;
  if ((rc = end_timing(c))) return rc;
  HS_CUDA(cudaMemcpyAsync(best, cand, sizeof(hs_cand), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaMemcpyAsync(n_feasible, cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  if (!exhaustive && best->index >= 0) best->index = original_index(sd, cmp, best->index);
  return HS_OK;
}

int hs_search_rank(hs_ctx* c, const hs_entry* table, const int32_t* n_degrees, int32_t M, hs_cand* ranked,
                   int64_t* n_ranked, int8_t* first_bad) {
  if (!c || !table || !n_degrees || !ranked || !n_ranked || !first_bad) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  hs::SpaceDesc sd;
  int32_t m_off;
  int64_t P;
  if ((rc = build_space(table, n_degrees, M, &sd, &m_off, &P))) return rc;
  if (P > (int64_t(1) << 26)) return fail(HS_ERR_UNSUPPORTED, "space too large to rank in full (use hs_search_best)");
  double* tot;
  int8_t* fb;
  uint8_t* flag;
  int64_t *sel, *nsel, *idx2;
  uint64_t *keys, *keys2;
  hs_cand* out;
  if ((rc = ensure_t(c, S_TOTAL, (size_t)P, &tot)) || (rc = ensure_t(c, S_FIRSTBAD, (size_t)P, &fb)) ||
      (rc = ensure_t(c, S_FLAG, (size_t)P, &flag)) || (rc = ensure_t(c, S_SELIDX, (size_t)P, &sel)) ||
      (rc = ensure_t(c, S_NSEL, 1, &nsel)) || (rc = ensure_t(c, S_KEYS, (size_t)P, &keys)) ||
      (rc = ensure_t(c, S_KEYS2, (size_t)P, &keys2)) || (rc = ensure_t(c, S_IDX2, (size_t)P, &idx2)) ||
      (rc = ensure_t(c, S_RANKED, (size_t)P, &out)))
    return rc;
  void* tmp;
  if ((rc = ensure(c, S_CUBTMP, hs::sort_workspace_bytes(P), &tmp))) return rc;
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_search_score(sd, m_off, P, tot, fb, flag, c->stream));
  HS_CUDA(hs::select_flagged(flag, P, sel, nsel, tmp, c->stream));
  const unsigned g = (unsigned)((P + 255) / 256);
  k_orderable_keys<<<g, 256, 0, c->stream>>>(tot, sel, nsel, keys);
  HS_CUDA(cudaGetLastError());
  int64_t h_nsel = 0;
  HS_CUDA(cudaMemcpyAsync(&h_nsel, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  if (h_nsel > 0) {
    // (key, index) pairs by key: ties keep the index order of the selection
    HS_CUDA(hs::sort_pairs_u64(keys, reinterpret_cast<uint64_t*>(sel), keys2, reinterpret_cast<uint64_t*>(idx2),
                               h_nsel, 0, 64, tmp, c->stream));
    k_gather_ranked<<<g, 256, 0, c->stream>>>(tot, sel, nsel, out);
    HS_CUDA(cudaGetLastError());
  }
  c->launches += 5;
  if ((rc = end_timing(c))) return rc;
  if (h_nsel > 0)
    HS_CUDA(cudaMemcpyAsync(ranked, out, sizeof(hs_cand) * h_nsel, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaMemcpyAsync(first_bad, fb, (size_t)P, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  *n_ranked = h_nsel;
  return HS_OK;
}

namespace {
int search_topk_impl(hs_ctx* c, const hs_entry* table, const int32_t* nd, int32_t M, int64_t k, int32_t shard,
                     int32_t n_shards, bool has_after, double after_total, int64_t after_index, hs_cand* out,
                     int64_t* n_out, int64_t* n_feasible);
}

int hs_search_topk(hs_ctx* c, const hs_entry* table, const int32_t* nd, int32_t M, int64_t k, int32_t shard,
                   int32_t n_shards, hs_cand* out, int64_t* n_out, int64_t* n_feasible) {
  return search_topk_impl(c, table, nd, M, k, shard, n_shards, false, 0.0, -1, out, n_out, n_feasible);
}

int hs_search_topk_after(hs_ctx* c, const hs_entry* table, const int32_t* nd, int32_t M, int64_t k,
                         double after_total, int64_t after_index, hs_cand* out, int64_t* n_out,
                         int64_t* n_feasible) {
  return search_topk_impl(c, table, nd, M, k, 0, 1, after_index >= 0, after_total, after_index, out, n_out,
                          n_feasible);
}

namespace {
int search_topk_impl(hs_ctx* c, const hs_entry* table, const int32_t* nd, int32_t M, int64_t k, int32_t shard,
                     int32_t n_shards, bool has_after, double after_total, int64_t after_index, hs_cand* out,
                     int64_t* n_out, int64_t* n_feasible) {
  if (!c || !table || !nd || !out || !n_out || !n_feasible) return fail(HS_ERR_ARG, "null argument");
  if (M < 1 || M > HS_MAX_MACHINES) return fail(HS_ERR_ARG, "n_machines out of range");
  if (k < 0 || n_shards < 1 || shard < 0 || shard >= n_shards) return fail(HS_ERR_ARG, "bad k / shard");
  int rc;
  if ((rc = use_device(c))) return rc;
  hs::FeasSpace fs;
  std::memset(&fs, 0, sizeof(fs));
  fs.M = M;
  long double F = 1;
  int64_t stride = 1;
  for (int32_t i = M - 1; i >= 0; --i) {
    if (nd[i] < 1 || nd[i] > HS_MAX_DEGREES) return fail(HS_ERR_ARG, "n_degrees out of range");
    fs.stride[i] = stride;
    stride *= nd[i];
    int32_t ok = 0;
    for (int32_t d = 0; d < nd[i]; ++d) {
      const hs_entry& e = table[i * HS_MAX_DEGREES + d];
      if (e.status != HS_ENTRY_OK) continue;
      if (std::isnan(e.contribution)) return fail(HS_ERR_UNSUPPORTED, "a feasible contribution is NaN");
      fs.C[i * HS_MAX_DEGREES + ok] = e.contribution;
      fs.orig[i * HS_MAX_DEGREES + ok] = d;
      ++ok;
    }
    fs.D[i] = ok;
    F *= ok;
  }
  *n_out = 0;
  *n_feasible = 0;
  if (F == 0) return HS_OK;
  if (F > 4.6e18L) return fail(HS_ERR_ARG, "feasible space exceeds 2^62");
  const int64_t DL = fs.D[M - 1];
  const int64_t items = (int64_t)(F / DL);
  const int64_t ib = items * shard / n_shards, ie = items * (shard + 1) / n_shards;
  const int64_t nf = (ie - ib) * DL;
  *n_feasible = nf;
  int64_t K = k < nf ? k : nf;
  if (K == 0) return HS_OK;
  uint64_t bkey = ~0ull;  // no boundary: every key is below it
  if (has_after) {
    double x = after_total;
    if (x == 0.0) x = 0.0;  // -0.0 and 0.0 tie
    const uint64_t u = (uint64_t)*reinterpret_cast<const int64_t*>(&x);
    bkey = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  }
  const int64_t bidx = has_after ? after_index : -1;
  const int64_t CAP = (int64_t)1 << 20;
  unsigned long long *d_hist, *d_cnt;
  uint64_t *d_key, *d_key2;
  int64_t *d_idx, *d_idx2;
  if ((rc = ensure_t(c, S_TK_HIST, 4096, &d_hist)) || (rc = ensure_t(c, S_TK_CNT, 1, &d_cnt)) ||
      (rc = ensure_t(c, S_TK_KEY, (size_t)CAP, &d_key)) || (rc = ensure_t(c, S_TK_IDX, (size_t)CAP, &d_idx)) ||
      (rc = ensure_t(c, S_TK_KEY2, (size_t)CAP, &d_key2)) || (rc = ensure_t(c, S_TK_IDX2, (size_t)CAP, &d_idx2)))
    return rc;
  int blocks = hs::sm_count() * 8;
  const int64_t nb = (ie - ib + 255) / 256;
  if (nb < blocks) blocks = (int)(nb > 0 ? nb : 1);
  std::vector<unsigned long long> h(4096);
  uint64_t prefix = 0;
  int64_t need = K, above = 0;
  int shift = 52;
  uint64_t thr = 0;
  bool uploaded = false;
  if ((rc = begin_timing(c))) return rc;
  for (;; shift -= 12) {
    HS_CUDA(cudaMemsetAsync(d_hist, 0, 4096 * sizeof(unsigned long long), c->stream));
    HS_CUDA(hs::launch_topk_pass(fs, !uploaded, 0, ib, ie, shift, prefix, 0, d_hist, d_cnt, d_key, d_idx, CAP, blocks,
                                 c->stream, bkey, bidx));
    uploaded = true;
    c->launches += 1;
    HS_CUDA(cudaMemcpyAsync(h.data(), d_hist, 4096 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    if (shift == 52 && has_after) {  // candidates after the boundary: fewer than k near the end
      int64_t left = 0;
      for (int bb = 0; bb < 4096; ++bb) left += (int64_t)h[bb];
      if (left < need) need = K = left;
      if (K == 0) {
        if ((rc = end_timing(c))) return rc;
        return HS_OK;
      }
    }
    int bsel = -1;
    int64_t cum = 0;
    for (int bb = 4095; bb >= 0; --bb) {
      if (cum + (int64_t)h[bb] >= need) {
        bsel = bb;
        break;
      }
      cum += (int64_t)h[bb];
    }
    if (bsel < 0) return fail(HS_ERR_CUDA, "top-k radix select lost candidates");
    need -= cum;
    above += cum;
    prefix = (shift == 52) ? (uint64_t)bsel : ((prefix << 12) | (uint64_t)bsel);
    thr = prefix << shift;
    if (above + (int64_t)h[bsel] <= CAP || shift == 4) break;
  }
  HS_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), c->stream));
  HS_CUDA(hs::launch_topk_pass(fs, false, 1, ib, ie, shift, prefix, thr, d_hist, d_cnt, d_key, d_idx, CAP, blocks,
                               c->stream, bkey, bidx));
  c->launches += 1;
  unsigned long long got = 0;
  HS_CUDA(cudaMemcpyAsync(&got, d_cnt, sizeof(got), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  if ((int64_t)got > CAP) return fail(HS_ERR_UNSUPPORTED, "more than 2^20 candidates tie at the top-k boundary");
  const int n = (int)got;
  // stable sorts: by index ascending, then by total descending (~key ascending)
  void* tmp;
  if ((rc = ensure(c, S_CUBTMP, hs::sort_workspace_bytes(n), &tmp))) return rc;
  HS_CUDA(hs::sort_pairs_u64(reinterpret_cast<uint64_t*>(d_idx), d_key, reinterpret_cast<uint64_t*>(d_idx2), d_key2,
                             n, 0, 64, tmp, c->stream));
  HS_CUDA(hs::launch_invert_keys(d_key, n, c->stream));
  HS_CUDA(hs::sort_pairs_u64(d_key, reinterpret_cast<uint64_t*>(d_idx), d_key2, reinterpret_cast<uint64_t*>(d_idx2),
                             n, 0, 64, tmp, c->stream));
  c->launches += 3;
  if ((rc = end_timing(c))) return rc;
  std::vector<uint64_t> hk((size_t)K);
  std::vector<int64_t> hi((size_t)K);
  HS_CUDA(cudaMemcpyAsync(hk.data(), d_key, sizeof(uint64_t) * K, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaMemcpyAsync(hi.data(), d_idx, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  for (int64_t j = 0; j < K; ++j) {
    const uint64_t key = ~hk[j];
    const uint64_t u = (key >> 63) ? (key & 0x7fffffffffffffffull) : ~key;
    double v;
    std::memcpy(&v, &u, 8);
    out[j].total = v;
    out[j].index = hi[j];
  }
  *n_out = K;
  return HS_OK;
}
}  // namespace

namespace {

int check_dist(const hs_dist& d) {
  if (d.kind < HS_DIST_LOGNORMAL_LEN || d.kind > HS_DIST_NORMAL_LEN) return fail(HS_ERR_ARG, "unknown distribution");
  if (d.kind != HS_DIST_EXP_CUMSUM && d.cap < 1) return fail(HS_ERR_ARG, "length cap must be >= 1");
  if (d.kind == HS_DIST_UNIFORM_LEN && d.lo > d.hi) return fail(HS_ERR_ARG, "uniform needs lo <= hi");
  return HS_OK;
}

// hs_replay / hs_replay_seeded: host buffers, traces replayed in kPipe chunks
// (copy of chunk i+1 overlaps the replay of chunk i); seeded arrivals and
// predictions are drawn on the chunk's stream right before its replay.
// cuStreamWriteValue32 (driver API, through the runtime's entry-point
// query): the copy stream publishes "phase p resident" without a kernel, so
// the replay kernel can wait on it even while it occupies every SM.
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
  static const WriteValue32Fn fn = []() -> WriteValue32Fn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<WriteValue32Fn>(p);
  }();
  return fn;
}

// The device address of a page-locked, device-mapped host buffer (nullptr for
// pageable memory): the replay then writes the assignments straight into the
// caller's buffer while it runs -- one 32-byte store per warp per 32 requests
// -- instead of a device buffer copied back after the kernel.
uint8_t* mapped_host(uint8_t* host) {
  if (!host) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer ? static_cast<uint8_t*>(a.devicePointer) : nullptr;
}

int replay_host(hs_ctx* c, const hs_instance* inst, const hs_policy* pol, const hs_trace_batch* b,
                const hs_replay_seeds* seeds, uint8_t* assign, double* depart, hs_inst_metrics* metrics,
                hs_trace_result* result) {
  if (!c || !inst || !pol || !b || !metrics || !result || !b->offsets) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  const int64_t T = b->n_traces;
  if (T < 0) return fail(HS_ERR_ARG, "n_traces < 0");
  const int64_t* off = b->offsets;
  if (off[0] != 0) return fail(HS_ERR_ARG, "offsets[0] must be 0");
  const int64_t total = off[T];
  const bool gen_arr = seeds && seeds->arrival_state;
  const bool gen_pred = seeds && seeds->predictor_state;
  if (gen_arr && b->arrival) return fail(HS_ERR_ARG, "seeded arrivals need batch->arrival = NULL");
  if (gen_pred && seeds->pred_cap < 1) return fail(HS_ERR_ARG, "pred_cap must be >= 1");
  if (total > 0 && (!b->input_len || !b->output_len || (!gen_pred && !b->pred_output_len)))
    return fail(HS_ERR_ARG, "null trace");
  hs::ReplayConst base;
  if ((rc = make_const(inst, pol, b->arrival != nullptr || gen_arr, &base))) return rc;
  int64_t max_q;
  if ((rc = check_offsets(off, T, &max_q))) return rc;
  if ((rc = ensure_pipeline(c))) return rc;
  const int N = pol->n_instances;
  // predictions identical to the outputs (oracle predictor): copy once
  const bool p_is_o = !gen_pred && b->pred_output_len == b->output_len;
  hs_pcg64_state *dSA = nullptr, *dSP = nullptr;
  if (gen_arr && (rc = ensure_t(c, S_RNG_ST, (size_t)(T > 0 ? T : 1), &dSA))) return rc;
  if (gen_pred && (rc = ensure_t(c, S_RNG_ST2, (size_t)(T > 0 ? T : 1), &dSP))) return rc;
  if (gen_arr && T > 0)
    HS_CUDA(cudaMemcpyAsync(dSA, seeds->arrival_state, sizeof(hs_pcg64_state) * T, cudaMemcpyHostToDevice, c->stream));
  if (gen_pred && T > 0)
    HS_CUDA(cudaMemcpyAsync(dSP, seeds->predictor_state, sizeof(hs_pcg64_state) * T, cudaMemcpyHostToDevice,
                            c->stream));
  int64_t* dOff;
  int32_t *dI, *dO, *dP;
  double* dT = nullptr;
  uint8_t* dA = nullptr;
  double* dDep = nullptr;
  hs_inst_metrics* dM;
  hs_trace_result* dR;
  void* dQ;
  const size_t tq = (size_t)(total > 0 ? total : 1);
  if ((rc = ensure_t(c, S_OFF, (size_t)T + 1, &dOff)) || (rc = ensure_t(c, S_I, tq, &dI)) ||
      (rc = ensure_t(c, S_O, tq, &dO)) || (rc = ensure_t(c, S_METRICS, (size_t)(T > 0 ? T : 1) * N, &dM)) ||
      (rc = ensure_t(c, S_RESULT, (size_t)(T > 0 ? T : 1), &dR)) ||
      (rc = ensure(c, S_WREC, tq * hs::kQRecBytes, &dQ)))
    return rc;
  if (p_is_o) {
    dP = dO;
  } else if ((rc = ensure_t(c, S_P, tq, &dP))) {
    return rc;
  }
  if ((b->arrival || gen_arr) && (rc = ensure_t(c, S_T, tq, &dT))) return rc;
  uint8_t* const zA = mapped_host(assign);
  if (zA) {
    dA = zA;
  } else if (assign && (rc = ensure_t(c, S_ASSIGN, tq, &dA))) {
    return rc;
  }
  const size_t dep_w = (pol->flags & HS_REPLAY_ORDER_KEYS) ? 3 : 1;  // doubles per request in `depart`
  if (depart && (rc = ensure_t(c, S_DEPART, tq * dep_w, &dDep))) return rc;
  // requests that never retire (a failed trace) read back as NaN
  if (dDep) HS_CUDA(cudaMemsetAsync(dDep, 0xff, sizeof(double) * dep_w * tq, c->stream));
  HS_CUDA(cudaMemcpyAsync(dOff, off, sizeof(int64_t) * (T + 1), cudaMemcpyHostToDevice, c->stream));
  // Streamed replay (equal-length traces, the batched-replay shape): every
  // trace is launched once the first of kPhases phases of every trace is
  // resident; the copy stream then moves phase p of all traces with one 2-D
  // copy per array and publishes p + 1 to a progress word the kernel reads
  // before it consumes a request block of that phase.  The PCIe transfer
  // hides under the replay instead of delaying the last chunk.  Heaps are
  // sized from phase 0's min(I + O); a trace that outgrows that estimate
  // reports CAPACITY and the call is redone on the exactly-sized path below.
  const int64_t sq = T > 0 ? off[1] : 0;
  bool equal = T > 0 && sq >= 256 && sq % 32 == 0 && !std::getenv("HS_NO_STREAM");
  for (int64_t t = 1; equal && t <= T; ++t) equal = off[t] == t * sq;
  const WriteValue32Fn wv = equal ? write_value32() : nullptr;
  if (wv) {
    constexpr int64_t kPhases = 16;
    const int64_t L = ((sq + kPhases - 1) / kPhases + 31) / 32 * 32;
    const int64_t nphase = (sq + L - 1) / L;
    uint32_t* dProg;
    int32_t* d_min;
    if ((rc = ensure_t(c, S_PROGRESS, 1, &dProg)) || (rc = ensure_t(c, S_MINNEED, kPipe, &d_min))) return rc;
    auto copy_phase = [&](int64_t p) -> int {
      const int64_t a = p * L, w = (sq - a) < L ? (sq - a) : L;
      const size_t s4 = (size_t)sq * 4, s8 = (size_t)sq * 8;
      HS_CUDA(cudaMemcpy2DAsync(dI + a, s4, b->input_len + a, s4, (size_t)w * 4, (size_t)T, cudaMemcpyHostToDevice,
                                c->stream));
      HS_CUDA(cudaMemcpy2DAsync(dO + a, s4, b->output_len + a, s4, (size_t)w * 4, (size_t)T, cudaMemcpyHostToDevice,
                                c->stream));
      if (!p_is_o && !gen_pred)
        HS_CUDA(cudaMemcpy2DAsync(dP + a, s4, b->pred_output_len + a, s4, (size_t)w * 4, (size_t)T,
                                  cudaMemcpyHostToDevice, c->stream));
      if (dT && !gen_arr)
        HS_CUDA(cudaMemcpy2DAsync(dT + a, s8, b->arrival + a, s8, (size_t)w * 8, (size_t)T, cudaMemcpyHostToDevice,
                                  c->stream));
      if (wv((CUstream)c->stream, (CUdeviceptr)dProg, (cuuint32_t)(p + 1), 0) != CUDA_SUCCESS)
        return fail(HS_ERR_CUDA, "cuStreamWriteValue32 failed");
      return HS_OK;
    };
    cudaStream_t ks = c->ks[0];
    if ((rc = begin_timing(c))) return rc;
    HS_CUDA(cudaMemsetAsync(dProg, 0, sizeof(uint32_t), c->stream));
    HS_CUDA(cudaEventRecord(c->ev_min[1], c->stream));  // offsets + generator states are on the device
    HS_CUDA(cudaStreamWaitEvent(ks, c->ev_min[1], 0));
    if (gen_arr) {  // drawn while phase 0 is in flight
      hs::RngConst g{};
      g.n_dists = 1;
      g.dist[0] = hs_dist{HS_DIST_EXP_CUMSUM, 0, 0, 0, seeds->arrival_scale, 0.0};
      g.out[0] = dT;
      HS_CUDA(hs::launch_rng_generate(g, dSA, dOff, 0, T, nullptr, ks));
      c->launches += 1;
    }
    if (gen_pred) {
      hs::RngConst g{};
      g.n_dists = 1;
      g.dist[0] = hs_dist{HS_DIST_NORMAL_LEN, seeds->pred_cap, 0, 0, seeds->pred_mean, seeds->pred_stddev};
      g.out[0] = dP;
      HS_CUDA(hs::launch_rng_generate(g, dSP, dOff, 0, T, nullptr, ks));
      c->launches += 1;
    }
    if ((rc = copy_phase(0))) return rc;
    HS_CUDA(cudaMemsetAsync(d_min, 0x7f, sizeof(int32_t), c->stream));
    HS_CUDA(hs::launch_min_need_2d(dI, dO, T, L < sq ? L : sq, sq, d_min, c->stream));
    c->launches += 1;
    HS_CUDA(cudaMemcpyAsync(c->pinned_min, d_min, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaEventRecord(c->ev_copy[0], c->stream));
    HS_CUDA(cudaEventSynchronize(c->ev_copy[0]));
    hs::ReplayConst rs = base;
    size_heaps(rs, inst, c->pinned_min[0], sq);
    const size_t heap_bytes = (size_t)T * rs.heap_stride * hs::kHEntBytes;
    HS_CUDA(cudaStreamWaitEvent(ks, c->ev_copy[0], 0));
    void* heap = nullptr;
    // (cudaMemGetInfo costs milliseconds per call: try the allocation instead)
    const cudaError_t ae = cudaMallocAsync(&heap, heap_bytes, ks);
    if (ae == cudaErrorMemoryAllocation) {  // all heaps at once do not fit: the chunked path below
      (void)cudaGetLastError();
      HS_CUDA(cudaStreamSynchronize(ks));
      HS_CUDA(cudaStreamSynchronize(c->stream));
      goto chunked;
    }
    HS_CUDA(ae);
    HS_CUDA(hs::launch_replay(rs, T, dOff, dI, dO, dP, dT, dA, dDep, dM, dR, dQ, static_cast<uint64_t*>(heap), ks,
                              nullptr, nullptr, nullptr, 0, 0, dProg, (int)L));
    c->launches += 1;
    HS_CUDA(cudaFreeAsync(heap, ks));
    HS_CUDA(cudaEventRecord(c->ev_done[0], ks));
    for (int64_t p = 1; p < nphase; ++p)
      if ((rc = copy_phase(p))) return rc;
    HS_CUDA(cudaStreamWaitEvent(c->stream, c->ev_done[0], 0));
    if ((rc = end_timing(c))) return rc;
    HS_CUDA(cudaMemcpyAsync(metrics, dM, sizeof(hs_inst_metrics) * T * N, cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaMemcpyAsync(result, dR, sizeof(hs_trace_result) * T, cudaMemcpyDeviceToHost, c->stream));
    if (assign && !zA && total > 0) HS_CUDA(cudaMemcpyAsync(assign, dA, total, cudaMemcpyDeviceToHost, c->stream));
    if (depart && total > 0)
      HS_CUDA(cudaMemcpyAsync(depart, dDep, sizeof(double) * dep_w * total, cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaStreamSynchronize(c->stream));
    bool redo = false;
    for (int64_t t = 0; t < T; ++t) redo |= result[t].error == HS_TRACE_CAPACITY;
    if (!redo) return HS_OK;
    // phase-0 sizing was too small for some trace: exact sizing below (the
    // device already holds every input; the chunked path copies them again)
    // (the generator kernel advanced the device copies of the states: restore them)
    if (gen_arr)
      HS_CUDA(cudaMemcpyAsync(dSA, seeds->arrival_state, sizeof(hs_pcg64_state) * T, cudaMemcpyHostToDevice,
                              c->stream));
    if (gen_pred)
      HS_CUDA(cudaMemcpyAsync(dSP, seeds->predictor_state, sizeof(hs_pcg64_state) * T, cudaMemcpyHostToDevice,
                              c->stream));
  }
chunked:
  // Chunks of traces: copy chunk i on the copy stream while earlier chunks
  // replay on their own streams; each chunk sizes its heaps exactly from
  // its own min(I + O).
  const int64_t nch = T < kPipe ? (T > 0 ? T : 0) : kPipe;
  std::vector<hs::ReplayConst> rcs((size_t)(nch > 0 ? nch : 1), base);
  std::vector<void*> heaps((size_t)(nch > 0 ? nch : 1), nullptr);
  auto bounds = [&](int64_t i, int64_t* t0, int64_t* t1) {
    *t0 = T * i / nch;
    *t1 = T * (i + 1) / nch;
  };
  auto enqueue_copy = [&](int64_t i) -> int {
    int64_t t0, t1;
    bounds(i, &t0, &t1);
    const int64_t a = off[t0], n = off[t1] - off[t0];
    if (n > 0) {
      HS_CUDA(cudaMemcpyAsync(dI + a, b->input_len + a, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
      HS_CUDA(cudaMemcpyAsync(dO + a, b->output_len + a, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
      if (!p_is_o && !gen_pred)
        HS_CUDA(cudaMemcpyAsync(dP + a, b->pred_output_len + a, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                                c->stream));
      if (dT && !gen_arr) HS_CUDA(cudaMemcpyAsync(dT + a, b->arrival + a, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    }
    HS_CUDA(cudaEventRecord(c->ev_copy[i], c->stream));
    HS_CUDA(cudaStreamWaitEvent(c->aux, c->ev_copy[i], 0));
    int32_t* d_min;
    int r2;
    if ((r2 = ensure_t(c, S_MINNEED, kPipe, &d_min))) return r2;
    HS_CUDA(cudaMemsetAsync(d_min + i, 0x7f, sizeof(int32_t), c->aux));
    if (n > 0) {
      HS_CUDA(hs::launch_min_need(dI + a, dO + a, n, d_min + i, c->aux));
      c->launches += 1;
    }
    HS_CUDA(cudaMemcpyAsync(c->pinned_min + i, d_min + i, sizeof(int32_t), cudaMemcpyDeviceToHost, c->aux));
    HS_CUDA(cudaEventRecord(c->ev_min[i], c->aux));
    return HS_OK;
  };
  auto launch_chunk = [&](int64_t i) -> int {
    int64_t t0, t1;
    bounds(i, &t0, &t1);
    HS_CUDA(cudaEventSynchronize(c->ev_min[i]));
    int64_t mq = 0;
    for (int64_t t = t0; t < t1; ++t) mq = (off[t + 1] - off[t]) > mq ? (off[t + 1] - off[t]) : mq;
    hs::ReplayConst& rci = rcs[i];
    size_heaps(rci, inst, c->pinned_min[i], mq);
    cudaStream_t ks = c->ks[i % kPipe];
    HS_CUDA(cudaStreamWaitEvent(ks, c->ev_copy[i], 0));
    const size_t hb = (size_t)(t1 - t0 > 0 ? t1 - t0 : 1) * rci.heap_stride * hs::kHEntBytes;
    HS_CUDA(cudaMallocAsync(&heaps[i], hb, ks));
    if (gen_arr) {
      hs::RngConst g{};
      g.n_dists = 1;
      g.dist[0] = hs_dist{HS_DIST_EXP_CUMSUM, 0, 0, 0, seeds->arrival_scale, 0.0};
      g.out[0] = dT;
      HS_CUDA(hs::launch_rng_generate(g, dSA, dOff, t0, t1, nullptr, ks));
      c->launches += 1;
    }
    if (gen_pred) {
      hs::RngConst g{};
      g.n_dists = 1;
      g.dist[0] = hs_dist{HS_DIST_NORMAL_LEN, seeds->pred_cap, 0, 0, seeds->pred_mean, seeds->pred_stddev};
      g.out[0] = dP;
      HS_CUDA(hs::launch_rng_generate(g, dSP, dOff, t0, t1, nullptr, ks));
      c->launches += 1;
    }
    HS_CUDA(hs::launch_replay(rci, t1 - t0, dOff + t0, dI, dO, dP, dT, dA, dDep, dM + t0 * N, dR + t0, dQ,
                              static_cast<uint64_t*>(heaps[i]), ks));
    c->launches += 1;
    HS_CUDA(cudaFreeAsync(heaps[i], ks));
    HS_CUDA(cudaEventRecord(c->ev_done[i], ks));
    return HS_OK;
  };
  if ((rc = begin_timing(c))) return rc;
  if (nch > 0 && (rc = enqueue_copy(0))) return rc;
  for (int64_t i = 0; i < nch; ++i) {
    if (i + 1 < nch && (rc = enqueue_copy(i + 1))) return rc;
    if ((rc = launch_chunk(i))) return rc;
  }
  for (int64_t i = 0; i < nch; ++i) HS_CUDA(cudaStreamWaitEvent(c->stream, c->ev_done[i], 0));
  if ((rc = end_timing(c))) return rc;
  if (T > 0) {
    HS_CUDA(cudaMemcpyAsync(metrics, dM, sizeof(hs_inst_metrics) * T * N, cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaMemcpyAsync(result, dR, sizeof(hs_trace_result) * T, cudaMemcpyDeviceToHost, c->stream));
  }
  if (assign && !zA && total > 0) HS_CUDA(cudaMemcpyAsync(assign, dA, total, cudaMemcpyDeviceToHost, c->stream));
  if (depart && total > 0)
    HS_CUDA(cudaMemcpyAsync(depart, dDep, sizeof(double) * dep_w * total, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}

}  // namespace

int hs_replay(hs_ctx* c, const hs_instance* inst, const hs_policy* pol, const hs_trace_batch* b, uint8_t* assign,
              double* depart, hs_inst_metrics* metrics, hs_trace_result* result) {
  return replay_host(c, inst, pol, b, nullptr, assign, depart, metrics, result);
}

int hs_replay_seeded(hs_ctx* c, const hs_instance* inst, const hs_policy* pol, const hs_trace_batch* b,
                     const hs_replay_seeds* seeds, uint8_t* assign, double* depart, hs_inst_metrics* metrics,
                     hs_trace_result* result) {
  if (!seeds) return fail(HS_ERR_ARG, "null seeds");
  return replay_host(c, inst, pol, b, seeds, assign, depart, metrics, result);
}

// numpy bit_generator.pyx SeedSequence (pool of 4 words, hashmix/mix) and
// pcg64.c pcg64_set_seed / pcg_setseq_128_srandom_r.
int hs_pcg64_seed(const uint32_t* entropy, int32_t n_words, hs_pcg64_state* out) {
  if (!out || n_words < 1 || !entropy) return fail(HS_ERR_ARG, "need at least one entropy word");
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_words ? entropy[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < n_words; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s]));
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  const uint64_t s0 = w[0] | ((uint64_t)w[1] << 32), s1 = w[2] | ((uint64_t)w[3] << 32);
  const uint64_t i0 = w[4] | ((uint64_t)w[5] << 32), i1 = w[6] | ((uint64_t)w[7] << 32);
  typedef unsigned __int128 u128;
  const u128 mult = ((u128)2549297995355413924ull << 64) | 4865540595714422341ull;
  const u128 initstate = ((u128)s0 << 64) | s1, initseq = ((u128)i0 << 64) | i1;
  const u128 inc = (initseq << 1) | 1u;
  u128 st = 0;
  st = st * mult + inc;
  st += initstate;
  st = st * mult + inc;
  out->state_hi = (uint64_t)(st >> 64);
  out->state_lo = (uint64_t)st;
  out->inc_hi = (uint64_t)(inc >> 64);
  out->inc_lo = (uint64_t)inc;
  out->has_uint32 = 0;
  out->uinteger = 0;
  return HS_OK;
}

int hs_pcg64_seed_u64(const uint64_t* seeds, int64_t n, hs_pcg64_state* out) {
  if (n < 0 || (n > 0 && (!seeds || !out))) return fail(HS_ERR_ARG, "null argument");
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t w[2] = {(uint32_t)seeds[i], (uint32_t)(seeds[i] >> 32)};
    int rc = hs_pcg64_seed(w, w[1] ? 2 : 1, out + i);
    if (rc) return rc;
  }
  return HS_OK;
}

int hs_rng_generate(hs_ctx* c, hs_pcg64_state* states, int32_t n_streams, const int64_t* offsets,
                    const hs_dist* dists, int32_t n_dists, void* const* out, int64_t* bad_index) {
  if (!c || !states || !offsets || !dists || !out) return fail(HS_ERR_ARG, "null argument");
  if (n_streams < 0) return fail(HS_ERR_ARG, "n_streams < 0");
  if (n_dists < 1 || n_dists > hs::kMaxDists) return fail(HS_ERR_ARG, "n_dists must be 1..4");
  if (offsets[0] != 0) return fail(HS_ERR_ARG, "offsets[0] must be 0");
  int rc;
  for (int32_t t = 0; t < n_streams; ++t)
    if (offsets[t + 1] < offsets[t]) return fail(HS_ERR_ARG, "offsets must be non-decreasing");
  hs::RngConst g{};
  g.n_dists = n_dists;
  for (int32_t j = 0; j < n_dists; ++j) {
    if ((rc = check_dist(dists[j]))) return rc;
    if (offsets[n_streams] > 0 && !out[j]) return fail(HS_ERR_ARG, "null output buffer");
    g.dist[j] = dists[j];
    g.out[j] = out[j];
  }
  if (n_streams == 0) return HS_OK;
  if ((rc = use_device(c))) return rc;
  hs_pcg64_state* dS;
  int64_t *dOff, *dBad;
  if ((rc = ensure_t(c, S_RNG_ST, (size_t)n_streams, &dS)) || (rc = ensure_t(c, S_RNG_OFF, (size_t)n_streams + 1, &dOff)) ||
      (rc = ensure_t(c, S_RNG_BAD, (size_t)n_streams, &dBad)))
    return rc;
  HS_CUDA(cudaMemcpyAsync(dS, states, sizeof(hs_pcg64_state) * n_streams, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemcpyAsync(dOff, offsets, sizeof(int64_t) * (n_streams + 1), cudaMemcpyHostToDevice, c->stream));
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_rng_generate(g, dS, dOff, 0, n_streams, dBad, c->stream));
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  HS_CUDA(cudaMemcpyAsync(states, dS, sizeof(hs_pcg64_state) * n_streams, cudaMemcpyDeviceToHost, c->stream));
  if (bad_index)
    HS_CUDA(cudaMemcpyAsync(bad_index, dBad, sizeof(int64_t) * n_streams, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}

int hs_replay_deployments(hs_ctx* c, const hs_instance* instances, const int32_t* inst_offsets, int32_t n_dep,
                          const hs_policy* pol, const int32_t* trace_dep, const hs_trace_batch* b, uint8_t* assign,
                          double* depart, hs_inst_metrics* metrics, hs_trace_result* result) {
  if (!c || !instances || !inst_offsets || !pol || !trace_dep || !b || !metrics || !result || !b->offsets)
    return fail(HS_ERR_ARG, "null argument");
  if (n_dep < 1) return fail(HS_ERR_ARG, "n_deployments must be >= 1");
  int rc;
  if ((rc = use_device(c))) return rc;
  // HS_DEBUG_PHASES=1: host wall time of each phase on stderr (diagnostic)
  static const bool dbg = std::getenv("HS_DEBUG_PHASES") != nullptr;
  auto tp0 = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(c->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hs_replay_deployments] %-12s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - tp0).count());
    tp0 = t;
  };
  const int64_t T = b->n_traces;
  const int64_t* off = b->offsets;
  if (T < 0 || off[0] != 0) return fail(HS_ERR_ARG, "bad offsets");
  const int64_t total = off[T];
  int64_t max_q;
  if ((rc = check_offsets(off, T, &max_q))) return rc;
  std::vector<hs::ReplayConst> deps((size_t)n_dep);
  int n_max = 0, max_types = 0;
  for (int32_t d = 0; d < n_dep; ++d) {
    hs_policy pd = *pol;
    pd.n_instances = inst_offsets[d + 1] - inst_offsets[d];
    if ((rc = make_const(instances + inst_offsets[d], &pd, b->arrival != nullptr, &deps[d]))) return rc;
    if (pd.n_instances > n_max) n_max = pd.n_instances;
    if (deps[d].n_types > max_types) max_types = deps[d].n_types;
  }
  for (int64_t t = 0; t < T; ++t)
    if (trace_dep[t] < 0 || trace_dep[t] >= n_dep) return fail(HS_ERR_ARG, "trace_deployment out of range");
  int64_t* dOff;
  int32_t *dI, *dO, *dP, *dTD, *dMin;
  double* dT = nullptr;
  uint8_t* dA = nullptr;
  double* dDep = nullptr;
  hs_inst_metrics* dM;
  hs_trace_result* dR;
  void *dQ, *dDeps;
  int64_t* dTH;
  const size_t tq = (size_t)(total > 0 ? total : 1);
  if ((rc = ensure_t(c, S_OFF, (size_t)T + 1, &dOff)) || (rc = ensure_t(c, S_I, tq, &dI)) ||
      (rc = ensure_t(c, S_O, tq, &dO)) || (rc = ensure_t(c, S_P, tq, &dP)) ||
      (rc = ensure_t(c, S_METRICS, (size_t)(T > 0 ? T : 1) * n_max, &dM)) ||
      (rc = ensure_t(c, S_RESULT, (size_t)(T > 0 ? T : 1), &dR)) || (rc = ensure(c, S_WREC, tq * hs::kQRecBytes, &dQ)) ||
      (rc = ensure(c, S_DEPS, sizeof(hs::ReplayConst) * n_dep, &dDeps)) ||
      (rc = ensure_t(c, S_TDEP, (size_t)(T > 0 ? T : 1), &dTD)) ||
      (rc = ensure_t(c, S_THEAP, (size_t)(T > 0 ? T : 1), &dTH)) || (rc = ensure_t(c, S_MINNEED, 2, &dMin)))
    return rc;
  if (b->arrival && (rc = ensure_t(c, S_T, tq, &dT))) return rc;
  // a page-locked, device-mapped caller buffer takes the assignments directly
  uint8_t* const zA = mapped_host(assign);
  if (zA) {
    dA = zA;
  } else if (assign && (rc = ensure_t(c, S_ASSIGN, tq, &dA))) {
    return rc;
  }
  const size_t dep_w = (pol->flags & HS_REPLAY_ORDER_KEYS) ? 3 : 1;  // doubles per request in `depart`
  if (depart && (rc = ensure_t(c, S_DEPART, tq * dep_w, &dDep))) return rc;
  // requests that never retire (a failed trace) read back as NaN
  if (dDep) HS_CUDA(cudaMemsetAsync(dDep, 0xff, sizeof(double) * dep_w * tq, c->stream));
  HS_CUDA(cudaMemcpyAsync(dOff, off, sizeof(int64_t) * (T + 1), cudaMemcpyHostToDevice, c->stream));
  if (total > 0) {
    HS_CUDA(cudaMemcpyAsync(dI, b->input_len, sizeof(int32_t) * total, cudaMemcpyHostToDevice, c->stream));
    HS_CUDA(cudaMemcpyAsync(dO, b->output_len, sizeof(int32_t) * total, cudaMemcpyHostToDevice, c->stream));
    // predictions identical to the outputs (oracle predictor): copy once
    if (b->pred_output_len == b->output_len)
      dP = dO;
    else
      HS_CUDA(cudaMemcpyAsync(dP, b->pred_output_len, sizeof(int32_t) * total, cudaMemcpyHostToDevice, c->stream));
    if (dT) HS_CUDA(cudaMemcpyAsync(dT, b->arrival, sizeof(double) * total, cudaMemcpyHostToDevice, c->stream));
  }
  phase("setup+copies");
  HS_CUDA(cudaMemsetAsync(dMin, 0x7f, sizeof(int32_t), c->stream));
  HS_CUDA(cudaMemsetAsync(dMin + 1, 0, sizeof(int32_t), c->stream));
  if (total > 0) {
    HS_CUDA(hs::launch_min_need(dI, dO, total, dMin, c->stream, dMin + 1));
    c->launches += 1;
  }
  int32_t need_stats[2] = {0, 0};  // min(I + O), max(O)
  HS_CUDA(cudaMemcpyAsync(need_stats, dMin, sizeof(need_stats), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  const int32_t min_need = need_stats[0];
  const int cal_bits = cal_bits_for(n_max, need_stats[1]);
  for (int32_t d = 0; d < n_dep; ++d)
    size_heaps(deps[d], instances + inst_offsets[d], min_need, max_q, n_max, cal_bits);
  std::vector<int64_t> theap((size_t)(T > 0 ? T : 1));
  int64_t hacc = 0;
  for (int64_t t = 0; t < T; ++t) {
    theap[t] = hacc;
    hacc += deps[trace_dep[t]].heap_stride;
  }
  phase("need+size");
  uint64_t* dHeap;
  if ((rc = ensure_t(c, S_HEAP, (size_t)(hacc > 0 ? hacc : 1) * 2, &dHeap))) return rc;
  HS_CUDA(cudaMemcpyAsync(dDeps, deps.data(), sizeof(hs::ReplayConst) * n_dep, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemcpyAsync(dTD, trace_dep, sizeof(int32_t) * T, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaMemcpyAsync(dTH, theap.data(), sizeof(int64_t) * T, cudaMemcpyHostToDevice, c->stream));
  if ((rc = begin_timing(c))) return rc;
  HS_CUDA(hs::launch_replay(deps[0], T, dOff, dI, dO, dP, dT, dA, dDep, dM, dR, dQ, dHeap, c->stream,
                            static_cast<const hs::ReplayConst*>(dDeps), dTD, dTH, n_max, max_types));
  c->launches += 1;
  if ((rc = end_timing(c))) return rc;
  phase("kernel");
  if (T > 0) {
    HS_CUDA(cudaMemcpyAsync(metrics, dM, sizeof(hs_inst_metrics) * T * n_max, cudaMemcpyDeviceToHost, c->stream));
    HS_CUDA(cudaMemcpyAsync(result, dR, sizeof(hs_trace_result) * T, cudaMemcpyDeviceToHost, c->stream));
  }
  if (assign && !zA && total > 0) HS_CUDA(cudaMemcpyAsync(assign, dA, total, cudaMemcpyDeviceToHost, c->stream));
  if (depart && total > 0)
    HS_CUDA(cudaMemcpyAsync(depart, dDep, sizeof(double) * dep_w * total, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  phase("results");
  return HS_OK;
}

int hs_replay_device(hs_ctx* c, const hs_instance* inst, const hs_policy* pol, const hs_trace_batch* b,
                     uint8_t* assign, double* depart, hs_inst_metrics* metrics, hs_trace_result* result) {
  if (!c || !inst || !pol || !b || !metrics || !result || !b->offsets) return fail(HS_ERR_ARG, "null argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  const int64_t T = b->n_traces;
  if (T < 0) return fail(HS_ERR_ARG, "n_traces < 0");
  std::vector<int64_t> off((size_t)T + 1);
  HS_CUDA(cudaMemcpyAsync(off.data(), b->offsets, sizeof(int64_t) * (T + 1), cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return replay_impl(c, inst, pol, T, b->offsets, off.data(), b->input_len, b->output_len, b->pred_output_len,
                     b->arrival, assign, depart, metrics, result);
}

int hs_device_alloc(hs_ctx* c, int64_t bytes, void** out) {
  if (!c || !out || bytes < 0) return fail(HS_ERR_ARG, "bad argument");
  int rc;
  if ((rc = use_device(c))) return rc;
  HS_CUDA(cudaMalloc(out, (size_t)(bytes > 0 ? bytes : 16)));
  return HS_OK;
}
int hs_device_free(hs_ctx* c, void* p) {
  if (!c) return fail(HS_ERR_ARG, "null ctx");
  use_device(c);
  if (p) HS_CUDA(cudaFree(p));
  return HS_OK;
}
int hs_memcpy_h2d(hs_ctx* c, void* dst, const void* src, int64_t bytes) {
  if (!c) return fail(HS_ERR_ARG, "null ctx");
  use_device(c);
  HS_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}
int hs_memcpy_d2h(hs_ctx* c, void* dst, const void* src, int64_t bytes) {
  if (!c) return fail(HS_ERR_ARG, "null ctx");
  use_device(c);
  HS_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, c->stream));
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}
int hs_device_synchronize(hs_ctx* c) {
  if (!c) return fail(HS_ERR_ARG, "null ctx");
  use_device(c);
  HS_CUDA(cudaStreamSynchronize(c->stream));
  return HS_OK;
}
int hs_host_alloc(hs_ctx* c, int64_t bytes, void** out) {
  if (!c || !out || bytes < 0) return fail(HS_ERR_ARG, "bad argument");
  use_device(c);
  HS_CUDA(cudaHostAlloc(out, (size_t)(bytes > 0 ? bytes : 16), cudaHostAllocPortable));
  return HS_OK;
}
int hs_host_free(hs_ctx* c, void* p) {
  if (!c) return fail(HS_ERR_ARG, "null ctx");
  if (p) HS_CUDA(cudaFreeHost(p));
  return HS_OK;
}

}  // extern "C"
