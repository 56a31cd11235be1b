// rng.cu -- numpy Generator(PCG64) streams on the device, bit-identical to
// the host draws the reference makes (cli.py:160-193 gen-trace lengths,
// simulator.py:112-124 arrivals, scheduling.py:87-95 predictor).
//
// One warp per stream.  PCG64 is an LCG, so lane l jumps straight to the
// (l+1)-th state after the warp's base state (s_{n} = A_n s + inc G_n with
// A_n = a^n, G_n = 1 + a + ... + a^(n-1), per-lane constants computed once):
// a warp sees 32 consecutive raw draws per round.  The ziggurat's fast path
// (one draw -> one value, ~99% of draws) is decided per lane; the first
// lane that misses it runs numpy's slow path (wedge / tail, further draws
// taken serially), after which the remaining lanes' draws are still the
// right ones when the slow path consumed few enough.  Values therefore leave
// in exactly numpy's order and the final state equals numpy's.  The
// exponential running sum (np.cumsum: out[i] = out[i-1] + g[i]) is a serial
// fp64 chain kept in lane 0 over a per-warp shared staging row.
#include "hs_device.cuh"
#include "hs_internal.h"
#include "../../include/hs_ziggurat_tables.h"

namespace hs {
namespace {

constexpr double kNorR = 3.6541528853610087963519472518;
constexpr double kNorInvR = 0.27366123732975827203338247596;
constexpr double kExpR = 7.6971174701310497140446280481;
constexpr int kWarps = 4;

struct U128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
  return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}
__device__ __forceinline__ U128 shfl128(U128 v, int src) {
  return {__shfl_sync(0xffffffffu, v.hi, src), __shfl_sync(0xffffffffu, v.lo, src)};
}
// pcg64.h pcg_output_xsl_rr_128_64
__device__ __forceinline__ uint64_t pcg_out(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ U128 pcg_mult() { return {2549297995355413924ull, 4865540595714422341ull}; }

struct Tabs {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
  uint64_t ke[256];
  double we[256];
  double fe[256];
};

// Warp generator: S is the warp-uniform base state; lane l's draw in a round
// is the output of A*S + C (the (l+1)-th step).
struct Gen {
  U128 S, inc, A, C;
  uint32_t has32, u32;
  int taken;  // draws consumed by the current slow path
  __device__ __forceinline__ U128 lane_state() const { return add128(mul128(A, S), C); }
  __device__ __forceinline__ uint64_t next64(U128& s) {
    s = add128(mul128(pcg_mult(), s), inc);
    ++taken;
    return pcg_out(s);
  }
  __device__ __forceinline__ double next_double(U128& s) {
    return __dmul_rn(__ull2double_rn(next64(s) >> 11), 1.0 / 9007199254740992.0);
  }
};

// distributions.c random_standard_normal: fast-path decode of one draw
__device__ __forceinline__ double zig_normal(uint64_t r, const Tabs& T, bool* fast, int* idx, uint64_t* rabs) {
  *idx = (int)(r & 0xff);
  r >>= 8;
  const bool neg = r & 1;
  *rabs = (r >> 1) & 0x000fffffffffffffull;
  double x = __dmul_rn(__ull2double_rn(*rabs), T.wi[*idx]);
  if (neg) x = -x;
  *fast = *rabs < T.ki[*idx];
  return x;
}
// distributions.c random_standard_exponential: fast-path decode
__device__ __forceinline__ double zig_exp(uint64_t r, const Tabs& T, bool* fast, int* idx) {
  uint64_t ri = r >> 3;
  *idx = (int)(ri & 0xff);
  ri >>= 8;
  *fast = ri < T.ke[*idx];
  return __dmul_rn(__ull2double_rn(ri), T.we[*idx]);
}

// Slow paths, executed warp-uniformly: r is the draw that missed the fast
// path (made from state s); further draws advance s.
__device__ __noinline__ double normal_slow(uint64_t r, U128& s, Gen& g, const Tabs& T) {
  bool of;
  for (;;) {
    bool fast;
    int idx;
    uint64_t rabs;
    const double x = zig_normal(r, T, &fast, &idx, &rabs);
    if (fast) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-kNorInvR, py_log1p(-g.next_double(s)));
        const double yy = -py_log1p(-g.next_double(s));
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1) ? -__dadd_rn(kNorR, xx) : __dadd_rn(kNorR, xx);
      }
    }
    const double u = g.next_double(s);
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(T.fi[idx - 1], T.fi[idx]), u), T.fi[idx]);
    if (lhs < py_exp(__dmul_rn(__dmul_rn(-0.5, x), x), kExpTab, &of)) return x;
    r = g.next64(s);
  }
}

__device__ __noinline__ double exp_slow(uint64_t r, U128& s, Gen& g, const Tabs& T) {
  bool of;
  for (;;) {
    bool fast;
    int idx;
    const double x = zig_exp(r, T, &fast, &idx);
    if (fast) return x;
    if (idx == 0) return __dsub_rn(kExpR, py_log1p(-g.next_double(s)));
    const double u = g.next_double(s);
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(T.fe[idx - 1], T.fe[idx]), u), T.fe[idx]);
    if (lhs < py_exp(-x, kExpTab, &of)) return x;
    r = g.next64(s);
  }
}

// int(min(max(round(v), 1), cap)); -1 when round() raises (v not finite).
__device__ __forceinline__ int32_t clamp_len(double v, int32_t cap) {
  if (!isfinite(v)) return -1;
  const double r = rint(v);
  if (r < 1.0) return 1;
  if (r > (double)cap) return cap;
  return (int32_t)r;
}

enum { Z_LOGNORMAL = 0, Z_NORMAL = 1, Z_EXPSUM = 2 };

// value of a standard draw z under the segment's transform
template <int K>
__device__ __forceinline__ int32_t to_len(double z, const hs_dist& d) {
  bool of;
  double v = __dadd_rn(d.p0, __dmul_rn(d.p1, z));  // random_normal: loc + scale * z
  if (K == Z_LOGNORMAL) v = py_exp(v, kExpTab, &of);  // random_lognormal: exp(normal)
  return clamp_len(v, d.cap);
}

template <int K>
__device__ void zig_segment(Gen& g, const hs_dist& d, int64_t n, void* out, const Tabs& T, double* row,
                            int64_t* bad, int lane) {
  int32_t* oi = static_cast<int32_t*>(out);
  double* od = static_cast<double*>(out);
  int64_t done = 0;
  double acc = 0.0;  // EXPSUM running sum (warp-uniform)
  while (done < n) {
    const U128 sl = g.lane_state();
    const uint64_t r = pcg_out(sl);
    bool fast;
    int idx;
    uint64_t rabs;
    const double x = (K == Z_EXPSUM) ? zig_exp(r, T, &fast, &idx) : zig_normal(r, T, &fast, &idx, &rabs);
    const uint32_t fm = __ballot_sync(0xffffffffu, fast);
    int j = 0;
    for (;;) {
      const uint32_t nf = ~fm & (0xffffffffu << j);
      const int k = nf ? __ffs(nf) - 1 : 32;
      const int e = (int)((int64_t)(k - j) < n - done ? (int64_t)(k - j) : n - done);
      const bool mine = lane >= j && lane < j + e;
      if (K == Z_EXPSUM) {
        if (mine) row[lane - j] = __dmul_rn(d.p0, x);  // random_exponential: scale * e
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < e) {
              acc = __dadd_rn(acc, row[i]);
              row[i] = acc;
            }
        }
        __syncwarp();
        if (mine) od[done + lane - j] = row[lane - j];
        acc = __shfl_sync(0xffffffffu, acc, 0);
        __syncwarp();
      } else if (mine) {
        const int32_t L = to_len<K>(x, d);
        oi[done + lane - j] = L < 0 ? 0 : L;
        if (L < 0 && *bad < 0) *bad = done + lane - j;
      }
      done += e;
      if (done == n) {  // e >= 1 here: the last value came from lane j + e - 1
        g.S = shfl128(sl, j + e - 1);
        return;
      }
      if (k == 32) {
        g.S = shfl128(sl, 31);
        break;
      }
      // lane k missed the fast path: numpy's slow path, warp-uniform
      U128 ss = shfl128(sl, k);
      const uint64_t rk = __shfl_sync(0xffffffffu, r, k);
      g.taken = 0;
      const double v = (K == Z_EXPSUM) ? exp_slow(rk, ss, g, T) : normal_slow(rk, ss, g, T);
      if (K == Z_EXPSUM) {
        acc = __dadd_rn(acc, __dmul_rn(d.p0, v));
        if (lane == 0) od[done] = acc;
      } else if (lane == 0) {
        const int32_t L = to_len<K>(v, d);
        oi[done] = L < 0 ? 0 : L;
        if (L < 0 && *bad < 0) *bad = done;
      }
      done += 1;
      if (done == n) {
        g.S = ss;
        return;
      }
      const int jn = k + 1 + g.taken;  // lanes >= jn still hold the next draws
      if (jn < 32) {
        j = jn;
        continue;
      }
      g.S = ss;
      break;
    }
  }
}

// random_bounded_uint64_fill (Lemire; the 32-bit path draws next_uint32,
// which splits one 64-bit draw low half first and buffers the high half).
// Rejected words are simply skipped, so a round is a stream compaction.
__device__ void uniform_segment(Gen& g, const hs_dist& d, int64_t n, int32_t* oi, int lane) {
  const uint64_t rng = (uint64_t)d.hi - (uint64_t)d.lo;
  const uint32_t lt = (1u << lane) - 1u;
  auto put = [&](int64_t i, uint64_t val) {
    const int64_t v = (int64_t)((uint64_t)d.lo + val);
    oi[i] = v < 1 ? 1 : (v > d.cap ? d.cap : (int32_t)v);
  };
  int64_t done = 0;
  if (rng == 0) {
    for (int64_t i = lane; i < n; i += 32) put(i, 0);
    return;
  }
  if (rng <= 0xffffffffull) {
    const bool full = rng == 0xffffffffull;
    const uint32_t rx = (uint32_t)rng + 1u;
    const uint32_t th = full ? 0u : (0xffffffffu - (uint32_t)rng) % rx;
    if (done < n && g.has32) {
      g.has32 = 0;
      const uint64_t m = full ? ((uint64_t)g.u32 << 32) : (uint64_t)g.u32 * rx;
      if (full || (uint32_t)m >= th) {
        if (lane == 0) put(done, m >> 32);
        ++done;
      }
    }
    while (done < n) {
      const U128 sl = g.lane_state();
      const uint64_t r = pcg_out(sl);
      const uint32_t c0 = (uint32_t)r, c1 = (uint32_t)(r >> 32);
      const uint64_t m0 = full ? ((uint64_t)c0 << 32) : (uint64_t)c0 * rx;
      const uint64_t m1 = full ? ((uint64_t)c1 << 32) : (uint64_t)c1 * rx;
      const bool a0 = full || (uint32_t)m0 >= th, a1 = full || (uint32_t)m1 >= th;
      const uint32_t b0 = __ballot_sync(0xffffffffu, a0), b1 = __ballot_sync(0xffffffffu, a1);
      const int pre = __popc(b0 & lt) + __popc(b1 & lt);
      const int total = __popc(b0) + __popc(b1);
      const int64_t rem = n - done;
      const int i0 = pre, i1 = pre + (a0 ? 1 : 0);
      if (a0 && i0 < rem) put(done + i0, m0 >> 32);
      if (a1 && i1 < rem) put(done + i1, m1 >> 32);
      // pcg64_next32 leaves uinteger = high half of the last split draw,
      // whether or not that half has been handed out since
      if (total < rem) {
        done += total;
        g.S = shfl128(sl, 31);
        g.u32 = __shfl_sync(0xffffffffu, c1, 31);
        continue;
      }
      // the value with index rem-1 is the last word consumed
      const bool l0 = a0 && i0 == rem - 1, l1 = a1 && i1 == rem - 1;
      const int L = __ffs(__ballot_sync(0xffffffffu, l0 || l1)) - 1;
      const bool high = __shfl_sync(0xffffffffu, l1 ? 1 : 0, L);
      g.S = shfl128(sl, L);
      g.u32 = __shfl_sync(0xffffffffu, c1, L);
      g.has32 = high ? 0u : 1u;
      done = n;
    }
    return;
  }
  const bool full = rng == ~0ull;
  const uint64_t rx = rng + 1;
  const uint64_t th = full ? 0ull : (~0ull - rng) % rx;
  while (done < n) {
    const U128 sl = g.lane_state();
    const uint64_t r = pcg_out(sl);
    const bool a = full || r * rx >= th;
    const uint64_t val = full ? r : __umul64hi(r, rx);
    const uint32_t b = __ballot_sync(0xffffffffu, a);
    const int pre = __popc(b & lt), total = __popc(b);
    const int64_t rem = n - done;
    if (a && pre < rem) put(done + pre, val);
    if (total < rem) {
      done += total;
      g.S = shfl128(sl, 31);
      continue;
    }
    const int L = __ffs(__ballot_sync(0xffffffffu, a && pre == rem - 1)) - 1;
    g.S = shfl128(sl, L);
    done = n;
  }
}

__device__ __forceinline__ int64_t warp_min64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

__global__ void __launch_bounds__(kWarps * 32, 8) k_rng_generate(const __grid_constant__ RngConst rc,
                                                               hs_pcg64_state* states, const int64_t* off,
                                                               int64_t s_begin, int64_t s_end, int64_t* bad_out) {
  __shared__ Tabs T;
  __shared__ double rows[kWarps][32];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    T.ki[i] = kZig_ki[i];
    T.wi[i] = kZig_wi[i];
    T.fi[i] = kZig_fi[i];
    T.ke[i] = kZig_ke[i];
    T.we[i] = kZig_we[i];
    T.fe[i] = kZig_fe[i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = s_begin + (int64_t)blockIdx.x * kWarps + warp;
  if (t >= s_end) return;
  const hs_pcg64_state st = states[t];
  Gen g;
  g.S = {st.state_hi, st.state_lo};
  g.inc = {st.inc_hi, st.inc_lo};
  g.has32 = st.has_uint32;
  g.u32 = st.uinteger;
  g.taken = 0;
  U128 A = {0, 1}, G = {0, 0};
  for (int i = 0; i < 32; ++i)
    if (i <= lane) {
      G = add128(mul128(pcg_mult(), G), U128{0, 1});
      A = mul128(pcg_mult(), A);
    }
  g.A = A;
  g.C = mul128(g.inc, G);
  const int64_t a = off[t], n = off[t + 1] - a;
  int64_t bad = -1;
  for (int j = 0; j < rc.n_dists; ++j) {
    const hs_dist& d = rc.dist[j];
    int64_t sb = -1;
    switch (d.kind) {
      case HS_DIST_LOGNORMAL_LEN:
        zig_segment<Z_LOGNORMAL>(g, d, n, static_cast<int32_t*>(rc.out[j]) + a, T, rows[warp], &sb, lane);
        break;
      case HS_DIST_NORMAL_LEN:
        zig_segment<Z_NORMAL>(g, d, n, static_cast<int32_t*>(rc.out[j]) + a, T, rows[warp], &sb, lane);
        break;
      case HS_DIST_EXP_CUMSUM:
        zig_segment<Z_EXPSUM>(g, d, n, static_cast<double*>(rc.out[j]) + a, T, rows[warp], &sb, lane);
        break;
      default:
        uniform_segment(g, d, n, static_cast<int32_t*>(rc.out[j]) + a, lane);
        break;
    }
    sb = warp_min64(sb < 0 ? INT64_MAX : sb);
    if (bad < 0 && sb != INT64_MAX) bad = sb;
  }
  if (lane == 0) {
    hs_pcg64_state o;
    o.state_hi = g.S.hi;
    o.state_lo = g.S.lo;
    o.inc_hi = st.inc_hi;
    o.inc_lo = st.inc_lo;
    o.has_uint32 = g.has32;
    o.uinteger = g.u32;
    states[t] = o;
    if (bad_out) bad_out[t] = bad;
  }
}

}  // namespace

cudaError_t launch_rng_generate(const RngConst& rc, hs_pcg64_state* d_states, const int64_t* d_off,
                                int64_t s_begin, int64_t s_end, int64_t* d_bad, cudaStream_t st) {
  if (s_end <= s_begin) return cudaSuccess;
  const int64_t blocks = (s_end - s_begin + kWarps - 1) / kWarps;
  k_rng_generate<<<(unsigned)blocks, kWarps * 32, 0, st>>>(rc, d_states, d_off, s_begin, s_end, d_bad);
  return cudaGetLastError();
}

}  // namespace hs
