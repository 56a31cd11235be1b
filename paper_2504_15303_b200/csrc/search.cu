// search.cu -- deployment-configuration search on the GPU.
//
// K1 k_table_build: one warp per (machine, tp degree).  Replaces the
//   per-machine body of planner.py:152-179 (estimate_system_throughput),
//   i.e. capacity.py:72-95 budget + feasibility and planner.py:51-118: the
//   greedy static-batch scan over the trace, batch pricing, CPython's
//   compensated sum of batch times and tokens / total_time.  The greedy scan
//   is sequential in batch boundaries; within a batch the warp tests 32
//   candidate extensions at once (warp prefix sum of inputs, prefix max of
//   outputs, one ballot), so a batch of width w costs ceil((w+1)/32) steps.
//
// K2 k_search_best: exhaustive argmax over the mixed-radix candidate space
//   of planner.py:213-228 (itertools.product, machine 0 most significant;
//   best = max total, ties -> lowest index, as ranked.sort's key).  Every
//   candidate's total is evaluated in the reference's left-to-right order
//   (planner.py:151,180): the shared prefix over the outer machines is kept
//   incrementally (odometer), and each candidate costs one DADD (prefix +
//   last contribution) and one DSETP.GT.OR against the thread's best.
//   Non-OK table entries hold -inf, so infeasible candidates evaluate to
//   -inf (or NaN) and can never satisfy `> best`.
//
// k_search_score: per-candidate total + first failing machine, for the full
//   ranking of small spaces (sorted afterwards with CUB).
#include <cmath>


#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {

// ----------------------------------------------------------------- K1
// planner.py:51-87 plan_static_batches for one instance, warp-cooperative:
// each round tests 32 extensions of the current batch at once (warp prefix
// sum of inputs, prefix max of outputs / inputs, one ballot for the first
// extension that no longer fits).  on_batch(stop, width, max_I, max_O) is
// called, warp-uniformly, for every batch in order.  Returns the index of a
// request that does not fit alone (planner.py:78-84), or -1.
template <class F>
__device__ __forceinline__ int64_t scan_batches(const int32_t* __restrict__ I, const int32_t* __restrict__ O,
                                                int64_t q, int64_t cap, int lane, F&& on_batch) {
  int64_t start = 0;
  while (start < q) {
    int64_t sumI = 0, maxO = 0, maxI = 0;  // carries of the batch so far
    int64_t pos = start, stop = start, bMO = 0, bMI = 0;
    for (;;) {
      const int64_t idx = pos + lane;
      const bool valid = idx < q;
      int64_t s = valid ? (int64_t)I[idx] : 0;
      int64_t mo = valid ? (int64_t)O[idx] : 0;
      int64_t mi = s;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int64_t ts = __shfl_up_sync(0xffffffffu, s, off);
        int64_t to = __shfl_up_sync(0xffffffffu, mo, off);
        int64_t ti = __shfl_up_sync(0xffffffffu, mi, off);
        if (lane >= off) {
          s += ts;
          mo = mo > to ? mo : to;
          mi = mi > ti ? mi : ti;
        }
      }
      const int64_t candI = sumI + s;
      const int64_t candMO = maxO > mo ? maxO : mo;
      const int64_t candMI = maxI > mi ? maxI : mi;
      const int64_t width = idx - start + 1;
      const int64_t tokens = sat_add(candI, sat_mul(width, candMO));
      const bool fail = !valid || tokens > cap;
      const unsigned bal = __ballot_sync(0xffffffffu, fail);
      if (bal) {
        const int f = __ffs(bal) - 1;
        stop = pos + f;
        const int src = f > 0 ? f - 1 : 0;
        const int64_t sMO = __shfl_sync(0xffffffffu, candMO, src);
        const int64_t sMI = __shfl_sync(0xffffffffu, candMI, src);
        bMO = f > 0 ? sMO : maxO;
        bMI = f > 0 ? sMI : maxI;
        break;
      }
      sumI = __shfl_sync(0xffffffffu, candI, 31);
      maxO = __shfl_sync(0xffffffffu, candMO, 31);
      maxI = __shfl_sync(0xffffffffu, candMI, 31);
      pos += 32;
    }
    if (stop == start) return start;
    on_batch(stop, stop - start, bMI, bMO);
    start = stop;
  }
  return -1;
}

__global__ void __launch_bounds__(128) k_table_build(const EntryDesc* __restrict__ desc, int n, SearchConst sc,
                                                     const int32_t* __restrict__ I, const int32_t* __restrict__ O,
                                                     hs_entry* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= n) return;
  const EntryDesc d = desc[e];
  hs_entry r;
  r.contribution = 0.0;
  r.rate = 0.0;
  r.budget = 0.0;
  r.slack = 0.0;
  r.tp_degree = d.tp;
  r.instance_count = d.tp > 0 ? d.own_count / d.tp : 0;
  r.bad_request = -1;
  r.token_count = 0;
  r.zero_div_int = 0;
  r._pad = 0;
  r.status = HS_ENTRY_OK;
  const int64_t q = sc.q;
  // token_count = sum(I + O) (planner.py:117)
  int64_t tok = 0;
  for (int64_t k = lane; k < q; k += 32) tok += (int64_t)I[k] + O[k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tok += __shfl_xor_sync(0xffffffffu, tok, off);
  r.token_count = tok;

  if (d.tp < 1 || d.spec_count % d.tp != 0) {
    r.status = HS_ENTRY_BAD_DEGREE;
  } else {
    // capacity.py:84-86: ((t*mem) * phi - delta) - weights
    double usable = __dmul_rn(i2d(d.tp * d.spec_mem), sc.phi);
    double budget = __dsub_rn(__dsub_rn(usable, i2d(sc.static_overhead)), i2d(sc.weights));
    double slack = __dsub_rn(budget, i2d(sc.required));
    r.budget = budget;
    r.slack = slack;
    if (!(slack >= 0.0)) {
      r.status = HS_ENTRY_INFEASIBLE_CONFIG;
    } else if (!d.present) {
      r.status = HS_ENTRY_MISSING_PARAMS;
    } else {
      PySum tot;
      tot.init();
      // planner.py:69-74 per_token*sum(I) + width*per_token*max(O) > budget,
      // exactly: the integer pt*X exceeds B iff X > floor(floor(B) / pt)
      const int64_t cap = budget >= 9.2e18 ? INT64_MAX : (int64_t)floor(budget) / sc.per_token;
      const int64_t bad = scan_batches(I, O, q, cap, lane, [&](int64_t, int64_t b, int64_t bMI, int64_t bMO) {
        // planner.py:90-101 estimate_batch_time
        tot.add(__dadd_rn(prefill_time(d.p, b, bMI), decode_time(d.p, b, bMI, bMO)));
      });
      if (bad >= 0) {  // planner.py:78-84
        r.status = HS_ENTRY_INFEASIBLE_REQUEST;
        r.bad_request = bad;
      }
      if (r.status == HS_ENTRY_OK) {
        const double total = tot.result();  // planner.py:46-48 sum(per_batch_time)
        if (tot.n == 0 || total == 0.0) {
          r.status = HS_ENTRY_ZERO_DIVISION;
          r.zero_div_int = tot.n == 0;
        } else {
          r.rate = __ddiv_rn(i2d(tok), total);                        // planner.py:118
          r.contribution = __dmul_rn(r.rate, i2d(r.instance_count));  // planner.py:168
        }
      }
    }
  }
  if (lane == 0) out[e] = r;
}

// planner.py:51-118 for one instance with an explicit KV budget (one warp):
// plan_static_batches (batch stops), time_batches (per-batch seconds, when
// params are given) and estimate_instance_throughput (token_count / total).
__global__ void k_plan_instance(double budget, int64_t per_token, PlanParams pp, const int32_t* __restrict__ I,
                                const int32_t* __restrict__ O, int64_t q, int64_t* __restrict__ stops,
                                double* __restrict__ times, int64_t* __restrict__ n_batches, hs_entry* out) {
  const int lane = threadIdx.x & 31;
  hs_entry r{};
  r.bad_request = -1;
  r.status = HS_ENTRY_OK;
  r.budget = budget;
  r.instance_count = 1;
  int64_t tok = 0;
  for (int64_t k = lane; k < q; k += 32) tok += (int64_t)I[k] + O[k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) tok += __shfl_xor_sync(0xffffffffu, tok, off);
  r.token_count = tok;
  const int64_t cap = budget >= 9.2e18 ? INT64_MAX : (int64_t)floor(budget) / per_token;
  PySum tot;
  tot.init();
  int64_t nb = 0;
  const int64_t bad = scan_batches(I, O, q, cap, lane, [&](int64_t stop, int64_t b, int64_t bMI, int64_t bMO) {
    if (pp.has) {
      const double t = __dadd_rn(prefill_time(pp.p, b, bMI), decode_time(pp.p, b, bMI, bMO));
      tot.add(t);
      if (lane == 0) times[nb] = t;
    }
    if (lane == 0) stops[nb] = stop;
    ++nb;
  });
  if (bad >= 0) {
    r.status = HS_ENTRY_INFEASIBLE_REQUEST;
    r.bad_request = bad;
  } else if (pp.has) {
    const double total = tot.result();
    if (tot.n == 0 || total == 0.0) {
      r.status = HS_ENTRY_ZERO_DIVISION;
      r.zero_div_int = tot.n == 0;
    } else {
      r.rate = __ddiv_rn(i2d(tok), total);
      r.contribution = r.rate;
    }
  }
  if (lane == 0) {
    *out = r;
    *n_batches = nb;
  }
}

cudaError_t launch_plan_instance(double budget, int64_t per_token, const PlanParams& pp, const int32_t* d_I,
                                 const int32_t* d_O, int64_t q, int64_t* d_stops, double* d_times, int64_t* d_nb,
                                 hs_entry* d_out, cudaStream_t st) {
  k_plan_instance<<<1, 32, 0, st>>>(budget, per_token, pp, d_I, d_O, q, d_stops, d_times, d_nb, d_out);
  return cudaGetLastError();
}

cudaError_t launch_table_build(const EntryDesc* d_desc, int n, const SearchConst& sc, const int32_t* d_I,
                               const int32_t* d_O, hs_entry* d_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int warps_per_block = 4;
  int blocks = (n + warps_per_block - 1) / warps_per_block;
  k_table_build<<<blocks, warps_per_block * 32, 0, st>>>(d_desc, n, sc, d_I, d_O, d_out);
  return cudaGetLastError();
}

// ----------------------------------------------------------------- K2
__constant__ SpaceDesc c_space;

// Levels of the product space (SpaceDesc is padded to M >= 4):
//   outer  machines 0 .. M-5   odometer, once per item (prefix sums kept)
//   mid    machines M-4, M-3   runtime loops, contributions in shared memory
//   inner1 machine  M-2        compile-time radix D1 (registers)
//   inner2 machine  M-1        compile-time radix DL (registers)
// An item = one outer prefix = D3*D2*D1*DL candidates.  Per candidate the fast
// path issues one DADD (prefix + last contribution, the reference's own
// left-to-right order) and one compare OR-ed into a `hit` predicate: a
// DSETP.GT.OR, or in non-negative spaces an ISETP on the total's high word
// (ge_or_hi below).
// h |= (v > b) as one DSETP.GT.OR per candidate (left to nvcc, a run of
// `hit |= v > best` is rewritten into a max-reduction costing ~8 ALU ops
// per candidate; ptxas folds the selp/setp pairs of consecutive calls).
__device__ __forceinline__ void gt_or(double v, double b, unsigned& h) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %0, 0;\n\tsetp.gt.or.f64 p, %1, %2, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "+r"(h)
      : "d"(v), "d"(b));
}

// Non-negative spaces (every OK contribution has a clear sign bit and is not
// NaN, checked on the host): every feasible total is >= +0.0, and for such
// doubles the high 32-bit word is monotone in the value, so
// h |= hi(v) >= thr with thr = max(hi(best), 0) never misses a v > best; it
// may report equal-high-word candidates (and NaN totals), which only send the
// item to the exact in-order re-scan.  One ISETP on the integer pipe instead
// of a DSETP on the half-rate FP64 pipe; infeasible totals (-inf) have a
// negative high word and never hit.
__device__ __forceinline__ void ge_or_hi(double v, int32_t thr, unsigned& h) {
  asm("{\n\t.reg .pred p, q;\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tsetp.ne.u32 q, %0, 0;\n\t"
      "setp.ge.or.s32 p, hi, %2, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "+r"(h)
      : "d"(v), "r"(thr));
}
__device__ __forceinline__ int32_t hi_threshold(double best) {
  const int32_t hb = (int32_t)(__double_as_longlong(best) >> 32);
  return hb > 0 ? hb : 0;
}

template <int D1, int DL>
struct Radix {
  static constexpr bool kStatic = D1 > 0 && DL > 0;
};

// Slow path: scan one item in index order, tracking (best, lowest index);
// candidates outside [lo, hi) (item-relative) are skipped.
__device__ __noinline__ void item_scan(const double* sC, int M, double s, bool prefix_ok, int64_t base, int64_t lo,
                                       int64_t hi, double& best, int64_t& bidx, int64_t& cnt, bool count) {
  const int D3 = c_space.D[M - 4], D2 = c_space.D[M - 3], D1 = c_space.D[M - 2], DL = c_space.D[M - 1];
  const double* C3 = &sC[(M - 4) * HS_MAX_DEGREES];
  const double* C2 = &sC[(M - 3) * HS_MAX_DEGREES];
  const double* C1 = &sC[(M - 2) * HS_MAX_DEGREES];
  const double* CL = &sC[(M - 1) * HS_MAX_DEGREES];
  int64_t c = 0;
  for (int d3 = 0; d3 < D3; ++d3) {
    const double s3 = __dadd_rn(s, C3[d3]);
    for (int d2 = 0; d2 < D2; ++d2) {
      const double s2 = __dadd_rn(s3, C2[d2]);
      for (int d1 = 0; d1 < D1; ++d1) {
        const double v1 = __dadd_rn(s2, C1[d1]);
        for (int dl = 0; dl < DL; ++dl, ++c) {
          if (c < lo || c >= hi) continue;
          const double v = __dadd_rn(v1, CL[dl]);
          const bool ok = prefix_ok && C3[d3] != -INFINITY && C2[d2] != -INFINITY && C1[d1] != -INFINITY &&
                          CL[dl] != -INFINITY;
          if (count && ok) ++cnt;
          if (ok && v > best) {
            best = v;
            bidx = base + c;
          }
        }
      }
    }
  }
}

template <int D1, int DL, bool NN>
__global__ void __launch_bounds__(256, 3) k_search_best(int64_t item_begin, int64_t item_end, int64_t begin,
                                                     int64_t end, int64_t chunk, double* blk_best,
                                                     int64_t* blk_idx, int64_t* blk_cnt) {
  __shared__ double sC[kMaxM * HS_MAX_DEGREES];
  __shared__ double rb[256 / 32];
  __shared__ int64_t ri[256 / 32], rc[256 / 32];
  const int M = c_space.M;
  for (int k = threadIdx.x; k < M * HS_MAX_DEGREES; k += blockDim.x) sC[k] = c_space.C[k];
  __syncthreads();
  const int D3 = c_space.D[M - 4], D2 = c_space.D[M - 3];
  const int64_t Din = (int64_t)D3 * D2 * c_space.D[M - 2] * c_space.D[M - 1];
  const int64_t inner_ok =
      c_space.okcnt[M - 4] * c_space.okcnt[M - 3] * c_space.okcnt[M - 2] * c_space.okcnt[M - 1];
  const double* C3 = &sC[(M - 4) * HS_MAX_DEGREES];
  const double* C2 = &sC[(M - 3) * HS_MAX_DEGREES];
  constexpr int R1 = D1 > 0 ? D1 : 1, RL = DL > 0 ? DL : 1;
  double C1[R1], CL[RL];
#pragma unroll
  for (int d = 0; d < R1; ++d) C1[d] = sC[(M - 2) * HS_MAX_DEGREES + d];
#pragma unroll
  for (int d = 0; d < RL; ++d) CL[d] = sC[(M - 1) * HS_MAX_DEGREES + d];

  double best = -INFINITY;
  int32_t thr = 0;  // NN: hi_threshold(best)
  int64_t bidx = -1, cnt = 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t it = item_begin + tid * chunk;
  int64_t it_end = it + chunk;
  if (it_end > item_end) it_end = item_end;
  if (it < it_end) {
    const int nouter = M - 4;  // machines 0 .. nouter-1
    int32_t dig[kMaxM];
    double ps[kMaxM];  // ps[i] = left-to-right sum of machines 0..i
    int64_t x = it;
    for (int i = nouter - 1; i >= 0; --i) {
      dig[i] = (int32_t)(x % c_space.D[i]);
      x /= c_space.D[i];
    }
    double acc = 0.0;
    for (int i = 0; i < nouter; ++i) {
      acc = __dadd_rn(acc, sC[i * HS_MAX_DEGREES + dig[i]]);
      ps[i] = acc;
    }
    double s = nouter > 0 ? ps[nouter - 1] : 0.0;
    for (; it < it_end; ++it) {
      const bool prefix_ok = s != -INFINITY && s == s;
      const int64_t base = it * Din;
      if (base < begin || base + Din > end) {
        item_scan(sC, M, s, prefix_ok, base, begin - base, end - base, best, bidx, cnt, true);
        if (NN) thr = hi_threshold(best);
      } else {
        // four independent hit accumulators: one predicate chain would
        // serialise every compare on the previous one's result
        unsigned hit = 0, h4[4] = {0u, 0u, 0u, 0u};
        if (Radix<D1, DL>::kStatic) {
          for (int d3 = 0; d3 < D3; ++d3) {
            const double s3 = __dadd_rn(s, C3[d3]);
            for (int d2 = 0; d2 < D2; ++d2) {
              const double s2 = __dadd_rn(s3, C2[d2]);
#pragma unroll
              for (int d1 = 0; d1 < R1; ++d1) {
                const double v1 = __dadd_rn(s2, C1[d1]);
#pragma unroll
                for (int dl = 0; dl < RL; ++dl) {
                  if (NN) ge_or_hi(__dadd_rn(v1, CL[dl]), thr, h4[(d1 * RL + dl) & 3]);
                  else gt_or(__dadd_rn(v1, CL[dl]), best, h4[(d1 * RL + dl) & 3]);
                }
              }
            }
          }
        } else {
          const int rD1 = c_space.D[M - 2], rDL = c_space.D[M - 1];
          const double* g1 = &sC[(M - 2) * HS_MAX_DEGREES];
          const double* gl = &sC[(M - 1) * HS_MAX_DEGREES];
          for (int d3 = 0; d3 < D3; ++d3) {
            const double s3 = __dadd_rn(s, C3[d3]);
            for (int d2 = 0; d2 < D2; ++d2) {
              const double s2 = __dadd_rn(s3, C2[d2]);
              for (int d1 = 0; d1 < rD1; ++d1) {
                const double v1 = __dadd_rn(s2, g1[d1]);
                for (int dl = 0; dl < rDL; ++dl) {
                  if (NN) ge_or_hi(__dadd_rn(v1, gl[dl]), thr, hit);
                  else gt_or(__dadd_rn(v1, gl[dl]), best, hit);
                }
              }
            }
          }
        }
        hit |= (h4[0] | h4[1]) | (h4[2] | h4[3]);
        if (hit) {
          item_scan(sC, M, s, prefix_ok, base, 0, Din, best, bidx, cnt, false);
          if (NN) thr = hi_threshold(best);
        }
        if (prefix_ok) cnt += inner_ok;
      }
      // odometer over the outer digits, recomputing the changed prefix sums
      if (nouter > 0) {
        int i = nouter - 1;
        while (i >= 0) {
          if (++dig[i] < c_space.D[i]) break;
          dig[i] = 0;
          --i;
        }
        if (i < 0) i = 0;
        double a = i > 0 ? ps[i - 1] : 0.0;
        for (int j = i; j < nouter; ++j) {
          a = __dadd_rn(a, sC[j * HS_MAX_DEGREES + dig[j]]);
          ps[j] = a;
        }
        s = a;
      }
    }
  }
  // block reduction: max total, then lowest index
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (oi >= 0 && (bidx < 0 || ob > best || (ob == best && oi < bidx))) {
      best = ob;
      bidx = oi;
    }
  }
  if (lane == 0) {
    rb[w] = best;
    ri[w] = bidx;
    rc[w] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      cnt += rc[k];
      if (ri[k] >= 0 && (bidx < 0 || rb[k] > best || (rb[k] == best && ri[k] < bidx))) {
        best = rb[k];
        bidx = ri[k];
      }
    }
    blk_best[blockIdx.x] = best;
    blk_idx[blockIdx.x] = bidx;
    blk_cnt[blockIdx.x] = cnt;
  }
}

__global__ void k_search_final(const double* blk_best, const int64_t* blk_idx, const int64_t* blk_cnt, int nblk,
                               hs_cand* out, int64_t* cnt_out) {
  __shared__ double rb[32];
  __shared__ int64_t ri[32], rc[32];
  double best = -INFINITY;
  int64_t bidx = -1, cnt = 0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) {
    cnt += blk_cnt[k];
    const double ob = blk_best[k];
    const int64_t oi = blk_idx[k];
    if (oi >= 0 && (bidx < 0 || ob > best || (ob == best && oi < bidx))) {
      best = ob;
      bidx = oi;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, off);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    if (oi >= 0 && (bidx < 0 || ob > best || (ob == best && oi < bidx))) {
      best = ob;
      bidx = oi;
    }
  }
  if (lane == 0) {
    rb[w] = best;
    ri[w] = bidx;
    rc[w] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      cnt += rc[k];
      if (ri[k] >= 0 && (bidx < 0 || rb[k] > best || (rb[k] == best && ri[k] < bidx))) {
        best = rb[k];
        bidx = ri[k];
      }
    }
    out->total = bidx >= 0 ? best : 0.0;
    out->index = bidx;
    *cnt_out = cnt;
  }
}

using BestKernel = void (*)(int64_t, int64_t, int64_t, int64_t, int64_t, double*, int64_t*, int64_t*);
constexpr int kMaxStaticRadix = 6;

template <int D1, int DL>
struct BestTable {
  static void fill(BestKernel (&t)[2][kMaxStaticRadix + 1][kMaxStaticRadix + 1]) {
    t[0][D1][DL] = k_search_best<D1, DL, false>;
    t[1][D1][DL] = k_search_best<D1, DL, true>;
    if constexpr (DL < kMaxStaticRadix) {
      BestTable<D1, DL + 1>::fill(t);
    } else if constexpr (D1 < kMaxStaticRadix) {
      BestTable<D1 + 1, 1>::fill(t);
    }
  }
};

cudaError_t launch_search_best(const SpaceDesc& sd, int64_t begin, int64_t end, int blocks, double* d_blk_best,
                               int64_t* d_blk_idx, int64_t* d_blk_cnt, hs_cand* d_out, int64_t* d_cnt_out,
                               cudaStream_t st) {
  static BestKernel table[2][kMaxStaticRadix + 1][kMaxStaticRadix + 1] = {};
  static bool filled = false;
  if (!filled) {
    BestTable<1, 1>::fill(table);
    filled = true;
  }
  cudaError_t e = cudaMemcpyToSymbolAsync(c_space, &sd, sizeof(SpaceDesc), 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  const int threads = 256;
  const int M = sd.M;
  const int64_t Din = (int64_t)sd.D[M - 4] * sd.D[M - 3] * sd.D[M - 2] * sd.D[M - 1];
  const int64_t item_begin = begin / Din;
  const int64_t item_end = end > begin ? (end + Din - 1) / Din : item_begin;
  const int64_t n_items = item_end - item_begin;
  const int64_t nthreads = (int64_t)blocks * threads;
  int64_t chunk = (n_items + nthreads - 1) / nthreads;
  if (chunk < 1) chunk = 1;
  const int D1 = sd.D[M - 2], DL = sd.D[M - 1];
  // non-negative space: every OK contribution has a clear sign bit and is not NaN
  bool nn = true;
  for (int i = 0; i < M && nn; ++i)
    for (int d = 0; d < sd.D[i]; ++d) {
      const double c = sd.C[i * HS_MAX_DEGREES + d];
      if (c != -INFINITY && (std::signbit(c) || std::isnan(c))) {
        nn = false;
        break;
      }
    }
  BestKernel k = nn ? k_search_best<0, 0, true> : k_search_best<0, 0, false>;
  if (D1 <= kMaxStaticRadix && DL <= kMaxStaticRadix) k = table[nn ? 1 : 0][D1][DL];
  k<<<blocks, threads, 0, st>>>(item_begin, item_end, begin, end, chunk, d_blk_best, d_blk_idx, d_blk_cnt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_search_final<<<1, 1024, 0, st>>>(d_blk_best, d_blk_idx, d_blk_cnt, blocks, d_out, d_cnt_out);
  return cudaGetLastError();
}

// --------------------------------------------------------- full ranking
// One thread per candidate: left-to-right total and the first machine whose
// entry is not OK (the one whose exception search_optimal_config records).
__global__ void k_search_score(int32_t m_off, int64_t P, double* __restrict__ total, int8_t* __restrict__ first_bad,
                               uint8_t* __restrict__ flag) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P) return;
  const int M = c_space.M;
  int32_t dig[kMaxM];
  int64_t x = c;
  for (int i = M - 1; i >= 0; --i) {
    dig[i] = (int32_t)(x % c_space.D[i]);
    x /= c_space.D[i];
  }
  double acc = 0.0;
  int fb = -1;
  for (int i = 0; i < M; ++i) {
    const double v = c_space.C[i * HS_MAX_DEGREES + dig[i]];
    // status is carried in okcnt bit tricks: -inf marks non-OK entries
    if (v == -INFINITY) {
      fb = i - m_off;
      break;
    }
    acc = __dadd_rn(acc, v);
  }
  total[c] = acc;
  first_bad[c] = (int8_t)fb;
  flag[c] = fb < 0;
}

cudaError_t launch_search_score(const SpaceDesc& sd, int32_t m_off, int64_t P, double* d_total, int8_t* d_first_bad,
                                uint8_t* d_flag, cudaStream_t st) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_space, &sd, sizeof(SpaceDesc), 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  if (P <= 0) return cudaSuccess;
  const int threads = 256;
  k_search_score<<<(unsigned)((P + threads - 1) / threads), threads, 0, st>>>(m_off, P, d_total, d_first_bad,
                                                                              d_flag);
  return cudaGetLastError();
}

}  // namespace hs
