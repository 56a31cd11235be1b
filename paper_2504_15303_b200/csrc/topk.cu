// topk.cu -- top-K deployment search (the head of planner.py:227's ranking)
// for spaces too large to rank in full (BASELINE config 5: top-1024 of a
// 5^16 space).
//
// Only feasible candidates can appear in the ranking (planner.py:225-226
// moves every other candidate to `infeasible`), so the enumeration runs over
// the feasible sub-product: machine i contributes its OK degrees only, and a
// candidate's index in the original mixed-radix space is rebuilt from the
// OK-degree positions.  Every feasible candidate's total is evaluated in the
// reference's left-to-right order (planner.py:151,180).
//
// Selection is exact: radix select on order-preserving 64-bit keys of the
// totals (12-bit digits, one histogram pass per digit, stopping as soon as
// the candidates at or above the current bucket fit the collect buffer),
// then one collect pass and a stable device sort by (total desc, index asc).

#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {

__constant__ FeasSpace c_feas;

__device__ __forceinline__ uint64_t key_of(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 and 0.0 tie (Python comparison)
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// mode 0: histogram of key digit (key >> shift) & 4095 among keys whose bits
// above shift+12 equal `prefix`; mode 1: collect keys >= thr.  Only
// candidates ranked after the boundary (bkey, bidx) take part -- key < bkey,
// or key == bkey and index > bidx (planner.py:227 order: total desc, index
// asc) -- so successive calls stream the ranking chunk by chunk.
template <int MODE>
__global__ void __launch_bounds__(256) k_topk_pass(int64_t item_begin, int64_t item_end, int64_t chunk, int shift,
                                                   uint64_t prefix, uint64_t thr, unsigned long long* hist,
                                                   unsigned long long* cnt, uint64_t* out_key, int64_t* out_idx,
                                                   int64_t cap, uint64_t bkey, int64_t bidx) {
  __shared__ unsigned int sh[MODE == 0 ? 4096 : 1];
  __shared__ double sC[kMaxM * HS_MAX_DEGREES];
  const int M = c_feas.M;
  for (int k = threadIdx.x; k < M * HS_MAX_DEGREES; k += blockDim.x) sC[k] = c_feas.C[k];
  if (MODE == 0)
    for (int k = threadIdx.x; k < 4096; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  const int DL = c_feas.D[M - 1];
  const double* CL = &sC[(M - 1) * HS_MAX_DEGREES];
  const int64_t strideL = c_feas.stride[M - 1];
  const int32_t* origL = &c_feas.orig[(M - 1) * HS_MAX_DEGREES];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t it = item_begin + tid * chunk;
  int64_t it_end = it + chunk;
  if (it_end > item_end) it_end = item_end;
  if (it < it_end) {
    const int nouter = M - 1;
    int32_t dig[kMaxM];
    double ps[kMaxM];
    int64_t pidx[kMaxM];  // original index contribution of machines 0..i
    int64_t x = it;
    for (int i = nouter - 1; i >= 0; --i) {
      dig[i] = (int32_t)(x % c_feas.D[i]);
      x /= c_feas.D[i];
    }
    double acc = 0.0;
    int64_t ia = 0;
    for (int i = 0; i < nouter; ++i) {
      acc = __dadd_rn(acc, sC[i * HS_MAX_DEGREES + dig[i]]);
      ia += (int64_t)c_feas.orig[i * HS_MAX_DEGREES + dig[i]] * c_feas.stride[i];
      ps[i] = acc;
      pidx[i] = ia;
    }
    double s = nouter > 0 ? ps[nouter - 1] : 0.0;
    int64_t sidx = nouter > 0 ? pidx[nouter - 1] : 0;
    for (; it < it_end; ++it) {
      for (int d = 0; d < DL; ++d) {
        const uint64_t key = key_of(__dadd_rn(s, CL[d]));
        if (key > bkey || (key == bkey && sidx + (int64_t)origL[d] * strideL <= bidx)) continue;  // not after
        if (MODE == 0) {
          if (shift + 12 >= 64 || (key >> (shift + 12)) == prefix) atomicAdd(&sh[(key >> shift) & 4095u], 1u);
        } else if (key >= thr) {
          const unsigned long long pos = atomicAdd(cnt, 1ull);
          if ((int64_t)pos < cap) {
            out_key[pos] = key;
            out_idx[pos] = sidx + (int64_t)origL[d] * strideL;
          }
        }
      }
      if (nouter > 0) {
        int i = nouter - 1;
        while (i >= 0) {
          if (++dig[i] < c_feas.D[i]) break;
          dig[i] = 0;
          --i;
        }
        if (i < 0) i = 0;
        double a = i > 0 ? ps[i - 1] : 0.0;
        int64_t ib = i > 0 ? pidx[i - 1] : 0;
        for (int j = i; j < nouter; ++j) {
          a = __dadd_rn(a, sC[j * HS_MAX_DEGREES + dig[j]]);
          ib += (int64_t)c_feas.orig[j * HS_MAX_DEGREES + dig[j]] * c_feas.stride[j];
          ps[j] = a;
          pidx[j] = ib;
        }
        s = a;
        sidx = ib;
      }
    }
  }
  if (MODE == 0) {
    __syncthreads();
    for (int k = threadIdx.x; k < 4096; k += blockDim.x)
      if (sh[k]) atomicAdd(&hist[k], (unsigned long long)sh[k]);
  }
}

cudaError_t launch_topk_pass(const FeasSpace& fs, bool upload, int mode, int64_t item_begin, int64_t item_end,
                             int shift, uint64_t prefix, uint64_t thr, unsigned long long* d_hist,
                             unsigned long long* d_cnt, uint64_t* d_key, int64_t* d_idx, int64_t cap, int blocks,
                             cudaStream_t st, uint64_t bkey, int64_t bidx) {
  cudaError_t e;
  if (upload) {
    e = cudaMemcpyToSymbolAsync(c_feas, &fs, sizeof(FeasSpace), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
  }
  const int threads = 256;
  const int64_t n_items = item_end - item_begin;
  if (n_items <= 0) return cudaSuccess;
  const int64_t nthreads = (int64_t)blocks * threads;
  int64_t chunk = (n_items + nthreads - 1) / nthreads;
  if (chunk < 1) chunk = 1;
  if (mode == 0)
    k_topk_pass<0><<<blocks, threads, 0, st>>>(item_begin, item_end, chunk, shift, prefix, thr, d_hist, d_cnt, d_key,
                                               d_idx, cap, bkey, bidx);
  else
    k_topk_pass<1><<<blocks, threads, 0, st>>>(item_begin, item_end, chunk, shift, prefix, thr, d_hist, d_cnt, d_key,
                                               d_idx, cap, bkey, bidx);
  return cudaGetLastError();
}

__global__ void k_invert_keys(uint64_t* key, int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) key[k] = ~key[k];  // ascending sort of ~key == descending totals
}

cudaError_t launch_invert_keys(uint64_t* d_key, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_invert_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_key, n);
  return cudaGetLastError();
}

}  // namespace hs
