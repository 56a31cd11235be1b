// sort.cu -- the ranking's device sort and stream compaction (hs_search_rank,
// the top-K's final order): a stable LSD radix sort of 64-bit keys carrying
// 64-bit values, 4-bit digits, and an order-preserving select of flagged
// indices.  Both are tiled the same way: a tile of kTile items per block, a
// per-(digit, tile) count, one exclusive scan over the counts, then a stable
// scatter in which each block walks its tile in rounds of 256 items (warp
// ballots give an item's rank among equal digits, a shared-memory prefix over
// the block's 8 warps orders the warps).  HBM-bound byte work: every pass
// reads and writes each (key, value) pair once.

#include <cuda_runtime.h>

#include <cstdint>

#include "hs_internal.h"

namespace hs {
namespace {

constexpr int kThreadsS = 256;
constexpr int kWarpsS = kThreadsS / 32;
constexpr int kRounds = 16;
constexpr int kTile = kThreadsS * kRounds;  // 4096 items per block
constexpr int kDigits = 16;                 // 4-bit digits

// counts[d * ntiles + tile] = items of the tile with digit d
__global__ void __launch_bounds__(kThreadsS) k_digit_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                          uint32_t* __restrict__ counts, int64_t ntiles) {
  __shared__ uint32_t h[kDigits];
  if (threadIdx.x < kDigits) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int r = 0; r < kRounds; ++r) {
    const int64_t i = base + (int64_t)r * kThreadsS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (kDigits - 1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kDigits) counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of n counts in place (one block); *total = the sum
__global__ void __launch_bounds__(1024) k_scan_counts(uint32_t* __restrict__ c, int64_t n, int64_t* total) {
  __shared__ uint64_t part[1024];
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = (int64_t)threadIdx.x * per;
  const int64_t e = b + per < n ? b + per : n;
  uint64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += c[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
    const uint64_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  uint64_t run = part[threadIdx.x] - s;
  for (int64_t i = b; i < e; ++i) {
    const uint32_t v = c[i];
    c[i] = (uint32_t)run;
    run += v;
  }
  if (threadIdx.x == 1023 && total) *total = (int64_t)part[1023];
}

// stable scatter of one 4-bit digit pass
__global__ void __launch_bounds__(kThreadsS) k_digit_scatter(const uint64_t* __restrict__ kin,
                                                             const uint64_t* __restrict__ vin, uint64_t* __restrict__ kout,
                                                             uint64_t* __restrict__ vout, int64_t n, int shift,
                                                             const uint32_t* __restrict__ offs, int64_t ntiles) {
  __shared__ uint32_t wcnt[kWarpsS][kDigits];
  __shared__ uint32_t base[kDigits];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x < kDigits) base[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  const unsigned lt = (1u << lane) - 1u;
  const int64_t tbase = (int64_t)blockIdx.x * kTile;
  for (int r = 0; r < kRounds; ++r) {
    const int64_t i = tbase + (int64_t)r * kThreadsS + threadIdx.x;
    const bool in = i < n;
    const uint64_t k = in ? kin[i] : 0ull;
    const uint64_t v = in ? vin[i] : 0ull;
    const int d = in ? (int)((k >> shift) & (kDigits - 1)) : -1;
    unsigned rank = 0;
#pragma unroll
    for (int dd = 0; dd < kDigits; ++dd) {
      const unsigned m = __ballot_sync(0xffffffffu, d == dd);
      if (d == dd) rank = __popc(m & lt);
      if (lane == 0) wcnt[w][dd] = __popc(m);
    }
    __syncthreads();  // wcnt complete (and base from the previous round)
    if (threadIdx.x < kDigits) {  // warp prefix per digit; advance the digit's base
      uint32_t s = base[threadIdx.x];
#pragma unroll
      for (int ww = 0; ww < kWarpsS; ++ww) {
        const uint32_t c = wcnt[ww][threadIdx.x];
        wcnt[ww][threadIdx.x] = s;
        s += c;
      }
      base[threadIdx.x] = s;
    }
    __syncthreads();
    if (in) {
      const uint32_t dst = wcnt[w][d] + rank;
      kout[dst] = k;
      vout[dst] = v;
    }
    __syncthreads();  // wcnt is rewritten by the next round
  }
}

__global__ void __launch_bounds__(kThreadsS) k_flag_count(const uint8_t* __restrict__ flag, int64_t n,
                                                          uint32_t* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * kTile;
  uint32_t c = 0;
  for (int r = 0; r < kRounds; ++r) {
    const int64_t i = base + (int64_t)r * kThreadsS + threadIdx.x;
    if (i < n && flag[i]) ++c;
  }
  __shared__ uint32_t h;
  if (threadIdx.x == 0) h = 0;
  __syncthreads();
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&h, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = h;
}

__global__ void __launch_bounds__(kThreadsS) k_flag_scatter(const uint8_t* __restrict__ flag, int64_t n,
                                                            const uint32_t* __restrict__ offs,
                                                            int64_t* __restrict__ out) {
  __shared__ uint32_t wcnt[kWarpsS];
  __shared__ uint32_t base;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = offs[blockIdx.x];
  const int64_t tbase = (int64_t)blockIdx.x * kTile;
  for (int r = 0; r < kRounds; ++r) {
    const int64_t i = tbase + (int64_t)r * kThreadsS + threadIdx.x;
    const bool f = i < n && flag[i];
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = base;
      for (int ww = 0; ww < kWarpsS; ++ww) {
        const uint32_t c = wcnt[ww];
        wcnt[ww] = s;
        s += c;
      }
      base = s;
    }
    __syncthreads();
    if (f) out[wcnt[w] + __popc(m & ((1u << lane) - 1u))] = i;
    __syncthreads();
  }
}

}  // namespace

size_t sort_workspace_bytes(int64_t n) {
  const int64_t nt = (n + kTile - 1) / kTile;
  return (size_t)(nt > 0 ? nt : 1) * kDigits * sizeof(uint32_t) + sizeof(int64_t);
}

cudaError_t sort_pairs_u64(uint64_t* keys, uint64_t* vals, uint64_t* keys_alt, uint64_t* vals_alt, int64_t n,
                           int begin_bit, int end_bit, void* workspace, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > (int64_t)UINT32_MAX) return cudaErrorInvalidValue;
  const int64_t nt = (n + kTile - 1) / kTile;
  uint32_t* counts = static_cast<uint32_t*>(workspace);
  const int passes = (end_bit - begin_bit + 3) / 4;
  uint64_t *ks = keys, *vs = vals, *kd = keys_alt, *vd = vals_alt;
  for (int p = 0; p < passes; ++p) {
    const int shift = begin_bit + 4 * p;
    k_digit_hist<<<(unsigned)nt, kThreadsS, 0, st>>>(ks, n, shift, counts, nt);
    k_scan_counts<<<1, 1024, 0, st>>>(counts, nt * kDigits, nullptr);
    k_digit_scatter<<<(unsigned)nt, kThreadsS, 0, st>>>(ks, vs, kd, vd, n, shift, counts, nt);
    uint64_t* t = ks;
    ks = kd;
    kd = t;
    t = vs;
    vs = vd;
    vd = t;
  }
  if (ks != keys) {  // an odd number of passes ends in the alternate buffers
    cudaMemcpyAsync(keys, ks, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(vals, vs, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st);
  }
  return cudaGetLastError();
}

cudaError_t select_flagged(const uint8_t* flag, int64_t n, int64_t* out, int64_t* d_count, void* workspace,
                           cudaStream_t st) {
  if (n <= 0) return cudaMemsetAsync(d_count, 0, sizeof(int64_t), st);
  const int64_t nt = (n + kTile - 1) / kTile;
  uint32_t* counts = static_cast<uint32_t*>(workspace);
  k_flag_count<<<(unsigned)nt, kThreadsS, 0, st>>>(flag, n, counts);
  k_scan_counts<<<1, 1024, 0, st>>>(counts, nt, d_count);
  k_flag_scatter<<<(unsigned)nt, kThreadsS, 0, st>>>(flag, n, counts, out);
  return cudaGetLastError();
}

}  // namespace hs
