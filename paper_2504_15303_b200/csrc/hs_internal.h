// hs_internal.h -- host-side glue shared by the C-ABI and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hetserve_b200.h"

namespace hs {

// One (machine, degree) work item of the table build.
struct EntryDesc {
  double p[8];
  int64_t own_count;   // accelerator_count of the machine itself (instance count)
  int64_t spec_count;  // accelerator_count of cluster.machine(name)
  int64_t spec_mem;    // accelerator_mem_bytes of cluster.machine(name)
  int32_t tp;
  int32_t present;
};

struct SearchConst {
  int64_t per_token;        // capacity.py:67-69
  int64_t required;         // capacity.py:93 per_token * (Imax + Omax)
  int64_t weights;          // capacity.py:85 param_count * bytes_per_param
  int64_t static_overhead;  // EngineOverheads.static_overhead_bytes
  double phi;               // EngineOverheads.mem_utilization_fraction
  int64_t q;
};

// Product space for K2: machines padded to M >= 4 (leading virtual
// machines with one degree and contribution +0.0 leave every total
// unchanged: (0.0 + 0.0) + C0 == 0.0 + C0).
constexpr int kMaxM = HS_MAX_MACHINES + 3;
struct SpaceDesc {
  int32_t M;
  int32_t D[kMaxM];
  int64_t okcnt[kMaxM];
  // contributions, -inf where the entry is not OK; [M][HS_MAX_DEGREES]
  double C[kMaxM * HS_MAX_DEGREES];
};

// Feasible sub-product for top-K: per machine its OK degrees only.
struct FeasSpace {
  int32_t M;
  int32_t D[kMaxM];                      // OK degrees per machine
  int64_t stride[kMaxM];                 // stride of the ORIGINAL mixed radix
  double C[kMaxM * HS_MAX_DEGREES];      // contribution of the d-th OK degree
  int32_t orig[kMaxM * HS_MAX_DEGREES];  // its original digit
};

constexpr int kMaxReplayInst = 256;  // up to 8 warps per trace (<= 255 instances: uint8 assignments)
constexpr int kMaxTypes = 32;         // distinct (params, budget) classes per deployment

struct ReplayConst {
  int32_t N;
  int32_t policy;
  int32_t n_types;
  int32_t has_arrival;
  int32_t mode;  // 0 continuous (simulator.py:272), 1 static (simulator.py:206)
  int32_t flags;  // replay.cu kOrderKeys | kTrackMax
  int32_t cal_bits;  // > 0: multi-warp traces keep retirements in a calendar of 2^cal_bits steps
  double theta;
  int64_t per_token;
  double wrr_total;
  int64_t heap_stride;                       // heap entries per trace
  int64_t heap_off[kMaxReplayInst + 1];
  int8_t inst_type[kMaxReplayInst];
  double type_p[kMaxTypes][8];
  double type_budget[kMaxTypes];
  int64_t type_cap_tokens[kMaxTypes];        // floor(floor(budget) / per_token)
  double wrr_weight[kMaxReplayInst];
};

struct PlanParams {
  double p[8];
  int32_t has;  // time the batches (estimate_batch_time) and compute the rate
  int32_t _pad;
};

// launchers (return cudaError_t as int)
cudaError_t launch_table_build(const EntryDesc* d_desc, int n, const SearchConst& sc, const int32_t* d_I,
                               const int32_t* d_O, hs_entry* d_out, cudaStream_t st);
cudaError_t launch_plan_instance(double budget, int64_t per_token, const PlanParams& pp, const int32_t* d_I,
                                 const int32_t* d_O, int64_t q, int64_t* d_stops, double* d_times, int64_t* d_nb,
                                 hs_entry* d_out, cudaStream_t st);
// workspace: 3 * blocks doubles/int64s
cudaError_t launch_search_best(const SpaceDesc& sd, int64_t begin, int64_t end, int blocks,
                               double* d_blk_best, int64_t* d_blk_idx, int64_t* d_blk_cnt,
                               hs_cand* d_out, int64_t* d_cnt_out, cudaStream_t st);
cudaError_t launch_search_score(const SpaceDesc& sd, int32_t m_real_offset, int64_t P, double* d_total,
                                int8_t* d_first_bad, uint8_t* d_flag, cudaStream_t st);
cudaError_t launch_topk_pass(const FeasSpace& fs, bool upload, int mode, int64_t item_begin, int64_t item_end,
                             int shift, uint64_t prefix, uint64_t thr, unsigned long long* d_hist,
                             unsigned long long* d_cnt, uint64_t* d_key, int64_t* d_idx, int64_t cap, int blocks,
                             cudaStream_t st, uint64_t bkey = ~0ull, int64_t bidx = -1);
cudaError_t launch_invert_keys(uint64_t* d_key, int64_t n, cudaStream_t st);
// d_out: min(I + O); d_max_out (optional): max(O)
cudaError_t launch_min_need(const int32_t* d_I, const int32_t* d_O, int64_t n, int32_t* d_out, cudaStream_t st,
                            int32_t* d_max_out = nullptr);
cudaError_t launch_min_need_2d(const int32_t* d_I, const int32_t* d_O, int64_t rows, int64_t width, int64_t pitch,
                               int32_t* d_out, cudaStream_t st);
// deps / trace_dep / trace_heap: per-trace deployments (config 5); when
// deps is null every trace uses rc and trace t's heap starts at t*stride.
cudaError_t launch_replay(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                          const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign,
                          double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result,
                          void* d_qrec, uint64_t* d_heap, cudaStream_t st, const ReplayConst* d_deps = nullptr,
                          const int32_t* d_trace_dep = nullptr, const int64_t* d_trace_heap = nullptr,
                          int n_max = 0, int max_types = 0, const uint32_t* d_progress = nullptr,
                          int phase_len = 0);
// sort.cu: stable LSD radix sort of (key, value) pairs by key bits
// [begin_bit, end_bit), in place (keys / vals; *_alt are scratch of n), and the
// ordered indices of the set flags (*d_count = how many).  workspace:
// sort_workspace_bytes(n).
size_t sort_workspace_bytes(int64_t n);
cudaError_t sort_pairs_u64(uint64_t* keys, uint64_t* vals, uint64_t* keys_alt, uint64_t* vals_alt, int64_t n,
                           int begin_bit, int end_bit, void* workspace, cudaStream_t st);
cudaError_t select_flagged(const uint8_t* flag, int64_t n, int64_t* out, int64_t* d_count, void* workspace,
                           cudaStream_t st);
constexpr int kQRecBytes = 24;  // replay.cu QRec
// retirement calendar (multi-warp traces): 2^cal_bits buckets, cal_bits <= kMaxCalBits
// (the summary bitmap is kCalSumWords 64-bit words per lane)
constexpr int kMaxCalBits = 14;
constexpr int kCalSumWords = 1 << (kMaxCalBits - 12);
constexpr int kHEntBytes = 16;  // replay.cu HEnt
// heap entries per lane kept in shared memory by a trace of w warps (replay.cu kHS)
#ifndef HS_REPLAY_HEAP_PREFIX
#define HS_REPLAY_HEAP_PREFIX 16
#endif
__host__ __device__ constexpr int replay_heap_prefix(int w) { return w > 4 ? 4 : HS_REPLAY_HEAP_PREFIX; }

// Seeded streams (rng.cu): up to kMaxDists distributions drawn in order from
// each stream; out[j] is indexed by the stream offsets.
constexpr int kMaxDists = 4;
struct RngConst {
  int32_t n_dists;
  int32_t _pad;
  hs_dist dist[kMaxDists];
  void* out[kMaxDists];
};
cudaError_t launch_rng_generate(const RngConst& rc, hs_pcg64_state* d_states, const int64_t* d_off,
                                int64_t s_begin, int64_t s_end, int64_t* d_bad, cudaStream_t st);

int sm_count();

}  // namespace hs
