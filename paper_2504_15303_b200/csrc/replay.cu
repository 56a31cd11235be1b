// replay.cu -- K3: batched continuous-batching replay with the capacity-aware
// scheduler, one warp per trace, one lane per instance.
//
// Replaces simulator.py:272-363 run_continuous with scheduling.py:216-346
// (Scheduler.evaluate / _min_max_choice / _commit / complete) and the
// baselines RR / WRR / SI / MB (scheduling.py:246-251, 314-333).
//
// Why lanes may advance independently: a STEP event of instance i reads and
// writes only instance i's run state and, through Scheduler.complete, only
// instance i's load / running tokens (simulator.py:330-355,
// scheduling.py:256-264).  Each instance has at most one pending step
// (simulator.py:292-295) and arrivals sort before steps at equal times
// (simulator.py:285-290).  So arrival a (time t_a) observes, for every
// instance, exactly the state after all of that instance's steps with
// t < t_a: the warp advances every lane's steps with t_next < t_a, then
// dispatches a with warp reductions.  Retirement order within a step is the
// active-list (admission) order, and admission order on an instance is
// dispatch order = trace order, so the retirement heap key
// (departure step, request index) reproduces it.
//
// Per-step bookkeeping: a request admitted at step k_a has generated =
// k - k_a at step k, so it retires at step k_a + O (simulator.py:334) and
// max(I + generated + 1) = max(I - k_a) + k + 1 (simulator.py:351); the
// max is tracked with a count and recomputed from the heap only when its
// last holder retires.  Between events the instance runs "pure" steps: no
// retirement is due before the heap minimum's step, and admission cannot
// succeed until a retirement frees KV or a dispatch fills an empty queue,
// so a pure step is just the decode-iteration price and the clock update
// (latency.py:95-97, simulator.py:352-355): 2 DMUL + 5 DADD in registers.
//
// The state-independent part of the OS workload (ideal batch size and
// per-request cost, scheduling.py:119-147) depends only on (request,
// instance class), so the warp prices 32 (arrival, class) pairs per SIMT
// pass into shared memory; the state-dependent factor exp(theta * usage)
// (capacity.py:98-106, scheduling.py:150-154) is cached per lane and
// recomputed only after the lane's running tokens change.  The min-max
// mapping (scheduling.py:299-312) is O(log N): the max of the loads and an
// argmin of peaks via REDUX on order-preserving 64-bit keys.
#include "hs_device.cuh"
#include <cstdlib>

#include "hs_internal.h"

namespace hs {


#ifdef HS_TIMERS
// Diagnostic build only (-DHS_TIMERS): per-warp cycle counts of the replay
// phases, summed over the launch: advance, price, evaluate, event-step parts,
// pass counters, then min-max (16), commit (17), final drain (18), whole trace (19).
__device__ unsigned long long g_timers[24];
// accumulated in registers (tacc[]) and flushed once per lane at kernel end
#define HS_T0(v) long long v = clock64()
#define HS_T1(slot, v) \
  do { tacc[slot] += (unsigned long long)(clock64() - v); } while (0)
#else
#define HS_T0(v)
#define HS_T1(slot, v)
#endif

constexpr int kWarps = 4;
// at most this many one-warp traces per SM run the pipelined pure loop
constexpr int kPipeTracesPerSM = 8;
// Resident blocks per SM that __launch_bounds__ asks for (of the block's real
// size, replay_block_threads: a 3-warp trace is a 96-thread block; bounding it
// as 128 threads cost config 5 8 %: 425 vs 393 ms).  One-warp traces
// (N <= 32) are issue-bound and gain from occupancy: 4 blocks (128 registers)
// beats 3 (168) by 17 % on config 4.  Multi-warp traces (W > 1) spill at 128
// registers (60-150 B) and lose more to the spills than they gain from the
// extra block: 3 blocks is 11 % faster on config 5 (K3).
#ifndef HS_REPLAY_MIN_BLOCKS
#define HS_REPLAY_MIN_BLOCKS 4
#endif
// the PIPE instantiation runs at most kPipeTracesPerSM traces (2 blocks) per SM,
// so it may take up to 256 registers (it uses ~160, no spills: 1024 traces 265.8 -> 260.4 ms)
#ifndef HS_REPLAY_PIPE_MIN_BLOCKS
#define HS_REPLAY_PIPE_MIN_BLOCKS 2
#endif
#ifndef HS_REPLAY_MIN_BLOCKS_MULTI
#define HS_REPLAY_MIN_BLOCKS_MULTI 3
#endif
constexpr unsigned FULL = 0xffffffffu;
// threads of a replay block: G trace groups of W warps (G = 4 / 2 / 1 for W = 1 / 2 / >= 3)
__host__ __device__ constexpr int replay_block_threads(int W) { return W * (W == 1 ? 4 : (W == 2 ? 2 : 1)) * 32; }

// Per-lane min-heap of retirement entries: key = departure step << 32 |
// request (orders retirements as the reference's active list does) and
// mk = I - k_admit (the quantity whose max gives the cached length).
// Entries [0, kHS) live in shared memory, the rest in global memory (kHS = 16;
// 4 for traces of more than 4 warps, whose 256 lanes share a block).
struct HEnt {
  uint64_t key;
  int64_t mk;
};
template <int kHS>
struct HeapT {
  HEnt* s;  // shared part, kHS entries
  HEnt* g;  // global part (entry i >= kHS at g[i - kHS])
  // Generic accessors (heap larger than kHS).  Kept out of line so nvcc
  // cannot if-convert them into loads of both the shared and the global
  // address, which would put a global round trip on every heap operation.
  __device__ __noinline__ HEnt get_any(int32_t i) const {
    if (i < kHS) return s[i];
    return g[i - kHS];
  }
  __device__ __noinline__ void set_any(int32_t i, HEnt v) const {
    if (i < kHS) s[i] = v;
    else g[i - kHS] = v;
  }
  __device__ __forceinline__ HEnt get(int32_t i, int32_t n) const { return n <= kHS ? s[i] : get_any(i); }
  __device__ __forceinline__ void push(int32_t& n, HEnt e) const {
    int32_t i = n++;
    if (n <= kHS) {  // shared memory only
      while (i > 0) {
        const int32_t p = (i - 1) >> 1;
        const HEnt hp = s[p];
        if (hp.key <= e.key) break;
        s[i] = hp;
        i = p;
      }
      s[i] = e;
      return;
    }
    while (i > 0) {
      const int32_t p = (i - 1) >> 1;
      const HEnt hp = get_any(p);
      if (hp.key <= e.key) break;
      set_any(i, hp);
      i = p;
    }
    set_any(i, e);
  }
  __device__ __forceinline__ void pop(int32_t& n) const {
    if (n <= kHS) {  // shared memory only
      const HEnt last = s[--n];
      int32_t i = 0;
      for (;;) {
        int32_t l = 2 * i + 1;
        if (l >= n) break;
        HEnt hl = s[l];
        if (l + 1 < n) {
          const HEnt hr = s[l + 1];
          if (hr.key < hl.key) {
            hl = hr;
            ++l;
          }
        }
        if (last.key <= hl.key) break;
        s[i] = hl;
        i = l;
      }
      if (n > 0) s[i] = last;
      return;
    }
    const HEnt last = get_any(--n);
    int32_t i = 0;
    for (;;) {
      int32_t l = 2 * i + 1;
      if (l >= n) break;
      HEnt hl = get_any(l);
      if (l + 1 < n) {
        const HEnt hr = get_any(l + 1);
        if (hr.key < hl.key) {
          hl = hr;
          ++l;
        }
      }
      if (last.key <= hl.key) break;
      set_any(i, hl);
      i = l;
    }
    if (n > 0) set_any(i, last);
  }
};

// Queue record of request a (written by the lane that owns the request):
// P and the recorded workload W at dispatch; next / nI / nO when the next
// request is enqueued behind it, so popping a head yields the new head's
// lengths in the same load.
struct QRec {
  int32_t next, nI, nO, P;
  double W;
};

// order-preserving key of a double (ascending); +0.0 and -0.0 share one key
// because Python's comparisons treat them as equal.
__device__ __forceinline__ uint64_t okey(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_okey(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k) {
  const unsigned hi = __reduce_max_sync(FULL, (unsigned)(k >> 32));
  const unsigned lo = __reduce_max_sync(FULL, (unsigned)(k >> 32) == hi ? (unsigned)k : 0u);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t k) {
  const unsigned hi = __reduce_min_sync(FULL, (unsigned)(k >> 32));
  const unsigned lo = __reduce_min_sync(FULL, (unsigned)(k >> 32) == hi ? (unsigned)k : 0xffffffffu);
  return ((uint64_t)hi << 32) | lo;
}

// Rarely touched per-lane state lives in shared memory.
struct Cold {
  double completion, wcur, err_t;
  double segmax;  // HS_REPLAY_ORDER_KEYS: running max of step times since the lane last went idle
  int64_t tok_count;
  int32_t req_count, err, err_req;
  int32_t ty;    // instance class (read from here: a per-lane constant-bank index serialises)
  int32_t nret;  // HS_REPLAY_ORDER_KEYS: retirements so far (per-lane processing order)
};

// ReplayConst.flags
constexpr int32_t kOrderKeys = 1;  // depart = (time, heap key, per-lane sequence) triples
constexpr int32_t kTrackMax = 2;   // step costs may be negative: every step is an event step
constexpr int32_t kMono = 4;       // decode coefficients >= 0: a pure run's clock never decreases

// One instance class of the deployment, staged in shared memory once per
// trace group: lanes read their class by index from shared memory instead of
// the constant bank, where per-lane indices serialise (the compiler
// rematerialises these values rather than keeping them in registers).
struct TypeRec {
  double p[8];
  double budget;
  int64_t cap_tok;  // floor(floor(budget) / per_token)
  double rbudget;   // RN(1 / budget): kv_usage's division by one FMA correction (div_rn_by)
};
constexpr int kTypeRecWords = sizeof(TypeRec) / sizeof(double);

// Cross-warp exchange for traces spanning W > 1 warps: one slot per warp of
// the trace group, a named barrier per group (ids 1..4).
struct Xch {
  uint64_t a, b;
  int32_t c, d;
};
// Per-instance record of one dispatch (multi-warp traces, OS / MB): the
// load's order key and the candidate key of load + w (~0: not a candidate).
struct DispRec {
  uint64_t lk, ko;
};
__device__ __forceinline__ void group_bar(int g, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(nthreads) : "memory");
}

template <int W, bool MULTI, bool CAL, bool PIPE>
__global__ void __launch_bounds__(replay_block_threads(W),
                                  W == 1 ? (PIPE ? HS_REPLAY_PIPE_MIN_BLOCKS : HS_REPLAY_MIN_BLOCKS)
                                         : (W > kWarps ? 1 : HS_REPLAY_MIN_BLOCKS_MULTI))
    k_replay(int64_t n_traces, const int64_t* __restrict__ off, const int32_t* __restrict__ gI,
             const int32_t* __restrict__ gO, const int32_t* __restrict__ gP, const double* __restrict__ gT,
             uint8_t* __restrict__ assign, double* __restrict__ depart, hs_inst_metrics* __restrict__ metrics,
             hs_trace_result* __restrict__ result, QRec* __restrict__ qrec_all, uint64_t* __restrict__ heap_all,
             const ReplayConst* __restrict__ deps, const int32_t* __restrict__ trace_dep,
             const int64_t* __restrict__ trace_heap, int n_max, int max_types, const uint32_t* progress,
             int32_t phase_len, const __grid_constant__ ReplayConst c_one) {
  constexpr int G = W == 1 ? 4 : (W == 2 ? 2 : 1);  // trace groups per block
  constexpr int kThreads = (W > kWarps ? W : kWarps) * 32;
  constexpr int kHS = replay_heap_prefix(W);
  using Heap = HeapT<kHS>;
  __shared__ uint64_t s_tab[256];
  __shared__ Cold s_cold[kThreads];
  // CAL: per-lane summary of the calendar's bucket bitmap (bit i: word i non-empty)
  __shared__ uint64_t s_csum[CAL ? kThreads : 1][kCalSumWords];
  __shared__ HEnt s_heap[kThreads][kHS];
  __shared__ Xch s_x[G][W];
  // W > 1, OS / MB: one published record per instance and one flag word per
  // warp per dispatch, double-buffered by arrival parity, so a dispatch
  // needs a single group barrier (every warp then reduces all W*32 records)
  __shared__ DispRec s_disp[W > 1 ? 2 : 1][G][W > 1 ? W * 32 : 1];
  __shared__ uint4 s_dflag[W > 1 ? 2 : 1][G][W];
  __shared__ uint32_t s_steps[G];
  extern __shared__ double s_cost[];  // [kWarps][32 * n_types] prices, then [G][n_types] TypeRec
  for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab[k] = kExpTab[k];
  if (threadIdx.x < G) s_steps[threadIdx.x] = 0;
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int g = wib / W, wsub = wib - g * W;
  const int64_t tr = (int64_t)blockIdx.x * G + g;
  if (tr >= n_traces) return;
  // single deployment: the kernel parameter (constant bank); per-trace
  // deployments: the trace's record in global memory
  const ReplayConst& c_rep = MULTI ? deps[trace_dep[tr]] : c_one;
  const int N = c_rep.N;
  const int NT = c_rep.n_types;
  const int policy = c_rep.policy;
  const int64_t pt = c_rep.per_token;
  const double theta = c_rep.theta;
  // shared-memory strides: the launch-wide class count (traces of one block
  // may run deployments with different class counts)
  const int NTS = MULTI ? max_types : NT;
  double* cost = s_cost + (size_t)wib * 32 * NTS;
  TypeRec* types = reinterpret_cast<TypeRec*>(s_cost + (size_t)(W * G) * 32 * NTS) + (size_t)g * NTS;
  for (int k = wsub * 32 + lane; k < NT * kTypeRecWords; k += W * 32) {
    const int t = k / kTypeRecWords, f = k - t * kTypeRecWords;
    double* dst = reinterpret_cast<double*>(types + t) + f;
    if (f < 8) *dst = c_rep.type_p[t][f];
    else if (f == 8) *dst = c_rep.type_budget[t];
    else if (f == 9) *reinterpret_cast<int64_t*>(dst) = c_rep.type_cap_tokens[t];
    else *dst = __ddiv_rn(1.0, c_rep.type_budget[t]);
  }
  if (W > 1) group_bar(g, W * 32);
  else __syncwarp();
  Cold& cold = s_cold[threadIdx.x];
  Xch* xg = s_x[g];
  // combine helper: every warp of the group publishes one slot, all read all
  auto xchg = [&](const Xch& mine, Xch* all) {
    if (W > 1) {
      if (lane == 0) xg[wsub] = mine;
      group_bar(g, W * 32);
#pragma unroll
      for (int w = 0; w < W; ++w) all[w] = xg[w];
      group_bar(g, W * 32);
    } else {
      all[0] = mine;
    }
  };

  const int64_t o = off[tr];
  const int64_t q = off[tr + 1] - o;
  const int32_t* I = gI + o;
  const int32_t* O = gO + o;
  const int32_t* P = gP + o;
  const double* T = gT ? gT + o : nullptr;
  QRec* R = qrec_all + o;
  // with kOrderKeys every request owns three doubles of `depart`
  double* DEP = depart ? depart + ((c_rep.flags & kOrderKeys) ? 3 * o : o) : nullptr;

  const int jj = wsub * 32 + lane;  // instance index of this lane
  const bool valid = jj < N;
  const int j = valid ? jj : 0;
  cold.ty = c_rep.inst_type[j];
  const int& ty = cold.ty;
  const TypeRec& trec = types[ty];
  const double* tp = trec.p;
  const double budget = trec.budget;
  const double p7 = tp[6], p8 = tp[7];
  const int64_t hbase = MULTI ? trace_heap[tr] : tr * c_rep.heap_stride;
  const Heap heap{s_heap[threadIdx.x], reinterpret_cast<HEnt*>(heap_all) + hbase + c_rep.heap_off[j]};
  const int64_t cap_tok = trec.cap_tok;  // floor(floor(budget) / per_token)
  const int32_t cap = (int32_t)(c_rep.heap_off[j + 1] - c_rep.heap_off[j]) + kHS;
  // CAL: the retirement calendar replaces the heap -- a ring of B = 2^cal_bits
  // buckets indexed by retirement step (B > every output length, so the
  // active steps (k, k + max O] never collide), each a list of requests in
  // admission order (= request order, the heap's tie-break) linked through
  // the retired queue records (QRec.next; QRec.nI holds I - k_admit), plus a
  // two-level bitmap of non-empty buckets: words in global memory after the
  // buckets, their summary in shared memory.
  const uint32_t cmask = CAL ? (1u << c_rep.cal_bits) - 1u : 0u;
  int2* const cal = reinterpret_cast<int2*>(reinterpret_cast<HEnt*>(heap_all) + hbase + c_rep.heap_off[j]);
  uint64_t* const csum = s_csum[CAL ? threadIdx.x : 0];
  int32_t topnext = -1;  // CAL: the next request of the top bucket's list
  if (CAL) {
    uint64_t* cb = reinterpret_cast<uint64_t*>(cal + cmask + 1);
    if (valid)
      for (uint32_t i = 0; i <= (cmask >> 6); ++i) cb[i] = 0ull;
#pragma unroll
    for (int i = 0; i < kCalSumWords; ++i) csum[i] = 0ull;
  }

  // hot per-lane state (registers)
  double load = 0.0, ex = 1.0;
  int64_t run_i = 0, run_p = 0, reserved = 0, cur_max = INT64_MIN, max_res = 0;
  uint32_t k = 0, kr = 0xffffffffu;  // steps executed; step of the next retirement
  double t_next = 0.0, cd = 0.0, A = 0.0, B = 0.0;  // clock, cached len (double), p5*b, p6*b
  // queue head: index, lengths, and its prefetched record
  int32_t qhead = -1, qtail = -1, hI = 0, hO = 0, hP = 0, hnext = -1, hnI = 0, hnO = 0;
  double hW = 0.0;
  // heap: size, minimum key and the prefetched payload of the minimum
  int32_t nact = 0, topI = 0, topO = 0, topP = 0;
  uint64_t topkey = 0;
  double topW = 0.0;
  bool sched = false, dirty = true, ex_over = false, max_dirty = false, blocked = false, lerr = false;
  cold.completion = 0.0;
  cold.segmax = -INFINITY;
  cold.nret = 0;
  cold.wcur = 0.0;
  cold.err_t = 0.0;
  cold.tok_count = 0;
  cold.req_count = 0;
  int32_t cnt_max = 0;  // holders of cur_max among the active requests (a register: -1.2 % / -4.3 %)
  cold.err = HS_TRACE_OK;
  cold.err_req = -1;
  uint32_t n_steps = 0;
  int64_t rr_next = 0;
#ifdef HS_TIMERS
  unsigned long long tacc[24] = {};
  const long long t_all0 = clock64();
#endif
  int32_t t_err = HS_TRACE_OK, t_err_inst = -1;
  int64_t t_err_req = -1;
  double t_err_val = 0.0;

  auto set_err = [&](int32_t code, int32_t r, double t) {
    cold.err = code;
    cold.err_req = r;
    cold.err_t = t;
    lerr = true;
  };

  // A full STEP event (simulator.py:330-355): retirements due at this step,
  // FCFS admission, prefill for newcomers, one decode iteration.
#ifdef HS_TIMERS
#define HS_LT0(v) const long long v = clock64()
#define HS_LT1(slot, v) tacc[slot] += (unsigned long long)(clock64() - v)
#else
#define HS_LT0(v)
#define HS_LT1(slot, v)
#endif
  // ---- CAL helpers
  // the head of a bucket (retirement step s_) becomes the top: its payload
  // (the pushed record holds O and I - k_admit, k_admit = s_ - max(O, 1):
  // one record load, not three scattered ones)
  auto cal_set_top = [&](uint32_t s_, int32_t r2) {
    topkey = ((uint64_t)s_ << 32) | (uint32_t)r2;
    const QRec q2 = R[r2];
    topO = q2.nO;
    topI = (int32_t)((int64_t)q2.nI + (int64_t)s_ - (int64_t)(q2.nO > 1 ? q2.nO : 1));
    topP = q2.P;
    topW = q2.W;
    topnext = q2.next;
  };
  // bucket of step s_ emptied: clear its bit; returns the bitmap word
  auto cal_clear = [&](uint32_t s_) -> uint64_t {
    uint64_t* cb = reinterpret_cast<uint64_t*>(cal + cmask + 1);
    const uint32_t b = s_ & cmask, wi = b >> 6;
    const uint64_t w = cb[wi] & ~(1ull << (b & 63));
    cb[wi] = w;
    if (!w) csum[wi >> 6] &= ~(1ull << (wi & 63));
    return w;
  };
  // the first non-empty bucket at or after step p, circularly (every active
  // step lies in [p, p + B)); w0 = the bitmap word holding p's bucket
  auto cal_next = [&](uint32_t p, uint64_t w0) {
    const uint64_t* cb = reinterpret_cast<const uint64_t*>(cal + cmask + 1);
    const uint32_t b0 = p & cmask, wi0 = b0 >> 6;
    uint64_t w = w0 & (~0ull << (b0 & 63));
    uint32_t wi = wi0;
    if (!w) {
      // summary bits after wi0, then around to wi0 itself (its bits below b0)
      const uint32_t ns = (((cmask >> 6) + 1) + 63) >> 6;
      const uint32_t s0 = wi0 >> 6, bw = wi0 & 63;
      wi = 0xffffffffu;
      for (uint32_t t = 0; t <= ns && wi == 0xffffffffu; ++t) {
        const uint32_t si = (s0 + t) & (ns - 1);  // ns is a power of two
        uint64_t m = csum[si];
        if (t == 0) m &= bw == 63 ? 0ull : (~0ull << (bw + 1));
        else if (t == ns) m &= bw == 63 ? ~0ull : ((2ull << bw) - 1ull);
        if (m) wi = si * 64 + (uint32_t)(__ffsll((long long)m) - 1);
      }
      w = cb[wi];
    }
    const uint32_t b = (wi << 6) + (uint32_t)(__ffsll((long long)w) - 1);
    cal_set_top(p + ((b - b0) & cmask), cal[b].x);
  };

  auto event_step = [&]() {
    const double t = t_next;
    sched = false;
    // the reference's heap pops a step once every earlier step of its busy
    // period has popped: its order key is the running max of their times
    // (== t whenever step costs are non-negative)
    if (c_rep.flags & kTrackMax) cold.segmax = t > cold.segmax ? t : cold.segmax;
#ifdef HS_TIMERS
    tacc[14] += nact > kHS ? 1 : 0;
    tacc[15] += nact;
#endif
    ++n_steps;
#ifdef HS_TIMERS
    tacc[7] += 1;
#endif
    HS_LT0(tr0);
    while (nact > 0 && (uint32_t)(topkey >> 32) == k) {
      // retire in (departure step, admission order); payload was prefetched
      const int32_t r = (int32_t)(topkey & 0xffffffffu);
      const int64_t Ir = topI, Or = topO, Pr = topP;
      const double wr = topW;
      if (CAL) {
        --nact;
        if (topnext >= 0) {  // the bucket's list goes on (same step)
          cal_set_top(k, topnext);
        } else {
          const uint64_t wk = cal_clear(k);
          if (nact > 0) {
            const uint32_t p = k + 1;
            const uint32_t wp = (p & cmask) >> 6;
            cal_next(p, wp == ((k & cmask) >> 6) ? wk : reinterpret_cast<const uint64_t*>(cal + cmask + 1)[wp]);
          }
        }
      } else {
        heap.pop(nact);
        if (nact > 0) {
          topkey = heap.s[0].key;  // the root always lives in shared memory
          const int32_t r2 = (int32_t)(topkey & 0xffffffffu);
          topI = I[r2];
          topO = O[r2];
          topP = R[r2].P;
          topW = R[r2].W;
        }
      }
      reserved -= Ir + Or;
      if (W > 1) {  // multi-warp traces count at retirement: off the barrier-paced dispatch
        cold.req_count += 1;
        cold.tok_count += Ir + Or;
      }
      cold.completion = t;
      if (DEP) {
        if (c_rep.flags & kOrderKeys) {
          DEP[3 * (int64_t)r] = t;
          DEP[3 * (int64_t)r + 1] = (c_rep.flags & kTrackMax) ? cold.segmax : t;
          DEP[3 * (int64_t)r + 2] = (double)cold.nret++;
        } else {
          DEP[r] = t;
        }
      }
      load = __dsub_rn(load, wr);  // Scheduler.complete: the recorded values
      run_i -= Ir;
      run_p -= Pr;
      dirty = true;
      if (run_i < 0 || run_p < 0) {
        set_err(HS_TRACE_NEGATIVE_RUNNING, r, t);
        return;
      }
      const int64_t ka = (int64_t)k - (Or > 1 ? Or : 1);
      if (Ir - ka == cur_max && --cnt_max == 0) max_dirty = true;
    }
    if (nact == 0) {
      cur_max = INT64_MIN;
      cnt_max = 0;
      max_dirty = false;
    }
    HS_LT1(3, tr0);
    HS_LT0(ta0);
    // admit FCFS (simulator.py:297-316)
    int64_t newly = 0, max_i_new = 0;
    while (qhead >= 0) {
      const int64_t need = (int64_t)hI + hO;
      // simulator.py:303 per_token * (reserved + need) > budget, exactly:
      // an integer X satisfies pt*X > B iff X > floor(floor(B) / pt)
      if (reserved + need > cap_tok) {
        if (nact == 0 && newly == 0) {
          set_err(HS_TRACE_INFEASIBLE_REQUEST, qhead, t);
          return;
        }
        break;
      }
      if ((!CAL && nact >= cap) || k > 0x7fffffffu) {
        set_err(HS_TRACE_CAPACITY, qhead, t);
        return;
      }
      const int32_t r = qhead;
      const int64_t Ir = hI, Or = hO, Pr = hP;
      const double wr = hW;
      if (r == qtail) {
        qhead = -1;
      } else {  // the next head's lengths came with the popped record
        qhead = hnext;
        hI = hnI;
        hO = hnO;
        const QRec nr = R[qhead];  // prefetch the new head's record
        hnext = nr.next;
        hnI = nr.nI;
        hnO = nr.nO;
        hP = nr.P;
        hW = nr.W;
      }
      reserved += need;
      if (Ir > max_i_new) max_i_new = Ir;
      ++newly;
      const uint32_t sstep = k + (uint32_t)(Or > 1 ? Or : 1);
      const uint64_t key = ((uint64_t)sstep << 32) | (uint32_t)r;
      if (nact == 0 || key < topkey) {
        topkey = key;
        topI = (int32_t)Ir;
        topO = (int32_t)Or;
        topP = (int32_t)Pr;
        topW = wr;
        topnext = -1;
      }
      const int64_t mk = Ir - (int64_t)k;
      if (CAL) {
        // append r to bucket sstep: its queue record becomes the list node
        uint64_t* cb = reinterpret_cast<uint64_t*>(cal + cmask + 1);
        const uint32_t b = sstep & cmask, wi = b >> 6;
        const uint64_t bit = 1ull << (b & 63);
        const uint64_t w = cb[wi];
        R[r].next = -1;
        R[r].nI = (int32_t)mk;
        R[r].nO = (int32_t)Or;
        if (w & bit) {
          const int32_t tl = cal[b].y;
          R[tl].next = r;
          cal[b].y = r;
          if (tl == (int32_t)(uint32_t)topkey) topnext = r;  // appended right behind the top
        } else {
          cal[b] = make_int2(r, r);
          cb[wi] = w | bit;
          csum[wi >> 6] |= 1ull << (wi & 63);
        }
        ++nact;
      } else {
        heap.push(nact, HEnt{key, mk});
      }
      if (mk > cur_max) {
        cur_max = mk;
        cnt_max = 1;
        max_dirty = false;
      } else if (mk == cur_max) {
        cnt_max += 1;
      }
    }
    blocked = true;  // queue empty or its head does not fit: nothing changes until an event
    // simulator.py:315 peak = max(peak, per_token*reserved / budget): the
    // quotient is monotone in the numerator, so the max of the quotients is
    // the quotient of the max reservation (divided once, at the end).
    if (newly && reserved > max_res) max_res = reserved;
    HS_LT1(4, ta0);
    HS_LT0(tc0_);
    if (nact == 0) {  // idle until the next dispatch (simulator.py:344-345)
      kr = 0xffffffffu;
      return;
    }
    double c = 0.0;
    if (newly) c = __dadd_rn(c, prefill_time(tp, newly, max_i_new));
    if (max_dirty || cnt_max <= 0) {  // the last holder of the max retired: rescan
      int64_t m = INT64_MIN;
      int32_t cm = 0;
#ifdef HS_TIMERS
      tacc[10] += 1;
      tacc[11] += nact;
#endif
      auto count = [&](int64_t mk) {
        if (mk > m) {
          m = mk;
          cm = 1;
        } else if (mk == m) {
          ++cm;
        }
      };
      if (CAL) {  // every active request: the non-empty buckets' lists
        const uint64_t* cb = reinterpret_cast<const uint64_t*>(cal + cmask + 1);
        const uint32_t ns = (((cmask >> 6) + 1) + 63) >> 6;
        for (uint32_t si = 0; si < ns; ++si) {
          for (uint64_t sm = csum[si]; sm; sm &= sm - 1) {
            const uint32_t wi = si * 64 + (uint32_t)(__ffsll((long long)sm) - 1);
            for (uint64_t w = cb[wi]; w; w &= w - 1) {
              const uint32_t b = (wi << 6) + (uint32_t)(__ffsll((long long)w) - 1);
              for (int32_t rr = cal[b].x; rr >= 0;) {
                const QRec qq = R[rr];
                count(qq.nI);
                rr = qq.next;
              }
            }
          }
        }
      } else {
        for (int32_t h = 0; h < nact; ++h) count(heap.get(h, nact).mk);
      }
      cur_max = m;
      cnt_max = cm;
      max_dirty = false;
    }
    const double db = i2d(nact);
    A = __dmul_rn(tp[4], db);
    B = __dmul_rn(tp[5], db);
    cd = i2d(cur_max + (int64_t)k + 1);
    // decode_iteration_time(cached, batch) = ((A*c + B) + p7*c) + p8
    const double dec = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, cd), B), __dmul_rn(p7, cd)), p8);
    c = __dadd_rn(c, dec);
    k += 1;
    cd = __dadd_rn(cd, 1.0);
    kr = (uint32_t)(topkey >> 32);
    t_next = __dadd_rn(t, c);
    sched = true;
    HS_LT1(5, tc0_);
  };

  // The earliest failing step event of the trace group (heap order: time,
  // then instance); false when no lane failed.
  auto resolve_step_err = [&]() -> bool {
    const unsigned eb = __ballot_sync(FULL, valid && lerr);
    if (W == 1 && !eb) return false;
    Xch mine{~0ull, 0, -1, -1};
    if (eb) {
      const uint64_t tk = (valid && lerr) ? okey(cold.err_t) : ~0ull;
      const uint64_t mt = warp_min_u64(tk);
      const int bl = __ffs(__ballot_sync(FULL, tk == mt)) - 1;
      mine.a = mt;
      mine.b = (uint64_t)(wsub * 32 + bl);
      mine.c = __shfl_sync(FULL, cold.err, bl);
      mine.d = __shfl_sync(FULL, cold.err_req, bl);
    }
    Xch all[W];
    xchg(mine, all);
    int best = -1;
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (all[w].c >= 0 && (best < 0 || all[w].a < all[best].a)) best = w;
    if (best < 0) return false;
    t_err = all[best].c;
    t_err_req = all[best].d;
    t_err_inst = (int32_t)all[best].b;
    t_err_val = from_okey(all[best].a);  // the failing step's time
    return true;
  };

  // Advance every lane's steps with t_next < t_limit (strict: steps at an
  // arrival's own time run after it), or every step when draining.
  auto advance = [&](double t_limit, bool drain, bool defer) -> bool {
    const double lim = drain ? INFINITY : t_limit;
    for (;;) {
      const bool want = valid && sched && (drain || t_next < t_limit) && !lerr;
      if (!__any_sync(FULL, want)) break;
#ifdef HS_TIMERS
      tacc[8] += 1;
      tacc[12] += __popc(__ballot_sync(FULL, want && !(blocked && k < kr)));
#endif
      // phase 1: lanes whose next step is an event (retirement due, or an
      // admission may succeed)

      if (want && ((c_rep.flags & kTrackMax) || !(blocked && k < kr))) event_step();
#ifdef HS_TIMERS
      __syncwarp();
      HS_T0(tpu);
#endif
      // phase 2: every lane whose next steps are pure runs them together,
      // up to its next event or the arrival time.  Two steps per iteration:
      // their prices depend only on the cached length, so both are computed
      // side by side and only the clock additions stay serial (the
      // reference's rounding order).
      const bool pure = valid && sched && !lerr && blocked && k < kr && (drain || t_next < t_limit) &&
                        !(c_rep.flags & kTrackMax);
      if (pure) {
        const uint32_t k0 = k;
        // decode price of a step with cached length x (latency.py:95-97)
        auto price = [&](double x) { return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, x), B), __dmul_rn(p7, x)), p8); };
        // Blocks of four steps, software-pipelined: the four prices of the
        // next block (they depend only on the cached length) are computed
        // while this block's four clock additions -- the only serial part,
        // in the reference's rounding order -- run.  Exit predicates are
        // evaluated off the chain; the state is taken at the first step that
        // may not run (extra additions are discarded).
        double c0 = price(cd), c1 = price(__dadd_rn(cd, 1.0)), c2 = price(__dadd_rn(cd, 2.0)),
               c3 = price(__dadd_rn(cd, 3.0));
        const bool mono = (c_rep.flags & kMono) != 0;
        for (;;) {
#ifdef HS_TIMERS
          if (lane == __ffs(__activemask()) - 1) tacc[9] += 1;
          tacc[13] += 1;
#endif
          const double t1 = __dadd_rn(t_next, c0);
          const double t2 = __dadd_rn(t1, c1);
          const double t3 = __dadd_rn(t2, c2);
          const double t4 = __dadd_rn(t3, c3);
          // monotone clocks: t4 < lim implies t1, t2, t3 < lim, so one test
          // admits the whole block; the per-step tests run on the block that
          // exits.  At full occupancy (issue-bound) the next block's prices are
          // computed only once the block is admitted (none wasted on exits);
          // PIPE (few traces per SM: latency-bound) computes them alongside
          // this block's clock chain, off the dependent path.
          double n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0;
          if (PIPE) {
            n0 = price(__dadd_rn(cd, 4.0));
            n1 = price(__dadd_rn(cd, 5.0));
            n2 = price(__dadd_rn(cd, 6.0));
            n3 = price(__dadd_rn(cd, 7.0));
          }
          const bool all4 = mono ? (k + 4 < kr && (drain || t4 < lim))
                                 : (k + 4 < kr && (drain || (t1 < lim && t2 < lim && t3 < lim && t4 < lim)));
          if (all4) {
            t_next = t4;
            cd = __dadd_rn(cd, 4.0);
            k += 4;
            if (PIPE) {
              c0 = n0;
              c1 = n1;
              c2 = n2;
              c3 = n3;
            } else {
              c0 = price(cd);
              c1 = price(__dadd_rn(cd, 1.0));
              c2 = price(__dadd_rn(cd, 2.0));
              c3 = price(__dadd_rn(cd, 3.0));
            }
            continue;
          }
          // step i+1 runs iff step i ran, k+i < kr and t_i < lim
          const bool g1 = k + 1 < kr && (t1 < lim || drain);
          const bool g2 = g1 && k + 2 < kr && (t2 < lim || drain);
          const bool g3 = g2 && k + 3 < kr && (t3 < lim || drain);
          const uint32_t n = 1u + (uint32_t)g1 + (uint32_t)g2 + (uint32_t)g3;
          t_next = g3 ? t4 : (g2 ? t3 : (g1 ? t2 : t1));
          cd = __dadd_rn(cd, (double)n);
          k += n;
          break;
        }
        n_steps += k - k0;
      }
#ifdef HS_TIMERS
      __syncwarp();
      HS_T1(6, tpu);
#endif
    }
    // defer: a multi-warp dispatch folds the error check into its exchange
    return defer ? false : resolve_step_err();
  };

  const bool is_static = c_rep.mode == 1;
  // classes held by this warp's lanes (HS_MAX_CLASSES <= 32)
  const unsigned warp_classes = __reduce_or_sync(FULL, valid ? 1u << ty : 0u);
  bool failed = false;
  uint8_t my_assign = 0;
  for (int64_t base = 0; base < q && !failed; base += 32) {
    const int n_in = (int)((q - base) < 32 ? (q - base) : 32);
    if (progress) {
      // streamed inputs (host path): phase p of every trace is resident once
      // *progress > p (the copy stream publishes it after the phase's copies)
      const uint32_t need = (uint32_t)((base + n_in - 1) / phase_len);
      int stalled = 0;
      if (lane == 0) {
        const long long t0 = clock64();
        uint32_t have;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(progress) : "memory");
        while (have <= need) {
          __nanosleep(256);
          if (clock64() - t0 > 20000000000ll) {  // ~10 s: report instead of hanging the device
            stalled = 1;
            break;
          }
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(progress) : "memory");
        }
      }
      stalled = __shfl_sync(FULL, stalled, 0);
      if (W > 1) {  // every warp of the trace group takes the same decision
        Xch all[W];
        xchg(Xch{0, 0, stalled, 0}, all);
#pragma unroll
        for (int w = 0; w < W; ++w) stalled |= all[w].c;
      }
      if (stalled) {
        t_err = HS_TRACE_STALLED;
        t_err_req = base;
        t_err_inst = -1;
        failed = true;
        break;
      }
    }
    int32_t cI = 0, cO = 0, cP = 0;
    double cT = 0.0;
    if (lane < n_in) {  // L2-coherent loads: streamed inputs arrive while the kernel runs
      cI = __ldcg(I + base + lane);
      cO = __ldcg(O + base + lane);
      cP = __ldcg(P + base + lane);
      cT = T ? __ldcg(T + base + lane) : 0.0;
    }
    // price (arrival, class) pairs: scheduling.py:119-147
    __syncwarp();
    HS_T0(tp0);
    if (policy != HS_POLICY_MB) {
      auto price_pair = [&](int tyk, int64_t Ia, int64_t Pa) {
        const double fl = py_floordiv(types[tyk].budget, i2d(pt * (Ia + Pa)));
        int64_t b = (int64_t)fl;
        if (b < 1) b = 1;
        const double* ctp = types[tyk].p;
        const double tot = __dadd_rn(prefill_time(ctp, b, Ia), decode_time(ctp, b, Ia, Pa));
        return (tot <= 0.0) ? -1.0 : __ddiv_rn(tot, i2d(b));
      };
      if (W > 1) {
        // a warp of a multi-warp trace prices only the classes its own
        // lanes hold: lane = arrival, one pass per class
        for (unsigned m = warp_classes; m; m &= m - 1) {
          const int tyk = __ffs(m) - 1;
          if (lane < n_in) cost[lane * NT + tyk] = price_pair(tyk, cI, cP);
        }
      } else {
        for (int pair0 = 0; pair0 < n_in * NT; pair0 += 32) {
          const int pair = pair0 + lane;
          const int al = pair / NT, tyk = pair - al * NT;
          const int srcl = al < 32 ? al : 0;
          const int64_t Ia = __shfl_sync(FULL, cI, srcl);
          const int64_t Pa = __shfl_sync(FULL, cP, srcl);
          if (pair < n_in * NT) cost[pair] = price_pair(tyk, Ia, Pa);
        }
      }
      __syncwarp();
    }
    HS_T1(1, tp0);
    for (int al = 0; al < n_in; ++al) {
      const int64_t a = base + al;
      const double ta = shfl_d(cT, al);
      HS_T0(ta0);
      const bool eval_all = policy == HS_POLICY_OS || policy == HS_POLICY_MB;
      // multi-warp OS / MB: the step-error check joins the dispatch's exchange
      const bool fused = W > 1 && eval_all;
      if (!is_static && advance(ta, false, fused)) {
        failed = true;
        break;
      }
      HS_T1(0, ta0);
      HS_T0(te0);
      const int64_t Ia = __shfl_sync(FULL, cI, al);
      const int64_t Oa = __shfl_sync(FULL, cO, al);
      const int64_t Pa = __shfl_sync(FULL, cP, al);
      // ---- choose (scheduling.py:235-254)
      int chosen = -1;
      if (!eval_all) {
        if (policy == HS_POLICY_SI) {
          chosen = 0;
        } else if (policy == HS_POLICY_RR) {
          chosen = (int)(rr_next % N);
          rr_next += 1;
        } else {  // smooth WRR: first strict maximum after adding the weights
          if (valid) cold.wcur = __dadd_rn(cold.wcur, c_rep.wrr_weight[jj]);
          const uint64_t wk = valid ? okey(cold.wcur) : 0ull;
          const uint64_t mk = warp_max_u64(wk);
          const unsigned wb = __ballot_sync(FULL, valid && wk == mk);
          Xch all[W];
          xchg(Xch{wb ? mk : 0ull, (uint64_t)(wsub * 32 + __ffs(wb) - 1), wb ? 1 : 0, 0}, all);
          int bw = -1;
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (all[w].c && (bw < 0 || all[w].a > all[bw].a)) bw = w;
          chosen = (int)all[bw].b;
          if (jj == chosen) cold.wcur = __dsub_rn(cold.wcur, c_rep.wrr_total);
        }
      }
      // ---- evaluate (scheduling.py:216-233) on the lanes that need it
      const bool need = valid && (eval_all || jj == chosen);
      double w = INFINITY;
      bool cerr = false, eerr = false;
      if (need) {
        double cst = 1.0;
        if (policy != HS_POLICY_MB) {
          cst = cost[al * NT + ty];
          cerr = cst < 0.0;
        }
        HS_T0(tx0);
        if (dirty) {  // capacity.py:98-106 kv_usage, scheduling.py:154 exp
#if HS_RECIP_DIV
          const double usage = div_rn_by(i2d(pt * (run_i + run_p)), budget, trec.rbudget);
#else
          const double usage = __ddiv_rn(i2d(pt * (run_i + run_p)), budget);
#endif
          bool of;
          ex = py_exp(__dmul_rn(theta, usage), s_tab, &of);
          ex_over = of;
          dirty = false;
        }
        eerr = ex_over;
        w = __dmul_rn(cst, ex);
        HS_T1(21, tx0);
      }
      HS_T1(2, te0);
      HS_T0(tm0);
      const unsigned errb = __ballot_sync(FULL, need && (cerr || eerr));
      bool any_err = errb != 0;
      const DispRec* drec = nullptr;
      if (fused) {
        // publish (load key, load + w) and the warp's error / candidate
        // masks; one barrier; every warp then sees the whole group
        const int buf = (int)(a & 1);
        const unsigned stepb = __ballot_sync(FULL, valid && lerr);
        // candidate key of own = load + w: its peak is max(own, top), so a NaN
        // own (never > top) ranks as the smallest key and +inf is no candidate
        const double own = __dadd_rn(load, w);
        const uint64_t ko = (need && !isinf(w)) ? (isnan(own) ? 0ull : (own < INFINITY ? okey(own) : ~0ull)) : ~0ull;
        s_disp[buf][g][jj] = DispRec{valid ? okey(load) : 0ull, ko};
        if (lane == 0) s_dflag[buf][g][wsub] = make_uint4(errb, stepb, 0u, 0u);
        HS_T0(tb0);
        group_bar(g, W * 32);
        HS_T1(20, tb0);
        drec = s_disp[buf][g];
        unsigned any_e = 0, any_s = 0;
#pragma unroll
        for (int w2 = 0; w2 < W; ++w2) {
          const uint4 f = s_dflag[buf][g][w2];
          any_e |= f.x;
          any_s |= f.y;
        }
        if (any_s) {  // a step before this arrival failed: that error wins
          resolve_step_err();
          failed = true;
          break;
        }
        any_err = any_e != 0;
      } else if (W > 1) {
        Xch all[W];
        xchg(Xch{0, 0, errb ? 1 : 0, 0}, all);
        any_err = false;
#pragma unroll
        for (int w = 0; w < W; ++w) any_err |= all[w].c != 0;
      }
      if (any_err) {  // the first instance in evaluation order raises
        Xch mine{0, 0, -1, 0};
        if (errb) {
          const int el = __ffs(errb) - 1;
          const bool ce = __shfl_sync(FULL, cerr, el);
          double cval = 0.0;
          if (lane == el && ce) {  // recompute the non-positive total for the message
            const double fl = py_floordiv(budget, i2d(pt * (Ia + Pa)));
            int64_t b = (int64_t)fl;
            if (b < 1) b = 1;
            cval = __dadd_rn(prefill_time(tp, b, Ia), decode_time(tp, b, Ia, Pa));
          }
          mine = Xch{(uint64_t)__double_as_longlong(shfl_d(cval, el)), (uint64_t)(wsub * 32 + el), ce ? 1 : 0, 0};
        }
        Xch all[W];
        xchg(mine, all);
        int bw = -1;
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (all[w].c >= 0 && (bw < 0 || all[w].b < all[bw].b)) bw = w;
        t_err = all[bw].c ? HS_TRACE_NONPOSITIVE_COST : HS_TRACE_EXP_OVERFLOW;
        t_err_inst = (int32_t)all[bw].b;
        t_err_req = a;
        t_err_val = __longlong_as_double((long long)all[bw].a);
        failed = true;
        break;
      }
      if (eval_all) {
        // _min_max_choice (scheduling.py:299-312): argmin (lowest index) of
        // peak_s = max(L_s + w_s, max_{j != s} L_j).  Since w_s >= 0 and
        // rounding is monotone, L_s + w_s >= L_s, so the max over j != s may
        // include s itself: peak_s = max(L_s + w_s, max_j L_j) -- one max
        // reduction instead of the top-2 of the loads.
        if (fused) {
          // the whole group's reduction from the published records, in
          // every warp.  With M = max load key and K_s = candidate key, the
          // peak key is max(K_s, M), so the minimum peak is max(min K, M) =:
          // thr and the choice is the lowest instance with K_s <= thr: the
          // max and the min reduce side by side, then one ballot per warp.
          uint64_t lm = 0, km = ~0ull, ko[W];
#pragma unroll
          for (int w2 = 0; w2 < W; ++w2) {
            const DispRec e = drec[w2 * 32 + lane];
            lm = e.lk > lm ? e.lk : lm;
            km = e.ko < km ? e.ko : km;
            ko[w2] = e.ko;
          }
          const uint64_t m1 = warp_max_u64(lm);
          const uint64_t kmin = warp_min_u64(km);
          const double top = from_okey(m1);
          const uint64_t thr = kmin > m1 ? kmin : m1;
          unsigned ci = 0xffffffffu;
          if (top < INFINITY && kmin != ~0ull) {  // a NaN or +inf top leaves no candidate
#pragma unroll
            for (int w2 = W - 1; w2 >= 0; --w2) {
              const unsigned b = __ballot_sync(FULL, ko[w2] <= thr);
              if (b) ci = (unsigned)(w2 * 32 + __ffs(b) - 1);
            }
          }
          if (ci == 0xffffffffu) {
            t_err = HS_TRACE_NO_INSTANCE;
            t_err_req = a;
            t_err_inst = -1;
            failed = true;
            break;
          }
          chosen = (int)ci;
        } else {  // W == 1 (multi-warp OS / MB traces take the fused path)
          // the same threshold form as above: the max-load and the
          // min-candidate reductions are independent, then one ballot
          const double own = __dadd_rn(load, w);
          const uint64_t kown =
              (need && !isinf(w)) ? (isnan(own) ? 0ull : (own < INFINITY ? okey(own) : ~0ull)) : ~0ull;
          const uint64_t m1 = warp_max_u64(valid ? okey(load) : 0ull);
          const uint64_t kmin = warp_min_u64(kown);
          const double top = from_okey(m1);
          const uint64_t thr = kmin > m1 ? kmin : m1;
          const bool any = top < INFINITY && kmin != ~0ull;  // a NaN or +inf top leaves no candidate
          const unsigned win = __ballot_sync(FULL, any && kown <= thr);
          if (!win) {
            t_err = HS_TRACE_NO_INSTANCE;
            t_err_req = a;
            t_err_inst = -1;
            failed = true;
            break;
          }
          chosen = __ffs(win) - 1;
        }
      }

      HS_T1(16, tm0);
      HS_T0(tc0);
      // ---- commit (scheduling.py:335-346) and enqueue (simulator.py:323-327)
      if (jj == chosen) {
        load = __dadd_rn(load, w);
        run_i += Ia;
        run_p += Pa;
        dirty = true;
        // InstanceMetrics request / token counts (simulator.py:338-341): in a
        // replay that completes, every dispatched request retires exactly
        // once, so one-warp traces (and static mode, which has no event
        // steps) accumulate them here, off the retirement path; multi-warp
        // continuous traces count at retirement instead, off the dispatch
        // that their barrier paces (a failed trace reports an error instead
        // of metrics)
        if (W == 1 || is_static) {
          cold.req_count += 1;
          cold.tok_count += Ia + Oa;
        }
        R[a].P = (int32_t)Pa;
        R[a].W = w;
        if (qhead < 0) {
          qhead = (int32_t)a;
          hI = (int32_t)Ia;
          hO = (int32_t)Oa;
          hP = (int32_t)Pa;
          hW = w;
          blocked = false;  // a new queue head may be admitted at the next step
        } else if (qtail == qhead) {  // the head's prefetched record gains its successor
          hnext = (int32_t)a;
          hnI = (int32_t)Ia;
          hnO = (int32_t)Oa;
          R[qtail].next = (int32_t)a;
        } else {
          QRec& tr_ = R[qtail];
          tr_.next = (int32_t)a;
          tr_.nI = (int32_t)Ia;
          tr_.nO = (int32_t)Oa;
        }
        qtail = (int32_t)a;
        if (!sched) {
          sched = true;
          t_next = ta;
          blocked = false;
          if (c_rep.flags & kTrackMax) cold.segmax = -INFINITY;  // a new busy period
        }
      }
      if (lane == al) my_assign = (uint8_t)chosen;
      HS_T1(17, tc0);

    }
    if (assign && wsub == 0 && lane < n_in && !failed) assign[o + base + lane] = my_assign;
  }
  HS_T0(tdr0);
  if (!failed && !is_static && advance(0.0, true, false)) failed = true;
  HS_T1(18, tdr0);
  if (!failed && is_static) {
    // run_static (simulator.py:229-247): each instance runs its assigned
    // requests (queue order = trace order) as greedy KV-feasible static
    // batches (planner.py:51-87 with the true output lengths), prices each
    // with estimate_batch_time (planner.py:90-101), advances its clock and
    // fires the completion hooks in batch order.
    bool bad = false;
    int32_t bad_r = -1;
    if (valid) {
      double clock = 0.0;
      int32_t r = qhead;
      while (r >= 0) {
        int64_t sumI = 0, maxO = 0, maxI = 0, width = 0;
        int32_t c = r, stop = -1;
        while (c >= 0) {
          const int64_t Ic = I[c], Oc = O[c];
          const int64_t cI = sumI + Ic, cMO = maxO > Oc ? maxO : Oc;
          if (sat_add(cI, sat_mul(width + 1, cMO)) > cap_tok) break;
          sumI = cI;
          maxO = cMO;
          if (Ic > maxI) maxI = Ic;
          ++width;
          c = (c == qtail) ? -1 : R[c].next;
        }
        stop = c;
        if (width == 0) {
          bad = true;
          bad_r = r;
          break;
        }
        const int64_t res_tok = sumI + width * maxO;
        if (res_tok > max_res) max_res = res_tok;
        clock = __dadd_rn(clock, __dadd_rn(prefill_time(tp, width, maxI), decode_time(tp, width, maxI, maxO)));
        for (int32_t m = r; m != stop;) {
          const QRec rec = R[m];
          load = __dsub_rn(load, rec.W);
          if (DEP) {
            if (c_rep.flags & kOrderKeys) {
              DEP[3 * (int64_t)m] = clock;
              DEP[3 * (int64_t)m + 1] = clock;
              DEP[3 * (int64_t)m + 2] = (double)cold.nret++;
            } else {
              DEP[m] = clock;
            }
          }
          m = (m == qtail) ? -1 : rec.next;
        }
        r = stop;
      }
      cold.completion = clock;
    }
    const unsigned bb = __ballot_sync(FULL, bad);
    Xch mine{0, 0, -1, 0};
    if (bb) {
      const int bl = __ffs(bb) - 1;
      mine = Xch{0, (uint64_t)(wsub * 32 + bl), 1, __shfl_sync(FULL, bad_r, bl)};
    }
    Xch all[W];
    xchg(mine, all);
    int bw = -1;
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (all[w].c > 0 && (bw < 0 || all[w].b < all[bw].b)) bw = w;
    if (bw >= 0) {  // the first instance (config order) whose plan fails raises
      t_err = HS_TRACE_INFEASIBLE_REQUEST;
      t_err_req = all[bw].d;
      t_err_inst = (int32_t)all[bw].b;
      failed = true;
    }
  }

#ifdef HS_TIMERS
  // warp-level phases (slots 0-2, 6) were timed by every lane: count lane 0;
  // event-step parts (3-5, 7) are per lane
  tacc[19] += (unsigned long long)(clock64() - t_all0);
  for (int sl = 0; sl < 24; ++sl) {
    const bool warp_slot = sl <= 2 || sl == 6 || sl == 8 || sl == 12 || sl >= 16;
    if (!warp_slot || lane == 0) atomicAdd(&g_timers[sl], tacc[sl]);
  }
#endif
  if (valid) {
    hs_inst_metrics m;
    m.completion_time = cold.completion;
    m.peak_kv_usage = max_res > 0 ? __ddiv_rn(i2d(pt * max_res), budget) : 0.0;
    m.residual_load = load;
    m.request_count = cold.req_count;
    m.token_count = cold.tok_count;
    metrics[tr * (int64_t)n_max + jj] = m;
  }
  int64_t steps_all = n_steps;
#pragma unroll
  for (int offs = 16; offs > 0; offs >>= 1) steps_all += __shfl_xor_sync(FULL, steps_all, offs);
  if (W > 1) {
    if (lane == 0) atomicAdd(&s_steps[g], (uint32_t)steps_all);
    group_bar(g, W * 32);
    steps_all = s_steps[g];
  }
  if (lane == 0 && wsub == 0) {
    hs_trace_result r;
    r.error = failed ? t_err : HS_TRACE_OK;
    r.err_instance = failed ? t_err_inst : -1;
    r.err_request = failed ? t_err_req : -1;
    r.err_value = failed ? t_err_val : 0.0;
    r.n_steps = steps_all;
    result[tr] = r;
  }
}

template <int W, bool MULTI, bool CAL, bool PIPE = false>
cudaError_t launch_w(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                     const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign, double* d_depart,
                     hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec, uint64_t* d_heap,
                     cudaStream_t st, const ReplayConst* d_deps, const int32_t* d_trace_dep,
                     const int64_t* d_trace_heap, int n_max, int max_types, const uint32_t* d_progress,
                     int phase_len) {
  constexpr int G = W == 1 ? 4 : (W == 2 ? 2 : 1);
  const int warps = W * G;
  const size_t smem = (size_t)warps * 32 * max_types * sizeof(double) + (size_t)G * max_types * sizeof(TypeRec);
  // static (heaps, per-lane state) + dynamic (price buffer) may exceed the
  // 48 KB default: opt in for the dynamic part every time
  cudaError_t e = cudaFuncSetAttribute(k_replay<W, MULTI, CAL, PIPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)((n_traces + G - 1) / G);
  k_replay<W, MULTI, CAL, PIPE><<<blocks, warps * 32, smem, st>>>(n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics,
                                                d_result, static_cast<QRec*>(d_qrec), d_heap, d_deps, d_trace_dep,
                                                d_trace_heap, n_max, max_types, d_progress, phase_len, rc);
  return cudaGetLastError();
}

// One-warp traces: the software-pipelined pure loop (next block's prices
// computed alongside this block's clock chain) pays when few traces share an
// SM (latency-bound); at full occupancy the kernel is issue-bound and the
// admit-then-price loop wins.  HS_REPLAY_PIPE=0/1 forces either (A/B runs).
static bool replay_pipelined(int64_t n_traces) {
  static const int force = [] {
    const char* e = std::getenv("HS_REPLAY_PIPE");
    return e ? std::atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  return n_traces <= (int64_t)kPipeTracesPerSM * sm_count();
}

cudaError_t launch_replay(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                          const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign,
                          double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec,
                          uint64_t* d_heap, cudaStream_t st, const ReplayConst* d_deps, const int32_t* d_trace_dep,
                          const int64_t* d_trace_heap, int n_max, int max_types, const uint32_t* d_progress,
                          int phase_len) {
  if (n_traces <= 0) return cudaSuccess;
  if (n_max <= 0) n_max = rc.N;
  if (max_types <= 0) max_types = rc.n_types;
  const int W = (n_max + 31) / 32;
#define HS_LW(w, m)                                                                                              \
  (cal ? launch_w<w, m, true>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics, d_result,  \
                              d_qrec, d_heap, st, d_deps, d_trace_dep, d_trace_heap, n_max, max_types, d_progress,  \
                              phase_len)                                                                           \
       : launch_w<w, m, false>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics, d_result, d_qrec, d_heap, \
                 st, d_deps, d_trace_dep, d_trace_heap, n_max, max_types, d_progress, phase_len))
  const bool multi = d_deps != nullptr;
  const bool cal = rc.cal_bits > 0;
  switch (W) {
    case 1:  // one-warp traces keep the shared-memory heap (calendars are for W > 1)
      if (cal) return cudaErrorInvalidValue;
      if (multi)
        return launch_w<1, true, false>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics,
                                        d_result, d_qrec, d_heap, st, d_deps, d_trace_dep, d_trace_heap, n_max,
                                        max_types, d_progress, phase_len);
      if (replay_pipelined(n_traces))
        return launch_w<1, false, false, true>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart,
                                               d_metrics, d_result, d_qrec, d_heap, st, d_deps, d_trace_dep,
                                               d_trace_heap, n_max, max_types, d_progress, phase_len);
      return launch_w<1, false, false>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics,
                                       d_result, d_qrec, d_heap, st, d_deps, d_trace_dep, d_trace_heap, n_max,
                                       max_types, d_progress, phase_len);
    case 2: return multi ? HS_LW(2, true) : HS_LW(2, false);
    case 3: return multi ? HS_LW(3, true) : HS_LW(3, false);
    case 4: return multi ? HS_LW(4, true) : HS_LW(4, false);
    case 5:
    case 6: return multi ? HS_LW(6, true) : HS_LW(6, false);  // idle lanes past N
    case 7:
    case 8: return multi ? HS_LW(8, true) : HS_LW(8, false);
    default: return cudaErrorInvalidValue;
  }
#undef HS_LW
}

// min over all requests of (I + O): sizes the per-instance active-set heaps
__global__ void k_min_need(const int32_t* __restrict__ I, const int32_t* __restrict__ O, int64_t n, int32_t* out,
                           int32_t* max_out) {
  int32_t m = INT32_MAX, mo = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = O[k];
    const int64_t v = (int64_t)I[k] + o;
    const int32_t vv = v > INT32_MAX ? INT32_MAX : (int32_t)v;
    m = vv < m ? vv : m;
    mo = o > mo ? o : mo;
  }
  m = __reduce_min_sync(FULL, (unsigned)m);
  mo = (int32_t)__reduce_max_sync(FULL, (unsigned)mo);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, m);
    if (max_out) atomicMax(max_out, mo);
  }
}

cudaError_t launch_min_need(const int32_t* d_I, const int32_t* d_O, int64_t n, int32_t* d_out, cudaStream_t st,
                            int32_t* d_max_out) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  const int cap = sm_count() * 8;
  if (blocks > cap) blocks = cap;
  k_min_need<<<blocks, 256, 0, st>>>(d_I, d_O, n, d_out, d_max_out);
  return cudaGetLastError();
}

// the same over the first `width` requests of each of `rows` equal-length
// traces (row pitch `pitch`): the streamed host path sizes its heaps from the
// first phase of every trace
__global__ void k_min_need_2d(const int32_t* __restrict__ I, const int32_t* __restrict__ O, int64_t rows,
                              int64_t width, int64_t pitch, int32_t* out) {
  int32_t m = INT32_MAX;
  const int64_t n = rows * width;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / width, e = r * pitch + (k - r * width);
    const int64_t v = (int64_t)I[e] + O[e];
    const int32_t vv = v > INT32_MAX ? INT32_MAX : (int32_t)v;
    m = vv < m ? vv : m;
  }
  m = __reduce_min_sync(FULL, (unsigned)m);
  if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

cudaError_t launch_min_need_2d(const int32_t* d_I, const int32_t* d_O, int64_t rows, int64_t width, int64_t pitch,
                               int32_t* d_out, cudaStream_t st) {
  if (rows <= 0 || width <= 0) return cudaSuccess;
  int blocks = (int)((rows * width + 255) / 256);
  const int cap = sm_count() * 8;
  if (blocks > cap) blocks = cap;
  k_min_need_2d<<<blocks, 256, 0, st>>>(d_I, d_O, rows, width, pitch, d_out);
  return cudaGetLastError();
}

}  // namespace hs

#ifdef HS_TIMERS
// diagnostic export of the timers build (not part of the ABI header)
extern "C" int hs_debug_timers(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaError_t e = cudaMemcpyFromSymbol(out, hs::g_timers, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(hs::g_timers, z, sizeof(z));
  }
  return e == cudaSuccess ? 0 : 1;
}
#endif
