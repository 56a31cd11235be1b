// replay_mt.cu -- K3, trace-group layout: four traces per warp, eight lanes
// per trace, each lane owning up to four instances (j = lane + 8k).
//
// Same semantics, bit for bit, as replay.cu (simulator.py:272-363
// run_continuous with scheduling.py:216-346 Scheduler.evaluate / choose /
// complete and the RR / WRR / SI / MB baselines); see replay.cu's header for
// why every instance may advance independently between arrivals.
//
// Why this layout: with one warp per trace and one lane per instance, each
// arrival costs as many SIMT passes as its busiest instance needs steps
// (~35 for the fastest class at config 4), while ~9 of 32 lanes do work, and
// every event step (retirement / admission, 1-2 lanes) costs a whole warp
// pass.  Here a lane steps its instances one after another, and the instances
// are dealt so that every lane owns one instance of each class when the
// deployment lists classes in blocks of eight (config 4: b200/h100/a800/v100
// x 8): every lane then carries the same step load, and four traces share
// every warp instruction.  The price is lockstep across the warp's four
// traces: an arrival costs the warp the steps of the trace with the longest
// inter-arrival gap.  Dispatch reductions are 3-level shuffles inside the
// eight-lane group.
//
// Used for continuous mode, one deployment of <= 32 instances, no order keys
// (launch_replay picks it; HS_REPLAY_LEGACY=1 forces replay.cu's kernel).
#include <cstdlib>

#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {
namespace {

constexpr int kL = 8;   // lanes per trace
constexpr int kG = 4;   // traces per warp
constexpr int kWPB = 2;  // warps per block
constexpr int kHS2 = 4;  // heap entries per instance in shared memory
constexpr unsigned FULL = 0xffffffffu;

struct HEnt {
  uint64_t key;
  int64_t mk;
};
struct QRec {  // replay.cu QRec (kQRecBytes)
  int32_t next, nI, nO, P;
  double W;
};
static_assert(sizeof(QRec) == kQRecBytes, "QRec layout");
static_assert(sizeof(HEnt) == kHEntBytes, "HEnt layout");

// Per-instance state in shared memory; the stepping state is in registers (Hot).
struct IState {
  double hW, topW, completion, ex, wcur;
  int64_t run_tot, reserved, cur_max, max_res, tok_count;
  uint64_t topkey;
  int32_t qhead, qtail, hI, hO, hP, hnext, hnI, hnO;
  int32_t nact, topI, topO, topP, req_count, cnt_max;
};

struct TypeRec {  // one instance class
  double p[8];
  double budget;
  int64_t cap_tok;  // floor(floor(budget) / per_token)
};

// Hot per-instance registers.
enum : uint32_t { F_VALID = 1, F_SCHED = 2, F_BLOCKED = 4, F_DIRTY = 8, F_EXOVER = 16, F_MAXDIRTY = 32, F_ERR = 64 };
struct Hot {
  double t_next, cd, A, B, load;
  uint32_t k, kr, fl;
};

__device__ __forceinline__ uint64_t okey(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_okey(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  return (uint64_t)__shfl_xor_sync(FULL, (long long)v, m);
}
// group (8-lane) reductions; every lane of the warp takes part
__device__ __forceinline__ uint64_t group_max_u64(uint64_t v) {
#pragma unroll
  for (int m = 4; m > 0; m >>= 1) {
    const uint64_t o = shfl_xor_u64(v, m);
    v = o > v ? o : v;
  }
  return v;
}
// min of (key, idx) pairs, ties on the lowest idx
__device__ __forceinline__ void group_min_key_idx(uint64_t& key, int& idx) {
#pragma unroll
  for (int m = 4; m > 0; m >>= 1) {
    const uint64_t ok = shfl_xor_u64(key, m);
    const int oi = __shfl_xor_sync(FULL, idx, m);
    if (ok < key || (ok == key && oi < idx)) {
      key = ok;
      idx = oi;
    }
  }
}
__device__ __forceinline__ void group_max_key_idx(uint64_t& key, int& idx) {
#pragma unroll
  for (int m = 4; m > 0; m >>= 1) {
    const uint64_t ok = shfl_xor_u64(key, m);
    const int oi = __shfl_xor_sync(FULL, idx, m);
    if (ok > key || (ok == key && oi < idx)) {
      key = ok;
      idx = oi;
    }
  }
}

// Heap of retirement entries (key = departure step << 32 | request, mk = I -
// k_admit): entries [0, kHS2) in shared memory, the rest in global memory.
struct Heap {
  HEnt* s;
  HEnt* g;
  __device__ __noinline__ HEnt get_any(int32_t i) const {
    if (i < kHS2) return s[i];
    return g[i - kHS2];
  }
  __device__ __noinline__ void set_any(int32_t i, HEnt v) const {
    if (i < kHS2) s[i] = v;
    else g[i - kHS2] = v;
  }
  __device__ __forceinline__ HEnt get(int32_t i, int32_t n) const { return n <= kHS2 ? s[i] : get_any(i); }
  __device__ __forceinline__ void push(int32_t& n, HEnt e) const {
    int32_t i = n++;
    if (n <= kHS2) {
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
    if (n <= kHS2) {
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

// Per-lane record of the earliest failing step among its instances.
struct LaneErr {
  double t;
  int32_t code, inst, req;
};

struct Ctx {
  const int32_t* I;
  const int32_t* O;
  QRec* R;
  double* DEP;
  int64_t pt;
};

// A full STEP event of one instance (simulator.py:330-355): retirements due
// at this step (in admission order), FCFS admission, prefill for newcomers,
// one decode iteration.  Returns false on a trace error (recorded in le).
__device__ __forceinline__ void event_step(Hot& h, IState& S, const Heap& heap, const TypeRec& tr, const Ctx& c,
                                           int32_t cap, int j, uint32_t& n_steps, LaneErr& le) {
  const double t = h.t_next;
  h.fl &= ~F_SCHED;
  ++n_steps;
  int32_t nact = S.nact;
  uint64_t topkey = S.topkey;
  int64_t reserved = S.reserved, run_tot = S.run_tot, cur_max = S.cur_max;
  int32_t cnt_max = S.cnt_max;
  bool max_dirty = (h.fl & F_MAXDIRTY) != 0;
  bool retired = false;
  while (nact > 0 && (uint32_t)(topkey >> 32) == h.k) {
    // retire in (departure step, admission order); payload was prefetched
    const int32_t r = (int32_t)(topkey & 0xffffffffu);
    const int64_t Ir = S.topI, Or = S.topO, Pr = S.topP;
    const double wr = S.topW;
    heap.pop(nact);
    if (nact > 0) {
      topkey = heap.s[0].key;  // the root always lives in shared memory
      const int32_t r2 = (int32_t)(topkey & 0xffffffffu);
      S.topI = c.I[r2];
      S.topO = c.O[r2];
      S.topP = c.R[r2].P;
      S.topW = c.R[r2].W;
    }
    reserved -= Ir + Or;
    retired = true;
    if (c.DEP) c.DEP[r] = t;
    h.load = __dsub_rn(h.load, wr);  // Scheduler.complete: the recorded values
    run_tot -= Ir + Pr;
    const int64_t ka = (int64_t)h.k - (Or > 1 ? Or : 1);
    if (Ir - ka == cur_max && --cnt_max == 0) max_dirty = true;
  }
  if (retired) {
    S.completion = t;
    h.fl |= F_DIRTY;
  }
  if (nact == 0) {
    cur_max = INT64_MIN;
    cnt_max = 0;
    max_dirty = false;
  }
  // admit FCFS (simulator.py:297-316)
  int64_t newly = 0, max_i_new = 0;
  int32_t qhead = S.qhead;
  bool fail = false;
  while (qhead >= 0) {
    const int64_t need = (int64_t)S.hI + S.hO;
    // simulator.py:303 per_token * (reserved + need) > budget, exactly
    if (reserved + need > tr.cap_tok) {
      if (nact == 0 && newly == 0) {
        if (t < le.t || (t == le.t && j < le.inst)) le = LaneErr{t, HS_TRACE_INFEASIBLE_REQUEST, j, qhead};
        h.fl |= F_ERR;
        fail = true;
      }
      break;
    }
    if (nact >= cap || h.k > 0x7fffffffu) {
      if (t < le.t || (t == le.t && j < le.inst)) le = LaneErr{t, HS_TRACE_CAPACITY, j, qhead};
      h.fl |= F_ERR;
      fail = true;
      break;
    }
    const int32_t r = qhead;
    const int64_t Ir = S.hI, Or = S.hO, Pr = S.hP;
    const double wr = S.hW;
    if (r == S.qtail) {
      qhead = -1;
    } else {  // the next head's lengths came with the popped record
      qhead = S.hnext;
      S.hI = S.hnI;
      S.hO = S.hnO;
      const QRec nr = c.R[qhead];  // prefetch the new head's record
      S.hnext = nr.next;
      S.hnI = nr.nI;
      S.hnO = nr.nO;
      S.hP = nr.P;
      S.hW = nr.W;
    }
    reserved += need;
    if (Ir > max_i_new) max_i_new = Ir;
    ++newly;
    const uint64_t key = ((uint64_t)(h.k + (uint32_t)(Or > 1 ? Or : 1)) << 32) | (uint32_t)r;
    if (nact == 0 || key < topkey) {
      topkey = key;
      S.topI = (int32_t)Ir;
      S.topO = (int32_t)Or;
      S.topP = (int32_t)Pr;
      S.topW = wr;
    }
    const int64_t mk = Ir - (int64_t)h.k;
    heap.push(nact, HEnt{key, mk});
    if (mk > cur_max) {
      cur_max = mk;
      cnt_max = 1;
      max_dirty = false;
    } else if (mk == cur_max) {
      cnt_max += 1;
    }
  }
  S.qhead = qhead;
  h.fl |= F_BLOCKED;  // queue empty or its head does not fit
  // simulator.py:315: the max of the quotients is the quotient of the max reservation
  if (newly && reserved > S.max_res) S.max_res = reserved;
  if (!fail && nact > 0) {
    double cst = 0.0;
    if (newly) cst = __dadd_rn(cst, prefill_time(tr.p, newly, max_i_new));
    if (max_dirty || cnt_max <= 0) {  // the last holder of the max retired: rescan
      int64_t m = INT64_MIN;
      int32_t cm = 0;
      for (int32_t q = 0; q < nact; ++q) {
        const int64_t mk = heap.get(q, nact).mk;
        if (mk > m) {
          m = mk;
          cm = 1;
        } else if (mk == m) {
          ++cm;
        }
      }
      cur_max = m;
      cnt_max = cm;
      max_dirty = false;
    }
    const double db = i2d(nact);
    h.A = __dmul_rn(tr.p[4], db);
    h.B = __dmul_rn(tr.p[5], db);
    h.cd = i2d(cur_max + (int64_t)h.k + 1);
    // decode_iteration_time(cached, batch) = ((A*c + B) + p7*c) + p8
    const double dec =
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(h.A, h.cd), h.B), __dmul_rn(tr.p[6], h.cd)), tr.p[7]);
    cst = __dadd_rn(cst, dec);
    h.k += 1;
    h.cd = __dadd_rn(h.cd, 1.0);
    h.kr = (uint32_t)(topkey >> 32);
    h.t_next = __dadd_rn(t, cst);
    h.fl |= F_SCHED;
  } else {
    h.kr = 0xffffffffu;  // idle until the next dispatch (simulator.py:344-345)
  }
  if (max_dirty) h.fl |= F_MAXDIRTY;
  else h.fl &= ~F_MAXDIRTY;
  S.nact = nact;
  S.topkey = topkey;
  S.reserved = reserved;
  S.run_tot = run_tot;
  S.cur_max = cur_max;
  S.cnt_max = cnt_max;
}

// Advance one instance's steps with t_next < t_limit (strict: steps at an
// arrival's own time run after it), or every step when draining.
__device__ __forceinline__ void advance(Hot& h, IState& S, const Heap& heap, const TypeRec& tr, const Ctx& c,
                                        int32_t cap, int j, double t_limit, bool drain, uint32_t& n_steps,
                                        LaneErr& le) {
  const double lim = t_limit;
  const double p7 = tr.p[6], p8 = tr.p[7];
  while ((h.fl & (F_VALID | F_SCHED | F_ERR)) == (F_VALID | F_SCHED) && (drain || h.t_next < lim)) {
    if (!(h.fl & F_BLOCKED) || h.k >= h.kr) {
      event_step(h, S, heap, tr, c, cap, j, n_steps, le);
      continue;
    }
    // pure steps: decode price and clock only, blocks of four, the next
    // block's prices computed while this block's clock additions (the only
    // serial part, in the reference's rounding order) run
    const uint32_t k0 = h.k;
    const double A = h.A, B = h.B;
    auto price = [&](double x) {
      return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, x), B), __dmul_rn(p7, x)), p8);
    };
    double cd = h.cd, tn = h.t_next;
    uint32_t k = h.k;
    const uint32_t kr = h.kr;
    double c0 = price(cd), c1 = price(__dadd_rn(cd, 1.0)), c2 = price(__dadd_rn(cd, 2.0)),
           c3 = price(__dadd_rn(cd, 3.0));
    for (;;) {
      const double t1 = __dadd_rn(tn, c0);
      const double t2 = __dadd_rn(t1, c1);
      const double t3 = __dadd_rn(t2, c2);
      const double t4 = __dadd_rn(t3, c3);
      const double cd4 = __dadd_rn(cd, 4.0);
      const double n0 = price(cd4), n1 = price(__dadd_rn(cd, 5.0)), n2 = price(__dadd_rn(cd, 6.0)),
                   n3 = price(__dadd_rn(cd, 7.0));
      // step i+1 runs iff step i ran, k+i < kr and t_i < lim
      const bool g1 = k + 1 < kr && (drain || t1 < lim);
      const bool g2 = g1 && k + 2 < kr && (drain || t2 < lim);
      const bool g3 = g2 && k + 3 < kr && (drain || t3 < lim);
      const bool g4 = g3 && k + 4 < kr && (drain || t4 < lim);
      if (!g4) {
        const uint32_t n = 1u + (uint32_t)g1 + (uint32_t)g2 + (uint32_t)g3;
        tn = g3 ? t4 : (g2 ? t3 : (g1 ? t2 : t1));
        cd = __dadd_rn(cd, (double)n);
        k += n;
        break;
      }
      tn = t4;
      cd = cd4;
      k += 4;
      c0 = n0;
      c1 = n1;
      c2 = n2;
      c3 = n3;
    }
    h.t_next = tn;
    h.cd = cd;
    h.k = k;
    n_steps += k - k0;
  }
}

// shared memory per block: [IState kWPB*K*32][HEnt kWPB*K*32*kHS2][TypeRec n_types]
template <int K>
__host__ __device__ constexpr size_t mt_smem_fixed() {
  return sizeof(IState) * kWPB * K * 32 + sizeof(HEnt) * kWPB * K * 32 * kHS2;
}

template <int K>
__global__ void __launch_bounds__(kWPB * 32, 4) k_replay_mt(
    int64_t n_traces, const int64_t* __restrict__ off, const int32_t* __restrict__ gI, const int32_t* __restrict__ gO,
    const int32_t* __restrict__ gP, const double* __restrict__ gT, uint8_t* __restrict__ assign,
    double* __restrict__ depart, hs_inst_metrics* __restrict__ metrics, hs_trace_result* __restrict__ result,
    QRec* __restrict__ qrec_all, uint64_t* __restrict__ heap_all, const uint32_t* progress, int32_t phase_len,
    const __grid_constant__ ReplayConst rc) {
  __shared__ uint64_t s_tab[256];
  extern __shared__ double4 s_dyn[];
  IState(*s_ist)[K][32] = reinterpret_cast<IState(*)[K][32]>(s_dyn);
  HEnt(*s_heap)[K][32][kHS2] =
      reinterpret_cast<HEnt(*)[K][32][kHS2]>(reinterpret_cast<char*>(s_dyn) + sizeof(IState) * kWPB * K * 32);
  TypeRec* s_types = reinterpret_cast<TypeRec*>(reinterpret_cast<char*>(s_dyn) + mt_smem_fixed<K>());
  for (int x = threadIdx.x; x < 256; x += blockDim.x) s_tab[x] = kExpTab[x];
  const int NT = rc.n_types;
  for (int x = threadIdx.x; x < NT * 10; x += blockDim.x) {
    const int t = x / 10, f = x - t * 10;
    double* dst = reinterpret_cast<double*>(s_types + t) + f;
    if (f < 8) *dst = rc.type_p[t][f];
    else if (f == 8) *dst = rc.type_budget[t];
    else *reinterpret_cast<int64_t*>(dst) = rc.type_cap_tokens[t];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int grp = lane >> 3;  // trace group within the warp
  const int l = lane & 7;     // lane within the group
  const int64_t warp_global = (int64_t)blockIdx.x * kWPB + wib;
  const int64_t tr_raw = warp_global * kG + grp;
  if (warp_global * kG >= n_traces) return;  // whole warp idle
  const bool tvalid = tr_raw < n_traces;
  const int64_t tr = tvalid ? tr_raw : n_traces - 1;
  const int N = rc.N;
  const int policy = rc.policy;
  const int64_t pt = rc.per_token;
  const double theta = rc.theta;
  const int64_t o = off[tr];
  const int64_t q = tvalid ? off[tr + 1] - o : 0;
  // every group walks arrival indices in lockstep up to the warp's longest trace
  int64_t qmax = q;
#pragma unroll
  for (int m = 8; m < 32; m <<= 1) {
    const int64_t oq = __shfl_xor_sync(FULL, (long long)qmax, m);
    qmax = oq > qmax ? oq : qmax;
  }
  const Ctx c{gI + o, gO + o, qrec_all + o, depart ? depart + o : nullptr, pt};
  const int32_t* P = gP + o;
  const double* T = gT ? gT + o : nullptr;

  Hot h[K];
  int ty[K];
  int32_t capk[K];
  Heap heap[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = l + kL * k;
    const bool v = tvalid && j < N;
    ty[k] = v ? rc.inst_type[j] : 0;
    h[k] = Hot{0.0, 0.0, 0.0, 0.0, 0.0, 0u, 0xffffffffu, v ? (F_VALID | F_DIRTY) : 0u};
    IState& S = s_ist[wib][k][lane];
    S = IState{};
    S.ex = 1.0;
    S.cur_max = INT64_MIN;
    S.qhead = -1;
    S.qtail = -1;
    const int jj = v ? j : 0;
    heap[k] = Heap{s_heap[wib][k][lane],
                   reinterpret_cast<HEnt*>(heap_all) + tr * rc.heap_stride + rc.heap_off[jj]};
    capk[k] = (int32_t)(rc.heap_off[jj + 1] - rc.heap_off[jj]) + kHS2;
  }
  __syncwarp();
  LaneErr le{INFINITY, HS_TRACE_OK, 0x7fffffff, -1};
  uint32_t n_steps = 0;
  int64_t rr_next = 0;
  bool failed = !tvalid;
  int32_t t_err = HS_TRACE_OK, t_err_inst = -1;
  int64_t t_err_req = -1;
  double t_err_val = 0.0;
  const bool eval_all = policy == HS_POLICY_OS || policy == HS_POLICY_MB;

  // trace error from the lanes' step errors: earliest (time, instance) wins
  auto step_error = [&]() -> bool {
    const bool mine = (h[0].fl & F_ERR) || (K > 1 && (h[K > 1 ? 1 : 0].fl & F_ERR)) ||
                      (K > 2 && (h[K > 2 ? 2 : 0].fl & F_ERR)) || (K > 3 && (h[K > 3 ? 3 : 0].fl & F_ERR));
    const unsigned gb = __ballot_sync(FULL, mine && !failed) & (0xffu << (grp * 8));
    if (!__any_sync(FULL, gb != 0)) return false;
    uint64_t key = mine ? okey(le.t) : ~0ull;
    int idx = mine ? le.inst : 0x7fffffff;
    group_min_key_idx(key, idx);
    const int src = __ffs(__ballot_sync(FULL, mine && le.inst == idx) & (0xffu << (grp * 8))) - 1;
    const int code = __shfl_sync(FULL, le.code, src < 0 ? lane : src);
    const int req = __shfl_sync(FULL, le.req, src < 0 ? lane : src);
    if (gb && !failed) {
      failed = true;
      t_err = code;
      t_err_inst = idx;
      t_err_req = req;
      t_err_val = from_okey(key);
    }
    return true;
  };

  uint64_t apack = 0;  // assignments of the current 8-arrival block (byte i = arrival base + i)
  int32_t bI = 0, bO = 0, bP = 0;
  double bT = 0.0;
  for (int64_t a = 0; a < qmax; ++a) {
    const int slot = (int)(a & 7);
    if (slot == 0) {
      if (progress) {
        // streamed inputs (host path): phase p is resident once *progress > p
        const int64_t last = (a + 7 < qmax ? a + 7 : qmax - 1);
        const uint32_t need = (uint32_t)(last / phase_len);
        int stalled = 0;
        if (lane == 0) {
          const long long t0 = clock64();
          uint32_t have;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(progress) : "memory");
          while (have <= need) {
            __nanosleep(256);
            if (clock64() - t0 > 20000000000ll) {
              stalled = 1;
              break;
            }
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(have) : "l"(progress) : "memory");
          }
        }
        if (__shfl_sync(FULL, stalled, 0)) {
          if (!failed) {
            failed = true;
            t_err = HS_TRACE_STALLED;
            t_err_req = a;
            t_err_inst = -1;
          }
          break;
        }
      }
      // lane l of the group holds arrival a + l of its trace
      const int64_t x = a + l;
      if (x < q) {  // L2-coherent loads: streamed inputs arrive while the kernel runs
        bI = __ldcg(c.I + x);
        bO = __ldcg(c.O + x);
        bP = __ldcg(P + x);
        bT = T ? __ldcg(T + x) : 0.0;
      }
    }
    const int src = (grp << 3) | slot;
    const int64_t Ia = __shfl_sync(FULL, bI, src);
    const int64_t Oa = __shfl_sync(FULL, bO, src);
    const int64_t Pa = __shfl_sync(FULL, bP, src);
    const double ta = shfl_d(bT, src);
    const bool act = !failed && a < q;

    // ---- advance every instance to the arrival (strictly earlier steps)
    if (act) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        advance(h[k], s_ist[wib][k][lane], heap[k], s_types[ty[k]], c, capk[k], l + kL * k, ta, false, n_steps,
                le);
    }
    step_error();
    const bool live = !failed && a < q;

    // ---- per-class price of this arrival (scheduling.py:119-147): lane l
    // prices class l (+8, +16, ...), the owners of each instance fetch theirs
    double cost[K];
#pragma unroll
    for (int k = 0; k < K; ++k) cost[k] = 1.0;
    if (policy != HS_POLICY_MB) {
      for (int base = 0; base < NT; base += kL) {  // NT is launch-uniform
        double v = 0.0;
        const int cl = base + l;
        if (live && cl < NT) {
          const TypeRec& ct = s_types[cl];
          const double fl = py_floordiv(ct.budget, i2d(pt * (Ia + Pa)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          const double tot = __dadd_rn(prefill_time(ct.p, b, Ia), decode_time(ct.p, b, Ia, Pa));
          v = (tot <= 0.0) ? -1.0 : __ddiv_rn(tot, i2d(b));
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int want = ty[k] - base;
          const double got = shfl_d(v, (grp << 3) | (want >= 0 && want < kL ? want : 0));
          if (want >= 0 && want < kL) cost[k] = got;
        }
      }
    }

    // ---- choose (scheduling.py:235-254)
    int chosen = -1;
    if (live && !eval_all) {
      if (policy == HS_POLICY_SI) {
        chosen = 0;
      } else if (policy == HS_POLICY_RR) {
        chosen = (int)(rr_next % N);
        rr_next += 1;
      }
    }
    if (policy == HS_POLICY_WRR) {  // smooth WRR: first strict maximum after adding the weights
      uint64_t key = 0;
      int idx = 0x7fffffff;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (live && (h[k].fl & F_VALID)) {
          IState& S = s_ist[wib][k][lane];
          S.wcur = __dadd_rn(S.wcur, rc.wrr_weight[l + kL * k]);
          const uint64_t wk = okey(S.wcur);
          if (wk > key) {
            key = wk;
            idx = l + kL * k;
          }
        }
      }
      group_max_key_idx(key, idx);
      chosen = live ? idx : -1;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (live && l + kL * k == chosen) {
          IState& S = s_ist[wib][k][lane];
          S.wcur = __dsub_rn(S.wcur, rc.wrr_total);
        }
    }
    // ---- evaluate (scheduling.py:216-233) on the instances that need it
    double w[K];
    int err_j = 0x7fffffff, err_code = 0;
    double err_val = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k] = INFINITY;
      const int j = l + kL * k;
      const bool need = live && (h[k].fl & F_VALID) && (eval_all || j == chosen);
      if (need) {
        IState& S = s_ist[wib][k][lane];
        if (h[k].fl & F_DIRTY) {  // capacity.py:98-106 kv_usage, scheduling.py:154 exp
          const TypeRec& t_ = s_types[ty[k]];
          const double usage = __ddiv_rn(i2d(pt * S.run_tot), t_.budget);
          bool of;
          S.ex = py_exp(__dmul_rn(theta, usage), s_tab, &of);
          h[k].fl = (h[k].fl & ~(F_DIRTY | F_EXOVER)) | (of ? F_EXOVER : 0u);
        }
        const bool cerr = cost[k] < 0.0, eerr = (h[k].fl & F_EXOVER) != 0;
        if ((cerr || eerr) && j < err_j) {  // the first instance in evaluation order raises
          err_j = j;
          err_code = cerr ? HS_TRACE_NONPOSITIVE_COST : HS_TRACE_EXP_OVERFLOW;
          if (cerr) {  // recompute the non-positive total for the message
            const TypeRec& t_ = s_types[ty[k]];
            const double fl = py_floordiv(t_.budget, i2d(pt * (Ia + Pa)));
            int64_t b = (int64_t)fl;
            if (b < 1) b = 1;
            err_val = __dadd_rn(prefill_time(t_.p, b, Ia), decode_time(t_.p, b, Ia, Pa));
          }
        }
        w[k] = __dmul_rn(cost[k], S.ex);
      }
    }
    {
      uint64_t ekey = (uint64_t)(uint32_t)err_j;
      int dummy = 0;
      group_min_key_idx(ekey, dummy);
      const int ej = (int)ekey;
      if (ej != 0x7fffffff) {
        const int own = (grp << 3) | (ej & 7);
        const int code = __shfl_sync(FULL, err_code, own);
        const double val = shfl_d(err_val, own);
        if (live) {
          failed = true;
          t_err = code;
          t_err_inst = ej;
          t_err_req = a;
          t_err_val = code == HS_TRACE_NONPOSITIVE_COST ? val : 0.0;
        }
      }
    }
    const bool go = live && !failed;
    if (eval_all) {
      // _min_max_choice (scheduling.py:299-312): argmin (lowest index) of
      // peak_s = max(L_s + w_s, max_j L_j) (w_s >= 0, rounding is monotone)
      uint64_t m1 = 0;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (h[k].fl & F_VALID) {
          const uint64_t lk = okey(h[k].load);
          m1 = lk > m1 ? lk : m1;
        }
      m1 = group_max_u64(m1);
      const double top = from_okey(m1);
      uint64_t pk = ~0ull;
      int pidx = 0x7fffffff;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double own = __dadd_rn(h[k].load, w[k]);
        const double peak = own > top ? own : top;
        const bool cand = go && (h[k].fl & F_VALID) && !isinf(w[k]) && peak < INFINITY;
        const uint64_t key = cand ? okey(peak) : ~0ull;
        if (key < pk) {
          pk = key;
          pidx = l + kL * k;
        }
      }
      group_min_key_idx(pk, pidx);
      if (go) {
        if (pk == ~0ull) {
          failed = true;
          t_err = HS_TRACE_NO_INSTANCE;
          t_err_req = a;
          t_err_inst = -1;
        } else {
          chosen = pidx;
        }
      }
    }

    // ---- commit (scheduling.py:335-346) and enqueue (simulator.py:323-327)
    if (live && !failed) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (l + kL * k != chosen) continue;
        IState& S = s_ist[wib][k][lane];
        Hot& hk = h[k];
        hk.load = __dadd_rn(hk.load, w[k]);
        S.run_tot += Ia + Pa;
        hk.fl |= F_DIRTY;
        // InstanceMetrics counts (simulator.py:338-341): every dispatched
        // request of a completed replay retires exactly once
        S.req_count += 1;
        S.tok_count += Ia + Oa;
        c.R[a].P = (int32_t)Pa;
        c.R[a].W = w[k];
        if (S.qhead < 0) {
          S.qhead = (int32_t)a;
          S.hI = (int32_t)Ia;
          S.hO = (int32_t)Oa;
          S.hP = (int32_t)Pa;
          S.hW = w[k];
          hk.fl &= ~F_BLOCKED;  // a new queue head may be admitted at the next step
        } else if (S.qtail == S.qhead) {  // the head's prefetched record gains its successor
          S.hnext = (int32_t)a;
          S.hnI = (int32_t)Ia;
          S.hnO = (int32_t)Oa;
          c.R[S.qtail].next = (int32_t)a;
        } else {
          QRec& tq = c.R[S.qtail];
          tq.next = (int32_t)a;
          tq.nI = (int32_t)Ia;
          tq.nO = (int32_t)Oa;
        }
        S.qtail = (int32_t)a;
        if (!(hk.fl & F_SCHED)) {
          hk.fl = (hk.fl | F_SCHED) & ~F_BLOCKED;
          hk.t_next = ta;
        }
      }
      apack |= (uint64_t)(uint8_t)chosen << (8 * slot);
    }
    // assignments leave in 8-byte words (one store per group per 8 arrivals)
    if (assign && l == 0 && (slot == 7 || a + 1 == q) && a < q) {
      const int64_t base = a - slot;
      uint8_t* dst = assign + o + base;
      const int nb = slot + 1;
      if (nb == 8 && ((uintptr_t)dst & 7) == 0 && !failed) {
        *reinterpret_cast<uint64_t*>(dst) = apack;
      } else {
        for (int b = 0; b < nb; ++b) dst[b] = (uint8_t)(apack >> (8 * b));
      }
    }
    if (slot == 7) apack = 0;
  }
  // drain: every remaining step
  if (!failed) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      advance(h[k], s_ist[wib][k][lane], heap[k], s_types[ty[k]], c, capk[k], l + kL * k, 0.0, true, n_steps, le);
  }
  step_error();

  if (tvalid) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = l + kL * k;
      if (!(h[k].fl & F_VALID)) continue;
      const IState& S = s_ist[wib][k][lane];
      hs_inst_metrics m;
      m.completion_time = S.completion;
      m.peak_kv_usage = S.max_res > 0 ? __ddiv_rn(i2d(pt * S.max_res), s_types[ty[k]].budget) : 0.0;
      m.residual_load = h[k].load;
      m.request_count = S.req_count;
      m.token_count = S.tok_count;
      metrics[tr * (int64_t)N + j] = m;
    }
  }
  int64_t steps_all = n_steps;
#pragma unroll
  for (int m = 4; m > 0; m >>= 1) steps_all += __shfl_xor_sync(FULL, steps_all, m);
  if (tvalid && l == 0) {
    hs_trace_result r;
    r.error = failed ? t_err : HS_TRACE_OK;
    r.err_instance = failed ? t_err_inst : -1;
    r.err_request = failed ? t_err_req : -1;
    r.err_value = failed ? t_err_val : 0.0;
    r.n_steps = steps_all;
    result[tr] = r;
  }
}

template <int K>
cudaError_t launch_k(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                     const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign, double* d_depart,
                     hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec, uint64_t* d_heap,
                     cudaStream_t st, const uint32_t* d_progress, int phase_len) {
  const size_t smem = mt_smem_fixed<K>() + (size_t)rc.n_types * sizeof(TypeRec);
  cudaError_t e = cudaFuncSetAttribute(k_replay_mt<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t per_block = (int64_t)kWPB * kG;
  const unsigned blocks = (unsigned)((n_traces + per_block - 1) / per_block);
  k_replay_mt<K><<<blocks, kWPB * 32, smem, st>>>(n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics,
                                                  d_result, static_cast<QRec*>(d_qrec), d_heap, d_progress,
                                                  phase_len, rc);
  return cudaGetLastError();
}

}  // namespace

bool replay_mt_eligible(const ReplayConst& rc, bool multi) {
  static const bool legacy = std::getenv("HS_REPLAY_LEGACY") != nullptr;
  return !legacy && !multi && rc.mode == 0 && rc.flags == 0 && rc.N >= 1 && rc.N <= kG * kL;
}

int replay_shared_heap(const ReplayConst& rc, bool multi) {
  return replay_mt_eligible(rc, multi) ? kHS2 : kHeapShared;
}

cudaError_t launch_replay_mt(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                             const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign,
                             double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec,
                             uint64_t* d_heap, cudaStream_t st, const uint32_t* d_progress, int phase_len) {
  if (n_traces <= 0) return cudaSuccess;
  const int K = (rc.N + kL - 1) / kL;
#define HS_LK(k) \
  launch_k<k>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics, d_result, d_qrec, d_heap, st, \
              d_progress, phase_len)
  switch (K) {
    case 1: return HS_LK(1);
    case 2: return HS_LK(2);
    case 3: return HS_LK(3);
    case 4: return HS_LK(4);
    default: return cudaErrorInvalidValue;
  }
#undef HS_LK
}

}  // namespace hs
