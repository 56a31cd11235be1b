// replay_mt.cu -- K3 without per-arrival stepping: event order from rigorous
// fp64 interval bounds, exact clocks recomputed in bulk from a segment log.
//
// Same results, bit for bit, as replay.cu (simulator.py:272-363
// run_continuous with scheduling.py:216-346 Scheduler.evaluate / choose /
// complete and the RR / WRR / SI / MB baselines); see replay.cu's header for
// why every instance may advance independently between arrivals.
//
// What an arrival at t_a needs from an instance is only which of its EVENT
// steps (a retirement, or an admission after a dispatch) happen before t_a:
// load and running tokens change at events only, and between two events the
// instance runs "pure" steps whose clock is t += price(cached length), with
// the batch fixed.  A retirement's step INDEX is known at admission
// (admission step + O, simulator.py:334), so the next event's index is known;
// only its TIME needs the serial fp64 sum of the pure steps' prices.  Instead
// of running that sum per arrival (per-instance step counts per arrival vary
// with the exponential arrival gaps and the instance speeds, so SIMT lanes
// idle), the kernel bounds it in O(1): with non-negative coefficients every
// price lies in [P(x)(1-u)^4, P(x)(1+u)^4] for the affine
// P(x) = (A + p7) x + (B + p8), and a chain of n additions of non-negative
// terms lies in [S(1-u)^n, S(1+u)^n] around the exact sum S (u = 2^-53);
// directed-rounding arithmetic evaluates both ends.  An event is due before
// t_a when the upper bound is below t_a and not due when the lower bound is at
// or above it; otherwise (a relative width of ~1e-13: practically never) the
// exact chain decides.  Every event appends a segment record (event step, its
// cost, the batch size, the cached length) to a per-instance ring in global
// memory, and the exact clock chains -- which the outputs need (departure and
// completion times) -- are rebuilt from the rings in bulk: every lane walks
// its instances' records with the pipelined four-step loop, all lanes at
// once, when a ring is half full and at the end of the trace.  The rounding
// order is the reference's throughout.
//
// Layout: a warp holds 32 / L traces, L lanes per trace, each lane owning
// instances j = lane + L * k (k < K): per arrival the lanes test event
// bounds, process their due events and take part in the dispatch reductions
// (log2 L shuffle levels inside the trace's lane group).
//
// Used, when HS_REPLAY_MT=1, for continuous mode, one deployment of <= 32
// instances, non-negative latency coefficients, no order keys.  Measured
// slower than replay.cu's kernel on config 4 (K3): the per-arrival
// event and dispatch work and the bulk catch-ups (whose lanes carry unequal
// pending steps) cost more than the per-arrival stepping they replace.  Kept
// opt-in and parity-tested (tests/test_gpu_replay_layouts.py).
#include <cstdlib>

#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {
namespace {

constexpr int kWPB = 2;    // warps per block
constexpr int kHS2 = 4;    // heap entries per instance in shared memory
constexpr int kRing = 16;  // segment records per instance
constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t NONE = 0xffffffffu;

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

// One event step of an instance: the exact clock chain is rebuilt from these.
enum : uint32_t { R_RESTART = 1, R_IDLE = 2 };
struct SegRec {
  uint32_t k;         // event step index
  int32_t first_ret;  // requests retiring at this step (linked through QRec.next when departures are wanted), -1 none
  uint32_t nact;      // batch size of the pure steps that follow (A = p5 * nact, B = p6 * nact)
  uint32_t flags;     // R_RESTART: the step starts a busy period at time t0; R_IDLE: last step of one
  double c_e;         // cost of this step: (0.0 + prefill) + decode
  double cd1;         // cached length of step k + 1
  double t0;          // R_RESTART: exact time of this step (the dispatch time)
};
static_assert(kRing * sizeof(SegRec) % sizeof(HEnt) == 0, "the rings live in the heap buffer");
constexpr int kRingEntries = (int)(kRing * sizeof(SegRec) / sizeof(HEnt));  // heap-buffer entries per instance

// Per-instance state in shared memory.
struct IState {
  double hW, topW, completion, ex, wcur, at;
  int64_t run_tot, reserved, cur_max, max_res, tok_count;
  uint64_t topkey;
  int32_t qhead, qtail, hI, hO, hP, hnext, hnI, hnO;
  int32_t nact, topI, topO, topP, req_count, cnt_max;
  uint32_t ak;     // anchor: T(ak) = at exactly, step ak's cost not yet added
  uint32_t ri;     // ring index of the record whose segment holds the anchor
  uint32_t rw;     // records written
  uint32_t kidle;  // step index the instance went idle at (its next busy period restarts there)
  uint32_t adone;  // the anchor sits on ring[ri].k with that record's outputs written
  int32_t ty;      // instance class
  int32_t _pad;
};

struct TypeRec {  // one instance class
  double p[8];
  double budget;
  int64_t cap_tok;  // floor(floor(budget) / per_token)
};

// Hot per-instance registers.
enum : uint32_t {
  F_VALID = 1, F_DIRTY = 2, F_EXOVER = 4, F_MAXDIRTY = 8, F_ERR = 16, F_RESTART = 32
};
struct Hot {
  double load;
  double Elo, Ehi;  // bounds of T(kn)
  double slo, shi;  // bounds of T(sk)
  double sce;       // cost of step sk
  double sA, sB;    // p5 * nact, p6 * nact of the segment's pure steps
  double scd;       // cached length of step sk + 1
  uint32_t sk, kn;  // segment start (an event step) and the next event step (NONE: idle)
  uint32_t fl;
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
// lane-group reductions (xor offsets below L stay inside the group); every lane takes part
template <int L>
__device__ __forceinline__ uint64_t group_max_u64(uint64_t v) {
#pragma unroll
  for (int m = L / 2; m > 0; m >>= 1) {
    const uint64_t o = shfl_xor_u64(v, m);
    v = o > v ? o : v;
  }
  return v;
}
template <int L>
__device__ __forceinline__ void group_min_key_idx(uint64_t& key, int& idx) {  // ties: lowest idx
#pragma unroll
  for (int m = L / 2; m > 0; m >>= 1) {
    const uint64_t ok = shfl_xor_u64(key, m);
    const int oi = __shfl_xor_sync(FULL, idx, m);
    if (ok < key || (ok == key && oi < idx)) {
      key = ok;
      idx = oi;
    }
  }
}
template <int L>
__device__ __forceinline__ void group_max_key_idx(uint64_t& key, int& idx) {  // ties: lowest idx
#pragma unroll
  for (int m = L / 2; m > 0; m >>= 1) {
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
  double wscale;  // diagnostic: widens the bounds (HS_REPLAY_WIDEN) to exercise the exact paths
};

// ---------------------------------------------------------------- bounds
// Bounds of T(sk + 1 + n): T(sk) in [slo, shi], then sce, then n pure steps
// priced at cached lengths scd, scd + 1, ...  All terms are >= 0.
__device__ __forceinline__ void seg_bounds(const Hot& h, double p7, double p8, double wscale, uint32_t n, double& L,
                                           double& U) {
  const double dn = (double)n;
  const double tri_lo = __dmul_rd(__dmul_rd(dn, __dsub_rd(dn, 1.0)), 0.5);
  const double tri_hi = __dmul_ru(__dmul_ru(dn, __dsub_ru(dn, 1.0)), 0.5);
  const double sx_lo = __dadd_rd(__dmul_rd(dn, h.scd), tri_lo);
  const double sx_hi = __dadd_ru(__dmul_ru(dn, h.scd), tri_hi);
  const double S_lo = __dadd_rd(__dmul_rd(__dadd_rd(h.sA, p7), sx_lo), __dmul_rd(dn, __dadd_rd(h.sB, p8)));
  const double S_hi = __dadd_ru(__dmul_ru(__dadd_ru(h.sA, p7), sx_hi), __dmul_ru(dn, __dadd_ru(h.sB, p8)));
  // each price within a factor (1 -+ u)^4 of its affine value; n + 1 chain additions
  const double m = __dmul_ru(dn + 2.0, 0x1p-53 * wscale);
  L = __dmul_rd(__dadd_rd(__dadd_rd(h.slo, h.sce), __dmul_rd(S_lo, 1.0 - 0x1p-50 * wscale)), __dsub_rd(1.0, m));
  U = __dmul_ru(__dadd_ru(__dadd_ru(h.shi, h.sce), __dmul_ru(S_hi, 1.0 + 0x1p-49 * wscale)),
                __dadd_ru(1.0, __dmul_ru(2.0, m)));
}

// ------------------------------------------------------- exact clock chain
// Walk one instance's exact clock chain forward from its anchor through its
// ring's segment records (the reference's rounding order: t = t + cost, step
// by step), writing departure / completion times at retiring steps.
//   TO_STEP: stop at step kt;  TO_TIME: stop at the first step after sk whose
//   time is >= t_target;  ALL: stop at the last record's event step.
enum CatchMode { TO_STEP = 0, TO_TIME = 1, ALL = 2 };
__device__ __noinline__ void catch_up(IState& S, uint32_t sk, const SegRec* ring, const TypeRec& tr, const Ctx& c,
                                      int mode, uint32_t kt, double t_target, uint32_t* k_out, double* t_out) {
  const double p5 = tr.p[4], p6 = tr.p[5], p7 = tr.p[6], p8 = tr.p[7];
  uint32_t r = S.ri;
  uint32_t k = S.ak;
  double t = S.at;
  bool at_event_done = S.adone != 0;  // anchor on ring[r].k, its outputs written
  const uint32_t rw = S.rw;
  const bool by_time = mode == TO_TIME;
  for (;;) {
    const SegRec rec = ring[r % kRing];
    if (k == rec.k) {
      if (!at_event_done) {
        if (rec.flags & R_RESTART) t = rec.t0;
        if (rec.first_ret >= 0) {
          S.completion = t;
          if (c.DEP)
            for (int32_t x = rec.first_ret; x >= 0; x = c.R[x].next) c.DEP[x] = t;
        }
        at_event_done = true;
      }
      if (mode == TO_STEP && k == kt) break;
      if (mode == ALL && r + 1 == rw) break;
      if (rec.flags & R_IDLE) {  // no step follows: the next record restarts at the same index
        if (r + 1 == rw) break;
        ++r;
        at_event_done = false;
        continue;
      }
      if (by_time && t >= t_target && k > sk) break;
      t = __dadd_rn(t, rec.c_e);
      k += 1;
      at_event_done = false;
    }
    // pure steps of this segment, up to the next record's event step
    const uint32_t kend = (r + 1 < rw) ? ring[(r + 1) % kRing].k : NONE;
    uint32_t stop = kend;
    if (mode == TO_STEP && kt < stop) stop = kt;
    if (k < stop && !(by_time && t >= t_target && k > sk)) {
      const double dnact = (double)rec.nact;
      const double A = __dmul_rn(p5, dnact), B = __dmul_rn(p6, dnact);
      auto price = [&](double x) {
        return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, x), B), __dmul_rn(p7, x)), p8);
      };
      double cd = __dadd_rn(rec.cd1, (double)(k - rec.k - 1));
      double c0 = price(cd), c1 = price(__dadd_rn(cd, 1.0)), c2 = price(__dadd_rn(cd, 2.0)),
             c3 = price(__dadd_rn(cd, 3.0));
      for (;;) {
        // step k (time t) costs c0: step k + 1 is at t1, ...
        const double t1 = __dadd_rn(t, c0);
        const double t2 = __dadd_rn(t1, c1);
        const double t3 = __dadd_rn(t2, c2);
        const double t4 = __dadd_rn(t3, c3);
        const double cd4 = __dadd_rn(cd, 4.0);
        const double n0 = price(cd4), n1 = price(__dadd_rn(cd, 5.0)), n2 = price(__dadd_rn(cd, 6.0)),
                     n3 = price(__dadd_rn(cd, 7.0));
        // step k + i is reached while k + i <= stop and, by time, the chain
        // stops at the first step whose time reaches the target
        const bool g1 = k + 1 <= stop && !(by_time && t1 >= t_target);
        const bool g2 = g1 && k + 2 <= stop && !(by_time && t2 >= t_target);
        const bool g3 = g2 && k + 3 <= stop && !(by_time && t3 >= t_target);
        const bool g4 = g3 && k + 4 <= stop && !(by_time && t4 >= t_target);
        if (!g4 || k + 4 == stop) {
          uint32_t n;
          double tn;
          if (g4) {
            n = 4;
            tn = t4;
          } else if (!g1) {  // k + 1 > stop is excluded above: step k + 1 reaches the target
            n = 1;
            tn = t1;
          } else if (!g2) {
            n = (k + 2 > stop) ? 1 : 2;
            tn = (k + 2 > stop) ? t1 : t2;
          } else if (!g3) {
            n = (k + 3 > stop) ? 2 : 3;
            tn = (k + 3 > stop) ? t2 : t3;
          } else {
            n = (k + 4 > stop) ? 3 : 4;
            tn = (k + 4 > stop) ? t3 : t4;
          }
          k += n;
          t = tn;
          break;
        }
        t = t4;
        cd = cd4;
        k += 4;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
      }
    }
    if (mode == TO_STEP && k == kt) break;
    if (by_time && t >= t_target && k > sk) break;
    if (k == kend) {  // the next record's event step
      ++r;
      at_event_done = false;
      continue;
    }
    break;
  }
  S.ri = r;
  S.ak = k;
  S.at = t;
  S.adone = (k == ring[r % kRing].k && at_event_done) ? 1u : 0u;
  if (k_out) *k_out = k;
  if (t_out) *t_out = t;
}

// Every lane brings its instances' exact chains up to their last records in
// ONE flattened loop: each iteration is a block of up to four pure steps or
// one record boundary of the lane's current instance, so the warp pays for
// the longest lane's total, not for the longest segment of every record in
// turn; the next record is loaded while the current segment's steps run.
template <int L, int K>
__device__ __forceinline__ void bulk_catch_up(IState* sl /* this lane's IState, slot stride 32 */,
                                              const SegRec* ring0 /* instance j's ring: ring0 + j * kRing */,
                                              const TypeRec* types, const Ctx& c, int l, unsigned valid_mask) {
  int slot = -1;
  IState* S = nullptr;
  const SegRec* ring = nullptr;
  uint32_t r = 0, rw = 0, k = 0, stop = 0;
  double t = 0.0, cd = 0.0, A = 0.0, B = 0.0, p7 = 0.0, p8 = 0.0;
  int phase = 0;  // 0: at ring[r].k, outputs pending; 1: at ring[r].k, outputs written; 2: pure steps
  SegRec rec, nrec;
  auto load_seg = [&]() {  // pure steps of record r, up to nrec.k
    const TypeRec& tr = types[S->ty];
    const double dn = (double)rec.nact;
    A = __dmul_rn(tr.p[4], dn);
    B = __dmul_rn(tr.p[5], dn);
    p7 = tr.p[6];
    p8 = tr.p[7];
    cd = __dadd_rn(rec.cd1, (double)(k - rec.k - 1));
    nrec = ring[(r + 1) % kRing];
    stop = nrec.k;
  };
  auto next_instance = [&]() -> bool {
    for (++slot; slot < K; ++slot) {
      if (!((valid_mask >> slot) & 1u)) continue;
      S = sl + slot * 32;
      rw = S->rw;
      if (rw == 0) continue;
      r = S->ri;
      k = S->ak;
      t = S->at;
      ring = ring0 + (int64_t)(l + L * slot) * kRing;
      rec = ring[r % kRing];
      if (k == rec.k) {
        phase = S->adone ? 1 : 0;
        if (phase == 1 && r + 1 == rw) continue;  // already at the last record
      } else {
        if (r + 1 == rw) continue;  // past the last record's event step
        phase = 2;
        load_seg();
      }
      return true;
    }
    return false;
  };
  bool active = next_instance();
  while (__any_sync(FULL, active)) {
    if (!active) continue;
    if (phase == 2) {
      // a block of up to four pure steps (the reference's order: t = t + price)
      const uint32_t n = (stop - k) < 4u ? (stop - k) : 4u;
      const auto price = [&](double x) {
        return __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, x), B), __dmul_rn(p7, x)), p8);
      };
      const double c0 = price(cd), c1 = price(__dadd_rn(cd, 1.0)), c2 = price(__dadd_rn(cd, 2.0)),
                   c3 = price(__dadd_rn(cd, 3.0));
      const double t1 = __dadd_rn(t, c0);
      const double t2 = __dadd_rn(t1, c1);
      const double t3 = __dadd_rn(t2, c2);
      const double t4 = __dadd_rn(t3, c3);
      t = n == 4 ? t4 : (n == 3 ? t3 : (n == 2 ? t2 : t1));
      cd = __dadd_rn(cd, (double)n);
      k += n;
      if (k == stop) {  // the next record's event step
        ++r;
        rec = nrec;
        phase = 0;
      }
      continue;
    }
    if (phase == 0) {  // event step: outputs at its exact time
      if (rec.flags & R_RESTART) t = rec.t0;
      if (rec.first_ret >= 0) {
        S->completion = t;
        if (c.DEP)
          for (int32_t x = rec.first_ret; x >= 0; x = c.R[x].next) c.DEP[x] = t;
      }
      phase = 1;
    }
    // phase 1: leave the event step
    if (r + 1 == rw) {  // the last record: anchor here, next instance
      S->ri = r;
      S->ak = k;
      S->at = t;
      S->adone = 1u;
      active = next_instance();
      continue;
    }
    if (rec.flags & R_IDLE) {  // the next record restarts at the same step index
      ++r;
      rec = ring[r % kRing];
      phase = 0;
      continue;
    }
    t = __dadd_rn(t, rec.c_e);
    k += 1;
    load_seg();
    phase = 2;
    if (k == stop) {
      ++r;
      rec = nrec;
      phase = 0;
    }
  }
}

// ----------------------------------------------------------------- events
// The STEP event of one instance at step h.kn (simulator.py:330-355):
// retirements due at this step (admission order), FCFS admission, prefill
// for newcomers, one decode iteration -- as replay.cu's event_step, with the
// step's time known within [Elo, Ehi]; appends the step's segment record.
__device__ __forceinline__ void event(Hot& h, IState& S, const Heap& heap, SegRec* ring, const TypeRec& tr,
                                      const Ctx& c, int32_t cap, int j, uint32_t& n_steps, LaneErr& le) {
  const uint32_t ke = h.kn;
  const bool restart = (h.fl & F_RESTART) != 0;
  n_steps += restart ? 1u : ke - h.sk;
  if (S.rw - S.ri >= (uint32_t)kRing)  // ring full (rare: the arrival loop drains the rings early)
    catch_up(S, h.sk, ring, tr, c, ALL, 0, 0.0, nullptr, nullptr);
  int32_t nact = S.nact;
  uint64_t topkey = S.topkey;
  int64_t reserved = S.reserved, run_tot = S.run_tot, cur_max = S.cur_max;
  int32_t cnt_max = S.cnt_max;
  bool max_dirty = (h.fl & F_MAXDIRTY) != 0;
  int32_t first_ret = -1;
  while (nact > 0 && (uint32_t)(topkey >> 32) == ke) {
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
    if (c.DEP) c.R[r].next = first_ret;  // departure chain of this step (the queue link is dead)
    first_ret = r;
    h.load = __dsub_rn(h.load, wr);  // Scheduler.complete: the recorded values
    run_tot -= Ir + Pr;
    const int64_t ka = (int64_t)ke - (Or > 1 ? Or : 1);
    if (Ir - ka == cur_max && --cnt_max == 0) max_dirty = true;
  }
  if (first_ret >= 0) h.fl |= F_DIRTY;
  if (nact == 0) {
    cur_max = INT64_MIN;
    cnt_max = 0;
    max_dirty = false;
  }
  // admit FCFS (simulator.py:297-316)
  int64_t newly = 0, max_i_new = 0;
  int32_t qhead = S.qhead;
  int32_t fail = 0, fail_req = -1;
  while (qhead >= 0) {
    const int64_t need = (int64_t)S.hI + S.hO;
    // simulator.py:303 per_token * (reserved + need) > budget, exactly
    if (reserved + need > tr.cap_tok) {
      if (nact == 0 && newly == 0) {
        fail = HS_TRACE_INFEASIBLE_REQUEST;
        fail_req = qhead;
      }
      break;
    }
    if (nact >= cap || ke > 0x7fffffffu) {
      fail = HS_TRACE_CAPACITY;
      fail_req = qhead;
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
    const uint64_t key = ((uint64_t)(ke + (uint32_t)(Or > 1 ? Or : 1)) << 32) | (uint32_t)r;
    if (nact == 0 || key < topkey) {
      topkey = key;
      S.topI = (int32_t)Ir;
      S.topO = (int32_t)Or;
      S.topP = (int32_t)Pr;
      S.topW = wr;
    }
    const int64_t mk = Ir - (int64_t)ke;
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
  // simulator.py:315: the max of the quotients is the quotient of the max reservation
  if (newly && reserved > S.max_res) S.max_res = reserved;
  SegRec rec;
  rec.k = ke;
  rec.first_ret = first_ret;
  rec.flags = restart ? R_RESTART : 0u;
  rec.t0 = restart ? h.Elo : 0.0;
  h.fl &= ~F_RESTART;
  if (!fail && nact > 0) {
    double cst = 0.0;
    if (newly) cst = __dadd_rn(cst, prefill_time(tr.p, newly, max_i_new));
    if (max_dirty || cnt_max <= 0) {  // the last holder of the max retired: rescan
      int64_t m = INT64_MIN;
      int32_t cm = 0;
      for (int32_t x = 0; x < nact; ++x) {
        const int64_t mk = heap.get(x, nact).mk;
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
    const double A = __dmul_rn(tr.p[4], db), B = __dmul_rn(tr.p[5], db);
    const double cd = i2d(cur_max + (int64_t)ke + 1);
    // decode_iteration_time(cached, batch) = ((A*c + B) + p7*c) + p8
    const double dec = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, cd), B), __dmul_rn(tr.p[6], cd)), tr.p[7]);
    cst = __dadd_rn(cst, dec);
    rec.nact = (uint32_t)nact;
    rec.c_e = cst;
    rec.cd1 = __dadd_rn(cd, 1.0);
    // the new segment starts at ke; the next event is the heap minimum's step
    h.slo = h.Elo;
    h.shi = h.Ehi;
    h.sce = cst;
    h.sA = A;
    h.sB = B;
    h.scd = rec.cd1;
    h.sk = ke;
    h.kn = (uint32_t)(topkey >> 32);
    seg_bounds(h, tr.p[6], tr.p[7], c.wscale, h.kn - ke - 1, h.Elo, h.Ehi);
  } else {
    rec.nact = 0;
    rec.c_e = 0.0;
    rec.cd1 = 0.0;
    rec.flags |= R_IDLE;
    h.sk = ke;
    h.kn = NONE;  // idle until the next dispatch (simulator.py:344-345)
    S.kidle = ke;
  }
  ring[S.rw % kRing] = rec;
  S.rw += 1;
  if (max_dirty) h.fl |= F_MAXDIRTY;
  else h.fl &= ~F_MAXDIRTY;
  S.nact = nact;
  S.topkey = topkey;
  S.reserved = reserved;
  S.run_tot = run_tot;
  S.cur_max = cur_max;
  S.cnt_max = cnt_max;
  if (fail) {  // the failing step's exact time orders errors across instances
    h.kn = NONE;
    double tf;
    catch_up(S, h.sk, ring, tr, c, TO_STEP, ke, 0.0, nullptr, &tf);
    if (tf < le.t || (tf == le.t && j < le.inst)) le = LaneErr{tf, fail, j, fail_req};
    h.fl |= F_ERR;
  }
}

// Process every event of one instance before t_a (every event when
// draining); returns true when the next one's order against t_a is
// undecided by the bounds (the caller resolves it exactly).
__device__ __forceinline__ bool events_before(Hot& h, IState& S, const Heap& heap, SegRec* ring, const TypeRec& tr,
                                              const Ctx& c, int32_t cap, int j, double t_a, bool drain,
                                              uint32_t& n_steps, LaneErr& le) {
  while ((h.fl & (F_VALID | F_ERR)) == F_VALID && h.kn != NONE) {
    if (drain || h.Ehi < t_a) {
      event(h, S, heap, ring, tr, c, cap, j, n_steps, le);
      continue;
    }
    return !(h.Elo >= t_a);
  }
  return false;
}

// The exact time of the pending event decides its order against t_a.  The
// anchor is put back afterwards: a dispatch may still need the exact chain
// from before that step (the first step at or after t_a, admission_step).
__device__ __forceinline__ void resolve_exact(Hot& h, IState& S, SegRec* ring, const TypeRec& tr, const Ctx& c) {
  const uint32_t ak = S.ak, ri = S.ri, adone = S.adone;
  const double at = S.at;
  double t;
  catch_up(S, h.sk, ring, tr, c, TO_STEP, h.kn, 0.0, nullptr, &t);
  S.ak = ak;
  S.ri = ri;
  S.adone = adone;
  S.at = at;
  h.Elo = t;
  h.Ehi = t;
}

// Dispatch to a busy instance whose queue was empty and whose new head fits:
// it is admitted at the first step at or after t_a (arrivals pop before steps
// at equal times), which becomes the next event when it precedes the pending
// retirement.  T(sk) < t_a <= T(kn), so that step is sk + 1 + n, n <= nmax.
__device__ __forceinline__ void admission_step(Hot& h, IState& S, SegRec* ring, const TypeRec& tr, const Ctx& c,
                                               double t_a) {
  const double p7 = tr.p[6], p8 = tr.p[7];
  const uint32_t nmax = h.kn - h.sk - 1;
  uint32_t lo = 0, hi = nmax;
  {
    // closed-form guess from the midpoint of the affine sum:
    // T(sk + 1 + n) ~ T(sk) + sce + a (n scd + n (n - 1) / 2) + b n
    const double a = h.sA + p7, b = h.sB + p8;
    const double c0 = 0.5 * (h.slo + h.shi) + h.sce - t_a;  // < 0 here
    const double B1 = a * (h.scd - 0.5) + b;
    double g = nmax;
    if (a > 0.0) g = (-B1 + sqrt(B1 * B1 - 2.0 * a * c0)) / a;
    else if (B1 > 0.0) g = -c0 / B1;
    if (!(g >= 0.0)) g = 0.0;
    uint32_t n = g >= (double)nmax ? nmax : (uint32_t)ceil(g);
    // narrow [lo, hi] around the guess with the rigorous bounds
    for (int it = 0; it < 3 && lo < hi; ++it) {
      double L, U;
      seg_bounds(h, p7, p8, c.wscale, n, L, U);
      if (L >= t_a) {
        hi = n;
        if (n == 0) break;
        seg_bounds(h, p7, p8, c.wscale, n - 1, L, U);
        if (U < t_a) {
          lo = n;
          break;
        }
        n = n - 1;
      } else {
        lo = n + 1;
        n = lo < nmax ? lo : nmax;
      }
    }
  }
  while (lo < hi) {  // smallest n whose lower bound reaches t_a (nmax: known to)
    const uint32_t mid = lo + ((hi - lo) >> 1);
    double L, U;
    seg_bounds(h, p7, p8, c.wscale, mid, L, U);
    if (L >= t_a) hi = mid;
    else lo = mid + 1;
  }
  bool ok = true;
  double mlo = h.Elo, mhi = h.Ehi;
  if (lo < nmax) {
    seg_bounds(h, p7, p8, c.wscale, lo, mlo, mhi);
    ok = mlo >= t_a;
  }
  if (ok && lo > 0) {
    double L, U;
    seg_bounds(h, p7, p8, c.wscale, lo - 1, L, U);
    ok = U < t_a;
  }
  if (ok) {
    if (lo == nmax) return;  // the pending event's step itself
    h.kn = h.sk + 1 + lo;
    h.Elo = mlo;
    h.Ehi = mhi;
    return;
  }
  // undecided by the bounds: walk the exact chain to the first step at/after t_a
  uint32_t m;
  double t;
  catch_up(S, h.sk, ring, tr, c, TO_TIME, 0, t_a, &m, &t);
  if (m >= h.kn) {  // the pending event's step (its exact time is now known)
    h.Elo = t;
    h.Ehi = t;
    return;
  }
  h.kn = m;
  h.Elo = t;
  h.Ehi = t;
}

// shared memory per block: [IState kWPB*K*32][HEnt kWPB*K*32*kHS2][TypeRec n_types][prices kWPB*32*n_types]
template <int K>
__host__ __device__ constexpr size_t mt_smem_fixed() {
  return sizeof(IState) * kWPB * K * 32 + sizeof(HEnt) * kWPB * K * 32 * kHS2;
}
__host__ __device__ inline size_t mt_smem_types(int n_types) { return sizeof(TypeRec) * (size_t)n_types; }

template <int L, int K>
__global__ void __launch_bounds__(kWPB * 32, 1) k_replay_mt(
    int64_t n_traces, const int64_t* __restrict__ off, const int32_t* __restrict__ gI, const int32_t* __restrict__ gO,
    const int32_t* __restrict__ gP, const double* __restrict__ gT, uint8_t* __restrict__ assign,
    double* __restrict__ depart, hs_inst_metrics* __restrict__ metrics, hs_trace_result* __restrict__ result,
    QRec* __restrict__ qrec_all, uint64_t* __restrict__ heap_all, const uint32_t* progress, int32_t phase_len,
    double wscale, const __grid_constant__ ReplayConst rc) {
  constexpr int G = 32 / L;  // traces per warp
  __shared__ uint64_t s_tab[256];
  extern __shared__ double4 s_dyn[];
  IState(*s_ist)[K][32] = reinterpret_cast<IState(*)[K][32]>(s_dyn);
  HEnt(*s_heap)[K][32][kHS2] =
      reinterpret_cast<HEnt(*)[K][32][kHS2]>(reinterpret_cast<char*>(s_dyn) + sizeof(IState) * kWPB * K * 32);
  TypeRec* s_types = reinterpret_cast<TypeRec*>(reinterpret_cast<char*>(s_dyn) + mt_smem_fixed<K>());
  const int NT = rc.n_types;
  // per-(arrival, class) prices of the current block of L arrivals: [warp][lane = arrival slot][class]
  double* s_price = reinterpret_cast<double*>(reinterpret_cast<char*>(s_types) + mt_smem_types(NT));
  for (int x = threadIdx.x; x < 256; x += blockDim.x) s_tab[x] = kExpTab[x];
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
  const int grp = lane / L;  // trace group within the warp
  const int l = lane % L;    // lane within the group
  const int gbase = grp * L;
  const int64_t warp_global = (int64_t)blockIdx.x * kWPB + wib;
  const int64_t tr_raw = warp_global * G + grp;
  if (warp_global * G >= n_traces) return;  // whole warp idle
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
  for (int m = L; m < 32; m <<= 1) {
    const int64_t oq = __shfl_xor_sync(FULL, (long long)qmax, m);
    qmax = oq > qmax ? oq : qmax;
  }
  const Ctx c{gI + o, gO + o, qrec_all + o, depart ? depart + o : nullptr, pt, wscale};
  const int32_t* P = gP + o;
  const double* T = gT ? gT + o : nullptr;

  Hot h[K];
  int ty[K];
  int32_t capk[K];
  Heap heap[K];
  SegRec* ring[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = l + L * k;
    const bool v = tvalid && j < N;
    ty[k] = v ? rc.inst_type[j] : 0;
    h[k] = Hot{};
    h[k].kn = NONE;
    h[k].fl = v ? (F_VALID | F_DIRTY) : 0u;
    IState& S = s_ist[wib][k][lane];
    S = IState{};
    S.ex = 1.0;
    S.cur_max = INT64_MIN;
    S.qhead = -1;
    S.qtail = -1;
    S.ty = ty[k];
    const int jj = v ? j : 0;
    HEnt* base = reinterpret_cast<HEnt*>(heap_all) + tr * rc.heap_stride;
    heap[k] = Heap{s_heap[wib][k][lane], base + rc.heap_off[jj]};
    capk[k] = (int32_t)(rc.heap_off[jj + 1] - rc.heap_off[jj]) + kHS2;
    ring[k] = reinterpret_cast<SegRec*>(base + rc.heap_off[N] + (int64_t)jj * kRingEntries);
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
  const unsigned gmask = (L == 32 ? FULL : (((1u << L) - 1u) << gbase));

  // trace error from the lanes' step errors: earliest (time, instance) wins
  auto step_error = [&]() {
    bool mine = false;
#pragma unroll
    for (int k = 0; k < K; ++k) mine |= (h[k].fl & F_ERR) != 0;
    if (!__any_sync(FULL, mine && !failed)) return;
    uint64_t key = mine ? okey(le.t) : ~0ull;
    int idx = mine ? le.inst : 0x7fffffff;
    group_min_key_idx<L>(key, idx);
    const unsigned sb = __ballot_sync(FULL, mine && le.inst == idx) & gmask;
    const int src = sb ? __ffs(sb) - 1 : lane;
    const int code = __shfl_sync(FULL, le.code, src);
    const int req = __shfl_sync(FULL, le.req, src);
    if ((__ballot_sync(FULL, mine) & gmask) && !failed) {
      failed = true;
      t_err = code;
      t_err_inst = idx;
      t_err_req = req;
      t_err_val = from_okey(key);
    }
  };
  // every lane brings its instances' exact chains up to their last records
  unsigned valid_mask = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) valid_mask |= (h[k].fl & F_VALID) ? (1u << k) : 0u;
  const SegRec* ring0 = reinterpret_cast<const SegRec*>(reinterpret_cast<HEnt*>(heap_all) + tr * rc.heap_stride +
                                                        rc.heap_off[N]);
  auto drain_rings = [&]() { bulk_catch_up<L, K>(&s_ist[wib][0][lane], ring0, s_types, c, l, valid_mask); };
  // all events before t_a (or all events), undecided ones resolved exactly
  auto process_events = [&](double t_a, bool drain) {
    for (;;) {
      unsigned amb = 0;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (events_before(h[k], s_ist[wib][k][lane], heap[k], ring[k], s_types[ty[k]], c, capk[k], l + L * k, t_a,
                          drain, n_steps, le))
          amb |= 1u << k;
      if (!amb) break;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (amb >> k & 1u) resolve_exact(h[k], s_ist[wib][k][lane], ring[k], s_types[ty[k]], c);
    }
  };

  uint64_t apack = 0;  // assignments of the current 8-arrival block (byte i = arrival base + i)
  int32_t bI = 0, bO = 0, bP = 0;
  double bT = 0.0;
  for (int64_t a = 0; a < qmax; ++a) {
    const int slot = (int)(a % L);
    if (slot == 0) {
      if (progress) {
        // streamed inputs (host path): phase p is resident once *progress > p
        const int64_t last = (a + L - 1 < qmax ? a + L - 1 : qmax - 1);
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
      // price (arrival, class) pairs of the block (scheduling.py:119-147): the
      // state-independent part of the workload, one arrival per lane
      if (policy != HS_POLICY_MB && !failed && x < q) {
        double* pr = s_price + (size_t)(wib * 32 + lane) * NT;
        for (int cl = 0; cl < NT; ++cl) {
          const TypeRec& ct = s_types[cl];
          const double fl = py_floordiv(ct.budget, i2d(pt * ((int64_t)bI + bP)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          const double tot = __dadd_rn(prefill_time(ct.p, b, bI), decode_time(ct.p, b, bI, bP));
          pr[cl] = (tot <= 0.0) ? -1.0 : __ddiv_rn(tot, i2d(b));
        }
      }
      __syncwarp();
    }
    {  // keep room in every ring: the exact chains are rebuilt in bulk
      bool full = false;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const IState& S = s_ist[wib][k][lane];
        full |= S.rw - S.ri >= (uint32_t)(kRing - 4);
      }
      if (__any_sync(FULL, full)) drain_rings();
    }
    const int src = gbase | slot;
    const int64_t Ia = __shfl_sync(FULL, bI, src);
    const int64_t Oa = __shfl_sync(FULL, bO, src);
    const int64_t Pa = __shfl_sync(FULL, bP, src);
    const double ta = shfl_d(bT, src);

    // ---- every event before the arrival (steps strictly earlier)
    if (!failed && a < q) process_events(ta, false);
    step_error();
    const bool live = !failed && a < q;

    // ---- this arrival's price for each instance's class (computed per block)
    double cost[K];
    const double* prow = s_price + (size_t)(wib * 32 + src) * NT;
#pragma unroll
    for (int k = 0; k < K; ++k) cost[k] = (policy != HS_POLICY_MB && live) ? prow[ty[k]] : 1.0;

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
          S.wcur = __dadd_rn(S.wcur, rc.wrr_weight[l + L * k]);
          const uint64_t wk = okey(S.wcur);
          if (wk > key) {
            key = wk;
            idx = l + L * k;
          }
        }
      }
      group_max_key_idx<L>(key, idx);
      chosen = live ? idx : -1;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (live && l + L * k == chosen) {
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
      const int j = l + L * k;
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
      group_min_key_idx<L>(ekey, dummy);
      const int ej = (int)ekey;
      if (ej != 0x7fffffff) {
        const int own = gbase | (ej % L);
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
      m1 = group_max_u64<L>(m1);
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
          pidx = l + L * k;
        }
      }
      group_min_key_idx<L>(pk, pidx);
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
        if (l + L * k != chosen) continue;
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
        const bool was_empty = S.qhead < 0;
        if (was_empty) {
          S.qhead = (int32_t)a;
          S.hI = (int32_t)Ia;
          S.hO = (int32_t)Oa;
          S.hP = (int32_t)Pa;
          S.hW = w[k];
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
        if (hk.kn == NONE) {
          // idle: a busy period starts with a step at exactly t_a
          // (schedule_step(idx, t), simulator.py:292-295)
          hk.kn = S.kidle;
          hk.Elo = ta;
          hk.Ehi = ta;
          hk.fl |= F_RESTART;
        } else if (was_empty && S.reserved + Ia + Oa <= s_types[ty[k]].cap_tok) {
          // a head that does not fit waits for a retirement: no new event
          admission_step(hk, S, ring[k], s_types[ty[k]], c, ta);
        }
      }
      apack |= (uint64_t)(uint8_t)chosen << (8 * (a & 7));
    }
    // assignments leave in 8-byte words (one store per group per 8 arrivals)
    if (assign && l == 0 && ((a & 7) == 7 || a + 1 == q) && a < q) {
      const int64_t base = a - (a & 7);
      uint8_t* dst = assign + o + base;
      const int nb = (int)(a & 7) + 1;
      if (nb == 8 && ((uintptr_t)dst & 7) == 0) {
        *reinterpret_cast<uint64_t*>(dst) = apack;
      } else {
        for (int b = 0; b < nb; ++b) dst[b] = (uint8_t)(apack >> (8 * b));
      }
    }
    if ((a & 7) == 7) apack = 0;
  }
  // drain: every remaining event, then every exact chain
  if (!failed) process_events(0.0, true);
  step_error();
  drain_rings();

  if (tvalid) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int j = l + L * k;
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
  for (int m = L / 2; m > 0; m >>= 1) steps_all += __shfl_xor_sync(FULL, steps_all, m);
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

template <int L, int K>
cudaError_t launch_k(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                     const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign, double* d_depart,
                     hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec, uint64_t* d_heap,
                     cudaStream_t st, const uint32_t* d_progress, int phase_len, double wscale) {
  const size_t smem = mt_smem_fixed<K>() + mt_smem_types(rc.n_types) + sizeof(double) * kWPB * 32 * rc.n_types;
  cudaError_t e = cudaFuncSetAttribute(k_replay_mt<L, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t per_block = (int64_t)kWPB * (32 / L);
  const unsigned blocks = (unsigned)((n_traces + per_block - 1) / per_block);
  k_replay_mt<L, K><<<blocks, kWPB * 32, smem, st>>>(n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart,
                                                     d_metrics, d_result, static_cast<QRec*>(d_qrec), d_heap,
                                                     d_progress, phase_len, wscale, rc);
  return cudaGetLastError();
}

int lanes_per_trace() {
  static const int v = [] {
    const char* e = std::getenv("HS_REPLAY_LANES");
    const int x = e ? std::atoi(e) : 16;
    return (x == 8 || x == 16 || x == 32) ? x : 16;
  }();
  return v;
}

}  // namespace

bool replay_mt_eligible(const ReplayConst& rc, bool multi) {
  // opt-in (HS_REPLAY_MT=1): measured slower than replay.cu's kernel (K3)
  static const bool on = std::getenv("HS_REPLAY_MT") != nullptr && std::getenv("HS_REPLAY_LEGACY") == nullptr;
  if (!on || multi || rc.mode != 0 || rc.flags != 0 || rc.N < 1 || rc.N > 32) return false;
  for (int t = 0; t < rc.n_types; ++t)  // the interval bounds need non-negative prices
    for (int f = 0; f < 8; ++f)
      if (!(rc.type_p[t][f] >= 0.0)) return false;
  return true;
}

int replay_shared_heap(const ReplayConst& rc, bool multi) {
  return replay_mt_eligible(rc, multi) ? kHS2 : kHeapShared;
}

int64_t replay_extra_heap_entries(const ReplayConst& rc, bool multi) {
  return replay_mt_eligible(rc, multi) ? (int64_t)rc.N * kRingEntries : 0;
}

cudaError_t launch_replay_mt(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                             const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign,
                             double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result, void* d_qrec,
                             uint64_t* d_heap, cudaStream_t st, const uint32_t* d_progress, int phase_len) {
  if (n_traces <= 0) return cudaSuccess;
  static const double wscale = [] {
    const char* e = std::getenv("HS_REPLAY_WIDEN");  // diagnostic only
    const double x = e ? std::atof(e) : 1.0;
    return x >= 1.0 ? x : 1.0;
  }();
  const int L = lanes_per_trace();
  const int K = (rc.N + L - 1) / L;
#define HS_LK(l, k)                                                                                              \
  launch_k<l, k>(rc, n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics, d_result, d_qrec, d_heap, \
                 st, d_progress, phase_len, wscale)
  if (L == 8) {
    switch (K) {
      case 1: return HS_LK(8, 1);
      case 2: return HS_LK(8, 2);
      case 3: return HS_LK(8, 3);
      case 4: return HS_LK(8, 4);
    }
  } else if (L == 16) {
    switch (K) {
      case 1: return HS_LK(16, 1);
      case 2: return HS_LK(16, 2);
    }
  } else {
    return HS_LK(32, 1);
  }
#undef HS_LK
  return cudaErrorInvalidValue;
}

}  // namespace hs
