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
// mapping (scheduling.py:299-312) is O(log N): top-2 of the loads and an
// argmin of peaks via REDUX on order-preserving 64-bit keys.
#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {

__constant__ ReplayConst c_rep;

constexpr int kWarps = 4;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ void heap_push(uint64_t* h, int32_t& n, uint64_t key) {
  int32_t i = n++;
  while (i > 0) {
    const int32_t p = (i - 1) >> 1;
    const uint64_t hp = h[p];
    if (hp <= key) break;
    h[i] = hp;
    i = p;
  }
  h[i] = key;
}

__device__ __forceinline__ void heap_pop(uint64_t* h, int32_t& n) {
  const uint64_t last = h[--n];
  int32_t i = 0;
  for (;;) {
    int32_t l = 2 * i + 1;
    if (l >= n) break;
    uint64_t hl = h[l];
    if (l + 1 < n) {
      const uint64_t hr = h[l + 1];
      if (hr < hl) {
        hl = hr;
        ++l;
      }
    }
    if (last <= hl) break;
    h[i] = hl;
    i = l;
  }
  if (n > 0) h[i] = last;
}

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
  double completion, peak, wcur, err_t;
  int64_t tok_count;
  int32_t req_count, qtail, cnt_max, err, err_req, _pad;
};

__global__ void __launch_bounds__(kWarps * 32, 7)
    k_replay(int64_t n_traces, const int64_t* __restrict__ off, const int32_t* __restrict__ gI,
             const int32_t* __restrict__ gO, const int32_t* __restrict__ gP, const double* __restrict__ gT,
             uint8_t* __restrict__ assign, double* __restrict__ depart, hs_inst_metrics* __restrict__ metrics,
             hs_trace_result* __restrict__ result, double* __restrict__ wrec, int32_t* __restrict__ qnext,
             uint64_t* __restrict__ heap_all) {
  __shared__ uint64_t s_tab[256];
  __shared__ Cold s_cold[kWarps * 32];
  extern __shared__ double s_cost[];  // [kWarps][32 * n_types]
  for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab[k] = kExpTab[k];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t tr = (int64_t)blockIdx.x * kWarps + wib;
  if (tr >= n_traces) return;
  const int N = c_rep.N;
  const int NT = c_rep.n_types;
  const int policy = c_rep.policy;
  const int64_t pt = c_rep.per_token;
  const double theta = c_rep.theta;
  double* cost = s_cost + (size_t)wib * 32 * NT;
  Cold& cold = s_cold[threadIdx.x];

  const int64_t o = off[tr];
  const int64_t q = off[tr + 1] - o;
  const int32_t* I = gI + o;
  const int32_t* O = gO + o;
  const int32_t* P = gP + o;
  const double* T = gT ? gT + o : nullptr;
  double* W = wrec + o;
  int32_t* QN = qnext + o;
  double* DEP = depart ? depart + o : nullptr;

  const bool valid = lane < N;
  const int j = valid ? lane : 0;
  const int ty = c_rep.inst_type[j];
  const double* tp = c_rep.type_p[ty];
  const double budget = c_rep.type_budget[ty];
  const double p7 = tp[6], p8 = tp[7];
  uint64_t* heap = heap_all + tr * c_rep.heap_stride + c_rep.heap_off[j];
  const int32_t cap = (int32_t)(c_rep.heap_off[j + 1] - c_rep.heap_off[j]);

  // hot per-lane state (registers)
  double load = 0.0, ex = 1.0;
  int64_t run_i = 0, run_p = 0, reserved = 0, cur_max = INT64_MIN;
  uint32_t k = 0, kr = 0xffffffffu;  // steps executed; step of the next retirement
  double t_next = 0.0, cd = 0.0, A = 0.0, B = 0.0;  // clock, cached len (double), p5*b, p6*b
  int32_t qhead = -1, hI = 0, hO = 0, nact = 0;
  bool sched = false, dirty = true, ex_over = false, max_dirty = false, blocked = false;
  cold.completion = 0.0;
  cold.peak = 0.0;
  cold.wcur = 0.0;
  cold.err_t = 0.0;
  cold.tok_count = 0;
  cold.req_count = 0;
  cold.qtail = -1;
  cold.cnt_max = 0;
  cold.err = HS_TRACE_OK;
  cold.err_req = -1;
  uint32_t n_steps = 0;
  int64_t rr_next = 0;
  int32_t t_err = HS_TRACE_OK, t_err_inst = -1;
  int64_t t_err_req = -1;
  double t_err_val = 0.0;

  // A full STEP event (simulator.py:330-355): retirements due at this step,
  // FCFS admission, prefill for newcomers, one decode iteration.
  auto event_step = [&]() {
    const double t = t_next;
    sched = false;
    ++n_steps;
    if (nact > 0 && (uint32_t)(heap[0] >> 32) == k) {
      do {  // retire in (departure step, admission order)
        const uint64_t top = heap[0];
        const int32_t r = (int32_t)(top & 0xffffffffu);
        heap_pop(heap, nact);
        const int64_t Ir = I[r], Or = O[r], Pr = P[r];
        const double wr = W[r];
        reserved -= Ir + Or;
        cold.completion = t;
        cold.req_count += 1;
        cold.tok_count += Ir + Or;
        if (DEP) DEP[r] = t;
        load = __dsub_rn(load, wr);  // Scheduler.complete: recorded values
        run_i -= Ir;
        run_p -= Pr;
        dirty = true;
        if (run_i < 0 || run_p < 0) {
          cold.err = HS_TRACE_NEGATIVE_RUNNING;
          cold.err_req = r;
          cold.err_t = t;
          return;
        }
        const int64_t ka = (int64_t)k - (Or > 1 ? Or : 1);
        if (Ir - ka == cur_max && --cold.cnt_max == 0) max_dirty = true;
      } while (nact > 0 && (uint32_t)(heap[0] >> 32) == k);
    }
    // admit FCFS (simulator.py:297-316)
    int64_t newly = 0, max_i_new = 0;
    while (qhead >= 0) {
      const int64_t need = (int64_t)hI + hO;
      if (int_gt_double(sat_mul(pt, reserved + need), budget)) {
        if (nact == 0 && newly == 0) {
          cold.err = HS_TRACE_INFEASIBLE_REQUEST;
          cold.err_req = qhead;
          cold.err_t = t;
          return;
        }
        break;
      }
      const int32_t r = qhead;
      const int64_t Ir = hI, Or = hO;
      qhead = (r == cold.qtail) ? -1 : QN[r];
      if (qhead >= 0) {
        hI = I[qhead];
        hO = O[qhead];
      }
      reserved += need;
      if (Ir > max_i_new) max_i_new = Ir;
      ++newly;
      if (nact >= cap || k > 0x7fffffffu) {
        cold.err = HS_TRACE_CAPACITY;
        cold.err_req = r;
        cold.err_t = t;
        return;
      }
      heap_push(heap, nact, ((uint64_t)(k + (uint32_t)(Or > 1 ? Or : 1)) << 32) | (uint32_t)r);
      const int64_t mk = Ir - (int64_t)k;
      if (mk > cur_max) {
        cur_max = mk;
        cold.cnt_max = 1;
        max_dirty = false;
      } else if (mk == cur_max) {
        cold.cnt_max += 1;
      }
    }
    blocked = true;  // queue empty or its head does not fit: nothing changes until an event
    if (newly) {
      const double u = __ddiv_rn(i2d(pt * reserved), budget);  // simulator.py:315
      if (u > cold.peak) cold.peak = u;
    }
    if (nact == 0) {  // idle until the next dispatch (simulator.py:344-345)
      kr = 0xffffffffu;
      return;
    }
    double c = 0.0;
    if (newly) c = __dadd_rn(c, prefill_time(tp, newly, max_i_new));
    if (max_dirty || cold.cnt_max <= 0) {  // the last holder of the max retired: rescan
      int64_t m = INT64_MIN;
      int32_t cm = 0;
      for (int32_t h = 0; h < nact; ++h) {
        const uint64_t key = heap[h];
        const int32_t r = (int32_t)(key & 0xffffffffu);
        const int64_t Or = O[r];
        const int64_t mk = (int64_t)I[r] - ((int64_t)(uint32_t)(key >> 32) - (Or > 1 ? Or : 1));
        if (mk > m) {
          m = mk;
          cm = 1;
        } else if (mk == m) {
          ++cm;
        }
      }
      cur_max = m;
      cold.cnt_max = cm;
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
    kr = (uint32_t)(heap[0] >> 32);
    t_next = __dadd_rn(t, c);
    sched = true;
  };

  // Advance every lane's steps with t_next < t_limit (strict: steps at an
  // arrival's own time run after it), or every step when draining.
  auto advance = [&](double t_limit, bool drain) -> bool {
    for (;;) {
      const bool want = valid && sched && (drain || t_next < t_limit) && cold.err == HS_TRACE_OK;
      if (!__any_sync(FULL, want)) break;
      if (want) {
        if (blocked && k < kr) {
          // pure steps: decode price + clock, no heap / queue traffic.  Two
          // steps per iteration: their prices depend only on the cached
          // length, so both are computed side by side and only the clock
          // additions stay serial (the reference's rounding order).
          const double lim = drain ? INFINITY : t_limit;
          const uint32_t k0 = k;
          for (;;) {
            const double cd1 = __dadd_rn(cd, 1.0);
            const double c0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, cd), B), __dmul_rn(p7, cd)), p8);
            const double c1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A, cd1), B), __dmul_rn(p7, cd1)), p8);
            const double t1 = __dadd_rn(t_next, c0);
            if (!(k + 1 < kr && (t1 < lim || drain))) {
              t_next = t1;
              cd = cd1;
              k += 1;
              break;
            }
            t_next = __dadd_rn(t1, c1);
            cd = __dadd_rn(cd1, 1.0);
            k += 2;
            if (!(k < kr && (t_next < lim || drain))) break;
          }
          n_steps += k - k0;
        } else {
          event_step();
        }
      }
    }
    const unsigned eb = __ballot_sync(FULL, valid && cold.err != HS_TRACE_OK);
    if (!eb) return false;
    // the earliest failing step event wins (heap order: time, then instance)
    const uint64_t tk = (valid && cold.err != HS_TRACE_OK) ? okey(cold.err_t) : ~0ull;
    const uint64_t mt = warp_min_u64(tk);
    const int bl = __ffs(__ballot_sync(FULL, tk == mt)) - 1;
    t_err = __shfl_sync(FULL, cold.err, bl);
    t_err_req = __shfl_sync(FULL, cold.err_req, bl);
    t_err_inst = bl;
    t_err_val = 0.0;
    return true;
  };

  bool failed = false;
  uint8_t my_assign = 0;
  for (int64_t base = 0; base < q && !failed; base += 32) {
    const int n_in = (int)((q - base) < 32 ? (q - base) : 32);
    int32_t cI = 0, cO = 0, cP = 0;
    double cT = 0.0;
    if (lane < n_in) {
      cI = I[base + lane];
      cO = O[base + lane];
      cP = P[base + lane];
      cT = T ? T[base + lane] : 0.0;
    }
    // price (arrival, class) pairs: scheduling.py:119-147
    __syncwarp();
    if (policy != HS_POLICY_MB) {
      for (int pair0 = 0; pair0 < n_in * NT; pair0 += 32) {
        const int pair = pair0 + lane;
        const int al = pair / NT, tyk = pair - al * NT;
        const int srcl = al < 32 ? al : 0;
        const int64_t Ia = __shfl_sync(FULL, cI, srcl);
        const int64_t Pa = __shfl_sync(FULL, cP, srcl);
        if (pair < n_in * NT) {
          const double fl = py_floordiv(c_rep.type_budget[tyk], i2d(pt * (Ia + Pa)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          const double* ctp = c_rep.type_p[tyk];
          const double tot = __dadd_rn(prefill_time(ctp, b, Ia), decode_time(ctp, b, Ia, Pa));
          cost[pair] = (tot <= 0.0) ? -1.0 : __ddiv_rn(tot, i2d(b));
        }
      }
      __syncwarp();
    }
    for (int al = 0; al < n_in; ++al) {
      const int64_t a = base + al;
      const double ta = shfl_d(cT, al);
      if (advance(ta, false)) {
        failed = true;
        break;
      }
      const int64_t Ia = __shfl_sync(FULL, cI, al);
      const int64_t Oa = __shfl_sync(FULL, cO, al);
      const int64_t Pa = __shfl_sync(FULL, cP, al);
      // ---- choose (scheduling.py:235-254)
      int chosen = -1;
      const bool eval_all = policy == HS_POLICY_OS || policy == HS_POLICY_MB;
      if (!eval_all) {
        if (policy == HS_POLICY_SI) {
          chosen = 0;
        } else if (policy == HS_POLICY_RR) {
          chosen = (int)(rr_next % N);
          rr_next += 1;
        } else {  // smooth WRR: first strict maximum after adding the weights
          if (valid) cold.wcur = __dadd_rn(cold.wcur, c_rep.wrr_weight[lane]);
          const uint64_t wk = valid ? okey(cold.wcur) : 0ull;
          const uint64_t mk = warp_max_u64(wk);
          chosen = __ffs(__ballot_sync(FULL, valid && wk == mk)) - 1;
          if (lane == chosen) cold.wcur = __dsub_rn(cold.wcur, c_rep.wrr_total);
        }
      }
      // ---- evaluate (scheduling.py:216-233) on the lanes that need it
      const bool need = valid && (eval_all || lane == chosen);
      double w = INFINITY;
      bool cerr = false, eerr = false;
      if (need) {
        double cst = 1.0;
        if (policy != HS_POLICY_MB) {
          cst = cost[al * NT + ty];
          cerr = cst < 0.0;
        }
        if (dirty) {  // capacity.py:98-106 kv_usage, scheduling.py:154 exp
          const double usage = __ddiv_rn(i2d(pt * (run_i + run_p)), budget);
          bool of;
          ex = py_exp(__dmul_rn(theta, usage), s_tab, &of);
          ex_over = of;
          dirty = false;
        }
        eerr = ex_over;
        w = __dmul_rn(cst, ex);
      }
      const unsigned errb = __ballot_sync(FULL, need && (cerr || eerr));
      if (errb) {  // the first instance in evaluation order raises
        const int el = __ffs(errb) - 1;
        const bool ce = __shfl_sync(FULL, cerr, el);
        double cval = 0.0;
        if (lane == el && ce) {  // recompute the non-positive total for the message
          const double fl = py_floordiv(budget, i2d(pt * (Ia + Pa)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          cval = __dadd_rn(prefill_time(tp, b, Ia), decode_time(tp, b, Ia, Pa));
        }
        t_err = ce ? HS_TRACE_NONPOSITIVE_COST : HS_TRACE_EXP_OVERFLOW;
        t_err_inst = el;
        t_err_req = a;
        t_err_val = shfl_d(cval, el);
        failed = true;
        break;
      }
      if (eval_all) {
        // _min_max_choice (scheduling.py:299-312):
        // peak_s = max(L_s + w_s, max_{j != s} L_j), argmin with lowest index
        const uint64_t lk = valid ? okey(load) : 0ull;
        const uint64_t m1 = warp_max_u64(lk);
        const unsigned at_max = __ballot_sync(FULL, valid && lk == m1);
        uint64_t m2;
        if (__popc(at_max) >= 2) {
          m2 = m1;
        } else {
          m2 = warp_max_u64(lk == m1 ? 0ull : lk);
        }
        const uint64_t ok_ = (lk == m1) ? m2 : m1;
        const double others = ok_ == 0ull ? -INFINITY : from_okey(ok_);
        const double own = __dadd_rn(load, w);
        const double peak = own > others ? own : others;
        const bool cand = need && !isinf(w) && peak < INFINITY;
        const uint64_t pk = cand ? okey(peak) : ~0ull;
        const uint64_t mp = warp_min_u64(pk);
        const unsigned win = __ballot_sync(FULL, cand && pk == mp);
        if (!win) {
          t_err = HS_TRACE_NO_INSTANCE;
          t_err_req = a;
          t_err_inst = -1;
          failed = true;
          break;
        }
        chosen = __ffs(win) - 1;
      }
      // ---- commit (scheduling.py:335-346) and enqueue (simulator.py:323-327)
      if (lane == chosen) {
        load = __dadd_rn(load, w);
        run_i += Ia;
        run_p += Pa;
        dirty = true;
        W[a] = w;
        if (qhead < 0) {
          qhead = (int32_t)a;
          hI = (int32_t)Ia;
          hO = (int32_t)Oa;
          blocked = false;  // a new queue head may be admitted at the next step
        } else {
          QN[cold.qtail] = (int32_t)a;
        }
        cold.qtail = (int32_t)a;
        if (!sched) {
          sched = true;
          t_next = ta;
          blocked = false;
        }
      }
      if (lane == al) my_assign = (uint8_t)chosen;
    }
    if (assign && lane < n_in && !failed) assign[o + base + lane] = my_assign;
  }
  if (!failed && advance(0.0, true)) failed = true;

  if (valid) {
    hs_inst_metrics m;
    m.completion_time = cold.completion;
    m.peak_kv_usage = cold.peak;
    m.residual_load = load;
    m.request_count = cold.req_count;
    m.token_count = cold.tok_count;
    metrics[tr * N + lane] = m;
  }
  int64_t steps_all = n_steps;
#pragma unroll
  for (int offs = 16; offs > 0; offs >>= 1) steps_all += __shfl_xor_sync(FULL, steps_all, offs);
  if (lane == 0) {
    hs_trace_result r;
    r.error = failed ? t_err : HS_TRACE_OK;
    r.err_instance = failed ? t_err_inst : -1;
    r.err_request = failed ? t_err_req : -1;
    r.err_value = failed ? t_err_val : 0.0;
    r.n_steps = steps_all;
    result[tr] = r;
  }
}

cudaError_t launch_replay(const ReplayConst& rc, int64_t n_traces, const int64_t* d_off, const int32_t* d_I,
                          const int32_t* d_O, const int32_t* d_P, const double* d_arr, uint8_t* d_assign,
                          double* d_depart, hs_inst_metrics* d_metrics, hs_trace_result* d_result, double* d_wrec,
                          int32_t* d_qnext, uint64_t* d_heap, cudaStream_t st) {
  cudaError_t e = cudaMemcpyToSymbolAsync(c_rep, &rc, sizeof(ReplayConst), 0, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  if (n_traces <= 0) return cudaSuccess;
  const size_t smem = (size_t)kWarps * 32 * rc.n_types * sizeof(double);
  if (smem > 32 * 1024) {
    e = cudaFuncSetAttribute(k_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const unsigned blocks = (unsigned)((n_traces + kWarps - 1) / kWarps);
  k_replay<<<blocks, kWarps * 32, smem, st>>>(n_traces, d_off, d_I, d_O, d_P, d_arr, d_assign, d_depart, d_metrics,
                                              d_result, d_wrec, d_qnext, d_heap);
  return cudaGetLastError();
}

// min over all requests of (I + O): sizes the per-instance active-set heaps
__global__ void k_min_need(const int32_t* __restrict__ I, const int32_t* __restrict__ O, int64_t n, int32_t* out) {
  int32_t m = INT32_MAX;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)I[k] + O[k];
    const int32_t vv = v > INT32_MAX ? INT32_MAX : (int32_t)v;
    m = vv < m ? vv : m;
  }
  m = __reduce_min_sync(FULL, (unsigned)m);
  if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

cudaError_t launch_min_need(const int32_t* d_I, const int32_t* d_O, int64_t n, int32_t* d_out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  const int cap = sm_count() * 8;
  if (blocks > cap) blocks = cap;
  k_min_need<<<blocks, 256, 0, st>>>(d_I, d_O, n, d_out);
  return cudaGetLastError();
}

}  // namespace hs
