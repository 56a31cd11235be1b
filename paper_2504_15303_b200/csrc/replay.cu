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
// Per-step bookkeeping is O(1) in registers: a request admitted at step k_a
// has generated = k - k_a at step k, so it retires at step k_a + O
// (simulator.py:334) and max(I + generated + 1) = max(I - k_a) + k + 1
// (simulator.py:351); the max is tracked with a count and recomputed from
// the heap only when its last holder retires.
//
// The state-independent part of the OS workload (ideal batch size and
// per-request cost, scheduling.py:119-147) depends only on (request,
// instance class), so the warp prices 32 (arrival, class) pairs per SIMT
// pass into shared memory; the state-dependent factor exp(theta * usage)
// (capacity.py:98-106, scheduling.py:150-154) is cached per lane and
// recomputed only after the lane's running tokens change.
#include "hs_device.cuh"
#include "hs_internal.h"

namespace hs {

__constant__ ReplayConst c_rep;

constexpr int kWarps = 4;

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

struct Lane {
  // scheduler state (scheduling.py:157-164)
  double load;
  double ex;  // cached exp(theta * usage)
  int64_t run_i, run_p;
  bool dirty, ex_over;
  // run state (simulator.py:259-269)
  int64_t reserved;
  uint32_t k;  // non-idle steps executed
  bool sched;
  double t_next;
  int32_t qhead, qtail, hI, hO;
  int32_t nact;
  uint64_t top;  // heap minimum (valid when nact > 0)
  int64_t cur_max;
  int32_t cnt_max;
  bool max_dirty;
  double completion, peak;
  int64_t req_count, tok_count;
  double wcur;
  // error from a step event
  int32_t err;
  int32_t err_req;
  double err_t;
};

__global__ void __launch_bounds__(kWarps * 32) k_replay(int64_t n_traces, const int64_t* __restrict__ off,
                                                        const int32_t* __restrict__ gI, const int32_t* __restrict__ gO,
                                                        const int32_t* __restrict__ gP, const double* __restrict__ gT,
                                                        uint8_t* __restrict__ assign, double* __restrict__ depart,
                                                        hs_inst_metrics* __restrict__ metrics,
                                                        hs_trace_result* __restrict__ result, double* __restrict__ wrec,
                                                        int32_t* __restrict__ qnext, uint64_t* __restrict__ heap_all) {
  __shared__ uint64_t s_tab[256];
  extern __shared__ double s_cost[];  // [kWarps][32 * n_types]
  for (int k = threadIdx.x; k < 256; k += blockDim.x) s_tab[k] = kExpTab[k];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t tr = (int64_t)blockIdx.x * kWarps + wib;
  if (tr >= n_traces) return;
  const unsigned FULL = 0xffffffffu;
  const int N = c_rep.N;
  const int NT = c_rep.n_types;
  const int policy = c_rep.policy;
  const int64_t pt = c_rep.per_token;
  const double theta = c_rep.theta;
  double* cost = s_cost + (size_t)wib * 32 * NT;

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
  double p[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) p[k] = c_rep.type_p[ty][k];
  const double budget = c_rep.type_budget[ty];
  uint64_t* heap = heap_all + tr * c_rep.heap_stride + c_rep.heap_off[j];
  const int32_t cap = (int32_t)(c_rep.heap_off[j + 1] - c_rep.heap_off[j]);

  Lane s;
  s.load = 0.0;
  s.ex = 1.0;
  s.run_i = s.run_p = 0;
  s.dirty = true;
  s.ex_over = false;
  s.reserved = 0;
  s.k = 0;
  s.sched = false;
  s.t_next = 0.0;
  s.qhead = s.qtail = -1;
  s.hI = s.hO = 0;
  s.nact = 0;
  s.top = 0;
  s.cur_max = INT64_MIN;
  s.cnt_max = 0;
  s.max_dirty = false;
  s.completion = 0.0;
  s.peak = 0.0;
  s.req_count = s.tok_count = 0;
  s.wcur = 0.0;
  s.err = HS_TRACE_OK;
  s.err_req = -1;
  s.err_t = 0.0;
  int64_t n_steps = 0;
  int64_t rr_next = 0;

  int32_t t_err = HS_TRACE_OK, t_err_inst = -1;
  int64_t t_err_req = -1;
  double t_err_val = 0.0;

  // One STEP event of this lane's instance (simulator.py:330-355).
  auto do_step = [&]() {
    const double t = s.t_next;
    s.sched = false;
    ++n_steps;
    // retire, in (departure step, admission order) = active-list order
    while (s.nact > 0 && (uint32_t)(s.top >> 32) == s.k) {
      const int32_t r = (int32_t)(s.top & 0xffffffffu);
      heap_pop(heap, s.nact);
      if (s.nact > 0) s.top = heap[0];
      const int64_t Ir = I[r], Or = O[r], Pr = P[r];
      s.reserved -= Ir + Or;
      s.completion = t;
      s.req_count += 1;
      s.tok_count += Ir + Or;
      if (DEP) DEP[r] = t;
      // Scheduler.complete (scheduling.py:256-264): subtract recorded values
      s.load = __dsub_rn(s.load, W[r]);
      s.run_i -= Ir;
      s.run_p -= Pr;
      s.dirty = true;
      if (s.run_i < 0 || s.run_p < 0) {
        s.err = HS_TRACE_NEGATIVE_RUNNING;
        s.err_req = r;
        s.err_t = t;
        return;
      }
      const int64_t ka = (int64_t)s.k - (Or > 1 ? Or : 1);
      if (Ir - ka == s.cur_max && --s.cnt_max == 0) s.max_dirty = true;
    }
    // admit FCFS (simulator.py:297-316)
    int64_t newly = 0, max_i_new = 0;
    while (s.qhead >= 0) {
      const int64_t need = (int64_t)s.hI + s.hO;
      if (int_gt_double(sat_mul(pt, s.reserved + need), budget)) {
        if (s.nact == 0 && newly == 0) {
          s.err = HS_TRACE_INFEASIBLE_REQUEST;
          s.err_req = s.qhead;
          s.err_t = t;
          return;
        }
        break;
      }
      const int32_t r = s.qhead;
      const int64_t Ir = s.hI, Or = s.hO;
      s.qhead = (r == s.qtail) ? -1 : QN[r];
      if (s.qhead >= 0) {
        s.hI = I[s.qhead];
        s.hO = O[s.qhead];
      }
      s.reserved += need;
      if (Ir > max_i_new) max_i_new = Ir;
      ++newly;
      if (s.nact >= cap) {
        s.err = HS_TRACE_CAPACITY;
        s.err_req = r;
        s.err_t = t;
        return;
      }
      const uint64_t key = ((uint64_t)(s.k + (uint32_t)(Or > 1 ? Or : 1)) << 32) | (uint32_t)r;
      heap_push(heap, s.nact, key);
      s.top = heap[0];
      const int64_t mk = Ir - (int64_t)s.k;
      if (mk > s.cur_max) {
        s.cur_max = mk;
        s.cnt_max = 1;
        s.max_dirty = false;
      } else if (mk == s.cur_max) {
        ++s.cnt_max;
      }
    }
    if (newly) {
      const double u = __ddiv_rn(i2d(pt * s.reserved), budget);  // simulator.py:315
      if (u > s.peak) s.peak = u;
    }
    if (s.nact == 0) return;  // idle until the next dispatch (simulator.py:344-345)
    double c = 0.0;
    if (newly) c = __dadd_rn(c, prefill_time(p, newly, max_i_new));
    if (s.max_dirty || s.cnt_max <= 0) {  // the last holder of the max retired: rescan
      int64_t m = INT64_MIN;
      int32_t cm = 0;
      for (int32_t h = 0; h < s.nact; ++h) {
        const uint64_t key = heap[h];
        const int32_t r = (int32_t)(key & 0xffffffffu);
        const int64_t Or = O[r];
        const int64_t ka = (int64_t)(uint32_t)(key >> 32) - (Or > 1 ? Or : 1);
        const int64_t mk = (int64_t)I[r] - ka;
        if (mk > m) {
          m = mk;
          cm = 1;
        } else if (mk == m) {
          ++cm;
        }
      }
      s.cur_max = m;
      s.cnt_max = cm;
      s.max_dirty = false;
    }
    const int64_t cached = s.cur_max + (int64_t)s.k + 1;
    c = __dadd_rn(c, decode_iteration_time(p, cached, s.nact));
    s.k += 1;
    s.t_next = __dadd_rn(t, c);  // simulator.py:355
    s.sched = true;
  };

  // Advance every lane's steps with t_next < t_limit (strict: steps at the
  // arrival's own time run after it), or all steps when drain.
  auto advance = [&](double t_limit, bool drain) -> bool {
    for (;;) {
      const bool want = valid && s.err == HS_TRACE_OK && s.sched && (drain || s.t_next < t_limit);
      if (!__any_sync(FULL, want)) break;
      if (want) do_step();
    }
    // earliest failing step event wins (heap order: time, then instance)
    const unsigned eb = __ballot_sync(FULL, s.err != HS_TRACE_OK);
    if (!eb) return false;
    double bt = s.err != HS_TRACE_OK ? s.err_t : INFINITY;
    int bl = s.err != HS_TRACE_OK ? lane : 64;
#pragma unroll
    for (int offs = 16; offs > 0; offs >>= 1) {
      const double ot = shfl_d(bt, lane ^ offs);
      const int ol = __shfl_xor_sync(FULL, bl, offs);
      if (ot < bt || (ot == bt && ol < bl)) {
        bt = ot;
        bl = ol;
      }
    }
    t_err = __shfl_sync(FULL, s.err, bl);
    t_err_req = __shfl_sync(FULL, s.err_req, bl);
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
          const double bud = c_rep.type_budget[tyk];
          const double fl = py_floordiv(bud, i2d(pt * (Ia + Pa)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          const double* tp = c_rep.type_p[tyk];
          const double tot = __dadd_rn(prefill_time(tp, b, Ia), decode_time(tp, b, Ia, Pa));
          cost[pair] = (tot <= 0.0) ? -1.0 : __ddiv_rn(tot, i2d(b));
        }
      }
      __syncwarp();
    }
    for (int al = 0; al < n_in; ++al) {
      const int64_t a = base + al;
      const double ta = shfl_d(cT, al);
      const int64_t Ia = __shfl_sync(FULL, cI, al);
      const int64_t Oa = __shfl_sync(FULL, cO, al);
      const int64_t Pa = __shfl_sync(FULL, cP, al);
      if (advance(ta, false)) {
        failed = true;
        break;
      }
      // ---- choose (scheduling.py:235-254)
      int chosen = -1;
      const bool eval_all = policy == HS_POLICY_OS || policy == HS_POLICY_MB;
      if (!eval_all) {
        if (policy == HS_POLICY_SI) {
          chosen = 0;
        } else if (policy == HS_POLICY_RR) {
          chosen = (int)(rr_next % N);
          rr_next += 1;
        } else {  // smooth WRR: first strict maximum after adding weights
          if (valid) s.wcur = __dadd_rn(s.wcur, c_rep.wrr_weight[lane]);
          double bv = valid ? s.wcur : -INFINITY;
          int bl = valid ? lane : 64;
#pragma unroll
          for (int offs = 16; offs > 0; offs >>= 1) {
            const double ov = shfl_d(bv, lane ^ offs);
            const int ol = __shfl_xor_sync(FULL, bl, offs);
            if (ov > bv || (ov == bv && ol < bl)) {
              bv = ov;
              bl = ol;
            }
          }
          chosen = bl;
          if (lane == chosen) s.wcur = __dsub_rn(s.wcur, c_rep.wrr_total);
        }
      }
      // ---- evaluate (scheduling.py:216-233) for the lanes that need it
      const bool need = valid && (eval_all || lane == chosen);
      double w = INFINITY;
      bool cerr = false, eerr = false;
      double cval = 0.0;
      if (need) {
        double cst;
        if (policy == HS_POLICY_MB) {
          cst = 1.0;
        } else {
          cst = cost[al * NT + ty];
          cerr = cst < 0.0;
        }
        if (s.dirty) {  // capacity.py:98-106 kv_usage, scheduling.py:154 exp
          const double usage = __ddiv_rn(i2d(pt * (s.run_i + s.run_p)), budget);
          bool of;
          s.ex = py_exp(__dmul_rn(theta, usage), s_tab, &of);
          s.ex_over = of;
          s.dirty = false;
        }
        eerr = s.ex_over;
        if (cerr) {
          // recompute the non-positive total for the error record
          const double fl = py_floordiv(budget, i2d(pt * (Ia + Pa)));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          cval = __dadd_rn(prefill_time(p, b, Ia), decode_time(p, b, Ia, Pa));
        } else if (eerr) {
          cval = __dmul_rn(theta, __ddiv_rn(i2d(pt * (s.run_i + s.run_p)), budget));
        }
        w = __dmul_rn(cst, s.ex);
      }
      const unsigned errb = __ballot_sync(FULL, need && (cerr || eerr));
      if (errb) {  // first instance in evaluation order raises
        const int el = __ffs(errb) - 1;
        const bool ce = __shfl_sync(FULL, cerr, el);
        t_err = ce ? HS_TRACE_NONPOSITIVE_COST : HS_TRACE_EXP_OVERFLOW;
        t_err_inst = el;
        t_err_req = a;
        t_err_val = shfl_d(cval, el);
        failed = true;
        break;
      }
      if (eval_all) {
        // _min_max_choice (scheduling.py:299-312) in O(log N):
        // peak_s = max(L_s + w_s, max_{j != s} L_j)
        double m1 = valid ? s.load : -INFINITY;
        int i1 = valid ? lane : 64;
#pragma unroll
        for (int offs = 16; offs > 0; offs >>= 1) {
          const double ov = shfl_d(m1, lane ^ offs);
          const int ol = __shfl_xor_sync(FULL, i1, offs);
          if (ov > m1 || (ov == m1 && ol < i1)) {
            m1 = ov;
            i1 = ol;
          }
        }
        double m2 = (valid && lane != i1) ? s.load : -INFINITY;
#pragma unroll
        for (int offs = 16; offs > 0; offs >>= 1) {
          const double ov = shfl_d(m2, lane ^ offs);
          m2 = ov > m2 ? ov : m2;
        }
        const double others = lane == i1 ? m2 : m1;
        const double own = __dadd_rn(s.load, w);
        const double peak = own > others ? own : others;
        const bool cand = need && !isinf(w) && peak < INFINITY;
        double bp = cand ? peak : INFINITY;
        int bl = cand ? lane : 64;
#pragma unroll
        for (int offs = 16; offs > 0; offs >>= 1) {
          const double ov = shfl_d(bp, lane ^ offs);
          const int ol = __shfl_xor_sync(FULL, bl, offs);
          if (ov < bp || (ov == bp && ol < bl)) {
            bp = ov;
            bl = ol;
          }
        }
        if (bl >= 64) {
          t_err = HS_TRACE_NO_INSTANCE;
          t_err_req = a;
          t_err_inst = -1;
          failed = true;
          break;
        }
        chosen = bl;
      }
      // ---- commit (scheduling.py:335-346) and enqueue (simulator.py:323-327)
      if (lane == chosen) {
        s.load = __dadd_rn(s.load, w);
        s.run_i += Ia;
        s.run_p += Pa;
        s.dirty = true;
        W[a] = w;
        if (s.qhead < 0) {
          s.qhead = (int32_t)a;
          s.hI = (int32_t)Ia;
          s.hO = (int32_t)Oa;
        } else {
          QN[s.qtail] = (int32_t)a;
        }
        s.qtail = (int32_t)a;
        if (!s.sched) {
          s.sched = true;
          s.t_next = ta;
        }
      }
      if (lane == al) my_assign = (uint8_t)chosen;
    }
    if (assign && lane < n_in && !failed) assign[o + base + lane] = my_assign;
  }
  if (!failed && advance(0.0, true)) failed = true;

  if (valid) {
    hs_inst_metrics m;
    m.completion_time = s.completion;
    m.peak_kv_usage = s.peak;
    m.residual_load = s.load;
    m.request_count = s.req_count;
    m.token_count = s.tok_count;
    metrics[tr * N + lane] = m;
  }
#pragma unroll
  for (int offs = 16; offs > 0; offs >>= 1) n_steps += __shfl_xor_sync(FULL, n_steps, offs);
  if (lane == 0) {
    hs_trace_result r;
    r.error = failed ? t_err : HS_TRACE_OK;
    r.err_instance = failed ? t_err_inst : -1;
    r.err_request = failed ? t_err_req : -1;
    r.err_value = failed ? t_err_val : 0.0;
    r.n_steps = n_steps;
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
  if (smem > 48 * 1024) {
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
#pragma unroll
  for (int offs = 16; offs > 0; offs >>= 1) {
    const int32_t o2 = __shfl_xor_sync(0xffffffffu, m, offs);
    m = o2 < m ? o2 : m;
  }
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
