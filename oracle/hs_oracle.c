/*
 * hs_oracle.c -- TEST INFRASTRUCTURE ONLY (see hs_oracle.h).
 *
 * Literal C restatement of the reference hot path.  Every function names the
 * reference lines it follows (paths relative to
 * /root/reference/pkg/src/hetserve).  Arithmetic follows CPython semantics:
 * left-to-right fp64 evaluation with no contraction (build with
 * -ffp-contract=off), exact integer arithmetic (__int128 where a Python int
 * could exceed int64), exact int-vs-float comparisons, CPython 3.12's
 * compensated sum(), CPython float floor division and glibc 2.39's exp.
 */
#include "hs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#include "../include/hs_exp_table.h"

typedef __int128 i128;

static double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }

/* ------------------------------------------------------------------------
 * glibc 2.39 exp, FMA ifunc variant (the one CPython's math.exp reaches on
 * an FMA/AVX2 x86-64 host).  Algorithm: sysdeps/ieee754/dbl-64/e_exp.c; the
 * fused operations are exactly those in libm.so.6's FMA body (vfmadd* at
 * libm+0x79b60 in the build container).
 * ---------------------------------------------------------------------- */
#define ORC_INVLN2N 0x1.71547652b82fep+7
#define ORC_SHIFT 0x1.8p52
#define ORC_NEGLN2HIN -0x1.62e42fefa0000p-8
#define ORC_NEGLN2LON -0x1.cf79abc9e3b3ap-47
#define ORC_C2 0x1.ffffffffffdbdp-2
#define ORC_C3 0x1.555555555543cp-3
#define ORC_C4 0x1.55555cf172b91p-5
#define ORC_C5 0x1.1111167a4d017p-7

static double orc_specialcase(double tmp, uint64_t sbits, uint64_t ki, int* overflow) {
  if ((ki & 0x80000000u) == 0) {
    sbits -= 1009ull << 52;
    double scale = u2d(sbits);
    double y = 0x1p1009 * fma(scale, tmp, scale);
    if (isinf(y)) *overflow = 1;
    return y;
  }
  sbits += 1022ull << 52;
  double scale = u2d(sbits);
  double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    double lo = (scale - y) + st;
    double hi = 1.0 + y;
    lo = ((1.0 - hi) + y) + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

double hs_oracle_exp(double x, int* overflow) {
  *overflow = 0;
  uint64_t ix = d2u(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 969u >= 63u) {
    if ((int32_t)(abstop - 969u) < 0) return 1.0 + x; /* tiny |x| */
    if (abstop >= 1033u) {
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      if (ix >> 63) return 0.0; /* underflow: CPython returns 0.0 */
      *overflow = 1;
      return INFINITY;
    }
    abstop = 0; /* 512 <= |x| < 1024: specialcase below */
  }
  double kd = fma(x, ORC_INVLN2N, ORC_SHIFT);
  uint64_t ki = d2u(kd);
  kd = kd - ORC_SHIFT;
  double r = fma(kd, ORC_NEGLN2HIN, x);
  r = fma(kd, ORC_NEGLN2LON, r);
  uint64_t idx = 2 * (ki % 128);
  uint64_t top = ki << 45;
  double tail = u2d(kExpTab[idx]);
  uint64_t sbits = kExpTab[idx + 1] + top;
  double a = fma(r, ORC_C3, ORC_C2);
  double t1 = r + tail;
  double r2 = r * r;
  double b = fma(r, ORC_C5, ORC_C4);
  double tmp = fma(a, r2, t1);
  double r4 = r2 * r2;
  tmp = fma(r4, b, tmp);
  if (abstop == 0) return orc_specialcase(tmp, sbits, ki, overflow);
  double scale = u2d(sbits);
  return fma(scale, tmp, scale);
}

/* CPython Objects/floatobject.c _float_div_mod -> floor quotient. */
double hs_oracle_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod) {
    if ((wx < 0) != (mod < 0)) {
      mod += wx;
      div -= 1.0;
    }
  }
  double fl;
  if (div) {
    fl = floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = copysign(0.0, vx / wx);
  }
  return fl;
}

/* CPython 3.12 Python/bltinmodule.c builtin_sum_impl, float items, start 0:
 * result = 0 + x0, then Neumaier compensation, compensation added at the
 * end only when non-zero and finite.  An empty sequence gives int 0. */
typedef struct { double f, c; int64_t n; } pysum_t;
static void pysum_init(pysum_t* s) { s->f = 0.0; s->c = 0.0; s->n = 0; }
static void pysum_add(pysum_t* s, double x) {
  if (s->n++ == 0) { s->f = 0.0 + x; return; }
  double t = s->f + x;
  if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
  else s->c += (x - t) + s->f;
  s->f = t;
}
static double pysum_result(const pysum_t* s) {
  double f = s->f;
  if (s->c != 0.0 && isfinite(s->c)) f += s->c;
  return f;
}
double hs_oracle_pysum(const double* xs, int64_t n) {
  pysum_t s; pysum_init(&s);
  for (int64_t i = 0; i < n; ++i) pysum_add(&s, xs[i]);
  return pysum_result(&s);
}

/* exact Python comparison int > float */
static int i128_gt_double(i128 v, double b) {
  if (b != b) return 0;
  if (b >= 0x1p120) return 0;
  if (b < -0x1p120) return 1;
  double fl = floor(b);
  i128 flv = (i128)fl;
  return v > flv;
}
/* Python float(int): correctly rounded */
static double i128_to_double(i128 v) { return (double)v; }

/* latency.py:90-92 prefill_time: p1*b*I + p2*b + p3*I + p4 */
static double prefill(const double* p, int64_t b, int64_t I) {
  double db = (double)b, dI = (double)I;
  return (((p[0] * db) * dI) + (p[1] * db)) + (p[2] * dI) + p[3];
}
/* latency.py:95-97 decode_iteration_time: p5*b*c + p6*b + p7*c + p8 */
static double decode_iter(const double* p, int64_t cached, int64_t b) {
  double db = (double)b, dc = (double)cached;
  return (((p[4] * db) * dc) + (p[5] * db)) + (p[6] * dc) + p[7];
}
/* latency.py:100-109 decode_time closed form */
static double decode_total(const double* p, int64_t b, int64_t I, int64_t O) {
  double S = i128_to_double((i128)O * I) + (i128_to_double((i128)O * (O + 1)) / 2.0);
  double db = (double)b;
  return ((p[4] * db) + p[6]) * S + ((p[5] * db) + p[7]) * (double)O;
}

/* capacity.py:67-69 */
static int64_t per_token_of(const hs_model* m) {
  return 2 * m->layers * m->hidden_dim * m->bytes_per_param;
}
/* capacity.py:72-86 kv_budget (divisibility checked by caller) */
static double kv_budget_of(const hs_model* model, const hs_engine* eng, int64_t tp, int64_t mem) {
  double usable = i128_to_double((i128)tp * mem) * eng->mem_utilization_fraction;
  return (usable - (double)eng->static_overhead_bytes) -
         i128_to_double((i128)model->param_count * model->bytes_per_param);
}

/* core.py:363-371 enumerate_tp_degrees */
static int32_t degrees_of(int64_t count, int32_t* out) {
  int32_t n = 0;
  for (int64_t t = 1; t <= count && n < HS_MAX_DEGREES; t *= 2)
    if (count % t == 0) out[n++] = (int32_t)t;
  return n;
}

/* planner.py:143-181 (one machine) = capacity.py:72-95 + planner.py:51-118 */
void hs_oracle_entry(const hs_model* model, const hs_engine* engine, const hs_limits* limits,
                     const hs_machine* machines, int32_t i, int32_t t, const double* p,
                     int present, const int32_t* I, const int32_t* O, int64_t q, hs_entry* e) {
  memset(e, 0, sizeof(*e));
  const hs_machine* own = &machines[i];
  const hs_machine* spec = &machines[own->spec_index];
  e->tp_degree = t;
  e->instance_count = own->accelerator_count / t;
  e->bad_request = -1;
  if (t < 1 || spec->accelerator_count % t != 0) { e->status = HS_ENTRY_BAD_DEGREE; return; }
  int64_t per_token = per_token_of(model);
  double budget = kv_budget_of(model, engine, t, spec->accelerator_mem_bytes);
  i128 required = (i128)per_token * (limits->max_input_len + limits->max_output_len);
  double slack = budget - i128_to_double(required);
  e->budget = budget;
  e->slack = slack;
  if (!(slack >= 0)) { e->status = HS_ENTRY_INFEASIBLE_CONFIG; return; }
  if (!present) { e->status = HS_ENTRY_MISSING_PARAMS; return; }
  /* planner.py:51-87 plan_static_batches, literal, then planner.py:104-106
   * time_batches (estimate_batch_time per batch, planner.py:90-101) */
  pysum_t tot; pysum_init(&tot);
  int64_t start = 0;
  while (start < q) {
    i128 input_sum = 0;
    int64_t max_output = 0;
    int64_t stop = start;
    while (stop < q) {
      i128 cand_inputs = input_sum + I[stop];
      int64_t cand_max_o = max_output > O[stop] ? max_output : O[stop];
      int64_t width = stop - start + 1;
      i128 reserved = (i128)per_token * cand_inputs + (i128)width * per_token * cand_max_o;
      if (i128_gt_double(reserved, budget)) break;
      input_sum = cand_inputs;
      max_output = cand_max_o;
      stop += 1;
    }
    if (stop == start) { e->status = HS_ENTRY_INFEASIBLE_REQUEST; e->bad_request = start; return; }
    int64_t mi = 0, mo = 0;
    for (int64_t k = start; k < stop; ++k) {
      if (I[k] > mi) mi = I[k];
      if (O[k] > mo) mo = O[k];
    }
    int64_t b = stop - start;
    pysum_add(&tot, prefill(p, b, mi) + decode_total(p, b, mi, mo));
    start = stop;
  }
  i128 tokens = 0;
  for (int64_t k = 0; k < q; ++k) tokens += (i128)I[k] + O[k];
  e->token_count = (int64_t)tokens;
  double total = pysum_result(&tot);
  if (tot.n == 0 || total == 0.0) {
    e->status = HS_ENTRY_ZERO_DIVISION;
    e->zero_div_int = tot.n == 0;
    return;
  }
  e->rate = i128_to_double(tokens) / total;
  e->contribution = e->rate * (double)e->instance_count;
  e->status = HS_ENTRY_OK;
}

int hs_oracle_tables(const hs_model* model, const hs_engine* engine, const hs_limits* limits,
                     const hs_machine* machines, int32_t M, const double* params,
                     const uint8_t* present, const int32_t* I, const int32_t* O, int64_t q,
                     hs_entry* table, int32_t* n_degrees) {
  if (M < 1 || M > HS_MAX_MACHINES) return HS_ERR_ARG;
  for (int32_t i = 0; i < M; ++i) {
    int32_t deg[HS_MAX_DEGREES];
    int32_t n;
    if (machines[i].fixed_degree > 0) { deg[0] = machines[i].fixed_degree; n = 1; }
    else n = degrees_of(machines[i].accelerator_count, deg);
    n_degrees[i] = n;
    for (int32_t d = 0; d < n; ++d)
      hs_oracle_entry(model, engine, limits, machines, i, deg[d],
                      params + ((int64_t)i * HS_MAX_DEGREES + d) * 8,
                      present[i * HS_MAX_DEGREES + d], I, O, q, &table[i * HS_MAX_DEGREES + d]);
  }
  return HS_OK;
}

/* planner.py:216-226: decode the product index (machine 0 most significant,
 * itertools.product order), then estimate_system_throughput literally. */
double hs_oracle_candidate_literal(const hs_model* model, const hs_engine* engine,
                                   const hs_limits* limits, const hs_machine* machines, int32_t M,
                                   const double* params, const uint8_t* present, const int32_t* I,
                                   const int32_t* O, int64_t q, int64_t index, int32_t* first_bad,
                                   int32_t* bad_status) {
  int32_t digit[HS_MAX_MACHINES];
  int32_t degs[HS_MAX_MACHINES][HS_MAX_DEGREES];
  int32_t nd[HS_MAX_MACHINES];
  for (int32_t i = 0; i < M; ++i) nd[i] = degrees_of(machines[i].accelerator_count, degs[i]);
  for (int32_t i = M - 1; i >= 0; --i) { digit[i] = (int32_t)(index % nd[i]); index /= nd[i]; }
  double total = 0.0;
  *first_bad = -1;
  *bad_status = HS_ENTRY_OK;
  for (int32_t i = 0; i < M; ++i) {
    hs_entry e;
    int32_t d = digit[i];
    hs_oracle_entry(model, engine, limits, machines, i, degs[i][d],
                    params + ((int64_t)i * HS_MAX_DEGREES + d) * 8, present[i * HS_MAX_DEGREES + d],
                    I, O, q, &e);
    if (e.status != HS_ENTRY_OK) { *first_bad = i; *bad_status = e.status; return 0.0; }
    total = total + e.contribution;
  }
  return total;
}

typedef struct {
  const hs_model* model; const hs_engine* engine; const hs_limits* limits; const hs_machine* machines;
  int32_t M; const double* params; const uint8_t* present; const int32_t* I; const int32_t* O; int64_t q;
  const int64_t* idx; int64_t n; double* totals; int32_t* first_bad; int64_t* next; pthread_mutex_t* mu;
} lit_job_t;

static void* literal_worker(void* arg) {
  lit_job_t* j = (lit_job_t*)arg;
  for (;;) {
    pthread_mutex_lock(j->mu);
    int64_t k = (*j->next)++;
    pthread_mutex_unlock(j->mu);
    if (k >= j->n) break;
    int32_t fb, st;
    double t = hs_oracle_candidate_literal(j->model, j->engine, j->limits, j->machines, j->M, j->params,
                                           j->present, j->I, j->O, j->q, j->idx[k], &fb, &st);
    j->totals[k] = t;
    j->first_bad[k] = fb;
  }
  return NULL;
}

/* The literal per-candidate reference loop over a list of candidate indices,
 * spread over nthreads (used as the CPU baseline of the search). */
int hs_oracle_candidates_literal(const hs_model* model, const hs_engine* engine, const hs_limits* limits,
                                 const hs_machine* machines, int32_t M, const double* params,
                                 const uint8_t* present, const int32_t* I, const int32_t* O, int64_t q,
                                 const int64_t* idx, int64_t n, int nthreads, double* totals, int32_t* first_bad) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  int64_t next = 0;
  lit_job_t job = {model, engine, limits, machines, M, params, present, I, O, q, idx, n, totals, first_bad, &next, &mu};
  for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, literal_worker, &job);
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  return HS_OK;
}

/* candidate total from the table, reference order (planner.py:151,180) */
static double table_total(const hs_entry* table, int32_t M, const int32_t* digit, int32_t* first_bad) {
  double acc = 0.0;
  *first_bad = -1;
  for (int32_t i = 0; i < M; ++i) {
    const hs_entry* e = &table[i * HS_MAX_DEGREES + digit[i]];
    if (e->status != HS_ENTRY_OK) { *first_bad = i; return 0.0; }
    acc = acc + e->contribution;
  }
  return acc;
}

static int64_t space_size(const int32_t* nd, int32_t M) {
  i128 p = 1;
  for (int32_t i = 0; i < M; ++i) { p *= nd[i]; if (p > ((i128)1 << 62)) return -1; }
  return (int64_t)p;
}

typedef struct {
  const hs_entry* table; const int32_t* nd; int32_t M; int64_t lo, hi;
  double best; int64_t idx; int64_t feas;
} best_job_t;

static void* best_worker(void* arg) {
  best_job_t* j = (best_job_t*)arg;
  double b = 0.0; int64_t bi = -1; int64_t feas = 0;
  int32_t digit[HS_MAX_MACHINES];
  int64_t x = j->lo;
  for (int32_t i = j->M - 1; i >= 0; --i) { digit[i] = (int32_t)(x % j->nd[i]); x /= j->nd[i]; }
  for (int64_t c = j->lo; c < j->hi; ++c) {
    int32_t fb;
    double t = table_total(j->table, j->M, digit, &fb);
    if (fb < 0) {
      ++feas;
      if (bi < 0 || t > b) { b = t; bi = c; }
    }
    for (int32_t i = j->M - 1; i >= 0; --i) { if (++digit[i] < j->nd[i]) break; digit[i] = 0; }
  }
  j->best = b; j->idx = bi; j->feas = feas;
  return NULL;
}

int hs_oracle_best(const hs_entry* table, const int32_t* nd, int32_t M, int64_t begin, int64_t end,
                   int nthreads, hs_cand* best, int64_t* n_feasible) {
  int64_t P = space_size(nd, M);
  if (P < 0 || begin < 0 || end > P || begin > end) return HS_ERR_ARG;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  best_job_t jobs[256];
  pthread_t th[256];
  int64_t chunk = (end - begin + nthreads - 1) / nthreads;
  for (int k = 0; k < nthreads; ++k) {
    int64_t lo = begin + chunk * k, hi = lo + chunk;
    if (lo > end) lo = end;
    if (hi > end) hi = end;
    best_job_t jb = {table, nd, M, lo, hi, 0.0, -1, 0};
    jobs[k] = jb;
    pthread_create(&th[k], NULL, best_worker, &jobs[k]);
  }
  double g_best = 0.0; int64_t g_idx = -1; int64_t g_feas = 0;
  for (int k = 0; k < nthreads; ++k) {
    pthread_join(th[k], NULL);
    g_feas += jobs[k].feas;
    if (jobs[k].idx >= 0 && (g_idx < 0 || jobs[k].best > g_best)) { g_best = jobs[k].best; g_idx = jobs[k].idx; }
  }
  best->total = g_best;
  best->index = g_idx;
  *n_feasible = g_feas;
  return HS_OK;
}

/* top-k of planner.py:227's order over shard `shard` of the feasible
 * sub-product (same contract as hs_search_topk): enumerate, keep the k best
 * in a heap whose root is the worst kept candidate. */
static int cmp_cand(const void* a, const void* b);
static int cand_worse(const hs_cand* a, const hs_cand* b) { /* a ranks after b */
  double ka = -a->total, kb = -b->total;
  if (ka != kb) return ka > kb;
  return a->index > b->index;
}
static void worst_sift_down(hs_cand* h, int64_t n, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && cand_worse(&h[l], &h[m])) m = l;
    if (r < n && cand_worse(&h[r], &h[m])) m = r;
    if (m == i) return;
    hs_cand t = h[i]; h[i] = h[m]; h[m] = t; i = m;
  }
}
int hs_oracle_topk(const hs_entry* table, const int32_t* nd, int32_t M, int64_t k, int32_t shard, int32_t n_shards,
                   hs_cand* out, int64_t* n_out, int64_t* n_feasible) {
  int32_t D[HS_MAX_MACHINES], orig[HS_MAX_MACHINES][HS_MAX_DEGREES];
  double C[HS_MAX_MACHINES][HS_MAX_DEGREES];
  int64_t stride[HS_MAX_MACHINES];
  int64_t st = 1;
  i128 F = 1;
  for (int32_t i = M - 1; i >= 0; --i) {
    stride[i] = st;
    st *= nd[i];
    int32_t ok = 0;
    for (int32_t d = 0; d < nd[i]; ++d) {
      const hs_entry* e = &table[i * HS_MAX_DEGREES + d];
      if (e->status != HS_ENTRY_OK) continue;
      C[i][ok] = e->contribution;
      orig[i][ok] = d;
      ++ok;
    }
    D[i] = ok;
    F *= ok;
  }
  *n_out = 0;
  *n_feasible = 0;
  if (F == 0) return HS_OK;
  int64_t items = (int64_t)(F / D[M - 1]);
  int64_t ib = items * shard / n_shards, ie = items * (shard + 1) / n_shards;
  *n_feasible = (ie - ib) * D[M - 1];
  int32_t dig[HS_MAX_MACHINES];
  int64_t x = ib;
  for (int32_t i = M - 2; i >= 0; --i) { dig[i] = (int32_t)(x % D[i]); x /= D[i]; }
  int64_t n = 0;
  for (int64_t it = ib; it < ie; ++it) {
    double pre = 0.0;
    int64_t pidx = 0;
    for (int32_t i = 0; i < M - 1; ++i) { pre = pre + C[i][dig[i]]; pidx += (int64_t)orig[i][dig[i]] * stride[i]; }
    for (int32_t d = 0; d < D[M - 1]; ++d) {
      hs_cand c = {pre + C[M - 1][d], pidx + (int64_t)orig[M - 1][d] * stride[M - 1]};
      if (n < k) {
        out[n] = c;
        int64_t i = n++;
        while (i > 0) {
          int64_t p = (i - 1) / 2;
          if (!cand_worse(&out[i], &out[p])) break;
          hs_cand t = out[i]; out[i] = out[p]; out[p] = t; i = p;
        }
      } else if (k > 0 && cand_worse(&out[0], &c)) {
        out[0] = c;
        worst_sift_down(out, n, 0);
      }
    }
    for (int32_t i = M - 2; i >= 0; --i) { if (++dig[i] < D[i]) break; dig[i] = 0; }
  }
  qsort(out, (size_t)n, sizeof(hs_cand), cmp_cand);
  *n_out = n;
  return HS_OK;
}

/* planner.py:227 ranked.sort(key=(-total, tp tuple)): stable sort of the
 * feasible candidates (product order) by descending total. */
static int cmp_cand(const void* a, const void* b) {
  const hs_cand* x = (const hs_cand*)a;
  const hs_cand* y = (const hs_cand*)b;
  double kx = -x->total, ky = -y->total;
  if (kx < ky) return -1;
  if (kx > ky) return 1;
  return (x->index > y->index) - (x->index < y->index);
}

int hs_oracle_rank(const hs_entry* table, const int32_t* nd, int32_t M, hs_cand* ranked,
                   int64_t* n_ranked, int8_t* first_bad) {
  int64_t P = space_size(nd, M);
  if (P < 0) return HS_ERR_ARG;
  int32_t digit[HS_MAX_MACHINES];
  for (int32_t i = 0; i < M; ++i) digit[i] = 0;
  int64_t n = 0;
  for (int64_t c = 0; c < P; ++c) {
    int32_t fb;
    double t = table_total(table, M, digit, &fb);
    first_bad[c] = (int8_t)fb;
    if (fb < 0) { ranked[n].total = t; ranked[n].index = c; ++n; }
    for (int32_t i = M - 1; i >= 0; --i) { if (++digit[i] < nd[i]) break; digit[i] = 0; }
  }
  qsort(ranked, (size_t)n, sizeof(hs_cand), cmp_cand);
  *n_ranked = n;
  return HS_OK;
}

/* ------------------------------------------------------------------------
 * Replay: simulator.py:272-363 run_continuous with the Scheduler of
 * scheduling.py:175-346, literal data structures (event heap, FCFS deque,
 * active list with order-preserving removal, O(N^2) min-max mapping).
 * ---------------------------------------------------------------------- */
typedef struct { double t; int32_t kind; int64_t tb; } ev_t;

static int ev_less(const ev_t* a, const ev_t* b) {
  if (a->t != b->t) return a->t < b->t;
  if (a->kind != b->kind) return a->kind < b->kind;
  return a->tb < b->tb;
}
typedef struct { ev_t* v; int64_t n, cap; } heap_t;
static void heap_push(heap_t* h, ev_t e) {
  if (h->n == h->cap) { h->cap = h->cap ? h->cap * 2 : 64; h->v = (ev_t*)realloc(h->v, sizeof(ev_t) * h->cap); }
  int64_t i = h->n++;
  h->v[i] = e;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_less(&h->v[i], &h->v[p])) break;
    ev_t tmp = h->v[i]; h->v[i] = h->v[p]; h->v[p] = tmp; i = p;
  }
}
static ev_t heap_pop(heap_t* h) {
  ev_t top = h->v[0];
  h->v[0] = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && ev_less(&h->v[l], &h->v[m])) m = l;
    if (r < h->n && ev_less(&h->v[r], &h->v[m])) m = r;
    if (m == i) break;
    ev_t tmp = h->v[i]; h->v[i] = h->v[m]; h->v[m] = tmp; i = m;
  }
  return top;
}

typedef struct { int64_t req; int64_t generated; } running_t;

typedef struct {
  /* _InstanceRun (simulator.py:259-269) */
  int64_t* queue; int64_t qh, qt;        /* deque as a ring over request ids */
  running_t* active; int64_t n_active, cap_active;
  int64_t reserved;
  int step_scheduled;
  double completion_time, peak;
  int64_t request_count, token_count;
  /* InstanceState (scheduling.py:157-164) */
  double load;
  int64_t run_i, run_p;
  double wrr_cur;
} inst_t;

int hs_oracle_replay_one(const hs_instance* inst, const hs_policy* pol, const int32_t* I,
                         const int32_t* O, const int32_t* P, const double* arrival, int64_t q,
                         uint8_t* assign, double* depart, hs_inst_metrics* metrics,
                         hs_trace_result* res) {
  const int32_t N = pol->n_instances;
  const int64_t per_token = pol->per_token;
  memset(res, 0, sizeof(*res));
  res->err_instance = -1;
  res->err_request = -1;
  inst_t* st = (inst_t*)calloc((size_t)N, sizeof(inst_t));
  double* w_rec = (double*)malloc(sizeof(double) * (q > 0 ? q : 1));
  for (int32_t j = 0; j < N; ++j) {
    st[j].queue = (int64_t*)malloc(sizeof(int64_t) * (q > 0 ? q : 1));
    st[j].cap_active = 16;
    st[j].active = (running_t*)malloc(sizeof(running_t) * 16);
  }
  double* weights = (double*)malloc(sizeof(double) * N);
  int64_t rr_next = 0;
  /* scheduling.py:326 total = sum(weights[i] for i in candidates) */
  double wrr_total = 0.0;
  if (pol->policy == HS_POLICY_WRR) {
    pysum_t s; pysum_init(&s);
    for (int32_t j = 0; j < N; ++j) pysum_add(&s, inst[j].wrr_weight);
    wrr_total = pysum_result(&s);
  }
  heap_t ev = {0, 0, 0};
  const int is_static = pol->mode == 1;
  for (int64_t s = 0; s < q; ++s) {
    ev_t e = {arrival ? arrival[s] : 0.0, 0, s};
    heap_push(&ev, e);
  }
  int err = 0;
  int64_t steps = 0;
  while (ev.n > 0 && !err) {
    ev_t e = heap_pop(&ev);
    double t = e.t;
    if (e.kind == 0) {
      /* ARRIVAL (simulator.py:320-328): choose (scheduling.py:235-254) */
      int64_t r = e.tb;
      int32_t chosen = -1;
      int evaluate_all = pol->policy == HS_POLICY_OS || pol->policy == HS_POLICY_MB;
      if (!evaluate_all) {
        if (pol->policy == HS_POLICY_SI) chosen = 0;
        else if (pol->policy == HS_POLICY_RR) { chosen = (int32_t)(rr_next % N); rr_next += 1; }
        else {
          chosen = 0;
          for (int32_t j = 0; j < N; ++j) {
            st[j].wrr_cur += inst[j].wrr_weight;
            if (st[j].wrr_cur > st[chosen].wrr_cur) chosen = j;
          }
          st[chosen].wrr_cur -= wrr_total;
        }
      }
      /* evaluate (scheduling.py:216-233) */
      for (int32_t j = 0; j < N && !err; ++j) {
        if (!evaluate_all && j != chosen) { weights[j] = INFINITY; continue; }
        double cost;
        if (pol->policy == HS_POLICY_MB) {
          cost = 1.0;
        } else {
          /* scheduling.py:119-128 ideal_batch_size */
          i128 per_req = (i128)per_token * ((int64_t)I[r] + P[r]);
          double fl = hs_oracle_floordiv(inst[j].budget, i128_to_double(per_req));
          int64_t b = (int64_t)fl;
          if (b < 1) b = 1;
          /* scheduling.py:136-147 per_request_cost */
          double total = prefill(inst[j].p, b, I[r]) + decode_total(inst[j].p, b, I[r], P[r]);
          if (total <= 0) {
            err = HS_TRACE_NONPOSITIVE_COST; res->err_instance = j; res->err_request = r; res->err_value = total;
            break;
          }
          cost = total / (double)b;
        }
        /* capacity.py:98-106 kv_usage, scheduling.py:150-154 workload */
        double usage = i128_to_double((i128)per_token * (st[j].run_i + st[j].run_p)) / inst[j].budget;
        int of;
        double ex = hs_oracle_exp(pol->theta * usage, &of);
        if (of) {
          err = HS_TRACE_EXP_OVERFLOW; res->err_instance = j; res->err_request = r; res->err_value = pol->theta * usage;
          break;
        }
        weights[j] = cost * ex;
      }
      if (err) break;
      if (evaluate_all) {
        /* scheduling.py:299-312 _min_max_choice, literal O(N^2) */
        double best_peak = INFINITY;
        int32_t best_idx = -1;
        for (int32_t s = 0; s < N; ++s) {
          double w = weights[s];
          if (isinf(w)) continue;
          double peak = 0.0;
          for (int32_t j = 0; j < N; ++j) {
            double v = st[j].load + (j == s ? w : 0.0);
            if (j == 0 || v > peak) peak = v;
          }
          if (peak < best_peak) { best_peak = peak; best_idx = s; }
        }
        if (best_idx < 0) { err = HS_TRACE_NO_INSTANCE; res->err_request = r; break; }
        chosen = best_idx;
      }
      /* _commit (scheduling.py:335-346) */
      st[chosen].load += weights[chosen];
      st[chosen].run_i += I[r];
      st[chosen].run_p += P[r];
      w_rec[r] = weights[chosen];
      if (assign) assign[r] = (uint8_t)chosen;
      st[chosen].queue[st[chosen].qt++] = r;
      if (is_static) continue; /* run_static: dispatch everything first (simulator.py:216-220) */
      if (!st[chosen].step_scheduled) {
        st[chosen].step_scheduled = 1;
        ev_t se = {t, 1, chosen};
        heap_push(&ev, se);
      }
      continue;
    }
    /* STEP (simulator.py:330-355) */
    int32_t j = (int32_t)e.tb;
    inst_t* run = &st[j];
    run->step_scheduled = 0;
    ++steps;
    /* retire, in active-list order */
    int64_t w = 0;
    for (int64_t a = 0; a < run->n_active; ++a) {
      running_t rr = run->active[a];
      if (rr.generated >= O[rr.req]) {
        int64_t r = rr.req;
        run->reserved -= (int64_t)I[r] + O[r];
        run->completion_time = t;
        run->request_count += 1;
        run->token_count += (int64_t)I[r] + O[r];
        if (depart) depart[r] = t;
        /* Scheduler.complete (scheduling.py:256-264) */
        run->load -= w_rec[r];
        run->run_i -= I[r];
        run->run_p -= P[r];
        if (run->run_i < 0 || run->run_p < 0) {
          err = HS_TRACE_NEGATIVE_RUNNING; res->err_instance = j; res->err_request = r;
        }
      } else {
        run->active[w++] = rr;
      }
    }
    run->n_active = w;
    if (err) break;
    /* admit (simulator.py:297-316) */
    double budget = inst[j].budget;
    int64_t newly = 0, max_i_new = 0;
    while (run->qh < run->qt) {
      int64_t r = run->queue[run->qh];
      int64_t need = (int64_t)I[r] + O[r];
      if (i128_gt_double((i128)per_token * (run->reserved + need), budget)) {
        if (run->n_active == 0 && newly == 0) {
          err = HS_TRACE_INFEASIBLE_REQUEST; res->err_instance = j; res->err_request = r;
        }
        break;
      }
      run->qh++;
      run->reserved += need;
      if (run->n_active + newly == run->cap_active) {
        run->cap_active *= 2;
        run->active = (running_t*)realloc(run->active, sizeof(running_t) * run->cap_active);
      }
      run->active[run->n_active + newly].req = r;
      run->active[run->n_active + newly].generated = 0;
      if (I[r] > max_i_new) max_i_new = I[r];
      ++newly;
    }
    if (err) break;
    if (newly) {
      double u = i128_to_double((i128)per_token * run->reserved) / budget;
      if (u > run->peak) run->peak = u;
    }
    if (run->n_active == 0 && newly == 0) continue;
    double cost = 0.0;
    if (newly) cost += prefill(inst[j].p, newly, max_i_new);
    run->n_active += newly;
    int64_t cached = 0;
    for (int64_t a = 0; a < run->n_active; ++a) {
      int64_t c = (int64_t)I[run->active[a].req] + run->active[a].generated + 1;
      if (a == 0 || c > cached) cached = c;
    }
    cost += decode_iter(inst[j].p, cached, run->n_active);
    for (int64_t a = 0; a < run->n_active; ++a) run->active[a].generated += 1;
    run->step_scheduled = 1;
    ev_t se = {t + cost, 1, j};
    heap_push(&ev, se);
  }
  if (!err && is_static) {
    /* simulator.py:229-247: per instance, plan_static_batches over its
     * assigned requests (planner.py:51-87), clock += estimate_batch_time,
     * complete() in batch order; the first failing instance raises. */
    for (int32_t j = 0; j < N && !err; ++j) {
      inst_t* run = &st[j];
      double clock = 0.0;
      int64_t a = run->qh;
      while (a < run->qt) {
        i128 input_sum = 0;
        int64_t max_o = 0, b = a;
        while (b < run->qt) {
          int64_t r = run->queue[b];
          i128 ci = input_sum + I[r];
          int64_t cmo = max_o > O[r] ? max_o : O[r];
          int64_t width = b - a + 1;
          i128 reserved = (i128)per_token * ci + (i128)width * per_token * cmo;
          if (i128_gt_double(reserved, inst[j].budget)) break;
          input_sum = ci;
          max_o = cmo;
          ++b;
        }
        if (b == a) {
          err = HS_TRACE_INFEASIBLE_REQUEST; res->err_instance = j; res->err_request = run->queue[a];
          break;
        }
        int64_t si = 0, mi = 0, mo = 0;
        for (int64_t x = a; x < b; ++x) {
          int64_t r = run->queue[x];
          si += I[r];
          if (I[r] > mi) mi = I[r];
          if (O[r] > mo) mo = O[r];
        }
        i128 reserved = (i128)per_token * (si + (b - a) * mo);
        double u = i128_to_double(reserved) / inst[j].budget;
        if (u > run->peak) run->peak = u;
        clock += prefill(inst[j].p, b - a, mi) + decode_total(inst[j].p, b - a, mi, mo);
        for (int64_t x = a; x < b; ++x) {
          int64_t r = run->queue[x];
          run->load -= w_rec[r];
          run->run_i -= I[r];
          run->run_p -= P[r];
          if (depart) depart[r] = clock;
          run->token_count += (int64_t)I[r] + O[r];
          run->request_count += 1;
        }
        a = b;
      }
      run->completion_time = clock;
    }
  }
  res->error = err;
  res->n_steps = steps;
  for (int32_t j = 0; j < N; ++j) {
    metrics[j].completion_time = st[j].completion_time;
    metrics[j].peak_kv_usage = st[j].peak;
    metrics[j].residual_load = st[j].load;
    metrics[j].request_count = st[j].request_count;
    metrics[j].token_count = st[j].token_count;
    free(st[j].queue);
    free(st[j].active);
  }
  free(ev.v);
  free(st);
  free(w_rec);
  free(weights);
  return HS_OK;
}

typedef struct {
  const hs_instance* inst; const hs_policy* pol; const hs_trace_batch* b;
  uint8_t* assign; double* depart; hs_inst_metrics* metrics; hs_trace_result* result;
  int64_t* next; pthread_mutex_t* mu;
} rep_job_t;

static void* replay_worker(void* arg) {
  rep_job_t* j = (rep_job_t*)arg;
  for (;;) {
    pthread_mutex_lock(j->mu);
    int64_t t = (*j->next)++;
    pthread_mutex_unlock(j->mu);
    if (t >= j->b->n_traces) break;
    int64_t o = j->b->offsets[t], q = j->b->offsets[t + 1] - o;
    hs_oracle_replay_one(j->inst, j->pol, j->b->input_len + o, j->b->output_len + o,
                         j->b->pred_output_len + o, j->b->arrival ? j->b->arrival + o : NULL, q,
                         j->assign ? j->assign + o : NULL, j->depart ? j->depart + o : NULL,
                         j->metrics + t * j->pol->n_instances, j->result + t);
  }
  return NULL;
}

int hs_oracle_replay(const hs_instance* inst, const hs_policy* pol, const hs_trace_batch* b,
                     int nthreads, uint8_t* assign, double* depart, hs_inst_metrics* metrics,
                     hs_trace_result* result) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  int64_t next = 0;
  rep_job_t job = {inst, pol, b, assign, depart, metrics, result, &next, &mu};
  for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, replay_worker, &job);
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  return HS_OK;
}

/* Batch forms for the exp tests: the port above, and libm's exp itself (the
 * function CPython's math.exp calls), over an array. */
void hs_oracle_exp_batch(const double* x, int64_t n, double* y, uint8_t* of) {
  for (int64_t i = 0; i < n; ++i) {
    int o;
    y[i] = hs_oracle_exp(x[i], &o);
    of[i] = (uint8_t)o;
  }
}
void hs_libm_exp_batch(const double* x, int64_t n, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = exp(x[i]);
}
