/*
 * hetserve_b200.h -- C ABI of the B200-native engine for the data-parallel
 * core of arXiv 2504.15303 (reference package `hetserve`).
 *
 * Every entry point replaces one reference Python function on the hot path
 * (paths relative to /root/reference/pkg/src/hetserve):
 *
 *   hs_search_tables   planner.py:143-181 estimate_system_throughput, one
 *                      machine at a time, for every (machine, tp degree):
 *                      capacity.py:72-95 kv_budget/check_memory_constraint,
 *                      planner.py:51-87 plan_static_batches,
 *                      planner.py:90-118 estimate_batch_time/time_batches/
 *                      estimate_instance_throughput.
 *   hs_search_best     planner.py:213-228 search_optimal_config product loop,
 *                      reduced to (best total, lowest index) over an index
 *                      range of the mixed-radix candidate space.
 *   hs_search_rank     planner.py:213-228 again, full ranking (ranked.sort
 *                      key (-total, tp tuple)) for spaces small enough to
 *                      materialise.
 *   hs_replay          simulator.py:272-363 run_continuous (or, with
 *                      hs_policy.mode = 1, simulator.py:206-250 run_static)
 *                      with scheduling.py:216-346 Scheduler.evaluate/choose/
 *                      complete, for a batch of independent traces.
 *
 * Conventions: plain pointers and sizes, caller-owned host buffers, calls are
 * synchronous (the reference API is synchronous).  One context per thread.
 * Return value: HS_OK or an hs_status code; hs_last_error() gives text.
 * Domain-level failures that the reference raises as exceptions are NOT call
 * failures: they are reported per table entry (hs_entry.status) or per trace
 * (hs_trace_result.error) so the Python shim can raise the same exception
 * type with the same fields.
 */
#ifndef HETSERVE_B200_H
#define HETSERVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 4
#define HS_MAX_DEGREES 32   /* power-of-two divisors of an accelerator count  */
#define HS_MAX_MACHINES 64
#define HS_MAX_INSTANCES 255 /* one lane per instance, up to 8 warps per trace; uint8 assignments */
#define HS_MAX_CLASSES 32    /* distinct (params, budget) instance classes      */

/* call status */
enum hs_status {
  HS_OK = 0,
  HS_ERR_ARG = 1,          /* bad argument (null pointer, size out of range) */
  HS_ERR_CUDA = 2,         /* CUDA runtime failure                           */
  HS_ERR_UNSUPPORTED = 3,  /* valid input the engine does not handle yet     */
  HS_ERR_NOMEM = 4
};

/* Per-(machine, degree) outcome: which exception estimate_system_throughput
 * (planner.py:143-181) raises for that machine, if any. */
enum hs_entry_status {
  HS_ENTRY_OK = 0,
  HS_ENTRY_INFEASIBLE_CONFIG = 1,  /* planner.py:156-163 InfeasibleConfigError */
  HS_ENTRY_MISSING_PARAMS = 2,     /* planner.py:164-166 SpecError             */
  HS_ENTRY_INFEASIBLE_REQUEST = 3, /* planner.py:78-84 InfeasibleRequestError  */
  HS_ENTRY_ZERO_DIVISION = 4,      /* planner.py:118 ZeroDivisionError (NOT caught
                                      by search_optimal_config: aborts it)     */
  HS_ENTRY_BAD_DEGREE = 5          /* capacity.py:79-83 SpecError (degree does
                                      not divide the named machine's count)    */
};

/* scheduling policies, scheduling.py:41 POLICIES */
enum hs_policy_kind { HS_POLICY_OS = 0, HS_POLICY_RR = 1, HS_POLICY_WRR = 2, HS_POLICY_SI = 3, HS_POLICY_MB = 4 };

/* Per-trace outcome of a replay: the exception run_continuous would raise. */
enum hs_trace_error {
  HS_TRACE_OK = 0,
  HS_TRACE_INFEASIBLE_REQUEST = 1, /* simulator.py:304-309 admit()                 */
  HS_TRACE_NONPOSITIVE_COST = 2,   /* scheduling.py:143-146 per_request_cost SpecError */
  HS_TRACE_EXP_OVERFLOW = 3,       /* scheduling.py:154 math.exp OverflowError      */
  HS_TRACE_NO_INSTANCE = 4,        /* scheduling.py:310-311 SchedulingError         */
  HS_TRACE_NEGATIVE_RUNNING = 5,   /* capacity.py:50-52 SpecError                   */
  HS_TRACE_CAPACITY = 6,           /* engine limit: active-set bound exceeded        */
  HS_TRACE_STALLED = 7             /* engine: streamed inputs did not arrive in time */
};

/* core.py:45-56 ModelSpec */
typedef struct {
  int64_t layers, hidden_dim, param_count, bytes_per_param;
} hs_model;

/* core.py:75-88 EngineOverheads */
typedef struct {
  double mem_utilization_fraction;
  int64_t static_overhead_bytes;
} hs_engine;

/* core.py:91-100 WorkloadLimits */
typedef struct {
  int64_t max_input_len, max_output_len;
} hs_limits;

/* core.py:59-72 MachineSpec, plus the index of the machine whose spec
 * cluster.machine(name) resolves to (core.py:161-165: first machine with that
 * name; == own index when names are unique).  fixed_degree = 0 enumerates
 * the machine's degrees (core.py:363-371); > 0 evaluates that one degree
 * (an explicit DeploymentConfig placement, planner.py:143-181). */
typedef struct {
  int64_t accelerator_count;
  int64_t accelerator_mem_bytes;
  int32_t spec_index;
  int32_t fixed_degree;
} hs_machine;

/* One (machine, degree) table entry = planner.py:167-179 MachineEstimate
 * plus the failure that replaces it. */
typedef struct {
  double contribution;   /* machine_tokens_per_sec = rate * instance_count */
  double rate;           /* instance_tokens_per_sec                      */
  double budget;         /* KV budget bytes (may be <= 0)                */
  double slack;          /* budget - required bytes                      */
  int64_t instance_count;
  int64_t bad_request;   /* request index for HS_ENTRY_INFEASIBLE_REQUEST */
  int64_t token_count;   /* sum(I + O) over the trace                      */
  int32_t tp_degree;
  int32_t status;        /* hs_entry_status */
  int32_t zero_div_int;  /* 1 when total_time was the int 0 (empty plan)   */
  int32_t _pad;
} hs_entry;

/* One candidate: (total, mixed-radix index; machine 0 most significant). */
typedef struct {
  double total;
  int64_t index;
} hs_cand;

/* Schedulable instance (scheduling.py:44-52 InstanceHandle). */
typedef struct {
  double p[8];           /* LatencyParams p1..p8 (latency.py:36-51)         */
  double budget;         /* KvBudget.total_bytes (> 0)                       */
  double wrr_weight;     /* PolicyConfig.wrr_weights[i] (WRR only)           */
  int32_t type;          /* class id: instances with bit-identical (p, budget)
                            share one; 0 <= type < n_instances              */
  int32_t _pad;
} hs_instance;

/* scheduling.py:98-116 PolicyConfig (predictor is applied host-side: the
 * engine consumes the predicted lengths as an array). */
typedef struct {
  int32_t policy;        /* hs_policy_kind */
  int32_t n_instances;
  double theta;
  int64_t per_token;     /* capacity.py:67-69 kv_bytes_per_token */
  int32_t mode;          /* 0 continuous batching (simulator.py:272-363),
                            1 static batching (simulator.py:206-250; rate=inf) */
  int32_t flags;         /* HS_REPLAY_* bits */
} hs_policy;

/* hs_policy.flags: `depart` receives three doubles per request instead of
 * one -- (departure time, heap key, per-instance sequence).  The reference's
 * event heap (simulator.py:285-355) pops a retiring step once every earlier
 * step of the instance's busy period has popped, so request_times order =
 * sort by (heap key, instance, sequence); the heap key is the running max of
 * the instance's step times since it last went idle (== the departure time
 * whenever step costs are non-negative). */
#define HS_REPLAY_ORDER_KEYS 1

/* simulator.py:82-88 InstanceMetrics + scheduler.loads() residual. */
typedef struct {
  double completion_time;
  double peak_kv_usage;
  double residual_load;
  int64_t request_count;
  int64_t token_count;
} hs_inst_metrics;

typedef struct {
  int32_t error;         /* hs_trace_error */
  int32_t err_instance;  /* instance index involved (or -1) */
  int64_t err_request;   /* request index within the trace (or -1) */
  double err_value;      /* offending value (e.g. non-positive batch time) */
  int64_t n_steps;       /* step events executed (statistics) */
} hs_trace_result;

/* A batch of traces laid out back to back (SoA).  Trace t owns requests
 * [offsets[t], offsets[t+1]).  arrival == NULL means rate = inf (all 0.0,
 * simulator.py:117-118). */
typedef struct {
  int64_t n_traces;
  const int64_t* offsets;
  const int32_t* input_len;
  const int32_t* output_len;
  const int32_t* pred_output_len;
  const double* arrival;
} hs_trace_batch;

/* ---- synthetic workload streams (numpy Generator(PCG64)) ---------------
 * The reference draws its synthetic inputs from numpy.random.default_rng(seed)
 * (numpy 2.3, bit generator PCG64 / XSL-RR 128/64):
 *   cli.py:160-193        gen-trace lengths: lognormal(mu, sigma) or
 *                         integers(lo, hi + 1), then int(min(max(round(v), 1), cap))
 *   simulator.py:112-124  arrivals: cumsum(exponential(1 / rate, q))
 *   scheduling.py:87-95   predictor: int(min(max(round(normal(mean, sd)), 1), cap))
 * hs_pcg64_state is numpy's pcg64_state: the 128-bit LCG state and increment
 * plus the buffered upper half a 32-bit draw leaves behind. */
typedef struct {
  uint64_t state_hi, state_lo;
  uint64_t inc_hi, inc_lo;
  uint32_t has_uint32;
  uint32_t uinteger;
} hs_pcg64_state;

typedef enum {
  HS_DIST_LOGNORMAL_LEN = 0, /* int32: clamp(round(exp(p0 + p1 * N(0,1))), 1, cap) */
  HS_DIST_UNIFORM_LEN = 1,   /* int32: clamp(integers(lo, hi + 1), 1, cap)          */
  HS_DIST_EXP_CUMSUM = 2,    /* fp64:  running sum of p0 * Exp(1)                  */
  HS_DIST_NORMAL_LEN = 3     /* int32: clamp(round(p0 + p1 * N(0,1)), 1, cap)       */
} hs_dist_kind;

typedef struct {
  int32_t kind;  /* hs_dist_kind */
  int32_t cap;   /* upper clamp of the *_LEN kinds (max_input_len / max_output_len) */
  int64_t lo;    /* UNIFORM_LEN: inclusive bounds, lo <= hi */
  int64_t hi;
  double p0;     /* LOGNORMAL: mu; EXP_CUMSUM: scale (= 1 / rate); NORMAL: mean */
  double p1;     /* LOGNORMAL: sigma; NORMAL: stddev */
} hs_dist;

/* Device generation of the seeded streams hs_replay_seeded consumes. */
typedef struct {
  const hs_pcg64_state* arrival_state;   /* [n_traces] or NULL (use batch->arrival) */
  double arrival_scale;                  /* 1 / rate */
  const hs_pcg64_state* predictor_state; /* [n_traces] or NULL (use batch->pred_output_len) */
  double pred_mean, pred_stddev;         /* predictor mode "normal" */
  int32_t pred_cap;                      /* limits.max_output_len */
  int32_t _pad;
} hs_replay_seeds;

typedef struct hs_ctx hs_ctx;

/* ---- context ---------------------------------------------------------- */
int hs_abi_version(void);
int hs_ctx_create(int device, hs_ctx** out);
int hs_ctx_destroy(hs_ctx* ctx);
const char* hs_last_error(void);
/* Kernel launches issued by this context since creation (evidence counter). */
int64_t hs_ctx_launch_count(const hs_ctx* ctx);
/* Device milliseconds of the last call's main kernel(s) (CUDA events on the
 * context's stream around the launches only: no copies, no host work). */
double hs_ctx_last_kernel_ms(const hs_ctx* ctx);
/* The context's cudaStream_t (so callers can bracket work with events). */
void* hs_ctx_stream(const hs_ctx* ctx);
/* Diagnostic: measured FP64 add throughput of this device (DADD/s). */
int hs_probe_fp64(hs_ctx* ctx, double* dadd_per_s);
/* CPython's math.exp (glibc 2.39, FMA ifunc body) as the replay kernels
 * evaluate it for workload() (scheduling.py:154): y[i] = exp(x[i]) and
 * overflow[i] = 1 where math.exp raises OverflowError.  Host arrays. */
int hs_exp_batch(hs_ctx* ctx, const double* x, int64_t n, double* y, uint8_t* overflow);
/* CPython float floor division x // w as the replay kernels evaluate it for
 * ideal_batch_size (scheduling.py:128: budget // (per_token * tokens)):
 * y[i] = x[i] // w[i].  Host arrays. */
int hs_floordiv_batch(hs_ctx* ctx, const double* x, const double* w, int64_t n, double* y);

/* The IEEE quotient x / b as the replay kernels evaluate kv_usage
 * (capacity.py:98-106: per_token * running_tokens / budget): from RN(1 / b)
 * with one FMA correction.  y[i] = x[i] / b[i], b finite and positive.  Host
 * arrays. */
int hs_div_batch(hs_ctx* ctx, const double* x, const double* b, int64_t n, double* y);

/* ---- deployment search ------------------------------------------------ */
/* Fill table[i * HS_MAX_DEGREES + d] for d < n_degrees[i] (degree list =
 * core.py:363-371 enumerate_tp_degrees of machines[i]).  params is
 * [M][HS_MAX_DEGREES][8] and params_present [M][HS_MAX_DEGREES], indexed by
 * the same degree position.  I/O are the trace's input/output lengths. */
int hs_search_tables(hs_ctx* ctx, const hs_model* model, const hs_engine* engine,
                     const hs_limits* limits, const hs_machine* machines, int32_t n_machines,
                     const double* params, const uint8_t* params_present,
                     const int32_t* input_len, const int32_t* output_len, int64_t n_requests,
                     hs_entry* table, int32_t* n_degrees);

/* planner.py:51-118 for ONE instance with an explicit KV budget (one warp):
 * plan_static_batches -> batch b is [stops[b-1], stops[b]) (stops[-1] = 0),
 * time_batches -> times[b] (estimate_batch_time, when params != NULL), and
 * estimate_instance_throughput -> entry->rate, with entry->status /
 * bad_request / zero_div_int as hs_search_tables reports them.  I, O, stops,
 * times are host arrays (stops / times with room for q entries). */
int hs_plan_instance(hs_ctx* ctx, double budget, int64_t per_token, const double* params, const int32_t* I,
                     const int32_t* O, int64_t q, int64_t* stops, double* times, int64_t* n_batches,
                     hs_entry* entry);

/* Argmax over candidate indices [begin, end) of the product space defined
 * by (table, n_degrees): best = max total, ties -> lowest index
 * (planner.py:227).  *n_feasible receives the number of feasible candidates
 * in the range.  best->index = -1 when none is feasible.  Every candidate is
 * decided: an infeasible one has a non-OK (machine, degree) entry and can
 * never win, so the kernel scores the feasible sub-product only (per machine
 * its OK degrees, an order-preserving compression of the mixed radix);
 * environment HS_SEARCH_EXHAUSTIVE=1 scores every candidate instead. */
int hs_search_best(hs_ctx* ctx, const hs_entry* table, const int32_t* n_degrees, int32_t n_machines,
                   int64_t begin, int64_t end, hs_cand* best, int64_t* n_feasible);

/* Rank every candidate of the space (size <= 2^26): feasible ones into
 * ranked[0 .. *n_ranked) ordered by (-total, index); for every candidate,
 * first_bad[c] = index of the first machine (config order) whose entry is
 * not OK, or -1 when feasible. */
int hs_search_rank(hs_ctx* ctx, const hs_entry* table, const int32_t* n_degrees, int32_t n_machines,
                   hs_cand* ranked, int64_t* n_ranked, int8_t* first_bad);

/* Top-k of the ranking (planner.py:227 order: total desc, index asc) over
 * shard `shard` of `n_shards` equal blocks of the FEASIBLE sub-product
 * (only feasible candidates are ranked).  out[0 .. *n_out) is sorted;
 * *n_feasible = feasible candidates in the shard.  Shard results merge by
 * the same order. */
int hs_search_topk(hs_ctx* ctx, const hs_entry* table, const int32_t* n_degrees, int32_t n_machines, int64_t k,
                   int32_t shard, int32_t n_shards, hs_cand* out, int64_t* n_out, int64_t* n_feasible);

/* The ranking streamed: the best k feasible candidates ranked AFTER the
 * candidate (after_total, after_index) in planner.py:227 order (total desc,
 * index asc) -- repeated calls with the last result as the boundary walk the
 * whole ranking of any space (hs_search_rank materialises at most 2^26).
 * after_index < 0: from the top.  *n_feasible = all feasible candidates. */
int hs_search_topk_after(hs_ctx* ctx, const hs_entry* table, const int32_t* n_degrees, int32_t n_machines, int64_t k,
                         double after_total, int64_t after_index, hs_cand* out, int64_t* n_out, int64_t* n_feasible);

/* ---- batched scheduler replay ------------------------------------------ */
/* Replay every trace of the batch on the same instance set.  assign
 * ([total requests], may be NULL) receives the chosen instance per request
 * (page-locked, device-mapped memory -- e.g. hs_host_alloc -- is written by the
 * kernel in place while it runs); depart ([total requests], may be NULL) the
 * departure time; metrics is [n_traces][n_instances]; result is [n_traces]. */
int hs_replay(hs_ctx* ctx, const hs_instance* instances, const hs_policy* policy,
              const hs_trace_batch* batch, uint8_t* assign, double* depart,
              hs_inst_metrics* metrics, hs_trace_result* result);

/* Per-trace deployments (BASELINE config 5: each of the top-k deployments
 * replayed on its own trace).  Deployment d owns instances
 * [inst_offsets[d], inst_offsets[d+1]) (types numbered per deployment);
 * trace t runs deployment trace_deployment[t]; policy->n_instances is
 * ignored.  metrics is [n_traces][max instances over deployments]; assign
 * and depart as for hs_replay (a page-locked assign buffer is written in place). */
int hs_replay_deployments(hs_ctx* ctx, const hs_instance* instances, const int32_t* inst_offsets,
                          int32_t n_deployments, const hs_policy* policy, const int32_t* trace_deployment,
                          const hs_trace_batch* batch, uint8_t* assign, double* depart, hs_inst_metrics* metrics,
                          hs_trace_result* result);

/* Device-resident variant for throughput measurement: every pointer in
 * batch / assign / depart / metrics / result is a DEVICE pointer (allocated
 * with hs_device_alloc); instances and policy are host structs. */
int hs_replay_device(hs_ctx* ctx, const hs_instance* instances, const hs_policy* policy,
                     const hs_trace_batch* batch, uint8_t* assign, double* depart,
                     hs_inst_metrics* metrics, hs_trace_result* result);

/* hs_replay with seeded device-side generation: when seeds->arrival_state
 * is set, trace t's arrivals are cumsum(arrival_scale * Exp(1)) drawn from
 * arrival_state[t] on the device (simulator.py:112-124; batch->arrival must
 * be NULL); when seeds->predictor_state is set, its predicted output lengths
 * are drawn on the device (scheduling.py:87-95, one normal per request in
 * trace order; batch->pred_output_len is ignored).  Host buffers as hs_replay. */
int hs_replay_seeded(hs_ctx* ctx, const hs_instance* instances, const hs_policy* policy,
                     const hs_trace_batch* batch, const hs_replay_seeds* seeds, uint8_t* assign,
                     double* depart, hs_inst_metrics* metrics, hs_trace_result* result);

/* ---- seeded streams ---------------------------------------------------- */
/* numpy.random.PCG64(SeedSequence(entropy)) initial state: entropy is the
 * little-endian 32-bit words of a non-negative int seed (numpy
 * bit_generator.pyx SeedSequence.generate_state + pcg64_set_seed). */
int hs_pcg64_seed(const uint32_t* entropy, int32_t n_words, hs_pcg64_state* out);
/* Batch form for integer seeds below 2^64: out[i] = PCG64(seeds[i]) (the
 * entropy words of a seed are its low and, when non-zero, high 32 bits). */
int hs_pcg64_seed_u64(const uint64_t* seeds, int64_t n, hs_pcg64_state* out);

/* Draw stream t's values for each distribution in order: dists[j] fills
 * out[j][offsets[t] .. offsets[t+1]) of its device buffer (int32 for the
 * *_LEN kinds, fp64 for EXP_CUMSUM), continuing the same generator (as
 * cmd_gen_trace draws inputs then outputs from one rng).  states (host, one
 * per stream) are advanced in place.  bad_index (host, optional, one per
 * stream) receives the first index whose length draw was not finite (the
 * reference raises OverflowError on round(inf)) or -1. */
int hs_rng_generate(hs_ctx* ctx, hs_pcg64_state* states, int32_t n_streams, const int64_t* offsets,
                    const hs_dist* dists, int32_t n_dists, void* const* out, int64_t* bad_index);

/* ---- live scheduler (the gateway's per-request path) -------------------
 * Replaces scheduling.py:175-346 Scheduler on the host: evaluate / choose /
 * complete / snapshot with the reference's arithmetic (CPython float //,
 * sum(), glibc exp), checks and state transitions, the in-flight table keyed
 * by the request id, one mutex (the reference's _lock), and an O(N) min-max
 * (scheduling.py:299-312 is O(N^2)).  instances[j]: p, budget, wrr_weight;
 * policy: policy, theta, per_token.  allowed: NULL = all, else n bytes. */
typedef struct hs_scheduler hs_scheduler;

typedef enum {
  HS_SCHED_OK = 0,
  HS_SCHED_NO_INSTANCE = 1,       /* SchedulingError("no instance available for scheduling")       */
  HS_SCHED_ALREADY_IN_FLIGHT = 2, /* SchedulingError("request ... is already in flight")           */
  HS_SCHED_NOT_IN_FLIGHT = 3,     /* SchedulingError("request ... is not in flight (double ...)")  */
  HS_SCHED_NONPOSITIVE_COST = 4,  /* SpecError("non-positive batch time ...")  (value = the total) */
  HS_SCHED_EXP_OVERFLOW = 5,      /* OverflowError("math range error")                              */
  HS_SCHED_NEGATIVE_RUNNING = 6,  /* SpecError("running token sums went negative; ...")            */
  HS_SCHED_ZERO_DIVISION = 7      /* ZeroDivisionError("float floor division by zero")             */
} hs_sched_error;

typedef struct {
  int32_t error;    /* hs_sched_error */
  int32_t instance; /* instance the error arose on, or -1 */
  double value;
} hs_sched_status;

int hs_sched_create(const hs_instance* instances, int32_t n, const hs_policy* policy, hs_scheduler** out);
int hs_sched_destroy(hs_scheduler* s);
/* Scheduler.evaluate: weights[n] (+inf where not allowed); no state change. */
int hs_sched_evaluate(hs_scheduler* s, int64_t input_len, int64_t predicted_output_len, const uint8_t* allowed,
                      double* weights, hs_sched_status* status);
/* Scheduler.choose: *chosen = instance index, dispatch bookkeeping committed. */
int hs_sched_choose(hs_scheduler* s, const char* request_id, int32_t id_len, int64_t input_len,
                    int64_t predicted_output_len, const uint8_t* allowed, int32_t* chosen, hs_sched_status* status);
/* Scheduler.complete: subtracts exactly what choose recorded. */
int hs_sched_complete(hs_scheduler* s, const char* request_id, int32_t id_len, hs_sched_status* status);
/* Scheduler.snapshot / loads / running_totals (any pointer may be NULL). */
int hs_sched_snapshot(hs_scheduler* s, double* loads, int64_t* running_totals, double* kv_usage, int64_t* oversized,
                      int64_t* in_flight);
/* Scheduler._states[j] (scheduling.py:157-164 InstanceState): read or
 * overwrite one instance's load, running token sums (RunningTokens
 * input_sum / predicted_output_sum) and oversized count, or replace its
 * handle (params, budget, wrr_weight) -- what the reference's tests and a
 * gateway reach into directly (tests/test_scheduling.py:142-143, 275;
 * tests/test_gateway.py:140-149).  Any out pointer may be NULL. */
int hs_sched_get_state(hs_scheduler* s, int32_t j, double* load, int64_t* input_sum, int64_t* pred_sum,
                       int64_t* oversized);
int hs_sched_set_state(hs_scheduler* s, int32_t j, double load, int64_t input_sum, int64_t pred_sum,
                       int64_t oversized);
int hs_sched_set_instance(hs_scheduler* s, int32_t j, const hs_instance* instance);

/* Device buffers for hs_replay_device. */
int hs_device_alloc(hs_ctx* ctx, int64_t bytes, void** out);
int hs_device_free(hs_ctx* ctx, void* ptr);
int hs_memcpy_h2d(hs_ctx* ctx, void* dst, const void* src, int64_t bytes);
int hs_memcpy_d2h(hs_ctx* ctx, void* dst, const void* src, int64_t bytes);
int hs_device_synchronize(hs_ctx* ctx);
/* Page-locked host buffers (for end-to-end transfers at full PCIe rate). */
int hs_host_alloc(hs_ctx* ctx, int64_t bytes, void** out);
int hs_host_free(hs_ctx* ctx, void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* HETSERVE_B200_H */
