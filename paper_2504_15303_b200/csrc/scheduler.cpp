// scheduler.cpp -- the live capacity-aware scheduler on the host (C++): the
// per-request path the reference's gateway takes (scheduling.py:175-346
// Scheduler; gateway.py:201-306 calls choose() / complete()).
//
// Same decisions, bit for bit, as the reference: the arithmetic follows the
// reference's operation order (CPython float floor division, builtin sum(),
// glibc exp -- the very libm function CPython's math.exp calls), checks run in
// the reference's order and raise the same conditions (as hs_sched_status
// codes the Python shim turns into the reference's exceptions), and the
// round-robin / weighted state advances before the chosen instance is
// evaluated, as in Scheduler.choose.  _min_max_choice is O(N): with the
// top-2 of the loads, max_{j != s} L_j is the top unless s holds it alone.
// Host code only (no CUDA); compiled without contraction (-ffp-contract=off).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hetserve_b200.h"

namespace hs {
int set_error(int code, const char* msg);
}

namespace {

struct InFlight {
  int32_t inst;
  double load_delta;
  int64_t input_len, pred_len;
};

struct Inst {
  double p[8];
  double budget;
  double wrr_weight;
  double load = 0.0;
  int64_t input_sum = 0, pred_sum = 0;
  int64_t oversized = 0;
};

// CPython Objects/floatobject.c float_floor_div (_float_div_mod), wx != 0
double py_floordiv(double vx, double wx) {
  double mod = std::fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) {
      mod += wx;
      div -= 1.0;
    }
  }
  double fl;
  if (div != 0.0) {
    fl = std::floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = std::copysign(0.0, vx / wx);
  }
  return fl;
}

// CPython 3.12 builtin sum() over floats with int start 0 (Neumaier)
double py_sum(const std::vector<double>& xs) {
  double f = 0.0, c = 0.0;
  bool first = true;
  for (double x : xs) {
    if (first) {
      f = 0.0 + x;
      first = false;
      continue;
    }
    const double t = f + x;
    if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  if (c != 0.0 && std::isfinite(c)) f += c;
  return f;
}

// latency.py:90-92 / 100-109 (same operation order as csrc/hs_device.cuh).
// The batch size only ever enters as float(b); b = int(x) of an integral
// float x converts back to x exactly, so it is carried as that double.
double prefill_time(const double* p, double db, int64_t I) {
  const double dI = (double)I;
  return ((p[0] * db * dI + p[1] * db) + p[2] * dI) + p[3];
}
double decode_time(const double* p, double db, int64_t I, int64_t O) {
  const double S = (double)(O * I) + (double)(O * (O + 1)) / 2.0;
  return (p[4] * db + p[6]) * S + (p[5] * db + p[7]) * (double)O;
}

}  // namespace

struct hs_scheduler {
  std::mutex mu;
  std::vector<Inst> inst;
  int32_t policy;
  double theta;
  int64_t per_token;
  int64_t rr_next = 0;
  std::vector<double> wrr_current;
  std::unordered_map<std::string, InFlight> in_flight;

  // Scheduler.evaluate for instance j (ideal_batch_size, per_request_cost,
  // kv_usage, workload: scheduling.py:119-154, capacity.py:98-106)
  int weight(int32_t j, int64_t I, int64_t P, double* w, hs_sched_status* st) const {
    const Inst& s = inst[j];
    double cost = 1.0;
    if (policy != HS_POLICY_MB) {
      const int64_t per_request = per_token * (I + P);
      if (per_request == 0) {
        *st = hs_sched_status{HS_SCHED_ZERO_DIVISION, j, 0.0};
        return 1;
      }
      // ideal_batch_size: max(1, int(budget // per_request))
      double db = py_floordiv(s.budget, (double)per_request);
      if (!(db >= 1.0)) db = 1.0;
      const double total = prefill_time(s.p, db, I) + decode_time(s.p, db, I, P);
      if (total <= 0.0) {
        *st = hs_sched_status{HS_SCHED_NONPOSITIVE_COST, j, total};
        return 1;
      }
      cost = total / db;
    }
    const double usage = (double)(per_token * (s.input_sum + s.pred_sum)) / s.budget;
    const double x = theta * usage;
    const double e = std::exp(x);
    if (std::isinf(e) && !std::isinf(x)) {  // CPython math.exp: OverflowError
      *st = hs_sched_status{HS_SCHED_EXP_OVERFLOW, j, x};
      return 1;
    }
    *w = cost * e;
    return 0;
  }

  int evaluate(int64_t I, int64_t P, const uint8_t* allowed, double* w, hs_sched_status* st) const {
    const int32_t n = (int32_t)inst.size();
    for (int32_t j = 0; j < n; ++j) {
      if (allowed && !allowed[j]) {
        w[j] = INFINITY;
        continue;
      }
      if (weight(j, I, P, &w[j], st)) return 1;
    }
    return 0;
  }

  // scheduling.py:299-312: argmin over s of max(L_s + w_s, max_{j != s} (L_j + 0.0)),
  // first strict improvement wins (lowest index among equal peaks)
  int32_t min_max(const double* w) const {
    const int32_t n = (int32_t)inst.size();
    int32_t a1 = -1;
    int cnt1 = 0;
    double m1 = -INFINITY, m2 = -INFINITY;
    for (int32_t j = 0; j < n; ++j) {
      const double l = inst[j].load;
      if (a1 < 0 || l > m1) {
        m2 = m1;
        m1 = l;
        a1 = j;
        cnt1 = 1;
      } else if (l == m1) {
        ++cnt1;
      } else if (l > m2) {
        m2 = l;
      }
    }
    if (cnt1 >= 2) m2 = m1;
    int32_t best = -1;
    double best_peak = INFINITY;
    for (int32_t s = 0; s < n; ++s) {
      if (std::isinf(w[s])) continue;
      const double others = (n == 1) ? -INFINITY : ((s == a1 || inst[s].load == m1) && cnt1 == 1 ? m2 : m1);
      const double own = inst[s].load + w[s];
      const double peak = own > others ? own : others;
      if (peak < best_peak) {
        best_peak = peak;
        best = s;
      }
    }
    return best;
  }
};

namespace {
int sched_fail(hs_sched_status* st, int32_t code) {
  *st = hs_sched_status{code, -1, 0.0};
  return HS_OK;
}
}  // namespace

extern "C" {

int hs_sched_create(const hs_instance* instances, int32_t n, const hs_policy* policy, hs_scheduler** out) {
  if (!instances || !policy || !out) return hs::set_error(HS_ERR_ARG, "null argument");
  if (n < 1) return hs::set_error(HS_ERR_ARG, "scheduler needs at least one instance");
  if (policy->policy < HS_POLICY_OS || policy->policy > HS_POLICY_MB) return hs::set_error(HS_ERR_ARG, "unknown policy");
  if (!(policy->theta > 0)) return hs::set_error(HS_ERR_ARG, "theta must be > 0");
  if (policy->per_token <= 0) return hs::set_error(HS_ERR_ARG, "per_token must be positive");
  hs_scheduler* s = new hs_scheduler();
  s->policy = policy->policy;
  s->theta = policy->theta;
  s->per_token = policy->per_token;
  s->inst.resize((size_t)n);
  for (int32_t j = 0; j < n; ++j) {
    if (!(instances[j].budget > 0)) {
      delete s;
      return hs::set_error(HS_ERR_ARG, "instance budget must be positive");
    }
    std::memcpy(s->inst[j].p, instances[j].p, sizeof(double) * 8);
    s->inst[j].budget = instances[j].budget;
    s->inst[j].wrr_weight = instances[j].wrr_weight;
  }
  s->wrr_current.assign((size_t)n, 0.0);
  *out = s;
  return HS_OK;
}

int hs_sched_destroy(hs_scheduler* s) {
  delete s;
  return HS_OK;
}

int hs_sched_evaluate(hs_scheduler* s, int64_t I, int64_t P, const uint8_t* allowed, double* w, hs_sched_status* st) {
  if (!s || !w || !st) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  *st = hs_sched_status{HS_SCHED_OK, -1, 0.0};
  s->evaluate(I, P, allowed, w, st);
  return HS_OK;
}

int hs_sched_choose(hs_scheduler* s, const char* id, int32_t id_len, int64_t I, int64_t P, const uint8_t* allowed,
                    int32_t* chosen, hs_sched_status* st) {
  if (!s || !id || id_len < 0 || !chosen || !st) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  *st = hs_sched_status{HS_SCHED_OK, -1, 0.0};
  *chosen = -1;
  const int32_t n = (int32_t)s->inst.size();
  std::vector<int32_t> cand;  // _candidates
  for (int32_t j = 0; j < n; ++j)
    if (!allowed || allowed[j]) cand.push_back(j);
  if (cand.empty()) return sched_fail(st, HS_SCHED_NO_INSTANCE);
  std::string key(id, (size_t)id_len);
  if (s->in_flight.count(key)) return sched_fail(st, HS_SCHED_ALREADY_IN_FLIGHT);
  std::vector<double> w((size_t)n, INFINITY);
  int32_t c;
  if (s->policy == HS_POLICY_OS || s->policy == HS_POLICY_MB) {
    if (s->evaluate(I, P, allowed, w.data(), st)) return HS_OK;
    c = s->min_max(w.data());
    if (c < 0) return sched_fail(st, HS_SCHED_NO_INSTANCE);
  } else {
    if (s->policy == HS_POLICY_SI) {
      c = (!allowed || allowed[0]) ? 0 : cand[0];
    } else if (s->policy == HS_POLICY_RR) {  // _next_round_robin
      c = cand[0];
      for (int32_t k = 0; k < n; ++k) {
        const int32_t idx = (int32_t)(s->rr_next % n);
        s->rr_next += 1;
        if (!allowed || allowed[idx]) {
          c = idx;
          break;
        }
      }
    } else {  // _next_weighted: smooth WRR over the candidates
      std::vector<double> ws;
      for (int32_t i : cand) ws.push_back(s->inst[i].wrr_weight);
      const double total = py_sum(ws);
      c = cand[0];
      for (int32_t i : cand) {
        s->wrr_current[i] += s->inst[i].wrr_weight;
        if (s->wrr_current[i] > s->wrr_current[c]) c = i;
      }
      s->wrr_current[c] -= total;
    }
    if (s->weight(c, I, P, &w[c], st)) return HS_OK;  // evaluate(request, allowed={chosen})
  }
  // _commit (scheduling.py:335-346)
  Inst& t = s->inst[c];
  const int64_t per_request = s->per_token * (I + P);
  // request_oversized: the exact int > float comparison (per_request > floor(budget))
  if (t.budget < 9.2e18 && per_request > (int64_t)std::floor(t.budget)) t.oversized += 1;
  t.load += w[c];
  t.input_sum += I;
  t.pred_sum += P;
  s->in_flight.emplace(std::move(key), InFlight{c, w[c], I, P});
  *chosen = c;
  return HS_OK;
}

int hs_sched_complete(hs_scheduler* s, const char* id, int32_t id_len, hs_sched_status* st) {
  if (!s || !id || id_len < 0 || !st) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  *st = hs_sched_status{HS_SCHED_OK, -1, 0.0};
  auto it = s->in_flight.find(std::string(id, (size_t)id_len));
  if (it == s->in_flight.end()) return sched_fail(st, HS_SCHED_NOT_IN_FLIGHT);
  const InFlight e = it->second;
  s->in_flight.erase(it);
  Inst& t = s->inst[e.inst];
  t.load -= e.load_delta;
  t.input_sum -= e.input_len;
  t.pred_sum -= e.pred_len;
  if (t.input_sum < 0 || t.pred_sum < 0) {
    *st = hs_sched_status{HS_SCHED_NEGATIVE_RUNNING, e.inst, 0.0};
  }
  return HS_OK;
}

int hs_sched_snapshot(hs_scheduler* s, double* loads, int64_t* running, double* usage, int64_t* oversized,
                      int64_t* in_flight) {
  if (!s) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  for (size_t j = 0; j < s->inst.size(); ++j) {
    const Inst& t = s->inst[j];
    if (loads) loads[j] = t.load;
    if (running) running[j] = t.input_sum + t.pred_sum;
    if (usage) usage[j] = (double)(s->per_token * (t.input_sum + t.pred_sum)) / t.budget;
    if (oversized) oversized[j] = t.oversized;
  }
  if (in_flight) *in_flight = (int64_t)s->in_flight.size();
  return HS_OK;
}

}  // extern "C"

// Scheduler._states view (scheduling.py:157-164 InstanceState): tests and
// gateways that read or poke one instance's bookkeeping directly
// (load, running tokens, oversized count, handle).
extern "C" {

int hs_sched_get_state(hs_scheduler* s, int32_t j, double* load, int64_t* input_sum, int64_t* pred_sum,
                       int64_t* oversized) {
  if (!s) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  if (j < 0 || (size_t)j >= s->inst.size()) return hs::set_error(HS_ERR_ARG, "instance index out of range");
  const Inst& t = s->inst[j];
  if (load) *load = t.load;
  if (input_sum) *input_sum = t.input_sum;
  if (pred_sum) *pred_sum = t.pred_sum;
  if (oversized) *oversized = t.oversized;
  return HS_OK;
}

int hs_sched_set_state(hs_scheduler* s, int32_t j, double load, int64_t input_sum, int64_t pred_sum,
                       int64_t oversized) {
  if (!s) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  if (j < 0 || (size_t)j >= s->inst.size()) return hs::set_error(HS_ERR_ARG, "instance index out of range");
  Inst& t = s->inst[j];
  t.load = load;
  t.input_sum = input_sum;
  t.pred_sum = pred_sum;
  t.oversized = oversized;
  return HS_OK;
}

int hs_sched_set_instance(hs_scheduler* s, int32_t j, const hs_instance* instance) {
  if (!s || !instance) return hs::set_error(HS_ERR_ARG, "null argument");
  std::lock_guard<std::mutex> g(s->mu);
  if (j < 0 || (size_t)j >= s->inst.size()) return hs::set_error(HS_ERR_ARG, "instance index out of range");
  if (!(instance->budget > 0)) return hs::set_error(HS_ERR_ARG, "instance budget must be positive");
  Inst& t = s->inst[j];
  std::memcpy(t.p, instance->p, sizeof(double) * 8);
  t.budget = instance->budget;
  t.wrr_weight = instance->wrr_weight;
  return HS_OK;
}

}  // extern "C"
