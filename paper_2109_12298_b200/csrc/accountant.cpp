// accountant.cpp — host-side privacy bookkeeping around the device step:
//   * NoiseSchedule / schedule_noise (reference optimizer.hpp:280-358): sigma per epoch, applied to
//     an optimizer through dpg_set_noise_multiplier;
//   * the RDP accountant of the subsampled Gaussian mechanism (reference SPEC.md:331-389, a spec-only
//     module of the reference): integer-order RDP in log space, additive composition, the
//     (epsilon, delta) conversion, and noise calibration by bisection;
// (The record export to the host, dpg_grad_sample_export, lives with the optimizer in model.cpp.)
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "dpg_internal.h"

using dpg::guard;
using dpg::raise;

namespace {

// the reference's ParameterError texts (optimizer.hpp:281-358)
void check_sigma(double sigma) {
  if (!(sigma >= 0.0)) raise(DPG_ERR_PARAMETER, "schedule sigma must be >= 0");
}

double log_add(double a, double b) {  // log(e^a + e^b)
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double m = std::max(a, b);
  return m + std::log1p(std::exp(-std::fabs(a - b)));
}

// (1/(alpha-1)) ln sum_k C(alpha,k) (1-q)^(alpha-k) q^k exp((k^2 - k) / (2 sigma^2)), log-sum-exp
double rdp_sg(double q, double sigma, int alpha) {
  if (!(q >= 0.0 && q <= 1.0)) raise(DPG_ERR_PARAMETER, "sampling rate q must be in [0, 1]");
  if (alpha < 2) raise(DPG_ERR_PARAMETER, "RDP order must be an integer >= 2");
  if (q == 0.0) return 0.0;
  if (!(sigma > 0.0)) raise(DPG_ERR_PARAMETER, "noise multiplier must be > 0 when q > 0");
  const double inv2s2 = 1.0 / (2.0 * sigma * sigma);
  if (q == 1.0) return alpha * inv2s2;  // only k = alpha survives
  const double lq = std::log(q), l1q = std::log1p(-q);
  const double lga = std::lgamma(alpha + 1.0);
  double acc = -INFINITY;
  for (int k = 0; k <= alpha; ++k) {
    const double lc = lga - std::lgamma(k + 1.0) - std::lgamma(alpha - k + 1.0);
    acc = log_add(acc, lc + (alpha - k) * l1q + k * lq + ((double)k * k - k) * inv2s2);
  }
  return std::max(0.0, acc / (alpha - 1));
}

struct Record {
  double sigma, q;
  int64_t steps;
};

}  // namespace

struct dpg_accountant {
  std::vector<int> orders;
  std::vector<Record> history;
};

namespace {

void curve_of(const std::vector<int>& orders, const std::vector<Record>& hist, std::vector<double>& out) {
  out.assign(orders.size(), 0.0);
  for (const Record& r : hist)
    for (size_t i = 0; i < orders.size(); ++i) out[i] += (double)r.steps * rdp_sg(r.q, r.sigma, orders[i]);
}

void to_eps(const std::vector<int>& orders, const std::vector<double>& curve, double delta, double* eps, int* best) {
  if (!(delta > 0.0 && delta < 1.0)) raise(DPG_ERR_PARAMETER, "delta must be in (0, 1)");
  double e = INFINITY;
  int b = orders.empty() ? 0 : orders.back();
  for (size_t i = 0; i < orders.size(); ++i) {
    const double v = curve[i] + std::log(1.0 / delta) / (orders[i] - 1);
    if (v < e) {  // ties keep the smaller order
      e = v;
      b = orders[i];
    }
  }
  if (eps) *eps = e;
  if (best) *best = b;
}

std::vector<int> default_orders() {
  std::vector<int> o;
  for (int a = 2; a <= 64; ++a) o.push_back(a);
  o.push_back(128);
  o.push_back(256);
  return o;
}

}  // namespace


// ---- NoiseSchedule (optimizer.hpp:280-351) ----
dpg_status dpg_noise_schedule_init(dpg_noise_schedule* s, int kind, double sigma0, double gamma, double factor,
                                   uint64_t period, const double* table, int64_t table_len) {
  return guard(nullptr, [&] {
    if (!s) raise(DPG_ERR_PARAMETER, "null schedule");
    dpg_noise_schedule r{};
    r.kind = kind;
    r.gamma = 1.0;
    r.factor = 1.0;
    r.period = 1;
    switch (kind) {
      case DPG_SCHEDULE_CONSTANT:
        check_sigma(sigma0);
        r.initial_sigma = r.current = sigma0;
        break;
      case DPG_SCHEDULE_EXPONENTIAL:
        check_sigma(sigma0);
        if (gamma < 0.0) raise(DPG_ERR_PARAMETER, "exponential schedule needs gamma >= 0");
        r.initial_sigma = r.current = sigma0;
        r.gamma = gamma;
        break;
      case DPG_SCHEDULE_STEP:
        check_sigma(sigma0);
        if (factor < 0.0) raise(DPG_ERR_PARAMETER, "step schedule needs factor >= 0");
        if (period == 0) raise(DPG_ERR_PARAMETER, "step schedule needs period >= 1");
        r.initial_sigma = r.current = sigma0;
        r.factor = factor;
        r.period = period;
        break;
      case DPG_SCHEDULE_CUSTOM:
        if (!table || table_len <= 0) raise(DPG_ERR_PARAMETER, "custom schedule needs at least one sigma");
        for (int64_t i = 0; i < table_len; ++i) check_sigma(table[i]);
        r.initial_sigma = r.current = table[0];
        r.table = table;
        r.table_len = table_len;
        break;
      default:
        raise(DPG_ERR_PARAMETER, "unknown schedule kind");
    }
    *s = r;
  });
}

double dpg_noise_schedule_sigma_at(const dpg_noise_schedule* s, uint64_t epoch) {
  if (!s) return NAN;
  switch (s->kind) {
    case DPG_SCHEDULE_CONSTANT: return s->initial_sigma;
    case DPG_SCHEDULE_EXPONENTIAL: return s->initial_sigma * std::pow(s->gamma, (double)epoch);
    case DPG_SCHEDULE_STEP: return s->initial_sigma * std::pow(s->factor, (double)(epoch / s->period));
    case DPG_SCHEDULE_CUSTOM:
      return s->table[std::min<uint64_t>(epoch, (uint64_t)(s->table_len - 1))];
  }
  return s->initial_sigma;
}

// schedule_noise (optimizer.hpp:354-358), applied to the optimizer when one is given
dpg_status dpg_schedule_noise(dpg_noise_schedule* s, uint64_t epoch, dpg_optimizer* opt, double* sigma) {
  if (!s) return DPG_ERR_PARAMETER;
  s->current = dpg_noise_schedule_sigma_at(s, epoch);
  if (sigma) *sigma = s->current;
  return opt ? dpg_set_noise_multiplier(opt, s->current) : DPG_OK;
}

// ---- RDP accountant ----
dpg_status dpg_rdp_subsampled_gaussian(double q, double sigma, int alpha, double* out) {
  return guard(nullptr, [&] {
    const double v = rdp_sg(q, sigma, alpha);
    if (out) *out = v;
  });
}

dpg_status dpg_accountant_create(const int* orders, int n, dpg_accountant** out) {
  if (!out) return DPG_ERR_PARAMETER;
  *out = nullptr;
  dpg_accountant* a = new dpg_accountant();
  const dpg_status st = guard(nullptr, [&] {
    if (orders && n > 0) {
      a->orders.assign(orders, orders + n);
      for (int o : a->orders)
        if (o < 2) raise(DPG_ERR_PARAMETER, "RDP orders must be integers >= 2");
      std::sort(a->orders.begin(), a->orders.end());
      a->orders.erase(std::unique(a->orders.begin(), a->orders.end()), a->orders.end());
    } else {
      a->orders = default_orders();
    }
  });
  if (st != DPG_OK) {
    delete a;
    return st;
  }
  *out = a;
  return DPG_OK;
}

void dpg_accountant_destroy(dpg_accountant* a) { delete a; }

int dpg_accountant_num_orders(const dpg_accountant* a) { return a ? (int)a->orders.size() : 0; }

// one record per logical step batch (virtual steps do not multiply invocations)
dpg_status dpg_accountant_step(dpg_accountant* a, double sigma, double q, int64_t steps) {
  return guard(nullptr, [&] {
    if (!a) raise(DPG_ERR_PARAMETER, "null accountant");
    if (steps < 0) raise(DPG_ERR_PARAMETER, "step count must be >= 0");
    rdp_sg(q, sigma, 2);  // validates (q, sigma)
    a->history.push_back({sigma, q, steps});
  });
}

dpg_status dpg_accountant_rdp(const dpg_accountant* a, int* orders, double* curve) {
  return guard(nullptr, [&] {
    if (!a) raise(DPG_ERR_PARAMETER, "null accountant");
    std::vector<double> c;
    curve_of(a->orders, a->history, c);
    for (size_t i = 0; i < c.size(); ++i) {
      if (orders) orders[i] = a->orders[i];
      if (curve) curve[i] = c[i];
    }
  });
}

dpg_status dpg_accountant_epsilon(const dpg_accountant* a, double delta, double* eps, int* best_order) {
  return guard(nullptr, [&] {
    if (!a) raise(DPG_ERR_PARAMETER, "null accountant");
    std::vector<double> c;
    curve_of(a->orders, a->history, c);
    to_eps(a->orders, c, delta, eps, best_order);
  });
}

// smallest sigma on the bisection grid (absolute tolerance 1e-3) with epsilon(sigma) <= target
dpg_status dpg_get_noise_multiplier(double target_eps, double delta, double q, int64_t steps, double sigma_min,
                                    double sigma_max, double* sigma) {
  return guard(nullptr, [&] {
    if (!(target_eps > 0.0)) raise(DPG_ERR_PARAMETER, "target epsilon must be > 0");
    if (steps < 0) raise(DPG_ERR_PARAMETER, "step count must be >= 0");
    if (!(sigma_min > 0.0 && sigma_max > sigma_min)) raise(DPG_ERR_PARAMETER, "need 0 < sigma_min < sigma_max");
    const std::vector<int> orders = default_orders();
    auto eps_at = [&](double s) {
      std::vector<double> c;
      curve_of(orders, {{s, q, steps}}, c);
      double e;
      to_eps(orders, c, delta, &e, nullptr);
      return e;
    };
    const double e_max = eps_at(sigma_max);
    if (e_max > target_eps)
      raise(DPG_ERR_PARAMETER, "noise calibration infeasible: epsilon at sigma_max " + std::to_string(sigma_max) +
                                   " is " + std::to_string(e_max) + " > target " + std::to_string(target_eps));
    if (eps_at(sigma_min) <= target_eps) {
      *sigma = sigma_min;
      return;
    }
    double lo = sigma_min, hi = sigma_max;  // eps(lo) > target >= eps(hi)
    while (hi - lo > 1e-3) {
      const double mid = 0.5 * (lo + hi);
      if (eps_at(mid) <= target_eps) hi = mid;
      else lo = mid;
    }
    *sigma = hi;
  });
}

