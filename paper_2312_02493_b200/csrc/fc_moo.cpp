// fc_moo.cpp — the adaptive-CR controller's decision functions
// (inc/moo.hpp:27-146, inc/netsched.hpp:50-58, inc/compress.hpp:145-165)
// behind the C-ABI, shared by the C++ façade (include/flexcomm_b200/moo.hpp)
// and the Python mirror (paper_2312_02493_b200/moo.py).
//
// The controller's choice must be the reference's choice on the same
// candidate statistics, so every expression keeps the reference's operation
// order in double precision (compiled with -ffp-contract=off), and
// tests/test_moo.py checks the results bit for bit against the unmodified
// reference headers (oracle/_ref).  The state machine (explore / refresh /
// apply) lives in the façades because it drives the trainer.
#include <cmath>
#include <cstdint>

#include "flexcomm_b200.h"

namespace {

inline bool valid_config(const fc_controller_config* c) {
  // ControllerConfig::validate, inc/moo.hpp:34-41
  if (!(c->c_low > 0.0 && c->c_low <= c->c_high && c->c_high <= 1.0)) return false;
  if (c->factor <= 1.0) return false;
  if (c->probe_iters < 1) return false;
  if (c->gain_threshold < 0.0) return false;
  return true;
}

inline double r3(double v) {
  // round_3sig, inc/moo.hpp:44-48: scale to three significant digits and
  // round half away from zero (std::round)
  if (v == 0.0) return 0.0;
  const double unit = std::pow(10.0, std::floor(std::log10(std::fabs(v))) - 2.0);
  return std::round(v / unit) * unit;
}

// objectives minimised by the controller: compression time, modelled sync
// time, inverse gain (inc/moo.hpp:76-77, 115-117)
inline void objectives(const fc_candidate& c, double o[3]) {
  o[0] = c.t_comp_avg;
  o[1] = c.t_sync_modeled;
  o[2] = 1.0 / c.gain_avg;
}

// a dominates b: no objective worse, at least one strictly better (:75-84)
inline bool dominates(const fc_candidate& a, const fc_candidate& b) {
  double x[3], y[3];
  objectives(a, x);
  objectives(b, y);
  bool none_worse = true, one_better = false;
  for (int i = 0; i < 3; ++i) {
    none_worse = none_worse && !(x[i] > y[i]);
    one_better = one_better || x[i] < y[i];
  }
  return none_worse && one_better;
}

}  // namespace

extern "C" {

int fc_controller_config_validate(const fc_controller_config* cfg) {
  if (!cfg) return FC_ERR_INVALID_ARGUMENT;
  return valid_config(cfg) ? FC_OK : FC_ERR_INVALID_ARGUMENT;
}

int fc_round_3sig(double v, double* out) {
  if (!out) return FC_ERR_INVALID_ARGUMENT;
  *out = r3(v);
  return FC_OK;
}

// candidate_ladder, inc/moo.hpp:52-65: geometric rungs from c_high down by
// `factor`; the first value below c_low·sqrt(factor) is replaced by c_low
// and ends the ladder.  *count is the full rung count even when cap is short.
int fc_candidate_ladder(const fc_controller_config* cfg, double* out, int cap, int* count) {
  if (!cfg || !count || (cap > 0 && !out)) return FC_ERR_INVALID_ARGUMENT;
  if (!valid_config(cfg)) return FC_ERR_INVALID_ARGUMENT;
  const double stop = cfg->c_low * std::sqrt(cfg->factor);
  int m = 0;
  for (double v = cfg->c_high;; v /= cfg->factor) {
    const bool last = v < stop;
    const double rung = last ? cfg->c_low : r3(v);
    if (m < cap) out[m] = rung;
    ++m;
    if (last) break;
  }
  *count = m;
  return FC_OK;
}

// trigger_gain, inc/moo.hpp:67-71, over the GainTracker window
// (inc/compress.hpp:145-165: the samples in push order, mean = sequential sum / n).
int fc_trigger_gain(double gain_ref, const double* samples, uint64_t count, double threshold,
                    int* fire) {
  if (!fire || (count && !samples)) return FC_ERR_INVALID_ARGUMENT;
  *fire = 0;
  if (count < 2) return FC_OK;
  if (!(gain_ref > 0.0)) return FC_OK;
  double sum = 0.0;
  for (uint64_t i = 0; i < count; ++i) sum += samples[i];
  const double mean = sum / static_cast<double>(count);
  *fire = std::fabs(mean - gain_ref) / gain_ref >= threshold ? 1 : 0;
  return FC_OK;
}

// pareto_front, inc/moo.hpp:88-102: mask[i] = 1 iff no candidate dominates i
// (the front keeps input order).
int fc_pareto_front(const fc_candidate* cands, int m, int* mask) {
  if (!cands || !mask || m < 1) return FC_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < m; ++i) {
    int keep = 1;
    for (int j = 0; j < m && keep; ++j)
      if (dominates(cands[j], cands[i])) keep = 0;
    mask[i] = keep;
  }
  return FC_OK;
}

// choose_cr, inc/moo.hpp:111-146: min-max normalise the objectives over the
// front, take the candidate nearest the ideal point (ties within 1e-12 go to
// the larger c, else the earlier one), then select_collective at its c.
int fc_choose_cr(const fc_candidate* front, int m, double alpha, double bandwidth, double m_bytes,
                 int n, int* chosen, int* collective) {
  if (!front || m < 1 || !chosen) return FC_ERR_INVALID_ARGUMENT;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int i = 0; i < m; ++i) {
    double o[3];
    objectives(front[i], o);
    for (int d = 0; d < 3; ++d) {
      lo[d] = o[d] < lo[d] ? o[d] : lo[d];
      hi[d] = hi[d] < o[d] ? o[d] : hi[d];
    }
  }
  int best = -1;
  double best_d = 0.0;
  for (int i = 0; i < m; ++i) {
    double o[3], ss = 0.0;
    objectives(front[i], o);
    for (int d = 0; d < 3; ++d) {
      const double span = hi[d] - lo[d];
      const double x = span > 0.0 ? (o[d] - lo[d]) / span : 0.0;
      ss += x * x;
    }
    const double dist = std::sqrt(ss);
    const bool closer = dist < best_d - 1e-12;
    const bool tie_larger = std::fabs(dist - best_d) <= 1e-12 && front[i].c > front[best < 0 ? 0 : best].c;
    if (best < 0 || closer || tie_larger) {
      best = i;
      best_d = dist;
    }
  }
  *chosen = best;
  if (collective) {
    const int s = fc_select_collective(alpha, bandwidth, m_bytes, front[best].c, n, collective, nullptr);
    if (s != FC_OK) return s;
  }
  return FC_OK;
}

// network_changed, inc/netsched.hpp:50-58: relative change of alpha or
// bandwidth above rel_threshold (scale = the larger magnitude; 0 when both 0).
int fc_network_changed(double alpha0, double bandwidth0, double alpha1, double bandwidth1,
                       double rel_threshold, int* changed) {
  if (!changed) return FC_ERR_INVALID_ARGUMENT;
  auto rel = [](double a, double b) {
    const double s = std::fmax(std::fabs(a), std::fabs(b));
    return s == 0.0 ? 0.0 : std::fabs(a - b) / s;
  };
  *changed = (rel(alpha0, alpha1) > rel_threshold || rel(bandwidth0, bandwidth1) > rel_threshold) ? 1 : 0;
  return FC_OK;
}

}  // extern "C"
