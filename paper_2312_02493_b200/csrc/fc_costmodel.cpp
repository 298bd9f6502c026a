// fc_costmodel.cpp — the reference's alpha-beta collective cost model and its
// closed-form selection (inc/costmodel.hpp:12-203; paper Eqs. 4a/4b/5a-c,
// PAPER.md:701-856), exposed through the C-ABI so the C++ facade, the
// Python host mirror and the MOO controller share one implementation.
//
// The north star keeps this model UNCHANGED and only recalibrates its
// NetParams to NVLink (see calibrate.py).  Selection parity is bit-exact, so
// every expression below is evaluated in the same operation order as the
// reference (left-to-right products, log2 of double(N)), and the file is
// compiled with -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <string>

#include "flexcomm_b200.h"

namespace {

thread_local std::string g_cm_err;

struct Net {
  double alpha, bw;
  double beta() const { return 8.0 / bw; }  // seconds per byte (NetParams::beta)
};

struct Msg {
  double m, c;
  int n;
};

int validate(double alpha, double bw, double m, double c, int n) {
  if (alpha < 0.0) return 1;
  if (!(bw > 0.0)) return 2;
  if (m < 4.0) return 3;
  if (!(c > 0.0 && c <= 1.0)) return 4;
  if (n < 1) return 5;
  return 0;
}

// Eight costs in CostBreakdown order: ps, ring_ar, tree_ar, broadcast,
// allgather_dense, ag_compressed, art_ring, art_tree.
void costs(const Net& net, const Msg& s, double out[8]) {
  const double lg = std::log2(static_cast<double>(s.n));
  const double nm1 = s.n - 1;
  const double beta = net.beta();
  // inc/costmodel.hpp:54-56
  out[0] = 2.0 * net.alpha + 2.0 * (s.n - 1) * s.m * beta;
  // :58-61
  out[1] = 2.0 * nm1 * net.alpha + 2.0 * (nm1 / s.n) * s.m * beta;
  // :63-66
  out[2] = 2.0 * net.alpha * lg + 2.0 * lg * s.m * beta;
  // :68-71
  out[3] = net.alpha * lg + lg * s.m * beta;
  // :73-76
  out[4] = net.alpha * lg + (s.n - 1) * s.m * beta;
  // :79-82  (2Mc bytes: values plus indices)
  out[5] = net.alpha * lg + 2.0 * s.m * s.c * beta * (s.n - 1);
  const double mc = s.m * s.c;
  // :85-90  Eq. (4a)
  out[6] = net.alpha * (2.0 * nm1 + lg) + mc * beta * (2.0 * nm1 / s.n + lg);
  // :92-96  Eq. (4b)
  out[7] = 3.0 * net.alpha * lg + 3.0 * mc * beta * lg;
}

}  // namespace

extern "C" {

int fc_cost_primitives(double alpha, double bandwidth, double m_bytes, double c, int n,
                       double* out8) {
  if (int v = validate(alpha, bandwidth, m_bytes, c, n)) {
    (void)v;
    return FC_ERR_INVALID_ARGUMENT;
  }
  costs(Net{alpha, bandwidth}, Msg{m_bytes, c, n}, out8);
  return FC_OK;
}

// inc/costmodel.hpp:153-167: strict '<' argmin in the order AG, ART_RING,
// ART_TREE (ties go to AG, then ART_RING); N < 2 is an invalid argument.
int fc_select_collective(double alpha, double bandwidth, double m_bytes, double c, int n,
                         int* choice, double* costs_out) {
  if (validate(alpha, bandwidth, m_bytes, c, n)) return FC_ERR_INVALID_ARGUMENT;
  if (n < 2) return FC_ERR_INVALID_ARGUMENT;
  double b[8];
  costs(Net{alpha, bandwidth}, Msg{m_bytes, c, n}, b);
  int ch = 0;
  double best = b[5];
  if (b[6] < best) {
    best = b[6];
    ch = 1;
  }
  if (b[7] < best) ch = 2;
  if (choice) *choice = ch;
  if (costs_out)
    for (int i = 0; i < 8; ++i) costs_out[i] = b[i];
  return FC_OK;
}

// Closed forms, Eq. (5a-c) (inc/costmodel.hpp:124-146):
//   which 0 = ring over tree, 1 = ring over AG, 2 = tree over AG.
int fc_prefer(double alpha, double bandwidth, double m_bytes, double c, int n, int which,
              int* out) {
  if (validate(alpha, bandwidth, m_bytes, c, n)) return FC_ERR_INVALID_ARGUMENT;
  const Net net{alpha, bandwidth};
  const double lg = std::log2(static_cast<double>(n));
  const double nm1 = n - 1;
  const double mc = m_bytes * c;
  bool r;
  switch (which) {
    case 0: r = net.alpha * (nm1 - lg) < mc * net.beta() * (lg - nm1 / n); break;
    case 1: r = net.alpha < mc * net.beta() * (1.0 - 1.0 / n - lg / (2.0 * nm1)); break;
    case 2: r = net.alpha < mc * net.beta() * (nm1 / lg - 1.5); break;
    default: return FC_ERR_INVALID_ARGUMENT;
  }
  *out = r ? 1 : 0;
  return FC_OK;
}

// inc/costmodel.hpp:180-203; pair 0 ring/tree, 1 ring/AG, 2 tree/AG.
// *has = 0 for "no crossover in (0, 1]".
int fc_crossover_cr(double alpha, double bandwidth, double m_bytes, int n, int pair, double* c_out,
                    int* has) {
  if (n < 2) return FC_ERR_INVALID_ARGUMENT;
  if (alpha < 0.0 || !(bandwidth > 0.0)) return FC_ERR_INVALID_ARGUMENT;
  const Net net{alpha, bandwidth};
  const double lg = std::log2(static_cast<double>(n));
  const double nm1 = n - 1;
  double coeff = 0.0;
  *has = 0;
  *c_out = 0.0;
  switch (pair) {
    case 0:
      if (nm1 - lg <= 0.0 || lg - nm1 / n <= 0.0) return FC_OK;
      coeff = (lg - nm1 / n) / (nm1 - lg);
      break;
    case 1: coeff = 1.0 - 1.0 / n - lg / (2.0 * nm1); break;
    case 2: coeff = nm1 / lg - 1.5; break;
    default: return FC_ERR_INVALID_ARGUMENT;
  }
  if (coeff <= 0.0) return FC_OK;
  const double c = (net.alpha / net.beta()) / (m_bytes * coeff);
  if (c > 1.0) return FC_OK;
  *has = 1;
  *c_out = c;
  return FC_OK;
}

// inc/costmodel.hpp:171-175: M implied by a measured compressed allgather.
int fc_derive_m_from_ag(double alpha, double bandwidth, double c, int n, double seconds,
                        double* m_out) {
  if (alpha < 0.0 || !(bandwidth > 0.0) || n < 2) return FC_ERR_INVALID_ARGUMENT;
  const Net net{alpha, bandwidth};
  const double lg = std::log2(static_cast<double>(n));
  *m_out = (seconds - net.alpha * lg) / (2.0 * c * net.beta() * (n - 1));
  return FC_OK;
}

}  // extern "C"
