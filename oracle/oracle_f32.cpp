// ORACLE — test infrastructure only.  Never linked into, imported by or
// executed on the product path; only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load it, and only as the checker.
//
// fp32 restatement of the reference's hot path (the reference is fp64,
// /root/reference/proj/include/flexcomm).  Each function follows the cited
// reference lines step by step with `double` replaced by `float` for values
// and `size_t` by `uint32_t` for indices, so that multi-step runs (where the
// reference's fp64 error-feedback sum would differ from the GPU's fp32 sum)
// have a bit-exact CPU answer.  It is pinned against the reference itself
// (oracle/_ref, tests/test_oracle.py) on every case where fp32 and fp64
// coincide, and against the reference tests' hand-executed vectors
// (tests/golden/).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <numeric>
#include <vector>

#include "fc_synth.h"

namespace {

// inc/compress.hpp:28-33
uint64_t k_of(double c, uint64_t g) {
  double raw = std::ceil(c * static_cast<double>(g) - 1e-9);
  uint64_t k = raw <= 0.0 ? 0 : static_cast<uint64_t>(raw);
  return std::min<uint64_t>(std::max<uint64_t>(k, 1), g);
}

// inc/compress.hpp:38-53: nth_element on (|v| desc, index asc), keep k,
// sort ascending.  The (|v|, index) order is carried by one packed 64-bit key
// per element -- high word the magnitude's bit pattern (for finite floats
// |a| > |b| <=> (bits(a) & 0x7fffffff) > (bits(b) & 0x7fffffff), and +0/-0
// share 0, exactly fabs's order), low word the complemented index (so a
// larger key means a lower index among equal magnitudes) -- so that
// nth_element runs over a contiguous array instead of an index permutation
// with a random-access comparator.  Same selection (the first k elements of
// the same total order), same output order; seconds instead of minutes at
// the BASELINE sizes.
inline uint64_t packed_key(const float* v, uint64_t i) {
  uint32_t b;
  std::memcpy(&b, v + i, 4);
  return (static_cast<uint64_t>(b & 0x7fffffffu) << 32) | (0xffffffffull - i);
}

void select_topk_indices(const float* v, uint64_t g, uint64_t k, std::vector<uint32_t>& out) {
  std::vector<uint64_t> key(g);
  for (uint64_t i = 0; i < g; ++i) key[i] = packed_key(v, i);
  std::nth_element(key.begin(), key.begin() + static_cast<std::ptrdiff_t>(k - 1), key.end(),
                   std::greater<uint64_t>());
  out.resize(k);
  for (uint64_t j = 0; j < k; ++j) out[j] = static_cast<uint32_t>(0xffffffffull - (key[j] & 0xffffffffull));
  std::sort(out.begin(), out.end());
}

// inc/compress.hpp:132-136 (values widened to double, sequential order)
double squared_norm(const float* v, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double x = v[i];
    s += x * x;
  }
  return s;
}

// inc/compress.hpp:67-79 topk_layerwise: per layer (offset, length) the exact
// top-k_of(c, length) of that slice; layers in map order.  No map -> exact.
void select_layerwise(const float* v, uint64_t g, double c, int nl, const uint64_t* off,
                      const uint64_t* len, std::vector<uint32_t>& out) {
  out.clear();
  if (nl <= 0) {
    select_topk_indices(v, g, k_of(c, g), out);
    return;
  }
  for (int l = 0; l < nl; ++l) {
    std::vector<uint32_t> part;
    select_topk_indices(v + off[l], len[l], k_of(c, len[l]), part);
    for (uint32_t i : part) out.push_back(static_cast<uint32_t>(i + off[l]));
  }
}

// inc/compress.hpp:81-112 topk_threshold: bisect t in [0, max|v|] (doubles)
// for `rounds` rounds, stopping when exactly k elements have |v| >= t; keep
// every element with |v| >= t (count may differ from k).
void select_threshold(const float* v, uint64_t g, double c, int rounds, std::vector<uint32_t>& out) {
  const uint64_t k = k_of(c, g);
  double hi = 0.0;
  for (uint64_t i = 0; i < g; ++i) hi = std::max(hi, static_cast<double>(std::fabs(v[i])));
  double lo = 0.0, t = 0.0;
  for (int r = 0; r < rounds; ++r) {
    t = (lo + hi) / 2.0;
    uint64_t count = 0;
    for (uint64_t i = 0; i < g; ++i)
      if (static_cast<double>(std::fabs(v[i])) >= t) ++count;
    if (count == k) break;
    if (count > k) lo = t;
    else hi = t;
  }
  out.clear();
  for (uint64_t i = 0; i < g; ++i)
    if (static_cast<double>(std::fabs(v[i])) >= t) out.push_back(static_cast<uint32_t>(i));
}

// inc/artopk.hpp:115-123 run_compressor (kind 0 exact, 1 layerwise, 2 threshold)
void compress(int kind, const float* v, uint64_t g, double c, int nl, const uint64_t* off,
              const uint64_t* len, int rounds, std::vector<uint32_t>& out) {
  if (kind == 1) select_layerwise(v, g, c, nl, off, len, out);
  else if (kind == 2) select_threshold(v, g, c, rounds, out);
  else select_topk_indices(v, g, k_of(c, g), out);
}

}  // namespace

extern "C" {

uint64_t orc_k_of(double c, uint64_t g) {
  if (!(c > 0.0 && c <= 1.0) || g == 0) return 0;
  return k_of(c, g);
}

// inc/compress.hpp:57-65 topk_exact
uint64_t orc_topk_exact(const float* v, uint64_t g, double c, uint32_t* idx_out, float* val_out) {
  if (!(c > 0.0 && c <= 1.0) || g == 0) return 0;
  const uint64_t k = k_of(c, g);
  std::vector<uint32_t> idx;
  select_topk_indices(v, g, k, idx);
  for (uint64_t j = 0; j < k; ++j) {
    if (idx_out) idx_out[j] = idx[j];
    if (val_out) val_out[j] = v[idx[j]];
  }
  return k;
}

double orc_squared_norm(const float* v, uint64_t n) { return squared_norm(v, n); }

// topk_exact at several ratios of one vector (the C5 ladder): the packed key
// array is built once and re-partitioned per k (nth_element only needs a
// permutation of the keys).  idx_out[r] receives k_of(cs[r], g) indices.
int orc_topk_multi(const float* v, uint64_t g, const double* cs, int ncs, uint32_t** idx_out) {
  if (g == 0 || ncs < 1) return 1;
  std::vector<uint64_t> key(g);
  for (uint64_t i = 0; i < g; ++i) key[i] = packed_key(v, i);
  for (int r = 0; r < ncs; ++r) {
    if (!(cs[r] > 0.0 && cs[r] <= 1.0)) return 1;
    const uint64_t k = k_of(cs[r], g);
    std::nth_element(key.begin(), key.begin() + static_cast<std::ptrdiff_t>(k - 1), key.end(),
                     std::greater<uint64_t>());
    uint32_t* o = idx_out[r];
    for (uint64_t j = 0; j < k; ++j) o[j] = static_cast<uint32_t>(0xffffffffull - (key[j] & 0xffffffffull));
    std::sort(o, o + k);
  }
  return 0;
}

// inc/artopk.hpp:62-111 artopk_step (Alg. 1), fp32.
// g_o: n*g, res: n*g (in/out), agg_out: g, bidx_out: k (may be NULL),
// norms_out: n (VAR scores; may be NULL).  Returns k, or 0 on bad input.
uint64_t orc_artopk_step(int n, uint64_t g, const float* g_o, float* res, double c, int mode,
                         long step, int op, float* agg_out, int* sel_out, uint32_t* bidx_out,
                         double* norms_out) {
  if (n < 1 || g == 0 || !(c > 0.0 && c <= 1.0)) return 0;
  const uint64_t k = k_of(c, g);
  std::vector<std::vector<float>> ge(n, std::vector<float>(g));
  std::vector<std::vector<uint32_t>> local(n);
  std::vector<double> norms(n, 0.0);
  for (int r = 0; r < n; ++r) {
    // error_feedback, inc/compress.hpp:114-120: g_e = g_o; g_e += res
    for (uint64_t i = 0; i < g; ++i) ge[r][i] = g_o[r * g + i] + res[r * g + i];
    select_topk_indices(ge[r].data(), g, k, local[r]);
    std::vector<float> vals(k);
    for (uint64_t j = 0; j < k; ++j) vals[j] = ge[r][local[r][j]];
    norms[r] = squared_norm(vals.data(), k);
  }
  int sel;
  if (mode == 0) {
    sel = static_cast<int>(step % n);  // select_star, inc/artopk.hpp:27-30
    if (sel < 0) return 0;
  } else {
    sel = 0;  // select_var, inc/artopk.hpp:35-48 (strict >, ties -> lowest rank)
    for (int r = 1; r < n; ++r)
      if (norms[r] > norms[sel]) sel = r;
  }
  const std::vector<uint32_t>& indices = local[sel];
  std::vector<std::vector<float>> contrib(n, std::vector<float>(k));
  for (int r = 0; r < n; ++r) {
    for (uint64_t j = 0; j < k; ++j) contrib[r][j] = ge[r][indices[j]];
    // residual before reduction: g_e with zeros at the broadcast indices
    for (uint64_t i = 0; i < g; ++i) res[r * g + i] = ge[r][i];
    for (uint64_t j = 0; j < k; ++j) res[r * g + indices[j]] = 0.0f;
  }
  // allreduce, inc/collectives.hpp:82-87: rank-ascending sum, then /N (Avg)
  std::vector<float> out = contrib[0];
  for (int r = 1; r < n; ++r)
    for (uint64_t j = 0; j < k; ++j) out[j] += contrib[r][j];
  if (op == 1)
    for (uint64_t j = 0; j < k; ++j) out[j] /= static_cast<float>(n);
  // densify, inc/core.hpp:72-81
  std::memset(agg_out, 0, g * sizeof(float));
  for (uint64_t j = 0; j < k; ++j) agg_out[indices[j]] = out[j];
  if (sel_out) *sel_out = sel;
  if (bidx_out)
    for (uint64_t j = 0; j < k; ++j) bidx_out[j] = indices[j];
  if (norms_out)
    for (int r = 0; r < n; ++r) norms_out[r] = norms[r];
  return k;
}

// inc/artopk.hpp:128-161 ag_step (Exact compressor), fp32.
uint64_t orc_ag_step(int n, uint64_t g, const float* g_o, float* res, double c, float* agg_out) {
  if (n < 1 || g == 0 || !(c > 0.0 && c <= 1.0)) return 0;
  const uint64_t k = k_of(c, g);
  std::vector<std::vector<uint32_t>> idx(n);
  std::vector<std::vector<float>> val(n);
  std::vector<float> ge(g);
  for (int r = 0; r < n; ++r) {
    for (uint64_t i = 0; i < g; ++i) ge[i] = g_o[r * g + i] + res[r * g + i];
    select_topk_indices(ge.data(), g, k, idx[r]);
    val[r].resize(k);
    for (uint64_t j = 0; j < k; ++j) val[r][j] = ge[idx[r][j]];
    // residual_update, inc/compress.hpp:122-130: res = g_e; res[idx] -= val
    for (uint64_t i = 0; i < g; ++i) res[r * g + i] = ge[i];
    for (uint64_t j = 0; j < k; ++j) res[r * g + idx[r][j]] -= val[r][j];
  }
  for (uint64_t i = 0; i < g; ++i) agg_out[i] = 0.0f;
  for (int r = 0; r < n; ++r)
    for (uint64_t j = 0; j < k; ++j) agg_out[idx[r][j]] += val[r][j];
  for (uint64_t i = 0; i < g; ++i) agg_out[i] /= static_cast<float>(n);
  return k;
}

// Layerwise / threshold Top-k of one vector (no error feedback).  Writes
// the selection (count returned; idx/val must hold g entries).
uint64_t orc_topk_kind(const float* v, uint64_t g, double c, int kind, int nl, const uint64_t* off,
                       const uint64_t* len, int rounds, uint32_t* idx_out, float* val_out) {
  if (!(c > 0.0 && c <= 1.0) || g == 0) return 0;
  std::vector<uint32_t> idx;
  compress(kind, v, g, c, nl, off, len, rounds, idx);
  for (size_t j = 0; j < idx.size(); ++j) {
    if (idx_out) idx_out[j] = idx[j];
    if (val_out) val_out[j] = v[idx[j]];
  }
  return idx.size();
}

// inc/artopk.hpp:128-161 ag_step with any compressor, fp32.  counts_out[r]
// (may be NULL) gets each worker's selection size.  Returns max count.
uint64_t orc_ag_step_kind(int n, uint64_t g, const float* g_o, float* res, double c, int kind, int nl,
                          const uint64_t* off, const uint64_t* len, int rounds, float* agg_out,
                          uint64_t* counts_out) {
  if (n < 1 || g == 0 || !(c > 0.0 && c <= 1.0)) return 0;
  std::vector<std::vector<uint32_t>> idx(n);
  std::vector<std::vector<float>> val(n);
  std::vector<float> ge(g);
  uint64_t maxk = 0;
  for (int r = 0; r < n; ++r) {
    for (uint64_t i = 0; i < g; ++i) ge[i] = g_o[r * g + i] + res[r * g + i];
    compress(kind, ge.data(), g, c, nl, off, len, rounds, idx[r]);
    val[r].resize(idx[r].size());
    for (size_t j = 0; j < idx[r].size(); ++j) val[r][j] = ge[idx[r][j]];
    for (uint64_t i = 0; i < g; ++i) res[r * g + i] = ge[i];
    for (size_t j = 0; j < idx[r].size(); ++j) res[r * g + idx[r][j]] -= val[r][j];
    maxk = std::max<uint64_t>(maxk, idx[r].size());
    if (counts_out) counts_out[r] = idx[r].size();
  }
  for (uint64_t i = 0; i < g; ++i) agg_out[i] = 0.0f;
  for (int r = 0; r < n; ++r)
    for (size_t j = 0; j < idx[r].size(); ++j) agg_out[idx[r][j]] += val[r][j];
  for (uint64_t i = 0; i < g; ++i) agg_out[i] /= static_cast<float>(n);
  return maxk;
}

// Dense sync, inc/trainer.hpp:240-244 -> allreduce(g_o), collectives.hpp:82-87
void orc_dense(int n, uint64_t g, const float* g_o, int op, float* agg_out) {
  for (uint64_t i = 0; i < g; ++i) agg_out[i] = g_o[i];
  for (int r = 1; r < n; ++r)
    for (uint64_t i = 0; i < g; ++i) agg_out[i] += g_o[r * g + i];
  if (op == 1)
    for (uint64_t i = 0; i < g; ++i) agg_out[i] /= static_cast<float>(n);
}

// Host twin of the device generator (include/fc_synth.h).
void orc_fill_synth(float* dst, uint64_t g, uint64_t seed, uint32_t rank, uint64_t step, int dist) {
  const uint64_t key = fc_stream_key(seed, rank, step);
  for (uint64_t i = 0; i < g; ++i) dst[i] = fc_synth_value(key, i, dist);
}

}  // extern "C"
