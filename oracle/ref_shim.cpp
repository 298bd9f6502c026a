// ORACLE — test infrastructure only (see oracle/oracle_f32.cpp header).
//
// C-ABI shim around the UNMODIFIED reference implementation.  This file
// contains no reference code: it #includes the reference headers where they
// lie (/root/reference/proj/include, via -I in oracle/Makefile) and exposes
// flexcomm::artopk_step / ag_step / topk_exact / k_of / select_collective /
// the Controller pieces through plain pointers, so that tests can pin the
// fp32 restatement against the real thing and bench.py can time the
// reference's CPU path on the GPU box's host.  Built into oracle/_ref/.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fc_synth.h"
#include "flexcomm/artopk.hpp"
#include "flexcomm/collectives.hpp"
#include "flexcomm/compress.hpp"
#include "flexcomm/core.hpp"
#include "flexcomm/costmodel.hpp"
#include "flexcomm/moo.hpp"
#include "flexcomm/netsched.hpp"

using namespace flexcomm;

namespace {

int code_of(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::out_of_range&) {
    return 2;
  } catch (const std::runtime_error&) {
    return 3;
  } catch (...) {
    return 9;
  }
}

struct RefState {
  int n = 1;
  std::size_t g = 0;
  std::vector<DenseGrad> g_o;
  ResidualStore res;
  DenseGrad last;
  int last_sel = -1;
  SimClock clock;
};

}  // namespace

extern "C" {

// ---- stateless wrappers ---------------------------------------------------

int ref_k_of(double c, uint64_t g, uint64_t* k) {
  try {
    *k = k_of(CompressionRatio(c), g);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_topk_exact(const double* v, uint64_t g, double c, uint64_t* idx_out, double* val_out,
                   uint64_t* k_out) {
  try {
    DenseGrad d;
    d.values.assign(v, v + g);
    SparseGrad s = topk_exact(d, CompressionRatio(c));
    for (std::size_t j = 0; j < s.indices.size(); ++j) {
      if (idx_out) idx_out[j] = s.indices[j];
      if (val_out) val_out[j] = s.values[j];
    }
    *k_out = s.indices.size();
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// One artopk_step over caller arrays: g_o n*g (in), res n*g (in/out),
// agg g (out).  sync_charge = seconds charged to SimClock Sync.
int ref_artopk_step(int n, uint64_t g, const double* g_o, double* res, double c, int mode,
                    int algo, long step, int op, double payload_scale, double alpha,
                    double bandwidth, double* agg, int* sel, double* sync_charge) {
  try {
    SimClock clk;
    Cluster cluster(n, NetParams(alpha, bandwidth), &clk);
    std::vector<DenseGrad> grads(static_cast<std::size_t>(n));
    ResidualStore store(n, g);
    for (int r = 0; r < n; ++r) {
      grads[r].values.assign(g_o + r * g, g_o + (r + 1) * g);
      store.of(r).assign(res + r * g, res + (r + 1) * g);
    }
    auto out = artopk_step(cluster, grads, store, CompressionRatio(c),
                           mode == 0 ? SelectionMode::STAR : SelectionMode::VAR,
                           algo == 0 ? ReduceAlgo::Ring : ReduceAlgo::Tree, step, nullptr,
                           op == 0 ? ReduceOp::Sum : ReduceOp::Avg, payload_scale);
    for (int r = 0; r < n; ++r) std::memcpy(res + r * g, store.of(r).data(), g * sizeof(double));
    std::memcpy(agg, out.aggregate.values.data(), g * sizeof(double));
    *sel = out.selected_rank;
    if (sync_charge) *sync_charge = clk.of(Category::Sync);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_ag_step(int n, uint64_t g, const double* g_o, double* res, double c, double payload_scale,
                double alpha, double bandwidth, double* agg, double* sync_charge) {
  try {
    SimClock clk;
    Cluster cluster(n, NetParams(alpha, bandwidth), &clk);
    std::vector<DenseGrad> grads(static_cast<std::size_t>(n));
    ResidualStore store(n, g);
    for (int r = 0; r < n; ++r) {
      grads[r].values.assign(g_o + r * g, g_o + (r + 1) * g);
      store.of(r).assign(res + r * g, res + (r + 1) * g);
    }
    auto out = ag_step(cluster, grads, store, CompressionRatio(c), CompressorKind::Exact,
                       payload_scale);
    for (int r = 0; r < n; ++r) std::memcpy(res + r * g, store.of(r).data(), g * sizeof(double));
    std::memcpy(agg, out.values.data(), g * sizeof(double));
    if (sync_charge) *sync_charge = clk.of(Category::Sync);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// topk_layerwise / topk_threshold (inc/compress.hpp:67-112) on one vector;
// kind 1 layerwise (nl layers, offsets/lengths), kind 2 threshold.  Writes
// the selection; returns its size or -code.
long ref_topk_kind(const double* v, uint64_t g, double c, int kind, int nl, const uint64_t* off,
                   const uint64_t* len, int rounds, uint64_t* idx_out, double* val_out) {
  try {
    DenseGrad d;
    d.values.assign(v, v + g);
    for (int l = 0; l < nl; ++l) d.layer_map.push_back({"L" + std::to_string(l), off[l], len[l]});
    SparseGrad s = kind == 1 ? topk_layerwise(d, CompressionRatio(c))
                             : topk_threshold(d, CompressionRatio(c), rounds);
    for (std::size_t j = 0; j < s.indices.size(); ++j) {
      idx_out[j] = s.indices[j];
      val_out[j] = s.values[j];
    }
    return static_cast<long>(s.indices.size());
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// ag_step with a compressor kind (inc/artopk.hpp:128-161); the gradients carry
// the layer map (error_feedback copies it into g_e).
int ref_ag_step_kind(int n, uint64_t g, const double* g_o, double* res, double c, int kind, int nl,
                     const uint64_t* off, const uint64_t* len, int rounds, double* agg) {
  try {
    SimClock clk;
    Cluster cluster(n, NetParams(0.001, 1e9), &clk);
    std::vector<DenseGrad> grads(static_cast<std::size_t>(n));
    ResidualStore store(n, g);
    for (int r = 0; r < n; ++r) {
      grads[r].values.assign(g_o + r * g, g_o + (r + 1) * g);
      for (int l = 0; l < nl; ++l) grads[r].layer_map.push_back({"L" + std::to_string(l), off[l], len[l]});
      store.of(r).assign(res + r * g, res + (r + 1) * g);
    }
    auto out = ag_step(cluster, grads, store, CompressionRatio(c), static_cast<CompressorKind>(kind), 1.0,
                       rounds);
    for (int r = 0; r < n; ++r) std::memcpy(res + r * g, store.of(r).data(), g * sizeof(double));
    std::memcpy(agg, out.values.data(), g * sizeof(double));
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// select_collective (inc/costmodel.hpp:153-167); costs_out gets the eight
// CostBreakdown fields in declaration order.
int ref_select_collective(double alpha, double bandwidth, double m_bytes, double c, int n,
                          int* choice, double* costs_out) {
  try {
    auto ch = select_collective(NetParams(alpha, bandwidth), MessageSpec(m_bytes, c, n));
    *choice = static_cast<int>(ch.collective);
    if (costs_out) {
      const CostBreakdown& b = ch.costs;
      const double v[8] = {b.ps, b.ring_ar, b.tree_ar, b.broadcast, b.allgather_dense,
                           b.ag_compressed, b.art_ring, b.art_tree};
      std::memcpy(costs_out, v, sizeof(v));
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// crossover_cr (inc/costmodel.hpp:180-203); returns 0 with *has=0 for nullopt.
int ref_crossover_cr(double alpha, double bandwidth, double m_bytes, int n, int pair, double* c,
                     int* has) {
  try {
    auto r = crossover_cr(NetParams(alpha, bandwidth), m_bytes, n,
                          static_cast<CollectivePair>(pair));
    *has = r.has_value() ? 1 : 0;
    *c = r.value_or(0.0);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// candidate_ladder (inc/moo.hpp:52-65); returns the rung count.
int ref_candidate_ladder(double c_low, double c_high, double factor, double* out, int cap) {
  try {
    ControllerConfig cfg;
    cfg.c_low = c_low;
    cfg.c_high = c_high;
    cfg.factor = factor;
    auto l = candidate_ladder(cfg);
    for (int i = 0; i < (int)l.size() && i < cap; ++i) out[i] = l[i];
    return (int)l.size();
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// pareto_front + choose_cr (inc/moo.hpp:88-146) over m candidates given as
// (c, gain_avg, t_comp_avg, t_sync_modeled) rows.  front_mask[i] = 1 if row
// i is on the front; returns the chosen c via *chosen and the collective.
int ref_choose_cr(const double* rows, int m, double alpha, double bandwidth, double m_bytes, int n,
                  int* front_mask, double* chosen, int* collective) {
  try {
    std::vector<CandidateCR> cands;
    for (int i = 0; i < m; ++i)
      cands.push_back({rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]});
    auto front = pareto_front(cands);
    for (int i = 0; i < m; ++i) {
      front_mask[i] = 0;
      for (const auto& f : front)
        if (f.c == cands[i].c && f.gain_avg == cands[i].gain_avg &&
            f.t_comp_avg == cands[i].t_comp_avg && f.t_sync_modeled == cands[i].t_sync_modeled)
          front_mask[i] = 1;
    }
    auto ch = choose_cr(front, NetParams(alpha, bandwidth), m_bytes, n);
    *chosen = ch.candidate.c;
    *collective = static_cast<int>(ch.collective);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// round_3sig (inc/moo.hpp:44-48)
double ref_round_3sig(double v) { return round_3sig(v); }

// trigger_gain (inc/moo.hpp:67-71) after pushing `count` samples into a
// GainTracker of the given window (inc/compress.hpp:145-165); -code on error.
int ref_trigger_gain(double gain_ref, const double* samples, uint64_t count, uint64_t window,
                     double threshold) {
  try {
    GainTracker t(window);
    for (uint64_t i = 0; i < count; ++i) t.push(samples[i]);
    return trigger_gain(gain_ref, t, threshold) ? 1 : 0;
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

// network_changed (inc/netsched.hpp:50-58)
int ref_network_changed(double a0, double b0, double a1, double b1, double rel) {
  return network_changed(NetParams(a0, b0), NetParams(a1, b1), rel) ? 1 : 0;
}

// params_at (inc/netsched.hpp:38-46) over m segments (start_epoch, alpha, bandwidth)
int ref_params_at(const double* segs, int m, long epoch, double* alpha, double* bandwidth) {
  try {
    NetworkSchedule s;
    for (int i = 0; i < m; ++i)
      s.segments.push_back({static_cast<long>(segs[3 * i]), NetParams(segs[3 * i + 1], segs[3 * i + 2])});
    auto p = params_at(s, epoch);
    *alpha = p.alpha;
    *bandwidth = p.bandwidth;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// ---- persistent state for the CPU baseline timing --------------------------
// Gradients come from the same synthetic generator as the device
// (include/fc_synth.h), widened to double; only the reference call itself is
// timed (std::chrono::steady_clock).

void* ref_state_create(int n, uint64_t g) {
  try {
    auto* s = new RefState();
    s->n = n;
    s->g = g;
    s->g_o.resize(static_cast<std::size_t>(n));
    for (auto& d : s->g_o) d.values.assign(g, 0.0);
    s->res = ResidualStore(n, g);
    return s;
  } catch (...) {
    return nullptr;
  }
}

void ref_state_destroy(void* p) { delete static_cast<RefState*>(p); }

void ref_state_fill_synth(void* p, int worker, uint64_t seed, uint32_t rank, uint64_t step, int dist) {
  auto* s = static_cast<RefState*>(p);
  const uint64_t key = fc_stream_key(seed, rank, step);
  auto& v = s->g_o[static_cast<std::size_t>(worker)].values;
  for (std::size_t i = 0; i < s->g; ++i) v[i] = static_cast<double>(fc_synth_value(key, i, dist));
}

// Returns seconds spent inside flexcomm::artopk_step (or ag_step when
// mode == 2); < 0 on error.
double ref_state_step(void* p, double c, int mode, int algo, long step) {
  auto* s = static_cast<RefState*>(p);
  try {
    Cluster cluster(s->n, NetParams(1e-5, 900e9 * 8), &s->clock);
    auto t0 = std::chrono::steady_clock::now();
    if (mode == 2) {
      s->last = ag_step(cluster, s->g_o, s->res, CompressionRatio(c));
      s->last_sel = -1;
    } else {
      auto r = artopk_step(cluster, s->g_o, s->res, CompressionRatio(c),
                           mode == 0 ? SelectionMode::STAR : SelectionMode::VAR,
                           algo == 0 ? ReduceAlgo::Ring : ReduceAlgo::Tree, step);
      s->last_sel = r.selected_rank;
      s->last = std::move(r.aggregate);
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (...) {
    return -1.0;
  }
}

int ref_state_selected(void* p) { return static_cast<RefState*>(p)->last_sel; }

void ref_state_aggregate(void* p, double* out) {
  auto* s = static_cast<RefState*>(p);
  std::memcpy(out, s->last.values.data(), s->g * sizeof(double));
}

void ref_state_residual(void* p, int worker, double* out) {
  auto* s = static_cast<RefState*>(p);
  std::memcpy(out, s->res.of(worker).data(), s->g * sizeof(double));
}

}  // extern "C"
