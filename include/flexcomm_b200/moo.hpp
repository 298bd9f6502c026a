// flexcomm_b200/moo.hpp — the reference's adaptive-CR controller
// (inc/moo.hpp) over the B200 sync path, with the sync side of its Trainer
// (inc/trainer.hpp) re-based on device state.
//
//   reference                                  here
//   ----------------------------------------   -----------------------------------
//   ControllerConfig, CandidateCR, CrChoice    same names (inc/moo.hpp:20-107)
//   round_3sig, candidate_ladder               fc_round_3sig / fc_candidate_ladder
//   trigger_gain, pareto_front, choose_cr      fc_trigger_gain / fc_pareto_front / fc_choose_cr
//   GainTracker                                GainTracker (inc/compress.hpp:145-165)
//   NetworkSchedule, params_at,                same (inc/netsched.hpp:13-58)
//     network_changed
//   Controller                                 Controller (same state machine, :159-271)
//   Trainer                                    SyncTrainer: the sync side only
//
// The decision arithmetic runs in the library (csrc/fc_moo.cpp), bit-exact
// with the reference (tests/test_moo.py).  SyncTrainer differs from the
// reference Trainer where the device path makes it so: its trajectory is
// the HBM residual store (snapshot/restore = fc_snapshot/fc_restore), the
// compression time of a step is measured with CUDA events (max over ranks)
// instead of the 0.5 ns/element model (inc/trainer.hpp:344-359), and the
// gradients come from a caller-supplied source (default: the synthetic
// generator); the toy model and its SGD update are out of scope.
#pragma once

#include <cmath>
#include <deque>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "flexcomm_b200/flexcomm.hpp"

namespace flexcomm {
namespace b200 {

struct ControllerConfig {
  double c_low = 0.001;
  double c_high = 0.1;
  double factor = 3.0;
  int probe_iters = 10;
  double gain_threshold = 0.10;

  fc_controller_config raw() const { return {c_low, c_high, factor, probe_iters, gain_threshold}; }
  void validate() const {
    const fc_controller_config c = raw();
    if (fc_controller_config_validate(&c) != FC_OK)
      throw std::invalid_argument(
          "invalid controller config (need 0 < c_low <= c_high <= 1, factor > 1, probe_iters >= 1, "
          "gain_threshold >= 0)");
  }
};

inline double round_3sig(double v) {
  double out = 0;
  check(fc_round_3sig(v, &out));
  return out;
}

inline std::vector<double> candidate_ladder(const ControllerConfig& cfg) {
  cfg.validate();
  const fc_controller_config c = cfg.raw();
  int n = 0;
  check(fc_candidate_ladder(&c, nullptr, 0, &n));
  std::vector<double> out(static_cast<std::size_t>(n));
  check(fc_candidate_ladder(&c, out.data(), n, &n));
  return out;
}

struct GainTracker {
  std::size_t window = 50;
  std::deque<double> samples;
  explicit GainTracker(std::size_t w = 50) : window(w) {
    if (window == 0) throw std::invalid_argument("window must be positive");
  }
  void push(double g) {
    samples.push_back(g);
    if (samples.size() > window) samples.pop_front();
  }
  std::size_t count() const { return samples.size(); }
  double mean() const {
    if (samples.empty()) throw std::runtime_error("no gain samples");
    double s = 0.0;
    for (double v : samples) s += v;
    return s / static_cast<double>(samples.size());
  }
};

inline bool trigger_gain(double gain_ref, const GainTracker& t, double threshold) {
  std::vector<double> s(t.samples.begin(), t.samples.end());
  int fire = 0;
  check(fc_trigger_gain(gain_ref, s.data(), s.size(), threshold, &fire));
  return fire != 0;
}

using CandidateCR = fc_candidate;  // {c, gain_avg, t_comp_avg, t_sync_modeled}

inline std::vector<CandidateCR> pareto_front(const std::vector<CandidateCR>& cands) {
  if (cands.empty()) throw std::invalid_argument("empty candidate set");
  std::vector<int> mask(cands.size());
  check(fc_pareto_front(cands.data(), static_cast<int>(cands.size()), mask.data()));
  std::vector<CandidateCR> front;
  for (std::size_t i = 0; i < cands.size(); ++i)
    if (mask[i]) front.push_back(cands[i]);
  return front;
}

struct CrChoice {
  CandidateCR candidate{1.0, 1.0, 0.0, 0.0};
  Collective collective = Collective::AG;
};

inline CrChoice choose_cr(const std::vector<CandidateCR>& front, const NetParams& net, double m_bytes,
                          int n) {
  if (front.empty()) throw std::invalid_argument("empty pareto front");
  MessageSpec(m_bytes, 1.0, n);  // the reference's argument validation
  if (n < 2) throw std::invalid_argument("selection undefined for single worker");
  int chosen = 0, coll = 0;
  check(fc_choose_cr(front.data(), static_cast<int>(front.size()), net.alpha, net.bandwidth, m_bytes, n,
                     &chosen, &coll));
  return {front[static_cast<std::size_t>(chosen)], static_cast<Collective>(coll)};
}

// ---- network schedule (inc/netsched.hpp:13-58) ---------------------------------
struct Segment {
  long start_epoch = 0;
  NetParams net;
};

struct NetworkSchedule {
  std::vector<Segment> segments;
  void validate() const {
    if (segments.empty()) throw std::invalid_argument("empty network schedule");
    if (segments.front().start_epoch != 0) throw std::invalid_argument("first segment must start at epoch 0");
    for (std::size_t i = 1; i < segments.size(); ++i)
      if (segments[i].start_epoch <= segments[i - 1].start_epoch)
        throw std::invalid_argument("segment start epochs must be strictly ascending");
  }
};

inline NetParams params_at(const NetworkSchedule& s, long epoch) {
  if (epoch < 0) throw std::invalid_argument("epoch must be >= 0");
  s.validate();
  NetParams cur = s.segments.front().net;
  for (const auto& seg : s.segments)
    if (seg.start_epoch <= epoch) cur = seg.net;
  return cur;
}

inline bool network_changed(const NetParams& prev, const NetParams& cur, double rel_threshold = 0.0) {
  int ch = 0;
  check(fc_network_changed(prev.alpha, prev.bandwidth, cur.alpha, cur.bandwidth, rel_threshold, &ch));
  return ch != 0;
}

// ---- the Trainer's sync side on the device ------------------------------------------
enum class SyncMode { Dense, AG, STAR, VAR };

struct SyncConfig {
  long epochs = 5;
  long steps_per_epoch = 10;
  double c = 1.0;
  bool adaptive = false;
  SyncMode mode = SyncMode::STAR;
  ReduceAlgo reduce_algo = ReduceAlgo::Ring;
  ReduceOp reduce_op = ReduceOp::Avg;
  bool error_feedback = true;
  std::size_t gain_window = 50;
  double size_bytes_override = 0.0;
  double net_change_threshold = 0.0;
  double t_compute = 0.0;  // seconds charged per step for the (external) backward pass
  double t_io = 0.0;
  uint64_t seed = 42;
  int dist = 0;  // fc_fill_synthetic distribution: 0 normal, 1 ties, 2 layered

  void validate() const {
    if (epochs < 1) throw std::invalid_argument("epochs must be >= 1");
    if (steps_per_epoch < 1) throw std::invalid_argument("steps_per_epoch must be >= 1");
    if (!(c > 0.0 && c <= 1.0)) throw std::invalid_argument("compression ratio out of (0,1]");
    if (t_io < 0.0 || t_compute < 0.0) throw std::invalid_argument("t_io / t_compute must be >= 0");
    if (gain_window == 0) throw std::invalid_argument("window must be positive");
  }
};

struct StepMetrics {  // inc/trainer.hpp:84-96 (the model's loss is out of scope)
  long step = 0;
  double t_compute = 0.0, t_comp_decomp = 0.0, t_sync = 0.0, t_io = 0.0, t_step = 0.0;
  double gain = 1.0;
  double cr_used = 1.0;
  std::string collective_used;
  int selected_rank = -1;
};

class SyncTrainer {
 public:
  struct Snapshot {
    unsigned long generation = 0;
    GainTracker tracker;
    long step_index = 0;
    double current_c = 1.0;
    Collective current_collective = Collective::AG;
  };
  // fills this step's gradients into the context (default: synthetic)
  using GradSource = std::function<void(SyncTrainer&, long step)>;

  SyncTrainer(std::shared_ptr<Context> ctx, SyncConfig cfg, NetworkSchedule sched, GradSource src = {})
      : ctx_(std::move(ctx)), cfg_(cfg), sched_(std::move(sched)), src_(std::move(src)), tracker_(cfg.gain_window) {
    cfg_.validate();
    sched_.validate();
    current_c_ = cfg_.c;
    current_collective_ = cfg_.mode == SyncMode::AG ? Collective::AG
                          : cfg_.reduce_algo == ReduceAlgo::Ring ? Collective::ART_RING
                                                                 : Collective::ART_TREE;
  }

  int n() const { return ctx_->world(); }
  const SyncConfig& config() const { return cfg_; }
  Context& context() { return *ctx_; }
  SimClock& clock() { return clock_; }
  long step_index() const { return step_index_; }
  long total_steps() const { return cfg_.epochs * cfg_.steps_per_epoch; }
  long epoch_of(long step) const { return step / cfg_.steps_per_epoch; }
  NetParams net_at_step(long step) const { return params_at(sched_, epoch_of(step)); }
  double m_eff() const {
    return cfg_.size_bytes_override > 0.0 ? cfg_.size_bytes_override : 4.0 * static_cast<double>(ctx_->grad_len());
  }
  GainTracker& gain_tracker() { return tracker_; }
  const std::vector<StepMetrics>& metrics() const { return metrics_; }
  double current_c() const { return current_c_; }
  Collective current_collective() const { return current_collective_; }
  void set_compression(double c, Collective coll) {
    if (!(c > 0.0 && c <= 1.0)) throw std::invalid_argument("compression ratio out of (0,1]");
    if (c != current_c_) tracker_ = GainTracker(cfg_.gain_window);
    current_c_ = c;
    current_collective_ = coll;
  }
  bool probe_mode() const { return probe_; }
  void set_probe_mode(bool on) { probe_ = on; }

  Snapshot snapshot() {
    ctx_->snapshot();
    return {++gen_, tracker_, step_index_, current_c_, current_collective_};
  }
  void restore(const Snapshot& s) {
    if (s.generation != gen_) throw std::runtime_error("restore of a superseded snapshot (one device slot)");
    ctx_->restore();
    tracker_ = s.tracker;
    step_index_ = s.step_index;
    current_c_ = s.current_c;
    current_collective_ = s.current_collective;
  }

  StepMetrics step() {
    fc_ctx* c = ctx_->get();
    StepMetrics m;
    m.step = step_index_;
    m.cr_used = effective_c();
    m.t_io = cfg_.t_io;
    m.t_compute = cfg_.t_compute;
    if (src_) {
      src_(*this, step_index_);
    } else {
      for (int w = 0; w < ctx_->n_local(); ++w)
        check(fc_fill_synthetic(c, w, cfg_.seed, static_cast<uint32_t>(ctx_->rank() + w),
                                static_cast<uint64_t>(step_index_), cfg_.dist));
    }
    fc_step_stats st{};
    double gain = 1.0, t_comp = 0.0;
    const SyncMode mode = effective_mode();
    if (mode == SyncMode::Dense) {
      check(fc_dense_step(c, cfg_.reduce_algo == ReduceAlgo::Ring ? FC_RING : FC_TREE,
                          cfg_.reduce_op == ReduceOp::Sum ? FC_SUM : FC_AVG, &st));
      m.collective_used = cfg_.reduce_algo == ReduceAlgo::Ring ? "RING_AR" : "TREE_AR";
    } else if (mode == SyncMode::AG) {
      check(fc_ag_step(c, m.cr_used, FC_EXACT, &st));
      check(fc_moo_metrics(c, 1, &st, &gain, &t_comp));
      m.collective_used = "AG";
    } else {
      ReduceAlgo algo = current_collective_ == Collective::ART_TREE ? ReduceAlgo::Tree : cfg_.reduce_algo;
      if (current_collective_ == Collective::ART_RING) algo = ReduceAlgo::Ring;
      check(fc_artopk_step(c, m.cr_used, mode == SyncMode::VAR ? FC_VAR : FC_STAR,
                           algo == ReduceAlgo::Ring ? FC_RING : FC_TREE, step_index_,
                           cfg_.reduce_op == ReduceOp::Sum ? FC_SUM : FC_AVG, &st));
      check(fc_moo_metrics(c, 0, &st, &gain, &t_comp));
      m.selected_rank = st.selected_rank;
      m.collective_used = algo == ReduceAlgo::Ring ? "ART_RING" : "ART_TREE";
    }
    m.t_sync = st.ms_exchange * 1e-3;
    m.gain = gain;
    tracker_.push(gain);
    m.t_comp_decomp = t_comp;
    charge(Category::Sync, m.t_sync);
    charge(Category::Compression, m.t_comp_decomp);
    charge(Category::Compute, m.t_compute);
    charge(Category::Io, m.t_io);
    m.t_step = m.t_compute + m.t_sync + m.t_io + m.t_comp_decomp;
    if (!cfg_.error_feedback) check(fc_reset_residuals(c));
    ++step_index_;
    return m;
  }

  using StepHook = std::function<void(SyncTrainer&, long step, long epoch, const NetParams&)>;
  void run(const StepHook& hook = {}) {
    while (step_index_ < total_steps()) {
      if (hook) hook(*this, step_index_, epoch_of(step_index_), net_at_step(step_index_));
      metrics_.push_back(step());
    }
  }

 private:
  SyncMode effective_mode() const {
    if (!cfg_.adaptive) return cfg_.mode;
    if (current_collective_ == Collective::AG) return SyncMode::AG;
    return cfg_.mode == SyncMode::VAR ? SyncMode::VAR : SyncMode::STAR;
  }
  double effective_c() const { return cfg_.adaptive ? current_c_ : cfg_.c; }
  void charge(Category cat, double s) { clock_.charge(probe_ ? Category::Exploration : cat, s); }

  std::shared_ptr<Context> ctx_;
  SyncConfig cfg_;
  NetworkSchedule sched_;
  GradSource src_;
  SimClock clock_;
  GainTracker tracker_;
  std::vector<StepMetrics> metrics_;
  long step_index_ = 0;
  double current_c_ = 1.0;
  Collective current_collective_ = Collective::AG;
  bool probe_ = false;
  unsigned long gen_ = 0;
};

// ---- the controller (inc/moo.hpp:148-271) -----------------------------------------------
struct ControllerEvent {
  long step = 0;
  std::string trigger;  // "gain" or "network"
  double chosen_c = 1.0;
  Collective collective = Collective::AG;
  std::size_t front_size = 0;
};

class Controller {
 public:
  explicit Controller(ControllerConfig cfg) : cfg_(cfg) { cfg_.validate(); }

  const std::vector<ControllerEvent>& events() const { return events_; }
  const std::vector<CandidateCR>& candidates() const { return candidates_; }
  const ControllerConfig& config() const { return cfg_; }

  void on_step(SyncTrainer& t, long step, long /*epoch*/, const NetParams& net) {
    if (!initialized_) {
      explore(t, net);
      refresh_sync(t, net);
      apply_selection(t, net);
      gain_ref_ = gain_of(t.current_c());
      prev_net_ = net;
      initialized_ = true;
      return;
    }
    if (trigger_gain(gain_ref_, t.gain_tracker(), cfg_.gain_threshold)) {
      explore(t, net);
      refresh_sync(t, net);
      gain_ref_ = gain_of(t.current_c());
      events_.push_back({step, "gain", t.current_c(), t.current_collective(), pareto_front(candidates_).size()});
    }
    if (network_changed(prev_net_, net, t.config().net_change_threshold)) {
      refresh_sync(t, net);
      const CrChoice chosen = apply_selection(t, net);
      gain_ref_ = chosen.candidate.gain_avg;
      events_.push_back({step, "network", chosen.candidate.c, chosen.collective, pareto_front(candidates_).size()});
    }
    prev_net_ = net;
  }

  SyncTrainer::StepHook hook() {
    return [this](SyncTrainer& t, long step, long epoch, const NetParams& net) { on_step(t, step, epoch, net); };
  }

  void explore(SyncTrainer& t, const NetParams& net) {
    const auto snap = t.snapshot();
    t.set_probe_mode(true);
    std::vector<CandidateCR> fresh;
    for (double c : candidate_ladder(cfg_)) {
      t.restore(snap);
      const Collective coll =
          t.n() >= 2 ? select_collective(net, MessageSpec(t.m_eff(), c, t.n())).collective : Collective::ART_RING;
      t.set_compression(c, coll);
      double gain_sum = 0.0, comp_sum = 0.0;
      bool ok = true;
      for (int i = 0; i < cfg_.probe_iters; ++i) {
        try {
          const StepMetrics m = t.step();
          gain_sum += m.gain;
          comp_sum += m.t_comp_decomp;
        } catch (const device_error&) {
          throw;  // not a property of the candidate
        } catch (const std::runtime_error&) {
          ok = false;  // divergent probe: candidate discarded
          break;
        }
      }
      if (ok) fresh.push_back({c, gain_sum / cfg_.probe_iters, comp_sum / cfg_.probe_iters, 0.0});
    }
    t.restore(snap);
    t.set_probe_mode(false);
    if (fresh.empty()) throw std::runtime_error("all exploration candidates diverged");
    candidates_ = std::move(fresh);
  }

  void refresh_sync(SyncTrainer& t, const NetParams& net) {
    for (auto& cand : candidates_) {
      const auto ch = select_collective(net, MessageSpec(t.m_eff(), cand.c, t.n()));
      switch (ch.collective) {
        case Collective::AG: cand.t_sync_modeled = ch.costs.ag_compressed; break;
        case Collective::ART_RING: cand.t_sync_modeled = ch.costs.art_ring; break;
        case Collective::ART_TREE: cand.t_sync_modeled = ch.costs.art_tree; break;
      }
    }
  }

 private:
  CrChoice apply_selection(SyncTrainer& t, const NetParams& net) {
    const auto chosen = choose_cr(pareto_front(candidates_), net, t.m_eff(), t.n());
    t.set_compression(chosen.candidate.c, chosen.collective);
    return chosen;
  }
  double gain_of(double c) const {
    for (const auto& cand : candidates_)
      if (cand.c == c) return cand.gain_avg;
    return -1.0;
  }

  ControllerConfig cfg_;
  std::vector<CandidateCR> candidates_;
  std::vector<ControllerEvent> events_;
  double gain_ref_ = -1.0;
  NetParams prev_net_;
  bool initialized_ = false;
};

}  // namespace b200
}  // namespace flexcomm
