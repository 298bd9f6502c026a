// flexcomm_b200/flexcomm.hpp — C++ façade with the reference's hot-path
// signatures over the B200 C-ABI (include/flexcomm_b200.h).
//
// A caller of the reference (/root/reference/proj/include/flexcomm) switches
// by including this header and using namespace flexcomm::b200 instead of
// flexcomm for the hot path:
//
//   reference                                  here
//   ----------------------------------------   -----------------------------
//   artopk_step   inc/artopk.hpp:62-111        b200::artopk_step (same args)
//   ag_step       inc/artopk.hpp:128-161       b200::ag_step
//   select_star   inc/artopk.hpp:27-30         b200::select_star
//   k_of          inc/compress.hpp:28-33       b200::k_of
//   topk_exact    inc/compress.hpp:57-65       b200::topk_exact
//   Cluster       inc/collectives.hpp:15-33    b200::Cluster (+ device context)
//   ResidualStore inc/core.hpp:84-95           b200::ResidualStore (lives in HBM)
//   select_collective / cost_* / crossover_cr  b200::select_collective / ...
//                 inc/costmodel.hpp:54-203
//
// Semantics kept: argument order and defaults, the SimClock wire charges the
// reference's Cluster makes (same byte counts, payload_scale on gradient
// payloads only, 4-byte floor, nothing charged at N=1), exceptions
// (std::invalid_argument / std::out_of_range / std::runtime_error).
// Differences (documented in INTEGRATION.md): values are fp32 on the device
// (inputs are converted; results widened back to double), and ResidualStore
// is device-resident (of() returns a host copy).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "flexcomm_b200.h"

namespace flexcomm {
namespace b200 {

// ---- status -> the reference's exception types ------------------------------
// CUDA / NCCL failures are runtime_errors too, but never a property of the data.
struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int s) {
  if (s == FC_OK) return;
  const std::string msg = std::string(fc_status_string(s)) + ": " + fc_last_error();
  switch (s) {
    case FC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FC_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case FC_ERR_CUDA:
    case FC_ERR_NCCL: throw device_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// ---- vocabulary (inc/artopk.hpp:13, inc/collectives.hpp:35-36, ...) ---------
enum class SelectionMode { STAR, VAR };
enum class ReduceOp { Sum, Avg };
enum class ReduceAlgo { Ring, Tree };
enum class CompressorKind { Exact, Layerwise, Threshold };
enum class Collective { AG, ART_RING, ART_TREE };
enum class Category { Compute, Sync, Compression, Io, Exploration };

struct CompressionRatio {
  double c = 1.0;
  CompressionRatio() = default;
  explicit CompressionRatio(double value) : c(value) {
    if (!(c > 0.0 && c <= 1.0)) throw std::invalid_argument("compression ratio must be in (0, 1]");
  }
};

inline std::size_t k_of(CompressionRatio c, std::size_t g) {
  uint64_t k = 0;
  check(fc_k_of(c.c, g, &k));
  return static_cast<std::size_t>(k);
}

inline int select_star(long step, int n) {
  int r = 0;
  check(fc_select_star(step, n, &r));
  return r;
}

struct LayerSpan {  // inc/core.hpp:11-15
  std::string name;
  std::size_t offset = 0;
  std::size_t length = 0;
};

struct DenseGrad {
  std::vector<double> values;
  std::vector<LayerSpan> layer_map;  // used by the Layerwise compressor
  std::size_t size() const { return values.size(); }
};

struct SparseGrad {
  std::vector<std::size_t> indices;
  std::vector<double> values;
  std::size_t total_len = 0;
  std::size_t nnz() const { return indices.size(); }
};

// ---- cost model (inc/costmodel.hpp) ----------------------------------------
struct NetParams {
  double alpha = 0.0;
  double bandwidth = 1e9;
  NetParams() = default;
  NetParams(double a, double bw) : alpha(a), bandwidth(bw) {
    if (alpha < 0.0) throw std::invalid_argument("alpha must be >= 0");
    if (!(bandwidth > 0.0)) throw std::invalid_argument("bandwidth must be > 0");
  }
  double beta() const { return 8.0 / bandwidth; }
};

struct MessageSpec {
  double m_bytes = 4.0;
  double c = 1.0;
  int n = 1;
  MessageSpec() = default;
  MessageSpec(double m, double cr, int workers) : m_bytes(m), c(cr), n(workers) {
    if (m_bytes < 4.0) throw std::invalid_argument("message must be >= 4 bytes");
    if (!(c > 0.0 && c <= 1.0)) throw std::invalid_argument("compression ratio out of (0,1]");
    if (n < 1) throw std::invalid_argument("worker count must be >= 1");
  }
};

struct CostBreakdown {
  double ps = 0, ring_ar = 0, tree_ar = 0, broadcast = 0, allgather_dense = 0, ag_compressed = 0,
         art_ring = 0, art_tree = 0;
};

inline CostBreakdown cost_primitives(const NetParams& net, const MessageSpec& msg) {
  double v[8];
  check(fc_cost_primitives(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n, v));
  return {v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
}
inline double cost_ring_ar(const NetParams& n, const MessageSpec& m) { return cost_primitives(n, m).ring_ar; }
inline double cost_tree_ar(const NetParams& n, const MessageSpec& m) { return cost_primitives(n, m).tree_ar; }
inline double cost_broadcast(const NetParams& n, const MessageSpec& m) { return cost_primitives(n, m).broadcast; }
inline double cost_allgather_dense(const NetParams& n, const MessageSpec& m) {
  return cost_primitives(n, m).allgather_dense;
}

struct CollectiveChoice {
  Collective collective = Collective::AG;
  CostBreakdown costs;
};

inline CollectiveChoice select_collective(const NetParams& net, const MessageSpec& msg) {
  int ch = 0;
  double v[8];
  check(fc_select_collective(net.alpha, net.bandwidth, msg.m_bytes, msg.c, msg.n, &ch, v));
  return {static_cast<Collective>(ch), {v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]}};
}

enum class CollectivePair { RING_VS_TREE, RING_VS_AG, TREE_VS_AG };
inline std::optional<double> crossover_cr(const NetParams& net, double m_bytes, int n,
                                          CollectivePair between) {
  double c = 0;
  int has = 0;
  check(fc_crossover_cr(net.alpha, net.bandwidth, m_bytes, n, static_cast<int>(between), &c, &has));
  if (!has) return std::nullopt;
  return c;
}

// ---- simulated clock (inc/netsched.hpp:60-90): the façade keeps the
// reference's analytic wire charges so its accounting tests still hold -------
struct SimClock {
  double acc[5] = {0, 0, 0, 0, 0};
  void charge(Category cat, double seconds) {
    if (seconds < 0.0) throw std::invalid_argument("negative duration");
    acc[static_cast<int>(cat)] += seconds;
  }
  double of(Category cat) const { return acc[static_cast<int>(cat)]; }
  double now() const { return acc[0] + acc[1] + acc[2] + acc[3] + acc[4]; }
};

struct SelectionLog {
  std::vector<std::pair<long, int>> entries;
  std::vector<long> counts;
  void record(long step, int rank, int n) {
    if (counts.empty()) counts.assign(static_cast<std::size_t>(n), 0);
    entries.emplace_back(step, rank);
    counts.at(static_cast<std::size_t>(rank))++;
  }
};

// ---- device context -------------------------------------------------------------
class Context {
 public:
  // loopback: n logical workers on one GPU (the reference's in-process Cluster)
  Context(int n, std::size_t grad_len, int device = 0, double max_cr = 1.0, unsigned flags = 0) {
    fc_opts o{};
    o.device = device;
    o.n_local = n;
    o.world = n;
    o.rank = 0;
    o.nccl_uid = nullptr;
    o.grad_len = grad_len;
    o.max_cr = max_cr;
    o.flags = flags;
    init(o);
  }
  // one worker per process: world ranks over NCCL (uid from fc_get_unique_id on rank 0)
  Context(int world, int rank, const unsigned char* nccl_uid, std::size_t grad_len, int device,
          double max_cr = 1.0, unsigned flags = 0) {
    fc_opts o{};
    o.device = device;
    o.n_local = 1;
    o.world = world;
    o.rank = rank;
    o.nccl_uid = nccl_uid;
    o.grad_len = grad_len;
    o.max_cr = max_cr;
    o.flags = flags;
    init(o);
  }
  ~Context() {
    if (ctx_) fc_destroy(ctx_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  fc_ctx* get() const { return ctx_; }
  std::size_t grad_len() const { return g_; }
  int n_local() const { return n_local_; }
  int world() const { return world_; }
  int rank() const { return rank_; }

  // fp64 <-> fp32 conversion by the library's host thread pool through
  // pinned staging chunks pipelined with the copy engine (fc_*_f64)
  void set_grad(int worker, const std::vector<double>& g) {
    if (g.size() != g_) throw std::invalid_argument("gradient length mismatch");
    check(fc_set_grad_f64(ctx_, worker, g.data()));
  }
  void set_residual(int worker, const std::vector<double>& r) {
    if (r.size() != g_) throw std::invalid_argument("residual length mismatch");
    check(fc_set_residual_f64(ctx_, worker, r.data()));
  }
  std::vector<double> residual(int worker) {
    std::vector<double> out(g_);
    check(fc_get_residual_f64(ctx_, worker, out.data()));
    return out;
  }
  std::vector<double> aggregate() {
    std::vector<double> out(g_);
    check(fc_get_aggregate_f64(ctx_, out.data()));
    return out;
  }
  // into an existing vector (no allocation when it already holds G values)
  void aggregate_into(std::vector<double>& out) {
    if (out.size() != g_) out.resize(g_);
    check(fc_get_aggregate_f64(ctx_, out.data()));
  }
  SparseGrad topk(int worker) {
    uint64_t k = 0;
    check(fc_get_topk(ctx_, worker, nullptr, nullptr, &k));
    std::vector<uint32_t> idx(k);
    std::vector<float> val(k);
    check(fc_get_topk(ctx_, worker, idx.data(), val.data(), &k));
    SparseGrad s;
    s.total_len = g_;
    s.indices.assign(idx.begin(), idx.end());
    s.values.assign(val.begin(), val.end());
    return s;
  }
  fc_worker_stats worker_stats(int worker) {
    fc_worker_stats w{};
    check(fc_get_worker_stats(ctx_, worker, &w));
    return w;
  }
  void snapshot() { check(fc_snapshot(ctx_)); }
  void restore() { check(fc_restore(ctx_)); }

 private:
  void init(const fc_opts& o) {
    check(fc_create(&ctx_, &o));
    g_ = o.grad_len;
    int nl = 0, w = 0, r = 0;
    check(fc_num_workers(ctx_, &nl, &w, &r));
    n_local_ = nl;
    world_ = w;
    rank_ = r;
  }
  fc_ctx* ctx_ = nullptr;
  std::size_t g_ = 0;
  int n_local_ = 1, world_ = 1, rank_ = 0;
};

// The reference's Cluster (inc/collectives.hpp:15-33) plus the device context
// that holds the workers' state.
struct Cluster {
  int n = 1;
  NetParams net;
  SimClock* clock = nullptr;
  Category charge_category = Category::Sync;
  std::shared_ptr<Context> ctx;

  Cluster(int workers, NetParams net_params, SimClock* clk, std::shared_ptr<Context> context)
      : n(workers), net(net_params), clock(clk), ctx(std::move(context)) {
    if (n < 1) throw std::invalid_argument("worker count must be >= 1");
    if (!ctx || ctx->world() != n) throw std::invalid_argument("context worker count != cluster size");
  }
  void charge(double seconds) const {
    if (clock) clock->charge(charge_category, seconds);
  }
  MessageSpec msg(double payload_bytes) const {
    return MessageSpec(payload_bytes > 4.0 ? payload_bytes : 4.0, 1.0, n);
  }
};

// Device-resident residual store (inc/core.hpp:84-95); of() returns a copy.
class ResidualStore {
 public:
  explicit ResidualStore(std::shared_ptr<Context> ctx) : ctx_(std::move(ctx)) {}
  std::vector<double> of(int worker) const {
    if (worker < 0 || worker >= ctx_->n_local()) throw std::out_of_range("worker index out of range");
    return ctx_->residual(worker);
  }
  void set(int worker, const std::vector<double>& r) { ctx_->set_residual(worker, r); }
  void reset() { check(fc_reset_residuals(ctx_->get())); }

 private:
  std::shared_ptr<Context> ctx_;
};

struct ArtopkResult {
  DenseGrad aggregate;
  int selected_rank = 0;
};

namespace detail {
inline void upload(const Cluster& cluster, const std::vector<DenseGrad>& g_o) {
  Context& c = *cluster.ctx;
  if (g_o.size() != static_cast<std::size_t>(c.n_local()))
    throw std::invalid_argument("gradient count != worker count");
  for (int r = 0; r < c.n_local(); ++r) {
    if (g_o[static_cast<std::size_t>(r)].size() != c.grad_len())
      throw std::invalid_argument("gradient length mismatch");
    c.set_grad(r, g_o[static_cast<std::size_t>(r)].values);
  }
}
}  // namespace detail

// inc/artopk.hpp:62-111.  g_o holds this context's workers (all N in
// loopback, the local worker under NCCL).
inline ArtopkResult artopk_step(const Cluster& cluster, const std::vector<DenseGrad>& g_o,
                                ResidualStore& /*residuals: device-resident in cluster.ctx*/,
                                CompressionRatio c, SelectionMode mode, ReduceAlgo algo, long step,
                                SelectionLog* log = nullptr, ReduceOp op = ReduceOp::Avg,
                                double payload_scale = 1.0) {
  detail::upload(cluster, g_o);
  fc_step_stats st{};
  check(fc_artopk_step(cluster.ctx->get(), c.c, mode == SelectionMode::STAR ? FC_STAR : FC_VAR,
                       algo == ReduceAlgo::Ring ? FC_RING : FC_TREE, step,
                       op == ReduceOp::Sum ? FC_SUM : FC_AVG, &st));
  if (log) log->record(step, st.selected_rank, cluster.n);
  if (cluster.n > 1) {  // the reference's analytic wire charges (collectives.hpp:52-92)
    if (mode == SelectionMode::VAR) cluster.charge(cost_allgather_dense(cluster.net, cluster.msg(4.0 * cluster.n)));
    const double wire = 4.0 * static_cast<double>(st.k) * payload_scale;
    cluster.charge(cost_broadcast(cluster.net, cluster.msg(wire)));
    cluster.charge(algo == ReduceAlgo::Ring ? cost_ring_ar(cluster.net, cluster.msg(wire))
                                            : cost_tree_ar(cluster.net, cluster.msg(wire)));
  }
  ArtopkResult out;
  out.aggregate.values = cluster.ctx->aggregate();
  out.selected_rank = st.selected_rank;
  return out;
}

// artopk_step writing into a caller-owned result: the same step, but the
// aggregate reuses out.aggregate's storage instead of returning a fresh
// 8G-byte vector by value (on a host where first-touching 1.1 GB costs
// hundreds of milliseconds, that allocation dominates the call; see
// tests/cpp/bench_facade.cpp).  Not in the reference's API -- an addition.
inline void artopk_step_into(ArtopkResult& out, const Cluster& cluster, const std::vector<DenseGrad>& g_o,
                             ResidualStore& /*device-resident*/, CompressionRatio c, SelectionMode mode,
                             ReduceAlgo algo, long step, SelectionLog* log = nullptr, ReduceOp op = ReduceOp::Avg,
                             double payload_scale = 1.0) {
  detail::upload(cluster, g_o);
  fc_step_stats st{};
  check(fc_artopk_step(cluster.ctx->get(), c.c, mode == SelectionMode::STAR ? FC_STAR : FC_VAR,
                       algo == ReduceAlgo::Ring ? FC_RING : FC_TREE, step,
                       op == ReduceOp::Sum ? FC_SUM : FC_AVG, &st));
  if (log) log->record(step, st.selected_rank, cluster.n);
  if (cluster.n > 1) {
    if (mode == SelectionMode::VAR) cluster.charge(cost_allgather_dense(cluster.net, cluster.msg(4.0 * cluster.n)));
    const double wire = 4.0 * static_cast<double>(st.k) * payload_scale;
    cluster.charge(cost_broadcast(cluster.net, cluster.msg(wire)));
    cluster.charge(algo == ReduceAlgo::Ring ? cost_ring_ar(cluster.net, cluster.msg(wire))
                                            : cost_tree_ar(cluster.net, cluster.msg(wire)));
  }
  cluster.ctx->aggregate_into(out.aggregate.values);
  out.selected_rank = st.selected_rank;
}

// inc/artopk.hpp:128-161, every compressor on the device (Layerwise uses
// g_o's layer map, like error_feedback's copy of it in the reference).
inline DenseGrad ag_step(const Cluster& cluster, const std::vector<DenseGrad>& g_o,
                         ResidualStore& /*device-resident*/, CompressionRatio c,
                         CompressorKind compressor = CompressorKind::Exact,
                         double payload_scale = 1.0, int threshold_rounds = 25) {
  detail::upload(cluster, g_o);
  if (compressor == CompressorKind::Layerwise) {
    std::vector<uint64_t> off, len;
    for (const auto& l : g_o.front().layer_map) {
      off.push_back(l.offset);
      len.push_back(l.length);
    }
    check(fc_set_layer_map(cluster.ctx->get(), off.data(), len.data(), static_cast<int>(off.size())));
  }
  if (compressor == CompressorKind::Threshold) check(fc_set_threshold_rounds(cluster.ctx->get(), threshold_rounds));
  const int kind = compressor == CompressorKind::Exact ? FC_EXACT
                   : compressor == CompressorKind::Layerwise ? FC_LAYERWISE
                                                             : FC_THRESHOLD;
  fc_step_stats st{};
  check(fc_ag_step(cluster.ctx->get(), c.c, kind, &st));
  if (cluster.n > 1)
    cluster.charge(cost_allgather_dense(
        cluster.net, cluster.msg(2.0 * 4.0 * static_cast<double>(st.k) * payload_scale)));
  DenseGrad agg;
  agg.values = cluster.ctx->aggregate();
  return agg;
}

// inc/compress.hpp:57-65 on the device (one-worker context, cached per G).
inline SparseGrad topk_exact(const DenseGrad& g, CompressionRatio c) {
  if (g.size() == 0) throw std::invalid_argument("empty gradient (G == 0)");
  thread_local std::unique_ptr<Context> ctx;
  if (!ctx || ctx->grad_len() != g.size()) ctx.reset(new Context(1, g.size()));
  ctx->set_grad(0, g.values);
  check(fc_topk_exact(ctx->get(), 0, c.c, nullptr));
  return ctx->topk(0);
}

}  // namespace b200
}  // namespace flexcomm
