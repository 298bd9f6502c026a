// Reference-style tests of the C++ façade (include/flexcomm_b200/flexcomm.hpp)
// on a B200.  Each test restates a reference test (file:line under
// /root/reference/proj/tests) against flexcomm::b200; where the reference
// computes its expectation in fp64, the restatement computes it with the fp32
// arithmetic the device uses (inputs are fp32-representable), and says so.
#include <algorithm>
#include <numeric>
#include <random>
#include <set>

#include "flexcomm_b200/flexcomm.hpp"
#include "flexcomm_b200/moo.hpp"
#include "mini_test.hpp"

using namespace flexcomm::b200;

namespace {

std::shared_ptr<Context> make_ctx(int n, std::size_t g) { return std::make_shared<Context>(n, g); }

Cluster make_cluster(int n, SimClock* clk, std::shared_ptr<Context> ctx) {
  return Cluster(n, NetParams(0.001, 1e9), clk, std::move(ctx));
}

std::vector<DenseGrad> random_grads(std::mt19937_64& rng, int n, std::size_t g) {
  std::normal_distribution<float> dist(0.0f, 1.0f);  // fp32-representable inputs
  std::vector<DenseGrad> out(static_cast<std::size_t>(n));
  for (auto& grad : out) {
    grad.values.resize(g);
    for (double& v : grad.values) v = dist(rng);
  }
  return out;
}

}  // namespace

// tests/test_artopk.cpp:28-53
TEST(Artopk, HandExecutedTwoWorkerStep) {
  SimClock clk;
  auto ctx = make_ctx(2, 3);
  auto cluster = make_cluster(2, &clk, ctx);
  std::vector<DenseGrad> g_o(2);
  g_o[0].values = {2.0, 0.0, 1.0};
  g_o[1].values = {3.0, 4.0, 2.0};
  ResidualStore residuals(ctx);
  auto res = artopk_step(cluster, g_o, residuals, CompressionRatio(1.0 / 3.0), SelectionMode::STAR,
                         ReduceAlgo::Ring, 0);
  EXPECT_EQ(res.selected_rank, 0);
  EXPECT_TRUE(res.aggregate.values == (std::vector<double>{2.5, 0.0, 0.0}));
  EXPECT_TRUE(residuals.of(0) == (std::vector<double>{0.0, 0.0, 1.0}));
  EXPECT_TRUE(residuals.of(1) == (std::vector<double>{0.0, 4.0, 2.0}));
  auto res2 = artopk_step(cluster, g_o, residuals, CompressionRatio(1.0 / 3.0),
                          SelectionMode::STAR, ReduceAlgo::Ring, 1);
  EXPECT_EQ(res2.selected_rank, 1);
  EXPECT_TRUE(res2.aggregate.values == (std::vector<double>{0.0, 4.0, 0.0}));
  EXPECT_TRUE(residuals.of(0) == (std::vector<double>{2.0, 0.0, 2.0}));
  EXPECT_TRUE(residuals.of(1) == (std::vector<double>{3.0, 0.0, 4.0}));
}

// tests/test_artopk.cpp:55-104 (expectations in the device's fp32 arithmetic)
TEST(Artopk, BruteForceAgainstDefinition) {
  std::mt19937_64 rng(17);
  std::uniform_int_distribution<int> nw(1, 4);
  std::uniform_int_distribution<std::size_t> glen(1, 16);
  std::uniform_real_distribution<double> crs(0.05, 1.0);
  for (int trial = 0; trial < 100; ++trial) {
    const int n = nw(rng);
    const std::size_t g = glen(rng);
    auto g_o = random_grads(rng, n, g);
    auto ctx = make_ctx(n, g);
    ResidualStore residuals(ctx);
    SimClock clk;
    auto cluster = make_cluster(n, &clk, ctx);
    for (long step = 0; step < 3; ++step) {
      CompressionRatio c(crs(rng));
      std::vector<std::vector<float>> g_e(static_cast<std::size_t>(n), std::vector<float>(g));
      for (int r = 0; r < n; ++r) {
        auto rr = residuals.of(r);
        for (std::size_t i = 0; i < g; ++i)
          g_e[r][i] = static_cast<float>(g_o[r].values[i]) + static_cast<float>(rr[i]);
      }
      auto res = artopk_step(cluster, g_o, residuals, c, SelectionMode::STAR, ReduceAlgo::Ring, step);
      ASSERT_EQ(res.selected_rank, static_cast<int>(step % n));
      for (std::size_t i = 0; i < g; ++i) {
        if (res.aggregate.values[i] == 0.0) continue;
        float expect = g_e[0][i];
        for (int r = 1; r < n; ++r) expect += g_e[r][i];
        expect /= static_cast<float>(n);
        ASSERT_EQ(res.aggregate.values[i], static_cast<double>(expect));
      }
      for (int r = 0; r < n; ++r) {
        auto rr = residuals.of(r);
        for (std::size_t i = 0; i < g; ++i) {
          const float kept = g_e[r][i] - static_cast<float>(rr[i]);
          if (rr[i] != 0.0) ASSERT_EQ(kept, 0.0f);
          ASSERT_EQ(kept + static_cast<float>(rr[i]), g_e[r][i]);
        }
      }
    }
  }
}

// tests/test_artopk.cpp:106-113
TEST(SelectStar, RoundRobinIsUniform) {
  const int n = 4;
  const long m = 25;
  SelectionLog log;
  for (long step = 0; step < m * n; ++step) log.record(step, select_star(step, n), n);
  for (long count : log.counts) EXPECT_EQ(count, m);
  EXPECT_THROW(select_star(0, 0), std::invalid_argument);
}

// tests/test_artopk.cpp:115-130, through the VAR mode of artopk_step
TEST(SelectVar, ArgmaxOfCompressedNormWithLowRankTies) {
  SimClock clk;
  auto ctx = make_ctx(3, 4);
  auto cluster = make_cluster(3, &clk, ctx);
  ResidualStore residuals(ctx);
  std::vector<DenseGrad> g_o(3);
  g_o[0].values = {2.0, 0.0, 0.0, 0.0};
  g_o[1].values = {0.0, -3.0, 0.0, 0.0};
  g_o[2].values = {0.0, 0.0, 3.0, 0.0};  // ties with rank 1 at norm 9
  auto res = artopk_step(cluster, g_o, residuals, CompressionRatio(0.25), SelectionMode::VAR,
                         ReduceAlgo::Ring, 0);
  EXPECT_EQ(res.selected_rank, 1);
  const double wire = 4.0;
  EXPECT_DOUBLE_EQ(clk.of(Category::Sync),
                   cost_allgather_dense(cluster.net, cluster.msg(4.0 * 3)) +
                       cost_broadcast(cluster.net, cluster.msg(wire)) +
                       cost_ring_ar(cluster.net, cluster.msg(wire)));
}

// tests/test_artopk.cpp:159-185
TEST(Artopk, WireAccounting) {
  std::mt19937_64 rng(41);
  const int n = 4;
  const std::size_t g = 40;
  auto g_o = random_grads(rng, n, g);
  SimClock clk;
  auto ctx = make_ctx(n, g);
  auto cluster = make_cluster(n, &clk, ctx);
  ResidualStore residuals(ctx);
  CompressionRatio c(0.25);  // k = 10
  artopk_step(cluster, g_o, residuals, c, SelectionMode::STAR, ReduceAlgo::Ring, 0);
  const double wire = 4.0 * 10;
  EXPECT_DOUBLE_EQ(clk.of(Category::Sync), cost_broadcast(cluster.net, cluster.msg(wire)) +
                                               cost_ring_ar(cluster.net, cluster.msg(wire)));
  SimClock clk2;
  auto ctx2 = make_ctx(n, g);
  auto cluster2 = make_cluster(n, &clk2, ctx2);
  ResidualStore residuals2(ctx2);
  artopk_step(cluster2, g_o, residuals2, c, SelectionMode::VAR, ReduceAlgo::Tree, 0, nullptr,
              ReduceOp::Avg, 100.0);
  const double scaled = wire * 100.0;
  EXPECT_DOUBLE_EQ(clk2.of(Category::Sync),
                   cost_allgather_dense(cluster2.net, cluster2.msg(4.0 * n)) +
                       cost_broadcast(cluster2.net, cluster2.msg(scaled)) +
                       cost_tree_ar(cluster2.net, cluster2.msg(scaled)));
}

// tests/test_artopk.cpp:187-202 (0.1 / 0.2 restated as their fp32 values)
TEST(AgStep, AveragesContributionsByWorkerCount) {
  SimClock clk;
  auto ctx = make_ctx(2, 3);
  auto cluster = make_cluster(2, &clk, ctx);
  ResidualStore residuals(ctx);
  std::vector<DenseGrad> g_o(2);
  g_o[0].values = {4.0, 0.1, 0.0};
  g_o[1].values = {0.2, 6.0, 0.0};
  auto agg = ag_step(cluster, g_o, residuals, CompressionRatio(1.0 / 3.0));
  EXPECT_TRUE(agg.values == (std::vector<double>{2.0, 3.0, 0.0}));
  EXPECT_TRUE(residuals.of(0) == (std::vector<double>{0.0, (double)0.1f, 0.0}));
  EXPECT_TRUE(residuals.of(1) == (std::vector<double>{(double)0.2f, 0.0, 0.0}));
  EXPECT_DOUBLE_EQ(clk.of(Category::Sync), cost_allgather_dense(cluster.net, cluster.msg(2.0 * 4.0 * 1)));
}

// tests/test_artopk.cpp:204-225 (Exact compressor; identity in fp32)
TEST(AgStep, ErrorFeedbackIdentityAcrossSteps) {
  std::mt19937_64 rng(53);
  const int n = 3;
  const std::size_t g = 32;
  auto ctx = make_ctx(n, g);
  ResidualStore residuals(ctx);
  SimClock clk;
  auto cluster = make_cluster(n, &clk, ctx);
  for (int step = 0; step < 20; ++step) {
    auto g_o = random_grads(rng, n, g);
    std::vector<std::vector<float>> g_e(n, std::vector<float>(g));
    for (int r = 0; r < n; ++r) {
      auto rr = residuals.of(r);
      for (std::size_t i = 0; i < g; ++i) g_e[r][i] = (float)g_o[r].values[i] + (float)rr[i];
    }
    ag_step(cluster, g_o, residuals, CompressionRatio(0.25));
    for (int r = 0; r < n; ++r) {
      auto rr = residuals.of(r);
      for (std::size_t i = 0; i < g; ++i) {
        const float kept = g_e[r][i] - (float)rr[i];
        ASSERT_EQ(kept + (float)rr[i], g_e[r][i]);
      }
    }
  }
}

// tests/test_compress.cpp:38-48
TEST(KOf, ExactValues) {
  EXPECT_EQ(k_of(CompressionRatio(1.0), 17), 17u);
  EXPECT_EQ(k_of(CompressionRatio(0.5), 10), 5u);
  EXPECT_EQ(k_of(CompressionRatio(0.1), 10), 1u);
  EXPECT_EQ(k_of(CompressionRatio(0.01), 10), 1u);
  EXPECT_EQ(k_of(CompressionRatio(0.3), 10), 3u);
  EXPECT_EQ(k_of(CompressionRatio(0.31), 10), 4u);
  EXPECT_THROW(k_of(CompressionRatio(0.5), 0), std::invalid_argument);
  EXPECT_THROW(CompressionRatio(0.0), std::invalid_argument);
  EXPECT_THROW(CompressionRatio(1.5), std::invalid_argument);
}

// tests/test_compress.cpp:50-64
TEST(TopkExact, MatchesFullSortOracle) {
  std::mt19937_64 rng(7);
  std::uniform_int_distribution<std::size_t> glen(1, 2000);
  std::uniform_real_distribution<double> crs(0.001, 1.0);
  std::normal_distribution<float> dist(0.0f, 1.0f);
  for (int trial = 0; trial < 100; ++trial) {
    DenseGrad g;
    g.values.resize(glen(rng));
    for (double& v : g.values) v = dist(rng);
    CompressionRatio c(crs(rng));
    auto s = topk_exact(g, c);
    const std::size_t k = k_of(c, g.size());
    ASSERT_EQ(s.nnz(), k);
    std::vector<std::size_t> idx(g.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
      double ma = std::fabs(g.values[a]), mb = std::fabs(g.values[b]);
      if (ma != mb) return ma > mb;
      return a < b;
    });
    idx.resize(k);
    std::sort(idx.begin(), idx.end());
    EXPECT_TRUE(s.indices == idx);
    for (std::size_t i = 0; i < k; ++i) EXPECT_EQ(s.values[i], g.values[s.indices[i]]);
  }
}

// tests/test_compress.cpp:66-71
TEST(TopkExact, TieBreaksToLowerIndex) {
  DenseGrad g;
  g.values = {1.0, -1.0, 1.0, -2.0, 1.0};
  auto s = topk_exact(g, CompressionRatio(0.6));
  EXPECT_TRUE(s.indices == (std::vector<std::size_t>{0, 1, 3}));
}

// tests/test_costmodel.cpp:10-44
TEST(CostModel, HandComputedCells) {
  NetParams net(0.010, 10e9);
  EXPECT_DOUBLE_EQ(net.beta(), 8.0 / 10e9);
  EXPECT_THROW(NetParams(-1.0, 1e9), std::invalid_argument);
  MessageSpec msg(4e8, 1.0, 8);
  EXPECT_NEAR(cost_ring_ar(net, msg), 0.70, 1e-12);
  EXPECT_NEAR(cost_tree_ar(net, msg), 1.98, 1e-12);
  EXPECT_NEAR(cost_primitives(net, msg).ps, 4.50, 1e-12);
  EXPECT_NEAR(cost_broadcast(net, msg), 0.01 * 3 + 3 * 4e8 * 8e-10, 1e-12);
  EXPECT_NEAR(cost_allgather_dense(net, msg), 0.01 * 3 + 7 * 4e8 * 8e-10, 1e-12);
  NetParams n2(0.001, 1e9);
  MessageSpec m2(4e7, 0.01, 8);
  const double mc = 4e7 * 0.01, beta = 8.0 / 1e9;
  auto b = cost_primitives(n2, m2);
  EXPECT_NEAR(b.ag_compressed, 0.001 * 3 + 2 * mc * beta * 7, 1e-12);
  EXPECT_NEAR(b.art_ring, 0.001 * (14 + 3) + mc * beta * (14.0 / 8 + 3), 1e-12);
  EXPECT_NEAR(b.art_tree, 3 * 0.001 * 3 + 3 * mc * beta * 3, 1e-12);
  EXPECT_THROW(select_collective(n2, MessageSpec(4e7, 0.01, 1)), std::invalid_argument);
}

// Trainer::snapshot/restore (inc/trainer.hpp:160-190) as used by the MOO
// explore (inc/moo.hpp:205, 232): the device residuals replay exactly.
TEST(Snapshot, RestoreReplaysExactly) {
  std::mt19937_64 rng(3);
  const int n = 2;
  const std::size_t g = 5000;
  auto ctx = make_ctx(n, g);
  ResidualStore residuals(ctx);
  SimClock clk;
  auto cluster = make_cluster(n, &clk, ctx);
  auto g_o = random_grads(rng, n, g);
  artopk_step(cluster, g_o, residuals, CompressionRatio(0.01), SelectionMode::STAR, ReduceAlgo::Ring, 0);
  ctx->snapshot();
  std::vector<std::vector<double>> outs;
  for (long s = 1; s < 4; ++s)
    outs.push_back(artopk_step(cluster, g_o, residuals, CompressionRatio(0.01), SelectionMode::VAR,
                               ReduceAlgo::Tree, s)
                       .aggregate.values);
  ctx->restore();
  for (long s = 1; s < 4; ++s)
    EXPECT_TRUE(artopk_step(cluster, g_o, residuals, CompressionRatio(0.01), SelectionMode::VAR,
                            ReduceAlgo::Tree, s)
                    .aggregate.values == outs[s - 1]);
}

TEST(Errors, MapToReferenceExceptions) {
  auto ctx = make_ctx(2, 100);
  SimClock clk;
  auto cluster = make_cluster(2, &clk, ctx);
  ResidualStore residuals(ctx);
  std::vector<DenseGrad> one(1);
  one[0].values.assign(100, 1.0);
  EXPECT_THROW(artopk_step(cluster, one, residuals, CompressionRatio(0.1), SelectionMode::STAR,
                           ReduceAlgo::Ring, 0),
               std::invalid_argument);
  EXPECT_THROW(residuals.of(2), std::out_of_range);
  EXPECT_THROW(Cluster(0, NetParams(0.001, 1e9), &clk, ctx), std::invalid_argument);
}

// tests/test_moo.cpp:29-46
TEST(Ladder, DefaultRungsAndFactorTen) {
  ControllerConfig cfg;
  EXPECT_TRUE(candidate_ladder(cfg) == (std::vector<double>{0.1, 0.0333, 0.0111, 0.0037, 0.001}));
  cfg.factor = 10.0;
  EXPECT_TRUE(candidate_ladder(cfg) == (std::vector<double>{0.1, 0.01, 0.001}));
  cfg.c_low = cfg.c_high = 0.05;
  EXPECT_TRUE(candidate_ladder(cfg) == (std::vector<double>{0.05}));
  cfg.c_low = 0.2;
  EXPECT_THROW(candidate_ladder(cfg), std::invalid_argument);
  EXPECT_DOUBLE_EQ(round_3sig(123456.0), 123000.0);
}

// tests/test_moo.cpp:97-113
TEST(Knee, PicksBalancedCandidateAndTiesGoToLargerRatio) {
  auto cand = [](double c, double tc, double ts, double inv_gain) {
    return CandidateCR{c, 1.0 / inv_gain, tc, ts};
  };
  std::vector<CandidateCR> front = {cand(0.1, 1.0, 9.0, 9.0), cand(0.01, 5.0, 5.0, 5.0),
                                    cand(0.001, 9.0, 9.0, 1.0)};
  auto ch = choose_cr(front, NetParams(0.001, 10e9), 4e7, 8);
  EXPECT_EQ(ch.candidate.c, 0.01);
  EXPECT_TRUE(ch.collective == select_collective(NetParams(0.001, 10e9), MessageSpec(4e7, 0.01, 8)).collective);
  std::vector<CandidateCR> tie = {cand(0.01, 1.0, 2.0, 2.0), cand(0.1, 2.0, 1.0, 2.0)};
  EXPECT_EQ(choose_cr(tie, NetParams(0.001, 10e9), 4e7, 8).candidate.c, 0.1);
  EXPECT_THROW(choose_cr({}, NetParams(0.001, 10e9), 4e7, 8), std::invalid_argument);
}

// tests/test_moo.cpp:115-135 on device residuals
TEST(Controller, ExploreRestoresTrajectory) {
  auto ctx = make_ctx(2, 50000);
  NetworkSchedule sched;
  sched.segments = {{0, NetParams(0.001, 10e9)}};
  SyncConfig cfg;
  cfg.adaptive = true;
  cfg.c = 0.01;
  SyncTrainer trainer(ctx, cfg, sched);
  trainer.step();
  const auto r0 = ctx->residual(0), r1 = ctx->residual(1);
  const long step_before = trainer.step_index();
  ControllerConfig cc;
  cc.probe_iters = 3;
  Controller controller(cc);
  controller.explore(trainer, sched.segments[0].net);
  EXPECT_TRUE(ctx->residual(0) == r0);
  EXPECT_TRUE(ctx->residual(1) == r1);
  EXPECT_EQ(trainer.step_index(), step_before);
  EXPECT_TRUE(!trainer.probe_mode());
  EXPECT_TRUE(trainer.clock().of(Category::Exploration) > 0.0);
  EXPECT_EQ(controller.candidates().size(), candidate_ladder(controller.config()).size());
  for (const auto& c : controller.candidates()) {
    EXPECT_TRUE(c.gain_avg > 0.0 && c.gain_avg <= 1.0);
    EXPECT_TRUE(c.t_comp_avg > 0.0);
  }
}

// tests/test_moo.cpp:137-169
TEST(Controller, HookSelectsOnFirstStepAndOnNetworkChange) {
  auto ctx = make_ctx(2, 40000);
  NetworkSchedule sched;
  sched.segments = {{0, NetParams(0.001, 25e9)}, {1, NetParams(0.001, 1e9)}};
  SyncConfig cfg;
  cfg.adaptive = true;
  cfg.size_bytes_override = 4e7;
  cfg.epochs = 2;
  cfg.steps_per_epoch = 4;
  SyncTrainer trainer(ctx, cfg, sched);
  Controller controller{ControllerConfig()};
  trainer.run(controller.hook());
  std::vector<ControllerEvent> net_events;
  for (const auto& e : controller.events())
    if (e.trigger == "network") net_events.push_back(e);
  ASSERT_EQ(net_events.size(), 1u);
  EXPECT_EQ(net_events[0].step, cfg.steps_per_epoch);
  EXPECT_TRUE(net_events[0].chosen_c >= 0.001 && net_events[0].chosen_c <= 0.1);
  EXPECT_TRUE(net_events[0].front_size >= 1u);
  EXPECT_EQ(trainer.metrics().size(), 8u);
}

// tests/test_compress.cpp:73-78 through ag_step at N=1 (the aggregate is the selection)
TEST(TopkLayerwise, AppliesRatioPerLayer) {
  auto ctx = make_ctx(1, 8);
  SimClock clk;
  auto cluster = make_cluster(1, &clk, ctx);
  ResidualStore residuals(ctx);
  std::vector<DenseGrad> g(1);
  g[0].values = {5.0, 0.1, 0.2, 0.3, 0.01, 9.0, 0.02, 0.03};
  g[0].layer_map = {{"L0", 0, 4}, {"L1", 4, 4}};
  auto agg = ag_step(cluster, g, residuals, CompressionRatio(0.25), CompressorKind::Layerwise);
  EXPECT_TRUE(agg.values == (std::vector<double>{5.0, 0, 0, 0, 0, 9.0, 0, 0}));
}

// tests/test_compress.cpp:93-98 through ag_step at N=1
TEST(TopkThreshold, FullRatioKeepsEverything) {
  std::mt19937_64 rng(3);
  auto ctx = make_ctx(1, 97);
  SimClock clk;
  auto cluster = make_cluster(1, &clk, ctx);
  ResidualStore residuals(ctx);
  auto g = random_grads(rng, 1, 97);
  auto agg = ag_step(cluster, g, residuals, CompressionRatio(1.0), CompressorKind::Threshold, 1.0, 25);
  EXPECT_TRUE(agg.values == g[0].values);
  EXPECT_THROW(ag_step(cluster, g, residuals, CompressionRatio(1.0), CompressorKind::Threshold, 1.0, 0),
               std::invalid_argument);
}

int main() { return mt::run_all(); }
