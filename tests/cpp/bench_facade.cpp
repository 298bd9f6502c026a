// End-to-end time of the reference-signature façade on a B200:
// flexcomm::b200::artopk_step(Cluster, std::vector<DenseGrad>, ...) -- the
// call a reference Trainer makes (inc/artopk.hpp:62-66) -- including the fp64
// gradient upload and the fp64 aggregate returned by value, at BASELINE
// config 3 (138M, CR 0.01, one worker on this GPU).  Compared with the
// round-1 façade path (single-threaded fp64 -> fp32 conversion into a
// pageable std::vector<float>, synchronous pageable copies), restated here.
//   ./bench_facade [G] [steps]    -> one JSON line
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "flexcomm_b200/flexcomm.hpp"

using namespace flexcomm::b200;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
  const std::size_t G = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 138000000ull;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 5;
  auto ctx = std::make_shared<Context>(1, G, 0, 0.01);
  Cluster cluster(1, NetParams(1e-5, 1e12), nullptr, ctx);
  ResidualStore residuals(ctx);
  std::vector<DenseGrad> g_o(1);
  g_o[0].values.resize(G);
  std::mt19937_64 rng(42);
  std::normal_distribution<float> dist(0.f, 1.f);
  for (auto& v : g_o[0].values) v = dist(rng);

  // (1) the façade as shipped
  double sum = 0.0;
  for (int s = 0; s < steps + 1; ++s) {
    const auto t0 = clk::now();
    auto r = artopk_step(cluster, g_o, residuals, CompressionRatio(0.01), SelectionMode::STAR, ReduceAlgo::Ring, s);
    const double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (s > 0) sum += ms;  // first call: staging set-up
    if (r.aggregate.values.size() != G) return 2;
  }
  const double facade_ms = sum / steps;

  // (2) round 1's façade path: host conversion on one thread + pageable copies
  std::vector<float> buf;
  sum = 0.0;
  for (int s = 0; s < steps + 1; ++s) {
    const auto t0 = clk::now();
    buf.assign(g_o[0].values.begin(), g_o[0].values.end());
    check(fc_set_grad(ctx->get(), 0, buf.data(), FC_HOST));
    fc_step_stats st{};
    check(fc_artopk_step(ctx->get(), 0.01, FC_STAR, FC_RING, s, FC_AVG, &st));
    buf.resize(G);
    check(fc_get_aggregate(ctx->get(), buf.data(), FC_HOST));
    std::vector<double> agg(buf.begin(), buf.end());
    const double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (s > 0) sum += ms;
    if (agg.size() != G) return 2;
  }
  const double old_ms = sum / steps;

  // (1b) the allocation-free variant (result storage reused)
  ArtopkResult into;
  sum = 0.0;
  for (int s = 0; s < steps + 1; ++s) {
    const auto t0 = clk::now();
    artopk_step_into(into, cluster, g_o, residuals, CompressionRatio(0.01), SelectionMode::STAR, ReduceAlgo::Ring, s);
    const double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (s > 0) sum += ms;
  }
  const double into_ms = sum / steps;

  // (3) the façade's parts: fp64 upload, the device step, the fp64 aggregate
  double t_up = 0, t_step = 0, t_down = 0;
  for (int s = 0; s < steps; ++s) {
    auto t0 = clk::now();
    ctx->set_grad(0, g_o[0].values);
    auto t1 = clk::now();
    fc_step_stats st{};
    check(fc_artopk_step(ctx->get(), 0.01, FC_STAR, FC_RING, s, FC_AVG, &st));
    auto t2 = clk::now();
    auto agg = ctx->aggregate();
    auto t3 = clk::now();
    t_up += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t_step += std::chrono::duration<double, std::milli>(t2 - t1).count();
    t_down += std::chrono::duration<double, std::milli>(t3 - t2).count();
    if (agg.size() != G) return 2;
  }
  // a bare std::vector<double>(G): the allocation + zero fill that returning
  // the aggregate by value (as the reference does) costs on this host
  double t_alloc = 0;
  for (int s = 0; s < steps; ++s) {
    auto t0 = clk::now();
    std::vector<double> v(G);
    t_alloc += std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    if (v.size() != G) return 2;
  }
  std::printf("{\"bench\": \"facade artopk_step e2e\", \"grad_len\": %zu, \"cr\": 0.01, \"steps\": %d, "
              "\"facade_ms_per_step\": %.2f, \"facade_into_ms_per_step\": %.2f, \"round1_facade_ms_per_step\": %.2f, "
              "\"parts_ms\": {\"set_grad_f64\": %.2f, \"step\": %.3f, \"aggregate_f64\": %.2f, "
              "\"vector_double_G_alloc_zero\": %.2f}, \"h2d_bytes\": %zu, \"d2h_bytes\": %zu}\n",
              G, steps, facade_ms, into_ms, old_ms, t_up / steps, t_step / steps, t_down / steps, t_alloc / steps, 4 * G,
              4 * G);
  return 0;
}
