// Micro-benchmark of the peer gather's pieces at C3 size (G = 138M, k = 1.38M
// sorted random indices): remote index/value pulls, the local random gather of
// g_e, local and remote stores -- each alone and combined.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cstdlib>

template <bool kRemoteIdx, bool kPullVals, bool kGather, bool kPush>
__global__ void k_g(const uint4* __restrict__ idx_remote, const uint4* __restrict__ idx_local,
                    const uint4* __restrict__ vals_remote, const float* __restrict__ ge, uint64_t nq,
                    uint4* __restrict__ mine, float4* __restrict__ contrib, uint4* __restrict__ selcopy,
                    float4* __restrict__ peer) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += nt) {
    const uint4 ci = kRemoteIdx ? __ldcv(idx_remote + q) : __ldcs(idx_local + q);
    uint4 cv = make_uint4(0, 0, 0, 0);
    if (kPullVals) cv = __ldcv(vals_remote + q);
    float4 g = make_float4(0, 0, 0, 0);
    if (kGather) {
      g.x = __ldcs(ge + ci.x);
      g.y = __ldcs(ge + ci.y);
      g.z = __ldcs(ge + ci.z);
      g.w = __ldcs(ge + ci.w);
    } else {
      g.x = (float)ci.x;
    }
    mine[q] = ci;
    contrib[q] = g;
    if (kPullVals) selcopy[q] = cv;
    if (kPush) __stcg(peer + q, g);
  }
}

int main(int argc, char** argv) {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const uint64_t G = 138000000, k = 1380000, nq = k / 4;
  std::vector<unsigned> h(G / 100 * 100 / 100);
  std::mt19937_64 rng(1);
  std::vector<unsigned> idx(k);
  {
    std::vector<char> pick(G, 0);
    uint64_t c = 0;
    while (c < k) {
      const uint64_t i = rng() % G;
      if (!pick[i]) { pick[i] = 1; ++c; }
    }
    c = 0;
    for (uint64_t i = 0; i < G && c < k; ++i) if (pick[i]) idx[c++] = (unsigned)i;
  }
  void *r_idx, *r_vals, *r_peer;
  cudaSetDevice(1);
  cudaMalloc(&r_idx, k * 4);
  cudaMalloc(&r_vals, k * 4);
  cudaMalloc(&r_peer, k * 4);
  cudaMemcpy(r_idx, idx.data(), k * 4, cudaMemcpyHostToDevice);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  void *l_idx, *ge, *mine, *contrib, *selcopy;
  cudaMalloc(&l_idx, k * 4);
  cudaMalloc(&ge, G * 4);
  cudaMalloc(&mine, k * 4);
  cudaMalloc(&contrib, k * 4);
  cudaMalloc(&selcopy, k * 4);
  cudaMemcpy(l_idx, idx.data(), k * 4, cudaMemcpyHostToDevice);
  cudaMemset(ge, 0, G * 4);
  void* flush;
  cudaMalloc(&flush, 256ull << 20);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {  // L2 fetch granularity hint (bytes)
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit: %zu\n", v);
  } else {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit (default): %zu\n", v);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int grid) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 256ull << 20);  // evict L2
      cudaEventRecord(e0);
      kern<<<grid, 256>>>((const uint4*)r_idx, (const uint4*)l_idx, (const uint4*)r_vals, (const float*)ge, nq,
                          (uint4*)mine, (float4*)contrib, (uint4*)selcopy, (float4*)r_peer);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) best = std::min(best, ms);
    }
    printf("%-48s grid %5d: %7.1f us\n", name, grid, best * 1e3);
  };
  for (int grid : {sms * 8}) {
    run("local idx only (writes)", k_g<false, false, false, false>, grid);
    run("local idx + gather", k_g<false, false, true, false>, grid);
    run("remote idx", k_g<true, false, false, false>, grid);
    run("remote idx + vals", k_g<true, true, false, false>, grid);
    run("remote idx + gather", k_g<true, false, true, false>, grid);
    run("remote idx + vals + gather + push (full)", k_g<true, true, true, true>, grid);
    run("local idx + gather + push", k_g<false, false, true, true>, grid);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
