// Micro-benchmark: DRAM bytes and time of 1.38M random 4-byte reads (sorted
// indices into a 552 MB buffer) with different load instructions / cache hints.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>

template <int kMode>
__device__ __forceinline__ float ld(const float* p) {
  float v;
  if constexpr (kMode == 0) return __ldcs(p);
  else if constexpr (kMode == 1) return __ldcg(p);
  else if constexpr (kMode == 2) return __ldg(p);
  else if constexpr (kMode == 3) return __ldcv(p);
  else if constexpr (kMode == 4) return __ldlu(p);
  else if constexpr (kMode == 5) { asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 6) { asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 7) { asm volatile("ld.global.L1::evict_first.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 8) { asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 9) { asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 10) { asm volatile("ld.global.cg.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 11) { asm volatile("ld.global.cs.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 12) { asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else if constexpr (kMode == 13) { asm volatile("ld.global.L1::no_allocate.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
  else { asm volatile("ld.global.lu.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }
}

template <int kMode>
__global__ void k_g(const uint4* __restrict__ idx, const float* __restrict__ ge, uint64_t nq, float4* __restrict__ out) {
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += nt) {
    const uint4 ci = __ldcs(idx + q);
    float4 g;
    g.x = ld<kMode>(ge + ci.x);
    g.y = ld<kMode>(ge + ci.y);
    g.z = ld<kMode>(ge + ci.z);
    g.w = ld<kMode>(ge + ci.w);
    out[q] = g;
  }
}

int main() {
  const uint64_t G = 138000000, k = 1380000, nq = k / 4;
  std::mt19937_64 rng(1);
  std::vector<unsigned> idx(k);
  {
    std::vector<char> pick(G, 0);
    uint64_t c = 0;
    while (c < k) { const uint64_t i = rng() % G; if (!pick[i]) { pick[i] = 1; ++c; } }
    c = 0;
    for (uint64_t i = 0; i < G && c < k; ++i) if (pick[i]) idx[c++] = (unsigned)i;
  }
  void *d_idx, *ge, *out, *flush;
  cudaMalloc(&d_idx, k * 4);
  cudaMalloc(&ge, G * 4);
  cudaMalloc(&out, k * 4);
  cudaMalloc(&flush, 256ull << 20);
  cudaMemcpy(d_idx, idx.data(), k * 4, cudaMemcpyHostToDevice);
  cudaMemset(ge, 0, G * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemsetAsync(flush, r, 256ull << 20);
      cudaEventRecord(e0);
      kern<<<sms * 8, 256>>>((const uint4*)d_idx, (const float*)ge, nq, (float4*)out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) best = best < ms ? best : ms;
    }
    printf("%-40s %7.1f us\n", name, best * 1e3);
  };
  run("ld.cs", k_g<0>);
  run("ld.cg", k_g<1>);
  run("ld.nc (ldg)", k_g<2>);
  run("ld.cv", k_g<3>);
  run("ld.lu", k_g<4>);
  run("ld.L1::no_allocate", k_g<5>);
  run("ld.L2::64B", k_g<6>);
  run("ld.L1::evict_first.L2::64B", k_g<7>);
  run("ld.relaxed.gpu", k_g<8>);
  run("ld.nc.L1::no_allocate", k_g<9>);
  run("ld.cg.L2::64B", k_g<10>);
  run("ld.cs.L2::64B", k_g<11>);
  run("ld.nc.L1::no_allocate.L2::64B", k_g<12>);
  run("ld.L1::no_allocate.L2::64B", k_g<13>);
  run("ld.lu.L2::64B", k_g<14>);
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
