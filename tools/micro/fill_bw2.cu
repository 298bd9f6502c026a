// Micro-benchmark: write patterns for the 552 MB dense decode (grid-stride,
// block-contiguous, 16 KB tiles with per-thread vector stores, TMA bulk).
#include <cstdio>
#include <cstdint>

__global__ void k_gs(float4* p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void k_contig(float4* p, uint64_t n4) {
  const uint64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const uint64_t e = min(n4, (blockIdx.x + 1) * per);
  for (uint64_t i = blockIdx.x * per + threadIdx.x; i < e; i += blockDim.x) p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int kV8>
__global__ void k_tiles(float* p, uint64_t n) {  // 4096-float tiles, tile-stride over blocks
  const uint64_t nt = n / 4096;
  for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    float* q = p + t * 4096;
    if (kV8) {
      for (unsigned i = threadIdx.x; i < 512; i += blockDim.x) {
        float z = 0.f;
        asm volatile("st.global.v8.f32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(q + 8 * i), "f"(z) : "memory");
      }
    } else {
      for (unsigned i = threadIdx.x; i < 1024; i += blockDim.x)
        reinterpret_cast<float4*>(q)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

int main() {
  const uint64_t n = 138000000 / 4096 * 4096;
  float* p;
  cudaMalloc(&p, n * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-36s %7.1f us  %7.1f GB/s\n", name, best * 1e3, n * 4 / (best * 1e-3) / 1e9);
  };
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 0, n * 4); });
  for (int m : {6, 8, 16, 32, 64}) {
    char nm[64];
    snprintf(nm, sizeof nm, "grid-stride v4 %d blk/SM", m);
    run(nm, [&] { k_gs<<<sms * m, 256>>>((float4*)p, n / 4); });
    snprintf(nm, sizeof nm, "block-contig v4 %d blk/SM", m);
    run(nm, [&] { k_contig<<<sms * m, 256>>>((float4*)p, n / 4); });
    snprintf(nm, sizeof nm, "16KB tiles v4 %d blk/SM", m);
    run(nm, [&] { k_tiles<0><<<sms * m, 256>>>(p, n); });
    snprintf(nm, sizeof nm, "16KB tiles v8 %d blk/SM", m);
    run(nm, [&] { k_tiles<1><<<sms * m, 256>>>(p, n); });
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
