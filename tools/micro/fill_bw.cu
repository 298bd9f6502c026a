// Micro-benchmark: write-only bandwidth of a 552 MB fill (the dense decode's
// floor) with different store paths.
#include <cstdio>
#include <cstdint>

__global__ void k_st(float4* p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__global__ void k_stcs(float4* p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_float4(0.f, 0.f, 0.f, 0.f));
}
__global__ void k_stcg(float4* p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    __stcg(p + i, make_float4(0.f, 0.f, 0.f, 0.f));
}
__global__ void k_v8(float* p, uint64_t n8) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n8; i += (uint64_t)gridDim.x * blockDim.x) {
    float z = 0.f;
    asm volatile("st.global.v8.f32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"l"(p + 8 * i), "f"(z) : "memory");
  }
}
// TMA bulk stores of a zeroed 16 KB shared tile, one elected thread per block
__global__ void k_bulk(float* p, uint64_t n, unsigned tile) {
  extern __shared__ __align__(128) float s[];
  for (unsigned i = threadIdx.x; i < tile / 4; i += blockDim.x) s[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t nt = n * 4 / tile;
    for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + t * (tile / 4)),
                   "r"((unsigned)__cvta_generic_to_shared(s)), "r"(tile)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const uint64_t n = 138000000;
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
  for (int m : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "st.v4 %d blk/SM", m);
    run(nm, [&] { k_st<<<sms * m, 256>>>((float4*)p, n / 4); });
    snprintf(nm, sizeof nm, "st.cs.v4 %d blk/SM", m);
    run(nm, [&] { k_stcs<<<sms * m, 256>>>((float4*)p, n / 4); });
    snprintf(nm, sizeof nm, "st.cg.v4 %d blk/SM", m);
    run(nm, [&] { k_stcg<<<sms * m, 256>>>((float4*)p, n / 4); });
    snprintf(nm, sizeof nm, "st.v8 %d blk/SM", m);
    run(nm, [&] { k_v8<<<sms * m, 256>>>(p, n / 8); });
  }
  run("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 0, n * 4); });
  for (unsigned tile : {16384u, 32768u}) {
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile);
    for (int m : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "TMA bulk %u B, %d blk/SM", tile, m);
      run(nm, [&] { k_bulk<<<sms * m, 128, tile>>>(p, n, tile); });
    }
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
