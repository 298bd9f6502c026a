// Micro-benchmark: does a kernel that writes with TMA bulk stores (or reads
// with TMA bulk loads) complete later after its blocks' last instruction
// than one using plain stores?  globaltimer marks: A's latest block end vs
// B's earliest block start (B launched right behind A on the same stream).
#include <cstdio>
#include <cstdint>

__device__ unsigned long long g_t[4];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int kMode>  // 0 plain stores, 1 bulk stores, 2 bulk loads
__global__ void k_a(float* dst, size_t per_block) {
  extern __shared__ __align__(128) float sm[];
  float* d = dst + blockIdx.x * (per_block / 4);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (kMode == 0) {
    for (size_t i = threadIdx.x; i < per_block / 4; i += blockDim.x) d[i] = 1.0f;
  } else if (kMode == 1) {
    if (threadIdx.x == 0) {
      for (size_t o = 0; o < per_block; o += 16384) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(sm);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)d + o), "r"(sa),
                     "r"(16384)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t[0], gt());
}
__global__ void k_b() {
  if (threadIdx.x == 0) atomicMin(&g_t[1], gt());
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_block = 4u << 20;
  float* d;
  cudaMalloc(&d, per_block * sms);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_a<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_a<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 2; ++mode) {
    double acc = 0;
    for (int r = 0; r < 12; ++r) {
      unsigned long long init[4] = {0, ~0ull, 0, 0};
      cudaMemcpyToSymbol(g_t, init, sizeof(init));
      if (mode == 0) k_a<0><<<sms, 256, smem>>>(d, per_block);
      else k_a<1><<<sms, 256, smem>>>(d, per_block);
      k_b<<<sms, 256>>>();
      cudaDeviceSynchronize();
      unsigned long long t[4];
      cudaMemcpyFromSymbol(t, g_t, sizeof(t));
      if (r >= 2) acc += (double)(t[1] - t[0]) / 1e3;
    }
    printf("%s: A last block end -> B first block start: %.2f us\n", mode ? "bulk stores" : "plain stores", acc / 10);
  }
  return 0;
}
