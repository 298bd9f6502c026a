// Micro-benchmark: NVLink peer bandwidth between GPU 0 and GPU 1 with SM
// loads / stores (4- and 16-byte, various grids) and the copy engine.
#include <cstdio>
#include <cstdint>

template <typename T>
__global__ void k_copy(const T* __restrict__ src, T* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcv(src + i);
}
template <typename T>
__global__ void k_copy_u4(const T* __restrict__ src, T* __restrict__ dst, uint64_t n) {  // 4 loads in flight
  const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 4 * st) {
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * st < n) v[u] = __ldcv(src + i + u * st);
#pragma unroll
    for (int u = 0; u < 4; ++u) if (i + u * st < n) dst[i + u * st] = v[u];
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  const size_t bytes = 64ull << 20;
  void *a0, *b0, *a1;
  cudaSetDevice(1);
  cudaMalloc(&a1, bytes);
  cudaMemset(a1, 1, bytes);
  cudaDeviceEnablePeerAccess(0, 0);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&a0, bytes);
  cudaMalloc(&b0, bytes);
  cudaMemset(a0, 2, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto&& fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %8.1f GB/s  (%.1f us per 64 MB)\n", name, bytes * 10 / (ms * 1e-3) / 1e9, ms * 100);
  };
  timeit("CE peer copy 1->0", [&] { cudaMemcpyPeerAsync(b0, 0, a1, 1, bytes); });
  timeit("CE peer copy 0->1", [&] { cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes); });
  for (int mult : {1, 2, 4, 8, 16}) {
    char nm[96];
    snprintf(nm, sizeof nm, "SM read  u32  grid %3dx256", sms * mult);
    timeit(nm, [&] { k_copy<unsigned><<<sms * mult, 256>>>((const unsigned*)a1, (unsigned*)b0, bytes / 4); });
    snprintf(nm, sizeof nm, "SM read  u32x4inflight grid %3dx256", sms * mult);
    timeit(nm, [&] { k_copy_u4<unsigned><<<sms * mult, 256>>>((const unsigned*)a1, (unsigned*)b0, bytes / 4); });
    snprintf(nm, sizeof nm, "SM read  uint4 grid %3dx256", sms * mult);
    timeit(nm, [&] { k_copy<uint4><<<sms * mult, 256>>>((const uint4*)a1, (uint4*)b0, bytes / 16); });
    snprintf(nm, sizeof nm, "SM write u32  grid %3dx256", sms * mult);
    timeit(nm, [&] { k_copy<unsigned><<<sms * mult, 256>>>((const unsigned*)a0, (unsigned*)a1, bytes / 4); });
    snprintf(nm, sizeof nm, "SM write uint4 grid %3dx256", sms * mult);
    timeit(nm, [&] { k_copy<uint4><<<sms * mult, 256>>>((const uint4*)a0, (uint4*)a1, bytes / 16); });
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
