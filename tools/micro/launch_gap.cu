// Micro-benchmark: back-to-back launch cost of a 148x1024 kernel with ~200 KB
// dynamic shared memory, normal vs cooperative launch, empty vs a short spin,
// and with/without a grid barrier.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_empty(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }
__global__ void k_sync(int* p) {
  cg::this_grid().sync();
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
__global__ void k_small(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1; }

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d;
  cudaMalloc(&d, 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_sync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 200;
  auto run = [&](const char* name, auto f) {
    for (int i = 0; i < 10; ++i) f();
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < N; ++i) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %7.2f us/launch\n", name, ms * 1e3 / N);
  };
  void* args[] = {&d};
  run("normal 148x1024, 200KB smem, empty", [&] { k_empty<<<sms, 1024, smem, s>>>(d); });
  run("cooperative 148x1024, 200KB smem, empty", [&] {
    cudaLaunchCooperativeKernel((void*)k_empty, sms, 1024, args, smem, s);
  });
  run("cooperative 148x1024, 200KB smem, grid.sync", [&] {
    cudaLaunchCooperativeKernel((void*)k_sync, sms, 1024, args, smem, s);
  });
  run("normal 148x256, no smem, empty", [&] { k_small<<<sms, 256, 0, s>>>(d); });
  run("normal 888x256, no smem, empty", [&] { k_small<<<sms * 6, 256, 0, s>>>(d); });
  run("alternating normal(200KB)/normal(0KB)", [&] {
    k_empty<<<sms, 1024, smem, s>>>(d);
    k_small<<<sms * 6, 256, 0, s>>>(d);
  });
  run("alternating coop(200KB)/normal(0KB)", [&] {
    cudaLaunchCooperativeKernel((void*)k_empty, sms, 1024, args, smem, s);
    k_small<<<sms * 6, 256, 0, s>>>(d);
  });
  return 0;
}
