// Micro-benchmark: per-step overhead of a 3-kernel chain shaped like the sync
// step (EF: 148x256 / 200 KB smem; select: cooperative 148x1024 / 200 KB;
// decode: 888x256 / 32 KB), each spinning ~20 us, with plain launches vs
// programmatic dependent launch (griddepcontrol).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void spin(long long cyc) {
  const long long t0 = clock64();
  while (clock64() - t0 < cyc) {
  }
}
template <bool kPdl, bool kCoop>
__global__ void k_stage(long long cyc, int* p) {
  if (kPdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  spin(cyc);
  if (kCoop) cg::this_grid().sync();
  if (kPdl) asm volatile("griddepcontrol.launch_dependents;");
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d;
  cudaMalloc(&d, 4);
  const int big = 200 * 1024, dec = 32 * 1024;
  cudaFuncSetAttribute(k_stage<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_stage<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_stage<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaFuncSetAttribute(k_stage<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long long cyc = 20 * 1965;  // ~20 us at 1965 MHz
  auto launch = [&](auto kern, int grid, int block, int smem, bool pdl, bool coop) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (pdl) {
      at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[n].val.programmaticStreamSerializationAllowed = 1;
      ++n;
    }
    if (coop) {
      at[n].id = cudaLaunchAttributeCooperative;
      at[n].val.cooperative = 1;
      ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, cyc, d);
    if (e != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(e));
  };
  auto step = [&](bool pdl) {
    if (pdl) {
      launch(k_stage<true, false>, sms, 256, big, true, false);
      launch(k_stage<true, true>, sms, 1024, big, true, true);
      launch(k_stage<true, false>, sms * 6, 256, dec, true, false);
    } else {
      launch(k_stage<false, false>, sms, 256, big, false, false);
      launch(k_stage<false, true>, sms, 1024, big, false, true);
      launch(k_stage<false, false>, sms * 6, 256, dec, false, false);
    }
  };
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int i = 0; i < 20; ++i) step(pdl);
    cudaStreamSynchronize(s);
    const int N = 200;
    cudaEventRecord(a, s);
    for (int i = 0; i < N; ++i) step(pdl);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.2f us per 3-kernel step (3 x 20 us of work)\n", pdl ? "PDL  " : "plain", ms * 1e3 / N);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
