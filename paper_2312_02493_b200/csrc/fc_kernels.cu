// fc_kernels.cu — sm_100a kernels of the Top-k gradient-sync hot path.
//
// Reference algorithm (all in /root/reference/proj/include/flexcomm):
//   error_feedback        compress.hpp:114-120   -> k_ef (fused)
//   select_topk_indices   compress.hpp:38-53     -> k_sample, k_ef (candidate
//                                                   emission), k_refine{1,2},
//                                                   k_tile_count, k_tile_scan,
//                                                   k_emit
//   artopk gather/residual artopk.hpp:92-102     -> k_gather_zero
//   densify               core.hpp:72-81         -> k_tile_bounds + k_decode_ar
//   ag_step scatter-add   artopk.hpp:151-159     -> k_tile_bounds + k_decode_ag
//   allreduce (loopback)  collectives.hpp:82-87  -> summed inside k_decode_ar
//
// Everything is HBM-bound integer/fp32 streaming work: no tensor cores.
// DESIGN.md §4 gives each kernel's algorithmic bytes and roofline.
#include <atomic>
#include <cstdio>

#include "fc_device.cuh"
#include "fc_synth.h"

namespace fcb {

static std::atomic<uint64_t> g_launches{0};
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }
static inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// ---------------------------------------------------------------- helpers ---
__device__ __forceinline__ unsigned key_of(float v) { return __float_as_uint(v) & 0x7fffffffu; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Exclusive block scan; s_warp must hold B/32 + 1 entries.
template <int B>
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* s_warp,
                                                              unsigned long long* total) {
  constexpr int W = B / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long inc = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long x = lane < W ? s_warp[lane] : 0ull;
    const unsigned long long xi = warp_incl_scan(x);
    if (lane < W) s_warp[lane] = xi - x;
    if (lane == W - 1) s_warp[W] = xi;
  }
  __syncthreads();
  const unsigned long long r = inc - v + s_warp[warp];
  if (total) *total = s_warp[W];
  __syncthreads();
  return r;
}

// Deterministic (fixed-tree) block sum of doubles; result valid in all threads.
template <int B>
__device__ __forceinline__ double block_sum(double v, double* s_red) {
  constexpr int W = B / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

// All blocks call this at their end; true in exactly one (the last) block.
__device__ __forceinline__ bool last_block_done(unsigned* counter) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// Scanning a histogram from its top bin down, find the bin b with
//   above(b) < target <= above(b) + hist[b]
// where above(b) = sum of bins > b.  Block-uniform result; false if the whole
// histogram holds fewer than `target` entries.  hist lives in global memory
// (read through L2: it was filled by other blocks' atomics).
template <int B>
__device__ bool block_select_top(const unsigned* hist, int nb, unsigned long long target,
                                 unsigned& bin, unsigned long long& above) {
  __shared__ unsigned long long s_scan[B / 32 + 1];
  __shared__ unsigned s_bin;
  __shared__ unsigned long long s_above;
  __shared__ int s_found;
  const int per = (nb + B - 1) / B;
  const int top = nb - per * (int)threadIdx.x;
  const int bot = top - per < 0 ? 0 : top - per;
  unsigned long long sum = 0;
  for (int b = top - 1; b >= bot; --b) sum += __ldcg(hist + b);
  if (threadIdx.x == 0) s_found = 0;
  const unsigned long long ex = block_excl_scan<B>(sum, s_scan, nullptr);
  if (top > bot && ex < target && target <= ex + sum) {
    unsigned long long acc = ex;
    for (int b = top - 1; b >= bot; --b) {
      const unsigned h = __ldcg(hist + b);
      if (target <= acc + h) {
        s_bin = (unsigned)b;
        s_above = acc;
        s_found = 1;
        break;
      }
      acc += h;
    }
  }
  __syncthreads();
  const bool f = s_found != 0;
  bin = s_bin;
  above = s_above;
  __syncthreads();
  return f;
}

// ------------------------------------------------------------- synthetic ---
__global__ void k_fill_synth(float* __restrict__ dst, uint64_t G, uint64_t key, int dist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < G;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = fc_synth_value(key, i, dist);
}

void launch_fill_synth(float* dst, uint64_t G, uint64_t key, int dist, cudaStream_t s) {
  k_fill_synth<<<num_sms() * 8, kThreads, 0, s>>>(dst, G, key, dist);
  count_launch();
}

// ------------------------------------------------------------------ sample ---
// Strided sample of 32768 error-fed magnitudes -> the candidate bound digit.
// The bound only decides how many elements the EF pass copies out; exactness
// never depends on it (a miss triggers the full fallback).
__global__ void __launch_bounds__(kThreads) k_sample(const float* __restrict__ g_o,
                                                     const float* __restrict__ ge, uint64_t G,
                                                     uint64_t k, Ctl* __restrict__ ctl, int add,
                                                     int force_fb) {
  __shared__ unsigned s_h[kBins1];
  for (int b = threadIdx.x; b < kBins1; b += kThreads) s_h[b] = 0;
  __syncthreads();
  const uint64_t s = blockIdx.x * (uint64_t)kThreads + threadIdx.x;
  const uint64_t i = ((2 * s + 1) * G) / (2ull * kSamples);
  float v = ge[i];
  if (add) v = g_o[i] + v;
  atomicAdd(&s_h[key_of(v) >> kShift1], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kBins1; b += kThreads)
    if (s_h[b]) atomicAdd(&ctl->hist_s[b], s_h[b]);
  if (!last_block_done(&ctl->done_sample)) return;
  const double mean = (double)k / (double)G * (double)kSamples;
  const double target = 1.5 * mean + 6.0 * sqrt(mean) + 8.0;
  unsigned Ld = 0;
  if (force_fb) {
    Ld = kBins1 - 1;
  } else if (target < (double)kSamples) {
    unsigned bin;
    unsigned long long above;
    if (block_select_top<kThreads>(ctl->hist_s, kBins1, (unsigned long long)target, bin, above))
      Ld = bin;
  }
  if (threadIdx.x == 0) ctl->L_digit = Ld;
}

void launch_sample(const float* g_o, const float* ge, uint64_t G, uint64_t k, Ctl* ctl, int add,
                   int force_fallback, cudaStream_t s) {
  k_sample<<<kSampleBlocks, kThreads, 0, s>>>(g_o, ge, G, k, ctl, add, force_fallback);
  count_launch();
}

// ---------------------------------------------------------- error feedback ---
// g_e = g_o + residual, written in place over the residual (12 B/elem), with
//  - ||g_e||^2 (fp64, fixed block order),
//  - kEmit: every element with key >= L (the sampled bound) is copied, in
//    index order within its 8192-element tile, to the candidate arrays, and
//    counted in a 4096-bin histogram of its top 12 key bits.
// Persistent grid with a static tile schedule (deterministic partials).
template <bool kAdd, bool kEmit>
__global__ void __launch_bounds__(kThreads) k_ef(const float* __restrict__ g_o,
                                                 float* __restrict__ ge, uint64_t G, uint64_t k,
                                                 Ctl* __restrict__ ctl, TileWs w, int gated) {
  if (gated && *(volatile unsigned*)&ctl->fallback == 0) return;
  __shared__ unsigned s_h[kEmit ? kBins1 : 1];
  __shared__ unsigned long long s_lo[2][kThreads / 32], s_hi[2][kThreads / 32];
  __shared__ unsigned s_base[2];
  __shared__ double s_red[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (kEmit)
    for (int b = tid; b < kBins1; b += kThreads) s_h[b] = 0;
  const unsigned Lkey = kEmit ? (*(volatile unsigned*)&ctl->L_digit) << kShift1 : 0u;
  __syncthreads();

  double nacc = 0.0;
  const uint64_t ntiles = (G + kTile - 1) >> kTileShift;
  int par = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, par ^= 1) {
    const uint64_t base = t << kTileShift;
    float v[kVec * 4];
    unsigned valid = 0xffffffffu;
    if (base + kTile <= G) {
      const float4* go4 = reinterpret_cast<const float4*>(g_o + base);
      float4* ge4 = reinterpret_cast<float4*>(ge + base);
      float4 A[kVec], Bv[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        Bv[j] = __ldcs(ge4 + j * kThreads + tid);
        if (kAdd) A[j] = __ldcs(go4 + j * kThreads + tid);
      }
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        float4 r = Bv[j];
        if (kAdd) {
          r.x = A[j].x + r.x;
          r.y = A[j].y + r.y;
          r.z = A[j].z + r.z;
          r.w = A[j].w + r.w;
          __stcs(ge4 + j * kThreads + tid, r);
        }
        v[4 * j + 0] = r.x;
        v[4 * j + 1] = r.y;
        v[4 * j + 2] = r.z;
        v[4 * j + 3] = r.w;
      }
    } else {
      valid = 0;
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint64_t i = base + (uint64_t)(j * kThreads + tid) * 4 + e;
          float r = 0.f;
          if (i < G) {
            r = ge[i];
            if (kAdd) {
              r = g_o[i] + r;
              ge[i] = r;
            }
            valid |= 1u << (j * 4 + e);
          }
          v[j * 4 + e] = r;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      float s = v[4 * j] * v[4 * j];
      s = fmaf(v[4 * j + 1], v[4 * j + 1], s);
      s = fmaf(v[4 * j + 2], v[4 * j + 2], s);
      s = fmaf(v[4 * j + 3], v[4 * j + 3], s);
      nacc += (double)s;
    }
    if (kEmit) {
      unsigned mask = 0;
#pragma unroll
      for (int q = 0; q < kVec * 4; ++q) mask |= (key_of(v[q]) >= Lkey ? 1u : 0u) << q;
      mask &= valid;
      // Per-slot counts packed as 4 x 16-bit lanes: slots 0-3 in lo, 4-7 in hi.
      unsigned long long lo = 0, hi = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo |= (unsigned long long)__popc((mask >> (4 * j)) & 0xFu) << (16 * j);
        hi |= (unsigned long long)__popc((mask >> (4 * (j + 4))) & 0xFu) << (16 * j);
      }
      const unsigned long long ilo = warp_incl_scan(lo), ihi = warp_incl_scan(hi);
      if (lane == 31) {
        s_lo[par][warp] = ilo;
        s_hi[par][warp] = ihi;
      }
      __syncthreads();
      unsigned long long wlo = 0, whi = 0, tlo = 0, thi = 0;
#pragma unroll
      for (int q = 0; q < kThreads / 32; ++q) {
        const unsigned long long a = s_lo[par][q], b = s_hi[par][q];
        if (q < warp) {
          wlo += a;
          whi += b;
        }
        tlo += a;
        thi += b;
      }
      const unsigned long long elo = ilo - lo + wlo, ehi = ihi - hi + whi;
      unsigned sb[kVec];
      unsigned run = 0;
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        sb[j] = run;
        run += (unsigned)(((j < 4 ? tlo : thi) >> (16 * (j & 3))) & 0xFFFFu);
      }
      if (tid == 0) {
        const unsigned cb = run ? atomicAdd(&ctl->cand_count, run) : 0u;
        s_base[par] = cb;
        w.off[t] = cb;
        w.cnt[t] = run;
      }
      __syncthreads();
      if (mask) {
        const unsigned cb = s_base[par];
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          const unsigned m4 = (mask >> (4 * j)) & 0xFu;
          if (!m4) continue;
          unsigned pos = cb + sb[j] + (unsigned)(((j < 4 ? elo : ehi) >> (16 * (j & 3))) & 0xFFFFu);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (m4 & (1u << e)) {
              const float x = v[4 * j + e];
              w.cand_idx[pos] = (unsigned)(base + (uint64_t)(j * kThreads + tid) * 4 + e);
              w.cand_val[pos] = x;
              atomicAdd(&s_h[key_of(x) >> kShift1], 1u);
              ++pos;
            }
          }
        }
      }
    }
  }

  if (kEmit) {
    __syncthreads();
    for (int b = tid; b < kBins1; b += kThreads)
      if (s_h[b]) atomicAdd(&ctl->hist1[b], s_h[b]);
  }
  const double bsum = block_sum<kThreads>(nacc, s_red);
  if (tid == 0) w.ef_part[blockIdx.x] = bsum;
  if (!last_block_done(gated ? &ctl->done_fbe : &ctl->done_ef)) return;

  // ---- last block: ||g_e||^2 and the first radix digit of the threshold ----
  if (!gated) {
    double acc = 0.0;
    for (unsigned i = tid; i < gridDim.x; i += kThreads) acc += __ldcg(w.ef_part + i);
    const double tot = block_sum<kThreads>(acc, s_red);
    if (tid == 0) ctl->ge_norm2 = tot;
  }
  if (kEmit) {
    const unsigned M = __ldcg(&ctl->cand_count);
    if ((unsigned long long)M < k) {
      if (tid == 0) ctl->fallback = 1;
      return;
    }
    unsigned bin;
    unsigned long long above;
    block_select_top<kThreads>(ctl->hist1, kBins1, k, bin, above);
    if (tid == 0) {
      ctl->b1 = bin;
      ctl->need1 = k - above;
    }
  }
}

static int g_ef_grid = 0;
int ef_grid_size() {
  if (!g_ef_grid) {
    int occ = 0, o2 = 0, o3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ef<true, true>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_ef<true, false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_ef<false, true>, kThreads, 0);
    if (o2 < occ) occ = o2;
    if (o3 < occ) occ = o3;
    if (occ < 1) occ = 1;
    g_ef_grid = num_sms() * occ;
  }
  return g_ef_grid;
}

void launch_ef(const float* g_o, float* ge, uint64_t G, uint64_t k, Ctl* ctl, const TileWs& w,
               int add, int emit, cudaStream_t s) {
  const int grid = (int)w.ef_grid;
  if (add && emit)
    k_ef<true, true><<<grid, kThreads, 0, s>>>(g_o, ge, G, k, ctl, w, 0);
  else if (add)
    k_ef<true, false><<<grid, kThreads, 0, s>>>(g_o, ge, G, k, ctl, w, 0);
  else
    k_ef<false, true><<<grid, kThreads, 0, s>>>(g_o, ge, G, k, ctl, w, 0);
  count_launch();
}

// ---------------------------------------------------------------- fallback ---
// Only runs when the sampled bound kept fewer than k elements: full digit-1
// histogram of g_e, then an exact re-emission with L = the k-th element's
// digit (so the candidate set provably contains the whole top-k).
__global__ void __launch_bounds__(kThreads) k_fb_hist(const float* __restrict__ ge, uint64_t G,
                                                      uint64_t k, Ctl* __restrict__ ctl) {
  if (*(volatile unsigned*)&ctl->fallback == 0) return;
  __shared__ unsigned s_h[kBins1];
  for (int b = threadIdx.x; b < kBins1; b += kThreads) s_h[b] = 0;
  __syncthreads();
  const uint64_t n4 = G / 4;
  const float4* ge4 = reinterpret_cast<const float4*>(ge);
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * kThreads) {
    const float4 x = __ldcs(ge4 + i);
    atomicAdd(&s_h[key_of(x.x) >> kShift1], 1u);
    atomicAdd(&s_h[key_of(x.y) >> kShift1], 1u);
    atomicAdd(&s_h[key_of(x.z) >> kShift1], 1u);
    atomicAdd(&s_h[key_of(x.w) >> kShift1], 1u);
  }
  if (blockIdx.x == 0)
    for (uint64_t i = n4 * 4 + threadIdx.x; i < G; i += kThreads)
      atomicAdd(&s_h[key_of(ge[i]) >> kShift1], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kBins1; b += kThreads)
    if (s_h[b]) atomicAdd(&ctl->hist_fb[b], s_h[b]);
  if (!last_block_done(&ctl->done_fbh)) return;
  unsigned bin;
  unsigned long long above;
  block_select_top<kThreads>(ctl->hist_fb, kBins1, k, bin, above);
  if (threadIdx.x == 0) {
    ctl->L_digit = bin;
    ctl->cand_count = 0;
  }
  for (int b = threadIdx.x; b < kBins1; b += kThreads) ctl->hist1[b] = 0;
}

void launch_fallback(float* ge, uint64_t G, uint64_t k, Ctl* ctl, const TileWs& w, cudaStream_t s) {
  k_fb_hist<<<num_sms() * 4, kThreads, 0, s>>>(ge, G, k, ctl);
  count_launch();
  k_ef<false, true><<<(int)w.ef_grid, kThreads, 0, s>>>(nullptr, ge, G, k, ctl, w, 1);
  count_launch();
}

// ------------------------------------------------------------------ refine ---
// Digits 2 and 3 of the exact threshold, over the (small) candidate set only.
__global__ void __launch_bounds__(kThreads) k_refine1(Ctl* __restrict__ ctl, TileWs w) {
  __shared__ unsigned s_h[kBins2];
  for (int b = threadIdx.x; b < kBins2; b += kThreads) s_h[b] = 0;
  __syncthreads();
  const unsigned M = *(volatile unsigned*)&ctl->cand_count;
  const unsigned b1 = *(volatile unsigned*)&ctl->b1;
  for (unsigned j = blockIdx.x * kThreads + threadIdx.x; j < M; j += gridDim.x * kThreads) {
    const unsigned key = key_of(__ldcg(w.cand_val + j));
    if ((key >> kShift1) == b1) atomicAdd(&s_h[(key >> kShift2) & (kBins2 - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins2; b += kThreads)
    if (s_h[b]) atomicAdd(&ctl->hist2[b], s_h[b]);
  if (!last_block_done(&ctl->done_r1)) return;
  const unsigned long long need1 = __ldcg(&ctl->need1);
  unsigned bin;
  unsigned long long above;
  block_select_top<kThreads>(ctl->hist2, kBins2, need1, bin, above);
  if (threadIdx.x == 0) {
    ctl->b2 = bin;
    ctl->need2 = need1 - above;
  }
}

__global__ void __launch_bounds__(kThreads) k_refine2(uint64_t k, Ctl* __restrict__ ctl, TileWs w) {
  __shared__ unsigned s_h[kBins3];
  for (int b = threadIdx.x; b < kBins3; b += kThreads) s_h[b] = 0;
  __syncthreads();
  const unsigned M = *(volatile unsigned*)&ctl->cand_count;
  const unsigned hi = ((*(volatile unsigned*)&ctl->b1) << 12) | (*(volatile unsigned*)&ctl->b2);
  for (unsigned j = blockIdx.x * kThreads + threadIdx.x; j < M; j += gridDim.x * kThreads) {
    const unsigned key = key_of(__ldcg(w.cand_val + j));
    if ((key >> kShift2) == hi) atomicAdd(&s_h[key & (kBins3 - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins3; b += kThreads)
    if (s_h[b]) atomicAdd(&ctl->hist3[b], s_h[b]);
  if (!last_block_done(&ctl->done_r2)) return;
  const unsigned long long need2 = __ldcg(&ctl->need2);
  unsigned bin;
  unsigned long long above;
  block_select_top<kThreads>(ctl->hist3, kBins3, need2, bin, above);
  if (threadIdx.x == 0) {
    const unsigned long long needT = need2 - above;
    ctl->T = (hi << kShift2) | bin;
    ctl->needT = needT;
    ctl->count_gt = k - needT;
  }
}

void launch_refine(uint64_t k, Ctl* ctl, const TileWs& w, cudaStream_t s) {
  const int grid = num_sms() * 2;
  k_refine1<<<grid, kThreads, 0, s>>>(ctl, w);
  count_launch();
  k_refine2<<<grid, kThreads, 0, s>>>(k, ctl, w);
  count_launch();
}

// --------------------------------------------------------- ordered emission ---
// (1) per tile: candidates above / equal to T; (2) one-block scan giving each
// tile its output offset and how many of its ties it keeps (lowest index
// first: ties are taken in global index order); (3) per tile: ordered write
// of the selected (index, value) pairs, optional residual zeroing (AG:
// residual_update, compress.hpp:122-130) and the fp64 sum of squares.
__global__ void __launch_bounds__(kThreads) k_tile_count(const Ctl* __restrict__ ctl, TileWs w) {
  const unsigned T = *(volatile const unsigned*)&ctl->T;
  const int lane = threadIdx.x & 31;
  const unsigned nw = gridDim.x * (kThreads / 32);
  for (unsigned t = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); t < w.ntiles; t += nw) {
    const unsigned cnt = w.cnt[t], off = w.off[t];
    unsigned gt = 0, eq = 0;
    for (unsigned c0 = 0; c0 < cnt; c0 += 32) {
      const unsigned c = c0 + lane;
      if (c < cnt) {
        const unsigned key = key_of(__ldcg(w.cand_val + off + c));
        gt += key > T;
        eq += key == T;
      }
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    if (lane == 0) {
      w.gt[t] = gt;
      w.eq[t] = eq;
    }
  }
}

constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const Ctl* __restrict__ ctl, TileWs w) {
  __shared__ unsigned long long s_scan[kScanThreads / 32 + 1];
  const unsigned long long needT = *(volatile const unsigned long long*)&ctl->needT;
  const unsigned n = w.ntiles;
  const unsigned chunk = (n + kScanThreads - 1) / kScanThreads;
  const unsigned t0 = min(n, threadIdx.x * chunk), t1 = min(n, t0 + chunk);
  unsigned long long eqs = 0;
  for (unsigned t = t0; t < t1; ++t) eqs += w.eq[t];
  unsigned long long ep = block_excl_scan<kScanThreads>(eqs, s_scan, nullptr);
  unsigned long long sels = 0;
  for (unsigned t = t0; t < t1; ++t) {
    const unsigned eq = w.eq[t];
    const unsigned long long take = ep >= needT ? 0ull : min((unsigned long long)eq, needT - ep);
    w.take[t] = (unsigned)take;
    ep += eq;
    sels += w.gt[t] + take;
  }
  unsigned long long sp = block_excl_scan<kScanThreads>(sels, s_scan, nullptr);
  for (unsigned t = t0; t < t1; ++t) {
    w.out[t] = (unsigned)sp;
    sp += w.gt[t] + w.take[t];
  }
}

__global__ void __launch_bounds__(kThreads) k_emit(Ctl* __restrict__ ctl, TileWs w,
                                                   unsigned* __restrict__ out_idx,
                                                   float* __restrict__ out_val,
                                                   float* __restrict__ ge, int zero_own) {
  __shared__ double s_red[kThreads / 32];
  const unsigned T = *(volatile const unsigned*)&ctl->T;
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  const unsigned nw = gridDim.x * (kThreads / 32);
  for (unsigned t = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); t < w.ntiles; t += nw) {
    const unsigned cnt = w.cnt[t], off = w.off[t], out = w.out[t], take = w.take[t];
    unsigned eq_seen = 0, written = 0;
    double acc = 0.0;
    for (unsigned c0 = 0; c0 < cnt; c0 += 32) {
      const unsigned c = c0 + lane;
      const bool in = c < cnt;
      const float val = in ? __ldcg(w.cand_val + off + c) : 0.f;
      const unsigned idx = in ? __ldcg(w.cand_idx + off + c) : 0u;
      const unsigned key = key_of(val);
      const bool is_eq = in && key == T;
      const unsigned eqb = __ballot_sync(0xffffffffu, is_eq);
      const bool sel = in && (key > T || (is_eq && eq_seen + __popc(eqb & lt) < take));
      const unsigned sb = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const unsigned pos = out + written + __popc(sb & lt);
        out_idx[pos] = idx;
        out_val[pos] = val;
        if (zero_own) ge[idx] = 0.f;
        acc = fma((double)val, (double)val, acc);
      }
      written += __popc(sb);
      eq_seen += __popc(eqb);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) w.norm[t] = acc;
  }
  if (!last_block_done(&ctl->done_emit)) return;
  double acc = 0.0;
  for (unsigned t = threadIdx.x; t < w.ntiles; t += kThreads) acc += __ldcg(w.norm + t);
  const double tot = block_sum<kThreads>(acc, s_red);
  if (threadIdx.x == 0) ctl->topk_norm2 = tot;
}

void launch_emit(Ctl* ctl, const TileWs& w, unsigned* out_idx, float* out_val, float* ge,
                 int zero_own, cudaStream_t s) {
  const int grid = num_sms() * 4;
  k_tile_count<<<grid, kThreads, 0, s>>>(ctl, w);
  count_launch();
  k_tile_scan<<<1, kScanThreads, 0, s>>>(ctl, w);
  count_launch();
  k_emit<<<grid, kThreads, 0, s>>>(ctl, w, out_idx, out_val, ge, zero_own);
  count_launch();
}

// ------------------------------------------------------------ gather/zero ---
// contrib[j] = g_e[bidx[j]]; residual[bidx[j]] = 0 (artopk.hpp:92-102), and
// the kept energy sum_j g_e[bidx[j]]^2 for the gain (trainer.hpp:387-396).
constexpr int kGatherUnroll = 4;
__global__ void __launch_bounds__(kThreads) k_gather_zero(const unsigned* __restrict__ bidx,
                                                          uint64_t k, float* __restrict__ ge,
                                                          float* __restrict__ contrib,
                                                          Ctl* __restrict__ ctl,
                                                          double* __restrict__ part) {
  __shared__ double s_red[kThreads / 32];
  double acc = 0.0;
  const uint64_t step = (uint64_t)gridDim.x * kThreads;
  for (uint64_t j0 = blockIdx.x * (uint64_t)kThreads + threadIdx.x; j0 < k;
       j0 += step * kGatherUnroll) {
    unsigned ii[kGatherUnroll];
    float vv[kGatherUnroll];
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      const uint64_t j = j0 + u * step;
      ii[u] = j < k ? __ldcs(bidx + j) : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) vv[u] = ii[u] != 0xffffffffu ? ge[ii[u]] : 0.f;
#pragma unroll
    for (int u = 0; u < kGatherUnroll; ++u) {
      if (ii[u] != 0xffffffffu) {
        contrib[j0 + u * step] = vv[u];
        ge[ii[u]] = 0.f;
        acc = fma((double)vv[u], (double)vv[u], acc);
      }
    }
  }
  const double b = block_sum<kThreads>(acc, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
  if (!last_block_done(&ctl->done_gather)) return;
  double a2 = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += kThreads) a2 += __ldcg(part + i);
  const double tot = block_sum<kThreads>(a2, s_red);
  if (threadIdx.x == 0) ctl->kept_norm2 = tot;
}

void launch_gather_zero(const unsigned* bidx, uint64_t k, float* ge, float* contrib, Ctl* ctl,
                        double* part, cudaStream_t s) {
  k_gather_zero<<<num_sms() * 4, kThreads, 0, s>>>(bidx, k, ge, contrib, ctl, part);
  count_launch();
}

// ------------------------------------------------------------------ decode ---
// bounds[t] = first j with idx[j] >= t * kDecTile (per list), so every decode
// tile finds its slice of the sorted index list without a search.
__global__ void k_tile_bounds(const unsigned* __restrict__ idx, uint64_t k, uint64_t list_stride,
                              int nlists, uint64_t ntd, unsigned* __restrict__ bounds) {
  const uint64_t per = k + 1;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < per * nlists;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = q / per, j = q - r * per;
    const unsigned* id = idx + r * list_stride;
    unsigned* bd = bounds + r * (ntd + 1);
    const uint64_t hi = j < k ? (uint64_t)(id[j] >> kDecShift) : ntd;
    const uint64_t lo = j == 0 ? 0 : (uint64_t)(id[j - 1] >> kDecShift) + 1;
    for (uint64_t t = lo; t <= hi; ++t) bd[t] = (unsigned)j;
  }
}

void launch_tile_bounds(const unsigned* idx, uint64_t k, uint64_t list_stride, int nlists,
                        uint64_t G, unsigned* bounds, cudaStream_t s) {
  const uint64_t ntd = (G + kDecTile - 1) >> kDecShift;
  const uint64_t work = (k + 1) * nlists;
  int grid = (int)std::min<uint64_t>((work + kThreads - 1) / kThreads, (uint64_t)num_sms() * 8);
  if (grid < 1) grid = 1;
  k_tile_bounds<<<grid, kThreads, 0, s>>>(idx, k, list_stride, nlists, ntd, bounds);
  count_launch();
}

__device__ __forceinline__ void store_tile(const float* __restrict__ tile, float* __restrict__ agg,
                                           uint64_t t0, uint64_t G) {
  if (t0 + kDecTile <= G) {
    const float4* s4 = reinterpret_cast<const float4*>(tile);
    float4* d4 = reinterpret_cast<float4*>(agg + t0);
#pragma unroll
    for (int q = 0; q < kDecTile / 4 / kThreads; ++q) __stcs(d4 + q * kThreads + threadIdx.x, s4[q * kThreads + threadIdx.x]);
  } else {
    for (uint64_t i = threadIdx.x; t0 + i < G; i += kThreads) agg[t0 + i] = tile[i];
  }
}

// AR decode (densify, core.hpp:72-81): zeros everywhere except the broadcast
// indices, which get the allreduced value.  In loopback the allreduce itself
// happens here, in the reference's order: v = c_0; v += c_r (r ascending);
// v /= N for Avg (collectives.hpp:82-87).
__global__ void __launch_bounds__(kThreads) k_decode_ar(const unsigned* __restrict__ idx,
                                                        const unsigned* __restrict__ bounds,
                                                        const float* __restrict__ lists,
                                                        int nlists, uint64_t list_stride,
                                                        int divide, float divisor,
                                                        float* __restrict__ agg, uint64_t G) {
  __shared__ __align__(16) float tile[kDecTile];
  const uint64_t ntd = (G + kDecTile - 1) >> kDecShift;
  for (uint64_t t = blockIdx.x; t < ntd; t += gridDim.x) {
    const uint64_t t0 = t << kDecShift;
    float4* t4 = reinterpret_cast<float4*>(tile);
#pragma unroll
    for (int q = 0; q < kDecTile / 4 / kThreads; ++q)
      t4[q * kThreads + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    const unsigned lo = __ldg(bounds + t), hi = __ldg(bounds + t + 1);
    __syncthreads();
    for (unsigned j = lo + threadIdx.x; j < hi; j += kThreads) {
      float v = lists[j];
      for (int l = 1; l < nlists; ++l) v += lists[(uint64_t)l * list_stride + j];
      if (divide) v = v / divisor;
      tile[idx[j] - (unsigned)t0] = v;
    }
    __syncthreads();
    store_tile(tile, agg, t0, G);
    __syncthreads();
  }
}

void launch_decode_ar(const unsigned* idx, const unsigned* bounds, const float* lists, int nlists,
                      uint64_t list_stride, int divide, float divisor, float* agg, uint64_t G,
                      cudaStream_t s) {
  k_decode_ar<<<num_sms() * 8, kThreads, 0, s>>>(idx, bounds, lists, nlists, list_stride, divide,
                                                  divisor, agg, G);
  count_launch();
}

// AG decode (ag_step, artopk.hpp:151-159): agg = 0; agg[idx_r] += val_r for
// r ascending; every element /= N.  Indices are unique within a rank, so each
// rank's scatter into the shared-memory tile is race-free; ranks are
// separated by a barrier to keep the reference's summation order.
__global__ void __launch_bounds__(kThreads) k_decode_ag(const unsigned* __restrict__ packs,
                                                        uint64_t pack_stride, uint64_t k,
                                                        int nranks,
                                                        const unsigned* __restrict__ bounds,
                                                        float divisor, float* __restrict__ agg,
                                                        uint64_t G) {
  __shared__ __align__(16) float tile[kDecTile];
  const uint64_t ntd = (G + kDecTile - 1) >> kDecShift;
  for (uint64_t t = blockIdx.x; t < ntd; t += gridDim.x) {
    const uint64_t t0 = t << kDecShift;
    float4* t4 = reinterpret_cast<float4*>(tile);
#pragma unroll
    for (int q = 0; q < kDecTile / 4 / kThreads; ++q)
      t4[q * kThreads + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    for (int r = 0; r < nranks; ++r) {
      const unsigned* bd = bounds + (uint64_t)r * (ntd + 1);
      const unsigned lo = __ldg(bd + t), hi = __ldg(bd + t + 1);
      const unsigned* id = packs + (uint64_t)r * pack_stride;
      const float* va = reinterpret_cast<const float*>(id + k);
      for (unsigned j = lo + threadIdx.x; j < hi; j += kThreads) tile[id[j] - (unsigned)t0] += va[j];
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kDecTile / 4 / kThreads; ++q) {
      float4 x = t4[q * kThreads + threadIdx.x];
      x.x = x.x / divisor;
      x.y = x.y / divisor;
      x.z = x.z / divisor;
      x.w = x.w / divisor;
      t4[q * kThreads + threadIdx.x] = x;
    }
    __syncthreads();
    store_tile(tile, agg, t0, G);
    __syncthreads();
  }
}

void launch_decode_ag(const unsigned* packs, uint64_t pack_stride, uint64_t k, int nranks,
                      const unsigned* bounds, float divisor, float* agg, uint64_t G,
                      cudaStream_t s) {
  k_decode_ag<<<num_sms() * 8, kThreads, 0, s>>>(packs, pack_stride, k, nranks, bounds, divisor,
                                                  agg, G);
  count_launch();
}

// Dense baseline (trainer.hpp:240-244): out = sum_r lists[r] (r ascending), /N.
__global__ void k_dense_sum(const float* __restrict__ lists, int nlists, uint64_t list_stride,
                            int divide, float divisor, float* __restrict__ out, uint64_t G) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < G;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float v = lists[i];
    for (int l = 1; l < nlists; ++l) v += lists[(uint64_t)l * list_stride + i];
    if (divide) v = v / divisor;
    out[i] = v;
  }
}

void launch_dense_sum(const float* lists, int nlists, uint64_t list_stride, int divide,
                      float divisor, float* out, uint64_t G, cudaStream_t s) {
  k_dense_sum<<<num_sms() * 8, kThreads, 0, s>>>(lists, nlists, list_stride, divide, divisor, out,
                                                  G);
  count_launch();
}

}  // namespace fcb
