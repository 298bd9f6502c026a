// fc_device.cuh — device-side layout shared by the kernels and the host
// context.  See DESIGN.md §3 for the data layout in HBM and the per-kernel
// roofline budgets.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fcb {

// ---- geometry ---------------------------------------------------------------
constexpr int kThreads = 256;                 // every streaming kernel
constexpr int kVec = 8;                       // float4 per thread per tile
constexpr int kTile = kThreads * kVec * 4;    // 8192 elements per EF tile
constexpr int kTileShift = 13;
static_assert((1 << kTileShift) == kTile, "tile must be a power of two");

constexpr int kDecTile = 4096;                // dense decode tile (smem floats)
constexpr int kDecShift = 12;
static_assert((1 << kDecShift) == kDecTile, "decode tile must be a power of two");

// Magnitude key of an fp32 value: the IEEE bits with the sign cleared.  For
// finite values, |a| > |b| <=> key(a) > key(b) as unsigned integers, and
// |a| == |b| <=> key(a) == key(b) (+0 and -0 share key 0), which is exactly
// the reference's fabs comparator (inc/compress.hpp:44-48).
// The 31-bit key is resolved in three radix digits: 12 | 12 | 7 bits.
constexpr int kShift1 = 19, kBins1 = 4096;    // bits 30..19 (exponent + 3 mantissa)
constexpr int kShift2 = 7, kBins2 = 4096;     // bits 18..7
constexpr int kBins3 = 128;                   // bits 6..0

constexpr int kSampleBlocks = 128;            // 128 x 256 = 32768 samples
constexpr int kSamples = kSampleBlocks * kThreads;

// Per-worker control block, zeroed at the start of every step (one memset).
struct Ctl {
  unsigned L_digit;       // candidate bound: key >= L_digit << kShift1
  unsigned fallback;      // 1 => sampled bound missed, full re-emission ran
  unsigned cand_count;    // M: candidates emitted
  unsigned done_sample, done_ef, done_fbh, done_fbe, done_r1, done_r2, done_emit, done_gather;
  unsigned b1, b2, T;     // radix digits and the final threshold key
  unsigned pad0;
  unsigned long long need1, need2, needT, count_gt;
  double ge_norm2, topk_norm2, kept_norm2;
  unsigned hist_s[kBins1];   // sample histogram (digit 1)
  unsigned hist1[kBins1];    // candidate histogram (digit 1)
  unsigned hist_fb[kBins1];  // full histogram (fallback only)
  unsigned hist2[kBins2];
  unsigned hist3[kBins3];
};

// Per-worker tile workspace (one entry per 8192-element EF tile).
struct TileWs {
  unsigned* off;     // start of the tile's candidate run in cand_*
  unsigned* cnt;     // candidates in the tile
  unsigned* gt;      // candidates with key > T
  unsigned* eq;      // candidates with key == T
  unsigned* out;     // output offset of the tile's selected elements
  unsigned* take;    // ties at T the tile contributes (lowest indices first)
  double* norm;      // sum of squares of the tile's selected values
  unsigned* cand_idx;
  float* cand_val;
  double* ef_part;   // one per EF block (fixed grid => deterministic)
  double* g_part;    // one per gather block
  unsigned ntiles;
  unsigned ef_grid;
};

}  // namespace fcb

// Kernel launchers (fc_kernels.cu).  All take the context stream.
namespace fcb {
void launch_fill_synth(float* dst, uint64_t G, uint64_t key, int dist, cudaStream_t s);
void launch_sample(const float* g_o, const float* ge, uint64_t G, uint64_t k, Ctl* ctl, int add,
                   int force_fallback, cudaStream_t s);
void launch_ef(const float* g_o, float* ge, uint64_t G, uint64_t k, Ctl* ctl, const TileWs& w,
               int add, int emit, cudaStream_t s);
void launch_fallback(float* ge, uint64_t G, uint64_t k, Ctl* ctl, const TileWs& w, cudaStream_t s);
void launch_refine(uint64_t k, Ctl* ctl, const TileWs& w, cudaStream_t s);
void launch_emit(Ctl* ctl, const TileWs& w, unsigned* out_idx, float* out_val, float* ge,
                 int zero_own, cudaStream_t s);
void launch_gather_zero(const unsigned* bidx, uint64_t k, float* ge, float* contrib, Ctl* ctl,
                        double* part, cudaStream_t s);
void launch_tile_bounds(const unsigned* idx, uint64_t k, uint64_t list_stride, int nlists,
                        uint64_t G, unsigned* bounds, cudaStream_t s);
void launch_decode_ar(const unsigned* idx, const unsigned* bounds, const float* lists, int nlists,
                      uint64_t list_stride, int divide, float divisor, float* agg, uint64_t G,
                      cudaStream_t s);
void launch_decode_ag(const unsigned* packs, uint64_t pack_stride, uint64_t k, int nranks,
                      const unsigned* bounds, float divisor, float* agg, uint64_t G,
                      cudaStream_t s);
void launch_dense_sum(const float* lists, int nlists, uint64_t list_stride, int divide,
                      float divisor, float* out, uint64_t G, cudaStream_t s);
int ef_grid_size();
uint64_t launches();
}  // namespace fcb
