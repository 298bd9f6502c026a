// fc_device.cuh — device-side layout shared by the kernels and the host
// context.  See DESIGN.md §3 for the data layout in HBM and §4 for the
// per-kernel roofline budgets.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fcb {

// ---- geometry ---------------------------------------------------------------
constexpr int kThreads = 256;                 // every streaming kernel
constexpr int kVec = 8;                       // float4 per lane per chunk
// A chunk is the unit of the error-feedback pass and of the candidate
// bookkeeping: one warp, 8 x 512-byte coalesced segments, 1024 elements.
constexpr int kChunk = 32 * kVec * 4;
constexpr int kChunkShift = 10;
static_assert((1 << kChunkShift) == kChunk, "chunk must be a power of two");

constexpr int kDecTile = 4096;                // dense decode tile (smem floats)
constexpr int kDecShift = 12;
constexpr int kDecChunks = kDecTile / kChunk;
static_assert((1 << kDecShift) == kDecTile, "decode tile must be a power of two");

// Magnitude key of an fp32 value: the IEEE bits with the sign cleared.  For
// finite values, |a| > |b| <=> key(a) > key(b) as unsigned integers, and
// |a| == |b| <=> key(a) == key(b) (+0 and -0 share key 0), which is exactly
// the reference's fabs comparator (inc/compress.hpp:44-48).
// The 31-bit key is resolved in three radix digits (12 | 8 | 11 bits) by
// k_select over the candidates the error-feedback pass emits.
constexpr int kShift1 = 19, kBins1 = 4096;    // bits 30..19 (exponent + 3 mantissa)

constexpr int kSamples = 32768;                // candidate-bound sample size
constexpr int kSpecBins = 5;                   // speculative level-2 buckets (previous target bucket +- 2)
constexpr int kMaxGrid = 256;                  // grid of the one-block-per-SM kernels (>= SM count)

// Per-worker control block.  Each worker has two, used by alternate steps; the
// EF pass of one step zeroes the other for the next step.
struct Ctl {
  unsigned Lkey;          // candidate bound: every element with key >= Lkey
  unsigned fallback;      // 1 => sampled bound missed, full re-emission ran
  unsigned cand_count;    // M: candidates emitted
  unsigned done_gather, done_red;  // last-block counters
  unsigned ef_next;       // EF work queue: next chunk to hand out
  unsigned bar_ef, bar_sel;  // software grid barriers of the EF / select kernels
  unsigned pad_err;       // (timeouts go to the context's sticky error words, ChunkWs::err)
  unsigned maxkey;        // threshold compressor: max |g_e| key
  unsigned tfail;         // threshold: 1 final t below the candidate bound, 2 output > capacity
  unsigned long long kout;      // threshold: elements selected
  unsigned long long tcnt[64];  // threshold: per-round counts
  unsigned b1, b2, T;     // radix digits and the final threshold key
  unsigned pad0;
  unsigned long long need1, needT, count_gt;
  double ge_norm2, topk_norm2, kept_norm2;
  unsigned long long tphase[8];  // %globaltimer at k_select phase boundaries (diagnostics)
  unsigned long long tphase_ef[4];  // ... and at k_ef's (start, sampled, bound, end)
  unsigned long long tphase_ef2[4];  // k_ef: sample loaded, local histogram flushed; k_select: emission sub-phases
  unsigned long long tphase_sx[8];   // k_select_x sub-phases (block 0; diagnostics)
  unsigned hist_s[kBins1];   // sample histogram (digit 1)
  unsigned hist_s2[256];     // sample histogram of bits 18..11 inside the bound's bucket
  unsigned hist_s2w[kSpecBins * 256];  // the same, speculatively, for the buckets around the previous step's
  unsigned hist1[kBins1];    // candidate histogram, key bits 30..19 (k_select)
  unsigned hist_fb[kBins1];  // full histogram (fallback only)
  unsigned hist2[256];       // bits 18..11 of bucket-b1 candidates
  unsigned hist3[2048];      // bits 10..0
  unsigned hist_w[4096];     // window histogram: key bits 30..11 relative to Lkey (k_select)
  unsigned done_sel;         // k_select_x: last-block counter (finalisation)
  unsigned done_slice;       // k_fetch_gather two-stage broadcast: slice pulled
  unsigned lb_flag[kMaxGrid];             // k_select_x look-back: block b's total is in
  unsigned long long lb_tot[kMaxGrid];    // ... (gt << 32) | eq of block b
};

// Per-worker chunk workspace.  Chunk c's candidates occupy the fixed slot
// [c*kChunk, c*kChunk + cnt[c]) of cand_idx / cand_val.
struct ChunkWs {
  unsigned* cnt;              // candidates in the chunk
  unsigned* off;              // k_select scratch: (gt << 16) | eq per chunk
  unsigned long long* btot;   // k_select: per-block (gt, eq) totals
  double* bnorm;              // k_select: per-block sum of squares of selected values
  unsigned* cand_idx;
  float* cand_val;
  double* cnorm;              // per chunk: sum of g_e^2 (fp64), reduced in chunk order on demand
  double* g_part;             // one per gather block
  unsigned long long* tblk;   // diagnostics: %globaltimer at each EF block's start and end
  unsigned* err;              // the context's sticky error words (host-mapped; see kErr*)
  unsigned* skeys;            // kSamples sampled |g_e| keys (the EF pass's candidate bound)
  unsigned* segcnt;           // candidates per EF segment (EfLayout::seg_id), written by the EF pass
  unsigned* lastb1;           // the previous sampled EF pass's target bucket + 1 (0: none)
  unsigned nchunks;
  unsigned ef_grid;
  unsigned coop;              // grid-barrier kernels launched cooperatively (default)
  unsigned batch;             // EF work-queue batch (chunks per ticket) = candidate packing
};

// Candidate layout written by the EF pass and read by the select.  The EF
// work queue hands out aligned batches of B consecutive chunks covering
// [0, bnd) (bnd = the first multiple of B at or after 90 % of the chunks,
// capped at nchunks), then single chunks; one warp processes a batch in chunk
// order and writes the batch's candidate runs back to back from the batch's
// first slot (B * 1024 slots, never overflowing).  A "segment" is a batch or
// a single chunk: its candidates are contiguous from slot seg_base(c) << 10.
// B = 1 is the plain per-chunk layout (the threshold select, the fallback).
struct EfLayout {
  unsigned B, bnd, nbat;
  __host__ __device__ EfLayout(unsigned nchunks, unsigned b) {
    B = b < 1 ? 1u : b;
    const unsigned big = nchunks - nchunks / 10;
    const unsigned long long up = ((unsigned long long)big + B - 1) / B * B;
    bnd = B == 1 ? 0u : (unsigned)(up < nchunks ? up : nchunks);
    nbat = (bnd + B - 1) / B;
  }
  __host__ __device__ bool seg_start(unsigned c) const { return c >= bnd || c % B == 0; }
  __host__ __device__ bool seg_last(unsigned c, unsigned nchunks) const {
    return c >= bnd || c % B == B - 1 || c + 1 == bnd || c + 1 == nchunks;
  }
  // segment number: batch c / B in [0, bnd), then one per single chunk
  __host__ __device__ unsigned seg_id(unsigned c) const { return c < bnd ? c / B : nbat + (c - bnd); }
  __host__ __device__ unsigned seg_base(unsigned c) const { return c >= bnd ? c : c - c % B; }
};
// Batch size for a gradient of nchunks chunks on an EF grid of `blocks`
// 8-warp blocks: 16 when every warp gets >= 4 such batches, 4 when it gets
// >= 2 of 4, else 1 (small gradients: balance beats packing).
__host__ __device__ inline unsigned ef_batch(uint64_t nchunks, unsigned blocks) {
  const uint64_t warps = (uint64_t)blocks * 8;
  return nchunks >= 64 * warps ? 16u : nchunks >= 8 * warps ? 4u : 1u;
}

// Sticky error words of a context (pinned host memory mapped into the device,
// never reset by a step: the host reads them without synchronising and clears
// them only after reporting).  A kernel that times out stores 1 into its word.
constexpr int kErrBarrier = 0;  // a software grid barrier timed out (blocks not co-resident)
constexpr int kErrPeer = 1;     // a peer-exchange epoch wait timed out (a peer is late or gone)
constexpr int kErrWords = 2;

// Zeros owed to a residual store: the residual must be +0 at the set bits of
// `zmap`.  Applied by the next error-feedback pass instead of k random
// read-modify-write stores.  zmap is a plain bitmap of G
// bits (word i >> 5, bit i & 31): word c*32 + lane covers exactly the 32
// elements lane `lane` owns in the EF pass; the decode kernels build it while
// they scatter the (sorted) index list.
struct Pending {
  const unsigned* zmap = nullptr;
};
__host__ __device__ inline unsigned zmap_word(uint64_t i) { return (unsigned)(i >> 5); }
__host__ __device__ inline unsigned zmap_bit(uint64_t i) { return 1u << ((unsigned)i & 31u); }

// Kernel launchers (fc_kernels.cu).  All take the context stream.
void launch_fill_synth(float* dst, uint64_t G, uint64_t key, int dist, cudaStream_t s);
// EF pass (+ candidate emission when emit).  opts bit 0: fused sample of the
// candidate bound (one grid barrier inside), bit 1: force the fallback, bit 2:
// every element is a candidate (bound 0).  ctl_next:
// the worker's other control block, zeroed for the next step (nullable).
// Returns a cudaError_t.
int launch_ef(const float* g_o, float* ge, uint64_t G, uint64_t k, Ctl* ctl, const ChunkWs& w,
              Pending pz, int add, int emit, int opts, Ctl* ctl_next, cudaStream_t s);
// Returns a cudaError_t value (0 = success).
// ---- peer-memory exchange over NVLink (one process per GPU) ----------------
// Every rank owns an exchange buffer: two parities (alternate steps) of an
// index list and a contribution list (kmax entries each) and two epoch flags
// (list ready, contribution ready), mapped into every peer with CUDA IPC.
constexpr int kMaxPeers = 8;
struct PeerBufs {
  unsigned* list[kMaxPeers];
  float* contrib[kMaxPeers];
  float* reduced[kMaxPeers];             // rank r: the reduced values (every slice, pushed by its owner)
  float* inbox[kMaxPeers];               // rank r: N x 2 parities of contributions pushed to it
  unsigned* bounds[kMaxPeers];           // AG: the chunk bounds of rank r's list (2 parities)
  // rank r's mailbox, N x 8 words: box[r][src * 8 + slot] = the epoch src
  // published for slot 0 (list), 1 (contribution), 2 (reduced slice), 3
  // (two-stage broadcast: its list slice), 5 (teardown barrier); slot 4
  // holds src's ||top-k||^2 (double).  Producers store into every rank's box,
  // consumers poll their own (local) box.
  unsigned long long* box[kMaxPeers];
  int n = 0, rank = 0;
  unsigned* err = nullptr;               // this rank's sticky error words (ChunkWs::err)
  unsigned long long timeout_ns = 0;     // epoch waits give up (and report) after this long
  uint64_t kmax = 0;                     // parity stride of list/contrib/reduced/inbox (multiple of 4)
  uint64_t nb = 0, nbs = 0;              // bounds entries (nchunks + 1), parity stride (multiple of 4)
};
// AG over peer memory: once every rank published `epoch`, copy every rank's
// list (indices, values) and chunk bounds into local arrays laid out as the
// NCCL allgather + k_bounds would have produced them.
void launch_collect_packs(const PeerBufs& pb, int par, unsigned long long epoch, uint64_t k, unsigned* packs,
                          unsigned* bounds, cudaStream_t s);
// bounds_out (nullable): nchunks+1 entries, bounds_out[c] = first output
// position whose index is >= c * kChunk (what k_bounds computes from a list)
// ef_out: the array the EF pass wrote g_e to (read only by the fallback).
// Exact Top-k (SelectMode{} default) or, with rounds > 0, the reference's
// threshold compressor (inc/compress.hpp:81-112): bisection over the
// candidates, then every element with |g_e| >= t (count in ctl->kout, at
// most kcap).  idx_base is added to the emitted indices.
struct SelectMode {
  int rounds = 0;
  uint64_t kcap = 0;
  unsigned idx_base = 0;
  // peer exchange: after the selection, publish it (slot 0 -- and slot 1 --
  // = epoch in every rank's mailbox, system-scope release) for the peers
  // that read it over NVLink
  bool publish = false;
  PeerBufs pb;
  unsigned long long epoch = 0;
  bool publish_contrib = true;  // the values are this rank's contribution (STAR's selected rank)
};
int launch_select(uint64_t k, Ctl* ctl, const ChunkWs& w, const float* ef_out, uint64_t G,
                  unsigned* out_idx, float* out_val, unsigned* bounds_out, const SelectMode& m,
                  cudaStream_t s);
// out = sum of parts[0..n) in a fixed order (one block), e.g. ||g_e||^2 from
// the per-chunk partials of the last EF pass.
void launch_sum_fixed(const double* parts, uint64_t n, double* out, cudaStream_t s);
void launch_sumsq_fixed(const float* v, uint64_t n, double* out, double* parts, cudaStream_t s);
// diagnostics: %globaltimer marks of the last decode (start, end)
void read_tdiag(unsigned long long* out8);
// Peer memory, STAR non-selected ranks (sel >= 0) or every rank in VAR (sel <
// 0: the winner is the argmax of the published ||top-k||^2, written to
// *sel_out): wait for the selected list (epoch), copy it (own list, parity
// par), gather this rank's g_e at it into its contribution list, write the
// decode's chunk bounds, and push the contribution to where it is summed
// (two ranks: the peer's inbox, plus -- STAR -- the selected rank's values
// pulled into this rank's inbox; N > 2: each slice into its owner's inbox),
// then publish it (slot 1 = epoch).  Every later read is local.
__device__ __host__ inline float* inbox_of(const PeerBufs& pb, int dst, int src, int par) {
  return pb.inbox[dst] + ((uint64_t)src * 2 + (uint64_t)par) * pb.kmax;
}
// Owner of list position j when k positions are cut into n slices
// [k r / n, k (r+1) / n).
__device__ __host__ inline int slice_owner(uint64_t j, uint64_t k, int n) {
  int r = (int)((j * (uint64_t)n) / k);
  while (r + 1 < n && (k * (uint64_t)(r + 1)) / (uint64_t)n <= j) ++r;
  while (r > 0 && (k * (uint64_t)r) / (uint64_t)n > j) --r;
  return r;
}
// The selected list's chunk bounds are pulled from its exchange buffer
// (pb.bounds, written by its select) into `bounds`.  ||kept||^2 is not
// formed here (launch_sumsq_fixed over the contribution, on demand).
// tree != 0 (ART-Tree): the whole contribution goes to the root's (sel's)
// inbox instead (see launch_reduce_root).
void launch_fetch_gather(const PeerBufs& pb, int sel, int par, int tree, unsigned long long epoch,
                         const float* ge, uint64_t k, unsigned* bounds, uint64_t nch, Ctl* ctl, int* sel_out,
                         unsigned long long* tblk, cudaStream_t s);  // tblk: per-block marks (diagnostics)
// ART-Tree allreduce over peer memory (see k_reduce_root): the root
// (star_sel, or *dsel when star_sel < 0) sums every contribution in rank
// order, pushes the result into every rank's reduced area, publishes slot 2.
void launch_reduce_root(const PeerBufs& pb, int par, unsigned long long epoch, uint64_t k, int divide,
                        float divisor, int star_sel, const int* dsel, Ctl* ctl, cudaStream_t s);
// Reduce-scatter over peer memory (N > 2): once every rank published its
// contribution (`epoch`), rank r sums slice r of the list in rank order
// (collectives.hpp:82-87, /divisor when divide) from its inbox (the STAR
// selected rank `star_sel`, which runs no gather, is read from its own
// values), pushes the slice into every rank's reduced area and publishes it
// (slot 2).
void launch_reduce_slice(const PeerBufs& pb, int par, unsigned long long epoch, uint64_t k, int divide,
                         float divisor, int star_sel, Ctl* ctl, cudaStream_t s);
// Dense decode once every rank published `epoch`: value j is the sum of this
// rank's contribution and its inbox copy of the peer's (two ranks; /divisor
// when divide) or, with `reduced`, this rank's reduced area.  Local reads only.
// wait_root: -1 waits for every rank's publish (ring), >= 0 for that rank's
// (ART-Tree root), -2 for the rank in *dsel (ART-Tree, VAR winner).
void launch_decode_ar_peers(const PeerBufs& pb, int par, unsigned long long epoch, const unsigned* idx,
                            const unsigned* bounds, uint64_t k, int divide, float divisor, bool reduced,
                            float* agg, uint64_t G, unsigned* zmap, int wait_root, const int* dsel,
                            cudaStream_t s);
// Exchange diagnostics (fc_diag_exchange_ms): publish slots (mask bits) of
// `epoch` without a select; wait like the peer decode (root < 0: every rank);
// a sorted spread index list standing in for a selection.
void launch_publish(const PeerBufs& pb, unsigned long long epoch, unsigned mask, cudaStream_t s);
void launch_peer_barrier(const PeerBufs& pb, cudaStream_t s);
void launch_wait_slot(const PeerBufs& pb, int slot, unsigned long long epoch, int root, cudaStream_t s);
void launch_spread_list(unsigned* out, uint64_t k, uint64_t G, uint64_t shift, cudaStream_t s);
// select_var on the device: winner of the N scores into *sel_out, this rank's
// list (or zeros) into masked; a sum-allreduce of masked broadcasts the list.
void launch_var_mask(const double* scores, int n, int rank, const unsigned* idx, uint64_t k, unsigned* masked,
                     int* sel_out, cudaStream_t s);
// bounds (nullable): also write the decode's chunk bounds of bidx (nch+1)
void launch_gather(const unsigned* bidx, uint64_t k, const float* ge, float* contrib, Ctl* ctl,
                   double* part, unsigned* bounds, uint64_t nch, cudaStream_t s);
void launch_bounds(const unsigned* idx, uint64_t k, uint64_t list_stride, int nlists, uint64_t G,
                   unsigned* bounds, cudaStream_t s);
void launch_zero_at(const unsigned* idx, uint64_t k, float* ge, cudaStream_t s);
// In-place AR decode (one kernel): the previous support `prev` (kp indices)
// zeroed, this step's k values written at idx (chunk bounds `bounds`; local:
// rank-ascending sum of nlists lists), in whole 32-byte sectors; the new
// support kept in `keep` (must not alias prev); owed-zero words follow.
void launch_agg_update(const unsigned* prev, uint64_t kp, const unsigned* idx, uint64_t k, const unsigned* bounds,
                       const float* lists, int nlists, uint64_t list_stride, int divide,
                       float divisor, float* agg, uint64_t G, unsigned* zmap, unsigned* keep,
                       cudaStream_t s);
// The previous support's part alone (sectors / words this step's list does
// not own), needing no exchanged value: the peer paths launch it before
// their waits and the rest with kp = 0 after them.
void launch_agg_clear(const unsigned* prev, uint64_t kp, const unsigned* idx, uint64_t k, const unsigned* bounds,
                      float* agg, uint64_t G, unsigned* zmap, cudaStream_t s);
// ... the same over the peer exchanges (values as launch_decode_ar_peers
// reads them, after its publish waits)
void launch_agg_update_peers(const PeerBufs& pb, int par, unsigned long long epoch, const unsigned* prev,
                             uint64_t kp, const unsigned* idx, uint64_t k, const unsigned* bounds, int divide,
                             float divisor, bool reduced, float* agg, uint64_t G, unsigned* zmap, unsigned* keep,
                             int wait_root, const int* dsel, cudaStream_t s);
// Decodes also write the zero map(s) of the decoded index list(s).
void launch_decode_ar(const unsigned* idx, const unsigned* bounds, const float* lists, int nlists,
                      uint64_t list_stride, int divide, float divisor, float* agg, uint64_t G,
                      unsigned* zmap, cudaStream_t s);
// zmaps: nmaps maps of nchunks*32 words; map m belongs to rank (map_rank0 + m)
void launch_decode_ag(const unsigned* packs, uint64_t pack_stride, uint64_t k, int nranks,
                      const unsigned* bounds, float divisor, float* agg, uint64_t G,
                      unsigned* zmaps, int map_rank0, int nmaps, cudaStream_t s);
void launch_dense_sum(const float* lists, int nlists, uint64_t list_stride, int divide,
                      float divisor, float* out, uint64_t G, cudaStream_t s);
// topk_layerwise for the map's small layers in one launch (one block per
// layer, exact top-k, index order): layer b = layers[b] (offset into g_e,
// length, k, first pack position); per-layer ||top-k||^2 into norms (nullable).
struct SmallLayer {
  unsigned off, len, k, out;
};
// Layers up to this many elements take the one-launch small-layer path (one
// block per layer, staged whole in its shared memory); longer ones the
// segmented EF-emission + select, whose blocks are split by layer length
// (round 2: with the bound at 1M, VGG-16's 590K-element convolutions kept
// one SM busy for 820 us while the rest of the GPU idled).
constexpr unsigned kSmallLayerMax = 49152;

// Segmented launches (layerwise compressor): one k_ef emission pass and one
// k_select_x over several large layers at once.  Blocks [b0, b0 + nb) of the
// launch work on segment s as if they were a whole grid of nb blocks over
// its own slice, control block, workspace and output slot (grid barriers,
// look-back and last-block finalisation count the segment's blocks).
constexpr int kMaxSegs = 16;
struct SegEntry {
  const float* src;   // the layer's g_e (16-byte aligned)
  uint64_t len, k;
  Ctl* ctl;
  Ctl* ctl_next;      // zeroed by the EF pass (the segment's next step)
  ChunkWs ws;         // the segment's chunk arrays (offset views of the worker's)
  unsigned b0, nb;
  unsigned idx_base;  // the layer's offset, added to the output indices
  unsigned* out_idx;
  float* out_val;
};
struct SegTab {
  int n;
  SegEntry e[kMaxSegs];
};
int launch_ef_segs(const SegTab* d_tab, int nblocks, int opts, bool coop, cudaStream_t s);
int launch_select_segs(const SegTab* d_tab, int nblocks, bool coop, cudaStream_t s);
bool select_fits(unsigned nch, unsigned nblocks, unsigned batch);
void launch_topk_small(const float* ge, const SmallLayer* layers, int nlayers, unsigned* out_idx, float* out_val,
                       double* norms, cudaStream_t s);
int ef_grid_size();
uint64_t launches();
__host__ __device__ inline uint64_t nchunks_of(uint64_t G) { return (G + kChunk - 1) >> kChunkShift; }

}  // namespace fcb

namespace fcb {
void launch_triad(const float* a, float* b, uint64_t n, int blocks_per_sm, cudaStream_t s);
void launch_fill_zero(float* b, uint64_t n, int blocks_per_sm, cudaStream_t s);
}  // namespace fcb
