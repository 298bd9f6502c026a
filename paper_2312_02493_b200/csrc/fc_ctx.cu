// fc_ctx.cu — host side of the C-ABI (include/flexcomm_b200.h).
//
// Orchestrates one step of the reference protocol over the kernels in
// fc_kernels.cu and NCCL:
//   artopk_step  inc/artopk.hpp:62-111   -> fc_artopk_step
//   ag_step      inc/artopk.hpp:128-161  -> fc_ag_step
//   Dense sync   inc/trainer.hpp:240-244 -> fc_dense_step
//   topk_exact   inc/compress.hpp:57-65  -> fc_topk_exact
// Loopback contexts hold all N logical workers on one device and perform the
// collectives in HBM with the reference's rank-ascending order; NCCL contexts
// hold one worker per process (one GPU each) and use a Ring-forced and a
// Tree-forced communicator (ReduceAlgo, inc/collectives.hpp:36).
//
// Residual zeroing (artopk.hpp:99-101, compress.hpp:122-130) is recorded as a
// pending-zero list per worker and applied by the next error-feedback pass;
// every path that exposes the residual store materialises it first, so the
// observable state is exactly the reference's.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "fc_device.cuh"
#include "fc_synth.h"
#include "flexcomm_b200.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(FC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define NCCL_TRY(x)                                                                        \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) return fail(FC_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define LAUNCHED() CUDA_TRY(cudaGetLastError())
#define TRY(x)                  \
  do {                          \
    int s_ = (x);               \
    if (s_ != FC_OK) return s_; \
  } while (0)

uint64_t k_of_host(double c, uint64_t g) {
  // inc/compress.hpp:28-33 verbatim semantics: clamp(ceil(c*G - 1e-9), 1, G)
  const double raw = std::ceil(c * static_cast<double>(g) - 1e-9);
  uint64_t k = raw <= 0.0 ? 0 : static_cast<uint64_t>(raw);
  return std::min<uint64_t>(std::max<uint64_t>(k, 1), g);
}

bool cr_valid(double c) { return c > 0.0 && c <= 1.0; }

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

struct Worker {
  float* g_o = nullptr;
  float* ge = nullptr;  // the residual store; holds g_e between EF and gather
  float* snap = nullptr;
  fcb::Ctl* ctl = nullptr;      // this step's control block
  fcb::Ctl* ctl_buf[2] = {};    // alternate steps; each EF zeroes the other one
  int ctl_next = 0;             // the clean one the next EF pass uses
  size_t ctl_bytes = 0;
  fcb::ChunkWs ws{};
  unsigned* pack = nullptr;  // [idx k | val k], capacity 2*kmax
  float* contrib = nullptr;  // capacity kmax
  bool has_topk = false;
  const float* kept_vals = nullptr;  // peer gather: the contribution whose ||.||^2 is the kept mass
  uint64_t kept_k = 0;
  uint64_t topk_k = 0;
  const unsigned* topk_idx = nullptr;  // where the last select wrote its output
  const float* topk_val = nullptr;
  bool kept_is_topk = false;  // gather skipped: kept energy == ||top-k||^2
  fcb::Pending pz{};          // zeros owed to `ge` (zero map, read by the next EF)
  // layerwise segments: control blocks (two sets, alternate steps), sample
  // keys and speculation words per segment
  fcb::Ctl* seg_ctl[2] = {};  // [group * kMaxSegs + segment]
  unsigned* seg_skeys = nullptr;
  unsigned* seg_lastb1 = nullptr;
  int seg_cap = 0;             // groups the arrays hold
  int seg_par = 0;
  const unsigned* pz_idx = nullptr;  // the same zeros as a sorted index list
  uint64_t pz_k = 0;
};

}  // namespace

struct fc_ctx {
  int device = 0, n_local = 1, world = 1, rank = 0;
  uint64_t G = 0, gstride = 0, kmax = 0, nch = 0;  // gstride: per-worker stride (256 B aligned)
  unsigned flags = 0;
  bool nccl = false;
  ncclComm_t comm_ring = nullptr, comm_tree = nullptr;
  cudaStream_t stream = nullptr;
  // FC_HOST_ASYNC copies: an upload stream and a download stream, ordered
  // against the compute stream with events
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  // ART-Ring slice ranks clear the previous support beside their
  // reduce-scatter kernel: fork / join events around this stream
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // per (gradient set, worker): upload done / last kernel reading it done
  std::vector<cudaEvent_t> ev_go_ready, ev_go_free;
  std::vector<char> go_pending, go_read;
  // per aggregate buffer: decode done / download done
  cudaEvent_t ev_agg_ready[2] = {}, ev_agg_free[2] = {};
  bool agg_pending[2] = {}, agg_written[2] = {};
  // FC_FLAG_PIPELINE: two gradient sets (uploads of step s+1 overlap step s)
  // and two aggregates (the download of step s overlaps the decode of s+1)
  int nbuf = 1;
  float* g_o_set[2] = {};
  int in_set = 0;      // the gradient set the next step reads
  float* agg_buf[2] = {};
  int agg_cur = 0;     // the buffer holding the last decoded aggregate (== agg)
  std::vector<Worker> w;
  std::vector<void*> allocs;
  float* g_o_all = nullptr;
  float* ge_all = nullptr;
  float* agg = nullptr;
  unsigned* pack_all = nullptr;
  float* contrib_all = nullptr;
  float* reduced = nullptr;
  unsigned* bidx = nullptr;
  unsigned* ag_recv = nullptr;
  unsigned* bounds = nullptr;  // nlists x (nch + 1)
  unsigned* zmaps = nullptr;   // n_local x (nch * 32) zero maps
  unsigned* agg_support = nullptr;  // indices of agg's nonzero support (incremental decode)
  unsigned* agg_support_next = nullptr;  // where an in-place step keeps its support (swapped after)
  uint64_t agg_support_k = 0;
  bool agg_incr = false;            // agg == densify(agg_support) and zmap 0 == its bits
  uint64_t incr_div = 80;           // in-place update when k <= G / incr_div (FC_INCR_DIV overrides)
  // compressors of the AG path (inc/artopk.hpp:113-123)
  std::vector<uint64_t> layer_off, layer_len;  // layer map (Layerwise), sorted, disjoint
  int thresh_rounds = 25;                      // Threshold bisection rounds
  float* scratch = nullptr;                    // G floats, for layer slices not 16-byte aligned
  fcb::SmallLayer* h_small = nullptr;          // small layers' table (pinned) and its device copy
  fcb::SmallLayer* d_small = nullptr;
  int n_small = 0;
  double small_cr = -1.0;
  uint64_t small_ktot = 0;
  // layerwise large layers: segment tables per (worker, parity, group),
  // pinned host copies and their device copies; rebuilt with the CR
  fcb::SegTab* h_seg = nullptr;
  fcb::SegTab* d_seg = nullptr;
  size_t seg_tab_cap = 0;       // tables h_seg / d_seg hold
  size_t seg_ntab = 0;          // EF tables; the select's follow them
  int seg_groups = 0;
  std::vector<int> seg_blocks, seg_blocks_sel;  // co-resident blocks of each group's EF / select launch
  double seg_cr = -1.0;
  uint64_t seg_ktot = 0;
  double* dnorms = nullptr;
  double* h_norms = nullptr;  // pinned
  // sticky error words (pinned, mapped into the device): set by a kernel whose
  // grid barrier or peer wait timed out, never reset by a step; checked by
  // every step call (without synchronising), fc_sync and fc_join, cleared
  // once reported
  unsigned* h_err = nullptr;
  unsigned* d_err = nullptr;  // the same words, device view
  // fp64 host buffers (fc_*_f64, the reference's DenseGrad): per host thread a
  // pinned fp32 staging chunk and an event (created on first use)
  std::vector<float*> f64_stage;
  std::vector<cudaEvent_t> f64_ev;
  unsigned f64_threads = 0;
  int* dsel = nullptr;        // VAR winner chosen on the device (NCCL)
  // peer-memory exchange (NCCL contexts, 1 < world <= 8, every rank's
  // exchange buffer mapped into every other with CUDA IPC over NVLink)
  bool p2p = false;
  bool peer_only = false;           // FC_FLAG_PEER_ONLY: no NCCL, handles exchanged by the caller
  cudaIpcMemHandle_t my_handle{};
  fcb::PeerBufs pb{};
  void* xbuf = nullptr;
  std::vector<void*> peer_maps;
  unsigned long long epoch = 0;
  bool sel_on_device = false; // the last step's selected rank is in *dsel
  bool has_agg = false;
  // phase events (recorded only for calls that asked for step statistics)
  cudaEvent_t ev[5] = {};
  bool timing = false;
  bool phase_stats = false;
  // EF-kernel timing (dominant kernel, for the roofline)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ef_pending;
  std::vector<cudaEvent_t> ev_pool;
  double ef_ms_sum = 0.0;
  uint64_t ef_n = 0;
  unsigned ef_period = 1, ef_calls = 0;  // time every ef_period-th EF launch

  template <typename T>
  int alloc(T** p, uint64_t count) {
    void* q = nullptr;
    CUDA_TRY(cudaMalloc(&q, std::max<uint64_t>(count, 1) * sizeof(T)));
    allocs.push_back(q);
    *p = static_cast<T*>(q);
    return FC_OK;
  }
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {

int check_worker(const fc_ctx* c, int worker) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (worker < 0 || worker >= c->n_local) return fail(FC_ERR_OUT_OF_RANGE, "worker index out of range");
  return FC_OK;
}

// The compute stream must not read worker i's gradient before its async
// upload landed (called before any kernel that reads g_o).
int go_slot(const fc_ctx* c, int i) { return c->in_set * c->n_local + i; }
int wait_grad(fc_ctx* c, int i) {
  const int q = go_slot(c, i);
  if (c->go_pending[q]) {
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_go_ready[q], 0));
    c->go_pending[q] = 0;
  }
  return FC_OK;
}
// ... and an async upload must not overwrite g_o before the EF pass read it.
int grad_consumed(fc_ctx* c, int i) {
  const int q = go_slot(c, i);
  CUDA_TRY(cudaEventRecord(c->ev_go_free[q], c->stream));
  c->go_read[q] = 1;
  return FC_OK;
}
// After a step read its gradients: the next uploads go to the other set.
void advance_input(fc_ctx* c) {
  if (c->nbuf < 2) return;
  c->in_set ^= 1;
  for (int i = 0; i < c->n_local; ++i) c->w[i].g_o = c->g_o_set[c->in_set] + (uint64_t)i * c->gstride;
  c->g_o_all = c->g_o_set[c->in_set];
}
// A decode must not overwrite the aggregate while an async download reads it.
int wait_agg_free(fc_ctx* c, int b) {
  if (c->agg_pending[b]) {
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_agg_free[b], 0));
    c->agg_pending[b] = false;
  }
  return FC_OK;
}
// The buffer a step decodes into (the other one when pipelined), once its
// download (if any) has finished.
int agg_target(fc_ctx* c, int* b) {
  *b = c->nbuf == 2 ? c->agg_cur ^ 1 : 0;
  return wait_agg_free(c, *b);
}
int agg_written(fc_ctx* c, int b) {
  c->agg_cur = b;
  c->agg = c->agg_buf[b];
  CUDA_TRY(cudaEventRecord(c->ev_agg_ready[b], c->stream));
  c->agg_written[b] = true;
  return FC_OK;
}

int copy_in(fc_ctx* c, float* dst, const float* src, int memkind) {
  if (!src) return fail(FC_ERR_INVALID_ARGUMENT, "null source pointer");
  if (memkind == FC_HOST_ASYNC) return fail(FC_ERR_INVALID_ARGUMENT, "async copies only for gradients");
  CUDA_TRY(cudaMemcpyAsync(dst, src, c->G * sizeof(float),
                           memkind == FC_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           c->stream));
  if (!(c->flags & FC_FLAG_ASYNC) || memkind != FC_DEVICE) CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int copy_out(fc_ctx* c, float* dst, const float* src, uint64_t n, int memkind) {
  if (!dst) return fail(FC_ERR_INVALID_ARGUMENT, "null destination pointer");
  CUDA_TRY(cudaMemcpyAsync(dst, src, n * sizeof(float),
                           memkind == FC_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

void record(fc_ctx* c, int i) {
  if (c->timing && c->phase_stats) cudaEventRecord(c->ev[i], c->stream);
}

// Write the owed zeros now (the residual store is about to be observed).
int materialize(fc_ctx* c, Worker& w) {
  if (w.pz_idx && w.pz_k) {
    fcb::launch_zero_at(w.pz_idx, w.pz_k, w.ge, c->stream);
    LAUNCHED();
  }
  w.pz = fcb::Pending{};
  w.pz_idx = nullptr;
  w.pz_k = 0;
  return FC_OK;
}

int materialize_all(fc_ctx* c) {
  for (auto& w : c->w) TRY(materialize(c, w));
  return FC_OK;
}

// EF + (optionally) candidate emission for worker i; times the EF kernel of
// local worker 0 (the dominant kernel) for the roofline.
// Switch worker w to its clean control block; returns the other one (which
// the EF pass about to run zeroes for the next step).
fcb::Ctl* take_ctl(Worker& w) {
  w.ctl = w.ctl_buf[w.ctl_next];
  w.ctl_next ^= 1;
  return w.ctl_buf[w.ctl_next];
}

int run_ef(fc_ctx* c, int i, uint64_t k, bool topk) {
  Worker& w = c->w[i];
  const int force_fb = std::getenv("FC_FORCE_FALLBACK") != nullptr ? 2 : 0;
  fcb::Ctl* next = take_ctl(w);
  TRY(wait_grad(c, i));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (i == 0 && c->timing && (c->ef_calls++ % c->ef_period) == 0) {
    e0 = c->take_event();
    e1 = c->take_event();
    cudaEventRecord(e0, c->stream);
  }
  // EF, with the candidate bound sampled in the same kernel when Top-k follows
  const int e = fcb::launch_ef(w.g_o, w.ge, c->G, k, w.ctl, w.ws, w.pz, 1, topk ? 1 : 0,
                               topk ? (1 | force_fb) : 0, next, c->stream);
  if (e) return fail(FC_ERR_CUDA, std::string("k_ef launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  LAUNCHED();
  TRY(grad_consumed(c, i));
  w.pz = fcb::Pending{};  // consumed
  w.pz_idx = nullptr;
  w.pz_k = 0;
  if (e0) {
    cudaEventRecord(e1, c->stream);
    c->ef_pending.emplace_back(e0, e1);
  }
  return FC_OK;
}

// Top-k of worker i into its pack; also writes the chunk bounds of the
// selection into bounds slot i (so a decode of this list needs no k_bounds).
int run_select(fc_ctx* c, int i, uint64_t k, const float* ef_out = nullptr,
               const fcb::SelectMode& mode = fcb::SelectMode{}, unsigned* out_idx = nullptr,
               float* out_val = nullptr, unsigned* out_bounds = nullptr) {
  Worker& w = c->w[i];
  // exact: [idx k | val k]; threshold (count unknown): [idx kmax | val kmax]
  const uint64_t voff = mode.rounds > 0 ? c->kmax : k;
  if (!out_idx) {
    out_idx = w.pack;
    out_val = reinterpret_cast<float*>(w.pack + voff);
  }
  w.topk_idx = out_idx;
  w.topk_val = out_val;
  const int e = fcb::launch_select(k, w.ctl, w.ws, ef_out ? ef_out : w.ge, c->G, out_idx, out_val,
                                   out_bounds ? out_bounds : c->bounds + (uint64_t)i * (c->nch + 1), mode,
                                   c->stream);
  if (e) return fail(FC_ERR_CUDA, std::string("k_select launch: ") +
                                      cudaGetErrorString(static_cast<cudaError_t>(e)));
  LAUNCHED();
  w.has_topk = true;
  w.topk_k = k;
  return FC_OK;
}

// Segment tables of the layerwise large layers (rebuilt when the CR or the
// selection size changes): layers in map order, groups of up to kMaxSegs;
// in a group the co-resident blocks are split by layer length (at least one
// each), and the layers' chunk arrays are consecutive views of the worker's.
int build_segs(fc_ctx* c, double cr, uint64_t ktot) {
  if (c->seg_cr == cr && c->seg_ktot == ktot) return FC_OK;
  struct Big {
    uint64_t off, len, k, acc, soff;
  };
  std::vector<Big> big;
  uint64_t acc = 0, soff = 0;
  for (size_t l = 0; l < c->layer_off.size(); ++l) {
    const uint64_t off = c->layer_off[l], len = c->layer_len[l], kl = k_of_host(cr, len);
    if (len > fcb::kSmallLayerMax) {
      big.push_back(Big{off, len, kl, acc, off % 4 ? soff : ~uint64_t(0)});
      if (off % 4) soff += (len + 3) & ~uint64_t(3);
    }
    acc += kl;
  }
  if (soff && !c->scratch) TRY(c->alloc(&c->scratch, c->G + 4 * fcb::kMaxSegs));
  const int ng = (int)((big.size() + fcb::kMaxSegs - 1) / fcb::kMaxSegs);
  CUDA_TRY(cudaStreamSynchronize(c->stream));  // the previous tables are no longer read
  c->seg_groups = ng;
  c->seg_blocks.assign(ng, 0);
  c->seg_blocks_sel.assign(ng, 0);
  // tables [EF | select] x (worker, parity, group): the two launches split
  // the blocks differently (below)
  const size_t ntab = (size_t)c->n_local * 2 * ng;
  if (2 * ntab > c->seg_tab_cap) {  // (kept across CR changes; grown only for a map with more groups)
    if (c->h_seg) cudaFreeHost(c->h_seg);
    c->h_seg = nullptr;
    CUDA_TRY(cudaMallocHost(&c->h_seg, 2 * ntab * sizeof(fcb::SegTab)));
    TRY(c->alloc(&c->d_seg, 2 * ntab));
    c->seg_tab_cap = 2 * ntab;
  }
  c->seg_ntab = ntab;
  if (ng == 0) {
    c->seg_cr = cr;
    c->seg_ktot = ktot;
    return FC_OK;
  }
  const unsigned total = c->w[0].ws.ef_grid;
  for (int i = 0; i < c->n_local; ++i) {
    Worker& w = c->w[i];
    if (w.seg_cap < ng) {  // every (group, segment) has its own control blocks: the groups run in turn
      const uint64_t ns = (uint64_t)ng * fcb::kMaxSegs;
      for (auto& cb : w.seg_ctl) {
        TRY(c->alloc(&cb, ns));
        CUDA_TRY(cudaMemsetAsync(cb, 0, ns * sizeof(fcb::Ctl), c->stream));
      }
      TRY(c->alloc(&w.seg_skeys, ns * fcb::kSamples));
      TRY(c->alloc(&w.seg_lastb1, ns));
      CUDA_TRY(cudaMemsetAsync(w.seg_lastb1, 0, ns * sizeof(unsigned), c->stream));
      w.seg_cap = ng;
    }
    // (a new table may use a segment's control blocks in the other parity
    // order than their last use: start from clean ones)
    for (auto& cb : w.seg_ctl)
      CUDA_TRY(cudaMemsetAsync(cb, 0, (uint64_t)w.seg_cap * fcb::kMaxSegs * sizeof(fcb::Ctl), c->stream));
    w.seg_par = 0;
    float* vals = reinterpret_cast<float*>(w.pack + ktot);
    for (int g = 0; g < ng; ++g) {
      const size_t a = (size_t)g * fcb::kMaxSegs, b = std::min(big.size(), a + fcb::kMaxSegs);
      const int n = (int)(b - a);
      // blocks by length, at least `floor` each, the rest proportionally.
      // The EF pass streams (its time ~ the longest per-block slice):
      // floor 1.  The select is latency-bound per block (a one-block
      // segment runs every phase over all its candidates alone): floor 3.
      uint64_t lsum = 0;
      for (size_t q = a; q < b; ++q) lsum += big[q].len;
      auto split = [&](unsigned floor) {
        if ((unsigned)n * floor > total) floor = 1;
        std::vector<unsigned> nb(n, floor);
        unsigned left = total > (unsigned)n * floor ? total - n * floor : 0;
        unsigned used = 0;
        for (int q = 0; q < n; ++q) {
          const unsigned x = (unsigned)((double)left * (double)big[a + q].len / (double)lsum);
          nb[q] += x;
          used += x;
        }
        for (unsigned r = used; r < left; ++r) {  // remainder to the largest layers' shares
          int best = 0;
          double worst = 0.0;
          for (int q = 0; q < n; ++q) {
            const double per = (double)big[a + q].len / nb[q];
            if (per > worst) worst = per, best = q;
          }
          ++nb[best];
        }
        return nb;
      };
      const std::vector<unsigned> nb = split(1), nbs = split(3);
      unsigned b0 = 0;
      uint64_t co = 0;  // chunk offset of the layer in the worker's arrays
      for (int p = 0; p < 2; ++p) {
        fcb::SegTab& t = c->h_seg[((size_t)i * 2 + p) * ng + g];
        t.n = n;
        b0 = 0;
        co = 0;
        for (int q = 0; q < n; ++q) {
          const Big& L = big[a + q];
          fcb::SegEntry& e = t.e[q];
          const unsigned nch = (unsigned)fcb::nchunks_of(L.len);
          e.src = L.soff == ~uint64_t(0) ? w.ge + L.off : c->scratch + L.soff;
          e.len = L.len;
          e.k = L.k;
          const uint64_t sq = (uint64_t)g * fcb::kMaxSegs + q;
          e.ctl = w.seg_ctl[p] + sq;
          e.ctl_next = w.seg_ctl[p ^ 1] + sq;
          e.ws = w.ws;
          e.ws.nchunks = nch;
          e.ws.ef_grid = nb[q];
          e.ws.batch = fcb::ef_batch(nch, nb[q]);
          e.ws.cnt = w.ws.cnt + co;
          e.ws.cand_idx = w.ws.cand_idx + (co << fcb::kChunkShift);
          e.ws.cand_val = w.ws.cand_val + (co << fcb::kChunkShift);
          e.ws.cnorm = w.ws.cnorm + c->nch + co;
          e.ws.segcnt = w.ws.segcnt + co;
          e.ws.bnorm = w.ws.bnorm + b0;
          e.ws.tblk = w.ws.tblk + 2 * (uint64_t)b0;
          e.ws.skeys = w.seg_skeys + sq * fcb::kSamples;
          e.ws.lastb1 = w.seg_lastb1 + sq;
          e.b0 = b0;
          e.nb = nb[q];
          e.idx_base = (unsigned)L.off;
          e.out_idx = w.pack + L.acc;
          e.out_val = vals + L.acc;
          b0 += nb[q];
          co += nch;
        }
        // the select's table: the same segments over its own block split
        fcb::SegTab& ts = c->h_seg[ntab + ((size_t)i * 2 + p) * ng + g];
        ts = t;
        unsigned s0 = 0;
        for (int q = 0; q < n; ++q) {
          fcb::SegEntry& e = ts.e[q];
          e.ws.bnorm = w.ws.bnorm + s0;
          e.ws.tblk = w.ws.tblk + 2 * (uint64_t)s0;
          e.b0 = s0;
          e.nb = nbs[q];
          if (!fcb::select_fits(e.ws.nchunks, nbs[q], e.ws.batch))
            return fail(FC_ERR_OUT_OF_RANGE, "layer too long for its share of the segmented select");
          s0 += nbs[q];
        }
        c->seg_blocks_sel[g] = (int)s0;
      }
      c->seg_blocks[g] = (int)b0;
    }
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_seg, c->h_seg, 2 * ntab * sizeof(fcb::SegTab), cudaMemcpyHostToDevice, c->stream));
  c->seg_cr = cr;
  c->seg_ktot = ktot;
  return FC_OK;
}

// Layerwise Top-k (inc/compress.hpp:67-79) of worker i's error-fed gradient
// into its pack [idx ktot | val ktot], layers in map order: every layer of
// at most kSmallLayerMax elements in ONE launch (k_topk_small, one block per
// layer); each larger layer through the EF kernel's candidate emission on
// its slice + k_select_x (layer offset added to the indices).
int run_layerwise(fc_ctx* c, int i, double cr, uint64_t ktot) {
  Worker& w = c->w[i];
  const int force_fb = std::getenv("FC_FORCE_FALLBACK") != nullptr ? 2 : 0;
  float* vals = reinterpret_cast<float*>(w.pack + ktot);
  // the small layers' table (pinned host -> device), rebuilt when c changes
  const size_t nl = c->layer_off.size();
  if (c->small_cr != cr || c->small_ktot != ktot) {
    if (!c->h_small) {
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      CUDA_TRY(cudaMallocHost(&c->h_small, nl * sizeof(fcb::SmallLayer)));
      TRY(c->alloc(&c->d_small, nl));
    } else {
      CUDA_TRY(cudaStreamSynchronize(c->stream));  // the previous table's upload is done
    }
    uint64_t acc = 0;
    c->n_small = 0;
    for (size_t l = 0; l < nl; ++l) {
      const uint64_t len = c->layer_len[l], kl = k_of_host(cr, len);
      if (len <= fcb::kSmallLayerMax)
        c->h_small[c->n_small++] = fcb::SmallLayer{(unsigned)c->layer_off[l], (unsigned)len, (unsigned)kl, (unsigned)acc};
      acc += kl;
    }
    if (c->n_small)
      CUDA_TRY(cudaMemcpyAsync(c->d_small, c->h_small, c->n_small * sizeof(fcb::SmallLayer), cudaMemcpyHostToDevice,
                               c->stream));
    c->small_cr = cr;
    c->small_ktot = ktot;
  }
  fcb::launch_topk_small(w.ge, c->d_small, c->n_small, w.pack, vals, nullptr, c->stream);
  LAUNCHED();
  // the large layers: segmented launches, up to kMaxSegs layers per EF
  // emission pass + select pair (the blocks split by layer size)
  TRY(build_segs(c, cr, ktot));
  const int par = w.seg_par;
  w.seg_par ^= 1;
  {
    uint64_t soff = 0;
    for (size_t l = 0; l < nl; ++l) {  // slices the bulk copies cannot read in place
      const uint64_t off = c->layer_off[l], len = c->layer_len[l];
      if (len <= fcb::kSmallLayerMax || off % 4 == 0) continue;
      CUDA_TRY(cudaMemcpyAsync(c->scratch + soff, w.ge + off, len * sizeof(float), cudaMemcpyDeviceToDevice,
                               c->stream));
      soff += (len + 3) & ~uint64_t(3);
    }
  }
  const bool coop = w.ws.coop != 0;
  for (int g = 0; g < c->seg_groups; ++g) {
    const fcb::SegTab* tab = c->d_seg + ((size_t)i * 2 + par) * c->seg_groups + g;
    int e = fcb::launch_ef_segs(tab, c->seg_blocks[g], 1 | force_fb, coop, c->stream);
    if (e) return fail(FC_ERR_CUDA, std::string("k_ef (segments) launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
    LAUNCHED();
    e = fcb::launch_select_segs(tab + c->seg_ntab, c->seg_blocks_sel[g], coop, c->stream);
    if (e) return fail(FC_ERR_CUDA, std::string("k_select_x (segments) launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
    LAUNCHED();
  }
  // ||g_c||^2 of the whole selection (gain input) into this step's control block
  fcb::launch_sumsq_fixed(vals, ktot, &w.ctl->topk_norm2, w.ws.g_part, c->stream);
  LAUNCHED();
  w.has_topk = true;
  w.topk_k = ktot;
  w.kept_is_topk = true;
  return FC_OK;
}

// Threshold compressor (inc/compress.hpp:81-112) of worker i: bisection in
// k_select over the EF pass's candidates; the selection size is read back.
int run_threshold(fc_ctx* c, int i, uint64_t k, uint64_t* kout) {
  Worker& w = c->w[i];
  fcb::SelectMode m;
  m.rounds = c->thresh_rounds;
  m.kcap = c->kmax;
  TRY(run_select(c, i, k, nullptr, m));
  unsigned tfail = 0;
  CUDA_TRY(cudaMemcpyAsync(&tfail, &w.ctl->tfail, sizeof(tfail), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (tfail == 1) {
    // the final t fell below the candidate bound: every element a candidate
    fcb::Ctl* next = take_ctl(w);
    const int e = fcb::launch_ef(nullptr, w.ge, c->G, k, w.ctl, w.ws, fcb::Pending{}, 0, 1, 4, next,
                                 c->stream);
    if (e) return fail(FC_ERR_CUDA, std::string("k_ef launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
    LAUNCHED();
    TRY(run_select(c, i, k, nullptr, m));
    CUDA_TRY(cudaMemcpyAsync(&tfail, &w.ctl->tfail, sizeof(tfail), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  if (tfail == 2)
    return fail(FC_ERR_INVALID_ARGUMENT, "threshold selection larger than the context's max_cr capacity");
  if (tfail) return fail(FC_ERR_RUNTIME, "threshold selection failed");
  unsigned long long ko = 0;
  CUDA_TRY(cudaMemcpy(&ko, &w.ctl->kout, sizeof(ko), cudaMemcpyDeviceToHost));
  *kout = ko;
  w.kept_is_topk = true;
  return FC_OK;
}

// Folds completed EF-kernel event pairs into the running mean (events are
// recycled, so long runs do not accumulate them).
int drain_ef_events(fc_ctx* c) {
  for (auto& pr : c->ef_pending) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, pr.first, pr.second));
    c->ef_ms_sum += ms;
    c->ef_n += 1;
    c->ev_pool.push_back(pr.first);
    c->ev_pool.push_back(pr.second);
  }
  c->ef_pending.clear();
  return FC_OK;
}

// Timeouts recorded by the kernels (sticky words in mapped host memory, so
// this needs no synchronisation: it sees every report of a kernel that has
// finished).  A grid-barrier timeout means the EF / select blocks were not
// co-resident; a peer-wait timeout that a peer was late or gone.  Either way
// the step's results cannot be trusted.  A report is cleared once returned.
int check_errors(fc_ctx* c) {
  if (!c->h_err) return FC_OK;
  volatile unsigned* e = c->h_err;
  const unsigned bar = e[fcb::kErrBarrier], peer = e[fcb::kErrPeer];
  if (!bar && !peer) return FC_OK;
  e[fcb::kErrBarrier] = 0;
  e[fcb::kErrPeer] = 0;
  if (peer)
    return fail(FC_ERR_RUNTIME, "peer exchange timed out waiting for another rank (late or gone); "
                                "the step's results are invalid");
  return fail(FC_ERR_RUNTIME, "grid barrier timed out (kernel blocks not co-resident)");
}

int finish_step(fc_ctx* c, fc_step_stats* st, uint64_t k, int sel, int coll, double hbm, double bus,
                uint64_t launches0) {
  if (!st) {
    if (!(c->flags & FC_FLAG_ASYNC)) {
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      TRY(drain_ef_events(c));
    }
    return check_errors(c);  // async: reports of earlier steps that have finished
  }
  std::memset(st, 0, sizeof(*st));
  st->selected_rank = sel;
  if (sel < 0 && c->sel_on_device && !(c->flags & FC_FLAG_ASYNC)) {
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    CUDA_TRY(cudaMemcpy(&st->selected_rank, c->dsel, sizeof(int), cudaMemcpyDeviceToHost));
  }
  st->collective = coll;
  st->k = k;
  st->hbm_bytes = hbm;
  st->bus_bytes = bus;
  st->launches = fcb::launches() - launches0;
  if (c->flags & FC_FLAG_ASYNC) return check_errors(c);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  TRY(drain_ef_events(c));
  if (c->timing && c->phase_stats) {
    float a = 0, b = 0, d = 0, e = 0, t = 0;
    cudaEventElapsedTime(&a, c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&b, c->ev[1], c->ev[2]);
    cudaEventElapsedTime(&d, c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&e, c->ev[3], c->ev[4]);
    cudaEventElapsedTime(&t, c->ev[0], c->ev[4]);
    st->ms_ef = a;
    st->ms_select = b;
    st->ms_exchange = d;
    st->ms_decode = e;
    st->ms_total = t;
  }
  for (int i = 0; i < c->n_local; ++i) {
    unsigned fb = 0;
    CUDA_TRY(cudaMemcpy(&fb, &c->w[i].ctl->fallback, sizeof(fb), cudaMemcpyDeviceToHost));
    st->fallback |= fb ? 1 : 0;
  }
  return check_errors(c);
}

}  // namespace

extern "C" {

const char* fc_status_string(int status) {
  switch (status) {
    case FC_OK: return "ok";
    case FC_ERR_INVALID_ARGUMENT: return "invalid argument";
    case FC_ERR_OUT_OF_RANGE: return "out of range";
    case FC_ERR_RUNTIME: return "runtime error";
    case FC_ERR_CUDA: return "CUDA error";
    case FC_ERR_NCCL: return "NCCL error";
    case FC_ERR_NO_DEVICE: return "no CUDA device";
  }
  return "unknown status";
}

const char* fc_last_error(void) { return g_err.c_str(); }
int fc_abi_version(void) { return FC_ABI_VERSION; }
uint64_t fc_launch_count(void) { return fcb::launches(); }

int fc_k_of(double c, uint64_t grad_len, uint64_t* k_out) {
  if (!cr_valid(c)) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio must be in (0, 1]");
  if (grad_len == 0) return fail(FC_ERR_INVALID_ARGUMENT, "empty gradient (G == 0)");
  if (!k_out) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  *k_out = k_of_host(c, grad_len);
  return FC_OK;
}

int fc_select_star(long step, int n, int* rank_out) {
  if (n < 1) return fail(FC_ERR_INVALID_ARGUMENT, "worker count must be >= 1");
  if (!rank_out) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  *rank_out = static_cast<int>(step % n);
  return FC_OK;
}

int fc_get_unique_id(unsigned char uid_out[FC_NCCL_UID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == FC_NCCL_UID_BYTES, "nccl uid size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(uid_out, &id, sizeof(id));
  return FC_OK;
}

static int create_impl(fc_ctx* c, const fc_opts* o) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(FC_ERR_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
  if (o->device < 0 || o->device >= ndev) return fail(FC_ERR_INVALID_ARGUMENT, "bad device ordinal");
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, o->device));
  if (prop.major != 10) return fail(FC_ERR_NO_DEVICE, "device is not sm_100 (B200)");
  if (o->grad_len == 0) return fail(FC_ERR_INVALID_ARGUMENT, "empty gradient (G == 0)");
  if (o->grad_len >= (1ull << 31)) return fail(FC_ERR_INVALID_ARGUMENT, "G must be < 2^31");
  if (o->n_local < 1) return fail(FC_ERR_INVALID_ARGUMENT, "worker count must be >= 1");
  c->device = o->device;
  c->G = o->grad_len;
  c->flags = o->flags;
  c->timing = !(o->flags & FC_FLAG_NO_TIMING);
  c->peer_only = (o->flags & FC_FLAG_PEER_ONLY) != 0;
  if (c->peer_only) {
    if (o->nccl_uid) return fail(FC_ERR_INVALID_ARGUMENT, "a peer-only context takes no NCCL id");
    if (o->world < 2 || o->world > fcb::kMaxPeers)
      return fail(FC_ERR_INVALID_ARGUMENT, "a peer-only context needs 2 <= world <= 8");
  }
  c->nccl = o->nccl_uid != nullptr || c->peer_only;  // one worker per process
  c->n_local = o->n_local;
  if (c->nccl) {
    if (o->n_local != 1) return fail(FC_ERR_INVALID_ARGUMENT, "NCCL contexts hold one worker");
    if (o->world < 1 || o->rank < 0 || o->rank >= o->world)
      return fail(FC_ERR_INVALID_ARGUMENT, "bad world/rank");
    c->world = o->world;
    c->rank = o->rank;
  } else {
    c->world = o->n_local;
    c->rank = 0;
  }
  const double max_cr = o->max_cr > 0.0 ? o->max_cr : 1.0;
  if (!cr_valid(max_cr)) return fail(FC_ERR_INVALID_ARGUMENT, "max_cr must be in (0, 1]");
  c->kmax = k_of_host(max_cr, c->G);
  c->nch = fcb::nchunks_of(c->G);

  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->s_aux, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
  for (int b = 0; b < 2; ++b) {
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_agg_ready[b], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_agg_free[b], cudaEventDisableTiming));
  }
  c->nbuf = (o->flags & FC_FLAG_PIPELINE) ? 2 : 1;
  c->ev_go_ready.assign(2 * c->n_local, nullptr);
  c->ev_go_free.assign(2 * c->n_local, nullptr);
  c->go_pending.assign(2 * c->n_local, 0);
  c->go_read.assign(2 * c->n_local, 0);
  for (int i = 0; i < 2 * c->n_local; ++i) {
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_go_ready[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_go_free[i], cudaEventDisableTiming));
  }

  const uint64_t G = c->G, N = c->n_local;
  c->gstride = align_up(G, 64);
  const uint64_t GS = c->gstride;
  const unsigned nch = (unsigned)c->nch;
  const unsigned ef_grid = (unsigned)fcb::ef_grid_size();
  for (int b = 0; b < c->nbuf; ++b) {
    TRY(c->alloc(&c->g_o_set[b], N * GS));
    TRY(c->alloc(&c->agg_buf[b], G));
    CUDA_TRY(cudaMemsetAsync(c->g_o_set[b], 0, N * GS * sizeof(float), c->stream));
    CUDA_TRY(cudaMemsetAsync(c->agg_buf[b], 0, G * sizeof(float), c->stream));
  }
  c->g_o_all = c->g_o_set[0];
  c->agg = c->agg_buf[0];
  TRY(c->alloc(&c->ge_all, N * GS));
  TRY(c->alloc(&c->pack_all, N * 2 * c->kmax));
  TRY(c->alloc(&c->contrib_all, N * c->kmax));
  const uint64_t nl = std::max<uint64_t>(N, (uint64_t)c->world);
  TRY(c->alloc(&c->bounds, nl * (c->nch + 1) + 4));  // (+4: vector pulls of a padded row)
  TRY(c->alloc(&c->zmaps, N * c->nch * 32));
  TRY(c->alloc(&c->agg_support, c->kmax));
  TRY(c->alloc(&c->agg_support_next, c->kmax));
  CUDA_TRY(cudaMemsetAsync(c->zmaps, 0, N * c->nch * 32 * sizeof(unsigned), c->stream));
  // zero agg == densify(empty support); pipelined contexts always decode densely
  c->agg_incr = !(o->flags & (FC_FLAG_DENSE_DECODE | FC_FLAG_PIPELINE));
  c->agg_support_k = 0;
  if (const char* e = std::getenv("FC_INCR_DIV")) c->incr_div = std::strtoull(e, nullptr, 10);
  if (c->nccl) {
    TRY(c->alloc(&c->reduced, c->kmax));
    TRY(c->alloc(&c->bidx, c->kmax));
    TRY(c->alloc(&c->ag_recv, (uint64_t)c->world * 2 * c->kmax));
    // [0, W): VAR scores; [W, W+3): this rank's MOO metrics; [W+3, 4W+3): gathered
    TRY(c->alloc(&c->dnorms, 4 * (uint64_t)c->world + 3));
    TRY(c->alloc(&c->dsel, 1));
  }
  CUDA_TRY(cudaMallocHost(&c->h_norms, 3 * sizeof(double) * std::max(c->world, c->n_local)));
  CUDA_TRY(cudaHostAlloc(&c->h_err, 64, cudaHostAllocMapped));
  std::memset(c->h_err, 0, 64);
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_err), c->h_err, 0));
  CUDA_TRY(cudaMemsetAsync(c->ge_all, 0, N * GS * sizeof(float), c->stream));
  c->w.resize(N);
  for (uint64_t i = 0; i < N; ++i) {
    Worker& w = c->w[i];
    w.g_o = c->g_o_all + i * GS;
    w.ge = c->ge_all + i * GS;
    w.pack = c->pack_all + i * 2 * c->kmax;
    w.contrib = c->contrib_all + i * c->kmax;
    w.ctl_bytes = sizeof(fcb::Ctl);
    for (auto& cb : w.ctl_buf) {
      TRY(c->alloc(&cb, 1));
      CUDA_TRY(cudaMemsetAsync(cb, 0, w.ctl_bytes, c->stream));
    }
    w.ctl = w.ctl_buf[0];
    fcb::ChunkWs& s = w.ws;
    s.nchunks = nch;
    s.ef_grid = ef_grid;
    s.err = c->d_err;
    s.coop = (o->flags & FC_FLAG_NO_COOPERATIVE) ? 0u : 1u;
    s.batch = fcb::ef_batch(nch, ef_grid);  // packed candidate layout (EfLayout)
    TRY(c->alloc(&s.off, nch));
    TRY(c->alloc(&s.cnt, nch + fcb::kMaxSegs));
    TRY(c->alloc(&s.btot, 4096));
    TRY(c->alloc(&s.bnorm, 4096));
    // (+kMaxSegs chunks: a segmented layer pass rounds every layer up to whole chunks)
    TRY(c->alloc(&s.cand_idx, ((uint64_t)nch + fcb::kMaxSegs) << fcb::kChunkShift));
    TRY(c->alloc(&s.cand_val, ((uint64_t)nch + fcb::kMaxSegs) << fcb::kChunkShift));
    TRY(c->alloc(&s.cnorm, 2 * (uint64_t)nch + fcb::kMaxSegs));  // [full EF pass | layer passes]
    TRY(c->alloc(&s.g_part, 4096));
    TRY(c->alloc(&s.skeys, fcb::kSamples));
    TRY(c->alloc(&s.segcnt, nch + 1 + fcb::kMaxSegs));
    TRY(c->alloc(&s.lastb1, 1));
    CUDA_TRY(cudaMemsetAsync(s.lastb1, 0, sizeof(unsigned), c->stream));
    TRY(c->alloc(&s.tblk, 2 * (uint64_t)ef_grid));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));

  if (c->nccl && !c->peer_only) {
    ncclUniqueId id;
    std::memcpy(&id, o->nccl_uid, sizeof(id));
    const bool force = std::getenv("FC_NCCL_NO_FORCE_ALGO") == nullptr;
    const char* prev = std::getenv("NCCL_ALGO");
    std::string saved = prev ? prev : "";
    if (force) setenv("NCCL_ALGO", "Ring", 1);
    ncclResult_t r = ncclCommInitRank(&c->comm_ring, c->world, id, c->rank);
    if (r == ncclSuccess) {
      if (force) setenv("NCCL_ALGO", "Tree", 1);
      r = ncclCommSplit(c->comm_ring, 0, c->rank, &c->comm_tree, nullptr);
    }
    if (force) {
      if (prev) setenv("NCCL_ALGO", saved.c_str(), 1);
      else unsetenv("NCCL_ALGO");
    }
    NCCL_TRY(r);
  }
  return FC_OK;
}

// ---- the peer-memory exchange buffers --------------------------------------
// Layout of one rank's exchange buffer (parity strides are multiples of 4
// elements: 16-byte rows for vector pulls).
struct XLayout {
  uint64_t kst, nbs, list_b, contrib_b, bounds_b, inbox_b, box_b, total;
  XLayout(const fc_ctx* c) {
    const int N = c->world;
    kst = align_up(c->kmax, 4);
    nbs = align_up(c->nch + 1, 4);
    list_b = align_up(2 * kst * sizeof(unsigned), 256);
    contrib_b = align_up(2 * kst * sizeof(float), 256);
    bounds_b = align_up(2 * nbs * sizeof(unsigned), 256);
    inbox_b = align_up(N * 2 * kst * sizeof(float), 256);
    box_b = align_up(N * 8 * sizeof(unsigned long long), 256);
    total = list_b + 2 * contrib_b + inbox_b + bounds_b + box_b;
  }
};

// Allocate and export this rank's exchange buffer.
int p2p_alloc(fc_ctx* c, cudaIpcMemHandle_t* mine, int* ok) {
  const XLayout L(c);
  CUDA_TRY(cudaMalloc(&c->xbuf, L.total));
  CUDA_TRY(cudaMemset(c->xbuf, 0, L.total));
  *ok = cudaIpcGetMemHandle(mine, c->xbuf) == cudaSuccess ? 1 : 0;
  cudaGetLastError();
  return FC_OK;
}

// Map every peer's buffer (handles in rank order); *ok = 0 if any failed
// (nothing stays mapped then).
int p2p_open(fc_ctx* c, const cudaIpcMemHandle_t* hs, int* ok) {
  const int N = c->world;
  std::vector<unsigned char*> base(N, nullptr);
  base[c->rank] = static_cast<unsigned char*>(c->xbuf);
  for (int r = 0; r < N && *ok; ++r) {
    if (r == c->rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      *ok = 0;
      break;
    }
    c->peer_maps.push_back(p);
    base[r] = static_cast<unsigned char*>(p);
  }
  if (!*ok) {
    for (void* p : c->peer_maps) cudaIpcCloseMemHandle(p);
    c->peer_maps.clear();
    return FC_OK;
  }
  const XLayout L(c);
  c->pb.n = N;
  c->pb.rank = c->rank;
  c->pb.err = c->d_err;
  if (!c->pb.timeout_ns) c->pb.timeout_ns = 120ull * 1000000000ull;
  c->pb.kmax = L.kst;
  c->pb.nb = c->nch + 1;
  c->pb.nbs = L.nbs;
  for (int r = 0; r < N; ++r) {
    unsigned char* x = base[r];
    c->pb.list[r] = reinterpret_cast<unsigned*>(x);
    c->pb.contrib[r] = reinterpret_cast<float*>(x + L.list_b);
    c->pb.reduced[r] = reinterpret_cast<float*>(x + L.list_b + L.contrib_b);
    c->pb.inbox[r] = reinterpret_cast<float*>(x + L.list_b + 2 * L.contrib_b);
    c->pb.bounds[r] = reinterpret_cast<unsigned*>(x + L.list_b + 2 * L.contrib_b + L.inbox_b);
    c->pb.box[r] = reinterpret_cast<unsigned long long*>(x + L.list_b + 2 * L.contrib_b + L.inbox_b + L.bounds_b);
  }
  c->p2p = true;
  return FC_OK;
}

// NCCL contexts: map every rank's exchange buffer into every other rank (CUDA
// IPC handles allgathered over NCCL); used only if every rank succeeds.
// FC_NO_P2P=1 keeps the NCCL collectives.  Peer-only contexts
// (FC_FLAG_PEER_ONLY) allocate the buffer here and attach in fc_peer_attach,
// with the handles exchanged by the caller.
int setup_p2p(fc_ctx* c) {
  const int N = c->world;
  if (c->peer_only) {
    cudaIpcMemHandle_t mine{};
    int ok = 1;
    TRY(p2p_alloc(c, &mine, &ok));
    if (!ok) return fail(FC_ERR_CUDA, "cudaIpcGetMemHandle failed for the exchange buffer");
    c->my_handle = mine;
    return FC_OK;
  }
  if (!c->nccl || N < 2 || N > fcb::kMaxPeers || std::getenv("FC_NO_P2P")) return FC_OK;
  cudaIpcMemHandle_t mine{};
  int ok = 1;
  TRY(p2p_alloc(c, &mine, &ok));
  unsigned char* dh = nullptr;
  int* dok = nullptr;
  CUDA_TRY(cudaMalloc(&dh, (N + 1) * sizeof(cudaIpcMemHandle_t)));
  CUDA_TRY(cudaMalloc(&dok, sizeof(int)));
  CUDA_TRY(cudaMemcpy(dh + N * sizeof(cudaIpcMemHandle_t), &mine, sizeof(mine), cudaMemcpyHostToDevice));
  NCCL_TRY(ncclAllGather(dh + N * sizeof(cudaIpcMemHandle_t), dh, sizeof(cudaIpcMemHandle_t), ncclUint8,
                         c->comm_ring, c->stream));
  std::vector<cudaIpcMemHandle_t> hs(N);
  CUDA_TRY(cudaMemcpyAsync(hs.data(), dh, N * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  TRY(p2p_open(c, hs.data(), &ok));
  // every rank must take the same path
  CUDA_TRY(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
  NCCL_TRY(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm_ring, c->stream));
  CUDA_TRY(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  cudaFree(dh);
  cudaFree(dok);
  if (!ok && c->p2p) {  // a peer failed: everyone falls back to NCCL
    for (void* p : c->peer_maps) cudaIpcCloseMemHandle(p);
    c->peer_maps.clear();
    c->p2p = false;
  }
  return FC_OK;
}

// Operations on the NCCL communicators are not available in peer-only
// contexts (and steps need the peer mappings there).
int need_comm(fc_ctx* c, const char* what) {
  if (c->nccl && c->world > 1 && !c->comm_ring)
    return fail(FC_ERR_INVALID_ARGUMENT,
                std::string(what) + " needs NCCL communicators (this is a peer-only context"
                + (c->p2p ? ")" : " not attached yet: fc_peer_attach)"));
  return FC_OK;
}

int fc_create(fc_ctx** out, const fc_opts* opts) {
  if (!out || !opts) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  fc_ctx* c = new fc_ctx();
  int s = create_impl(c, opts);
  if (s == FC_OK) s = setup_p2p(c);
  if (s != FC_OK) {
    std::string msg = g_err;
    fc_destroy(c);
    g_err = msg;
    return s;
  }
  *out = c;
  return FC_OK;
}

int fc_destroy(fc_ctx* c) {
  if (!c) return FC_OK;
  cudaSetDevice(c->device);
  if (c->s_h2d) cudaStreamSynchronize(c->s_h2d);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->s_d2h) cudaStreamSynchronize(c->s_d2h);
  if (c->s_aux) cudaStreamSynchronize(c->s_aux);
  // Peer memory: a peer may still be reading this rank's exchange buffer
  // (AG's collect_packs waits only for the publish, not for the readers), so
  // every rank first passes a barrier that is stream-ordered after all of its
  // own kernels -- once it completes, no rank has an exchange kernel left.
  if (c->p2p && c->comm_ring && c->dsel) {
    if (ncclAllReduce(c->dsel, c->dsel, 1, ncclInt32, ncclMax, c->comm_ring, c->stream) == ncclSuccess)
      cudaStreamSynchronize(c->stream);
  } else if (c->p2p && c->peer_only) {  // the same barrier through the mailboxes
    fcb::launch_peer_barrier(c->pb, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  for (void* p : c->peer_maps) cudaIpcCloseMemHandle(p);
  if (c->xbuf) cudaFree(c->xbuf);
  if (c->comm_tree) ncclCommDestroy(c->comm_tree);
  if (c->comm_ring) ncclCommDestroy(c->comm_ring);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& w : c->w)
    if (w.snap) cudaFree(w.snap);
  if (c->h_norms) cudaFreeHost(c->h_norms);
  if (c->h_err) cudaFreeHost(c->h_err);
  if (c->h_small) cudaFreeHost(c->h_small);
  if (c->h_seg) cudaFreeHost(c->h_seg);
  for (float* q : c->f64_stage) cudaFreeHost(q);
  for (cudaEvent_t e : c->f64_ev) cudaEventDestroy(e);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& pr : c->ef_pending) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  if (c->s_aux) cudaStreamDestroy(c->s_aux);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (auto e : c->ev_go_ready)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_go_free)
    if (e) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    if (c->ev_agg_ready[b]) cudaEventDestroy(c->ev_agg_ready[b]);
    if (c->ev_agg_free[b]) cudaEventDestroy(c->ev_agg_free[b]);
  }
  delete c;
  return FC_OK;
}

int fc_num_workers(const fc_ctx* c, int* n_local, int* world, int* rank) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (n_local) *n_local = c->n_local;
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return FC_OK;
}

int fc_set_grad(fc_ctx* c, int worker, const float* src, int memkind) {
  TRY(check_worker(c, worker));
  CUDA_TRY(cudaSetDevice(c->device));
  if (memkind == FC_HOST_ASYNC) {
    if (!src) return fail(FC_ERR_INVALID_ARGUMENT, "null source pointer");
    // after the last reader of g_o (previous EF pass), before the next one
    const int q = go_slot(c, worker);
    if (c->go_read[q]) CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, c->ev_go_free[q], 0));
    CUDA_TRY(cudaMemcpyAsync(c->w[worker].g_o, src, c->G * sizeof(float), cudaMemcpyHostToDevice,
                             c->s_h2d));
    CUDA_TRY(cudaEventRecord(c->ev_go_ready[q], c->s_h2d));
    c->go_pending[q] = 1;
    return FC_OK;
  }
  TRY(wait_grad(c, worker));
  return copy_in(c, c->w[worker].g_o, src, memkind);
}

// ---- fp64 host buffers (the reference's DenseGrad is std::vector<double>) --
// A host thread pool converts chunk j (fp64 -> fp32, or back) through its own
// pinned staging chunk while the copy engine moves the previous ones: PCIe
// carries fp32 only, and no single-threaded conversion pass or pageable copy
// sits on the path.  Thread t handles chunks t, t + T, ...
namespace {
constexpr uint64_t kF64Chunk = 4ull << 20;  // floats per staging chunk (16 MB)

int f64_setup(fc_ctx* c) {
  if (c->f64_threads) return FC_OK;
  const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
  const unsigned T = std::min(8u, std::max(1u, hw / 2));
  for (unsigned t = 0; t < T; ++t) {
    float* q = nullptr;
    cudaEvent_t e = nullptr;
    CUDA_TRY(cudaMallocHost(&q, kF64Chunk * sizeof(float)));
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->f64_stage.push_back(q);
    c->f64_ev.push_back(e);
  }
  c->f64_threads = T;
  return FC_OK;
}

// dev[0, n) <- (float) src[0, n), chunked through the staging on stream s
int f64_upload(fc_ctx* c, float* dev, const double* src, uint64_t n, cudaStream_t s) {
  TRY(f64_setup(c));
  const unsigned T = c->f64_threads;
  const uint64_t nchk = (n + kF64Chunk - 1) / kF64Chunk;
  std::vector<int> rc(T, FC_OK);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      cudaSetDevice(c->device);
      for (uint64_t j = t; j < nchk; j += T) {
        const uint64_t a = j * kF64Chunk, m = std::min(kF64Chunk, n - a);
        if (cudaEventSynchronize(c->f64_ev[t]) != cudaSuccess) { rc[t] = FC_ERR_CUDA; return; }
        float* q = c->f64_stage[t];
        for (uint64_t i = 0; i < m; ++i) q[i] = static_cast<float>(src[a + i]);
        if (cudaMemcpyAsync(dev + a, q, m * sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaEventRecord(c->f64_ev[t], s) != cudaSuccess) { rc[t] = FC_ERR_CUDA; return; }
      }
    });
  for (auto& x : th) x.join();
  for (int r : rc)
    if (r != FC_OK) return fail(r, "fp64 upload: CUDA copy failed");
  return FC_OK;
}

// dst[0, n) <- (double) dev[0, n), after everything queued on `after`
int f64_download(fc_ctx* c, double* dst, const float* dev, uint64_t n, cudaStream_t after) {
  TRY(f64_setup(c));
  const unsigned T = c->f64_threads;
  cudaEvent_t ready = c->take_event();
  CUDA_TRY(cudaEventRecord(ready, after));
  const uint64_t nchk = (n + kF64Chunk - 1) / kF64Chunk;
  std::vector<int> rc(T, FC_OK);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      cudaSetDevice(c->device);
      cudaStream_t s = nullptr;
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamWaitEvent(s, ready, 0) != cudaSuccess) { rc[t] = FC_ERR_CUDA; return; }
      float* q = c->f64_stage[t];
      for (uint64_t j = t; j < nchk; j += T) {
        const uint64_t a = j * kF64Chunk, m = std::min(kF64Chunk, n - a);
        if (cudaMemcpyAsync(q, dev + a, m * sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) { rc[t] = FC_ERR_CUDA; break; }
        for (uint64_t i = 0; i < m; ++i) dst[a + i] = q[i];
      }
      cudaStreamDestroy(s);
    });
  for (auto& x : th) x.join();
  c->ev_pool.push_back(ready);
  for (int r : rc)
    if (r != FC_OK) return fail(r, "fp64 download: CUDA copy failed");
  return FC_OK;
}
}  // namespace

int fc_set_grad_f64(fc_ctx* c, int worker, const double* src) {
  TRY(check_worker(c, worker));
  if (!src) return fail(FC_ERR_INVALID_ARGUMENT, "null source pointer");
  CUDA_TRY(cudaSetDevice(c->device));
  // after the last reader of this gradient buffer, like an FC_HOST_ASYNC upload
  const int q = go_slot(c, worker);
  if (c->go_read[q]) CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, c->ev_go_free[q], 0));
  TRY(f64_upload(c, c->w[worker].g_o, src, c->G, c->s_h2d));
  CUDA_TRY(cudaEventRecord(c->ev_go_ready[q], c->s_h2d));
  c->go_pending[q] = 1;
  if (!(c->flags & FC_FLAG_ASYNC)) CUDA_TRY(cudaStreamSynchronize(c->s_h2d));
  return FC_OK;
}

int fc_set_residual_f64(fc_ctx* c, int worker, const double* src) {
  TRY(check_worker(c, worker));
  if (!src) return fail(FC_ERR_INVALID_ARGUMENT, "null source pointer");
  CUDA_TRY(cudaSetDevice(c->device));
  Worker& w = c->w[worker];
  w.pz = fcb::Pending{};  // overwritten wholesale: owed zeros are void
  w.pz_idx = nullptr;
  w.pz_k = 0;
  CUDA_TRY(cudaStreamSynchronize(c->stream));  // no kernel is using the residual store
  TRY(f64_upload(c, w.ge, src, c->G, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_get_residual_f64(fc_ctx* c, int worker, double* dst) {
  TRY(check_worker(c, worker));
  if (!dst) return fail(FC_ERR_INVALID_ARGUMENT, "null destination pointer");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize(c, c->w[worker]));
  return f64_download(c, dst, c->w[worker].ge, c->G, c->stream);
}

int fc_get_aggregate_f64(fc_ctx* c, double* dst) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (!dst) return fail(FC_ERR_INVALID_ARGUMENT, "null destination pointer");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(wait_agg_free(c, c->agg_cur));
  return f64_download(c, dst, c->agg, c->G, c->stream);
}

int fc_grad_ptr(fc_ctx* c, int worker, float** p) {
  TRY(check_worker(c, worker));
  if (!p) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  *p = c->w[worker].g_o;
  return FC_OK;
}

int fc_fill_synthetic(fc_ctx* c, int worker, uint64_t seed, uint32_t rank, uint64_t step, int dist) {
  TRY(check_worker(c, worker));
  if (dist < FC_DIST_NORMAL || dist > FC_DIST_LAYERED) return fail(FC_ERR_INVALID_ARGUMENT, "bad distribution");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(wait_grad(c, worker));
  fcb::launch_fill_synth(c->w[worker].g_o, c->G, fc_stream_key(seed, rank, step), dist, c->stream);
  LAUNCHED();
  TRY(grad_consumed(c, worker));  // a later async upload must follow the fill
  if (!(c->flags & FC_FLAG_ASYNC)) CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_set_residual(fc_ctx* c, int worker, const float* src, int memkind) {
  TRY(check_worker(c, worker));
  CUDA_TRY(cudaSetDevice(c->device));
  Worker& w = c->w[worker];
  w.pz = fcb::Pending{};  // overwritten wholesale: owed zeros are void
  w.pz_idx = nullptr;
  w.pz_k = 0;
  return copy_in(c, w.ge, src, memkind);
}

int fc_get_residual(fc_ctx* c, int worker, float* dst, int memkind) {
  TRY(check_worker(c, worker));
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize(c, c->w[worker]));
  return copy_out(c, dst, c->w[worker].ge, c->G, memkind);
}

int fc_residual_ptr(fc_ctx* c, int worker, float** p) {
  TRY(check_worker(c, worker));
  if (!p) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize(c, c->w[worker]));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  *p = c->w[worker].ge;
  return FC_OK;
}

int fc_reset_residuals(fc_ctx* c) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  for (auto& w : c->w) {
    w.pz = fcb::Pending{};
    w.pz_idx = nullptr;
    w.pz_k = 0;
  }
  CUDA_TRY(cudaMemsetAsync(c->ge_all, 0, (uint64_t)c->n_local * c->gstride * sizeof(float), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_get_aggregate(fc_ctx* c, float* dst, int memkind) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  if (memkind == FC_HOST_ASYNC) {
    if (!dst) return fail(FC_ERR_INVALID_ARGUMENT, "null destination pointer");
    // after this step's decode, before the next one (which waits on ev_agg_free)
    const int b = c->agg_cur;
    if (c->agg_written[b]) CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->ev_agg_ready[b], 0));
    CUDA_TRY(cudaMemcpyAsync(dst, c->agg, c->G * sizeof(float), cudaMemcpyDeviceToHost, c->s_d2h));
    CUDA_TRY(cudaEventRecord(c->ev_agg_free[b], c->s_d2h));
    c->agg_pending[b] = true;
    return FC_OK;
  }
  TRY(wait_agg_free(c, c->agg_cur));
  return copy_out(c, dst, c->agg, c->G, memkind);
}

int fc_aggregate_ptr(fc_ctx* c, float** p) {
  if (!c || !p) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  *p = c->agg;
  return FC_OK;
}

int fc_get_topk(fc_ctx* c, int worker, uint32_t* idx, float* val, uint64_t* k_out) {
  TRY(check_worker(c, worker));
  const Worker& w = c->w[worker];
  if (!w.has_topk) return fail(FC_ERR_RUNTIME, "no top-k was computed for this worker in the last step");
  if (k_out) *k_out = w.topk_k;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const unsigned* ti = w.topk_idx ? w.topk_idx : w.pack;
  const float* tv = w.topk_val ? w.topk_val : reinterpret_cast<const float*>(w.pack + w.topk_k);
  if (idx) CUDA_TRY(cudaMemcpy(idx, ti, w.topk_k * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  if (val) CUDA_TRY(cudaMemcpy(val, tv, w.topk_k * sizeof(float), cudaMemcpyDeviceToHost));
  return FC_OK;
}

int fc_get_worker_stats(fc_ctx* c, int worker, fc_worker_stats* out) {
  TRY(check_worker(c, worker));
  if (!out) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  CUDA_TRY(cudaSetDevice(c->device));
  Worker& wk = c->w[worker];
  // ||g_e||^2 of the last EF pass, summed over its per-chunk partials in chunk order
  fcb::launch_sum_fixed(wk.ws.cnorm, c->nch, &wk.ctl->ge_norm2, c->stream);
  // ||kept||^2 of a peer gather: over its contribution list, in list order
  if (wk.kept_vals) fcb::launch_sumsq_fixed(wk.kept_vals, wk.kept_k, &wk.ctl->kept_norm2, wk.ws.g_part, c->stream);
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  fcb::Ctl h;
  CUDA_TRY(cudaMemcpy(&h, wk.ctl, offsetof(fcb::Ctl, hist_s), cudaMemcpyDeviceToHost));
  out->ge_norm2 = h.ge_norm2;
  out->kept_norm2 = c->w[worker].kept_is_topk ? h.topk_norm2 : h.kept_norm2;
  out->topk_norm2 = h.topk_norm2;
  out->threshold_key = h.T;
  out->candidates = h.cand_count;
  out->count_above = h.count_gt;
  out->fallback = h.fallback ? 1 : 0;
  return FC_OK;
}

int fc_snapshot(fc_ctx* c) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize_all(c));
  for (auto& w : c->w) {
    if (!w.snap) CUDA_TRY(cudaMalloc(&w.snap, c->G * sizeof(float)));
    CUDA_TRY(cudaMemcpyAsync(w.snap, w.ge, c->G * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_restore(fc_ctx* c) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  for (auto& w : c->w) {
    if (!w.snap) return fail(FC_ERR_RUNTIME, "restore without snapshot");
    w.pz = fcb::Pending{};
    w.pz_idx = nullptr;
    w.pz_k = 0;
    CUDA_TRY(cudaMemcpyAsync(w.ge, w.snap, c->G * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return FC_OK;
}

int fc_peer_handle(fc_ctx* c, unsigned char out[FC_PEER_HANDLE_BYTES]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == FC_PEER_HANDLE_BYTES, "IPC handle size");
  if (!c || !out) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  if (!c->peer_only) return fail(FC_ERR_INVALID_ARGUMENT, "not a peer-only context (FC_FLAG_PEER_ONLY)");
  std::memcpy(out, &c->my_handle, sizeof(c->my_handle));
  return FC_OK;
}

int fc_peer_attach(fc_ctx* c, const unsigned char* handles) {
  if (!c || !handles) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  if (!c->peer_only) return fail(FC_ERR_INVALID_ARGUMENT, "not a peer-only context (FC_FLAG_PEER_ONLY)");
  if (c->p2p) return fail(FC_ERR_INVALID_ARGUMENT, "already attached");
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<cudaIpcMemHandle_t> hs(c->world);
  std::memcpy(hs.data(), handles, c->world * sizeof(cudaIpcMemHandle_t));
  if (std::memcmp(&hs[c->rank], &c->my_handle, sizeof(c->my_handle)) != 0)
    return fail(FC_ERR_INVALID_ARGUMENT, "handles[rank] is not this context's handle (rank order?)");
  int ok = 1;
  TRY(p2p_open(c, hs.data(), &ok));
  if (!ok) return fail(FC_ERR_CUDA, "cudaIpcOpenMemHandle failed for a peer's exchange buffer");
  return FC_OK;
}

int fc_set_peer_timeout(fc_ctx* c, double seconds) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (!(seconds > 0.0) || seconds > 1e7) return fail(FC_ERR_INVALID_ARGUMENT, "timeout must be in (0, 1e7] s");
  c->pb.timeout_ns = (unsigned long long)(seconds * 1e9);
  return FC_OK;
}

int fc_peer_exchange(fc_ctx* c, int* enabled) {
  if (!c || !enabled) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  *enabled = c->p2p ? 1 : 0;
  return FC_OK;
}

int fc_aggregate_in_place(fc_ctx* c, int* in_place) {
  if (!c || !in_place) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  *in_place = c->agg_incr ? 1 : 0;
  return FC_OK;
}

int fc_moo_metrics(fc_ctx* c, int ag, const fc_step_stats* st, double* gain, double* t_comp_s) {
  if (!c || !st || !gain || !t_comp_s) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  TRY(need_comm(c, "fc_moo_metrics"));
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  // this process's workers: (gain_r, t_comp, degenerate_r) triples.  A
  // degenerate gradient (inc/trainer.hpp:391-393) is not returned early: the
  // flag travels with the metrics so that every rank fails the same way and
  // the ranks stay in lockstep (no rank left waiting in the allgather)
  const double tc = (st->ms_ef + st->ms_select + st->ms_decode) * 1e-3;
  std::vector<double> mine(3 * (size_t)c->n_local);
  for (int i = 0; i < c->n_local; ++i) {
    fc_worker_stats ws{};
    TRY(fc_get_worker_stats(c, i, &ws));
    const bool degenerate = !(ws.ge_norm2 > 0.0);
    double g = degenerate ? 0.0 : (ag ? ws.topk_norm2 : ws.kept_norm2) / ws.ge_norm2;
    if (!ag) g = std::min(std::max(g, 0.0), 1.0);  // std::clamp(kept / ge, 0, 1)
    mine[3 * i] = g;
    mine[3 * i + 1] = tc;
    mine[3 * i + 2] = degenerate ? 1.0 : 0.0;
  }
  const int N = c->world;
  double* all = c->h_norms;  // 3N pinned doubles, rank order
  if (c->nccl) {
    double* send = c->dnorms + N;
    double* recv = c->dnorms + N + 3;
    CUDA_TRY(cudaMemcpyAsync(send, mine.data(), 3 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(ncclAllGather(send, recv, 3, ncclFloat64, c->comm_ring, c->stream));
    CUDA_TRY(cudaMemcpyAsync(all, recv, 3 * sizeof(double) * N, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  } else {
    for (int i = 0; i < 3 * N; ++i) all[i] = mine[i];
  }
  // gain_sum / n in rank order (inc/trainer.hpp:364-369, 387-396)
  double sum = 0.0, tmax = 0.0;
  for (int r = 0; r < N; ++r) {
    if (all[3 * r + 2] != 0.0) return fail(FC_ERR_RUNTIME, "degenerate gradient");
    sum += all[3 * r];
    tmax = std::max(tmax, all[3 * r + 1]);
  }
  *gain = sum / N;
  *t_comp_s = tmax;
  return FC_OK;
}

int fc_sync(fc_ctx* c) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->s_h2d));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->s_d2h));
  return check_errors(c);
}

int fc_join(fc_ctx* c) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaEvent_t a = c->take_event(), b = c->take_event();
  CUDA_TRY(cudaEventRecord(a, c->s_h2d));
  CUDA_TRY(cudaEventRecord(b, c->s_d2h));
  CUDA_TRY(cudaStreamWaitEvent(c->stream, a, 0));
  CUDA_TRY(cudaStreamWaitEvent(c->stream, b, 0));
  c->ev_pool.push_back(a);  // safe: a recorded event may be re-recorded later
  c->ev_pool.push_back(b);
  return check_errors(c);
}

int fc_stream(fc_ctx* c, void** stream_out) {
  if (!c || !stream_out) return fail(FC_ERR_INVALID_ARGUMENT, "null argument");
  *stream_out = c->stream;
  return FC_OK;
}

int fc_set_ef_timing_period(fc_ctx* c, int period) {
  if (!c || period < 1) return fail(FC_ERR_INVALID_ARGUMENT, "period must be >= 1");
  c->ef_period = (unsigned)period;
  c->ef_calls = 0;
  return FC_OK;
}

int fc_ef_kernel_timing(fc_ctx* c, double* mean_ms, uint64_t* launches, int reset) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  TRY(drain_ef_events(c));
  if (mean_ms) *mean_ms = c->ef_n ? c->ef_ms_sum / (double)c->ef_n : 0.0;
  if (launches) *launches = c->ef_n;
  if (reset) {
    c->ef_ms_sum = 0.0;
    c->ef_n = 0;
  }
  return FC_OK;
}

// Diagnostics: mean device time (CUDA events around each launch) of one
// kernel of the path, or of a reference streaming kernel, on worker 0's
// buffers.  Not on the hot path; used for roofline calibration.
//   0/1/2  triad b += a over G floats, 3/4/8 blocks per SM (EF's access pattern)
//   3      write-only zero fill of G floats (decode's access pattern)
//   4      EF, no emission, no owed zeros        5  EF + candidate emission
//   6      EF + emission + owed zeros (zero map of the last AR/AG step)
int fc_diag_kernel_ms(fc_ctx* c, int which, int iters, double* ms_out) {
  if (!c || !ms_out || iters < 1) return fail(FC_ERR_INVALID_ARGUMENT, "bad argument");
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize_all(c));
  Worker& w = c->w[0];
  const uint64_t k = std::max<uint64_t>(1, c->kmax / 10);
  cudaEvent_t e0 = c->take_event(), e1 = c->take_event();
  double sum = 0.0;
  for (int it = 0; it < iters + 1; ++it) {
    if (which >= 4) CUDA_TRY(cudaMemsetAsync(w.ctl, 0, w.ctl_bytes, c->stream));  // work queue, bound
    fcb::Pending pz{};
    if (which == 6) pz.zmap = c->zmaps;
    cudaEventRecord(e0, c->stream);
    switch (which) {
      case 0: fcb::launch_triad(w.g_o, w.ge, c->G & ~uint64_t(3), 3, c->stream); break;
      case 1: fcb::launch_triad(w.g_o, w.ge, c->G & ~uint64_t(3), 4, c->stream); break;
      case 2: fcb::launch_triad(w.g_o, w.ge, c->G & ~uint64_t(3), 8, c->stream); break;
      case 3: fcb::launch_fill_zero(c->agg, c->G & ~uint64_t(3), 8, c->stream); break;
      case 4: fcb::launch_ef(w.g_o, w.ge, c->G, k, w.ctl, w.ws, pz, 1, 0, 0, nullptr, c->stream); break;
      case 5:
      case 6: fcb::launch_ef(w.g_o, w.ge, c->G, k, w.ctl, w.ws, pz, 1, 1, 1, nullptr, c->stream); break;
      default: return fail(FC_ERR_INVALID_ARGUMENT, "unknown diagnostic kernel");
    }
    LAUNCHED();
    cudaEventRecord(e1, c->stream);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it > 0) sum += ms;  // first launch is a warm-up
  }
  c->ev_pool.push_back(e0);
  c->ev_pool.push_back(e1);
  *ms_out = sum / iters;
  return FC_OK;
}

// Diagnostics for the NVLink calibration of the cost model: mean device time
// (CUDA events, this rank) of one NCCL collective on the context's comms:
//   0 broadcast of `bytes` from rank 0      1 ring allreduce of bytes/4 floats
//   2 tree allreduce of bytes/4 floats      3 allgather of `bytes` per rank
//   4 ART-Ring = broadcast(bytes) + ring allreduce(bytes)
//   5 ART-Tree = broadcast(bytes) + tree allreduce(bytes)
//   6 AG-compressed = allgather(2 * bytes)   (values + indices, cost_ag_compressed)
// All ranks must call with the same arguments (collective).
int fc_diag_collective_ms(fc_ctx* c, int which, uint64_t bytes, int iters, double* ms_out) {
  if (!c || !ms_out || iters < 1) return fail(FC_ERR_INVALID_ARGUMENT, "bad argument");
  if (!c->nccl) return fail(FC_ERR_INVALID_ARGUMENT, "needs an NCCL context");
  TRY(need_comm(c, "fc_diag_collective_ms"));
  const uint64_t cap = c->kmax * 4;  // bytes available in bidx / reduced / pack
  const uint64_t need = (which == 3 || which == 6) ? (which == 6 ? 2 * bytes : bytes) : bytes;
  if (need > 2 * cap || (which != 3 && which != 6 && bytes > cap) || bytes < 4)
    return fail(FC_ERR_INVALID_ARGUMENT, "message larger than the context's buffers");
  CUDA_TRY(cudaSetDevice(c->device));
  Worker& w = c->w[0];
  const size_t nf = bytes / 4;
  auto once = [&]() -> int {
    switch (which) {
      case 0: NCCL_TRY(ncclBroadcast(w.pack, c->bidx, nf, ncclUint32, 0, c->comm_ring, c->stream)); break;
      case 1: NCCL_TRY(ncclAllReduce(w.contrib, c->reduced, nf, ncclFloat32, ncclSum, c->comm_ring, c->stream)); break;
      case 2: NCCL_TRY(ncclAllReduce(w.contrib, c->reduced, nf, ncclFloat32, ncclSum, c->comm_tree, c->stream)); break;
      case 3: NCCL_TRY(ncclAllGather(w.pack, c->ag_recv, nf, ncclUint32, c->comm_ring, c->stream)); break;
      case 4:
      case 5:
        NCCL_TRY(ncclBroadcast(w.pack, c->bidx, nf, ncclUint32, 0, c->comm_ring, c->stream));
        NCCL_TRY(ncclAllReduce(w.contrib, c->reduced, nf, ncclFloat32, ncclSum,
                               which == 4 ? c->comm_ring : c->comm_tree, c->stream));
        break;
      case 6: NCCL_TRY(ncclAllGather(w.pack, c->ag_recv, 2 * nf, ncclUint32, c->comm_ring, c->stream)); break;
      default: return fail(FC_ERR_INVALID_ARGUMENT, "unknown collective");
    }
    return FC_OK;
  };
  for (int i = 0; i < 3; ++i) TRY(once());
  cudaEvent_t e0 = c->take_event(), e1 = c->take_event();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaEventRecord(e0, c->stream));
  for (int i = 0; i < iters; ++i) TRY(once());
  CUDA_TRY(cudaEventRecord(e1, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  c->ev_pool.push_back(e0);
  c->ev_pool.push_back(e1);
  *ms_out = ms / iters;
  return FC_OK;
}

// Diagnostics for the NVLink calibration of the cost model on the exchange
// the product actually runs (peer memory): mean device ms per exchange of
// k (index, value) pairs, this rank, all ranks calling alike (collective):
//   0 AG        every rank publishes its list; k_collect_packs pulls all N
//   1 ART-Ring  the root (rotating as STAR does) publishes; the others'
//               k_fetch_gather pulls the list, gathers g_e and pushes; N > 2
//               k_reduce_slice (reduce-scatter + allgather by stores)
//   2 ART-Tree  as 1, then k_reduce_root (reduce to the root + broadcast)
// each followed by the wait the peer decode performs before reading (the
// decode itself is compression-side work and is not timed).  The lists are
// spread index sets (sorted, k over [0, G)); the selects are replaced by a
// publish.  Without peer mappings the NCCL equivalents are timed
// (fc_diag_collective_ms 6 / 4 / 5 with 4k-byte messages).
int fc_diag_exchange_ms(fc_ctx* c, int which, uint64_t k, int iters, double* ms_out) {
  if (!c || !ms_out || iters < 1 || which < 0 || which > 2) return fail(FC_ERR_INVALID_ARGUMENT, "bad argument");
  if (!c->nccl || c->world < 2) return fail(FC_ERR_INVALID_ARGUMENT, "needs a multi-rank NCCL context");
  if (k < 1 || k > c->kmax || k > c->G) return fail(FC_ERR_INVALID_ARGUMENT, "k outside [1, min(kmax, G)]");
  if (!c->p2p) return fc_diag_collective_ms(c, which == 0 ? 6 : which == 1 ? 4 : 5, 4 * k, iters, ms_out);
  CUDA_TRY(cudaSetDevice(c->device));
  TRY(materialize_all(c));
  Worker& w = c->w[0];
  const int N = c->world;
  // this rank's list in both parities (+ its chunk bounds, as a select writes them)
  for (int q = 0; q < 2; ++q) {
    unsigned* lst = c->pb.list[c->rank] + q * c->pb.kmax;
    fcb::launch_spread_list(lst, k, c->G, (uint64_t)c->rank % std::max<uint64_t>(1, c->G / k), c->stream);
    fcb::launch_bounds(lst, k, 0, 1, c->G, c->pb.bounds[c->rank] + q * c->pb.nbs, c->stream);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  auto once = [&](int it) -> int {
    const unsigned long long epoch = ++c->epoch;
    const int par = (int)(epoch & 1);
    const int sel = it % N;
    // a fresh control block per exchange (its last-block counters)
    fcb::Ctl* next = take_ctl(w);
    CUDA_TRY(cudaMemsetAsync(next, 0, sizeof(fcb::Ctl), c->stream));
    if (which == 0) {
      fcb::launch_publish(c->pb, epoch, 1u, c->stream);
      fcb::launch_collect_packs(c->pb, par, epoch, k, c->ag_recv, c->bounds, c->stream);
    } else {
      const bool tree = which == 2, rs = !tree && N > 2;
      if (c->rank == sel) {
        fcb::launch_publish(c->pb, epoch, 3u, c->stream);  // list + its values (the contribution)
      } else {
        fcb::launch_fetch_gather(c->pb, sel, par, tree, epoch, w.ge, k, c->bounds, c->nch, w.ctl, nullptr,
                                 reinterpret_cast<unsigned long long*>(w.ws.g_part), c->stream);
      }
      if (rs) fcb::launch_reduce_slice(c->pb, par, epoch, k, 1, (float)N, sel, w.ctl, c->stream);
      if (tree && c->rank == sel)
        fcb::launch_reduce_root(c->pb, par, epoch, k, 1, (float)N, sel, c->dsel, w.ctl, c->stream);
      fcb::launch_wait_slot(c->pb, rs || tree ? 2 : 1, epoch, tree ? sel : -1, c->stream);
    }
    CUDA_TRY(cudaGetLastError());
    return FC_OK;
  };
  for (int i = 0; i < 3; ++i) TRY(once(i));
  cudaEvent_t e0 = c->take_event(), e1 = c->take_event();
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  TRY(check_errors(c));
  CUDA_TRY(cudaEventRecord(e0, c->stream));
  for (int i = 0; i < iters; ++i) TRY(once(3 + i));
  CUDA_TRY(cudaEventRecord(e1, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  TRY(check_errors(c));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  c->ev_pool.push_back(e0);
  c->ev_pool.push_back(e1);
  *ms_out = ms / iters;
  // the lists are no longer a selection: nothing may treat them as one
  for (auto& wk : c->w) wk.has_topk = false;
  c->has_agg = false;
  return FC_OK;
}

// Diagnostics: %globaltimer (ns) at k_select's phase boundaries in the last
// step of `worker` (block 0): start, staged, digit 1/2/3, counted, emitted, end.
int fc_diag_select_phases(fc_ctx* c, int worker, uint64_t* out12) {
  TRY(check_worker(c, worker));
  if (!out12) return fail(FC_ERR_INVALID_ARGUMENT, "null output");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpy(out12, &c->w[worker].ctl->tphase[0], 24 * sizeof(uint64_t),
                      cudaMemcpyDeviceToHost));
  return FC_OK;
}

int fc_diag_seg_phases(fc_ctx* c, int worker, uint64_t* out, int nmax, int* nseg) {
  TRY(check_worker(c, worker));
  if (!out || !nseg || nmax < 0) return fail(FC_ERR_INVALID_ARGUMENT, "bad output");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  Worker& w = c->w[worker];
  *nseg = 0;
  if (!c->h_seg || c->seg_groups == 0 || !w.seg_ctl[0]) return FC_OK;
  const int par = w.seg_par ^ 1;  // the parity the last layerwise step used
  int n = 0;
  for (int g = 0; g < c->seg_groups; ++g) {
    const fcb::SegTab& t = c->h_seg[((size_t)worker * 2 + par) * c->seg_groups + g];
    for (int q = 0; q < t.n && n < nmax; ++q, ++n) {
      // per segment: len, blocks, then 24 marks (select tphase[8],
      // tphase_ef[4], tphase_ef2[4], tphase_sx[8]) of its block 0
      uint64_t* o = out + (size_t)n * 26;
      o[0] = t.e[q].len;
      o[1] = t.e[q].nb;
      CUDA_TRY(cudaMemcpy(o + 2, &t.e[q].ctl->tphase[0], 24 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    }
  }
  *nseg = n;
  return FC_OK;
}

int fc_diag_ef_blocks(fc_ctx* c, int worker, uint64_t* out, int n) {
  TRY(check_worker(c, worker));
  if (!out || n < 0) return fail(FC_ERR_INVALID_ARGUMENT, "bad output");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  const int m = std::min<int>(n, 2 * (int)c->w[worker].ws.ef_grid);
  CUDA_TRY(cudaMemcpy(out, c->w[worker].ws.tblk, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  // followed by the last AR decode's start and end marks, then (n >= m + 8)
  // the peer exchange's: fetch-gather wait start / start / flag published,
  // decode wait start, reduce-slice start / flag published
  if (n >= m + 2) {
    unsigned long long t[8];
    fcb::read_tdiag(t);
    for (int i = 0; i < 8 && m + i < n; ++i) out[m + i] = t[i];
  }
  // then the peer gather's per-block (start, end) marks
  if (n > m + 8)
    CUDA_TRY(cudaMemcpy(out + m + 8, c->w[worker].ws.g_part, std::min<int>(n - m - 8, 4096) * sizeof(uint64_t),
                        cudaMemcpyDeviceToHost));
  return FC_OK;
}

// ------------------------------------------------------------ hot path -----

int fc_topk_exact(fc_ctx* c, int worker, double cr, fc_step_stats* st) {
  TRY(check_worker(c, worker));
  if (!cr_valid(cr)) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio must be in (0, 1]");
  const uint64_t k = k_of_host(cr, c->G);
  if (k > c->kmax) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio above the context's max_cr");
  CUDA_TRY(cudaSetDevice(c->device));
  // the packs are about to be rewritten: settle any zeros that reference them
  TRY(materialize_all(c));
  const uint64_t l0 = fcb::launches();
  c->phase_stats = st != nullptr;
  Worker& w = c->w[worker];
  const int force_fb = std::getenv("FC_FORCE_FALLBACK") != nullptr ? 2 : 0;
  record(c, 0);
  fcb::Ctl* next = take_ctl(w);
  TRY(wait_grad(c, worker));
  // the "error-fed" vector is the gradient itself (no residual added)
  const int e = fcb::launch_ef(nullptr, w.g_o, c->G, k, w.ctl, w.ws, fcb::Pending{}, 0, 1,
                               1 | force_fb, next, c->stream);
  if (e) return fail(FC_ERR_CUDA, std::string("k_ef launch: ") + cudaGetErrorString(static_cast<cudaError_t>(e)));
  TRY(grad_consumed(c, worker));
  LAUNCHED();
  record(c, 1);
  TRY(run_select(c, worker, k, w.g_o));
  record(c, 2);
  record(c, 3);
  record(c, 4);
  return finish_step(c, st, k, -1, -1, 4.0 * c->G + 16.0 * k, 0.0, l0);
}

int fc_artopk_step(fc_ctx* c, double cr, int mode, int algo, long step, int op, fc_step_stats* st) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (!cr_valid(cr)) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio must be in (0, 1]");
  if (mode != FC_STAR && mode != FC_VAR) return fail(FC_ERR_INVALID_ARGUMENT, "unknown selection mode");
  if (algo != FC_RING && algo != FC_TREE) return fail(FC_ERR_INVALID_ARGUMENT, "unknown reduce algo");
  if (op != FC_SUM && op != FC_AVG) return fail(FC_ERR_INVALID_ARGUMENT, "unknown reduce op");
  const uint64_t k = k_of_host(cr, c->G);
  if (k > c->kmax) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio above the context's max_cr");
  const int N = c->world;
  int sel = -1;
  if (mode == FC_STAR) {
    sel = static_cast<int>(step % N);  // select_star, inc/artopk.hpp:27-30
    if (sel < 0) return fail(FC_ERR_INVALID_ARGUMENT, "broadcast: bad source rank");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  const uint64_t l0 = fcb::launches();
  c->phase_stats = st != nullptr;
  for (auto& w : c->w) {
    w.has_topk = false;
    w.kept_is_topk = false;
    w.kept_vals = nullptr;
  }
  // STAR over peer memory: the selected rank's select publishes its list and
  // values in its exchange buffer (parity of this step's epoch), the other
  // ranks fetch the list and gather, and every rank's decode sums the
  // contributions in rank order straight from peer memory
  const bool p2p_star = c->p2p && N > 1;  // STAR and VAR
  const unsigned long long epoch = p2p_star ? ++c->epoch : 0;
  const int par = (int)(epoch & 1);

  if (!p2p_star) TRY(need_comm(c, "this step"));
  // in-place update of the aggregate (§3.5): ~2k whole-sector writes
  // (32 B each, scattered) against the 4G-byte dense write; the measured
  // break-even sets incr_div
  const bool incr_ok = !(c->flags & FC_FLAG_DENSE_DECODE) && c->nbuf == 1 && c->incr_div &&
                       k * c->incr_div <= c->G;
  bool early_clear = false;  // the previous support cleared before the exchange's waits
  bool aux_join = false;     // ... on s_aux: join before the write
  // (1) error feedback on every worker; Top-k where its result is consumed
  record(c, 0);
  for (int i = 0; i < c->n_local; ++i) {
    const bool topk = mode == FC_VAR || (c->rank + i) == sel;
    TRY(run_ef(c, i, k, topk));
  }
  advance_input(c);
  if (p2p_star && mode == FC_STAR && c->rank != sel && incr_ok && c->agg_incr && c->agg_support_k) {
    // a STAR rank that does not select waits for the selected rank's list
    // from here (~its select): the previous support's sectors are zeroed in
    // that wait -- all of them (this step's list is not known yet; the write
    // rewrites its own sectors after)
    int ob0 = 0;
    TRY(agg_target(c, &ob0));
    fcb::launch_agg_clear(c->agg_support, c->agg_support_k, nullptr, 0, nullptr, c->agg_buf[ob0], c->G,
                          c->zmaps, c->stream);
    early_clear = true;
  }
  record(c, 1);
  for (int i = 0; i < c->n_local; ++i) {
    const bool topk = mode == FC_VAR || (c->rank + i) == sel;
    if (!topk) continue;
    if (p2p_star) {
      fcb::SelectMode m;
      m.publish = true;
      m.pb = c->pb;
      m.epoch = epoch;
      m.publish_contrib = mode == FC_STAR;  // VAR: contributions come from the gather
      TRY(run_select(c, i, k, nullptr, m, c->pb.list[c->rank] + par * c->pb.kmax,
                     c->pb.contrib[c->rank] + par * c->pb.kmax, c->pb.bounds[c->rank] + par * c->pb.nbs));
    } else {
      TRY(run_select(c, i, k));
    }
  }
  record(c, 2);

  // (2) VAR: allgather of N ||top-k||^2, argmax, ties -> lowest rank
  //     (select_var, inc/artopk.hpp:35-48)
  if (mode == FC_VAR && N == 1) sel = 0;  // argmax over one worker
  const bool var_device = mode == FC_VAR && N > 1 && c->nccl;  // winner found on the device
  const bool p2p_var = p2p_star && mode == FC_VAR;
  c->sel_on_device = var_device;
  if (mode == FC_VAR && N > 1 && !c->nccl) {
    for (int i = 0; i < N; ++i)
      CUDA_TRY(cudaMemcpyAsync(c->h_norms + i, &c->w[i].ctl->topk_norm2, sizeof(double),
                               cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    sel = 0;
    for (int r = 1; r < N; ++r)
      if (c->h_norms[r] > c->h_norms[sel]) sel = r;
  }


  // (3) broadcast of the selected index set, gather, allreduce of the k
  //     values (artopk.hpp:87-104); the zeros at bidx become owed zeros
  const unsigned* bsrc = nullptr;
  const float* contrib0 = nullptr;
  const unsigned* own_bounds = nullptr;  // chunk bounds of bsrc, when a local select wrote them
  if (p2p_star) {
    Worker& w = c->w[0];
    if (p2p_var || c->rank != sel) {  // VAR: every rank (winner found on the device)
      fcb::launch_fetch_gather(c->pb, p2p_var ? -1 : sel, par, algo == FC_TREE, epoch, w.ge, k, c->bounds,
                               c->nch, w.ctl,
                               p2p_var ? c->dsel : nullptr, reinterpret_cast<unsigned long long*>(w.ws.g_part),
                               c->stream);
      w.kept_vals = c->pb.contrib[c->rank] + par * c->pb.kmax;  // ||kept||^2 on demand
      w.kept_k = k;
      own_bounds = c->bounds;  // the selected list's bounds, pulled
    } else {
      w.kept_is_topk = true;
      own_bounds = c->pb.bounds[c->rank] + par * c->pb.nbs;  // written by the local select
    }
    LAUNCHED();
    bsrc = c->pb.list[c->rank] + par * c->pb.kmax;  // local copy of the selected list
    // the previous support needs no exchanged value: clear it now, while
    // this rank waits for its peers (the selected rank for the others'
    // contributions, the others for the root's or the peer's values).  An
    // ART-Ring rank that reduces a slice for the others has no such window
    // on its stream (the clear would delay its slice, hence everyone's
    // decode: N = 4 0.525 ms): it clears on the auxiliary stream beside
    // the slice kernel
    const bool ring_slice = algo != FC_TREE && N > 2 && (mode == FC_VAR || c->rank != sel);
    if (incr_ok && c->agg_incr && c->agg_support_k && !early_clear) {
      int ob0 = 0;
      TRY(agg_target(c, &ob0));
      if (!ring_slice) {
        fcb::launch_agg_clear(c->agg_support, c->agg_support_k, bsrc, k, own_bounds, c->agg_buf[ob0], c->G,
                              c->zmaps, c->stream);
      } else {
        // beside the reduce-scatter slice (an NVLink-bound kernel), on the
        // auxiliary stream; the write joins it after the waits
        CUDA_TRY(cudaEventRecord(c->ev_fork, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->s_aux, c->ev_fork, 0));
        fcb::launch_agg_clear(c->agg_support, c->agg_support_k, bsrc, k, own_bounds, c->agg_buf[ob0], c->G,
                              c->zmaps, c->s_aux);
        CUDA_TRY(cudaEventRecord(c->ev_join, c->s_aux));
        aux_join = true;
      }
      early_clear = true;
    }
  } else if (c->nccl && N == 1) {
    // a single rank: broadcast and allreduce are identities
    Worker& w = c->w[0];
    bsrc = w.pack;
    contrib0 = reinterpret_cast<const float*>(w.pack + k);
    w.kept_is_topk = true;
    own_bounds = c->bounds;
  } else if (var_device) {
    // VAR: allgather of the N scores, winner on the device, its list
    // broadcast as a sum-allreduce of (winner ? list : 0); every rank
    // gathers g_e at the list (the winner's gather returns its own values)
    Worker& w = c->w[0];
    NCCL_TRY(ncclAllGather(&w.ctl->topk_norm2, c->dnorms, 1, ncclFloat64, c->comm_ring, c->stream));
    unsigned* masked = reinterpret_cast<unsigned*>(w.contrib);
    fcb::launch_var_mask(c->dnorms, N, c->rank, w.pack, k, masked, c->dsel, c->stream);
    LAUNCHED();
    NCCL_TRY(ncclAllReduce(masked, c->bidx, k, ncclUint32, ncclSum, c->comm_ring, c->stream));
    bsrc = c->bidx;
    fcb::launch_gather(bsrc, k, w.ge, w.contrib, w.ctl, w.ws.g_part, c->bounds, c->nch, c->stream);
    LAUNCHED();
    contrib0 = w.contrib;
    own_bounds = c->bounds;
    NCCL_TRY(ncclAllReduce(contrib0, c->reduced, k, ncclFloat32, ncclSum,
                           algo == FC_TREE ? c->comm_tree : c->comm_ring, c->stream));
  } else if (c->nccl) {
    Worker& w = c->w[0];
    NCCL_TRY(ncclBroadcast(w.pack, c->bidx, k, ncclUint32, sel, c->comm_ring, c->stream));
    bsrc = c->bidx;
    if (c->rank == sel) {
      // the selected worker's contribution is its own top-k values
      contrib0 = reinterpret_cast<const float*>(w.pack + k);
      w.kept_is_topk = true;
      own_bounds = c->bounds;
    } else {
      // the gather also writes the decode's chunk bounds of the broadcast list
      fcb::launch_gather(bsrc, k, w.ge, w.contrib, w.ctl, w.ws.g_part, c->bounds, c->nch, c->stream);
      LAUNCHED();
      contrib0 = w.contrib;
      own_bounds = c->bounds;
    }
    NCCL_TRY(ncclAllReduce(contrib0, c->reduced, k, ncclFloat32, ncclSum,
                           algo == FC_TREE ? c->comm_tree : c->comm_ring, c->stream));
  } else {
    bsrc = c->w[sel].pack;
    own_bounds = c->bounds + (uint64_t)sel * (c->nch + 1);
    for (int i = 0; i < c->n_local; ++i) {
      Worker& w = c->w[i];
      if (i == sel) {
        // g_e at its own top-k indices are its top-k values
        contrib0 = reinterpret_cast<const float*>(w.pack + k);
        w.kept_is_topk = true;
        if (N > 1)
          CUDA_TRY(cudaMemcpyAsync(w.contrib, contrib0, k * sizeof(float), cudaMemcpyDeviceToDevice,
                                   c->stream));
        continue;
      }
      fcb::launch_gather(bsrc, k, w.ge, w.contrib, w.ctl, w.ws.g_part, nullptr, 0, c->stream);
      LAUNCHED();
    }
  }
  record(c, 3);

  // (4) densify (core.hpp:72-81); /N for Avg (collectives.hpp:85-87)
  const float* lists = (c->nccl || N == 1) ? (N == 1 ? contrib0 : c->reduced) : c->contrib_all;
  const int nlists = c->nccl ? 1 : N;
  const uint64_t lstride = c->nccl ? 0 : c->kmax;
  int ob = 0;
  TRY(agg_target(c, &ob));
  float* aggw = c->agg_buf[ob];
  if (p2p_star) {
    // ART-Ring, N > 2: reduce-scatter (each rank sums its slice of the list
    // from every rank's contribution, rank order) and an allgather by NVLink
    // stores into every rank's reduced area; two ranks: the decode sums both
    // contributions directly (one fewer launch).  ART-Tree: reduce to the
    // root (the selected rank), which broadcasts the reduced list.  Both sum
    // in rank order, bit-exact with the reference (collectives.hpp:82-87).
    const bool tree = algo == FC_TREE;
    const bool rs = !tree && N > 2;
    if (rs)
      fcb::launch_reduce_slice(c->pb, par, epoch, k, op == FC_AVG, (float)N, mode == FC_STAR ? sel : -1,
                               c->w[0].ctl, c->stream);
    if (tree && (mode == FC_VAR || c->rank == sel))  // (VAR: only the winner works; found on the device)
      fcb::launch_reduce_root(c->pb, par, epoch, k, op == FC_AVG, (float)N, mode == FC_STAR ? sel : -1, c->dsel,
                              c->w[0].ctl, c->stream);
    const int wait_root = tree ? (mode == FC_STAR ? sel : -2) : -1;
    if (aux_join) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    if (incr_ok && c->agg_incr) {
      fcb::launch_agg_update_peers(c->pb, par, epoch, c->agg_support, early_clear ? 0 : c->agg_support_k, bsrc, k,
                                   own_bounds,
                                   op == FC_AVG, (float)N, rs || tree, aggw, c->G, c->zmaps, c->agg_support_next,
                                   wait_root, c->dsel, c->stream);
      std::swap(c->agg_support, c->agg_support_next);
    } else {
      fcb::launch_decode_ar_peers(c->pb, par, epoch, bsrc, own_bounds, k, op == FC_AVG, (float)N, rs || tree,
                                  aggw, c->G, c->zmaps, wait_root, c->dsel, c->stream);
      if (incr_ok)
        CUDA_TRY(cudaMemcpyAsync(c->agg_support, bsrc, k * sizeof(unsigned), cudaMemcpyDeviceToDevice,
                                 c->stream));
    }
  } else if (incr_ok && c->agg_incr) {
    // in place: zero the previous support, write this one (same dense content)
    if (!own_bounds) {
      fcb::launch_bounds(bsrc, k, 0, 1, c->G, c->bounds, c->stream);
      own_bounds = c->bounds;
    }
    fcb::launch_agg_update(c->agg_support, c->agg_support_k, bsrc, k, own_bounds, lists, nlists, lstride,
                           op == FC_AVG, (float)N, aggw, c->G, c->zmaps, c->agg_support_next, c->stream);
    std::swap(c->agg_support, c->agg_support_next);
  } else {
    if (!own_bounds) {
      fcb::launch_bounds(bsrc, k, 0, 1, c->G, c->bounds, c->stream);
      own_bounds = c->bounds;
    }
    fcb::launch_decode_ar(bsrc, own_bounds, lists, nlists, lstride, op == FC_AVG, (float)N, aggw,
                          c->G, c->zmaps, c->stream);
    if (incr_ok)
      CUDA_TRY(cudaMemcpyAsync(c->agg_support, bsrc, k * sizeof(unsigned), cudaMemcpyDeviceToDevice,
                               c->stream));
  }
  LAUNCHED();
  c->agg_incr = incr_ok;
  c->agg_support_k = incr_ok ? k : 0;
  record(c, 4);
  c->has_agg = true;
  TRY(agg_written(c, ob));
  for (auto& w : c->w) {  // every worker owes zeros at the broadcast indices
    w.pz.zmap = c->zmaps;
    w.pz_idx = bsrc;
    w.pz_k = k;
  }

  const double nl = c->n_local;
  const double hbm = nl * 12.0 * c->G + 4.0 * c->G + 32.0 * k * (mode == FC_VAR ? nl : 1.0) +
                     (mode == FC_VAR ? 8.0 * N : 0.0);
  const double bus = N > 1 ? 4.0 * k + 2.0 * (N - 1) / N * 4.0 * k + (mode == FC_VAR ? 8.0 * (N - 1) : 0.0)
                           : 0.0;
  return finish_step(c, st, k, sel, algo == FC_TREE ? 2 : 1, hbm, bus, l0);
}

int fc_ag_step(fc_ctx* c, double cr, int compressor, fc_step_stats* st) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (!cr_valid(cr)) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio must be in (0, 1]");
  if (compressor != FC_EXACT && compressor != FC_LAYERWISE && compressor != FC_THRESHOLD)
    return fail(FC_ERR_INVALID_ARGUMENT, "unknown compressor");
  // topk_layerwise without a layer map is topk_exact (compress.hpp:68)
  if (compressor == FC_LAYERWISE && c->layer_off.empty()) compressor = FC_EXACT;
  const uint64_t k = k_of_host(cr, c->G);
  uint64_t kk = k;  // per-worker selection size when it is the same on every worker
  if (compressor == FC_LAYERWISE) {
    kk = 0;
    for (uint64_t len : c->layer_len) kk += k_of_host(cr, len);
  }
  if (kk > c->kmax) return fail(FC_ERR_INVALID_ARGUMENT, "compression ratio above the context's max_cr");
  const int N = c->world;
  CUDA_TRY(cudaSetDevice(c->device));
  const uint64_t l0 = fcb::launches();
  c->phase_stats = st != nullptr;

  if (!(c->p2p && compressor == FC_EXACT && N > 1)) TRY(need_comm(c, "this AG step"));
  // (1) error feedback + compression per worker (compress.hpp:114-130)
  // (the threshold select reads per-chunk candidate slots: unpacked layout)
  for (auto& w : c->w) w.ws.batch = compressor == FC_THRESHOLD ? 1u : fcb::ef_batch(c->nch, w.ws.ef_grid);
  record(c, 0);
  std::vector<uint64_t> kr(N, kk);  // selection size of every rank
  std::vector<uint64_t> mine(c->n_local, kk);
  for (int i = 0; i < c->n_local; ++i) TRY(run_ef(c, i, k, compressor != FC_LAYERWISE));
  advance_input(c);
  record(c, 1);
  // Exact AG over peer memory: each rank's select publishes its list, values
  // and chunk bounds in its exchange buffer; one pull kernel replaces the
  // allgather and k_bounds
  const bool p2p_ag = c->p2p && compressor == FC_EXACT && N > 1;
  const unsigned long long epoch = p2p_ag ? ++c->epoch : 0;
  const int par = (int)(epoch & 1);
  for (int i = 0; i < c->n_local; ++i) {
    if (compressor == FC_EXACT && p2p_ag) {
      fcb::SelectMode m;
      m.publish = true;
      m.pb = c->pb;
      m.epoch = epoch;
      TRY(run_select(c, i, k, nullptr, m, c->pb.list[c->rank] + par * c->pb.kmax,
                     c->pb.contrib[c->rank] + par * c->pb.kmax, c->pb.bounds[c->rank] + par * c->pb.nbs));
      c->w[i].kept_is_topk = true;
    } else if (compressor == FC_EXACT) {
      TRY(run_select(c, i, k));
      c->w[i].kept_is_topk = true;
    } else if (compressor == FC_LAYERWISE) {
      TRY(run_layerwise(c, i, cr, kk));
    } else {
      TRY(run_threshold(c, i, k, &mine[i]));
    }
  }
  record(c, 2);

  // (2) allgather of the (index, value) pairs (collectives.hpp:39-56)
  const unsigned* packs;
  uint64_t stride, voff;  // between ranks' lists; from a list's indices to its values
  bool local_bounds = compressor == FC_EXACT;  // bounds written by the local selects
  if (compressor == FC_THRESHOLD) {
    if (!c->nccl) {
      for (int r = 0; r < N; ++r) kr[r] = mine[r];
    } else if (N == 1) {
      kr[0] = mine[0];
    } else {
      // sizes differ per rank: exchange them, then allgather padded lists
      double* dk = c->dnorms + N;
      double* dks = c->dnorms + N + 2;
      const double mk = (double)mine[0];
      CUDA_TRY(cudaMemcpyAsync(dk, &mk, sizeof(double), cudaMemcpyHostToDevice, c->stream));
      NCCL_TRY(ncclAllGather(dk, dks, 1, ncclFloat64, c->comm_ring, c->stream));
      CUDA_TRY(cudaMemcpyAsync(c->h_norms, dks, N * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(cudaStreamSynchronize(c->stream));
      for (int r = 0; r < N; ++r) kr[r] = (uint64_t)c->h_norms[r];
    }
    kk = *std::max_element(kr.begin(), kr.end());
  }
  if (p2p_ag) {
    fcb::launch_collect_packs(c->pb, par, epoch, kk, c->ag_recv, c->bounds, c->stream);
    LAUNCHED();
    packs = c->ag_recv;
    stride = 2 * kk;
    voff = kk;
    local_bounds = true;  // collected with the lists
  } else if (c->nccl && N == 1) {
    packs = c->w[0].pack;  // allgather over one rank: identity
    stride = 2 * c->kmax;
    voff = compressor == FC_THRESHOLD ? c->kmax : kk;
  } else if (c->nccl) {
    Worker& w = c->w[0];
    if (compressor == FC_THRESHOLD) {
      // [idx kmax | val kmax] -> [idx kk | val kk] (padding is never read:
      // the decode only visits each list's first kr[r] entries)
      CUDA_TRY(cudaMemcpyAsync(w.contrib, w.pack + c->kmax, mine[0] * sizeof(float),
                               cudaMemcpyDeviceToDevice, c->stream));
      CUDA_TRY(cudaMemcpyAsync(w.pack + kk, w.contrib, mine[0] * sizeof(float), cudaMemcpyDeviceToDevice,
                               c->stream));
    }
    NCCL_TRY(ncclAllGather(w.pack, c->ag_recv, 2 * kk, ncclUint32, c->comm_ring, c->stream));
    packs = c->ag_recv;
    stride = 2 * kk;
    voff = kk;
    local_bounds = false;
  } else {
    packs = c->pack_all;
    stride = 2 * c->kmax;
    voff = compressor == FC_THRESHOLD ? c->kmax : kk;
  }
  record(c, 3);

  // (3) rank-ordered scatter-add, every element / N (artopk.hpp:151-159)
  if (!local_bounds) {
    if (compressor == FC_THRESHOLD) {
      for (int r = 0; r < N; ++r)
        fcb::launch_bounds(packs + (uint64_t)r * stride, kr[r], 0, 1, c->G,
                           c->bounds + (uint64_t)r * (c->nch + 1), c->stream);
    } else {
      fcb::launch_bounds(packs, kk, stride, N, c->G, c->bounds, c->stream);
    }
  }
  int ob = 0;
  TRY(agg_target(c, &ob));
  fcb::launch_decode_ag(packs, stride, voff, N, c->bounds, (float)N, c->agg_buf[ob], c->G, c->zmaps,
                        c->nccl ? c->rank : 0, c->n_local, c->stream);
  LAUNCHED();
  c->agg_incr = false;  // the aggregate's support is now a union of N lists
  record(c, 4);
  c->has_agg = true;
  TRY(agg_written(c, ob));
  // residual_update (compress.hpp:122-130): g_e - g_e = +0 at own indices
  for (int i = 0; i < c->n_local; ++i) {
    const int r = c->nccl ? c->rank : i;
    Worker& w = c->w[i];
    w.pz.zmap = c->zmaps + (uint64_t)i * c->nch * 32;
    w.pz_idx = packs + (uint64_t)r * stride;
    w.pz_k = kr[r];
  }

  const double nl = c->n_local;
  const double hbm = nl * (12.0 * c->G + 8.0 * kk) + 4.0 * c->G + 12.0 * N * kk;
  const double bus = N > 1 ? (N - 1) * 8.0 * kk : 0.0;
  return finish_step(c, st, compressor == FC_THRESHOLD ? mine[0] : kk, -1, 0, hbm, bus, l0);
}

int fc_set_layer_map(fc_ctx* c, const uint64_t* offsets, const uint64_t* lengths, int nlayers) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (nlayers < 0 || (nlayers > 0 && (!offsets || !lengths)))
    return fail(FC_ERR_INVALID_ARGUMENT, "bad layer map");
  std::vector<uint64_t> off(offsets, offsets + nlayers), len(lengths, lengths + nlayers);
  for (int l = 0; l < nlayers; ++l) {
    if (len[l] == 0) return fail(FC_ERR_INVALID_ARGUMENT, "layer of length 0 (k_of needs G > 0)");
    if (off[l] + len[l] > c->G) return fail(FC_ERR_OUT_OF_RANGE, "layer beyond the gradient");
    if (l > 0 && off[l] < off[l - 1] + len[l - 1])
      return fail(FC_ERR_INVALID_ARGUMENT, "layers must be sorted and disjoint");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));  // a queued table upload is done
  if (c->h_small) {
    cudaFreeHost(c->h_small);
    c->h_small = nullptr;  // (d_small stays in the context's allocations; a new one is made)
  }
  c->small_cr = -1.0;
  c->seg_cr = -1.0;  // (tables rebuilt on the next layerwise step)
  c->layer_off = std::move(off);
  c->layer_len = std::move(len);
  return FC_OK;
}

int fc_set_threshold_rounds(fc_ctx* c, int rounds) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (rounds < 1) return fail(FC_ERR_INVALID_ARGUMENT, "rounds must be >= 1");  // compress.hpp:84
  if (rounds > 64) return fail(FC_ERR_INVALID_ARGUMENT, "at most 64 bisection rounds on B200");
  c->thresh_rounds = rounds;
  return FC_OK;
}

int fc_dense_step(fc_ctx* c, int algo, int op, fc_step_stats* st) {
  if (!c) return fail(FC_ERR_INVALID_ARGUMENT, "null context");
  if (algo != FC_RING && algo != FC_TREE) return fail(FC_ERR_INVALID_ARGUMENT, "unknown reduce algo");
  if (op != FC_SUM && op != FC_AVG) return fail(FC_ERR_INVALID_ARGUMENT, "unknown reduce op");
  const int N = c->world;
  TRY(need_comm(c, "the dense step"));
  CUDA_TRY(cudaSetDevice(c->device));
  const uint64_t l0 = fcb::launches();
  c->phase_stats = st != nullptr;
  record(c, 0);
  record(c, 1);
  record(c, 2);
  for (int i = 0; i < c->n_local; ++i) TRY(wait_grad(c, i));
  int ob = 0;
  TRY(agg_target(c, &ob));
  float* aggw = c->agg_buf[ob];
  if (c->nccl && N > 1) {
    // Avg inside the collective (ncclAvg): no extra pass over the 4G-byte
    // aggregate; NCCL's summation order makes this path 1e-5-relative, like
    // every NCCL allreduce here
    NCCL_TRY(ncclAllReduce(c->w[0].g_o, aggw, c->G, ncclFloat32, op == FC_AVG ? ncclAvg : ncclSum,
                           algo == FC_TREE ? c->comm_tree : c->comm_ring, c->stream));
    record(c, 3);
  } else {  // loopback, or a single NCCL rank (allreduce = identity)
    record(c, 3);
    fcb::launch_dense_sum(c->g_o_all, c->n_local, c->gstride, op == FC_AVG, (float)N, aggw, c->G,
                          c->stream);
  }
  for (int i = 0; i < c->n_local; ++i) TRY(grad_consumed(c, i));
  advance_input(c);
  CUDA_TRY(cudaGetLastError());
  c->agg_incr = false;
  record(c, 4);
  c->has_agg = true;
  TRY(agg_written(c, ob));
  const double bus = N > 1 ? 2.0 * (N - 1) / N * 4.0 * c->G : 0.0;
  return finish_step(c, st, c->G, -1, algo == FC_TREE ? 2 : 1, 12.0 * c->G, bus, l0);
}

}  // extern "C"
