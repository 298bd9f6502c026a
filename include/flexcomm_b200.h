/*
 * flexcomm_b200.h — C-ABI of the B200-native Top-k gradient-sync path.
 *
 * This is the drop-in boundary for the hot path of the reference
 * (arXiv 2312.02493, "flexcomm", /root/reference/proj/include/flexcomm).
 * The reference is header-only C++ with no FFI; its hot path is the pair
 *
 *   artopk_step(const Cluster&, const std::vector<DenseGrad>& g_o,
 *               ResidualStore&, CompressionRatio, SelectionMode, ReduceAlgo,
 *               long step, SelectionLog*, ReduceOp, double payload_scale)
 *                                           -- inc/artopk.hpp:62-111
 *   ag_step(const Cluster&, const std::vector<DenseGrad>&, ResidualStore&,
 *           CompressionRatio, CompressorKind, double, int)
 *                                           -- inc/artopk.hpp:128-161
 *
 * plus the pieces they call (error_feedback compress.hpp:114, topk_exact
 * compress.hpp:57, select_star/select_var artopk.hpp:27/35, the three
 * collectives collectives.hpp:39-94, densify core.hpp:72).  Every entry
 * point below names the reference symbol it replaces.  The C++ facade in
 * include/flexcomm_b200/ re-exposes the reference signatures on top of it
 * and re-throws the reference's exception types from the status codes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All functions return an fc_status;
 *    fc_last_error() gives a thread-local message for the last failure.
 *  - One host thread per context; calls are not reentrant.  Work is ordered
 *    on the context's CUDA stream; a step returns after completion unless
 *    FC_FLAG_ASYNC was given at creation.
 *  - The ABI owns every device buffer (gradients, residuals, aggregate,
 *    workspaces).  Host pointers passed in are caller-owned and only read /
 *    written during the call.  *_ptr() getters give zero-copy device
 *    pointers for callers whose gradients already live in HBM.
 *  - Values are fp32, indices uint32 (G < 2^31).  The reference is fp64 with
 *    size_t indices; the facade converts.
 */
#ifndef FLEXCOMM_B200_H_
#define FLEXCOMM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 1

/* Status codes.  The facade maps them onto the reference's exceptions
 * (inc/artopk.hpp:68-78, inc/core.hpp:49,91, inc/compress.hpp:20-29,140). */
typedef enum fc_status {
  FC_OK = 0,
  FC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  FC_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range    */
  FC_ERR_RUNTIME = 3,          /* std::runtime_error   */
  FC_ERR_CUDA = 4,             /* CUDA runtime failure (runtime_error)  */
  FC_ERR_NCCL = 5,             /* NCCL failure (runtime_error)          */
  FC_ERR_NO_DEVICE = 6         /* no sm_100 device: the path never falls back to CPU */
} fc_status;

/* inc/artopk.hpp:13 */
typedef enum fc_selection_mode { FC_STAR = 0, FC_VAR = 1 } fc_selection_mode;
/* inc/collectives.hpp:36 */
typedef enum fc_reduce_algo { FC_RING = 0, FC_TREE = 1 } fc_reduce_algo;
/* inc/collectives.hpp:35 */
typedef enum fc_reduce_op { FC_SUM = 0, FC_AVG = 1 } fc_reduce_op;
/* inc/artopk.hpp:113 (only Exact is on the path; the others are §8f "next") */
typedef enum fc_compressor { FC_EXACT = 0, FC_LAYERWISE = 1, FC_THRESHOLD = 2 } fc_compressor;
/* memory kind of a caller pointer */
/* FC_HOST_ASYNC: pinned host memory, the copy is queued on a copy engine and
 * the call returns at once.  Uploads (fc_set_grad) are ordered after the
 * previous step's error-feedback pass and before the next one; downloads
 * (fc_get_aggregate) after the step's decode and before the next decode, so
 * a caller can overlap step s's aggregate download with step s+1's gradient
 * upload (PCIe is full duplex).  Host data is valid after fc_sync(). */
typedef enum fc_memkind { FC_HOST = 0, FC_DEVICE = 1, FC_HOST_ASYNC = 2 } fc_memkind;

/* creation flags */
#define FC_FLAG_ASYNC 0x1u        /* do not synchronize at the end of a step      */
#define FC_FLAG_NO_TIMING 0x2u    /* skip per-phase CUDA events                   */
#define FC_FLAG_DENSE_DECODE 0x4u /* always rewrite the whole aggregate; otherwise
                                     AR steps at k <= G/80 update it in place (zero
                                     the previous support, write the new one), so
                                     callers must treat fc_aggregate_ptr() memory
                                     as read-only                                 */
#define FC_FLAG_PIPELINE 0x8u     /* host-fed pipelining: two gradient buffer sets
                                     and two aggregate buffers, so FC_HOST_ASYNC
                                     uploads for step s+1 and the download of step
                                     s-1 overlap step s (fc_grad_ptr / the
                                     aggregate pointer alternate between buffers;
                                     implies FC_FLAG_DENSE_DECODE)                */
#define FC_FLAG_NO_COOPERATIVE 0x10u /* launch the two grid-barrier kernels (error
                                     feedback, select) without the cooperative
                                     attribute: co-residency is then only checked
                                     against the static occupancy, and blocks kept
                                     off the GPU by other streams' kernels make the
                                     bounded barriers time out (reported as
                                     FC_ERR_RUNTIME) instead of the launch waiting */

#define FC_FLAG_PEER_ONLY 0x20u  /* one worker per process over peer memory WITHOUT
                                     NCCL (2 <= world <= 8, nccl_uid NULL): the
                                     caller exchanges the exchange-buffer handles
                                     (fc_peer_handle -> allgather -> fc_peer_attach);
                                     STAR / VAR AR-Top-k and exact AG only (several
                                     ranks may share a GPU, which NCCL forbids) */

#define FC_NCCL_UID_BYTES 128
#define FC_PEER_HANDLE_BYTES 64

typedef struct fc_opts {
  int device;           /* CUDA ordinal for this context                       */
  int n_local;          /* logical workers held by this context (loopback)     */
  int world;            /* total workers; == n_local for loopback              */
  int rank;             /* this context's first global rank                    */
  const unsigned char* nccl_uid; /* FC_NCCL_UID_BYTES, NULL => loopback          */
  uint64_t grad_len;    /* G, 1 <= G < 2^31                                     */
  double max_cr;        /* largest compression ratio that will be used (sizes
                           the k-length buffers); 0 => 1.0                     */
  unsigned flags;
} fc_opts;

/* Per-step statistics.  Phase times come from CUDA events on the context
 * stream (0 when FC_FLAG_NO_TIMING).  Byte counters are algorithmic bytes
 * (SURVEY §8d), not measured traffic. */
typedef struct fc_step_stats {
  int selected_rank;        /* ART: broadcasting worker; AG: -1               */
  int collective;           /* 0 AG, 1 ART_RING, 2 ART_TREE                    */
  uint64_t k;               /* k_of(c, G), inc/compress.hpp:28                 */
  float ms_total;           /* first kernel -> last kernel of the step         */
  float ms_ef;              /* error feedback (+ candidate emission)           */
  float ms_select;          /* threshold select + ordered compaction           */
  float ms_exchange;        /* VAR norm exchange, broadcast, gather, allreduce
                               or allgather                                    */
  float ms_decode;          /* dense decode                                    */
  double hbm_bytes;         /* algorithmic HBM bytes, this context             */
  double bus_bytes;         /* NCCL-tests bus bytes, this context              */
  uint64_t launches;        /* kernels this library launched for the step      */
  int fallback;             /* 1 if the sampled candidate bound missed         */
} fc_step_stats;

/* Per-worker numbers of the last step (gain inputs, VAR norm, threshold). */
typedef struct fc_worker_stats {
  double ge_norm2;          /* ||g_e||^2                                       */
  double kept_norm2;        /* sum of g_e^2 at the broadcast / own indices     */
  double topk_norm2;        /* ||top-k values||^2 (VAR score, artopk.hpp:41)   */
  uint32_t threshold_key;   /* |v| bit pattern of the k-th largest magnitude   */
  uint64_t candidates;      /* elements kept by the sampled candidate bound    */
  uint64_t count_above;     /* elements strictly above the threshold           */
  int fallback;
} fc_worker_stats;

typedef struct fc_ctx fc_ctx;

/* ---- status / library ---------------------------------------------------- */
const char* fc_status_string(int status);
const char* fc_last_error(void);
int fc_abi_version(void);
/* number of kernel launches since library load (all contexts) */
uint64_t fc_launch_count(void);

/* ---- sizing helpers (host) ------------------------------------------------ */
/* k = clamp(ceil(c*G - 1e-9), 1, G)                     inc/compress.hpp:28-33 */
int fc_k_of(double c, uint64_t grad_len, uint64_t* k_out);
/* round-robin selection: step % n                       inc/artopk.hpp:27-30   */
int fc_select_star(long step, int n, int* rank_out);

/* ---- lifetime -------------------------------------------------------------- */
/* ncclGetUniqueId; rank 0 calls it and ships the bytes to the other ranks.  */
int fc_get_unique_id(unsigned char uid_out[FC_NCCL_UID_BYTES]);
/* Loopback (nccl_uid == NULL): n_local logical workers on one device; the
 * collectives are in-HBM with the reference's rank-ascending order, so the
 * results are bit-identical to the fp32 oracle (the analogue of the
 * reference's in-process Cluster, inc/collectives.hpp:15-33).
 * NCCL (nccl_uid != NULL): one worker per context, world ranks; one
 * Ring-forced and one Tree-forced communicator are created. */
int fc_create(fc_ctx** out, const fc_opts* opts);
int fc_destroy(fc_ctx* ctx);
int fc_num_workers(const fc_ctx* ctx, int* n_local, int* world, int* rank);

/* ---- state I/O (mirrors std::vector<DenseGrad> g_o and ResidualStore) ------ */
/* worker is a LOCAL index in [0, n_local); out of range => FC_ERR_OUT_OF_RANGE
 * (ResidualStore::of uses vector::at, inc/core.hpp:91). */
int fc_set_grad(fc_ctx* ctx, int worker, const float* src, int memkind);
int fc_grad_ptr(fc_ctx* ctx, int worker, float** dev_ptr);
/* fp64 host buffers, as the reference holds them (DenseGrad::values is a
 * std::vector<double>, inc/core.hpp:60-70): converted to / from fp32 by a
 * small host thread pool through pinned staging chunks pipelined with the
 * copy engine (PCIe carries fp32).  fc_set_grad_f64 returns once the upload
 * is queued in FC_FLAG_ASYNC contexts (the step waits for it; src must stay
 * valid until fc_sync), otherwise once it landed; the getters return the
 * data (synchronous). */
int fc_set_grad_f64(fc_ctx* ctx, int worker, const double* src);
int fc_set_residual_f64(fc_ctx* ctx, int worker, const double* src);
int fc_get_residual_f64(fc_ctx* ctx, int worker, double* dst);
int fc_get_aggregate_f64(fc_ctx* ctx, double* dst);
int fc_fill_synthetic(fc_ctx* ctx, int worker, uint64_t seed, uint32_t rank, uint64_t step,
                      int dist);
int fc_set_residual(fc_ctx* ctx, int worker, const float* src, int memkind);
int fc_get_residual(fc_ctx* ctx, int worker, float* dst, int memkind);
int fc_residual_ptr(fc_ctx* ctx, int worker, float** dev_ptr);
int fc_reset_residuals(fc_ctx* ctx);
/* dense aggregate of the last step (identical on every worker) */
int fc_get_aggregate(fc_ctx* ctx, float* dst, int memkind);
int fc_aggregate_ptr(fc_ctx* ctx, float** dev_ptr);
/* last top-k computed for a worker: ascending indices and their values.
 * idx/val may be NULL to query k only. */
int fc_get_topk(fc_ctx* ctx, int worker, uint32_t* idx, float* val, uint64_t* k_out);
int fc_get_worker_stats(fc_ctx* ctx, int worker, fc_worker_stats* out);
/* checkpoint-restore of the residual store for the MOO controller's explore
 * (Trainer::snapshot/restore, inc/trainer.hpp:160-190; moo.hpp:205,232) */
int fc_snapshot(fc_ctx* ctx);
int fc_restore(fc_ctx* ctx);

/* ---- the hot path ---------------------------------------------------------- */
/* AR-Top-k step (Alg. 1).  Replaces flexcomm::artopk_step, inc/artopk.hpp:62.
 * mode FC_STAR|FC_VAR, algo FC_RING|FC_TREE, op FC_SUM|FC_AVG.
 * Per worker: g_e = g_o + residual (in place in the residual store), exact
 * top-k of |g_e| (ties -> lower index); the selected worker's index set is
 * broadcast; each worker gathers g_e at those indices and zeroes its
 * residual there; the k values are allreduced; the dense aggregate is
 * decoded.  selected rank in stats->selected_rank (stats may be NULL). */
int fc_artopk_step(fc_ctx* ctx, double cr, int mode, int algo, long step, int op,
                   fc_step_stats* stats);
/* AG-Top-k step.  Replaces flexcomm::ag_step, inc/artopk.hpp:128-161.
 * Per worker EF + compression (run_compressor, artopk.hpp:115-123) +
 * residual_update; allgather of the (index,value) pairs; rank-ordered
 * scatter-add; every element divided by N.  compressor:
 *   FC_EXACT      topk_exact (compress.hpp:57-65)
 *   FC_LAYERWISE  topk_layerwise (compress.hpp:67-79): exact Top-k_of(c, len)
 *                 per layer of the map set by fc_set_layer_map (none: exact)
 *   FC_THRESHOLD  topk_threshold (compress.hpp:81-112): bisection of a
 *                 magnitude threshold (fc_set_threshold_rounds rounds, 25 by
 *                 default); the selection size may differ from k and per
 *                 worker (stats->k = this context's first worker's). */
int fc_ag_step(fc_ctx* ctx, double cr, int compressor, fc_step_stats* stats);
/* DenseGrad::layer_map (inc/core.hpp:11-23) of the gradients, for
 * FC_LAYERWISE: nlayers (offset, length) pairs, sorted and disjoint, length
 * >= 1 (nlayers = 0 clears it). */
int fc_set_layer_map(fc_ctx* ctx, const uint64_t* offsets, const uint64_t* lengths, int nlayers);
/* ag_step's threshold_rounds (inc/artopk.hpp:131; >= 1, at most 64 here). */
int fc_set_threshold_rounds(fc_ctx* ctx, int rounds);
/* Dense baseline: allreduce of g_o, inc/trainer.hpp:240-244 */
int fc_dense_step(fc_ctx* ctx, int algo, int op, fc_step_stats* stats);
/* Stand-alone exact top-k of a worker's gradient buffer (no error feedback);
 * replaces flexcomm::topk_exact, inc/compress.hpp:57.  Read with fc_get_topk. */
int fc_topk_exact(fc_ctx* ctx, int worker, double cr, fc_step_stats* stats);

/* ---- host cost model (inc/costmodel.hpp, kept unchanged) ------------------ */
/* NetParams{alpha s, bandwidth bit/s} x MessageSpec{m_bytes, c, n}.
 * out8 = CostBreakdown in declaration order: ps, ring_ar, tree_ar, broadcast,
 * allgather_dense, ag_compressed, art_ring, art_tree (costmodel.hpp:42-52). */
int fc_cost_primitives(double alpha, double bandwidth, double m_bytes, double c, int n,
                       double* out8);
/* select_collective, costmodel.hpp:153-167: choice 0 AG, 1 ART_RING, 2 ART_TREE */
int fc_select_collective(double alpha, double bandwidth, double m_bytes, double c, int n,
                         int* choice, double* costs8);
/* prefer_ring_over_tree / _ring_over_ag / _tree_over_ag (which = 0/1/2),
 * costmodel.hpp:124-146 */
int fc_prefer(double alpha, double bandwidth, double m_bytes, double c, int n, int which,
              int* out);
/* crossover_cr, costmodel.hpp:180-203 (pair 0 ring/tree, 1 ring/AG, 2 tree/AG) */
int fc_crossover_cr(double alpha, double bandwidth, double m_bytes, int n, int pair,
                    double* c_out, int* has);
/* derive_m_from_ag, costmodel.hpp:171-175 */
int fc_derive_m_from_ag(double alpha, double bandwidth, double c, int n, double seconds,
                        double* m_out);

/* ---- adaptive-CR controller (inc/moo.hpp, kept unchanged) ------------------ */
/* CandidateCR, inc/moo.hpp:20-25 */
typedef struct fc_candidate {
  double c;
  double gain_avg;
  double t_comp_avg;     /* seconds */
  double t_sync_modeled; /* seconds */
} fc_candidate;
/* ControllerConfig, inc/moo.hpp:27-32 (defaults 0.001, 0.1, 3, 10, 0.10) */
typedef struct fc_controller_config {
  double c_low;
  double c_high;
  double factor;
  int probe_iters;
  double gain_threshold;
} fc_controller_config;
/* ControllerConfig::validate, inc/moo.hpp:34-41 */
int fc_controller_config_validate(const fc_controller_config* cfg);
/* round_3sig, inc/moo.hpp:44-48 */
int fc_round_3sig(double v, double* out);
/* candidate_ladder, inc/moo.hpp:52-65: writes min(cap, count) rungs */
int fc_candidate_ladder(const fc_controller_config* cfg, double* out, int cap, int* count);
/* trigger_gain, inc/moo.hpp:67-71, over the GainTracker window samples in
 * push order (inc/compress.hpp:145-165) */
int fc_trigger_gain(double gain_ref, const double* samples, uint64_t count, double threshold,
                    int* fire);
/* pareto_front, inc/moo.hpp:88-102: mask[i] = 1 iff candidate i is undominated */
int fc_pareto_front(const fc_candidate* cands, int m, int* mask);
/* choose_cr, inc/moo.hpp:111-146 over a front of m candidates: *chosen = index
 * of the knee, *collective = select_collective at its c (may be NULL) */
int fc_choose_cr(const fc_candidate* front, int m, double alpha, double bandwidth, double m_bytes,
                 int n, int* chosen, int* collective);
/* network_changed, inc/netsched.hpp:50-58 */
int fc_network_changed(double alpha0, double bandwidth0, double alpha1, double bandwidth1,
                       double rel_threshold, int* changed);
/* Per-step controller inputs after fc_artopk_step / fc_ag_step (the Trainer's
 * artopk_with_gain / ag_step_with_gain, inc/trainer.hpp:361-398, with the
 * 0.5 ns/element compression model of :346-359 replaced by measurement):
 *   gain   = mean over all N workers, in rank order, of
 *            AR: clamp(kept_norm2 / ge_norm2, 0, 1);  AG (ag != 0): topk_norm2 / ge_norm2
 *   t_comp = compression + decompression seconds of the step (ms_ef +
 *            ms_select + ms_decode of `stats`), max over ranks.
 * Under NCCL the per-rank values are allgathered so every rank returns the
 * same numbers.  A worker with ge_norm2 == 0 is FC_ERR_RUNTIME ("degenerate
 * gradient", inc/trainer.hpp:391-393, inc/compress.hpp:140).  Needs stats
 * recorded by the step (not FC_FLAG_NO_TIMING). */
int fc_moo_metrics(fc_ctx* ctx, int ag, const fc_step_stats* stats, double* gain,
                   double* t_comp_s);

/* NCCL contexts with 1 < world <= 8: 1 if every rank's exchange buffer is
 * mapped into every other (CUDA IPC over NVLink) and STAR / VAR / exact-AG
 * steps exchange through peer memory (broadcast + allreduce as a
 * fetch-gather that pushes contributions into the consumers' inboxes, an
 * NVLink reduce-scatter for N > 2, and a decode that reads local memory;
 * epochs in per-rank mailboxes; rank-ordered sums, bit-exact with the
 * reference), 0 if they use NCCL collectives (FC_NO_P2P=1 in the environment
 * forces that). */
int fc_peer_exchange(fc_ctx* ctx, int* enabled);

/* *in_place = 1 if the last AR-Top-k step left the aggregate as an in-place
 * update (the previous support's sectors zeroed, this step's sectors
 * rewritten: identical content, k <= G / 80 without FC_FLAG_DENSE_DECODE /
 * FC_FLAG_PIPELINE, single-process or NCCL exchange), 0 if it was rewritten
 * whole. */
int fc_aggregate_in_place(fc_ctx* ctx, int* in_place);
/* FC_FLAG_PEER_ONLY contexts: this rank's exchange-buffer handle, and the
 * attachment of every rank's (world x FC_PEER_HANDLE_BYTES, rank order,
 * allgathered by the caller -- e.g. over a torch.distributed gloo group).
 * Steps need the attachment; every rank attaches before the first step. */
int fc_peer_handle(fc_ctx* ctx, unsigned char out[FC_PEER_HANDLE_BYTES]);
int fc_peer_attach(fc_ctx* ctx, const unsigned char* handles);

/* Peer-exchange epoch waits give up after `seconds` (default 120): the
 * waiting kernel skips its remaining reads and the timeout is reported as
 * FC_ERR_RUNTIME by the next step call, fc_sync or fc_join (the report is
 * sticky across steps until returned once).  Every rank should use the same
 * value.  seconds > 0. */
int fc_set_peer_timeout(fc_ctx* ctx, double seconds);

/* Synchronize the context's streams (for FC_FLAG_ASYNC / FC_HOST_ASYNC users).
 * Returns FC_ERR_RUNTIME if a kernel of an earlier step reported a timeout
 * (grid barrier or peer wait); every step call (also under FC_FLAG_ASYNC)
 * and fc_join report timeouts of steps that have already finished. */
int fc_sync(fc_ctx* ctx);
/* Order the compute stream after every queued FC_HOST_ASYNC copy (so an event
 * recorded on fc_stream() afterwards covers them). */
int fc_join(fc_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), so callers can record their own
 * CUDA events around steps on the stream the kernels run on. */
int fc_stream(fc_ctx* ctx, void** stream_out);
/* Device time of the last N kernels named by the phase (diagnostics): the
 * library keeps CUDA-event timings of its dominant kernel (error feedback)
 * for the roofline computation in bench.py.  Returns mean ms per launch
 * since the last reset and the number of launches timed. */
int fc_ef_kernel_timing(fc_ctx* ctx, double* mean_ms, uint64_t* launches, int reset);
/* Time only every period-th EF launch (default 1).  The event pair around
 * the kernel keeps it from overlapping its neighbours' launch (programmatic
 * dependent launch), so sampling keeps the measurement off most steps. */
int fc_set_ef_timing_period(fc_ctx* ctx, int period);
/* Diagnostics (roofline calibration, not the hot path): mean device ms of one
 * kernel on worker 0's buffers.  which: 0/1/2 reference triad b += a at
 * 3/4/8 blocks per SM, 3 write-only fill, 4 EF, 5 EF + candidate emission,
 * 6 EF + emission + owed zeros. */
int fc_diag_kernel_ms(fc_ctx* ctx, int which, int iters, double* ms_out);
/* Diagnostics: %globaltimer (ns) at the select kernel's phase boundaries of
 * the last step (8 marks: start, window resolved, window bin, low digits,
 * look-back, emitted, written, end), then the EF kernel's (start, sample
 * barrier passed, bound derived, end of block 0's stream), then two EF marks
 * (sample histogrammed, flushed) and two spare, then 8 select sub-phase marks
 * (values loaded, window flushed, in-bin pass, indices staged, output
 * written, bounds fixed, 2 spare): out12 holds 24 values (block 0). */
int fc_diag_select_phases(fc_ctx* ctx, int worker, uint64_t* out12);
/* Layerwise segments of the last FC_LAYERWISE step (diagnostics): per
 * segment 26 words -- layer length, blocks, and the 24 phase marks of
 * fc_diag_select_phases from the segment's own control block; at most nmax
 * segments, their number in *nseg. */
int fc_diag_seg_phases(fc_ctx* ctx, int worker, uint64_t* out, int nmax, int* nseg);
/* Diagnostics: %globaltimer (ns) at the start and end of every EF block of the
 * last step (2 x grid values, grid = number of SMs), followed (as n allows) by
 * the last decode's start and end and the peer exchange's marks: fetch-gather
 * wait start, gather start, contribution published; decode wait start;
 * reduce-slice start, slice published (8 more values, stale for kernels the
 * last step did not run), then the peer gather's per-block (start, end). */
int fc_diag_ef_blocks(fc_ctx* ctx, int worker, uint64_t* out, int n);
/* Diagnostics (NVLink calibration): mean device ms of one NCCL collective on
 * this context's communicators, all ranks calling alike.  which: 0 broadcast,
 * 1 ring allreduce, 2 tree allreduce, 3 allgather (bytes per rank),
 * 4 ART-Ring (broadcast + ring allreduce of `bytes`), 5 ART-Tree,
 * 6 AG-compressed (allgather of 2*bytes per rank). */
int fc_diag_collective_ms(fc_ctx* ctx, int which, uint64_t bytes, int iters, double* ms_out);
/* Diagnostics (NVLink calibration on the product's own exchange): mean device
 * ms of one exchange of k (index, value) pairs through the kernels the steps
 * run -- which: 0 AG (list publish + k_collect_packs), 1 ART-Ring (list
 * publish + fetch-gather + reduce-scatter/allgather by NVLink stores), 2
 * ART-Tree (fetch-gather + reduce to the root + broadcast) -- up to the point
 * where the decode could start (the decode itself is not timed).  The lists
 * are spread index sets standing in for selections; afterwards the context
 * holds no top-k / aggregate (run a step next).  Collective over the ranks.
 * Without peer mappings the NCCL equivalents (fc_diag_collective_ms 6/4/5 at
 * 4k bytes) are timed. */
int fc_diag_exchange_ms(fc_ctx* ctx, int which, uint64_t k, int iters, double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* FLEXCOMM_B200_H_ */
