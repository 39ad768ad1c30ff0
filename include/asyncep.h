/*
 * asyncep.h -- C ABI of the B200-native AsyncEP MoE-layer hot path
 * (arxiv/paper_2605_02960, "MoE-Prefill", S6.2 "Asynchronous Expert Parallelism").
 *
 * What the library computes (S2.2): for every local token x_t,
 *     logits = W_r x_t  (fp32)   ->  top-k experts S_t (desc. logit, ties -> lower id)
 *     w_tj   = softmax over the k selected logits (== softmax -> top-k -> renormalise)
 *     y_t    = r_t + sum_j w_tj * W_down[S_tj] ( silu(W_gate[S_tj] x_t) * (W_up[S_tj] x_t) )
 * with the four steps (1) router GEMM + softmax + top-k, (2) local permute/dispatch,
 * (3) grouped expert GEMM gate/up -> SwiGLU -> down, (4) weighted combine, all on the
 * caller's compute stream.  Concurrently the NEXT layer's expert
 * weights, sharded 1/N per GPU by expert index, are AllGathered into a double-buffered
 * slot on the caller's comm stream, ordered against compute by CUDA events.
 * asyncep_saturation_T is Eq. 1 in the per-layer token form.
 *
 * Conventions
 *  - Every pointer named "device" is a CUDA device pointer on the current device; all
 *    device buffers and both streams are allocated and OWNED BY THE CALLER and must
 *    outlive the context.  The library owns only the context, its CUDA events and its
 *    TMA descriptors.  The NCCL communicator is BORROWED (never destroyed).
 *  - All compute entry points enqueue work and return; no host synchronisation.
 *  - Every call returns an asyncep_status; asyncep_last_error() returns a thread-local
 *    message for the last failure.  Degenerate inputs (num_tokens == 0) compute nothing
 *    (the gather schedule's bookkeeping still runs, see asyncep_moe_forward).
 *  - Not thread-safe per context; one context per GPU per process.
 *  - Data types: bf16 = IEEE bfloat16 (2 B); e4m3 = OCP FP8 E4M3FN (1 B); fp32.
 */
#ifndef ASYNCEP_H
#define ASYNCEP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASYNCEP_ABI_VERSION 1

#if defined(__GNUC__)
#define ASYNCEP_API __attribute__((visibility("default")))
#else
#define ASYNCEP_API
#endif

typedef struct asyncep_ctx asyncep_ctx; /* opaque, owned by the library */

typedef enum {
  ASYNCEP_OK = 0,
  ASYNCEP_ERR_INVALID_ARG = 1,   /* bad shape / alignment / null / range              */
  ASYNCEP_ERR_UNSUPPORTED = 2,   /* valid but not implemented (e.g. dtype, no GPU)      */
  ASYNCEP_ERR_CUDA = 3,          /* a CUDA runtime/driver call failed                    */
  ASYNCEP_ERR_NCCL = 4,          /* NCCL missing or a collective failed                  */
  ASYNCEP_ERR_NOT_PREFETCHED = 5,/* forward(l) without prefetch(l) (gathered layers)     */
  ASYNCEP_ERR_WORKSPACE = 6      /* num_tokens > max_tokens                              */
} asyncep_status;

typedef enum { ASYNCEP_BF16 = 0, ASYNCEP_FP8_E4M3 = 1 } asyncep_dtype;

/* Debug / test flags (asyncep_config.flags).  Default 0 = the production path. */
#define ASYNCEP_FLAG_IDENTITY_EXPERTS 0x1 /* skip the grouped GEMM: Y_perm = X_perm (plumbing pin)      */
#define ASYNCEP_FLAG_SIMT_GEMM        0x2 /* CUDA-core grouped GEMM instead of tcgen05 (sanitizer runs) */
#define ASYNCEP_FLAG_STAGE_TIMING     0x4 /* record CUDA events around each stage (asyncep_stage_times) */
#define ASYNCEP_FLAG_SIMT_ROUTER      0x8 /* CUDA-core router logits instead of tcgen05                */
#define ASYNCEP_FLAG_XPERM           0x10 /* materialise X_perm and TMA-load it: the default (kept as
                                               an explicit spelling; overrides FUSED_DISPATCH)      */
#define ASYNCEP_FLAG_OFFLOAD         0x20 /* NEXT-2: expert_shard[l] may be NULL for offloaded layers  */
#define ASYNCEP_FLAG_NO_SWAP_TAILS   0x40 /* compute every expert's last row tile as a padded 256-row
                                               tile (default: swap-AB tail tiles where they pay:
                                               both BF16 GEMMs, the FP8 gate/up GEMM; S6) */
#define ASYNCEP_FLAG_SWAP_TAILS      0x80 /* swap-AB tail tiles (<= 240 rows) in both GEMMs and both
                                               dtypes (A/B and tests)                               */
#define ASYNCEP_FLAG_FUSED_DISPATCH 0x200 /* the fused dispatch: GEMM1's cp.async warps gather the
                                               token rows through src_tok and X_perm is never
                                               written (default: the dispatch writes X_perm and
                                               GEMM1 TMA-loads it; S6: FP8 10-12 %, BF16
                                               0.3-3 % faster per step)                             */
#define ASYNCEP_FLAG_MX_ACT         0x100 /* FP8 experts: the intermediate is quantised MX-style (e4m3,
                                               one E8M0 power-of-two scale per 32 columns, DESIGN.md
                                               R6b) inside the gate/up GEMM's epilogue and the down
                                               GEMM runs block-scaled MMAs (kind::mxf8f6f4); no
                                               separate quantisation pass.  Default: per-row scales
                                               (R6).  Requires expert_dtype == ASYNCEP_FP8_E4M3.     */

typedef struct {
  int32_t num_layers;      /* L                                                         */
  int32_t num_experts;     /* E (E % world_size == 0)                                   */
  int32_t top_k;           /* k, 1 <= k <= min(E, 16)                                   */
  int32_t hidden;          /* H, multiple of 64                                         */
  int32_t ffn;             /* h (expert FFN width), multiple of 128                     */
  int32_t expert_dtype;    /* asyncep_dtype of the expert weights                       */
  int32_t world_size;      /* N ranks sharing the expert shards                         */
  int32_t rank;            /* r, 0 <= r < N                                             */
  int32_t replicate_layer0;/* 1: layer 0 is fully resident on every rank */
  int32_t norm_topk;       /* 1: renormalise the k weights (reading R1); 0: raw softmax */
  int64_t max_tokens;      /* upper bound on num_tokens per forward (workspace sizing)  */
  float   gamma;           /* Eq. 1 jitter margin, >= 1 (PAPER.md:319 default 1.2)      */
  int32_t flags;           /* ASYNCEP_FLAG_*                                            */
} asyncep_config;

/*
 * Packed expert layout (the shard / slot format).  One expert is one contiguous blob:
 *   BF16:  [ W_gu : 2h x H bf16 | W_down : H x h bf16 ]
 *   FP8 :  [ W_gu : 2h x H e4m3 | W_down : H x h e4m3 | s_gu : 2h fp32 | s_down : H fp32 ]
 * both matrices row-major with the contraction dim (K) contiguous ("K-major").  W_gu rows
 * are gate/up interleaved in groups of 16: in 256-row block b, the 32-row group g holds gate
 * rows j = 128b + 16g + [0, 16) followed by the matching up rows, so one 256-wide GEMM N-tile
 * holds matching gate and up columns (SwiGLU fuses into its epilogue) and, with the weights as
 * the MMA's M operand (swap-AB tail tiles), each 32-lane TMEM quadrant holds 16 gate rows and
 * their up rows.  FP8 scales are per output row (dequantised weight = code * scale).
 * A layer is E blobs in expert order; rank r's shard is experts [r*E/N, (r+1)*E/N),
 * so the rank-major AllGather of shards IS the layer.
 */
ASYNCEP_API size_t asyncep_expert_bytes(const asyncep_config* cfg);   /* bytes of one packed expert    */
ASYNCEP_API size_t asyncep_slot_bytes(const asyncep_config* cfg);     /* E * expert_bytes (one layer)  */
ASYNCEP_API size_t asyncep_shard_bytes(const asyncep_config* cfg);    /* (E/N) * expert_bytes          */
ASYNCEP_API size_t asyncep_workspace_size(const asyncep_config* cfg); /* device scratch for forward    */

/*
 * Pack natural-layout weights of `count` experts into packed blobs at `out` (device).
 *   BF16: gate, up : [count, h, H] bf16; down : [count, H, h] bf16 (device, contiguous);
 *         scales must be NULL.
 *   FP8 : gate, up, down are e4m3 codes in the same shapes; gate_scale, up_scale :
 *         [count, h] fp32, down_scale : [count, H] fp32.
 * Enqueued on `stream` (cudaStream_t, may be NULL = legacy default stream).
 */
ASYNCEP_API asyncep_status asyncep_pack_experts(const asyncep_config* cfg, int32_t count,
                                    const void* gate, const void* up, const void* down,
                                    const float* gate_scale, const float* up_scale,
                                    const float* down_scale, void* out, void* stream);

/*
 * Create a context.
 *  nccl_comm     : ncclComm_t borrowed from the caller (torch ProcessGroupNCCL._comm_ptr());
 *                  may be NULL when world_size == 1.
 *  compute_stream, comm_stream : cudaStream_t, caller-owned (comm_stream may be NULL when
 *                  world_size == 1).
 *  router_w      : [L] device pointers, each [E, H] bf16 (replicated on every rank).
 *  expert_shard  : [L] device pointers to this rank's packed shard of layer l
 *                  (asyncep_shard_bytes each), except layer 0 when replicate_layer0 == 1,
 *                  where it is the full packed layer (asyncep_slot_bytes).  When
 *                  world_size == 1 every entry is the full packed layer.
 *  slot0, slot1  : 2 device buffers of asyncep_slot_bytes (NULL allowed if world_size==1).
 *  workspace     : asyncep_workspace_size bytes of device memory, 256-B aligned.
 * Errors: INVALID_ARG on any shape/alignment violation, NCCL if world_size > 1 and NCCL
 * symbols cannot be resolved in the process, CUDA on runtime failures.
 */
ASYNCEP_API asyncep_status asyncep_init(const asyncep_config* cfg, void* nccl_comm, void* compute_stream,
                            void* comm_stream, const void* const* router_w,
                            const void* const* expert_shard, void* slot0, void* slot1,
                            void* workspace, asyncep_ctx** out);

/*
 * Issue the background AllGather of layer `layer`'s expert shards into slot[layer % 2]
 * on the comm stream ("MoE gatherer").  Waits (on the device) until the
 * slot's previous occupant (layer - 2) has finished its GEMMs; records ag_done[layer%2].
 * No-op (returns OK) when world_size == 1 or (layer == 0 and replicate_layer0).
 */
ASYNCEP_API asyncep_status asyncep_prefetch_layer(asyncep_ctx* ctx, int32_t layer);

/*
 * Test hook: like asyncep_prefetch_layer but without NCCL -- copies the N shards given in
 * `shards` ([N] device pointers, each asyncep_shard_bytes) rank-major into the slot with
 * device-to-device copies on the comm stream, under the same event ordering.  Lets the
 * double-buffer / event machinery run on one GPU.  Requires world_size > 1.
 */
ASYNCEP_API asyncep_status asyncep_prefetch_layer_local(asyncep_ctx* ctx, int32_t layer,
                                            const void* const* shards);

/*
 * ---- NEXT-2: hybrid weight offload (PAPER.md:343-349 "two-channel pipeline", :630 "H2D
 * offloader") ----
 * The expert shards of layers >= 1 live in pinned host memory (host_shards[l], asyncep_shard_bytes
 * each; the full layer, asyncep_slot_bytes, when world_size == 1); only a sliding window of w
 * device buffers (window[i], same size) holds upcoming shards.  asyncep_stage_layer(l) copies
 * layer l's shard host->device into window[l % w] on h2d_stream, after the window buffer's
 * previous occupant (layer l - w) has been read (by its AllGather, or by its forward when
 * world_size == 1), and records h2d_done.  asyncep_prefetch_layer(l) then gathers from the
 * window (waiting h2d_done on the comm stream); with world_size == 1 the forward reads the
 * window buffer directly.  Layer 0 stays resident (replicated) as before.
 * The two channels (NVLink gather of l+1, PCIe staging of l+2..l+w) run concurrently, and
 * t_EP = max(t_AG, t_H2D).  Pinned host memory and window buffers are caller-owned.
 */
ASYNCEP_API asyncep_status asyncep_enable_offload(asyncep_ctx* ctx, const void* const* host_shards,
                                                  void* const* window, int32_t w, void* h2d_stream);
ASYNCEP_API asyncep_status asyncep_stage_layer(asyncep_ctx* ctx, int32_t layer);

/*
 * Copy-engine gather (the alternative to NCCL for step 5): `shards` [num_layers * world_size]
 * holds, for every layer l and rank r, a device pointer (in this process's address space:
 * CUDA-IPC-mapped for r != rank) to rank r's shard of layer l (entries of resident layers are
 * ignored).  From then on asyncep_prefetch_layer fills the slot with cudaMemcpyAsync copies over
 * NVLink on the comm stream -- copy engines, no SMs, so the gather overlaps the persistent GEMMs
 * that occupy every SM (an SM-based NCCL AllGather can only run in their gaps, or on SMs left free
 * with ASYNCEP_RESERVE_SMS).  Same slot layout, events and ordering rules as the NCCL path.
 * NULL reverts to NCCL.  The pointed-to shards must stay mapped while the context is used.
 */
ASYNCEP_API asyncep_status asyncep_set_peer_shards(asyncep_ctx* ctx, const void* const* shards);

/*
 * Gather transport of asyncep_prefetch_layer (and the copy mode of asyncep_prefetch_layer_local):
 *  ASYNCEP_GATHER_COPY_KERNEL  copy kernel over the IPC-mapped peer shards, small CTAs that
 *                              co-reside with the persistent GEMMs (needs asyncep_set_peer_shards);
 *  ASYNCEP_GATHER_COPY_ENGINE  one cudaMemcpyAsync per 64 MiB chunk over the peer shards (the
 *                              copy engines for peers on other GPUs; no SMs);
 *  ASYNCEP_GATHER_NCCL         ncclAllGather on the borrowed communicator (north_star's path);
 *  -1                          default: copy (ASYNCEP_GATHER_COPY env: kernel, or ce / memcpy) when
 *                              peer shards are set, else NCCL.
 * reserve_sms: SMs the persistent grouped GEMMs leave free (for NCCL's SM-based kernels, which do
 * not fit beside a GEMM CTA); 0 = all SMs.  Errors: INVALID_ARG, NCCL (no communicator).
 */
#define ASYNCEP_GATHER_COPY_KERNEL 0
#define ASYNCEP_GATHER_COPY_ENGINE 1
#define ASYNCEP_GATHER_NCCL 2
ASYNCEP_API asyncep_status asyncep_set_gather_transport(asyncep_ctx* ctx, int32_t transport, int32_t reserve_sms);

/* Communicator of the NCCL gather (ASYNCEP_GATHER_NCCL): e.g. a dedicated one whose NCCL config
 * caps its kernels at the SMs the GEMMs leave free (maxCTAs = reserve_sms); NULL = the context's
 * communicator.  Borrowed: it must outlive its use.  Errors: INVALID_ARG, NCCL (no NCCL loaded). */
ASYNCEP_API asyncep_status asyncep_set_gather_comm(asyncep_ctx* ctx, void* nccl_comm);

/* Measurement knob: CTAs of the co-resident copy kernel (0 = default: ASYNCEP_GATHER_CTAS, else
 * 1 per SM).  More CTAs keep more warps beside the GEMMs; NVLink latency needs ~1 MB in flight. */
ASYNCEP_API asyncep_status asyncep_set_gather_copy_ctas(asyncep_ctx* ctx, int32_t ctas);

/*
 * Startup gather-bandwidth probe for Eq. 1's t_EP (T "computed once at startup
 * from hardware and model configuration"; reading R12): one full gather of `layer` (a gathered
 * layer whose slot is free) with the current transport on the comm stream, nothing else
 * running; returns its time (ms) and the bytes each rank received ((N-1) x shard bytes).  The
 * slot is handed back unconsumed.  With NCCL it is collective: every rank must call it.
 * shards: NULL (peer shards / NCCL) or, in the one-GPU emulation, the N local shards of `layer`.
 */
ASYNCEP_API asyncep_status asyncep_probe_gather(asyncep_ctx* ctx, int32_t layer, const void* const* shards,
                                                double* ms_out, double* bytes_out);

/* The gather's transport primitive, exposed for measurement: a device-to-device (or NVLink
 * peer) copy of `bytes` on `stream` by a copy kernel of small CTAs that co-reside with the
 * persistent GEMM CTAs (the driver's D2D memcpy and NCCL kernels cannot start beside them).
 * ASYNCEP_GATHER_COPY=memcpy (alias ce) selects one cudaMemcpyAsync per copy instead (copy
 * engines for peer pointers on another GPU). */
ASYNCEP_API asyncep_status asyncep_gather_copy(void* dst, const void* src, size_t bytes, void* stream);

/*
 * Test / measurement hook for asyncep_prefetch_layer_local: pace the copies of the OTHER
 * ranks' shards at `bytes_per_s` (0 = unpaced) to emulate the NVLink receive bandwidth of
 * an N-rank AllGather on one GPU.  Each 64 MiB chunk is preceded on the comm stream by a
 * one-thread kernel that spins for chunk_bytes / bytes_per_s.
 */
ASYNCEP_API asyncep_status asyncep_set_link_emulation(asyncep_ctx* ctx, double bytes_per_s);

/*
 * Gated gather (every transport; §6.2: the grouped-GEMM time is what hides the gather).
 * on != 0: asyncep_prefetch_layer(_local) validates and claims the slot but holds the gather on the
 * host; the NEXT asyncep_moe_forward on this context enqueues it once its dispatch is enqueued, with
 * the comm stream waiting for the compute stream to get there (an event), so the gather's HBM traffic
 * overlaps the grouped GEMMs rather than the HBM-bound combine / router / dispatch.  The layer's own
 * forward also releases it (before its wait for the slot).  on == 0 enqueues every held gather at
 * once.  The startup probe (asyncep_probe_gather) is never held.  Errors: INVALID_ARG (ctx NULL), or
 * those of the held prefetches when on == 0.
 */
ASYNCEP_API asyncep_status asyncep_set_gather_gate(asyncep_ctx* ctx, int32_t on);

/*
 * The MoE FFN forward of layer `layer` on the compute stream.
 *  x         : [num_tokens, H] bf16 device, 16-B aligned rows.
 *  residual  : nullable [num_tokens, H] bf16 device; added to the output (reading R9).
 *  y         : [num_tokens, H] bf16 device output; may alias residual but not x.
 *  topk_ids_out [num_tokens, k] int32, topk_w_out [num_tokens, k] fp32,
 *  expert_counts_out [E] int32 : nullable device outputs (router decisions, in the
 *                  canonical order: descending logit, ties -> lower expert id).
 * Gathered layers require a prior asyncep_prefetch_layer(layer) (else NOT_PREFETCHED).
 * num_tokens == 0 computes nothing (x / y may be NULL) but keeps the schedule: a gathered layer must
 * still have been prefetched, a held (gated) gather is started, and the slot is released in stream
 * order after its gather, as a DP rank with an empty batch still takes part in every AllGather.
 * num_tokens > max_tokens -> WORKSPACE.
 */
ASYNCEP_API asyncep_status asyncep_moe_forward(asyncep_ctx* ctx, int32_t layer, const void* x,
                                   int64_t num_tokens, const void* residual, void* y,
                                   int32_t* topk_ids_out, float* topk_w_out,
                                   int32_t* expert_counts_out);

/*
 * ---- Contrast baseline: synchronous DP x EP (Table 1 "DPxEP") ----
 * Rank r permanently owns experts [r*E/N, (r+1)*E/N) of every layer and computes them for
 * the tokens of ALL ranks: per layer, one AllToAll dispatches each rank's permuted rows to
 * the owners of their experts and a second returns the expert outputs, both ON the critical
 * path of the compute stream (versus AsyncEP's off-path weight gather).  BF16 experts only.
 *
 * asyncep_ep_plan (host, pure): from this rank's per-expert row counts (send_counts [E]) and
 * the counts other ranks send to it (recv_counts [E]: source-major, E/N per source), the row
 * ranges of the exchange; rows of every expert are padded to 256 (the GEMM pair tile):
 *   send_off[d], send_rows[d]  : rows of this rank's X_perm going to rank d
 *   recv_off[s], recv_rows[s]  : rows arriving from rank s in the receive buffer
 *   group_off [E+1]            : receive-side row offset of group g = s*(E/N) + local expert
 * Returns the total receive rows through recv_total.
 */
ASYNCEP_API asyncep_status asyncep_ep_plan(const asyncep_config* cfg, const int32_t* send_counts,
                                           const int32_t* recv_counts, int64_t* send_off, int64_t* send_rows,
                                           int64_t* recv_off, int64_t* recv_rows, int64_t* group_off,
                                           int64_t* recv_total);
/* device bytes of the EP receive workspace for up to max_recv_rows received rows */
ASYNCEP_API size_t asyncep_ep_workspace_size(const asyncep_config* cfg, int64_t max_recv_rows);
/*
 * One synchronous DP x EP layer forward (host-synchronous: the exchanged counts are read back
 * to size the variable AllToAlls, as an EP layer must).  Uses the context's NCCL communicator
 * (ncclSend/ncclRecv groups on the compute stream; a device copy when world_size == 1 and no
 * communicator is given) and this rank's shard of `layer`.  x, residual, y as in
 * asyncep_moe_forward.  ERR_WORKSPACE if more than max_recv_rows rows arrive.  num_tokens == 0
 * at world_size > 1 still joins both AllToAlls (no rows sent; rows received for this rank's
 * experts are computed and returned).
 */
ASYNCEP_API asyncep_status asyncep_ep_forward(asyncep_ctx* ctx, int32_t layer, const void* x, int64_t num_tokens,
                                              const void* residual, void* y, void* ep_workspace,
                                              int64_t max_recv_rows);

/*
 * Saturation threshold, Eq. 1 in per-layer form (readings R11, R12):
 *   t_AG = (N-1)/N * E*3*H*h*b / ag_bytes_per_s;  T_FLOPs = gamma * t_AG * flops_per_s;
 *   T_tok = T_FLOPs / (6*k*H*h)  [tokens per GPU per layer].
 * Pure function (no context); N == 1 gives 0.  Outputs may be NULL.
 */
ASYNCEP_API asyncep_status asyncep_saturation_T(const asyncep_config* cfg, double flops_per_s,
                                    double ag_bytes_per_s, double* tokens_per_gpu_out,
                                    double* flops_out);

/*
 * Stage timing (ASYNCEP_FLAG_STAGE_TIMING, cf. the paper's gated per-layer CUDA-event
 * hooks).  Synchronises on the recorded events and returns, summed
 * over all forwards since the last reset, the milliseconds of each stage:
 *   [0] router  [1] permute  [2] exposed gather wait  [3] GEMM1 gate/up+SwiGLU
 *   [4] GEMM2 down (FP8: with the intermediate's quantisation pass)  [5] combine
 *   (n_stages <= 6), and the number of forwards counted.
 */
ASYNCEP_API asyncep_status asyncep_stage_times(asyncep_ctx* ctx, double* ms_out, int32_t n_stages,
                                   int64_t* forwards_out);
ASYNCEP_API asyncep_status asyncep_reset_stage_times(asyncep_ctx* ctx);

/*
 * Per-forward wall time (ms, CUDA events around the whole forward) of the last recorded
 * forwards, oldest first, with their layer ids (ASYNCEP_FLAG_STAGE_TIMING).  Writes up to n
 * entries; returns the count through n_out.  Synchronises on the recorded events.
 */
ASYNCEP_API asyncep_status asyncep_forward_times(asyncep_ctx* ctx, double* ms_out, int32_t* layer_out, int32_t n,
                                                 int32_t* n_out);

/*
 * Event timeline of the schedule (the per-layer view an nsys trace would give; nsys is not part of
 * this toolchain): asyncep_timeline_begin records an epoch on the compute stream (the comm stream
 * waits for it), then every forward (ASYNCEP_FLAG_STAGE_TIMING) and every gather is recorded until
 * asyncep_timeline_read, which synchronises, writes up to n records in issue order -- forwards
 * first as they flush, then gathers -- and ends the capture; n_out = records available.
 *   FORWARD: t0 = start (router), t1 = dispatch done (the wait for the slot begins), t2 = GEMM1
 *            start (the wait ended), t3 = end (combine)
 *   GATHER : t0 = start of the layer's gather on the comm stream, t1 = t2 = t3 = its end (ag_done)
 * Times are ms since the epoch.  Errors: INVALID_ARG (no timing flag / no begin), CUDA.
 */
#define ASYNCEP_TL_FORWARD 0
#define ASYNCEP_TL_GATHER 1
typedef struct {
  int32_t kind;  /* ASYNCEP_TL_* */
  int32_t layer;
  float t0, t1, t2, t3;
} asyncep_timeline_rec;
ASYNCEP_API asyncep_status asyncep_timeline_begin(asyncep_ctx* ctx);
ASYNCEP_API asyncep_status asyncep_timeline_read(asyncep_ctx* ctx, asyncep_timeline_rec* out, int32_t n,
                                                 int32_t* n_out);

/*
 * Calibrated saturation threshold, App. B.4 Eq. 3:
 *   T = gamma * (t_e / t_c) * C_dummy  [FLOPs],  collapsing to gamma * C_dummy when t_e <= t_c,
 * with t_c = wall time of the resident layer 0 and t_e = max wall time of the gathered layers
 * in one profile pass at n_ref tokens, C_dummy = f_tok * n_ref.  Pure; outputs may be NULL.
 */
ASYNCEP_API asyncep_status asyncep_calibrated_T(double gamma, double t_e, double t_c, double c_dummy,
                                                double* flops_out);

/*
 * NEXT-1 profile-run calibration, App. B.4, end to end: from the last
 * num_layers recorded forwards of `ctx` (one profile pass of the stack at n_ref tokens per GPU,
 * ASYNCEP_FLAG_STAGE_TIMING), t_c = the wall time of layer 0 (resident: pure compute) and
 * t_e = the max wall time of the layers >= 1 (each max(compute, transfer)); f_tok = 2HE + 6kHh
 * (router + experts, per token per layer), C_dummy = f_tok * n_ref, and T by
 * asyncep_calibrated_T (gamma <= 0: the config's gamma).  Outputs: T in FLOPs and in tokens per
 * GPU (T / f_tok), t_c and t_e in ms (each nullable).  Synchronises on the recorded events.
 * Errors: INVALID_ARG (no timing flag, fewer than num_layers forwards recorded, layer 0 absent).
 */
ASYNCEP_API asyncep_status asyncep_calibrate_T(asyncep_ctx* ctx, double gamma, int64_t n_ref, double* flops_out,
                                               double* tokens_out, double* t_c_out, double* t_e_out);

/*
 * ---- NEXT-4: saturation-bounded admission (frontend consumer of T; host only) ----
 * Algorithm 1 (App. A) with the Eq. 2 cost and the load
 * band [T, T + Delta_last].  Functional forms of Eq. 2 (reading R18):
 *   C_pfx(n)   = n f_tok + 2 n^2 HL
 *   C_sfx(S,P) = S f_tok + 2 S^2 HL + 4 S P HL          (HL = hidden x attention layers)
 * Requests are block-hash chains (block_size tokens per hash; hashes[chain_off[q] ..
 * chain_off[q+1]) for request q), prefix_len / suffix_len in tokens.
 */
typedef struct asyncep_router asyncep_router;
typedef struct {
  int32_t num_gpus;   /* N data-parallel GPUs                                  */
  int32_t block_size; /* tokens per hashed block (e.g. 16)       */
  double f_tok;       /* FLOPs per token of the linear terms                   */
  double attn_hl;     /* hidden x attention layers (quadratic attention terms) */
  double T_flops;     /* saturation threshold T [FLOPs], e.g. T_tok * f_tok    */
} asyncep_router_config;
ASYNCEP_API double asyncep_cost_delta(const asyncep_router_config* cfg, int64_t P, int64_t M, int64_t S); /* NaN on bad args */
ASYNCEP_API asyncep_status asyncep_router_create(const asyncep_router_config* cfg, asyncep_router** out);
ASYNCEP_API asyncep_status asyncep_router_destroy(asyncep_router* r);
ASYNCEP_API asyncep_status asyncep_router_set_T(asyncep_router* r, double T_flops);
ASYNCEP_API asyncep_status asyncep_router_loads(const asyncep_router* r, double* loads_out); /* [num_gpus] */
/* One round of Algorithm 1 over n_req queued requests in arrival order.  reset_loads = 1
 * starts the round with L_i = 0 (Alg. 1 line 1); 0 carries loads over (App. B.2 mode).
 * gpu_out[q] = assigned GPU, or -1 when every GPU is saturated (the request stays queued);
 * delta_out[q] = the charged cost (nullable). */
ASYNCEP_API asyncep_status asyncep_router_schedule_round(asyncep_router* r, int32_t reset_loads, int64_t n_req,
                                                         const int64_t* chain_off, const uint64_t* hashes,
                                                         const int64_t* prefix_len, const int64_t* suffix_len,
                                                         int32_t* gpu_out, double* delta_out, int64_t* admitted_out);
/* engine events (App. B.3): stored blocks pending -> committed; progress decays L_i by tokens*f_tok */
ASYNCEP_API asyncep_status asyncep_router_blocks_stored(asyncep_router* r, int32_t gpu, const uint64_t* hashes,
                                                        int64_t n);
ASYNCEP_API asyncep_status asyncep_router_progress(asyncep_router* r, int32_t gpu, int64_t tokens);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: the data-parallel attention layer before each MoE layer, KV-cache-free
 * (PAPER.md:275 "pure DP attention"; :311 "after computing attention locally, each GPU
 * evaluates the current MoE layer"; :351-353 "disables KV storage entirely and computes
 * attention on the fly").  The paper fixes no attention architecture; reading R19
 * (S3) is the Qwen3-MoE block:
 *     xn   = RMSNorm(x; w_ln1)
 *     qkv  = xn . W_qkv^T                 W_qkv [(Hq + 2 Hkv) d, H]: q rows, then k, then v
 *     q_h  = RoPE(RMSNorm(q_h; w_qn)), k_g = RoPE(RMSNorm(k_g; w_kn))   (per head of d)
 *     o    = causal softmax(q k^T / sqrt(d)) v per prompt, query head h reads kv head
 *            h / (Hq / Hkv) (grouped-query attention); positions restart at 0 per prompt
 *     x'   = x + o . W_o^T                W_o [H, Hq d]
 *     xn2  = RMSNorm(x'; w_ln2)           (the input of the MoE layer's router and experts)
 * Rotary embedding: rotate-half, inv_freq_i = theta^(-2i/d).  All tensors bf16, row-major,
 * device, caller-owned; fp32 accumulation.  Nothing is stored beyond the call (no KV cache).
 * Prompts are packed: prompt b holds tokens [cu_seqlens[b], cu_seqlens[b+1]).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t hidden;      /* H (multiple of 256)                                   */
  int32_t q_heads;     /* Hq (multiple of kv_heads)                             */
  int32_t kv_heads;    /* Hkv                                                   */
  int32_t head_dim;    /* d: must be 128                                        */
  int64_t max_tokens;  /* workspace sizing                                      */
  int64_t max_prompts; /* workspace sizing (0 = max_tokens)                     */
  double eps;          /* RMSNorm epsilon (Qwen3: 1e-6)                         */
  double rope_theta;   /* Qwen3: 1e6                                            */
} asyncep_attn_config;

/* Workspace bytes asyncep_attn_layer needs (xn, qkv, q, k, V^T, o, projection output, counters). */
ASYNCEP_API size_t asyncep_attn_workspace_size(const asyncep_attn_config* cfg);

/*
 * The attention core alone (step 4 of the layer above), on `stream`:
 *  q  [T, Hq, d], k [T, Hkv, d] bf16 device;  cu_seqlens [B+1] int32 device, non-decreasing,
 *  cu_seqlens[0] = 0, cu_seqlens[B] = T;  vt [Hkv, d, ldv] bf16 device = V transposed per kv
 *  head, prompt b's keys at columns [vt_cu[b], vt_cu[b] + len_b) (vt_cu [B+1] int32 device,
 *  every vt_cu[b] a multiple of 8 -- the TMA start along the contiguous dimension must be
 *  16-B aligned; columns outside the prompts must hold finite values); ldv % 8 == 0;
 *  o [T, Hq, d] bf16 output;  sched: one int32 of caller-owned device memory for the kernel's
 *  dynamic work-item scheduler (zeroed by the call on `stream`; concurrent calls need their own).
 * Causal within each prompt.  T == 0 is a no-op.  Errors: INVALID_ARG (d != 128, Hq % Hkv,
 * alignment), CUDA.
 */
ASYNCEP_API asyncep_status asyncep_attention(const asyncep_attn_config* cfg, const void* q, const void* k,
                                             const void* vt, int64_t ldv, const int32_t* vt_cu,
                                             const int32_t* cu_seqlens, int32_t B, int64_t T, void* o,
                                             int32_t* sched, void* stream);

/*
 * One full attention layer (the formulas above), on `stream`.
 *  x [T, H] bf16 device; cu_seqlens [B+1] int32 device; weights bf16 device: w_ln1 [H],
 *  w_qkv [(Hq + 2 Hkv) d, H], w_qn [d], w_kn [d], w_o [H, Hq d], w_ln2 [H];
 *  x_out [T, H] = x' and xn2_out [T, H] = RMSNorm(x'; w_ln2) (both bf16 device outputs,
 *  neither may alias x); workspace of asyncep_attn_workspace_size bytes, 256-B aligned.
 * T > max_tokens or B > max_prompts -> WORKSPACE; T == 0 is a no-op.
 */
ASYNCEP_API asyncep_status asyncep_attn_layer(const asyncep_attn_config* cfg, const void* x, int64_t T,
                                              const int32_t* cu_seqlens, int32_t B, const void* w_ln1,
                                              const void* w_qkv, const void* w_qn, const void* w_kn, const void* w_o,
                                              const void* w_ln2, void* x_out, void* xn2_out, void* workspace,
                                              size_t workspace_bytes, void* stream);

/* Number of kernels the library launched since context creation (host-side counter). */
ASYNCEP_API int64_t asyncep_kernel_launches(const asyncep_ctx* ctx);

ASYNCEP_API asyncep_status asyncep_destroy(asyncep_ctx* ctx);
ASYNCEP_API const char* asyncep_last_error(void);
ASYNCEP_API int32_t asyncep_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ASYNCEP_H */
