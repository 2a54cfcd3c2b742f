/*
 * comet_b200.h -- C ABI of the B200-native fused MoE layer (COMET,
 * arxiv 2502.19811) behind the reference package's layer API.
 *
 * The reference (`moepipe`, /root/reference/pkg/src/moepipe) is pure Python;
 * its "FFI" for this path is the Python function boundary
 *   execute_scheduled / execute_naive / execute_tp_sharded  (executor.py:132-246)
 * fed by resolve_layer0 / resolve_layer1 / sort_tokens_by_source
 *   (resolver.py:171-309) and the block split of select_split
 *   (assigner.py:260-292, simulator.py:45-65).
 * Each entry point below names the reference interface it replaces.  The
 * Python mirror (paper_2502_19811_b200/_lib.py) binds these with ctypes;
 * INTEGRATION.md shows the binding a maintainer adds to moepipe.
 *
 * Conventions
 *   - plain pointers and sizes only; device pointers are CUDA device memory
 *     owned by the caller unless stated; `stream` is a cudaStream_t.
 *   - every call is asynchronous on `stream` unless it says it synchronises.
 *   - return 0 on success; non-zero => comet_last_error() has the message
 *     (the Python layer raises ConfigurationError for COMET_EINVAL, the
 *     reference's error type, config.py:16-17).
 *   - a context is not re-entrant; one host thread per context.
 */
#ifndef COMET_B200_H_
#define COMET_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COMET_OK 0
#define COMET_EINVAL 1   /* bad shape / config / schedule -> ConfigurationError */
#define COMET_ECUDA 2    /* CUDA runtime / driver failure */
#define COMET_ECAP 3     /* index capacity exceeded */

/* Activation between the two expert GEMMs (executor.py:86-90 hook). */
#define COMET_ACT_IDENTITY 0
#define COMET_ACT_RELU 1
#define COMET_ACT_SILU 2
#define COMET_ACT_GELU_TANH 3
#define COMET_ACT_TANH 4

typedef struct comet_ctx comet_ctx;

/* Shape + sharding of one rank.  Mirrors ModelConfig / ParallelSpec
 * (config.py:23-128); m_cap bounds the global token count M per call. */
typedef struct comet_config {
  int rank, world, tp, ep, device;
  int E, topk, N, K; /* full K; each rank holds K / tp */
  int m_cap;
} comet_config;

/* Flat view of one rank's routing index (host copies made by
 * comet_index_download).  Field meaning follows the reference objects:
 *   counts          RoutingTable.expert_counts          routing.py:78-84
 *   transfer        RoutingTable.transfer_counts        routing.py:106-117
 *   row_off/token/src  sort_tokens_by_source layout     resolver.py:171-195
 *   tiles0          resolve_layer0 tiles (expert,row_start,row_stop,n_deps)
 *                                                       resolver.py:206-252
 *   tiles1, chunks  resolve_layer1 tiles (expert,row_start,row_stop,
 *                   col_start,col_stop,n_deps) and reduce chunks
 *                   (col_start,col_stop,first_tile,n_tiles) resolver.py:255-309
 * Arrays are caller-allocated with the capacities returned by
 * comet_index_sizes. */
typedef struct comet_index_host {
  int32_t meta[16];
  int32_t *counts, *transfer, *row_off, *n_local, *row_token, *row_src;
  int32_t *tiles0, *tiles1, *chunks;
  int32_t *pairs0, *pull_token, *pull_src;
} comet_index_host;

const char* comet_last_error(void);
int comet_version(void);

int comet_ctx_create(const comet_config* cfg, comet_ctx** out);
int comet_ctx_destroy(comet_ctx* ctx);

/* Symmetric heap (the paper's NVSHMEM buffer, buffer_bytes = dtype*M*N,
 * config.py:218-226): token-slot buffer + combine buffer + flags, same
 * size and offsets on every rank.  export writes a 64-byte CUDA IPC handle;
 * import takes world*64 bytes gathered from all ranks (torch.distributed
 * all_gather at init) and maps every peer over NVLink. */
int comet_symm_export(comet_ctx* ctx, void* handle64);
int comet_symm_import(comet_ctx* ctx, const void* handles);
/* In-process group (several ranks emulated on one device, or one process
 * driving several devices with peer access): link the contexts directly. */
int comet_link_local(comet_ctx** ctxs, int n);

/* Device pointer to this rank's token-slot buffer [m_cap, N] bf16: the
 * caller places its own tokens at rows [start_r, stop_r) before forward. */
void* comet_token_buffer(comet_ctx* ctx);
/* Device pointer to the [m_cap * topk] int32 routing buffer used by forward. */
void* comet_routing_buffer(comet_ctx* ctx);

/* moe_index_build for this rank from the global router output
 * d_experts[M, topk] (int32, ascending per token).  tile_rows / tile_cols
 * are the reference SharedTensorMeta knobs for the emitted tile lists
 * (resolver.py:32-96); the kernels always run 128-row tiles in 2-CTA pairs.
 * Bumps the context epoch (one forward = one epoch). */
int comet_index_build(comet_ctx* ctx, const int32_t* d_experts, int M, int tile_rows, int tile_cols,
                      void* stream);
/* Same, choosing what is emitted besides the kernels' work tables:
 * flags bit0 = reference outputs (tiles0/tiles1/chunks and the global
 * counts / transfer matrix), bit1 = combine token list (needed by comm-CTA
 * combine), bit2 = publish this rank's token-ready epoch to the peers, bit3 =
 * streamed-forward pair order, bit6 = the layer1 pair order comet_forward
 * uses (fold-level order per the FOLD_ORDER option).  comet_index_build =
 * flags 3; comet_forward builds only what its kernels consume (counts /
 * transfer are then stale). */
int comet_index_build_ex(comet_ctx* ctx, const int32_t* d_experts, int M, int tile_rows, int tile_cols,
                         int flags, void* stream);
/* Sizes of the index arrays after a build (synchronises the stream). */
int comet_index_sizes(comet_ctx* ctx, int32_t meta_out[16], void* stream);
/* Copy the index to host arrays (synchronises the stream). */
int comet_index_download(comet_ctx* ctx, comet_index_host* out, void* stream);

/* Publish "this rank's tokens are in its token buffer" to every peer. */
int comet_signal_tokens_ready(comet_ctx* ctx, void* stream);

/* layer0: NVLink dispatch (n_comm CTAs) fused with GroupGEMM FC1 +
 * activation.  w0t: [E_r, K/tp, N] bf16 (the rank's experts, K-major).
 * n_comm: communication CTAs (even, >= 0); group: pairs per L2 group. */
int comet_layer0(comet_ctx* ctx, const void* w0t, int activation, int n_comm, int group, void* stream);

/* layer1: GroupGEMM FC2 fused with the top-k (weighted) reduce and the
 * combine to source ranks.  w1t: [E_r, N, K/tp] bf16.  combine_w: global
 * [M, topk] fp32 (device) or NULL.  y_local: [M_r, N] bf16 output of this
 * rank's tokens.  n_comm >= 2, even; wave: n-blocks per column wave. */
int comet_layer1(comet_ctx* ctx, const void* w1t, const float* combine_w, void* y_local, int n_comm,
                 int wave, void* stream);

/* layer0 + layer1 in ONE persistent launch (what comet_forward runs): the
 * same work as comet_layer0 then comet_layer1 (n_comm1 = 0), with layer1
 * units claimed as soon as the layer0 H rows of their 256-row pair are
 * complete, and the dispatch CTAs joining the GEMMs once their rows are
 * pulled -- the paper's overlap carried across the layer boundary
 * (executor.py:200-217 runs the two loops back to back). */
int comet_layers(comet_ctx* ctx, const void* w0t, const void* w1t, const float* combine_w, void* y_local,
                 int activation, int n_comm0, int group0, int wave1, void* stream);

/* Remote half of the combine (world > 1): wait for every sender's partial
 * rows of this rank's tokens and sum them in ascending rank order
 * (executor.py:239-245).  Separate from comet_layer1 so that ranks emulated
 * on one device can enqueue all layer1 launches before any finish. */
int comet_combine_finish(comet_ctx* ctx, void* y_local, void* stream);

/* Whole layer forward of one rank: index build, token-ready signal,
 * layer0, layer1 (+ remote combine finish when world > 1). */
int comet_forward(comet_ctx* ctx, const int32_t* d_experts, int M, const void* w0t, const void* w1t,
                  const float* combine_w, void* y_local, int activation, int n_comm0, int n_comm1,
                  int group0, int wave1, void* stream);

/* End-to-end single-GPU forward on HOST buffers (world 1): h_x [M, N] bf16,
 * h_experts [M, topk] int32, h_combine_w [M, topk] fp32 or NULL (all pinned
 * host memory), result into h_y [M, N] bf16.  The token upload runs in
 * `chunks` token chunks on an internal copy stream, each publishing an epoch
 * flag (cuStreamWriteValue32); the ONE layer launch pulls rows as their
 * chunk lands (pairs in (row tile, expert) order), layer1's fused combine
 * writes output rows and counts them per chunk; a second copy stream
 * downloads chunk k once its count is complete (cuStreamWaitValue32).  The
 * call is asynchronous: `stream` waits for the download before anything
 * enqueued after it.  Same arithmetic as execute_naive (executor.py:132-148)
 * within the bf16 tolerance; replaces the reference's host-array call. */
int comet_forward_host(comet_ctx* ctx, const void* h_x, const int32_t* h_experts, const float* h_combine_w,
                       void* h_y, int M, const void* w0t, const void* w1t, int activation, int n_comm0, int group0,
                       int wave1, int chunks, void* stream);

/* Zero-copy single-GPU forward on pinned HOST buffers (world 1; same
 * arguments as comet_forward_host without `chunks`).  The host is treated as
 * the token-owning peer: n_comm0 dispatch CTAs read each token row ONCE from
 * h_x over PCIe (TMA bulk loads of mapped pinned memory), in the compute
 * claim order, and fan it out to the token's hosted rows, then join the
 * GEMMs; layer1's fused combine writes each finished output row straight
 * into h_y.  Requires topk <= 8 and N % 512 == 0.  Asynchronous on `stream`
 * (h_y is complete when the stream reaches the end of this call).  Same
 * arithmetic as execute_naive (executor.py:132-148) within the bf16
 * tolerance; replaces the reference's host-array call. */
int comet_forward_zerocopy(comet_ctx* ctx, const void* h_x, const int32_t* h_experts, const float* h_combine_w,
                           void* h_y, int M, const void* w0t, const void* w1t, int activation, int n_comm0,
                           int group0, int wave1, void* stream);

/* Device pointers of internal buffers (testing / profiling). */
void* comet_hidden_buffer(comet_ctx* ctx);   /* H [rows_pad_cap, K/tp] bf16 */
void* comet_yrows_buffer(comet_ctx* ctx);    /* layer1 rows [rows_pad_cap, N] bf16 */
int32_t comet_hidden_rows_cap(comet_ctx* ctx);

/* Per-CTA timeline of the layer kernels (globaltimer ns): `cap` records per
 * CTA and role (load, mma, tmem-wait, epilogue, comm); 0 disables.  dump
 * copies n_sm * 5 * cap * 2 uint64 {start, (task+1) << 40 | duration} and
 * clears the buffer (synchronises the device).  The Python side exports it
 * in the reference simulator's timeline CSV schema (simulator.py:235-245). */
int comet_timeline_enable(comet_ctx* ctx, int cap);
int comet_timeline_dump(comet_ctx* ctx, void* host_buf, size_t cap_bytes);

/* Launch timing of the layer kernel (moe_layer_kernel) alone: with `slots`
 * > 0, the next `slots` launches are bracketed by a cudaEvent pair recorded
 * on their launch stream (so the duration excludes the index build, the
 * local dispatch / combine kernels and host gaps).  read waits for the
 * recorded launches, writes min(cap, recorded) durations in ms to ms_out,
 * stores the count in *n_out and re-arms the ring.  0 slots disables.
 * Measurement aid for bench.py's roofline (no reference counterpart). */
int comet_kernel_timing_enable(comet_ctx* ctx, int slots);
int comet_kernel_timing_read(comet_ctx* ctx, float* ms_out, int cap, int* n_out);

/* GPU router front-end (no context).  Gate logits [M, E] (logits_dtype 0 =
 * fp32, 1 = bf16, row-major, device) -> d_experts [M, topk] int32, the top-k
 * expert ids stored ASCENDING per token: the reference router-output layout
 * RoutingTable.experts_per_token (routing.py:62-163, validated ascending and
 * distinct at 146-163) that comet_index_build consumes.  Selection is a
 * stable descending sort of the logits (ties -> smaller id, -0 == +0, NaN
 * below -inf); indices are bit-exact with oracle/moe_oracle.router_topk.
 * d_weights [M, topk] fp32 in the same ascending slot order -- the
 * combine_weights of executor.py:102-120 -- for norm 1 (softmax over the k
 * selected logits) or 2 (softmax over all E, selected entries); norm 0
 * writes no weights (d_weights may be NULL).  E <= 512, topk <= min(E, 32).
 * The reference has no router (build_routing, routing.py:283-307, is a
 * synthetic count generator): this replaces the model's gate in front of it. */
int comet_router_topk(const void* d_logits, int logits_dtype, int M, int E, int topk, int norm,
                      int32_t* d_experts, float* d_weights, void* stream);

/* Number of SMs and max co-resident 2-CTA clusters for the layer kernel. */
int comet_device_info(int device, int32_t out[4]);

/* Per-context kernel options (the knobs that are not call arguments).
 * Every option has a measured default; nothing is read from the
 * environment.  comet_set_option(ctx, opt, COMET_OPT_DEFAULT) restores the
 * default.  Options take effect at the next launch on the context.
 *   FUSED          1: both layers in one persistent launch (default 1)
 *   KSPLIT_MAX     split-K slices when a layer has fewer tiles than pairs,
 *                  0..8 (default 8)
 *   SPLIT_TAIL0    layer0's last partial round as 256-column halves (1)
 *   SPLIT1         layer1 units run as halves at the end: -1 automatic by
 *                  shape (default), 0 none, n the last n units
 *   DEDUP          world > 1: per-(token, rank) deduplicated NVLink pulls,
 *                  -1 automatic (default: on when a token can have several
 *                  hosted rows on a rank), 0 off, 1 on
 *   PULL_LOCAL     world > 1: dispatch CTAs place the local rows too (1)
 *   FOLD_ORDER     world > 1: layer1 pairs in fold-level order (0: its
 *                  level computation costs the index build 8-12 us and
 *                  PH EP4xTP2 ran 0.300 vs 0.282 ms, QW EP8 0.381 vs 0.376)
 *   GROUP1         layer1 pair-group size, 0 = layer0's group (0)
 *   CHUNK_ROWS     dispatch item rows 1..32; 0 = auto, ~one item per
 *                  dispatch CTA for M*topk/ep rows, clamped to 4..32 (0)
 *   PDL            programmatic dependent launch bitmask: 1 local dispatch,
 *                  2 layer kernel, 4 combine kernels, 8 index build (14)
 *   GRID           cap on the persistent grid in CTAs, 0 = every SM (0)
 *   FUSE1          world 1: fused epilogue combine instead of the combine
 *                  kernel (0)
 *   SPIN_TIMEOUT_MS  device flag waits trap after this long (600000 = 10
 *                  min; a straggling peer must not kill the job)
 *   ZC_DEDUP / ZC_INTERLEAVE / ZC_DOWNLOAD / ZC_ORDER / ZC_FOLD_ORDER
 *                  zero-copy forward: per-token PCIe dedup (1), layer1
 *                  groups interleaved at this lag (1), dispatch CTAs that
 *                  download the output (8), (row tile, expert) pair order
 *                  (0), fold-level order (0)
 *   STREAM_FUSE    streamed host forward: epilogue fold instead of the
 *                  dispatch-CTA combine (0)
 *   SEQUENTIAL     no overlap: layer0 GEMMs start after the WHOLE dispatch
 *                  (the all-to-all-then-GroupGEMM baseline of the cli; 0)
 *   STREAMK        1: layer1's single partial round (pairs/2 < tiles < pairs,
 *                  no fold chains) as head / tail K slices, the tails
 *                  filling the idle pairs (sched.cuh; measured no faster
 *                  than whole units at Mixtral EP=8 -- kept opt-in; 0)
 *   FOLD_STRIDE    fused combine: 0 = the token's last hosted row folds all
 *                  its other hosted rows; k >= 2 = chained folds -- every
 *                  k-th hosted row (and the last) folds the rows since the
 *                  previous folder plus that folder's weighted partial, so
 *                  a top-8 folder reads <= k rows instead of 7 (measured
 *                  slower: the intermediate folders' waits cost more than
 *                  the shorter last folds save, QW EP=8 0.360 -> 0.366 ms at
 *                  k = 2; 0) */
#define COMET_OPT_FUSED 0
#define COMET_OPT_KSPLIT_MAX 1
#define COMET_OPT_SPLIT_TAIL0 2
#define COMET_OPT_SPLIT1 3
#define COMET_OPT_DEDUP 4
#define COMET_OPT_PULL_LOCAL 5
#define COMET_OPT_FOLD_ORDER 6
#define COMET_OPT_GROUP1 7
#define COMET_OPT_CHUNK_ROWS 8
#define COMET_OPT_PDL 9
#define COMET_OPT_GRID 10
#define COMET_OPT_FUSE1 11
#define COMET_OPT_SPIN_TIMEOUT_MS 12
#define COMET_OPT_ZC_DEDUP 13
#define COMET_OPT_ZC_INTERLEAVE 14
#define COMET_OPT_ZC_DOWNLOAD 15
#define COMET_OPT_ZC_ORDER 16
#define COMET_OPT_ZC_FOLD_ORDER 17
#define COMET_OPT_STREAM_FUSE 18
#define COMET_OPT_SEQUENTIAL 19
#define COMET_OPT_STREAMK 20
#define COMET_OPT_FOLD_STRIDE 21
#define COMET_OPT_COUNT 22
#define COMET_OPT_DEFAULT (-2147483647 - 1)
int comet_set_option(comet_ctx* ctx, int opt, int value);
int comet_get_option(comet_ctx* ctx, int opt, int* value);

/* Host-side abort of device waits: a non-zero value makes every kernel of
 * this process that is spinning on a peer flag trap at its next timeout
 * check (about every 64 polls) instead of waiting out SPIN_TIMEOUT_MS --
 * for a watchdog that knows a peer is gone.  0 clears it. */
int comet_abort_waits(int value);

#ifdef __cplusplus
}
#endif

#endif /* COMET_B200_H_ */
