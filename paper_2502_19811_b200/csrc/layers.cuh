// Parameters of the fused layer kernels (shared by host launcher and device).
#pragma once

#include <cstdint>

#include <cuda_bf16.h>

#include "index.cuh"

// Timing-experiment switches (LayerArgs::debug) exist only in a build with
// -DCOMET_TIMING_EXPERIMENTS; the shipped library folds them to false.
#ifdef COMET_TIMING_EXPERIMENTS
#define COMET_DBG(v, bits) ((((v) & (bits)) != 0))
#else
#define COMET_DBG(v, bits) false
#endif

namespace comet {

enum TimelineRole : int { kRoleLoad = 0, kRoleMma = 1, kRoleTmemWait = 2, kRoleEpilogue = 3, kRoleComm = 4, kRoles = 5 };

constexpr int kLayerStages = 4;  // 48 KB smem stages per CTA (A 16 KB + two B halves 16 KB)

enum Activation : int { kActIdentity = 0, kActRelu = 1, kActSilu = 2, kActGeluTanh = 3, kActTanh = 4 };

struct LayerArgs {
  int layer;              // 0: dispatch + FC1 + act ; 1: FC2 + top-k combine
  int rank, world, tp, ep;
  int M, topk, n_embed;   // global tokens, experts per token, N
  int k_local;            // K / tp
  int e_lo;
  int experts_per_group;  // E / ep
  int n_compute;          // CTAs [0, n_compute) are compute (even); the rest comm
  int n_blocks;           // output 256-col blocks of this layer
  int k_blocks;           // 64-wide contraction blocks
  int b_rows;             // weight rows per expert in the 2D B view
  int order_group;        // layer0: pairs per group; layer1: n-blocks per wave
  int order_group2;       // layer1: pairs per group inside a wave (raster 1) / per outer group (raster 2)
  int raster;             // unit order: 0 layer0 groups, 1 layer1 waves, 2 pair groups then waves (fused)
  int activation;
  int split_tail;         // layer0 (alone): cut a mostly idle last round into 256-column half units
  int split_units;        // layer1: the last `split_units` full units run as 256-column halves
  int ksplit_max;         // split-K slices allowed when output tiles are fewer than pairs (0 = off)
  int streamk;            // layer1: stream-K tail (sched.cuh) instead of whole units in the last round
  float* part;            // split-K fp32 partials [tiles*NB][S][128][512] (<= pairs*2 CTA tiles)
  uint32_t* split_cnt;    // [1024] split-K counters of this layer (capi.cu comet_ctx::split_cnt)
  uint32_t epoch;
  int debug;              // timing-experiment bits, compiled in only with -DCOMET_TIMING_EXPERIMENTS
                          // (COMET_DBG; wrong results unless noted): 1: comm CTAs idle; 4: spin
                          // waits; 8: no MMA; 16: no loads; 64/128: no stores / no drain; 256: staged
                          // in smem, not stored; 512: packed only; 16384:
                          // st.global epilogue instead of TMA stores (correct)
  int sequential;         // layer0: GEMMs start after the WHOLE dispatch (COMET_OPT_SEQUENTIAL; the
                          // no-overlap baseline of the cli, correct results)

  // index (device)
  const int32_t* meta;
  const int32_t* pairs;       // [P*4] (e_local, pad_row, valid, key)
  const int32_t* gather_row;  // [Rpad] token ids of the padded layout (-1 = padding)
  const int32_t* pad_off;     // [E_r+1] padded block offset of each hosted expert
  const int32_t* n_local;     // [E_r] local (prefix) rows of each hosted expert
  __nv_bfloat16* xg;          // [Rpad_cap, N] layer0 A: dispatched rows, expert-sorted
  uint32_t* xg_ready;         // [Rpad_cap / 128] epoch when a 128-row tile of xg is filled
  uint32_t* xg_cnt;           // [Rpad_cap / 128] remote rows landed per tile (reset by its publisher)
  int chunk_rows;             // layer0 dispatch work item: rows of one tile (1..32)
  int dedup;                  // dispatch pulls each token once and fans it out (dispatch_rows_dedup)
  const int32_t* claim_of_tile;   // [Rpad/128] padded tile -> claim-order tile index
  const __nv_bfloat16* host_src;  // zero-copy forward: token rows read from pinned host memory
  // host-streamed forward (comet_forward_host, world 1): every row is pulled
  // by the dispatch CTAs once its token's upload chunk landed (chunk_ready
  // epoch, written by the copy stream); layer1 counts finished output halves
  // per token chunk (out_cnt) for the download stream to wait on
  int stream;                 // (kept for the host-streamed forward's bookkeeping)
  int pull_local;             // dispatch CTAs also place the local rows (no dispatch_local launch):
                              // every populated 128-row half is published by the dispatch
  const uint32_t* chunk_ready;
  int chunk_tokens;
  uint32_t* out_cnt;
  int stream_combine;         // layer0 (streamed forward): dispatch CTAs then reduce finished token
                              // chunks (comm::stream_combine) instead of joining the GEMMs
  int publish_tiles;          // layer1: publish tile_done epochs even without the fused combine
  const int32_t* pull_token;  // layer0 comm
  const int32_t* pull_src;
  const int32_t* tok_pos;     // [M*topk]
  const int32_t* combine_tok;
  const int32_t* row_dst;     // [Rpad] (src_rank << 24 | combine slot) of last-hosted rows, else -1
  const int32_t* row_widx;    // [Rpad] t * topk + slot of each padded row
  int fuse_combine;           // layer1: the epilogue of each token's last hosted row folds the
                              // earlier rows in and writes y (world 1) / pushes to the source rank
  int fold_stride;            // fused combine: 0 = that row folds all of them; k >= 2 = chained
                              // (COMET_OPT_FOLD_STRIDE): hosted rows c % k == k-1 fold too
  uint32_t* tile_done;        // [Rpad/128 * n_blocks * 2] epoch when a 128-row tile's yrows of a 256-column
                              // half of an n-block landed
  const float* combine_w;     // [M*topk] or null

  // buffers
  __nv_bfloat16* out;             // epilogue output: H (layer0) or yrows (layer1), row-major
  int out_ld;                     // its row length in elements (K_local or N)
  __nv_bfloat16* xs_local;        // [M_cap, N] this rank's symmetric token buffer
  const __nv_bfloat16* const* xs_peer;  // [world] peer token buffers (device array)
  uint32_t* tok_ready;            // [M_cap] epoch when xs_local[t] holds token t
  const uint32_t* x_ready;        // [world] epoch when peer's own tokens are in place
  const __nv_bfloat16* yrows;     // [Rpad_cap, N] layer1 per-(token,expert) rows
  __nv_bfloat16* y_local;         // [M_r, N] final output (world == 1 or finish kernel)
  __nv_bfloat16* const* cb_peer;  // [world] peer combine buffers [W*Mloc_cap, N]
  uint32_t* const* cb_flag_peer;  // [world] peer flags [W * n_blocks]
  uint32_t* nb_done;              // [n_blocks] layer1 compute completion counters
  uint32_t* nb_sent;              // [n_blocks] layer1 comm CTA completion counters
  int mloc_cap;                   // combine slots per sender

  // per-CTA timeline (optional, null = off): record r of CTA c, role k lives
  // at ((c * kRoles + k) * timeline_cap + r) * 2 as {start_ns, end_ns | tag}
  unsigned long long* timeline;
  int timeline_cap;
};

// One launch of the persistent layer kernel.  mode 0: layer0 alone; mode 1:
// layer1 alone; mode 2: layer0 then layer1 in ONE launch -- a layer1 unit
// starts as soon as the layer0 H rows of its 256-row pair are complete (per
// 128-row tile counters), so layer0's last round overlaps layer1's first.
// Work units are claimed dynamically (one atomic per unit, in sequence
// order): layer0 units, then layer1 units.  Dispatch CTAs (layer0 comm,
// [l[0].n_compute, grid)) join the compute pairs once their rows are pulled;
// layer1 combine CTAs (mode 1, [l[1].n_compute, grid)) never compute.
struct KernelArgs {
  LayerArgs l[2];
  int mode;
  int interleave;    // mode 2: >0 = layer1 group j follows layer0 group j + interleave (see unit_at)
  int n_dl;          // mode 2: the first n_dl dispatch CTAs then download final output rows to y_host
  __nv_bfloat16* y_host;  // zero-copy forward: [M, N] pinned host output (l[1].y_local is the device copy)
  uint32_t* sched;   // [0] unit claim counter, [1] CTA exit counter (both reset by the last CTA)
  uint32_t* h_cnt;   // [n_h] mode 2: layer0 256-column halves landed per (128-row H tile, n-block) (reset at exit)
  int n_h;
};

}  // namespace comet
