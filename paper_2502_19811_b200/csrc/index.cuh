// Device-side routing index of one rank: the reference's sorted layout and
// tile schedules (resolver.py:171-309) in flat integer form, plus the padded
// row layout and work-unit tables the fused layer kernels consume.
#pragma once

#include <cstdint>

namespace comet {

constexpr int kTileRows = 128;   // reference DEFAULT_TILE_ROWS (resolver.py:32) = one CTA's rows
constexpr int kPairRows = 256;   // rows per 2-CTA MMA pair (UMMA M = 256)
constexpr int kBlockN = 512;     // output columns per work unit (two UMMA N = 256 halves)
constexpr int kMaxWorld = 64;

// scalar slots in IndexDev::meta
enum MetaSlot : int {
  kMetaRows = 0,       // sum of hosted expert counts (unpadded rows)
  kMetaRowsPad = 1,    // rows in the 256-aligned padded layout
  kMetaTiles0 = 2,     // reference layer0 tiles
  kMetaPairs = 3,      // 256-row pair units per column block
  kMetaPull = 4,       // distinct remote tokens to pull (layer0 dispatch)
  kMetaTiles1 = 5,     // reference layer1 tiles (= chunks * tiles per chunk)
  kMetaChunks = 6,     // reference reduce chunks
  kMetaCombineTok = 7, // tokens with at least one hosted expert
  // 8..13: build phase timing probes (ns from kernel entry; CTA 0: phase 1a,
  // 1b, grid barrier, phase 2; last CTA: phase 3 start, end), 15: overflow flags
  kMetaSlots = 16
};

// IndexDev::flags: what the last CTA emits besides the pair tables.
constexpr int kIndexRefLists = 1;      // reference tiles0 / tiles1 / chunks (resolver API)
constexpr int kIndexCombineList = 2;   // combine token list (comm-CTA combine)
constexpr int kIndexSignal = 4;        // publish this rank's x_ready epoch to every peer
constexpr int kIndexStream = 8;        // host-streamed forward: pairs in (row tile, expert) order
constexpr int kIndexFoldOrder = 16;    // fused combine with fold chains: order pairs1 by fold level
constexpr int kIndexForwardOrder = 64; // host flag: add comet_forward's fold-order bit (COMET_OPT_FOLD_ORDER)
                                       // (experts whose rows are only folded in come first) and,
                                       // per token, the fused-combine folder = its row claimed LAST
constexpr int kIndexMaxChunks = 64;    // token chunks per hosted expert (host-checked)

struct IndexDev {
  // inputs
  const int32_t* experts;   // [M, topk] row-major, ascending per token
  int M, E, topk, tp, ep, rank, world;
  int e_lo, E_r;            // hosted experts [e_lo, e_lo + E_r)
  int tile_rows, tile_cols, n_embed;
  int flags;
  int mloc_cap;             // combine slots per sender in the symmetric combine buffer
  int tpt;                  // rotated token positions per thread per chunk (chunk = 1024 * tpt)
  uint32_t epoch;
  uint32_t* const* x_ready_peer;  // [world] peers' x_ready arrays (kIndexSignal)

  // outputs (device)
  int32_t* counts;      // [E]
  int32_t* transfer;    // [W*W]
  int32_t* row_off;     // [E_r+1] unpadded CSR offsets
  int32_t* pad_off;     // [E_r+1] 256-aligned offsets of each expert's block
  int32_t* n_local;     // [E_r]
  int32_t* row_token;   // [R]  layout order
  int32_t* row_src;     // [R]
  int32_t* gather_row;  // [Rpad] token id of each padded row, -1 = padding
  int32_t* tok_pos;     // [M*topk] padded row of hosted (token, slot), else -1
  int32_t* tiles0;      // [T0*4] (expert, row_start, row_stop, n_deps) in schedule order
  int32_t* tiles1;      // [T1*6] (expert, row_start, row_stop, col_start, col_stop, n_deps)
  int32_t* chunks;      // [C*4] (col_start, col_stop, first_tile, n_tiles)
  int32_t* pairs0;      // [P*4] (e_local, pad_row, valid_rows, key) layer0 claim order
  int32_t* pairs1;      // [P*4] (e_local, pad_row, valid_rows, 0) expert/row order
  int32_t* claim_of_tile;  // [Rpad/128] claim-order tile index (2 * pairs0 rank + half) of a padded tile
  int32_t* pull_token;  // [<=M] remote tokens in first-demand order
  int32_t* pull_src;    // [<=M]
  int32_t* combine_tok; // [<=M] tokens with a hosted expert, ascending (combine CTAs)
  int32_t* row_dst;     // [Rpad] (src_rank << 24 | combine slot) of a padded row holding its
                        // token's last hosted expert (fused combine), else -1
  int32_t* row_widx;    // [Rpad] t * topk + slot of the padded row (combine weight index)
  int32_t* meta;        // [kMetaSlots]
  // scratch
  int32_t* pair_key;    // [P_cap]
  uint32_t* done;       // [1] item-CTA completion counter (kIndexStream; self-resetting)
  uint32_t* p1_done;    // [1] fold-mask completion counter (kIndexFoldOrder; self-resetting)
  int32_t* chunk_cnt;   // [E_r * kIndexMaxChunks] hits per (hosted expert, token chunk)
  int32_t* chunk_loc;   // [E_r * kIndexMaxChunks] local-token hits per (hosted expert, chunk)
  uint32_t* chunk_flag; // [E_r * kIndexMaxChunks] build epoch when the item's counts landed (look-back)
  unsigned long long* fold_part;  // [grid * E_r] per-CTA fold-predecessor masks (kIndexFoldOrder)
  uint32_t* zero_words; // layer1 per-n-block counters, zeroed every build
  int n_zero_words;

  // capacities (checked on device; overflow sets meta[kMetaSlots-1])
  int cap_rows, cap_rows_pad, cap_tiles0, cap_tiles1, cap_pairs;
};

// Token -> source rank, contiguous pre-distribution with the remainder on
// the last rank (routing.py:86-95).
__host__ __device__ inline int src_rank_of(int t, int M, int W) {
  const int base = M / W;
  if (base == 0) return W - 1;
  const int r = t / base;
  return r < W - 1 ? r : W - 1;
}

__host__ __device__ inline int token_start_of(int r, int M, int W) { return r * (M / W); }
__host__ __device__ inline int token_stop_of(int r, int M, int W) {
  return r == W - 1 ? M : (r + 1) * (M / W);
}

}  // namespace comet
