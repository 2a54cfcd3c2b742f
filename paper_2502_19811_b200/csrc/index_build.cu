// moe_index_build: the routing index of one rank, built on the GPU.
//
// Bit-exact restatement of the reference's integer path:
//   expert_counts / transfer_counts       routing.py:78-117
//   sort_tokens_by_source                 resolver.py:171-195
//   resolve_layer0 (locality-first order) resolver.py:206-252
//   resolve_layer1 (column waves, chunks) resolver.py:255-309
//
// Key observation used for the layout: tokens are pre-distributed to ranks in
// contiguous, rank-monotone blocks (routing.py:86-104), so ordering an
// expert's rows by ((src - rank) mod W, token) is exactly the token order
// rotated to start at this rank's first token.  Each expert's block is then a
// stable stream compaction of the rotated token sequence -- work items of
// (hosted expert, token chunk), block-wide ballot scans, no sort.
//
// One launch: every CTA writes its token slice's non-hosted slots (and the
// reference counts / transfer matrix when asked); the item CTAs count each
// item's hits, publish them and look back at the earlier items (decoupled
// look-back: the rows before it, no grid barrier), then write its rows.  The
// last CTA has no items: it sums the items' published hit counts into each
// hosted expert's totals and builds the tile lists, the 2-CTA pair tables and
// the combine token list -- they need only those totals -- while the items
// look back and write their rows.  The tables are the build's longest serial stretch (~7 us,
// mostly first-touch instruction and constant fetch: the pair-table block
// takes 3.1 us the first time and 0.65 us when repeated in one launch), so
// overlapping them with the items instead of following a grid-wide
// completion count shortens the build.
#include <climits>
#include <cstdint>

#include "index.cuh"
#include "ptx.cuh"

namespace comet {

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxExperts = 1024;
constexpr int kSortSmemKeys = 8192;

// Exclusive block scan of one int per thread; returns the prefix, writes the
// block total to *total.  `ws` is kWarps ints of smem.
__device__ __forceinline__ int block_scan(int v, int* ws, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int s = lane < kWarps ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kWarps) ws[lane] = s;
  }
  __syncthreads();
  const int before = (warp ? ws[warp - 1] : 0) + x - v;
  *total = ws[kWarps - 1];
  __syncthreads();
  return before;
}

// Warp-aggregated shared-memory increment: lanes hitting the same counter are
// merged (match.any) so each distinct address takes one atomic per warp.
// Routing is highly concentrated (8 experts, or a single transfer cell at
// EP=1), so plain per-lane atomics serialise on a handful of addresses.
__device__ __forceinline__ void warp_add(int* base, int idx, bool active) {
  const unsigned act = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  const unsigned peers = __match_any_sync(act, idx);
  const int leader = __ffs(peers) - 1;
  if ((threadIdx.x & 31) == leader) atomicAdd(base + idx, __popc(peers));
}

__device__ __forceinline__ int slot_of(const int32_t* row, int topk, int e) {
  for (int s = 0; s < topk; ++s)
    if (row[s] == e) return s;
  return -1;
}

__device__ __forceinline__ long long tile_key(int ndeps, int e, int row_start) {
  return (static_cast<long long>(ndeps) << 42) | (static_cast<long long>(e) << 21) |
         static_cast<long long>(row_start);
}


// Token-chunk hits of hosted expert e: thread `tid` owns the rotated
// positions [c*T + tid*TPT, +TPT) (contiguous rows -> coalesced warp loads).
// Bit q of the result: position tid*TPT+q routes to e.
__device__ __forceinline__ uint64_t chunk_hits(const IndexDev& ix, int c, int T, int TPT, int e, int start,
                                               int n_own, int* n_loc) {
  const int M = ix.M, K = ix.topk;
  uint64_t hit = 0;
  int loc = 0;
#pragma unroll 4
  for (int q = 0; q < TPT; ++q) {
    const int i = c * T + threadIdx.x * TPT + q;
    int t = start + i;
    if (t >= M) t -= M;
    const bool f = i < M && slot_of(ix.experts + static_cast<long long>(min(t, M - 1)) * K, K, e) >= 0;
    hit |= static_cast<uint64_t>(f) << q;
    loc += (f && i < n_own);
  }
  *n_loc = loc;
  return hit;
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) index_build_kernel(IndexDev ix) {
  extern __shared__ long long sh_keys[];  // kSortSmemKeys (bookkeeping scratch, phase 3 keys)
  __shared__ int s_cnt[kMaxExperts];      // hosted expert totals, j-indexed
  __shared__ int s_off[kMaxExperts + 1];
  __shared__ int s_pad[kMaxExperts + 1];
  __shared__ int s_ws[kWarps];
  __shared__ int s_misc[8];

  ptx::pdl_launch_dependents();  // the dispatch / layer kernels may launch; they wait for this grid
  // launched with programmatic serialization (COMET_OPT_PDL bit 8): only the
  // launch overlapped the previous kernel (e.g. the last forward's combine),
  // which may still read this rank's index -- wait for it before any write
  ptx::pdl_wait();
  const int tid = threadIdx.x;
  unsigned long long tt0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt0));
  auto probe = [&](int k) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (tid == 0 && (blockIdx.x == 0 || k >= 4)) ix.meta[8 + k] = (int)(t1 - tt0);
  };
  const int M = ix.M, K = ix.topk, W = ix.world, E = ix.E, Er = ix.E_r;
  const int TPT = ix.tpt, T = kThreads * TPT;
  const int C = (M + T - 1) / T;  // token chunks (rotated order)
  const int items = Er * C;       // (hosted expert, chunk) work items
  const int start = token_start_of(ix.rank, M, W);
  const int n_own = token_stop_of(ix.rank, M, W) - start;

  // "my tokens are in place, my previous forward is done" -> every peer
  // (index.cuh kIndexSignal; replaces a separate signal launch)
  if ((ix.flags & kIndexSignal) && blockIdx.x == 0 && tid >= 32 && tid < 32 + W) {
    ptx::fence_acq_rel_sys();
    ptx::st_release_sys(ix.x_ready_peer[tid - 32] + ix.rank, ix.epoch);
  }
  if (blockIdx.x == 0)
    for (int i = tid; i < ix.n_zero_words; i += kThreads) ix.zero_words[i] = 0u;

  probe(0);
  // -------- phase 1 (independent of the row layout): bookkeeping over natural token slices: global
  // histogram (routing.py:78-84), transfer matrix (routing.py:106-117) and
  // the non-hosted tok_pos slots.  The hot path (no reference lists) needs
  // only the tok_pos slots --------
  if (!(ix.flags & kIndexRefLists)) {
    const int t_lo = static_cast<int>(static_cast<long long>(M) * blockIdx.x / gridDim.x);
    const int t_hi = static_cast<int>(static_cast<long long>(M) * (blockIdx.x + 1) / gridDim.x);
    for (int i = t_lo * K + tid; i < t_hi * K; i += kThreads) {
      const int e = __ldg(ix.experts + i);
      if (e < ix.e_lo || e >= ix.e_lo + Er) ix.tok_pos[i] = -1;
    }
  } else {
    int* s_tr = reinterpret_cast<int*>(sh_keys);  // W*W <= 4096 ints (host-checked)
    int* s_hist = s_tr + W * W;                   // E <= 1024 ints
    for (int i = tid; i < W * W; i += kThreads) s_tr[i] = 0;
    for (int i = tid; i < E; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    const int per_group = E / ix.ep;
    const int t_lo = static_cast<int>(static_cast<long long>(M) * blockIdx.x / gridDim.x);
    const int t_hi = static_cast<int>(static_cast<long long>(M) * (blockIdx.x + 1) / gridDim.x);
    for (int t0 = t_lo; t0 < t_hi; t0 += kThreads) {
      const int t = t0 + tid;
      const bool ok = t < t_hi;
      const int src = src_rank_of(ok ? t : t_lo, M, W);
      for (int sl = 0; sl < K; ++sl) {
        const int e = ok ? __ldg(ix.experts + static_cast<long long>(t) * K + sl) : 0;
        const int g = e / per_group;
        warp_add(s_hist, e, ok);
        for (int d = 0; d < ix.tp; ++d) warp_add(s_tr, src * W + g * ix.tp + d, ok);
        if (ok && (e < ix.e_lo || e >= ix.e_lo + Er)) ix.tok_pos[static_cast<long long>(t) * K + sl] = -1;
      }
    }
    __syncthreads();
    for (int i = tid; i < W * W; i += kThreads)
      if (s_tr[i]) atomicAdd(ix.transfer + i, s_tr[i]);  // zeroed by the host before launch
    for (int i = tid; i < E; i += kThreads)
      if (s_hist[i]) atomicAdd(ix.counts + i, s_hist[i]);
  }

  // fold-predecessor masks of this CTA's token slice: for a token with >= 2
  // hosted experts, the last hosted one (its fused-combine folder) must come
  // after every other hosted one in the layer1 order
  if (ix.flags & kIndexFoldOrder) {
    unsigned long long* s_pred = reinterpret_cast<unsigned long long*>(sh_keys);  // E_r <= 64 masks
    __syncthreads();
    for (int j = tid; j < Er; j += kThreads) s_pred[j] = 0ull;
    __syncthreads();
    const int t_lo = static_cast<int>(static_cast<long long>(M) * blockIdx.x / gridDim.x);
    const int t_hi = static_cast<int>(static_cast<long long>(M) * (blockIdx.x + 1) / gridDim.x);
    for (int t = t_lo + tid; t < t_hi; t += kThreads) {
      unsigned long long m = 0ull;
      int last = -1;
      for (int sl = 0; sl < K; ++sl) {
        const int j = __ldg(ix.experts + static_cast<long long>(t) * K + sl) - ix.e_lo;
        if (j < 0 || j >= Er) continue;
        if (last >= 0) m |= 1ull << last;
        last = j;
      }
      if (m) atomicOr(s_pred + last, m);
    }
    __syncthreads();
    for (int j = tid; j < Er; j += kThreads) ix.fold_part[static_cast<long long>(blockIdx.x) * Er + j] = s_pred[j];
    __syncthreads();
    // the table CTA reads every slice's masks: the CTA barrier orders the
    // writes before thread 0's release (cumulative)
    if (tid == 0) ptx::red_release_gpu_add(ix.p1_done, 1u);
  }

  probe(1);
  const bool table_cta = blockIdx.x == gridDim.x - 1;
  const int n_item_ctas = gridDim.x - 1;

  // -------- rows: one pass per (hosted expert, token chunk) item.  Count the
  // item's hits, publish the counts (epoch flag), look back at every earlier
  // item (experts before j: their padded totals; chunks before c: the rows
  // before this chunk -- a decoupled look-back, no grid barrier: every item
  // waits only on lower items, so the lowest unfinished one never waits),
  // then write the rows: a stable compaction of the rotated token order --------
  for (int it = table_cta ? items : static_cast<int>(blockIdx.x); it < items; it += n_item_ctas) {
    const int j = it / C, c = it - (it / C) * C, e = ix.e_lo + j;
    int loc;
    uint64_t hit = chunk_hits(ix, c, T, TPT, e, start, n_own, &loc);
    int tot, tot_loc;
    const int mine = block_scan(__popcll(hit), s_ws, &tot);
    block_scan(loc, s_ws, &tot_loc);
    if (tid == 0) {
      ix.chunk_cnt[it] = tot;
      ix.chunk_loc[it] = tot_loc;
      ptx::st_release_gpu(ix.chunk_flag + it, ix.epoch);
    }
    for (int q = tid; q <= j; q += kThreads) s_cnt[q] = 0;
    __syncthreads();
    for (int q = tid; q < it; q += kThreads) {
      { ptx::Spin sp; while (ptx::ld_acquire_gpu(ix.chunk_flag + q) != ix.epoch) sp.pause(32, 13); }
      const int n = __ldcg(ix.chunk_cnt + q);
      if (n) atomicAdd(s_cnt + q / C, n);  // experts < j: totals; expert j: rows before chunk c
    }
    __syncthreads();
    if (tid == 0) {
      int o = 0, pd = 0;
      for (int q = 0; q < j; ++q) {
        o += s_cnt[q];
        pd += (s_cnt[q] + kPairRows - 1) / kPairRows * kPairRows;
      }
      s_misc[0] = o;
      s_misc[2] = pd;
    }
    __syncthreads();
    const int before = s_cnt[j];
    const int base_row = s_misc[0], base_pad = s_misc[2];
    int pos = before + mine;
    while (hit) {
      const int q = __ffsll(hit) - 1;
      hit &= hit - 1;
      const int i = c * T + tid * TPT + q;
      int t = start + i;
      if (t >= M) t -= M;
      const int32_t* trow = ix.experts + static_cast<long long>(t) * K;
      const int sl = slot_of(trow, K, e);
      if (base_pad + pos < ix.cap_rows_pad) {
        // the token's last hosted expert (ascending slots) carries the fused
        // combine: its epilogue folds the earlier hosted rows in
        bool last = true;
        for (int s2 = sl + 1; s2 < K; ++s2) last &= !(trow[s2] >= ix.e_lo && trow[s2] < ix.e_lo + Er);
        const int sr = src_rank_of(t, M, W);
        const int slot = (W > 1 ? ix.rank * ix.mloc_cap : 0) + t - token_start_of(sr, M, W);
        ix.row_dst[base_pad + pos] = last ? ((sr << 24) | slot) : -1;
        ix.row_widx[base_pad + pos] = t * K + sl;
        ix.gather_row[base_pad + pos] = t;
      }
      if (base_row + pos < ix.cap_rows) {
        ix.row_token[base_row + pos] = t;
        ix.row_src[base_row + pos] = src_rank_of(t, M, W);
      }
      ix.tok_pos[static_cast<long long>(t) * K + sl] = base_pad + pos;
      ++pos;
    }
    if (c == C - 1) {  // padding rows of expert j's 256-aligned block
      const int cnt = before + tot;
      const int end = base_pad + (cnt + kPairRows - 1) / kPairRows * kPairRows;
      for (int r = base_pad + cnt + tid; r < end; r += kThreads)
        if (r < ix.cap_rows_pad) {
          ix.gather_row[r] = -1;
          ix.row_dst[r] = -1;
          ix.row_widx[r] = 0;
        }
    }
    __syncthreads();  // s_cnt / s_misc reuse
  }

  probe(3);
  if (!table_cta) {
    if (ix.flags & kIndexStream) {  // the stream pass below reads every item's tok_pos
      __syncthreads();
      if (tid == 0) ptx::red_release_gpu_add(ix.done, 1u);
    }
    return;
  }
  // -------- the table CTA: expert totals (all rows, rows of this rank's
  // tokens) from the items' published counts (each item publishes them before
  // its look-back and row writes), then the schedules --------
  __shared__ int s_nloc[kMaxExperts];
  for (int j = tid; j < Er; j += kThreads) {
    s_cnt[j] = 0;
    s_nloc[j] = 0;
  }
  __syncthreads();
  for (int q = tid; q < items; q += kThreads) {
    { ptx::Spin sp; while (ptx::ld_acquire_gpu(ix.chunk_flag + q) != ix.epoch) sp.pause(32, 13); }
    const int n = __ldcg(ix.chunk_cnt + q), l = __ldcg(ix.chunk_loc + q);
    if (n) atomicAdd(s_cnt + q / C, n);
    if (l) atomicAdd(s_nloc + q / C, l);
  }
  if ((ix.flags & kIndexFoldOrder) && tid == 0) {  // every slice's fold masks
    ptx::Spin sp;
    while (ptx::ld_acquire_gpu(ix.p1_done) < gridDim.x) sp.pause(32, 14);
    *ix.p1_done = 0u;  // nothing else reads it this launch; ready for the next
  }
  __syncthreads();
  probe(4);
  for (int j = tid; j < Er; j += kThreads) ix.n_local[j] = s_nloc[j];
  if (tid == 0) {
    int o = 0, pd = 0;
    for (int j = 0; j < Er; ++j) {
      s_off[j] = o;
      s_pad[j] = pd;
      o += s_cnt[j];
      pd += (s_cnt[j] + kPairRows - 1) / kPairRows * kPairRows;
    }
    s_off[Er] = o;
    s_pad[Er] = pd;
  }
  __syncthreads();
  for (int j = tid; j <= Er; j += kThreads) {
    ix.row_off[j] = s_off[j];
    ix.pad_off[j] = s_pad[j];
  }

  const int TR = ix.tile_rows;
  // tiles per expert (reference tile_rows) and pairs per expert (256 rows)
  __shared__ int s_t0[kMaxExperts + 1];
  __shared__ int s_p0[kMaxExperts + 1];
  if (tid == 0) {
    int t = 0, p = 0;
    for (int j = 0; j < Er; ++j) {
      s_t0[j] = t;
      s_p0[j] = p;
      const int c = s_cnt[j];
      t += (c + TR - 1) / TR;
      p += (c + kPairRows - 1) / kPairRows;
    }
    s_t0[Er] = t;
    s_p0[Er] = p;
  }
  __syncthreads();
  // layer1 pair order (pairs1): experts by (fold level, id) -- level = longest
  // chain of fold predecessors, so a folder's rows come after all the rows it
  // folds (no fold waits on units running alongside); natural order otherwise
  __shared__ int s_pord[kMaxExperts];  // first pairs1 index of expert j
  if (ix.flags & kIndexFoldOrder) {
    __shared__ unsigned long long s_fp[64];
    __shared__ int s_lvl[64];
    for (int j = tid; j < Er; j += kThreads) {
      unsigned long long m = 0ull;
      for (int c = 0; c < static_cast<int>(gridDim.x); ++c) m |= __ldcg(ix.fold_part + static_cast<long long>(c) * Er + j);
      s_fp[j] = m;
    }
    __syncthreads();
    if (tid == 0) {
      int max_lvl = 0;
      for (int j = 0; j < Er; ++j) {
        int l = 0;
        for (int q = 0; q < j; ++q)
          if ((s_fp[j] >> q) & 1ull) l = max(l, s_lvl[q] + 1);
        s_lvl[j] = l;
        max_lvl = max(max_lvl, l);
      }
      int off = 0;
      for (int l = 0; l <= max_lvl; ++l)
        for (int j = 0; j < Er; ++j)
          if (s_lvl[j] == l) {
            s_pord[j] = off;
            off += s_p0[j + 1] - s_p0[j];
          }
    }
  } else {
    for (int j = tid; j < Er; j += kThreads) s_pord[j] = s_p0[j];
  }
  __syncthreads();
  const int T0 = s_t0[Er], P = s_p0[Er];
  const bool ovf = T0 > ix.cap_tiles0 || P > ix.cap_pairs || s_pad[Er] > ix.cap_rows_pad ||
                   s_off[Er] > ix.cap_rows;

  // ---- layer0 tiles sorted by (n_deps, expert, row_start) ----
  auto tile_of = [&](int idx, int& j, int& rs, int& re, int& nd) {
    int lo = 0, hi = Er - 1;  // expert with s_t0[j] <= idx < s_t0[j+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_t0[mid] <= idx) lo = mid; else hi = mid - 1;
    }
    j = lo;
    const int c = s_cnt[j];
    rs = (idx - s_t0[j]) * TR;
    re = min(rs + TR, c);
    const int loc_end = min(re, s_nloc[j]);
    nd = (re - rs) - max(0, loc_end - rs);
  };
  const bool keys_in_smem = T0 <= kSortSmemKeys;
  const bool emit_lists = (ix.flags & kIndexRefLists) != 0;
  if (!ovf && emit_lists) {
    if (keys_in_smem) {
      for (int i = tid; i < T0; i += kThreads) {
        int j, rs, re, nd;
        tile_of(i, j, rs, re, nd);
        sh_keys[i] = tile_key(nd, ix.e_lo + j, rs);
      }
      __syncthreads();
    }
    for (int i = tid; i < T0; i += kThreads) {
      int j, rs, re, nd;
      tile_of(i, j, rs, re, nd);
      const long long k = tile_key(nd, ix.e_lo + j, rs);
      int rank = 0;
      for (int q = 0; q < T0; ++q) {
        long long kq;
        if (keys_in_smem) {
          kq = sh_keys[q];
        } else {
          int jq, rsq, req, ndq;
          tile_of(q, jq, rsq, req, ndq);
          kq = tile_key(ndq, ix.e_lo + jq, rsq);
        }
        rank += kq < k;
      }
      int* o = ix.tiles0 + rank * 4;
      o[0] = ix.e_lo + j; o[1] = rs; o[2] = re; o[3] = nd;
    }
  }
  __syncthreads();

  // ---- layer1 reference tiles: column block outer, (expert,row) inner ----
  const int TC = ix.tile_cols, NE = ix.n_embed;
  const int NCH = (NE + TC - 1) / TC;
  const long long T1 = static_cast<long long>(NCH) * T0;
  const bool ovf1 = emit_lists && T1 > ix.cap_tiles1;
  int4* s_tile = reinterpret_cast<int4*>(sh_keys);  // per-tile (expert, rs, re, nd) cache
  const bool tiles_in_smem = T0 <= kSortSmemKeys / 2;
  if (!ovf && !ovf1 && emit_lists) {
    if (tiles_in_smem) {
      for (int q = tid; q < T0; q += kThreads) {
        int j, rs, re, nd;
        tile_of(q, j, rs, re, nd);
        s_tile[q] = make_int4(ix.e_lo + j, rs, re, nd);
      }
      __syncthreads();
    }
    for (long long i = tid; i < T1; i += kThreads) {
      const int c = static_cast<int>(i / T0), q = static_cast<int>(i % T0);
      int4 tq;
      if (tiles_in_smem) {
        tq = s_tile[q];
      } else {
        int j, rs, re, nd;
        tile_of(q, j, rs, re, nd);
        tq = make_int4(ix.e_lo + j, rs, re, nd);
      }
      int* o = ix.tiles1 + i * 6;
      o[0] = tq.x; o[1] = tq.y; o[2] = tq.z;
      o[3] = c * TC; o[4] = min(c * TC + TC, NE); o[5] = tq.w;
    }
    for (int c = tid; c < NCH; c += kThreads) {
      int* o = ix.chunks + c * 4;
      o[0] = c * TC; o[1] = min(c * TC + TC, NE); o[2] = c * T0; o[3] = T0;
    }
  }
  __syncthreads();

  // ---- 2-CTA pair tables: natural order (layer1) and claim order (layer0) ----
  // A pair's claim key is the key of its last 128-row half, i.e. its position
  // in the reference order of 128-row tiles: locality-first is preserved.
  auto pair_of = [&](int idx, int& j, int& prow, int& valid, long long& key) {
    int lo = 0, hi = Er - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_p0[mid] <= idx) lo = mid; else hi = mid - 1;
    }
    j = lo;
    const int c = s_cnt[j];
    const int r0 = (idx - s_p0[j]) * kPairRows;
    prow = s_pad[j] + r0;
    valid = min(kPairRows, c - r0);
    const int last_rs = r0 + (valid > kTileRows ? kTileRows : 0);
    const int last_re = min(last_rs + kTileRows, c);
    const int nd = (last_re - last_rs) - max(0, min(last_re, s_nloc[j]) - last_rs);
    // streamed forward: row-tile-major across experts, so the first pairs
    // need only the first token chunks of the upload
    key = (ix.flags & kIndexStream) ? tile_key(r0 / kPairRows, ix.e_lo + j, r0) : tile_key(nd, ix.e_lo + j, last_rs);
  };
  long long* s_pkey = sh_keys;  // P keys (P <= kSortSmemKeys, else recomputed)
  const bool pkeys_in_smem = P <= kSortSmemKeys;
  if (!ovf) {
    if (pkeys_in_smem) {
      for (int i = tid; i < P; i += kThreads) {
        int j, prow, valid;
        long long key;
        pair_of(i, j, prow, valid, key);
        s_pkey[i] = key;
      }
      __syncthreads();
    }
    for (int i = tid; i < P; i += kThreads) {
      int j, prow, valid;
      long long key;
      pair_of(i, j, prow, valid, key);
      int* o = ix.pairs1 + (s_pord[j] + (i - s_p0[j])) * 4;
      int rank = 0;
      for (int q = 0; q < P; ++q) {
        long long kq;
        if (pkeys_in_smem) {
          kq = s_pkey[q];
        } else {
          int jq, pq, vq;
          pair_of(q, jq, pq, vq, kq);
        }
        rank += kq < key;
      }
      ix.pair_key[i] = rank;
      ix.claim_of_tile[prow >> 7] = 2 * rank;
      if (valid > kTileRows) ix.claim_of_tile[(prow >> 7) + 1] = 2 * rank + 1;
      // .w: bit h set when 128-row half h holds rows pulled from other ranks
      const int r0 = prow - s_pad[j];
      // streamed forward: every row is pulled by the dispatch CTAs (gated on
      // its upload chunk), so every populated half waits for its tile
      const int remote_mask = (ix.flags & kIndexStream)
                                  ? (1 | (valid > kTileRows ? 2 : 0))
                                  : ((min(r0 + kTileRows, s_cnt[j]) > s_nloc[j] ? 1 : 0) |
                                     (valid > kTileRows && r0 + valid > s_nloc[j] ? 2 : 0));
      o[0] = j; o[1] = prow; o[2] = valid; o[3] = remote_mask;
      int* o0 = ix.pairs0 + rank * 4;
      o0[0] = j; o0[1] = prow; o0[2] = valid; o0[3] = remote_mask;
    }
  }
  __syncthreads();

  const int Rpad = s_pad[Er];
  if (tid == 0) s_misc[2] = 0;  // pull list retired: remote rows are pulled per tile (comm.cuh)
  __syncthreads();

  // ---- streamed forward: the fused-combine folder of each token is its
  // hosted row in the LATEST (row tile, expert) pair -- every other row it
  // folds is claimed earlier, so fold waits never point forward ----
  if (ix.flags & kIndexStream) {  // every item CTA's rows (tok_pos) are in place
    if (tid == 0) {
      ptx::Spin sp;
      while (ptx::ld_acquire_gpu(ix.done) < gridDim.x - 1) sp.pause(32, 15);
      *ix.done = 0u;
    }
    __syncthreads();
  }
  if ((ix.flags & kIndexStream) && !ovf) {
    for (int t = tid; t < M; t += kThreads) {
      const int32_t* trow = ix.experts + static_cast<long long>(t) * K;
      long long best = -1;
      int best_s = -1;
      for (int s2 = 0; s2 < K; ++s2) {
        const int pos = __ldcg(ix.tok_pos + static_cast<long long>(t) * K + s2);
        if (pos < 0) continue;
        const int j = trow[s2] - ix.e_lo;
        const long long key = (static_cast<long long>((pos - s_pad[j]) / kPairRows) << 21) | j;
        if (key > best) { best = key; best_s = s2; }
      }
      const int sr = src_rank_of(t, M, W);
      const int slot = (W > 1 ? ix.rank * ix.mloc_cap : 0) + t - token_start_of(sr, M, W);
      for (int s2 = 0; s2 < K; ++s2) {
        const int pos = __ldcg(ix.tok_pos + static_cast<long long>(t) * K + s2);
        if (pos >= 0 && pos < ix.cap_rows_pad) ix.row_dst[pos] = s2 == best_s ? ((sr << 24) | slot) : -1;
      }
    }
    __syncthreads();
  }

  // ---- combine token list: tokens with >=1 hosted expert, ascending ----
  if (ix.flags & kIndexCombineList) {
    const int per = (M + kThreads - 1) / kThreads;
    uint64_t hits = 0;  // bit q: token tid*per+q has a hosted expert (per <= 64)
#pragma unroll 8
    for (int q = 0; q < per; ++q) {
      const int t = tid * per + q;
      int f = 0;
      if (t < M) {
        const int32_t* row = ix.experts + static_cast<long long>(t) * K;
        for (int s2 = 0; s2 < K; ++s2) {
          const int ev = __ldg(row + s2);
          f += (ev >= ix.e_lo && ev < ix.e_lo + Er);
        }
      }
      hits |= static_cast<uint64_t>(f > 0) << q;
    }
    int tot;
    int pos = block_scan(__popcll(hits), s_ws, &tot);
    for (int q = 0; q < per; ++q)
      if ((hits >> q) & 1) ix.combine_tok[pos++] = tid * per + q;
    if (tid == 0) s_misc[3] = tot;
  } else if (tid == 0) {
    s_misc[3] = 0;
  }
  __syncthreads();

  probe(5);
  if (tid == 0) {
    ix.meta[kMetaRows] = s_off[Er];
    ix.meta[kMetaRowsPad] = Rpad;
    ix.meta[kMetaTiles0] = T0;
    ix.meta[kMetaPairs] = P;
    ix.meta[kMetaPull] = ovf ? 0 : s_misc[2];
    ix.meta[kMetaTiles1] = static_cast<int>(T1);
    ix.meta[kMetaChunks] = NCH;
    ix.meta[kMetaCombineTok] = s_misc[3];
    ix.meta[kMetaSlots - 1] = (ovf ? 1 : 0) | (ovf1 ? 2 : 0);
  }
}

}  // namespace comet

// host: this unit's device-wait timeout (ptx::Spin)
cudaError_t set_spin_timeout_index(unsigned long long ns) {
  return cudaMemcpyToSymbol(comet::ptx::g_spin_timeout_ns, &ns, sizeof(ns));
}
cudaError_t set_abort_flag_index(const volatile uint32_t* p) {
  return cudaMemcpyToSymbol(comet::ptx::g_abort_flag, &p, sizeof(p));
}
