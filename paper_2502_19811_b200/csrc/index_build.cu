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
// stable stream compaction of the rotated token sequence -- one CTA per hosted
// expert, block-wide ballot scans, no sort.
//
// One launch: CTAs [0, E_r) build the per-expert layouts; CTA E_r writes the
// global counts, the transfer matrix and the non-hosted slots; the last CTA
// to finish (grid-wide completion counter) builds the tile lists, the 2-CTA
// pair tables, the deduplicated NVLink pull list and the combine token list.
#include <climits>
#include <cstdint>

#include "index.cuh"

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

}  // namespace

__global__ void __launch_bounds__(kThreads, 1) index_build_kernel(IndexDev ix) {
  extern __shared__ long long sh_keys[];  // kSortSmemKeys (phase 2 only)
  __shared__ int s_cnt[kMaxExperts];
  __shared__ int s_off[kMaxExperts + 1];
  __shared__ int s_pad[kMaxExperts + 1];
  __shared__ int s_ws[kWarps];
  __shared__ int s_misc[8];

  const int tid = threadIdx.x;
  const int M = ix.M, K = ix.topk, W = ix.world, E = ix.E, Er = ix.E_r;

  // -------- phase 0 (every CTA): global histogram + hosted offsets --------
  for (int e = tid; e < E; e += kThreads) s_cnt[e] = 0;
  __syncthreads();
  for (int i0 = 0; i0 < M * K; i0 += kThreads) {
    const int i = i0 + tid;
    warp_add(s_cnt, i < M * K ? ix.experts[i] : 0, i < M * K);
  }
  __syncthreads();
  if (tid == 0) {
    int o = 0, p = 0;
    for (int j = 0; j < Er; ++j) {
      s_off[j] = o;
      s_pad[j] = p;
      const int c = s_cnt[ix.e_lo + j];
      o += c;
      p += (c + kPairRows - 1) / kPairRows * kPairRows;
    }
    s_off[Er] = o;
    s_pad[Er] = p;
  }
  __syncthreads();

  const int start = token_start_of(ix.rank, M, W);
  const int n_own = token_stop_of(ix.rank, M, W) - start;

  if (blockIdx.x < Er) {
    // -------- per-expert layout: rotated-token stream compaction --------
    const int j = blockIdx.x, e = ix.e_lo + j;
    const int base_row = s_off[j], base_pad = s_pad[j];
    int running = 0, n_loc = 0;
    for (int c0 = 0; c0 < M; c0 += kThreads) {
      const int i = c0 + tid;
      int t = -1, s = -1;
      if (i < M) {
        t = start + i;
        if (t >= M) t -= M;
        s = slot_of(ix.experts + static_cast<long long>(t) * K, K, e);
      }
      const int f = s >= 0 ? 1 : 0;
      int tot;
      const int pos = running + block_scan(f, s_ws, &tot);
      if (f) {
        if (base_row + pos < ix.cap_rows) {
          ix.row_token[base_row + pos] = t;
          ix.row_src[base_row + pos] = src_rank_of(t, M, W);
        }
        if (base_pad + pos < ix.cap_rows_pad) ix.gather_row[base_pad + pos] = t;
        ix.tok_pos[static_cast<long long>(t) * K + s] = base_pad + pos;
      }
      if (i < n_own) n_loc += f;
      running += tot;
    }
    // local rows are exactly the rotated prefix [0, n_own)
    int tot;
    block_scan(n_loc, s_ws, &tot);
    if (tid == 0) ix.n_local[j] = tot;
    for (int r = base_pad + running + tid; r < s_pad[j + 1]; r += kThreads)
      if (r < ix.cap_rows_pad) ix.gather_row[r] = -1;
  } else {
    // -------- bookkeeping CTA: counts, transfer matrix, foreign slots --------
    int* s_tr = reinterpret_cast<int*>(sh_keys);  // W*W <= 4096 ints (host-checked)
    for (int e = tid; e < E; e += kThreads) ix.counts[e] = s_cnt[e];
    for (int i = tid; i < W * W; i += kThreads) s_tr[i] = 0;
    __syncthreads();
    const int per_group = E / ix.ep;
    for (int i0 = 0; i0 < M * K; i0 += kThreads) {
      const int i = i0 + tid;
      const bool ok = i < M * K;
      const int t = ok ? i / K : 0, e = ok ? ix.experts[i] : 0;
      const int src = src_rank_of(t, M, W);
      const int g = e / per_group;
      for (int d = 0; d < ix.tp; ++d) warp_add(s_tr, src * W + g * ix.tp + d, ok);
      if (ok && (e < ix.e_lo || e >= ix.e_lo + Er)) ix.tok_pos[i] = -1;
    }
    for (int i = tid; i < ix.n_zero_words; i += kThreads) ix.zero_words[i] = 0u;
    __syncthreads();
    for (int i = tid; i < W * W; i += kThreads) ix.transfer[i] = s_tr[i];
  }

  // -------- grid completion: the last CTA builds the schedules --------
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(ix.done, 1u);
    s_misc[1] = (prev == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (!s_misc[1]) return;
  __threadfence();

  // recompute hosted offsets (s_off may have been reused as scratch)
  if (tid == 0) {
    int o = 0, p = 0;
    for (int j = 0; j < Er; ++j) {
      s_off[j] = o;
      s_pad[j] = p;
      const int c = s_cnt[ix.e_lo + j];
      o += c;
      p += (c + kPairRows - 1) / kPairRows * kPairRows;
    }
    s_off[Er] = o;
    s_pad[Er] = p;
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
  __shared__ int s_nloc[kMaxExperts];
  for (int j = tid; j < Er; j += kThreads) s_nloc[j] = __ldcg(ix.n_local + j);
  __syncthreads();
  if (tid == 0) {
    int t = 0, p = 0;
    for (int j = 0; j < Er; ++j) {
      s_t0[j] = t;
      s_p0[j] = p;
      const int c = s_cnt[ix.e_lo + j];
      t += (c + TR - 1) / TR;
      p += (c + kPairRows - 1) / kPairRows;
    }
    s_t0[Er] = t;
    s_p0[Er] = p;
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
    const int c = s_cnt[ix.e_lo + j];
    rs = (idx - s_t0[j]) * TR;
    re = min(rs + TR, c);
    const int loc_end = min(re, s_nloc[j]);
    nd = (re - rs) - max(0, loc_end - rs);
  };
  const bool keys_in_smem = T0 <= kSortSmemKeys;
  if (!ovf) {
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
  const int C = (NE + TC - 1) / TC;
  const long long T1 = static_cast<long long>(C) * T0;
  const bool ovf1 = T1 > ix.cap_tiles1;
  if (!ovf && !ovf1) {
    for (long long i = tid; i < T1; i += kThreads) {
      const int c = static_cast<int>(i / T0), q = static_cast<int>(i % T0);
      int j, rs, re, nd;
      tile_of(q, j, rs, re, nd);
      int* o = ix.tiles1 + i * 6;
      o[0] = ix.e_lo + j; o[1] = rs; o[2] = re;
      o[3] = c * TC; o[4] = min(c * TC + TC, NE); o[5] = nd;
    }
    for (int c = tid; c < C; c += kThreads) {
      int* o = ix.chunks + c * 4;
      o[0] = c * TC; o[1] = min(c * TC + TC, NE); o[2] = c * T0; o[3] = T0;
    }
  }

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
    const int c = s_cnt[ix.e_lo + j];
    const int r0 = (idx - s_p0[j]) * kPairRows;
    prow = s_pad[j] + r0;
    valid = min(kPairRows, c - r0);
    const int last_rs = r0 + (valid > kTileRows ? kTileRows : 0);
    const int last_re = min(last_rs + kTileRows, c);
    const int nd = (last_re - last_rs) - max(0, min(last_re, s_nloc[j]) - last_rs);
    key = tile_key(nd, ix.e_lo + j, last_rs);
  };
  if (!ovf) {
    for (int i = tid; i < P; i += kThreads) {
      int j, prow, valid;
      long long key;
      pair_of(i, j, prow, valid, key);
      int* o = ix.pairs1 + i * 4;
      o[0] = j; o[1] = prow; o[2] = valid; o[3] = 0;
      int rank = 0;
      for (int q = 0; q < P; ++q) {
        int jq, pq, vq;
        long long kq;
        pair_of(q, jq, pq, vq, kq);
        rank += kq < key;
      }
      ix.pair_key[i] = rank;
      // .w: bit h set when 128-row half h holds rows pulled from other ranks
      const int r0 = prow - s_pad[j];
      const int remote_mask = (min(r0 + kTileRows, s_cnt[ix.e_lo + j]) > s_nloc[j] ? 1 : 0) |
                              (valid > kTileRows && r0 + valid > s_nloc[j] ? 2 : 0);
      int* o0 = ix.pairs0 + rank * 4;
      o0[0] = j; o0[1] = prow; o0[2] = valid; o0[3] = remote_mask;
      o[3] = remote_mask;
    }
  }
  __syncthreads();

  const int Rpad = s_pad[Er];
  if (tid == 0) s_misc[2] = 0;  // pull list retired: remote rows are pulled per tile (comm.cuh)
  __syncthreads();

  // ---- combine token list: tokens with >=1 hosted expert, ascending ----
  {
    int running = 0;
    for (int c0 = 0; c0 < M; c0 += kThreads) {
      const int t = c0 + tid;
      int f = 0;
      if (t < M) {
        const int32_t* row = ix.experts + static_cast<long long>(t) * K;
        for (int s = 0; s < K; ++s) f |= (row[s] >= ix.e_lo && row[s] < ix.e_lo + Er);
      }
      int tot;
      const int pos = running + block_scan(f, s_ws, &tot);
      if (f) ix.combine_tok[pos] = t;
      running += tot;
    }
    if (tid == 0) s_misc[3] = running;
  }
  __syncthreads();

  if (tid == 0) {
    ix.meta[kMetaRows] = s_off[Er];
    ix.meta[kMetaRowsPad] = Rpad;
    ix.meta[kMetaTiles0] = T0;
    ix.meta[kMetaPairs] = P;
    ix.meta[kMetaPull] = ovf ? 0 : s_misc[2];
    ix.meta[kMetaTiles1] = static_cast<int>(T1);
    ix.meta[kMetaChunks] = C;
    ix.meta[kMetaCombineTok] = s_misc[3];
    ix.meta[kMetaSlots - 1] = (ovf ? 1 : 0) | (ovf1 ? 2 : 0);
    *ix.done = 0u;  // self-reset for the next launch
  }
}

}  // namespace comet
