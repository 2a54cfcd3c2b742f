// Communication-CTA roles of the fused layer kernels (section 3.2.1,
// thread-block specialisation).  A communication CTA is a TMA bulk-copy
// engine: a loader warp computes the descriptors of kBatch jobs at a time
// (lane-parallel index loads), then each lane streams its job's row segments
// -- from local HBM or NVLink-mapped peer memory -- into its own smem ring
// slot; consumer warps drain the slots (bulk-store them, or reduce them).
#pragma once

#include <cuda_bf16.h>

#include "layers.cuh"
#include "ptx.cuh"

namespace comet {
namespace comm {

constexpr int kMaxSlots = 224;
constexpr int kReducers = 7;               // combine: warps 1..7 (higher warps idle)
constexpr int kBatch = 16;                 // jobs described per loader pass
constexpr uint32_t kRingBytes = 192 * 1024;
#ifndef COMET_FREE_LAG
#define COMET_FREE_LAG 2
#endif
constexpr int kFreeLag = COMET_FREE_LAG;   // dispatch: bulk-store groups in flight before a slot is reused
#ifndef COMET_PUB_LAG
#define COMET_PUB_LAG 8
#endif
constexpr int kPubLag = COMET_PUB_LAG;     // dispatch: groups in flight before a tile is published
constexpr int kJobSlots = 64;              // dedup dispatch ring slots (job descriptions in smem)
constexpr int kPubBatch = 8;               // dedup dispatch: completed jobs counted per publication pass

struct JobDesc {
  __nv_bfloat16* dst;
  float w[8];
};

struct CommSmem {
  uint64_t full[kMaxSlots];
  uint64_t empty[kMaxSlots];
  JobDesc desc[kMaxSlots];
  int pub_tile[64];  // tile | rows << 16 of a pending dispatch chunk
  int pub_rows[64];  // remote rows of that tile
  int pub_job[64];
  int2 pub_q[64][8];            // dedup dispatch: (claim tile, its pulled-row count) per destination
  int job_n[kJobSlots];         // dedup dispatch job in a ring slot: destination rows (<= 8)
  int4 job_dq[kJobSlots][8];    // (padded row, claim tile, tile's pulled-row count) per destination
  unsigned long long pub_t0[64];
  const __nv_bfloat16* xs_peer[kMaxWorld];
};

// Timeline record of a communication task (same buffer/format as the compute
// roles, moe_layers.cu tl_record): role kRoleComm, task = tile or n-block id.
__device__ __forceinline__ void comm_record(const LayerArgs& p, int idx, int task, uint64_t t0, uint64_t t1) {
  if (p.timeline == nullptr || idx >= p.timeline_cap) return;
  unsigned long long* r = p.timeline + ((static_cast<long long>(blockIdx.x) * kRoles + kRoleComm) * p.timeline_cap + idx) * 2;
  r[0] = t0;
  r[1] = (t1 - t0) | (static_cast<unsigned long long>(task + 1) << 40);
}

// Layer1 (world > 1): one contributor finished its rows of column block nb --
// a compute CTA's 128 epilogue-pushed rows of one unit (2 per full unit, 1
// per 256-column half unit), or a combine CTA's reduced tokens (1).  The
// contributor completing the count (4 per pair + one per combine CTA)
// publishes the block to every peer's combine flags.
__device__ __forceinline__ void nb_contributed(const LayerArgs& p, int nb, uint32_t amount, uint32_t target) {
  ptx::fence_acq_rel_sys();
  const uint32_t prev = ptx::atom_acq_rel_gpu_add(p.nb_sent + nb, amount);
  if (prev + amount == target) {
    ptx::fence_acq_rel_sys();
    for (int d = 0; d < p.world; ++d) ptx::st_release_sys(p.cb_flag_peer[d] + p.rank * p.n_blocks + nb, p.epoch);
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ CommSmem* comm_smem(uint8_t* smem) {
  return reinterpret_cast<CommSmem*>(smem + kRingBytes);
}

__device__ __forceinline__ void comm_init(const LayerArgs& p, uint8_t* smem, int n_slots) {
  CommSmem* cs = comm_smem(smem);
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_slots; ++i) {
      ptx::mbar_init(cs->full + i, 1);
      ptx::mbar_init(cs->empty + i, 1);
    }
    ptx::fence_mbar_init();
  }
  if (static_cast<int>(threadIdx.x) < p.world)  // zero-copy forward: the tokens come from pinned host memory
    cs->xs_peer[threadIdx.x] = p.host_src ? p.host_src : p.xs_peer[threadIdx.x];
  __syncthreads();
}

// Remote (NVLink) rows of 128-row tile q of the claim-ordered pair table: the
// local rows of every expert block are a prefix (resolver.py:171-195) and were
// already placed by dispatch_local_kernel, so a tile's remote rows are the
// suffix [padrow0, padrow0 + nr).  Returns false for tiles without any.
__device__ __forceinline__ bool remote_rows(const LayerArgs& p, int q, int& padrow0, int& nr) {
  const int4 pr = reinterpret_cast<const int4*>(p.pairs)[q >> 1];
  const int base = pr.y + kTileRows * (q & 1);
  const int rows = max(0, min(kTileRows, pr.z - kTileRows * (q & 1)));
  if (p.pull_local) {  // every row of every populated half (local rows included)
    padrow0 = base;
    nr = rows;
    return nr > 0;
  }
  if (!((pr.w >> (q & 1)) & 1)) return false;
  const int rel = base - p.pad_off[pr.x];                        // tile start within the expert block
  const int first = min(rows, max(0, p.n_local[pr.x] - rel));      // first remote row
  padrow0 = base + first;
  nr = rows - first;
  return nr > 0;
}

// A dispatch CTA that finished joins the compute pairs: its smem becomes
// stage buffers, so retire the ring barriers first (every bulk copy has
// completed: the storer waited for all groups, the loads were all consumed).
__device__ __forceinline__ void comm_release(const LayerArgs& p, uint8_t* smem) {
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_embed) * 2u;
  const int n_slots = min(p.dedup ? kJobSlots : kMaxSlots, static_cast<int>(kRingBytes / row_bytes));
  CommSmem* cs = comm_smem(smem);
  for (int i = threadIdx.x; i < n_slots; i += blockDim.x) {
    ptx::mbar_inval(cs->full + i);
    ptx::mbar_inval(cs->empty + i);
  }
}

// Dispatch work items: chunks of chunk_rows (default 32) remote rows of one 128-row tile,
// enumerated in the compute schedule's claim order (tile-major) and dealt
// round-robin to the dispatch CTAs, so a tile's rows are pulled by several
// CTAs at once.  fn(q, padrow0, r_begin, r_end, nr) for this CTA's items,
// called warp-uniformly.  Called by a whole warp: the lanes read the pair
// table of 32 tiles at once (a tile-by-tile walk is one dependent L2 round
// trip per tile -- ~16 per item at 64 dispatch CTAs, which made the walk, not
// the copies, set the dispatch rate: 0.6-0.9 us per row per CTA).
template <class F>
__device__ __forceinline__ void for_my_items(const LayerArgs& p, int cid, int n_comm, F&& fn) {
  const int lane = threadIdx.x & 31;
  const int n_tiles = 2 * p.meta[kMetaPairs];
  const int chunk = p.chunk_rows;  // 1..32
  int item = 0;
  for (int q0 = 0; q0 < n_tiles; q0 += 32) {
    int pr0 = 0, nr = 0;
    if (q0 + lane >= n_tiles || !remote_rows(p, q0 + lane, pr0, nr)) nr = 0;
    // items of each tile of the batch; this CTA's first item in each
    const int n_items = (nr + chunk - 1) / chunk;
    int before = n_items;  // inclusive prefix sum -> items before this lane's tile
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, before, o);
      if (lane >= o) before += v;
    }
    before -= n_items;
    unsigned has = __ballot_sync(0xffffffffu, n_items > 0 && ((cid - (item + before)) % n_comm + n_comm) % n_comm < n_items);
    while (has) {
      const int j = __ffs(has) - 1;
      has &= has - 1;
      const int nrj = __shfl_sync(0xffffffffu, nr, j);
      const int prj = __shfl_sync(0xffffffffu, pr0, j);
      const int bj = item + __shfl_sync(0xffffffffu, before, j);
      const int nij = (nrj + chunk - 1) / chunk;
      for (int i = ((cid - bj) % n_comm + n_comm) % n_comm; i < nij; i += n_comm)
        fn(q0 + j, prj, i * chunk, min(nrj, (i + 1) * chunk), nrj);
    }
    item += __shfl_sync(0xffffffffu, before + n_items, 31);
  }
}

// layer0 dispatch: fill the remote rows of the expert-sorted shared tensor xg
// (local rows were placed by dispatch_local_kernel) in the compute schedule's
// claim order (locality-first, resolver.py:206-252), pulling each row over
// NVLink from its source rank's token buffer.  A tile is published (ready
// epoch) by whichever CTA lands its last chunk (per-tile row counters).
__device__ void dispatch_rows(const LayerArgs& p, uint8_t* smem) {
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_embed) * 2u;  // <= kRingBytes / 8 (host-checked)
  const int n_slots = min(kMaxSlots, static_cast<int>(kRingBytes / row_bytes));
  comm_init(p, smem, n_slots);
  CommSmem* cs = comm_smem(smem);
  const int n_comm = gridDim.x - p.n_compute;
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    // ---- loader warp: lane-parallel index loads for a chunk, then lane 0
    // issues them in job order (slot waits never couple lanes of one batch) ----
    uint64_t ready_mask = 1ull << p.rank;
    int chunk_ok = -1;  // streamed forward: upload chunks [0, chunk_ok] are in HBM
    int k = 0;
    for_my_items(p, cid, n_comm, [&](int q, int padrow0, int rb, int re, int nr) {
      const int n = re - rb;
      const int t = lane < n ? p.gather_row[padrow0 + rb + lane] : 0;
      const int src = src_rank_of(t, p.M, p.world);
      // source ranks this item reads whose tokens are not known ready: every
      // such flag polled at once, one lane each (one system-scope round trip
      // instead of one per source rank)
      unsigned long long need = 0;
      for (int i = 0; i < n; ++i) need |= 1ull << __shfl_sync(0xffffffffu, src, i);
      need &= ~ready_mask;
      if (need) {
        for (int r = lane; r < p.world; r += 32)
          if ((need >> r) & 1) {
            ptx::Spin sp;
            while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.x_ready + r), p.epoch)) sp.pause(64, 7);
          }
        __syncwarp();
        ready_mask |= need;
      }
      for (int i = 0; i < n; ++i) {
        const int ti = __shfl_sync(0xffffffffu, t, i);
        const int si = __shfl_sync(0xffffffffu, src, i);
        if (lane == 0) {
          if (p.chunk_ready && ti / p.chunk_tokens > chunk_ok) {  // chunks land in order
            const int c = ti / p.chunk_tokens;
            { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.chunk_ready + c), p.epoch)) sp.pause(128, 8); }
            chunk_ok = c;
          }
          const int job = k + i;
          const int slot = job % n_slots;
          ptx::mbar_wait(cs->empty + slot, ((job / n_slots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(cs->full + slot, row_bytes);
          ptx::bulk_load(smem + slot * row_bytes, cs->xs_peer[si] + static_cast<long long>(ti) * p.n_embed,
                         row_bytes, cs->full + slot);
        }
      }
      k += n;
      __syncwarp();
    });
  } else if (warp == 1) {
    // ---- storer (lane 0; the warp walks the items): slot -> xg row; count
    // each chunk once its writes landed ----
    int k = 0, head = 0, tail = 0, n_rec = 0;
    auto publish_upto = [&](int done_job) {
      while (head != tail && cs->pub_job[head & 63] <= done_job) {
        const int e = head & 63;
        const int q = cs->pub_tile[e] & 0xFFFF, rows = cs->pub_tile[e] >> 16;
        const int nr = cs->pub_rows[e];
        ptx::fence_async_global();
        // end stamp taken before the count / release: a consumer that observes
        // the tile's flag always stamps a later time (measured dependency audit)
        const unsigned long long t_done = ptx::globaltimer();
        comm_record(p, n_rec++, q, cs->pub_t0[e], t_done);
        const uint32_t prev = ptx::atom_acq_rel_gpu_add(p.xg_cnt + q, static_cast<uint32_t>(rows));
        if (prev + static_cast<uint32_t>(rows) == static_cast<uint32_t>(nr)) {
          // last chunk of tile q: every CTA's rows are visible (acq_rel chain)
          p.xg_cnt[q] = 0u;  // no other access this launch; ready for the next
          ptx::st_release_gpu(p.xg_ready + q, p.epoch);
        }
        ++head;
      }
    };
    for_my_items(p, cid, n_comm, [&](int q, int padrow0, int rb, int re, int nr) {
      if (lane != 0) return;
      const unsigned long long t_item = ptx::globaltimer();
      for (int r = rb; r < re; ++r, ++k) {
        const int slot = k % n_slots;
        ptx::mbar_wait(cs->full + slot, (k / n_slots) & 1);
        ptx::bulk_store(p.xg + static_cast<long long>(padrow0 + r) * p.n_embed, smem + slot * row_bytes, row_bytes);
        ptx::bulk_commit();
        ptx::bulk_wait_read<kFreeLag>();
        if (k >= kFreeLag) ptx::mbar_arrive(cs->empty + (k - kFreeLag) % n_slots);
        if (k >= kPubLag) {
          ptx::bulk_wait<kPubLag>();
          publish_upto(k - kPubLag);
        }
      }
      const int e = tail & 63;
      cs->pub_tile[e] = q | ((re - rb) << 16);
      cs->pub_rows[e] = nr;
      cs->pub_job[e] = k - 1;
      cs->pub_t0[e] = t_item;
      ++tail;
      if (tail - head >= 60) {
        ptx::bulk_wait<0>();
        publish_upto(k);
      }
    });
    if (lane == 0) {
      ptx::bulk_wait<0>();
      publish_upto(k);
    }
  }
}

// Dedup (a7: one read per (token, rank)): the row of token t that pulls it is
// its hosted row in the earliest-claimed tile (ties: lower slot); the smem
// copy is bulk-stored to every hosted row of t.  One lane per row computes
// the row's job: whether it is the primary row and, if so, the destinations
// (padded row, claim tile, the tile's rows).  The loads are issued level by
// level over all top-k slots (tok_pos, then claim_of_tile, then the pair
// table) -- three dependent round trips per batch of 32 rows instead of a
// chain of ~3 per slot, which had made the loader's descriptor math, not the
// copies, set the dedup dispatch rate (QW EP=8: 112 vs 40 us).
__device__ __forceinline__ int dedup_job(const LayerArgs& p, int t, int pos, int4 (&dst)[8]) {
  const int K = p.topk;  // <= 8 (host-checked)
  int dpos[8], dq[8];
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2) dpos[s2] = s2 < K ? p.tok_pos[t * K + s2] : -1;
  const int my_s = p.row_widx[pos] - t * K;
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2) dq[s2] = dpos[s2] >= 0 ? p.claim_of_tile[dpos[s2] >> 7] : 0;
  int my_q = 0;
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2)
    if (s2 == my_s) my_q = dq[s2];
  bool prim = true;
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2)
    if (s2 != my_s && dpos[s2] >= 0 && (dq[s2] < my_q || (dq[s2] == my_q && s2 < my_s))) prim = false;
  if (!prim) return -1;
  int4 pr[8];
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2)
    if (dpos[s2] >= 0) pr[s2] = reinterpret_cast<const int4*>(p.pairs)[dq[s2] >> 1];
  int nd = 0;
#pragma unroll
  for (int s2 = 0; s2 < 8; ++s2) {
    if (dpos[s2] < 0) continue;
    // remote_rows() of claim tile dq: its populated rows (pull_local) or the
    // remote suffix of the expert block
    const int h = dq[s2] & 1;
    const int base = pr[s2].y + kTileRows * h;
    const int rows = max(0, min(kTileRows, pr[s2].z - kTileRows * h));
    int nrd = rows;
    if (!p.pull_local) {
      const int rel = base - p.pad_off[pr[s2].x];
      nrd = rows - min(rows, max(0, p.n_local[pr[s2].x] - rel));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j == nd) dst[j] = make_int4(dpos[s2], dq[s2], nrd, 0);
    ++nd;
  }
  return nd;
}

// layer0 dispatch, deduplicated per token (used by the zero-copy single-GPU
// forward, where every byte crosses PCIe): items in claim order as in
// dispatch_rows; the loader describes each job (destinations, their claim
// tiles and tile sizes) in smem, the storer fans the smem copy out and counts
// landed rows per claim tile in batches.
__device__ void dispatch_rows_dedup(const LayerArgs& p, uint8_t* smem) {
  const uint32_t row_bytes = static_cast<uint32_t>(p.n_embed) * 2u;
  const int n_slots = min(kJobSlots, static_cast<int>(kRingBytes / row_bytes));
  comm_init(p, smem, n_slots);
  CommSmem* cs = comm_smem(smem);
  const int n_comm = gridDim.x - p.n_compute;
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    uint64_t ready_mask = 1ull << p.rank;
    int k = 0;
    for_my_items(p, cid, n_comm, [&](int q, int padrow0, int rb, int re, int nr) {
      const int n = re - rb;
      const int pos = padrow0 + rb + lane;
      const int t = lane < n ? p.gather_row[pos] : 0;
      int4 dst[8];
      int nd = lane < n ? dedup_job(p, t, pos, dst) : -1;
      const bool prim = nd >= 0;
      const unsigned pm = __ballot_sync(0xffffffffu, prim);
      const int src = src_rank_of(t, p.M, p.world);
      nd = max(nd, 0);
      int jj = k;  // job index of this lane's row
      for (int i = 0; i < lane; ++i) jj += (pm >> i) & 1;
      for (int i = 0; i < n; ++i) {
        if (!((pm >> i) & 1)) continue;
        const int ti = __shfl_sync(0xffffffffu, t, i);
        const int si = __shfl_sync(0xffffffffu, src, i);
        if (lane == 0) ptx::mbar_wait(cs->empty + k % n_slots, ((k / n_slots) & 1) ^ 1);
        __syncwarp();
        if (lane == i) {  // the slot is free: describe the job for the storer
          cs->job_n[jj % n_slots] = nd;
          for (int q2 = 0; q2 < nd; ++q2) cs->job_dq[jj % n_slots][q2] = dst[q2];
        }
        __syncwarp();
        if (lane == 0) {
          if (!((ready_mask >> si) & 1)) {
            { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.x_ready + si), p.epoch)) sp.pause(64, 9); }
            ready_mask |= 1ull << si;
          }
          const int slot = k % n_slots;
          ptx::mbar_arrive_expect_tx(cs->full + slot, row_bytes);  // release: job description visible
          ptx::bulk_load(smem + slot * row_bytes, cs->xs_peer[si] + static_cast<long long>(ti) * p.n_embed,
                         row_bytes, cs->full + slot);
        }
        ++k;
      }
      __syncwarp();
    });
    if (lane == 0) {  // sentinel: no more jobs (arrival without bytes completes the phase)
      const int slot = k % n_slots;
      ptx::mbar_wait(cs->empty + slot, ((k / n_slots) & 1) ^ 1);
      cs->job_n[slot] = -1;
      ptx::mbar_arrive(cs->full + slot);
    }
  } else if (warp == 1 && lane == 0) {
    int k = 0, head = 0, tail = 0, n_rec = 0;
    constexpr int kAcc = 8;
    int acc_q[kAcc], acc_n[kAcc], acc_nr[kAcc];
    unsigned long long acc_t0[kAcc];
    int n_acc = 0;
    auto flush = [&](unsigned long long t_done) {
      for (int i = 0; i < n_acc; ++i) {
        const int qd = acc_q[i], nrd = acc_nr[i];
        const uint32_t prev = ptx::atom_acq_rel_gpu_add(p.xg_cnt + qd, static_cast<uint32_t>(acc_n[i]));
        if (prev + static_cast<uint32_t>(acc_n[i]) == static_cast<uint32_t>(nrd)) {
          p.xg_cnt[qd] = 0u;  // last rows of claim tile qd; ready for the next launch
          comm_record(p, n_rec++, qd, acc_t0[i], t_done);
          ptx::st_release_gpu(p.xg_ready + qd, p.epoch);
        }
      }
      n_acc = 0;
    };
    auto publish_upto = [&](int done_job) {
      if (head == tail || cs->pub_job[head & 63] > done_job) return;
      ptx::fence_async_global();
      const unsigned long long t_done = ptx::globaltimer();
      while (head != tail && cs->pub_job[head & 63] <= done_job) {
        const int e = head & 63;
        for (int s2 = 0; s2 < cs->pub_tile[e]; ++s2) {
          const int qd = cs->pub_q[e][s2].x, nrd = cs->pub_q[e][s2].y;
          int i = 0;
          while (i < n_acc && acc_q[i] != qd) ++i;
          if (i == n_acc) {
            if (n_acc == kAcc) {
              flush(t_done);
              i = 0;
            }
            acc_q[i] = qd;
            acc_nr[i] = nrd;
            acc_n[i] = 0;
            acc_t0[i] = cs->pub_t0[e];
            n_acc = i + 1;
          }
          ++acc_n[i];
        }
        ++head;
      }
      flush(t_done);
    };
    for (;; ++k) {  // jobs in the loader's order until its sentinel
      const unsigned long long t_job = ptx::globaltimer();
      const int slot = k % n_slots;
      ptx::mbar_wait(cs->full + slot, (k / n_slots) & 1);
      const int nd = cs->job_n[slot];
      if (nd < 0) break;
      const int e = tail & 63;
      for (int s2 = 0; s2 < nd; ++s2) {
        const int4 dq = cs->job_dq[slot][s2];
        ptx::bulk_store(p.xg + static_cast<long long>(dq.x) * p.n_embed, smem + slot * row_bytes, row_bytes);
        cs->pub_q[e][s2] = make_int2(dq.y, dq.z);
      }
      ptx::bulk_commit();
      ptx::bulk_wait_read<kFreeLag>();
      if (k >= kFreeLag) ptx::mbar_arrive(cs->empty + (k - kFreeLag) % n_slots);
      cs->pub_tile[e] = nd;
      cs->pub_job[e] = k;
      cs->pub_t0[e] = t_job;
      ++tail;
      if (k >= kPubLag && tail - head >= kPubLag + kPubBatch) {
        ptx::bulk_wait<kPubLag>();
        publish_upto(k - kPubLag);
      }
      if (tail - head >= 60) {
        ptx::bulk_wait<0>();
        publish_upto(k);
      }
    }
    ptx::bulk_wait<0>();
    publish_upto(k);
  }
}

// layer1 combine: once every pair finished column block nb, reduce each
// hosted token's expert rows (ascending slot = ascending expert, weighted when
// combine weights are given; executor.py:102-120) and write the result to the
// output (world == 1) or push the partial row to the token's source rank.
__device__ void combine_reduce(const LayerArgs& p, uint8_t* smem) {
  const int K = p.topk, N = p.n_embed, NB = p.n_blocks;
  constexpr uint32_t kSeg = kBlockN * 2;  // 1 KB of one expert row per 512-column block
  const uint32_t slot_bytes = K * kSeg;
  const int n_slots = min(kMaxSlots, static_cast<int>(kRingBytes / slot_bytes)) / kReducers * kReducers;
  comm_init(p, smem, n_slots);
  CommSmem* cs = comm_smem(smem);
  const int n_comm = gridDim.x - p.n_compute;
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = p.meta[kMetaPairs];
  const int n_tok = p.meta[kMetaCombineTok];
  const uint32_t target = 4u * static_cast<uint32_t>(P);  // nb_done counts 256-column halves per CTA
  const int start_r = token_start_of(p.rank, p.M, p.world);
  const int jobs = n_tok > cid ? (n_tok - cid + n_comm - 1) / n_comm : 0;  // tokens of this CTA per nb
  if (warp == 0) {
    // ---- loader warp ----
    if (p.world > 1) {  // every peer finished its previous forward (epoch barrier)
      if (lane < p.world)
        { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.x_ready + lane), p.epoch)) sp.pause(64, 10); }
      __syncwarp();
    }
    int k = 0;
    for (int nb = 0; nb < NB; ++nb) {
      const int nb_cols = p.out_ld - nb * static_cast<int>(kBlockN);  // a ragged last block <= 256 wide
      const uint32_t nb_target = (nb_cols > 0 && nb_cols <= static_cast<int>(kBlockN / 2)) ? target / 2 : target;
      if (lane == 0)
        { ptx::Spin sp; while (ptx::ld_acquire_gpu(p.nb_done + nb) < nb_target) sp.pause(128, 11); }
      __syncwarp();
      const unsigned long long t_nb = ptx::globaltimer();
      const uint32_t seg = min(kSeg, static_cast<uint32_t>(N - nb * kBlockN) * 2u);
      for (int j0 = 0; j0 < jobs; j0 += kBatch) {
        const int j = j0 + lane;
        if (lane < kBatch && j < jobs) {
          const int t = p.combine_tok[cid + j * n_comm];
          const int job = k + lane;
          const int slot = job % n_slots;
          JobDesc d;
          uint32_t bytes = 0;
          int pos[8];
          for (int s = 0; s < K; ++s) {
            pos[s] = p.tok_pos[t * K + s];
            d.w[s] = pos[s] < 0 ? 0.f : (p.combine_w ? p.combine_w[t * K + s] : 1.f);
            bytes += pos[s] >= 0 ? seg : 0u;
          }
          if (p.world == 1) {
            d.dst = p.y_local + static_cast<long long>(t - start_r) * N + nb * kBlockN;
          } else {
            const int dr = src_rank_of(t, p.M, p.world);
            const int cslot = p.rank * p.mloc_cap + (t - token_start_of(dr, p.M, p.world));
            d.dst = p.cb_peer[dr] + static_cast<long long>(cslot) * N + nb * kBlockN;
          }
          ptx::mbar_wait(cs->empty + slot, ((job / n_slots) & 1) ^ 1);
          cs->desc[slot] = d;
          ptx::mbar_arrive_expect_tx(cs->full + slot, bytes);  // release: desc visible to the reducer
          for (int s = 0; s < K; ++s)
            if (pos[s] >= 0)
              ptx::bulk_load(smem + slot * slot_bytes + s * kSeg,
                             p.yrows + static_cast<long long>(pos[s]) * N + nb * kBlockN, seg, cs->full + slot);
        }
        k += min(kBatch, jobs - j0);
        __syncwarp();
      }
      if (lane == 0) comm_record(p, nb, nb, t_nb, ptx::globaltimer());
    }
    return;
  }
  // ---- reducers: warp w takes jobs k with k % kReducers == w - 1 ----
  if (warp > kReducers) return;  // the layer kernel has more warps than reducers
  const int me = warp - 1;
  int k = 0;
  for (int nb = 0; nb < NB; ++nb) {
    for (int j = 0; j < jobs; ++j, ++k) {
      if (k % kReducers != me) continue;
      const int slot = k % n_slots;
      ptx::mbar_wait(cs->full + slot, (k / n_slots) & 1);
      const JobDesc& d = cs->desc[slot];
      __nv_bfloat16* dst = d.dst;
      float w[8];
      for (int s = 0; s < K; ++s) w[s] = d.w[s];
      uint4 o[kBlockN / 256];
#pragma unroll
      for (int h = 0; h < static_cast<int>(kBlockN / 256); ++h) {  // lane covers 8 columns per 256
        float acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.f;
        for (int s = 0; s < K; ++s) {
          if (w[s] == 0.f) continue;
          const uint4 v =
              *reinterpret_cast<const uint4*>(smem + slot * slot_bytes + s * kSeg + h * 512 + lane * 16);
          const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float2 f = __bfloat1622float2(hv[c]);
            acc[2 * c] += f.x * w[s];
            acc[2 * c + 1] += f.y * w[s];
          }
        }
        o[h].x = pack2(acc[0], acc[1]); o[h].y = pack2(acc[2], acc[3]);
        o[h].z = pack2(acc[4], acc[5]); o[h].w = pack2(acc[6], acc[7]);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(cs->empty + slot);
#pragma unroll
      for (int h = 0; h < static_cast<int>(kBlockN / 256); ++h)
        if (nb * kBlockN + h * 256 + lane * 8 < N) ptx::st_v4(dst + h * 256 + lane * 8, o[h]);
    }
    if (p.world > 1) {
      // all reducers of this CTA finished nb -> count the CTA; last CTA signals peers
      __threadfence_system();
      ptx::named_bar_sync(2, kReducers * 32);
      if (threadIdx.x == 32) {
        const int nb_cols = p.out_ld - nb * static_cast<int>(kBlockN);
        const uint32_t nb_target = (nb_cols > 0 && nb_cols <= static_cast<int>(kBlockN / 2)) ? target / 2 : target;
        nb_contributed(p, nb, 1u, nb_target + static_cast<uint32_t>(n_comm));
      }
    }
  }
}

// Streamed single-GPU forward (comet_forward_host): after their dispatch the
// dispatch CTAs reduce the top-k combine chunk by chunk (token chunk c outer,
// n-block inner) as soon as the layer1 tiles holding the chunk's rows are
// published, write y, and count each chunk's finished halves for the
// download stream (out_cnt).  Layer1 units never wait for each other.
__device__ void stream_combine(const LayerArgs& p, uint8_t* smem) {
  const int K = p.topk, N = p.n_embed, NB = p.n_blocks, M = p.M;
  constexpr uint32_t kSeg = kBlockN * 2;
  const uint32_t slot_bytes = K * kSeg;
  const int n_slots = min(kMaxSlots, static_cast<int>(kRingBytes / slot_bytes)) / kReducers * kReducers;
  comm_init(p, smem, n_slots);
  CommSmem* cs = comm_smem(smem);
  const int n_comm = gridDim.x - p.n_compute;  // (p = layer1 args with n_compute of layer0)
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ct = p.chunk_tokens;
  const int n_ch = (M + ct - 1) / ct;
  auto jobs_of = [&](int c) {
    const int n_tok = min(ct, M - c * ct);
    return n_tok > cid ? (n_tok - cid + n_comm - 1) / n_comm : 0;
  };
  if (warp == 0) {
    int k = 0;
    for (int c = 0; c < n_ch; ++c) {
      const int jobs = jobs_of(c);
      for (int nb = 0; nb < NB; ++nb) {
        const int cols = N - nb * static_cast<int>(kBlockN);
        const int h_hi = cols > static_cast<int>(kBlockN / 2) ? 1 : 0;
        const uint32_t seg = min(kSeg, static_cast<uint32_t>(cols) * 2u);
        for (int j0 = 0; j0 < jobs; j0 += kBatch) {
          const int j = j0 + lane;
          if (lane < kBatch && j < jobs) {
            const int t = c * ct + cid + j * n_comm;
            const int job = k + lane;
            const int slot = job % n_slots;
            JobDesc d;
            uint32_t bytes = 0;
            int pos[8];
            for (int s2 = 0; s2 < K; ++s2) {
              pos[s2] = p.tok_pos[t * K + s2];
              d.w[s2] = pos[s2] < 0 ? 0.f : (p.combine_w ? p.combine_w[t * K + s2] : 1.f);
              bytes += pos[s2] >= 0 ? seg : 0u;
              if (pos[s2] >= 0)  // the row's layer1 tile of this n-block is in memory
                for (int h = 0; h <= h_hi; ++h) {
                  const uint32_t* fl = p.tile_done + (static_cast<long long>(pos[s2] >> 7) * NB + nb) * 2 + h;
                  { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_gpu(fl), p.epoch)) sp.pause(128, 12); }
                }
            }
            ptx::fence_async_global();  // generic-proxy rows -> bulk (async proxy) loads
            d.dst = p.y_local + static_cast<long long>(t) * N + nb * kBlockN;
            ptx::mbar_wait(cs->empty + slot, ((job / n_slots) & 1) ^ 1);
            cs->desc[slot] = d;
            ptx::mbar_arrive_expect_tx(cs->full + slot, bytes);
            for (int s2 = 0; s2 < K; ++s2)
              if (pos[s2] >= 0)
                ptx::bulk_load(smem + slot * slot_bytes + s2 * kSeg,
                               p.yrows + static_cast<long long>(pos[s2]) * N + nb * kBlockN, seg, cs->full + slot);
          }
          k += min(kBatch, jobs - j0);
          __syncwarp();
        }
      }
    }
    return;
  }
  if (warp > kReducers) return;  // the layer kernel has more warps than reducers
  const int me = warp - 1;
  int k = 0;
  for (int c = 0; c < n_ch; ++c) {
    const int jobs = jobs_of(c);
    for (int nb = 0; nb < NB; ++nb) {
      for (int j = 0; j < jobs; ++j, ++k) {
        if (k % kReducers != me) continue;
        const int slot = k % n_slots;
        ptx::mbar_wait(cs->full + slot, (k / n_slots) & 1);
        const JobDesc& d = cs->desc[slot];
        __nv_bfloat16* dst = d.dst;
        float w[8];
        for (int s2 = 0; s2 < K; ++s2) w[s2] = d.w[s2];
        uint4 o[kBlockN / 256];
#pragma unroll
        for (int h = 0; h < static_cast<int>(kBlockN / 256); ++h) {
          float acc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = 0.f;
          for (int s2 = 0; s2 < K; ++s2) {  // ascending slot = ascending expert (executor.py:102-120)
            if (w[s2] == 0.f) continue;
            const uint4 v = *reinterpret_cast<const uint4*>(smem + slot * slot_bytes + s2 * kSeg + h * 512 + lane * 16);
            const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __bfloat1622float2(hv[q]);
              acc[2 * q] += f.x * w[s2];
              acc[2 * q + 1] += f.y * w[s2];
            }
          }
          o[h].x = pack2(acc[0], acc[1]); o[h].y = pack2(acc[2], acc[3]);
          o[h].z = pack2(acc[4], acc[5]); o[h].w = pack2(acc[6], acc[7]);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(cs->empty + slot);
#pragma unroll
        for (int h = 0; h < static_cast<int>(kBlockN / 256); ++h)
          if (nb * kBlockN + h * 256 + lane * 8 < N) ptx::st_v4(dst + h * 256 + lane * 8, o[h]);
      }
      // this CTA's tokens of chunk c are final for nb -> count them (copy engine reads y)
      ptx::named_bar_sync(2, kReducers * 32);
      if (threadIdx.x == 32 && jobs) {
        __threadfence_system();
        const int cols = N - nb * static_cast<int>(kBlockN);
        atomicAdd(p.out_cnt + c, static_cast<uint32_t>(jobs) * (cols > static_cast<int>(kBlockN / 2) ? 2u : 1u));
      }
    }
  }
}

}  // namespace comm
}  // namespace comet
