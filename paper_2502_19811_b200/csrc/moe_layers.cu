// COMET fused MoE layer kernels for sm_100a.
//
// moe_layer_kernel: ONE persistent launch runs both expert GEMMs of a rank
// (KernelArgs.mode 2; modes 0/1 run one layer), thread-block specialised
// (section 3.2.1).  CTAs [0, n_compute) form 2-CTA clusters: a
// scheduler warp claims 256x512 work units just in time (sched.cuh: the claim
// sequence), a TMA producer and a single-thread tcgen05.mma issuer
// (cta_group::2, 2 x 256-column fp32 accumulators in TMEM) run the mainloop,
// four epilogue warps drain TMEM.  CTAs [n_compute, grid) first pull this
// rank's rows of the expert-sorted token tensor (comm.cuh dispatch_rows:
// TMA bulk copies from the NVLink-mapped source ranks, in the compute claim
// order, publishing ready epochs per 128-row tile) and then join the GEMMs.
//
//   layer0 (resolve_layer0 + _hidden_row, resolver.py:206-252,
//   executor.py:86-90): units wait for their tiles' ready epochs; the
//   epilogue applies the activation and counts finished halves per H tile.
//
//   layer1 (resolve_layer1 + _output_columns + _combine, resolver.py:255-309,
//   executor.py:93-120): a unit starts when its H tiles are complete; the
//   epilogue of each token's last hosted row folds the earlier rows (ascending
//   slot, weighted) and writes the result (world 1) or pushes it into the
//   source rank's combine buffer over NVLink (combine_finish_kernel sums the
//   ranks' partials there).  Split-K and 256-column halves balance tails.

#include <cuda.h>
#include <cuda_bf16.h>

#include "comm.cuh"
#include "layers.cuh"
#include "ptx.cuh"
#include "sched.cuh"

namespace comet {

namespace {

// Work unit = 256 rows (a 2-CTA pair, 128 rows per CTA) x 512 output columns.
// Each k-step issues two UMMA 256x256x16 (cta_group::2) that share the A tile
// and use the two 256-column halves of the B block; both accumulators live in
// TMEM (2 x 256 fp32 columns = all 512).  Per SM and k-element this moves
// 128 A + 256 B rows for 128x512 MACs: 48 B/cycle at full rate instead of 64
// for a 256x256 pair tile (the L2->SM traffic and the power that costs set the
// sustained clock under the 1 kW cap).
// 12 warps: warp 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 unit
// scheduler (warpgroup 0, shrunk to kRegsCtl registers), warps 4-11 the
// epilogue (warpgroups 1-2, grown to kRegsEpi): two warps per TMEM lane
// quadrant (warp w reads lanes 32 (w % 4)..), one taking the even and one
// the odd 64-column chunks, so an accumulator drains twice as fast as with
// one warp per quadrant (the drain paces the next unit's first MMAs and the
// end of the launch).
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 128 + kEpiThreads;
// setmaxnreg moves registers inside the CTA's pool, i.e. what the launch
// allocated: 384 threads x 168 (the __launch_bounds__(384, 1) cap) = 64512
constexpr int kRegsCtl = 56;
constexpr int kRegsEpi = 224;
static_assert(128 * kRegsCtl + kEpiThreads * kRegsEpi <= kThreads * (65536 / kThreads / 8 * 8),
              "the register budgets exceed the CTA's launch allocation (setmaxnreg.inc would never succeed)");
constexpr int kStages = kLayerStages;
constexpr int kBlockK = 64;                              // bf16 elements = 128 B swizzle atom
constexpr uint32_t kSmemA = kTileRows * kBlockK * 2;     // 16 KB: this CTA's 128 A rows
constexpr uint32_t kSmemBh = 128 * kBlockK * 2;          // 16 KB: this CTA's 128 rows of one B half
constexpr uint32_t kSmemStage = kSmemA + 2 * kSmemBh;    // 48 KB
constexpr uint32_t kTmemCols = kBlockN;                  // 512 = both accumulators
constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(2 * kTileRows, kHalfN);
constexpr int kEpiThread0 = 128;                         // first epilogue thread
constexpr uint32_t kSmemEpiWarp = 32 * 128;              // one warp's 32 rows x 64 columns (bf16)
constexpr uint32_t kSmemEpi = kEpiWarps * kSmemEpiWarp;  // one staging buffer per epilogue warp
// a dispatch CTA's ring + bookkeeping live in the same dynamic smem
static_assert(comm::kRingBytes + sizeof(comm::CommSmem) <= kStages * kSmemStage + kSmemEpi,
              "dispatch ring and its bookkeeping exceed the layer kernel's shared memory");


// Timeline record: interval [t0, t1] of `role` for unit `task` on this CTA
// (globaltimer ns).  Exported as the reference simulator's timeline CSV
// (block_id, block_kind, task_id, start_ns, end_ns; simulator.py:235-245).
__device__ __forceinline__ void tl_record(const LayerArgs& p, int role, int idx, int task, uint64_t t0, uint64_t t1) {
  if (p.timeline == nullptr || idx >= p.timeline_cap) return;
  unsigned long long* r = p.timeline + ((static_cast<long long>(blockIdx.x) * kRoles + role) * p.timeline_cap + idx) * 2;
  r[0] = t0;
  r[1] = (t1 - t0) | (static_cast<unsigned long long>(task + 1) << 40);
}


template <int ACT>
__device__ __forceinline__ float activate(float x) {
  if constexpr (ACT == kActRelu) return fmaxf(x, 0.f);
  else if constexpr (ACT == kActSilu) return x / (1.f + __expf(-x));
  else if constexpr (ACT == kActGeluTanh) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.f + tanhf(u));
  } else if constexpr (ACT == kActTanh) return tanhf(x);
  else return x;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 64 fp32 accumulator columns -> activation -> 32 packed bf16 pairs.  The
// activation is resolved once per chunk (a runtime switch per element costs a
// jump-table branch per value).
template <int ACT>
__device__ __forceinline__ void pack_chunk(const uint32_t (&v0)[32], const uint32_t (&v1)[32], uint32_t (&pk)[32]) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    pk[i] = pack_bf16(activate<ACT>(__uint_as_float(v0[2 * i])), activate<ACT>(__uint_as_float(v0[2 * i + 1])));
#pragma unroll
  for (int i = 0; i < 16; ++i)
    pk[16 + i] = pack_bf16(activate<ACT>(__uint_as_float(v1[2 * i])), activate<ACT>(__uint_as_float(v1[2 * i + 1])));
}

// acc[0..32) += w * 32 bf16 already in registers (r[0..4) = 4 x uint4)
__device__ __forceinline__ void fold_regs(uint32_t (&acc)[32], const uint4* r, float w) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r[q]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(h[j]);
      acc[q * 8 + 2 * j] = __float_as_uint(fmaf(w, f.x, __uint_as_float(acc[q * 8 + 2 * j])));
      acc[q * 8 + 2 * j + 1] = __float_as_uint(fmaf(w, f.y, __uint_as_float(acc[q * 8 + 2 * j + 1])));
    }
  }
}
constexpr int kMaxFold = 7;  // earlier hosted rows of a token (top-k <= 8)
#ifndef COMET_HELP_POLL_NS
#define COMET_HELP_POLL_NS 8000
#endif
constexpr uint64_t kHelpPollNs = COMET_HELP_POLL_NS;  // split-K: how long an earlier slice polls for the last one

constexpr int kSchedSlots = 2;
constexpr int kLifeTask = (1 << 20) - 2;  // timeline task id of a CTA's lifetime record
// Readers of each claimed unit id: leader CTA producer + MMA + 8 epilogue
// warps, peer CTA producer + 8 epilogue warps (all arrive on the leader's
// slot-empty barrier).
constexpr uint32_t kSchedReaders = 2 * (1 + kEpiWarps) + 1;
// The producer asks for its next unit this many k-blocks before the end of
// the current unit's loads (~4 us of MMA: covers the claim's atomic and
// broadcast, keeps the claim-ahead short).
constexpr int kClaimLead = 8;


// Zero-copy forward, output side: a downloader CTA walks the layer1 units in
// sequence order (every n_dl-th), waits for each (128-row tile, 256-column
// half) to be final (tile_done epoch, published after the fused combine's
// folder rows were written to the device copy y_local) and copies the folder
// rows' 512-byte segments to pinned host memory.  Host writes leave the GEMM
// epilogues (a sysmem store backlog in an SM stalls its epilogue and, through
// TMEM, its MMAs) and run on these CTAs at PCIe rate.
__device__ void download_rows(const KernelArgs& f, int did) {
  const LayerArgs& p = f.l[1];
  const int NB = p.n_blocks, N = p.n_embed;
  const int P = p.meta[kMetaPairs];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_warps = blockDim.x >> 5;
  constexpr int kB = 4;  // row segments in flight per warp
  for (int u = did; u < P * NB; u += f.n_dl) {
    const Unit w = decode_unit(u, 1, p.raster, P, NB, p.order_group, p.order_group2);
    const int4 pr = reinterpret_cast<const int4*>(p.pairs)[w.pair];
    for (int cta = 0; cta < 2; ++cta) {
      const int rows = min(kTileRows, pr.z - kTileRows * cta);
      if (rows <= 0) continue;
      const int tile = (pr.y >> 7) + cta;
      for (int h = 0; h < 2; ++h) {
        if (lane == 0) {
          const uint32_t* fl = p.tile_done + (static_cast<long long>(tile) * NB + w.nb) * 2 + h;
          { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_gpu(fl), p.epoch)) sp.pause(128, 1); }
        }
        __syncwarp();
        const long long col = static_cast<long long>(w.nb) * kBlockN + h * kHalfN + lane * 8;
        for (int r0 = warp * kB; r0 < rows; r0 += n_warps * kB) {
          uint4 v[kB];
          int t[kB];
#pragma unroll
          for (int i = 0; i < kB; ++i) {
            const int rd = r0 + i < rows ? p.row_dst[tile * kTileRows + r0 + i] : -1;
            t[i] = rd >= 0 ? (rd & 0xFFFFFF) : -1;
            if (t[i] >= 0) v[i] = __ldcg(reinterpret_cast<const uint4*>(p.y_local + t[i] * static_cast<long long>(N) + col));
          }
#pragma unroll
          for (int i = 0; i < kB; ++i)
            if (t[i] >= 0) *reinterpret_cast<uint4*>(f.y_host + t[i] * static_cast<long long>(N) + col) = v[i];
        }
      }
    }
  }
}

// Compute role of a 2-CTA pair: scheduler (leader warp 3) claims units and
// broadcasts their ids to both CTAs; warp 0 TMA producer, warp 1 MMA issuer
// (leader), warps 4-7 epilogue.
__device__ __forceinline__ void compute_role(const KernelArgs& f, uint8_t* smem, const CUtensorMap* tm_a0,
                                             const CUtensorMap* tm_b0, const CUtensorMap* tm_a1,
                                             const CUtensorMap* tm_b1, const CUtensorMap* tm_s0,
                                             const CUtensorMap* tm_s1) {
  uint8_t* epi_smem = smem + kStages * kSmemStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_smem + kSmemEpi);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;       // accumulators ready (one per unit)
  uint64_t* tempty = bars + 2 * kStages + 1;  // [2]: accumulator half drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 3);
  uint64_t* sfull = bars + 2 * kStages + 4;                   // [kSchedSlots] unit id written
  uint64_t* sempty = sfull + kSchedSlots;                     // [kSchedSlots] unit id read by all
  uint64_t* sreq = sempty + kSchedSlots;                      // producer asks for the next unit
  int* sunit = reinterpret_cast<int*>(sreq + 1);              // [kSchedSlots]
  int* sflag = sunit + kSchedSlots;                           // epilogue: split-K finisher flag
  int* srow_chunk = sflag + 1;                                // epilogue: [128] output-row token chunk

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = blockIdx.x & 1;  // rank in the 2-CTA cluster
  const bool leader = cta == 0;
  const bool spin = COMET_DBG(f.l[f.mode == 1 ? 1 : 0].debug, 4);
  auto wait = [spin](uint64_t* bar, uint32_t parity) {
    if (spin) ptx::mbar_wait_spin(bar, parity);
    else ptx::mbar_wait(bar, parity);
  };

  if (warp == 0 && lane == 0) {
    if (f.mode != 1) {
      ptx::prefetch_tmap(tm_a0);
      ptx::prefetch_tmap(tm_b0);
    }
    if (f.mode != 0) {
      ptx::prefetch_tmap(tm_a1);
      ptx::prefetch_tmap(tm_b1);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(full + s, 2);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty + 0, 2 * kEpiThreads);
    ptx::mbar_init(tempty + 1, 2 * kEpiThreads);
    for (int s = 0; s < kSchedSlots; ++s) {
      ptx::mbar_init(sfull + s, 1);
      ptx::mbar_init(sempty + s, kSchedReaders);
    }
    ptx::mbar_init(sreq, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  ptx::pdl_wait();  // the prologue above overlapped the previous kernel's tail

  const int P = f.l[f.mode == 1 ? 1 : 0].meta[kMetaPairs];
  // pairs that compute: everything but layer1 combine CTAs (dispatch CTAs join)
  const int n_pairs =
      (f.mode == 1 ? f.l[1].n_compute : (f.l[0].stream_combine ? f.l[0].n_compute : static_cast<int>(gridDim.x))) >> 1;
  Sched s0, s1;
  const int total = seq_total(f, P, n_pairs, s0, s1);
  if (f.mode != 0) {
    const LayerArgs& p1 = f.l[1];
    if (p1.world > 1 && P == 0 && p1.n_compute == static_cast<int>(gridDim.x) && blockIdx.x == 0 &&
        threadIdx.x == 0)  // nothing hosted, no combine CTAs: publish empty blocks
      for (int nb = 0; nb < p1.n_blocks; ++nb)
        for (int d = 0; d < p1.world; ++d) ptx::st_release_sys(p1.cb_flag_peer[d] + p1.rank * p1.n_blocks + nb, p1.epoch);
  }
  // Reader side of the unit ring: lane 0 takes claim i, the warp gets it.
  auto next_unit = [&](int i) -> int {
    int g = 0;
    if (lane == 0) {
      const int slot = i % kSchedSlots;
      ptx::mbar_wait_cluster(sfull + slot, (i / kSchedSlots) & 1);
      g = reinterpret_cast<volatile int*>(sunit)[slot];
      if (leader) ptx::mbar_arrive(sempty + slot);
      else ptx::mbar_arrive_cluster(sempty + slot, 0);
    }
    return __shfl_sync(0xffffffffu, g, 0);
  };

  // Registers move from the single-lane control warps (warpgroup 0) to the
  // epilogue (warpgroups 1-2): each side changes its budget at the top of its
  // branch (ptxas allocates every region under the budget that dominates it).
  if (warp < 4) {
  ptx::setmaxnreg_dec<kRegsCtl>();
  if (warp == 3) {
    // ---------------- scheduler (leader CTA, one thread) ----------------
    // Claims just in time: unit i+1 is claimed when the producer asks for it,
    // a few k-blocks before the end of unit i's loads -- a pair never holds a
    // queued unit that an idle pair could have run (the tail is units of up
    // to ~150 us).
    if (leader && lane == 0) {
      for (int i = 0;; ++i) {
        const int slot = i % kSchedSlots;
        if (i > 0) ptx::mbar_wait(sreq, (i - 1) & 1);
        ptx::mbar_wait(sempty + slot, ((i / kSchedSlots) & 1) ^ 1);
        int g = static_cast<int>(atomicAdd(f.sched, 1u));
        if (g >= total) g = -1;
        sunit[slot] = g;
        ptx::st_shared_cluster(sunit + slot, 1, static_cast<uint32_t>(g));
        ptx::mbar_arrive(sfull + slot);
        ptx::mbar_arrive_release_cluster(sfull + slot, 1);
        if (g < 0) break;
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    bool seq_done = false;
    for (int it = 0;; ++it) {
      const int g = next_unit(it);
      if (g < 0) break;
      const Unit w = unit_at(f, g, P, s0, s1);
      const LayerArgs& p = f.l[w.layer];
      const CUtensorMap* ta = w.layer ? tm_a1 : tm_a0;
      const CUtensorMap* tb = w.layer ? tm_b1 : tm_b0;
      const int4 pr = reinterpret_cast<const int4*>(p.pairs)[w.pair];
      const int row0 = pr.y + kTileRows * static_cast<int>(cta);
      const int brow = pr.x * p.b_rows + w.nb * kBlockN + 128 * static_cast<int>(cta) + (w.half > 0 ? kHalfN : 0);
      if (lane == 0 && w.layer == 0 && p.sequential && !seq_done) {
        // "sequential" mode (no overlap, the cli's baseline): the first GEMM
        // waits for the WHOLE dispatch, like an all-to-all before GroupGEMM
        for (int q = 0; q < 2 * P; ++q)
          if (p.pull_local ? reinterpret_cast<const int4*>(p.pairs)[q >> 1].z > kTileRows * (q & 1)
                           : (reinterpret_cast<const int4*>(p.pairs)[q >> 1].w >> (q & 1)) & 1)
            { ptx::SpinCtl sp; while (!ptx::epoch_reached(ptx::ld_acquire_gpu(p.xg_ready + q), p.epoch)) sp.pause(64, 2); }
        seq_done = true;
      }
      if (lane == 0) {
        const bool pulled = p.pull_local ? pr.z > kTileRows * static_cast<int>(cta) : ((pr.w >> cta) & 1);
        if (w.layer == 0 && pulled && !COMET_DBG(p.debug, 1)) {
          // this CTA's 128 A rows include rows pulled over NVLink by a dispatch CTA
          const uint32_t* flag = p.xg_ready + (w.pair * 2 + static_cast<int>(cta));
          { ptx::SpinCtl sp; while (!ptx::epoch_reached(ptx::ld_acquire_gpu(flag), p.epoch)) sp.pause(32, 3); }
          ptx::fence_async_global();
        }
      }
      __syncwarp();
      // layer1 A = H rows written by the layer0 epilogues of this launch:
      // each 64-wide k-block is gated on the layer0 unit of its columns
      // (per (128-row tile, layer0 n-block) half counts), so a layer1 unit
      // starts as soon as its first H columns exist and reaches the columns
      // of layer0's last units (the leftover round) ~a unit time later
      const bool gate_h = w.layer == 1 && f.mode == 2;
      const uint32_t* hc = f.h_cnt + static_cast<long long>(row0 >> 7) * f.l[0].n_blocks;
      const uint64_t t_start = ptx::globaltimer();  // load interval starts once its A rows are ready
      const int kb0 = w.kb0, kb1 = w.kb1;
      const int kb_req = max(kb0, kb1 - kClaimLead);
      for (int kb = kb0; kb < kb1; ++kb) {
        wait(empty + stage, phase ^ 1);
        if (kb == kb_req && leader && lane == 0) ptx::mbar_arrive(sreq);  // claim the next unit now
        if (gate_h && lane == 0 && (kb == kb0 || (kb & (kBlockN / kBlockK - 1)) == 0)) {
          const int nb0 = kb / static_cast<int>(kBlockN / kBlockK);
          const uint32_t target = narrow_block(f.l[0], nb0) ? 1u : 2u;
          { ptx::SpinCtl sp; while (ptx::ld_acquire_gpu(hc + nb0) < target) sp.pause(32, 4); }
          ptx::fence_async_global();
        }
        if (lane == 0 && COMET_DBG(p.debug, 16)) {
          // debug: no data movement, complete the stage by arrivals only
          if (leader) ptx::mbar_arrive(full + stage);
          else ptx::mbar_arrive_cluster(full + stage, 0);
        } else if (lane == 0) {
          uint8_t* sa = smem + stage * kSmemStage;
          ptx::tma_load_2d_2sm(sa, ta, full + stage, kb * kBlockK, row0, ptx::kEvictNormal);
          ptx::tma_load_2d_2sm(sa + kSmemA, tb, full + stage, kb * kBlockK, brow, ptx::kEvictNormal);
          if (w.half < 0)
            ptx::tma_load_2d_2sm(sa + kSmemA + kSmemBh, tb, full + stage, kb * kBlockK, brow + kHalfN,
                                 ptx::kEvictNormal);
          if (leader) ptx::mbar_arrive_expect_tx(full + stage, w.half < 0 ? 2 * kSmemStage : 2 * (kSmemA + kSmemBh));
          else ptx::mbar_arrive_cluster(full + stage, 0);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) tl_record(p, kRoleLoad, it, g, t_start, ptx::globaltimer());
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA, one thread) ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      const int g = next_unit(it);
      if (g < 0) break;
      const Unit w = unit_at(f, g, P, s0, s1);
      const LayerArgs& p = f.l[w.layer];
      const bool two = w.half < 0;  // both accumulator halves (else only half 0)
      const uint32_t ephase = (it & 1) ^ 1;  // previous unit's drain of each half
      const int kb0 = w.kb0, kb1 = w.kb1;
      const uint64_t t_w = ptx::globaltimer();
      wait(tempty + 0, ephase);
      ptx::tc_fence_after();
      const uint64_t t_m = ptx::globaltimer();
      for (int kb = kb0; kb < kb1; ++kb) {
        wait(full + stage, phase);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + stage * kSmemStage);
        const uint64_t da = ptx::sdesc_kmajor_sw128(sa);
        const uint64_t db0 = ptx::sdesc_kmajor_sw128(sa + kSmemA);
        const uint64_t db1 = ptx::sdesc_kmajor_sw128(sa + kSmemA + kSmemBh);
        // one fixed issuing lane: tcgen05.commit tracks the MMAs of its own thread
        if (lane == 0 && !COMET_DBG(p.debug, 8)) {
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k)
            ptx::mma_bf16_2sm(tmem_base, da + 2 * k, db0 + 2 * k, kIdesc, (kb != kb0) || (k != 0));
        }
        __syncwarp();
        if (kb == kb0) {  // half 1 of the accumulator drains after half 0
          wait(tempty + 1, ephase);
          ptx::tc_fence_after();
        }
        if (lane == 0) {
          if (!COMET_DBG(p.debug, 8) && two) {
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k)
              ptx::mma_bf16_2sm(tmem_base + kHalfN, da + 2 * k, db1 + 2 * k, kIdesc, (kb != kb0) || (k != 0));
          }
          ptx::mma_commit_2sm(empty + stage, 0x3);
          if (kb == kb1 - 1) ptx::mma_commit_2sm(tfull, 0x3);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) {
        tl_record(p, kRoleTmemWait, it, g, t_w, t_m);
        tl_record(p, kRoleMma, it, g, t_m, ptx::globaltimer());
      }
    }
  }
  } else {
    // ---------------- epilogue: TMEM -> registers -> global ----------------
    ptx::setmaxnreg_inc<kRegsEpi>();
    const int ew = warp - 4;       // 0..7
    const int quad = ew & 3;       // TMEM lane quadrant = output rows 32 quad.. of the CTA's 128
    const int sub = ew >> 2;       // 0: even 64-column chunks, 1: odd
    for (int it = 0;; ++it) {
      const int g = next_unit(it);
      if (g < 0) break;
      const Unit w = unit_at(f, g, P, s0, s1);
      const LayerArgs& p = f.l[w.layer];
      const int NB = p.n_blocks;
      const int4 pr = reinterpret_cast<const int4*>(p.pairs)[w.pair];
      const int row0 = pr.y + kTileRows * static_cast<int>(cta);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
      const int col0 = w.half > 0 ? static_cast<int>(kHalfN) : 0;  // half unit: its columns
      const int cols_left = p.out_ld - w.nb * kBlockN - col0;      // ragged last n-block (e.g. K/tp = 3200)
      const int n_chunks = w.half < 0 ? static_cast<int>(kBlockN / 64) : static_cast<int>(kHalfN / 64);
      const int h_lo = w.half < 0 ? 0 : w.half, h_hi = w.half < 0 ? 1 : w.half;  // 256-col halves covered
      // Destination of this lane's row: the layer output, or -- fused combine,
      // the row of its token's last hosted expert -- the token's weighted sum
      // over its hosted experts (executor.py:102-120), written to y (world 1)
      // or pushed straight into the source rank's combine slot over NVLink.
      const int my_row = row0 + quad * 32 + lane;
      __nv_bfloat16* my_dst = p.out + static_cast<long long>(my_row) * p.out_ld + w.nb * kBlockN + col0;
      float scale = 1.f;
      int fold_t = -1;              // token of a folding row
      bool out_row = false;         // this row writes / pushes its token's final sum
      int nf = 0;                   // rows to fold in, their rows and weights (ascending slot)
      int fpos[kMaxFold];
      float fw[kMaxFold];
      if (w.layer == 1 && p.fuse_combine) {
        const int rd = p.row_dst[my_row];
        const bool real_row = kTileRows * static_cast<int>(cta) + quad * 32 + lane < pr.z;
        if (rd >= 0 || (p.fold_stride >= 2 && real_row)) {
          const int widx = p.row_widx[my_row];
          const int t = widx / p.topk, me = widx - t * p.topk;
          // chained folds (fold_stride k): hosted rows in ascending slot order
          // form a chain; rows whose chain index c has c % k == k-1, and the
          // last one, fold the rows since the previous folder (weighted) plus
          // that folder's row (already a weighted partial, weight 1); the
          // intermediate folders write their partial to their own yrows row.
          // k = 0: the last hosted row folds every other hosted row.
          const int k = p.fold_stride;
          int c = 0;
          if (k >= 2)
            for (int s2 = 0; s2 < me; ++s2) c += p.tok_pos[t * p.topk + s2] >= 0;
          if (rd >= 0 || c % k == k - 1) {
            out_row = rd >= 0;
            if (out_row) {
              __nv_bfloat16* base = p.world > 1 ? p.cb_peer[rd >> 24] : p.y_local;
              my_dst = base + static_cast<long long>(rd & 0xFFFFFF) * p.n_embed + w.nb * kBlockN + col0;
            }
            fold_t = t;
            if (p.combine_w) scale = p.combine_w[widx];
            const int g0 = k >= 2 ? c - c % k : 0;  // chain index of this folder's first own-group row
            // the rows to fold, ascending slot (k = 0: every other hosted row
            // -- only earlier slots unless the streamed forward picked a
            // non-last folder)
            int ci = 0;  // chain index of slot s2
#pragma unroll
            for (int s2 = 0; s2 < kMaxFold + 1; ++s2) {
              if (s2 >= p.topk) break;
              const int pos = p.tok_pos[t * p.topk + s2];
              if (pos < 0) continue;
              const int cs = ci++;
              if (s2 == me) continue;
              const bool prev_folder = k >= 2 && cs == g0 - 1;
              if (k >= 2 && (s2 > me || (cs < g0 && !prev_folder))) continue;
#pragma unroll
              for (int j = 0; j < kMaxFold; ++j)  // static register indexing
                if (j == nf) {
                  fpos[j] = pos;
                  fw[j] = prev_folder ? 1.f : (p.combine_w ? p.combine_w[t * p.topk + s2] : 1.f);
                }
              ++nf;
            }
          }
        }
      }
#ifndef COMET_NO_FOLD_PREFETCH
      // Fold rows were written by earlier units, up to a whole layer ago, and
      // the weight stream has since evicted most of them from L2: the
      // epilogue's register-limited loads (two rows in flight) then pay HBM
      // round trips (QW top-8 folders: ~35 us epilogues at the launch tail).
      // Pull this unit's column range of every fold row into L2 now, while
      // the MMAs still run: one bulk prefetch per (lane, fold row), the
      // quadrant's two warps taking alternate rows.  L2 is the coherence
      // point, so a prefetch that lands before a predecessor's stores is
      // harmless (the stores update the line; fold_wait orders the loads).
      if (fold_t >= 0 && cols_left > 0) {
        const int pcols = min(cols_left, n_chunks * 64);
#pragma unroll
        for (int j = 0; j < kMaxFold; ++j) {
          if (j >= nf) break;
          if ((j & 1) == sub)
            ptx::bulk_prefetch_l2(p.yrows + static_cast<long long>(fpos[j]) * p.n_embed + w.nb * kBlockN + col0,
                                  static_cast<uint32_t>(pcols) * 2u);
        }
      }
#endif
      wait(tfull, it & 1);
      ptx::tc_fence_after();
      const uint64_t t_e = ptx::globaltimer();
      // the rows this one folds live in units claimed before this one (same
      // n-block columns, lower sequence index): wait for their tiles
      auto fold_wait = [&]() {
        // (a split-tail half 1 of a narrow last n-block has no real columns:
        // nothing to fold, and its predecessors never publish that half)
        if (fold_t < 0 || cols_left <= 0) return;
#pragma unroll
        for (int j = 0; j < kMaxFold; ++j) {
          if (j >= nf) break;
          for (int h = h_lo; h <= h_hi; ++h) {
            const uint32_t* fl = p.tile_done + (static_cast<long long>(fpos[j] >> 7) * NB + w.nb) * 2 + h;
            { ptx::SpinEpi sp; while (!ptx::epoch_reached(ptx::ld_acquire_gpu(fl), p.epoch)) sp.pause(64, 5); }
          }
        }
      };
      const unsigned long long my_addr = reinterpret_cast<unsigned long long>(my_dst);
      // 64 fp32 columns of this lane's row -> (fold) -> activation -> bf16 ->
      // coalesced stores
      // contiguous destination rows (H, or yrows without the fused combine):
      // TMA tensor stores; fused-combine units write scattered token rows
      // (fused combine: a warp none of whose 32 rows writes a token's final
      // sum keeps its rows in yrows -- contiguous, so TMA stores too)
      const bool tma_out = (w.layer == 0 || !p.fuse_combine || !__any_sync(0xffffffffu, out_row))
                           && !COMET_DBG(p.debug, 16384);
      auto process = [&](int s, int seq, uint32_t (&v0)[32], uint32_t (&v1)[32]) {
        if (w.layer == 1) {  // no activation on FC2; fused combine: weight + earlier rows
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v0[i] = __float_as_uint(__uint_as_float(v0[i]) * scale);
            v1[i] = __float_as_uint(__uint_as_float(v1[i]) * scale);
          }
          // earlier hosted rows, ascending slot: two rows' loads in flight per
          // round trip (a serial load->fma chain made top-8 epilogues ~100 us)
#pragma unroll
          for (int j = 0; j < kMaxFold; j += 2) {
            if (j >= nf) break;
            uint4 ra[8], rb[8];
            const __nv_bfloat16* a = p.yrows + static_cast<long long>(fpos[j]) * p.n_embed + w.nb * kBlockN + col0 + s * 64;
#pragma unroll
            for (int q = 0; q < 8; ++q) ra[q] = *reinterpret_cast<const uint4*>(a + q * 8);
            const bool two = j + 1 < nf && j + 1 < kMaxFold;
            if (two) {
              const __nv_bfloat16* b =
                  p.yrows + static_cast<long long>(fpos[j + 1 < kMaxFold ? j + 1 : j]) * p.n_embed + w.nb * kBlockN + col0 + s * 64;
#pragma unroll
              for (int q = 0; q < 8; ++q) rb[q] = *reinterpret_cast<const uint4*>(b + q * 8);
            }
            fold_regs(v0, ra, fw[j]);
            fold_regs(v1, ra + 4, fw[j]);
            if (two) {
              fold_regs(v0, rb, fw[j + 1 < kMaxFold ? j + 1 : j]);
              fold_regs(v1, rb + 4, fw[j + 1 < kMaxFold ? j + 1 : j]);
            }
          }
        }
        uint32_t pk[32];
        switch (w.layer == 1 ? static_cast<int>(kActIdentity) : p.activation) {
          case kActRelu: pack_chunk<kActRelu>(v0, v1, pk); break;
          case kActSilu: pack_chunk<kActSilu>(v0, v1, pk); break;
          case kActGeluTanh: pack_chunk<kActGeluTanh>(v0, v1, pk); break;
          case kActTanh: pack_chunk<kActTanh>(v0, v1, pk); break;
          default: pack_chunk<kActIdentity>(v0, v1, pk); break;
        }
        // Coalesce through a per-warp smem transpose: each lane parks its
        // row's 128 B (XOR-swizzled 16 B granules, conflict-free), then each
        // store instruction writes 4 whole 128 B lines (8 lanes per row).
        // Only this warp touches its staging rows: __syncwarp suffices.
        // (seq: this warp's count of processed chunks; one staging buffer
        // per warp -- the quadrant's other warp stores the chunks between)
        uint8_t* stg = epi_smem + ew * kSmemEpiWarp;
        // TMA store: the staging rows (SW128 layout) of this warp's previous
        // chunk must be read out before they are overwritten
        if (tma_out && seq >= 1) {
          if (lane == 0) ptx::bulk_wait_read<0>();
          __syncwarp();
        }
        if (COMET_DBG(p.debug, 512)) {  // debug: pack only (no staging, no stores)
          if (pk[0] == 0x7fc07fc1u) p.split_cnt[0] = pk[1];  // keep the pack live
          return;
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) * 16)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        if (COMET_DBG(p.debug, 256)) return;  // debug: staged, not stored
        if (tma_out) {
          // rows row0+32*quad.. are contiguous in H / yrows: one async 2D tensor
          // store of the warp's 32 x 64 block (the swizzled staging layout is
          // the map's SWIZZLE_128B box) instead of 8 transposed st.global
          ptx::fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(w.layer ? tm_s1 : tm_s0, stg, w.nb * static_cast<int>(kBlockN) + col0 + s * 64,
                              row0 + quad * 32);
            ptx::bulk_commit();
          }
          return;
        }
        __syncwarp();
        const int gsub = lane & 7, rsub = lane >> 3;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + rsub;
          const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 128 + ((gsub ^ (r & 7)) * 16));
          __nv_bfloat16* rp = reinterpret_cast<__nv_bfloat16*>(__shfl_sync(0xffffffffu, my_addr, r));
          if (w.layer == 1 || f.mode == 2) ptx::st_v4(rp + s * 64 + gsub * 8, v);  // re-read in this launch
          else ptx::st_v4_cs(rp + s * 64 + gsub * 8, v);
        }
        __syncwarp();
      };
      // split-K: this slice's fp32 partial of the CTA's 128 x 512 tile, stored
      // column-quad major ([c/4][row][4]) so a warp's 32 rows of one quad are
      // 512 contiguous bytes (coalesced stores and reloads)
      const int S = w.np;
      const long long split_tile = static_cast<long long>(row0 >> 7) * NB + w.nb;
      float4* part_row = S > 1 ? reinterpret_cast<float4*>(p.part + (split_tile * S + w.ks) * kTileRows * kBlockN) +
                                     quad * 32 + lane
                               : nullptr;
      // Split-K finisher.  Two slices (the uneven layer1 tail split, or S = 2
      // split-K): roles are decided when the accumulator is ready -- the
      // slice that starts its epilogue last finishes the tile; the other
      // stores its fp32 partial and counts it as landed; the finisher waits
      // for it and drains its own accumulator adding the partial (0 + slice 0
      // + slice 1: IEEE addition commutes, so the value is the same whichever
      // slice finishes -- bitwise deterministic), so its own partial is never
      // written and re-read.  More slices (small-M split-K): every slice
      // stores its partial; the tile's 64-column chunks -- each the sum of
      // all S partials in slice order (deterministic) -- are finished by the
      // last slice to arrive and by earlier slices that see it arrive (see
      // below), so the reduction is spread over the slices (one CTA summing
      // all S x 8 chunks was ~40 us of dependent loads at the end of small-M
      // forwards); a half's completion is counted per chunk and published by
      // the CTA that completes it.
      const bool early = S == 2;
      bool finisher = S == 1;  // this CTA produces the tile's output (always, without split-K)
      uint32_t split_done = 0u;  // S > 2: the 256-column halves whose last chunk this slice finished
      uint32_t* landed = p.split_cnt + 256 + split_tile;
      const float4* rows0 =
          S > 1 ? reinterpret_cast<const float4*>(p.part + split_tile * S * kTileRows * kBlockN) + quad * 32 + lane : nullptr;
      if (early) {
        ptx::named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == kEpiThread0) *sflag = atomicAdd(p.split_cnt + split_tile, 1u) == 1u;
        ptx::named_bar_sync(1, kEpiThreads);
        finisher = *reinterpret_cast<volatile int*>(sflag) != 0;
        if (finisher) {
          if (threadIdx.x == kEpiThread0) {
            ptx::SpinEpi sp;
            while (ptx::ld_acquire_gpu(landed) < 1u) sp.pause(64, 6);
          }
          ptx::named_bar_sync(1, kEpiThreads);
          __threadfence();
        }
      }
      if (finisher) fold_wait();
      int seq = 0;
#pragma unroll 1
      for (int s = sub; s < n_chunks; s += 2) {
        // this warp's last chunk of its accumulator half: release the half
        const bool half_end = s + 2 >= n_chunks || ((s * 64) / static_cast<int>(kHalfN)) != (((s + 2) * 64) / static_cast<int>(kHalfN));
        if (COMET_DBG(p.debug, 128)) {  // debug: drain nothing
          if (half_end) {
            ptx::tc_fence_before();
            if (leader) ptx::mbar_arrive(tempty + (s * 64 >= static_cast<int>(kHalfN)));
            else ptx::mbar_arrive_cluster(tempty + (s * 64 >= static_cast<int>(kHalfN)), 0);
            if (w.half >= 0) {
              if (leader) ptx::mbar_arrive(tempty + 1);
              else ptx::mbar_arrive_cluster(tempty + 1, 0);
            }
          }
          continue;
        }
        uint32_t v0[32], v1[32];
        const bool red2 = early && finisher && s * 64 < cols_left;
        ptx::tmem_ld32(taddr + s * 64, v0);
        ptx::tmem_ld32(taddr + s * 64 + 32, v1);
        ptx::tmem_ld_wait();
        if (half_end) {
          // accumulator half drained: the next unit's MMAs may overwrite it
          // (a half unit used only half 0: release both)
          ptx::tc_fence_before();
          const int h = s * 64 >= static_cast<int>(kHalfN);
          if (leader) ptx::mbar_arrive(tempty + h);
          else ptx::mbar_arrive_cluster(tempty + h, 0);
          if (w.half >= 0) {
            if (leader) ptx::mbar_arrive(tempty + 1);
            else ptx::mbar_arrive_cluster(tempty + 1, 0);
          }
        }
        if (!finisher) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            part_row[(s * 16 + i) * kTileRows] = make_float4(__uint_as_float(v0[4 * i]), __uint_as_float(v0[4 * i + 1]),
                                                             __uint_as_float(v0[4 * i + 2]), __uint_as_float(v0[4 * i + 3]));
            part_row[(s * 16 + 8 + i) * kTileRows] =
                make_float4(__uint_as_float(v1[4 * i]), __uint_as_float(v1[4 * i + 1]), __uint_as_float(v1[4 * i + 2]),
                            __uint_as_float(v1[4 * i + 3]));
          }
          continue;
        }
        if (s * 64 >= cols_left || COMET_DBG(p.debug, 64)) continue;
        if (red2) {
          // 0 + slice 0 + slice 1 in slice order (IEEE addition commutes:
          // (0 + other) + own is that value whichever slice is this one)
          const float4* src = rows0 + static_cast<long long>(w.ks ^ 1) * (kTileRows * kBlockN / 4) + s * 16 * kTileRows;
#pragma unroll
          for (int hv = 0; hv < 2; ++hv) {
            uint32_t* v = hv ? v1 : v0;
            float4 q[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) q[i] = __ldcg(src + (hv * 8 + i) * kTileRows);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              v[4 * i] = __float_as_uint((0.f + q[i].x) + __uint_as_float(v[4 * i]));
              v[4 * i + 1] = __float_as_uint((0.f + q[i].y) + __uint_as_float(v[4 * i + 1]));
              v[4 * i + 2] = __float_as_uint((0.f + q[i].z) + __uint_as_float(v[4 * i + 2]));
              v[4 * i + 3] = __float_as_uint((0.f + q[i].w) + __uint_as_float(v[4 * i + 3]));
            }
          }
        }
        process(s, seq++, v0, v1);
      }
      if (tma_out) {  // this warp's tensor stores complete before the unit is counted
        if (lane == 0) ptx::bulk_wait<0>();
        __syncwarp();
      }
      if (early) {
        if (!finisher) {  // partial in memory -> landed
          __threadfence();
          ptx::named_bar_sync(1, kEpiThreads);
          if (threadIdx.x == kEpiThread0) ptx::red_release_gpu_add(landed, 1u);
        } else if (threadIdx.x == kEpiThread0) {  // both slices arrived and landed: reset for the next launch
          p.split_cnt[split_tile] = 0u;
          *landed = 0u;
        }
      } else if (S > 1) {
        // Partial stored -> arrive (acq_rel: the arrival count implies every
        // earlier arriver's partial is visible).  The last arriver finishes
        // the tile's chunks; an earlier arriver polls for the last arrival
        // for a few us and, if it sees it, helps: chunks are claimed one at a
        // time from a per-tile counter.  Nobody waits on a slice that has
        // not arrived beyond that bounded poll, so two slices of one tile
        // queued on one pair (consecutive claims of short slices) cannot
        // deadlock.  Every counter is reset by the launch's last CTA out.
        __threadfence();
        ptx::named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == kEpiThread0) {
          uint32_t* arrive = p.split_cnt + split_tile;
          bool help = ptx::atom_acq_rel_gpu_add(arrive, 1u) == static_cast<uint32_t>(S - 1);
          if (!help) {
            const uint64_t t0 = ptx::globaltimer();
            while (!(help = ptx::ld_acquire_gpu(arrive) >= static_cast<uint32_t>(S)) &&
                   ptx::globaltimer() - t0 < kHelpPollNs) {
            }
          }
          *sflag = help;
        }
        ptx::named_bar_sync(1, kEpiThreads);
        const bool help = *reinterpret_cast<volatile int*>(sflag) != 0;
        int mine[2] = {0, 0};  // (kEpiThread0) real chunks this CTA finished per 256-column half
        if (help) {
          __threadfence();
          fold_wait();
          uint32_t* next = p.split_cnt + 256 + split_tile;
          // two chunks per claim: the even-chunk warps take the first, the
          // odd-chunk warps the second
          for (int hseq = 0;; ++hseq) {
            ptx::named_bar_sync(1, kEpiThreads);  // the previous claim was read by every thread
            if (threadIdx.x == kEpiThread0) {
              const int c0 = static_cast<int>(atomicAdd(next, 2u));
              *sflag = c0;
              for (int c = c0; c < min(c0 + 2, n_chunks); ++c)
                if (c * 64 < cols_left) ++mine[w.half >= 0 ? w.half : (c * 64 >= static_cast<int>(kHalfN) ? 1 : 0)];
            }
            ptx::named_bar_sync(1, kEpiThreads);
            const int c0 = *reinterpret_cast<volatile int*>(sflag);
            if (c0 >= n_chunks) break;
            const int s = c0 + sub;
            if (s >= n_chunks || s * 64 >= cols_left || COMET_DBG(p.debug, 64)) continue;
            uint32_t v0[32], v1[32];
            float acc[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) acc[i] = 0.f;
            for (int k = 0; k < S; ++k) {
              const float4* src = rows0 + static_cast<long long>(k) * (kTileRows * kBlockN / 4) + s * 16 * kTileRows;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float4 q4 = __ldcg(src + i * kTileRows);
                acc[4 * i] += q4.x; acc[4 * i + 1] += q4.y; acc[4 * i + 2] += q4.z; acc[4 * i + 3] += q4.w;
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v0[i] = __float_as_uint(acc[i]);
              v1[i] = __float_as_uint(acc[32 + i]);
            }
            process(s, seq++, v0, v1);
          }
          if (tma_out) {
            if (lane == 0) ptx::bulk_wait<0>();
            __syncwarp();
          }
        }
        __threadfence();
        ptx::named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == kEpiThread0) {
          // a half is complete when all of its real chunks are (any CTA)
          uint32_t done = 0u;
          uint32_t* hc = p.split_cnt + 512 + 2 * split_tile;
          for (int h = 0; h < 2; ++h) {
            if (!mine[h]) continue;
            int real = 0;
            for (int c = 0; c < n_chunks; ++c)
              real += c * 64 < cols_left && (w.half >= 0 ? w.half : (c * 64 >= static_cast<int>(kHalfN) ? 1 : 0)) == h;
            if (atomicAdd(hc + h, static_cast<uint32_t>(mine[h])) + mine[h] == static_cast<uint32_t>(real)) done |= 1u << h;
          }
          *sflag = static_cast<int>(done);
        }
        ptx::named_bar_sync(1, kEpiThreads);
        split_done = static_cast<uint32_t>(*reinterpret_cast<volatile int*>(sflag));
      }
      // completion counted in real 256-column halves (half 1 of a narrow last
      // block -- a split-tail half -- covers none); split-K: by the finisher,
      // or (S > 2) per half by the slice that completed it
      const uint32_t done_mask = S > 2 ? split_done
                                 : !finisher ? 0u
                                 : w.half < 0 ? 3u
                                 : ((w.half == 1 && narrow_block(p, w.nb)) ? 0u : (1u << w.half));
      const uint32_t amount = __popc(done_mask);
      if (w.layer == 0 && f.mode == 2) {
        // this CTA's 128 H rows of the unit's columns are in memory -> count
        // them for the layer1 units that read the tile as their A operand
        ptx::fence_async_global();
        ptx::named_bar_sync(1, kEpiThreads);
        if (threadIdx.x == kEpiThread0 && amount) {
          __threadfence();
          ptx::red_release_gpu_add(f.h_cnt + static_cast<long long>(row0 >> 7) * NB + w.nb, amount);
        }
      } else if (w.layer == 1) {
        // this CTA's 128 rows of column block nb are in memory -> count them
        if (p.out_cnt && p.fuse_combine)
          if (sub == 0) srow_chunk[threadIdx.x - kEpiThread0] = (out_row && amount) ? fold_t / p.chunk_tokens : -1;
        // pushed rows become visible to the peer through the releasing
        // thread's system-scope fence in nb_contributed (cumulative over the
        // CTA's stores ordered before it by the barrier) -- one fence per CTA
        // instead of one per thread; rows written by TMA stores (completed
        // above) are ordered before the release by a proxy fence, as in layer0
        if (tma_out) ptx::fence_async_global();
        ptx::named_bar_sync(1, kEpiThreads);
        if (p.out_cnt && p.fuse_combine && threadIdx.x == kEpiThread0 && amount) {
          // streamed forward: these output rows' halves are final -> count
          // them per token chunk (rows are token-sorted: few runs) for the
          // download stream; one system fence covers the CTA's stores
          __threadfence_system();
          int run_c = -1, run_n = 0;
          for (int r = 0; r < 128; ++r) {
            const int cr = srow_chunk[r];
            if (cr != run_c) {
              if (run_c >= 0) atomicAdd(p.out_cnt + run_c, static_cast<uint32_t>(run_n) * amount);
              run_c = cr;
              run_n = 0;
            }
            run_n += cr >= 0;
          }
          if (run_c >= 0) atomicAdd(p.out_cnt + run_c, static_cast<uint32_t>(run_n) * amount);
        }
        if (threadIdx.x == kEpiThread0 && amount) {
          __threadfence();
          ptx::red_release_gpu_add(p.nb_done + w.nb, amount);
          if (p.fuse_combine || p.publish_tiles)
            for (int h = 0; h < 2; ++h)
              if ((done_mask >> h) & 1u)
                ptx::st_release_gpu(p.tile_done + (static_cast<long long>(row0 >> 7) * NB + w.nb) * 2 + h, p.epoch);
          if (p.world > 1)
            comm::nb_contributed(p, w.nb, amount,
                                 (narrow_block(p, w.nb) ? 2u : 4u) * static_cast<uint32_t>(P) +
                                     (gridDim.x - static_cast<uint32_t>(p.n_compute)));
        }
      }
      if (threadIdx.x == kEpiThread0) tl_record(p, kRoleEpilogue, it, g, t_e, ptx::globaltimer());
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, kTmemCols);
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
moe_layer_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_b0,
                 const __grid_constant__ CUtensorMap tm_a1, const __grid_constant__ CUtensorMap tm_b1,
                 const __grid_constant__ CUtensorMap tm_s0, const __grid_constant__ CUtensorMap tm_s1,
                 const __grid_constant__ KernelArgs f) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_last;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b = static_cast<int>(blockIdx.x);
  const uint64_t t_entry = ptx::globaltimer();
  bool compute = true;
  ptx::pdl_launch_dependents();  // the next kernel may start its launch / prologue
  if (f.mode == 1 && b >= f.l[1].n_compute) {
    // layer1 combine CTA (world 1, comm-CTA combine): reduces to the end
    ptx::pdl_wait();
    if (!COMET_DBG(f.l[1].debug, 1)) comm::combine_reduce(f.l[1], smem);
    compute = false;
  } else if (f.mode != 1 && b >= f.l[0].n_compute) {
    // layer0 dispatch CTA: pull the remote rows, then join the compute pairs
    ptx::pdl_wait();
    if (!COMET_DBG(f.l[0].debug, 1)) {
      if (f.l[0].dedup) comm::dispatch_rows_dedup(f.l[0], smem);
      else comm::dispatch_rows(f.l[0], smem);
    }
    __syncthreads();
    comm::comm_release(f.l[0], smem);
    __syncthreads();
    if (b - f.l[0].n_compute < f.n_dl) {  // zero-copy forward: download the output instead
      download_rows(f, b - f.l[0].n_compute);
      compute = false;
    } else if (f.l[0].stream_combine) {  // streamed forward: reduce finished token chunks instead
      LayerArgs pc = f.l[1];
      pc.n_compute = f.l[0].n_compute;
      comm::stream_combine(pc, smem);
      compute = false;
    }
  }
  if (compute) compute_role(f, smem, &tm_a0, &tm_b0, &tm_a1, &tm_b1, &tm_s0, &tm_s1);

  // The last CTA out resets the launch's claim counter and H-tile counters
  // (nothing reads them after every CTA has left).
  __syncthreads();
  {  // CTA lifetime (launch skew / prologue / tail): the last tmem-wait record, task kLifeTask
    const LayerArgs& pl = f.l[f.mode == 1 ? 1 : 0];
    if (threadIdx.x == 0) tl_record(pl, kRoleTmemWait, pl.timeline_cap - 1, kLifeTask, t_entry, ptx::globaltimer());
  }
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(f.sched + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (int i = threadIdx.x; i < f.n_h; i += blockDim.x) f.h_cnt[i] = 0u;
    for (int l = 0; l < 2; ++l)  // split-K counters (arrivals, chunk claims, finished chunks)
      if (f.l[l].split_cnt)
        for (int i = threadIdx.x; i < 1024; i += blockDim.x) f.l[l].split_cnt[i] = 0u;
    if (threadIdx.x == 0) {
      f.sched[0] = 0u;
      f.sched[1] = 0u;
    }
    __threadfence();
  }
}

// Final combine on the source rank (world > 1): sum the partial rows pushed by
// every contributing rank, ascending rank order (executor.py:239-245 for TP,
// 102-120 for experts split across EP groups).  One warp per (token, 1024-
// column segment): the contributor list comes from the token's router row,
// then each lane issues all its 16 B loads of every contributor before
// summing (latency-bound: ~8 loads in flight per lane, whole GPU).
__global__ void __launch_bounds__(256) combine_finish_kernel(const LayerArgs p, const __nv_bfloat16* cb,
                                                             const uint32_t* cb_flag, const int32_t* experts) {
  ptx::pdl_launch_dependents();
  ptx::pdl_wait();
  const int NB = p.n_blocks, N = p.n_embed, K = p.topk, W = p.world;
  const int start = token_start_of(p.rank, p.M, W);
  const int n_own = token_stop_of(p.rank, p.M, W) - start;
  for (int i = threadIdx.x; i < W * NB; i += blockDim.x)
    { ptx::Spin sp; while (!ptx::epoch_reached(ptx::ld_acquire_sys(cb_flag + i), p.epoch)) sp.pause(64, 6); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int vec = N / 8;
  constexpr int kU = 4;
  constexpr int kSegVec = 32 * kU;  // 16 B vectors per segment
  const int n_seg = (vec + kSegVec - 1) / kSegVec;
  const long long items = static_cast<long long>(n_own) * n_seg;
  for (long long item = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; item < items;
       item += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const int lt = static_cast<int>(item / n_seg), seg = static_cast<int>(item % n_seg);
    const int t = start + lt;
    // contributing ranks: every TP rank of each distinct EP group of t's
    // experts (ascending experts -> ascending groups -> ascending ranks)
    const int ge = lane < K ? experts[static_cast<long long>(t) * K + lane] / p.experts_per_group : -1;
    int groups[8];
    int ng = 0, last = -1;
    for (int s = 0; s < K; ++s) {
      const int g = __shfl_sync(0xffffffffu, ge, s);
      if (g != last) groups[ng++] = g;
      last = g;
    }
    const int c0 = seg * kSegVec + lane;
    float acc[kU][8];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[u][j] = 0.f;
    for (int gi = 0; gi < ng; ++gi) {
      for (int r = groups[gi] * p.tp; r < (groups[gi] + 1) * p.tp; ++r) {
        const __nv_bfloat16* row = cb + (static_cast<long long>(r) * p.mloc_cap + lt) * N;
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
          v[u] = c0 + u * 32 < vec ? ptx::ld_v4(row + (c0 + u * 32) * 8) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(h[j]);
            acc[u][2 * j] += f.x;
            acc[u][2 * j + 1] += f.y;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (c0 + u * 32 >= vec) continue;
      uint4 o;
      o.x = pack_bf16(acc[u][0], acc[u][1]); o.y = pack_bf16(acc[u][2], acc[u][3]);
      o.z = pack_bf16(acc[u][4], acc[u][5]); o.w = pack_bf16(acc[u][6], acc[u][7]);
      ptx::st_v4(p.y_local + static_cast<long long>(lt) * N + (c0 + u * 32) * 8, o);
    }
  }
}

// Local half of the layer0 dispatch: copy every row whose token lives on this
// rank from the token buffer into its slot of the expert-sorted shared tensor
// (HBM-bound; one warp per row, 16 B per lane per access, whole GPU).
__global__ void __launch_bounds__(256) dispatch_local_kernel(const int32_t* __restrict__ gather_row,
                                                             const int32_t* __restrict__ meta,
                                                             const __nv_bfloat16* __restrict__ xs,
                                                             __nv_bfloat16* __restrict__ xg, int n_embed, int M,
                                                             int world, int rank) {
  ptx::pdl_launch_dependents();
  ptx::pdl_wait();
  const int rows = meta[kMetaRowsPad];
  const int vec = n_embed / 8;
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int t = gather_row[r];
    if (t < 0 || src_rank_of(t, M, world) != rank) continue;
    const uint4* s = reinterpret_cast<const uint4*>(xs + static_cast<long long>(t) * n_embed);
    uint4* d = reinterpret_cast<uint4*>(xg + static_cast<long long>(r) * n_embed);
    int i = lane;
    for (; i + 7 * 32 < vec; i += 8 * 32) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ptx::ld_nc_v4(s + i + u * 32);
#pragma unroll
      for (int u = 0; u < 8; ++u) d[i + u * 32] = v[u];
    }
    for (; i < vec; i += 32) d[i] = ptx::ld_nc_v4(s + i);
  }
}

// Local top-k combine after layer1 (world == 1, or n_comm == 0): y[t] = left
// fold over t's expert rows in ascending slot order, weighted when combine
// weights are given (executor.py:102-120).  HBM-bound, whole GPU.
__global__ void __launch_bounds__(256) combine_local_kernel(const int32_t* __restrict__ tok_pos,
                                                            const float* __restrict__ combine_w,
                                                            const __nv_bfloat16* __restrict__ yrows,
                                                            __nv_bfloat16* __restrict__ y, int t0, int n_tok,
                                                            int topk, int n_embed) {
  ptx::pdl_launch_dependents();
  ptx::pdl_wait();
  const int vec = n_embed / 8;
  const long long items = static_cast<long long>(n_tok) * vec;
  for (long long it = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; it < items;
       it += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int lt = static_cast<int>(it / vec), c = static_cast<int>(it % vec) * 8;
    const int t = t0 + lt;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int s = 0; s < topk; ++s) {
      const int pos = tok_pos[t * topk + s];
      if (pos < 0) continue;
      const float w = combine_w ? combine_w[t * topk + s] : 1.f;
      const uint4 v = ptx::ld_nc_v4(yrows + static_cast<long long>(pos) * n_embed + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        acc[2 * j] += f.x * w;
        acc[2 * j + 1] += f.y * w;
      }
    }
    uint4 o;
    o.x = pack_bf16(acc[0], acc[1]); o.y = pack_bf16(acc[2], acc[3]);
    o.z = pack_bf16(acc[4], acc[5]); o.w = pack_bf16(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(y + static_cast<long long>(lt) * n_embed + c) = o;
  }
}

// Publish "my tokens are in my token-slot buffer" to every peer.
__global__ void signal_x_ready_kernel(uint32_t* const* x_ready_peer, int rank, int world, uint32_t epoch) {
  const int d = threadIdx.x;
  if (d < world) {
    ptx::fence_acq_rel_sys();
    ptx::st_release_sys(x_ready_peer[d] + rank, epoch);
  }
}

}  // namespace comet

// host: this unit's device-wait timeout (ptx::Spin)
cudaError_t set_spin_timeout_layers(unsigned long long ns) {
  return cudaMemcpyToSymbol(comet::ptx::g_spin_timeout_ns, &ns, sizeof(ns));
}
cudaError_t set_abort_flag_layers(const volatile uint32_t* p) {
  return cudaMemcpyToSymbol(comet::ptx::g_abort_flag, &p, sizeof(p));
}
