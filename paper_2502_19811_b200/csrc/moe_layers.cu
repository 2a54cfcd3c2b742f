// COMET fused MoE layer kernels for sm_100a.
//
// One persistent launch per layer, thread-block specialised (PAPER.md
// section 3.2.1): CTAs [0, n_compute) form 2-CTA clusters that run a
// tcgen05 GroupGEMM (UMMA 256x256x16, cta_group::2, accumulators in TMEM,
// operands staged by TMA); CTAs [n_compute, grid) are communication CTAs.
//
//   layer0 (reference resolve_layer0 + _hidden_row, resolver.py:206-252,
//   executor.py:86-90): comm CTAs pull each distinct remote token once over
//   NVLink into this rank's token-slot buffer, in the order the compute
//   schedule first needs it, and publish a per-token ready epoch; compute
//   pairs claim 256-row units in locality-first order, gather their A rows
//   straight from the token-slot buffer with TMA tile::gather4, and apply the
//   activation in the TMEM->register epilogue before a TMA store of H.
//
//   layer1 (resolve_layer1 + _output_columns + _combine, resolver.py:255-309,
//   executor.py:93-120): compute pairs walk column waves (n-block groups
//   outer, expert/row pairs inner) and count finished units per n-block;
//   comm CTAs reduce each finished column block over every token's hosted
//   experts in ascending expert order (weighted when combine weights are
//   given) and either write the layer output (world == 1) or push the
//   partial row to the token's source rank over NVLink.
#include <cuda.h>
#include <cuda_bf16.h>

#include "layers.cuh"
#include "ptx.cuh"

namespace comet {

namespace {

constexpr int kThreads = 256;
constexpr int kStages = 6;
constexpr int kBlockK = 64;                       // bf16 elements = 128 B swizzle atom
constexpr uint32_t kSmemA = kTileRows * kBlockK * 2;   // 16 KB
constexpr uint32_t kSmemB = 128 * kBlockK * 2;         // 16 KB (half of the 256-row B block)
constexpr uint32_t kSmemStage = kSmemA + kSmemB;
constexpr uint32_t kSmemEpi = kTileRows * 128;          // 128 rows x 64 bf16
constexpr uint32_t kAccCols = kBlockN;                  // fp32 columns per accumulator
constexpr uint32_t kTmemCols = 2 * kAccCols;
constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(2 * kTileRows, kBlockN);
constexpr int kEpiThread0 = 128;                        // first epilogue thread
constexpr int kCommWarps = kThreads / 32;

struct Unit {
  int pair, nb;
};

// Unit u -> (pair, n-block).  layer0: groups of `G` pairs, n-block middle,
// pair inner (weights block shared by the group, group's rows stay in L2);
// layer1: waves of `G` n-blocks, pair outer, n-block inner (the reference's
// column-wave order at wave granularity).
__device__ __forceinline__ Unit decode_unit(int u, int layer, int P, int NB, int G) {
  Unit r;
  if (layer == 0) {
    const int per_group = G * NB;
    const int g = u / per_group;
    const int base = g * G;
    const int ge = min(G, P - base);
    const int rem = u - g * per_group;
    r.nb = rem / ge;
    r.pair = base + rem % ge;
  } else {
    const int per_wave = P * G;
    const int w = u / per_wave;
    const int nb0 = w * G;
    const int we = min(G, NB - nb0);
    const int rem = u - w * per_wave;
    r.pair = rem / we;
    r.nb = nb0 + rem % we;
  }
  return r;
}

__device__ __forceinline__ float activate(float x, int act) {
  switch (act) {
    case kActRelu: return fmaxf(x, 0.f);
    case kActSilu: return x / (1.f + __expf(-x));
    case kActGeluTanh: {
      const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
      return 0.5f * x * (1.f + tanhf(u));
    }
    case kActTanh: return tanhf(x);
    default: return x;
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------ comm roles --
// layer0: pull distinct remote tokens (first-demand order) into xs_local.
__device__ void dispatch_pull(const LayerArgs& p) {
  const int n_comm = gridDim.x - p.n_compute;
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_pull = p.meta[kMetaPull];
  const int row_vec = p.n_embed / 8;  // uint4 per row
  uint64_t ready_mask = 0;            // peers whose tokens are known in place
  for (int q = cid * kCommWarps + warp; q < n_pull; q += n_comm * kCommWarps) {
    const int t = p.pull_token[q], src = p.pull_src[q];
    if (!((ready_mask >> src) & 1)) {
      if (lane == 0)
        while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.x_ready + src), p.epoch)) __nanosleep(64);
      __syncwarp();
      ready_mask |= 1ull << src;
    }
    const uint4* s = reinterpret_cast<const uint4*>(p.xs_peer[src] + static_cast<long long>(t) * p.n_embed);
    uint4* d = reinterpret_cast<uint4*>(p.xs_local + static_cast<long long>(t) * p.n_embed);
    int i = lane;
    for (; i + 96 < row_vec; i += 128) {
      const uint4 a = ptx::ld_nc_v4(s + i), b = ptx::ld_nc_v4(s + i + 32);
      const uint4 c = ptx::ld_nc_v4(s + i + 64), e = ptx::ld_nc_v4(s + i + 96);
      ptx::st_v4(d + i, a); ptx::st_v4(d + i + 32, b);
      ptx::st_v4(d + i + 64, c); ptx::st_v4(d + i + 96, e);
    }
    for (; i < row_vec; i += 32) ptx::st_v4(d + i, ptx::ld_nc_v4(s + i));
    __threadfence();
    __syncwarp();
    if (lane == 0) ptx::st_release_gpu(p.tok_ready + t, p.epoch);
  }
}

// layer1: per finished n-block, top-k reduce of each hosted token.
__device__ void combine_reduce(const LayerArgs& p) {
  const int n_comm = gridDim.x - p.n_compute;
  const int cid = blockIdx.x - p.n_compute;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = p.meta[kMetaPairs];
  const int n_tok = p.meta[kMetaCombineTok];
  const int NB = p.n_blocks, K = p.topk, N = p.n_embed;
  const uint32_t target = 2u * static_cast<uint32_t>(P);
  const int start_r = token_start_of(p.rank, p.M, p.world);
  if (p.world > 1) {
    // Every peer has finished its previous forward (it signalled this epoch's
    // tokens), so its combine buffer and flags may be overwritten.
    if (threadIdx.x < p.world)
      while (!ptx::epoch_reached(ptx::ld_acquire_sys(p.x_ready + threadIdx.x), p.epoch)) __nanosleep(64);
    __syncthreads();
  }
  for (int nb = 0; nb < NB; ++nb) {
    if (threadIdx.x == 0) {
      while (ptx::ld_acquire_gpu(p.nb_done + nb) < target) __nanosleep(128);
    }
    __syncthreads();
    const int col = nb * kBlockN + lane * 8;
    const bool col_ok = col < N;
    for (int i = cid * kCommWarps + warp; col_ok && i < n_tok; i += n_comm * kCommWarps) {
      const int t = p.combine_tok[i];
      float acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.f;
      for (int s = 0; s < K; ++s) {
        const int pos = p.tok_pos[t * K + s];
        if (pos < 0) continue;
        const float w = p.combine_w ? p.combine_w[t * K + s] : 1.f;
        const uint4 v = ptx::ld_v4(p.yrows + static_cast<long long>(pos) * N + col);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float2 f = __bfloat1622float2(h[c]);
          acc[2 * c] += (p.combine_w ? f.x * w : f.x);
          acc[2 * c + 1] += (p.combine_w ? f.y * w : f.y);
        }
      }
      uint4 o;
      o.x = pack_bf16(acc[0], acc[1]); o.y = pack_bf16(acc[2], acc[3]);
      o.z = pack_bf16(acc[4], acc[5]); o.w = pack_bf16(acc[6], acc[7]);
      if (p.world == 1) {
        ptx::st_v4(p.y_local + static_cast<long long>(t - start_r) * N + col, o);
      } else {
        const int dst = src_rank_of(t, p.M, p.world);
        const int slot = p.rank * p.mloc_cap + (t - token_start_of(dst, p.M, p.world));
        ptx::st_v4(p.cb_peer[dst] + static_cast<long long>(slot) * N + col, o);
      }
    }
    if (p.world > 1) {
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t prev = ptx::atom_acq_rel_gpu_add(p.nb_sent + nb, 1u);
        if (prev == static_cast<uint32_t>(n_comm) - 1) {
          ptx::fence_acq_rel_sys();
          for (int d = 0; d < p.world; ++d)
            ptx::st_release_sys(p.cb_flag_peer[d] + p.rank * NB + nb, p.epoch);
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 1)
moe_layer_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                 const __grid_constant__ CUtensorMap tm_out, const LayerArgs p) {
  if (static_cast<int>(blockIdx.x) >= p.n_compute) {
    if (p.layer == 0) dispatch_pull(p);
    else combine_reduce(p);
    return;
  }

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kSmemStage + 2 * kSmemEpi);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = blockIdx.x & 1;  // rank in the 2-CTA cluster
  const bool leader = cta == 0;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_a);
    ptx::prefetch_tmap(&tm_b);
    ptx::prefetch_tmap(&tm_out);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(full + s, 2);
      ptx::mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(tfull + a, 1);
      ptx::mbar_init(tempty + a, 2 * 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  const int P = p.meta[kMetaPairs];
  const int NB = p.n_blocks;
  const int U = P * NB;
  const int pair_id = blockIdx.x >> 1;
  const int n_pairs = p.n_compute >> 1;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int u = pair_id; u < U; u += n_pairs) {
      const Unit w = decode_unit(u, p.layer, P, NB, p.order_group);
      const int4 pr = reinterpret_cast<const int4*>(p.pairs)[w.pair];
      const int row0 = pr.y + kTileRows * static_cast<int>(cta);
      const int brow = pr.x * p.b_rows + w.nb * kBlockN + 128 * static_cast<int>(cta);
      int4 tok = make_int4(-1, -1, -1, -1);
      if (p.layer == 0) {
        tok = reinterpret_cast<const int4*>(p.gather_row + row0)[lane];
        if (p.world > 1) {
          const int tt[4] = {tok.x, tok.y, tok.z, tok.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int t = tt[i];
            if (t >= 0 && src_rank_of(t, p.M, p.world) != p.rank)
              while (!ptx::epoch_reached(ptx::ld_acquire_gpu(p.tok_ready + t), p.epoch)) __nanosleep(32);
          }
          ptx::fence_async_global();
          __syncwarp();
        }
      }
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        ptx::mbar_wait(empty + stage, phase ^ 1);
        uint8_t* sa = smem + stage * kSmemStage;
        uint8_t* sb = sa + kSmemA;
        if (p.layer == 0) {
          ptx::tma_gather4_2sm(sa + lane * 512, &tm_a, full + stage, kb * kBlockK, tok.x, tok.y, tok.z, tok.w);
        } else if (lane == 0) {
          ptx::tma_load_2d_2sm(sa, &tm_a, full + stage, kb * kBlockK, row0, ptx::kEvictNormal);
        }
        if (lane == 0) {
          ptx::tma_load_2d_2sm(sb, &tm_b, full + stage, kb * kBlockK, brow, ptx::kEvictNormal);
          if (leader) ptx::mbar_arrive_expect_tx(full + stage, 2 * kSmemStage);
          else ptx::mbar_arrive_cluster(full + stage, 0);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issuer (leader CTA, one thread) ----------------
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = pair_id; u < U; u += n_pairs, ++it) {
      const int a = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      ptx::mbar_wait(tempty + a, aphase ^ 1);
      ptx::tc_fence_after();
      const uint32_t dcol = tmem_base + a * kAccCols;
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        ptx::mbar_wait(full + stage, phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t sa = ptx::smem_u32(smem + stage * kSmemStage);
          const uint64_t da = ptx::sdesc_kmajor_sw128(sa);
          const uint64_t db = ptx::sdesc_kmajor_sw128(sa + kSmemA);
#pragma unroll
          for (int k = 0; k < kBlockK / 16; ++k)
            ptx::mma_bf16_2sm(dcol, da + 2 * k, db + 2 * k, kIdesc, (kb | k) != 0);
          ptx::mma_commit_2sm(empty + stage, 0x3);
          if (kb == p.k_blocks - 1) ptx::mma_commit_2sm(tfull + a, 0x3);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> regs -> smem -> TMA store ----------------
    const int ew = warp - 4;
    const int row = ew * 32 + lane;  // row of this CTA's 128-row half
    int it = 0, buf = 0;
    for (int u = pair_id; u < U; u += n_pairs, ++it) {
      const Unit w = decode_unit(u, p.layer, P, NB, p.order_group);
      const int4 pr = reinterpret_cast<const int4*>(p.pairs)[w.pair];
      const int row0 = pr.y + kTileRows * static_cast<int>(cta);
      const int a = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      ptx::mbar_wait(tfull + a, aphase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + a * kAccCols;
#pragma unroll 1
      for (int s = 0; s < kBlockN / 64; ++s) {
        uint32_t v0[32], v1[32];
        ptx::tmem_ld32(taddr + s * 64, v0);
        ptx::tmem_ld32(taddr + s * 64 + 32, v1);
        ptx::tmem_ld_wait();
        if (s == kBlockN / 64 - 1) {
          ptx::tc_fence_before();
          if (leader) ptx::mbar_arrive(tempty + a);
          else ptx::mbar_arrive_cluster(tempty + a, 0);
        }
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16(activate(__uint_as_float(v0[2 * i]), p.activation),
                            activate(__uint_as_float(v0[2 * i + 1]), p.activation));
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[16 + i] = pack_bf16(activate(__uint_as_float(v1[2 * i]), p.activation),
                                 activate(__uint_as_float(v1[2 * i + 1]), p.activation));
        if (threadIdx.x == kEpiThread0) ptx::bulk_wait_read<1>();
        ptx::named_bar_sync(1, 128);
        uint8_t* sbuf = smem + kStages * kSmemStage + buf * kSmemEpi;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = row * 128 + ((c ^ (row & 7)) * 16);
          *reinterpret_cast<uint4*>(sbuf + off) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        }
        ptx::fence_async_shared();
        ptx::named_bar_sync(1, 128);
        if (threadIdx.x == kEpiThread0) {
          ptx::tma_store_2d(&tm_out, sbuf, w.nb * kBlockN + s * 64, row0);
          ptx::bulk_commit();
        }
        buf ^= 1;
      }
      if (p.layer == 1 && threadIdx.x == kEpiThread0) {
        ptx::bulk_wait<0>();
        ptx::fence_async_global();
        ptx::red_release_gpu_add(p.nb_done + w.nb, 1u);
      }
    }
    if (threadIdx.x == kEpiThread0) ptx::bulk_wait<0>();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, kTmemCols);
}

// Final combine on the source rank (world > 1): sum the partial rows pushed by
// every contributing rank, ascending rank order (executor.py:239-245 for TP,
// 102-120 for experts split across EP groups).
__global__ void __launch_bounds__(256) combine_finish_kernel(const LayerArgs p, const __nv_bfloat16* cb,
                                                             const uint32_t* cb_flag, const int32_t* experts) {
  const int NB = p.n_blocks, N = p.n_embed, K = p.topk, W = p.world;
  const int start = token_start_of(p.rank, p.M, W);
  const int n_own = token_stop_of(p.rank, p.M, W) - start;
  for (int i = threadIdx.x; i < W * NB; i += blockDim.x)
    while (!ptx::epoch_reached(ptx::ld_acquire_sys(cb_flag + i), p.epoch)) __nanosleep(64);
  __syncthreads();
  const int vec = N / 8;
  const long long n_items = static_cast<long long>(n_own) * vec;
  for (long long it = blockIdx.x * blockDim.x + threadIdx.x; it < n_items;
       it += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int lt = static_cast<int>(it / vec), c = static_cast<int>(it % vec) * 8;
    const int t = start + lt;
    // contributing ranks: every TP rank of each distinct EP group of t's
    // experts, visited in ascending rank order
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    int last_group = -1;
    for (int s = 0; s < K; ++s) {
      const int g = experts[static_cast<long long>(t) * K + s] / p.experts_per_group;
      if (g == last_group) continue;
      last_group = g;
      for (int r = g * p.tp; r < (g + 1) * p.tp; ++r) {
        const uint4 v = ptx::ld_v4(cb + (static_cast<long long>(r) * p.mloc_cap + lt) * N + c);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(h[j]);
          acc[2 * j] += f.x;
          acc[2 * j + 1] += f.y;
        }
      }
    }
    uint4 o;
    o.x = pack_bf16(acc[0], acc[1]); o.y = pack_bf16(acc[2], acc[3]);
    o.z = pack_bf16(acc[4], acc[5]); o.w = pack_bf16(acc[6], acc[7]);
    ptx::st_v4(p.y_local + static_cast<long long>(lt) * N + c, o);
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
