// Row-gather copy engine microbenchmark (diagnostic tool, not product code).
// n_cta CTAs copy `rows` gathered 8 KB rows (random source permutation) from
// src to dst, the dispatch engine's data movement, in variants:
//   mode 0: TMA bulk load -> smem ring -> TMA bulk store, one storer thread
//           (release lag `lag` bulk groups)
//   mode 1: same, storer work split over 8 lanes (each its own bulk groups)
//   mode 2: register copies, one warp per row, 16 B per lane per access,
//           `unroll` accesses in flight per lane, all 8 warps
//   mode 3: TMA bulk load -> smem ring -> st.global from smem by 7 warps
// Prints GB/s (read bytes) per configuration.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <string>
#include <cstring>

#include "../paper_2502_19811_b200/csrc/ptx.cuh"

using namespace comet;

constexpr int kRowBytes = 8192;
constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads, 1) copy_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                        const int* __restrict__ perm, int rows, int n_slots, int lag,
                                                        int n_store_lanes) {
  extern __shared__ uint8_t raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + n_slots * kRowBytes);
  uint64_t* empty = full + n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_slots; ++i) {
      ptx::mbar_init(full + i, 1);
      ptx::mbar_init(empty + i, 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // rows of this CTA: r = blockIdx.x + j * gridDim.x
  const int my_rows = rows > (int)blockIdx.x ? (rows - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == 0) {
    // lane-parallel index loads, then one lane issues in job order (no
    // intra-warp convergence on slot waits)
    for (int j0 = 0; j0 < my_rows; j0 += 32) {
      const int jl = j0 + lane;
      const int tl = jl < my_rows ? perm[blockIdx.x + jl * gridDim.x] : 0;
      const int nb = my_rows - j0 < 32 ? my_rows - j0 : 32;
      for (int i = 0; i < nb; ++i) {
        const int t = __shfl_sync(0xffffffffu, tl, i);
        const int j = j0 + i;
        if (lane == 0) {
          const int slot = j % n_slots;
          ptx::mbar_wait(empty + slot, ((j / n_slots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(full + slot, kRowBytes);
          ptx::bulk_load(ring + slot * kRowBytes, src + (long long)t * kRowBytes, kRowBytes, full + slot);
        }
      }
      __syncwarp();
    }
  } else if (warp >= 1 && warp <= n_store_lanes && lane == 0) {
    // one storer thread per warp (independent bulk groups, no shared convergence)
    const int sl = warp - 1;
    int n = 0;
    for (int j = sl; j < my_rows; j += n_store_lanes, ++n) {
      const int r = blockIdx.x + j * gridDim.x;
      const int slot = j % n_slots;
      ptx::mbar_wait(full + slot, (j / n_slots) & 1);
      ptx::bulk_store(dst + (long long)r * kRowBytes, ring + slot * kRowBytes, kRowBytes);
      ptx::bulk_commit();
      if (lag == 0) {
        ptx::bulk_wait_read<0>();
        ptx::mbar_arrive(empty + slot);
      } else {
        ptx::bulk_wait_read<1>();
        const int jo = j - n_store_lanes;
        if (jo >= 0) ptx::mbar_arrive(empty + jo % n_slots);
      }
    }
    ptx::bulk_wait_read<0>();
    // release the tail so the loader never blocks (not needed at exit)
    ptx::bulk_wait<0>();
  }
}

template <int U>
__global__ void __launch_bounds__(kThreads, 1) copy_regs(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                         const int* __restrict__ perm, int rows) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (kThreads / 32) + warp, nw = gridDim.x * (kThreads / 32);
  for (int r = gw; r < rows; r += nw) {
    const uint4* s = reinterpret_cast<const uint4*>(src + (long long)perm[r] * kRowBytes);
    uint4* d = reinterpret_cast<uint4*>(dst + (long long)r * kRowBytes);
    for (int i = lane; i < kRowBytes / 16; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ptx::ld_nc_v4(s + i + u * 32);
#pragma unroll
      for (int u = 0; u < U; ++u) d[i + u * 32] = v[u];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) copy_tma_st(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                           const int* __restrict__ perm, int rows, int n_slots) {
  extern __shared__ uint8_t raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + n_slots * kRowBytes);
  uint64_t* empty = full + n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n_slots; ++i) {
      ptx::mbar_init(full + i, 1);
      ptx::mbar_init(empty + i, 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int my_rows = rows > (int)blockIdx.x ? (rows - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == 0) {
    // lane-parallel index loads, then one lane issues in job order (no
    // intra-warp convergence on slot waits)
    for (int j0 = 0; j0 < my_rows; j0 += 32) {
      const int jl = j0 + lane;
      const int tl = jl < my_rows ? perm[blockIdx.x + jl * gridDim.x] : 0;
      const int nb = my_rows - j0 < 32 ? my_rows - j0 : 32;
      for (int i = 0; i < nb; ++i) {
        const int t = __shfl_sync(0xffffffffu, tl, i);
        const int j = j0 + i;
        if (lane == 0) {
          const int slot = j % n_slots;
          ptx::mbar_wait(empty + slot, ((j / n_slots) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(full + slot, kRowBytes);
          ptx::bulk_load(ring + slot * kRowBytes, src + (long long)t * kRowBytes, kRowBytes, full + slot);
        }
      }
      __syncwarp();
    }
  } else {
    const int me = warp - 1, nst = kThreads / 32 - 1;
    for (int j = me; j < my_rows; j += nst) {
      const int r = blockIdx.x + j * gridDim.x;
      const int slot = j % n_slots;
      ptx::mbar_wait(full + slot, (j / n_slots) & 1);
      const uint4* s = reinterpret_cast<const uint4*>(ring + slot * kRowBytes);
      uint4* d = reinterpret_cast<uint4*>(dst + (long long)r * kRowBytes);
      uint4 v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = s[lane + u * 32];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(empty + slot);
#pragma unroll
      for (int u = 0; u < 16; ++u) d[lane + u * 32] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  const bool host_src = argc > 1 && std::string(argv[1]) == "host";
  const bool host_dst = argc > 1 && std::string(argv[1]) == "hostdst";
  const int rows = 16384;
  const size_t bytes = (size_t)rows * kRowBytes;
  uint8_t *src, *dst;
  int* perm;
  if (host_src) {  // zero-copy: pinned host memory read over PCIe by the kernels
    cudaHostAlloc(&src, bytes, cudaHostAllocMapped);
    memset(src, 1, bytes);
  } else {
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
  }
  if (host_dst)  // zero-copy writes: pinned host destination written over PCIe
    cudaHostAlloc(&dst, bytes, cudaHostAllocMapped);
  else
    cudaMalloc(&dst, bytes);
  cudaMalloc(&perm, rows * 4);
  std::vector<int> hp(rows);
  for (int i = 0; i < rows; ++i) hp[i] = i;
  std::shuffle(hp.begin(), hp.end(), std::mt19937(1));
  cudaMemcpy(perm, hp.data(), rows * 4, cudaMemcpyHostToDevice);
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(copy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(copy_tma_st, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, int ctas, auto launch) {
    for (int w = 0; w < 2; ++w) launch();
    cudaEventRecord(a);
    const int it = 3;
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    // verify a few rows arrived
    std::vector<uint8_t> chk(64);
    cudaMemcpy(chk.data(), dst, 64, cudaMemcpyDeviceToHost);
    printf("%-34s ctas=%3d  %8.1f GB/s total  %7.1f GB/s per CTA %s %s\n", name, ctas, bytes * it / (ms * 1e-3) / 1e9,
           bytes * it / (ms * 1e-3) / 1e9 / ctas, e == cudaSuccess ? "" : cudaGetErrorString(e), chk[0] == 1 ? "ok" : "BAD");
    cudaMemset(dst, 0, bytes);
  };
  printf("source: %s, destination: %s\n", host_src ? "pinned host (zero-copy)" : "device",
         host_dst ? "pinned host (zero-copy)" : "device");
  for (int ctas : {8, 16, 32, 64, 132}) {
    char nm[64];
    snprintf(nm, 64, "tma ring 24 slots, 1 storer lane");
    run(nm, ctas, [&] { copy_tma<<<ctas, kThreads, smem>>>(src, dst, perm, rows, 24, 1, 1); });
    run("regs unroll 8", ctas, [&] { copy_regs<8><<<ctas, kThreads>>>(src, dst, perm, rows); });
    run("regs unroll 1", ctas, [&] { copy_regs<1><<<ctas, kThreads>>>(src, dst, perm, rows); });
  }
  return 0;
}
