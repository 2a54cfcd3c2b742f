// Standalone TMA pipeline microbenchmark (diagnostic tool, not product code).
// Streams a [rows, cols] bf16 tensor through a kStages smem ring with the
// same producer / consumer protocol as the fused layer kernel, in variants:
//   mode 0: 1-CTA, consumer releases with mbarrier.arrive
//   mode 1: 1-CTA, consumer releases with tcgen05.commit (no MMA)
//   mode 2: 2-CTA cluster, .cta_group::2 loads credited to the leader, release by
//           tcgen05.commit multicast (the layer kernel's protocol)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

#include "../paper_2502_19811_b200/csrc/ptx.cuh"

using namespace comet;

constexpr int kStages = 6;
constexpr int kBox = 16384;  // 128 rows x 128 B

template <int mode>
__global__ void __launch_bounds__(128, 1) tma_stream(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2, int iters,
                                                     int rows_total, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * 2 * kBox);
  uint64_t* empty = full + kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + kStages);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr bool two = mode >= 2;
  const uint32_t cta = two ? (blockIdx.x & 1) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(full + s, two ? 2 : 1);
      ptx::mbar_init(empty + s, 1);
    }
    ptx::fence_mbar_init();
  }
  if (mode >= 1 && warp == 2) {
    if constexpr (two) ptx::tmem_alloc_2sm(tslot, 32);
    else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(ptx::smem_u32(tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  ptx::tc_fence_before();
  if (two) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const int unit = two ? blockIdx.x / 2 : blockIdx.x;
  const int n_units = two ? gridDim.x / 2 : gridDim.x;
  const long long t0 = clock64();
  if constexpr (mode >= 5) {
    // gather variants: A = 128 gathered rows (32 x gather4), B = one 128-row box
    if (warp != 1) {
      const int wslot = warp == 0 ? 0 : warp - 1;            // 0,1,2 (warps 0,2,3)
      const int n_issuers = mode == 5 ? 1 : 3;
      const bool issuer = (mode == 5 ? warp == 0 : true) && lane == 0;
      int stage = 0; uint32_t phase = 0;
      for (int i = 0; i < iters; ++i) {
        ptx::mbar_wait(empty + stage, phase ^ 1);
        if (issuer) {
          uint8_t* dst = smem + (stage * 2) * kBox;
          for (int g = wslot; g < 32; g += n_issuers) {
            const int r0 = ((unit * 131 + i * 17 + g * 4) * 97) % (rows_total - 4);
            ptx::tma_gather4_2sm(dst + g * 512, &tm2, full + stage, (i % 64) * 64, r0, r0 + 1, r0 + 2, r0 + 3);
          }
          if (warp == 0) {
            const int row = ((unit * 7 + i) * 256 + cta * 128) % (rows_total - 256);
            ptx::tma_load_2d_2sm(dst + kBox, &tm, full + stage, (i % 64) * 64, row, ptx::kEvictNormal);
            if (cta == 0) ptx::mbar_arrive_expect_tx(full + stage, 2 * 2 * kBox);
            else {
              uint32_t remote;
              asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(ptx::smem_u32(full + stage)));
              asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
            }
          }
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  }
  if (mode < 5 && warp == 0 && lane == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      ptx::mbar_wait(empty + stage, phase ^ 1);
      const int row = ((unit * 7 + i) * 256 + cta * 128) % (rows_total - 256);
      for (int b = 0; b < 2; ++b) {
        uint8_t* dst = smem + (stage * 2 + b) * kBox;
        if constexpr (two) ptx::tma_load_2d_2sm(dst, &tm, full + stage, (i % 32) * 64 + b * 64 * 32, row, ptx::kEvictNormal);
        else ptx::tma_load_2d(dst, &tm, full + stage, (i % 32) * 64 + b * 64 * 32, row, ptx::kEvictNormal);
      }
      if (!two || cta == 0) ptx::mbar_arrive_expect_tx(full + stage, (two ? 2 : 1) * 2 * kBox);
      else {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(ptx::smem_u32(full + stage)));
        if constexpr (mode == 2)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
        else if constexpr (mode == 3)
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
        else
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
      }
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1 && lane == 0 && cta == 0) {
    int stage = 0; uint32_t phase = 0;
    for (int i = 0; i < iters; ++i) {
      ptx::mbar_wait(full + stage, phase);
      ptx::tc_fence_after();
      if constexpr (mode == 0) ptx::mbar_arrive(empty + stage);
      else if constexpr (mode == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(ptx::smem_u32(empty + stage)) : "memory");
      else ptx::mma_commit_2sm(empty + stage, 0x3);
      if (++stage == kStages) { stage = 0; phase ^= 1; }
    }
  }
  ptx::tc_fence_before();
  if (two) ptx::cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (mode >= 1 && warp == 2) {
    if constexpr (two) ptx::tmem_dealloc_2sm(0, 32);
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(0));
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int grid = argc > 2 ? atoi(argv[2]) : 148;
  const int iters = 2000;
  const long long rows = 16384, cols = 4096;
  void* buf;
  cudaMalloc(&buf, rows * cols * 2);
  cudaMemset(buf, 0, rows * cols * 2);
  unsigned long long* out;
  cudaMalloc(&out, sizeof(unsigned long long) * grid);
  PFN_cuTensorMapEncodeTiled_v12000 fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap tm2;
  cuuint32_t box2[2] = {64, 1};
  fn(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = kStages * 2 * kBox + 2048;
  auto kern = mode == 0 ? tma_stream<0> : mode == 1 ? tma_stream<1> : mode == 2 ? tma_stream<2> : mode == 3 ? tma_stream<3> : mode == 4 ? tma_stream<4> : mode == 5 ? tma_stream<5> : tma_stream<6>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(128);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = mode >= 2 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaError_t le = cudaLaunchKernelEx(&lc, kern, tm, tm2, iters, (int)rows, out);
    if (le != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(le));
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * iters * 2 * kBox;
    printf("mode %d grid %d: %.3f ms  %.1f GB/s total  %.1f GB/s per CTA  (%s)\n", mode, grid, ms, bytes / ms / 1e6,
           bytes / ms / 1e6 / grid, cudaGetErrorString(e));
  }
  return 0;
}
