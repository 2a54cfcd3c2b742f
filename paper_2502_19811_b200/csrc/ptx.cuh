// Thin inline-PTX layer for sm_100a: mbarriers, TMA (tile / gather4 /
// 2-SM), tcgen05 (alloc, mma, commit, ld), proxy fences, and the
// acquire/release flag operations used between communication and compute
// CTAs (and across GPUs through NVLink-mapped peer memory).
//
// Written against the PTX ISA 8.6+ forms for sm_100a; the encodings of the
// shared-memory and instruction descriptors follow the tcgen05 "Matrix
// Descriptor" / "Instruction descriptor" tables (bit positions documented
// next to each builder).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

namespace comet {
namespace ptx {

// ---------------------------------------------------------------- basics --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n_threads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n_threads) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------- mbarrier --
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, 0x989680;\n\t"
      "@!P bra WAIT_%=;\n\t}"
      :: "r"(addr), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITS_%=;\n\t}"
      :: "r"(addr), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Arrive on the barrier at the same smem offset in CTA `cta` of the cluster.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  // Plain (default-semantics) remote arrive.  A `.release.cluster` arrive
  // waits for this thread's in-flight TMA loads and serialises the pipeline
  // (measured 4x lower per-SM load rate, tools/tma_bench.cu modes 2 vs 3).
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
}

// Release-ordered remote arrive (orders this thread's prior shared::cluster
// stores, e.g. a broadcast work-unit id, before the phase flip).  Only for
// threads without TMA loads in flight (see mbar_arrive_cluster).
__device__ __forceinline__ void mbar_arrive_release_cluster(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote) : "memory");
}

// Wait with cluster-scope acquire (pairs with mbar_arrive_release_cluster).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1, 0x989680;\n\t"
      "@!P bra WAITC_%=;\n\t}"
      :: "r"(addr), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// 32-bit store into the same smem offset of CTA `cta` of the cluster.
__device__ __forceinline__ void st_shared_cluster(void* local, uint32_t cta, uint32_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(cta));
  asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(remote), "r"(v) : "memory");
}

// Programmatic dependent launch: the next kernel in the stream may start
// (launch_dependents); block until the previous kernel finished and its
// memory is visible (wait).  No-ops for launches without the PDL attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ TMA --
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// Bulk L2 prefetch of `bytes` (multiple of 16, 16 B aligned) at `src`: no
// registers, no smem, no completion -- later plain loads of the range hit L2.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes)
               : "memory");
}

// 2D tile load; completion bytes land on `bar` of this CTA.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)),
         "r"(c0), "r"(c1), "l"(hint) : "memory");
}

// 2-SM variant: issued by both CTAs of a pair; the transaction bytes are
// credited to the barrier of the even (leader) CTA, whose shared::cluster
// address is this CTA's address with the peer bit (bit 24) cleared.
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const void* tmap, uint64_t* bar,
                                                int32_t c0, int32_t c1, uint64_t hint) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_leader),
         "r"(c0), "r"(c1), "l"(hint) : "memory");
}

__device__ __forceinline__ void tma_load_2d_2sm_nohint(void* dst, const void* tmap, uint64_t* bar,
                                                       int32_t c0, int32_t c1) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_leader),
         "r"(c0), "r"(c1) : "memory");
}

// Row gather: four rows (r0..r3) x box-width columns starting at column c0.
// cta_group::2 lets the completion go to the leader CTA's barrier.
__device__ __forceinline__ void tma_gather4_2sm(void* dst, const void* tmap, uint64_t* bar,
                                                int32_t c0, int32_t r0, int32_t r1, int32_t r2,
                                                int32_t r3) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_leader),
         "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

// 1-D bulk copies (global <-> shared), e.g. token rows for dispatch/combine.
// The global side may be an NVLink-mapped peer address.
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :: "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// Warpgroup register reallocation (every thread of the warpgroup executes it)
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(N)); }
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(N)); }

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}

// generic-proxy smem writes -> visible to the async proxy (TMA store source)
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// generic-proxy global writes (e.g. NVLink-pulled rows) -> visible to TMA reads
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Cache hints (createpolicy encodings used by CUTLASS' CacheHintSm90).
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// -------------------------------------------------------------- tcgen05 --
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, M=256 across the CTA pair (leader issues).
__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}

// MMA completion -> arrive on the barrier at this smem offset in every CTA of
// `mask` (both CTAs of the pair).
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      :: "r"(smem_u32(bar)), "h"(mask) : "memory");
}

// 32 lanes x 32-bit, 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major operand, 128-byte swizzle:
//   [0,14)  start address >> 4
//   [16,30) leading byte offset >> 4 (unused for swizzled K-major; 0)
//   [32,46) stride byte offset >> 4 = 1024 B between 8-row groups
//   [46,48) descriptor version = 1 (sm_100)
//   [49,52) base offset = 0 (stage buffers are 1024-byte aligned)
//   [61,64) layout = 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t sdesc_kmajor_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, both K-major.
//   [4,6) D fmt (1=f32)  [7,10) A fmt (1=bf16)  [10,13) B fmt (1=bf16)
//   [15] A major (0=K)   [16] B major (0=K)
//   [17,23) N >> 3       [24,29) M >> 4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ---------------------------------------------------- flags / memory order --
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_acq_rel_gpu_add(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// Flags carry the epoch of the forward that set them; wrap-safe ">=".
__device__ __forceinline__ bool epoch_reached(uint32_t flag, uint32_t epoch) {
  return static_cast<int32_t>(flag - epoch) >= 0;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// 16-byte streaming copies for P2P / HBM row moves.
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
// 32-byte (full L2 sector) streaming store, evict-first: STG.E.EF.ENL2.256.
// Used for the layer outputs so they do not evict the operand tiles that the
// GEMM re-reads from L2.
__device__ __forceinline__ void st_v8_cs(void* p, uint4 lo, uint4 hi) {
  const uint64_t a = (static_cast<uint64_t>(lo.y) << 32) | lo.x, b = (static_cast<uint64_t>(lo.w) << 32) | lo.z;
  const uint64_t c = (static_cast<uint64_t>(hi.y) << 32) | hi.x, d = (static_cast<uint64_t>(hi.w) << 32) | hi.z;
  asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_v8(void* p, uint4 lo, uint4 hi) {
  const uint64_t a = (static_cast<uint64_t>(lo.y) << 32) | lo.x, b = (static_cast<uint64_t>(lo.w) << 32) | lo.z;
  const uint64_t c = (static_cast<uint64_t>(hi.y) << 32) | hi.x, d = (static_cast<uint64_t>(hi.w) << 32) | hi.z;
  asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_v4_cs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Bounded spin for cross-CTA / cross-rank flag waits: sleeps `ns` per poll
// and, if one wait exceeds the timeout (a peer that never signals: a bug
// or a dead rank), prints the site and traps so the launch fails loudly
// instead of hanging the GPU.  The clock is read every 64 polls; the report
// is out of line (no stack or registers in the callers' hot code).
// per translation unit (no relocatable device code); set at context creation
// from COMET_OPT_SPIN_TIMEOUT_MS by each unit's set_spin_timeout_* (default
// 10 min), and the host abort word of comet_abort_waits (mapped pinned
// memory, polled with the clock)
static __device__ unsigned long long g_spin_timeout_ns = 600ull * 1000 * 1000 * 1000;
static __device__ const volatile uint32_t* g_abort_flag = nullptr;
// One out-of-line report per register-budget region (R): a noinline function
// called from regions with different setmaxnreg budgets makes ptxas compile
// every region under the smallest one, so the layer kernel's control warps
// (R = 1) and epilogue warps (R = 2) each get their own copy.
template <int R = 0>
__device__ __noinline__ void spin_timeout(int site, bool aborted) {
  printf("comet: device wait %s (site %d, block %d, thread %d)\n", aborted ? "aborted by the host" : "timed out",
         site, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));
  __trap();
}
template <int R = 0>
struct SpinT {
  unsigned n = 0;
  unsigned long long t0 = 0;
  __device__ __forceinline__ void pause(unsigned ns, int site) {
    __nanosleep(ns);
    if ((++n & 63u) != 0u) return;
    const unsigned long long t = globaltimer();
    if (t0 == 0) {
      t0 = t;
    } else if (t - t0 > g_spin_timeout_ns) {
      spin_timeout<R>(site, false);
    }
    // the host abort word lives in pinned host memory: a PCIe read, so it is
    // polled only by waits that already spun for > 1 ms (a straggling peer),
    // never on the microsecond-scale waits of a healthy forward
    if (t - t0 > 1000000ull && g_abort_flag != nullptr && *g_abort_flag != 0u) spin_timeout<R>(site, true);
  }
};
using Spin = SpinT<0>;
using SpinCtl = SpinT<1>;  // layer kernel control warps (setmaxnreg.dec region)
using SpinEpi = SpinT<2>;  // layer kernel epilogue warps (setmaxnreg.inc region)

}  // namespace ptx
}  // namespace comet
