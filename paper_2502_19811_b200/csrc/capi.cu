// C ABI (include/comet_b200.h): context, symmetric heap, launchers.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comet_b200.h"
#include "index.cuh"
#include "layers.cuh"

namespace comet {
__global__ void index_build_kernel(IndexDev ix);
__global__ void moe_layer_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_b0,
                                 const __grid_constant__ CUtensorMap tm_a1, const __grid_constant__ CUtensorMap tm_b1,
                                 const __grid_constant__ CUtensorMap tm_s0, const __grid_constant__ CUtensorMap tm_s1,
                                 const __grid_constant__ KernelArgs f);
__global__ void combine_finish_kernel(const LayerArgs p, const __nv_bfloat16* cb, const uint32_t* cb_flag,
                                      const int32_t* experts);
__global__ void signal_x_ready_kernel(uint32_t* const* x_ready_peer, int rank, int world, uint32_t epoch);
cudaError_t router_topk_launch(const void* logits, int logits_dtype, int M, int E, int topk, int norm,
                               int32_t* experts, float* weights, int n_sm, cudaStream_t stream);
__global__ void dispatch_local_kernel(const int32_t* gather_row, const int32_t* meta, const __nv_bfloat16* xs,
                                      __nv_bfloat16* xg, int n_embed, int M, int world, int rank);
__global__ void combine_local_kernel(const int32_t* tok_pos, const float* combine_w, const __nv_bfloat16* yrows,
                                     __nv_bfloat16* y, int t0, int n_tok, int topk, int n_embed);
}  // namespace comet
cudaError_t set_spin_timeout_index(unsigned long long ns);
cudaError_t set_spin_timeout_layers(unsigned long long ns);

using namespace comet;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(COMET_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                   \
  } while (0)

constexpr int kLayerThreads = 384;  // moe_layers.cu kThreads: 4 control + 8 epilogue warps
constexpr int kMaxStreamChunks = 64;  // token chunks of the host-streamed forward
constexpr size_t kLayerSmem = kLayerStages * 49152 + 32768 + 1024 + 1024;
constexpr int kIndexThreads = 1024;
constexpr size_t kIndexSmem = 8192 * sizeof(long long);

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Option defaults (comet_b200.h COMET_OPT_*), all measured (DESIGN.md §4/§6).
// PDL default 14: with bit 1 the host-pipeline test (forward_host, uneven
// token chunks) read a previous chunk's index in dispatch_local -- kept off.
#ifndef COMET_DEFAULT_SPIN_MS
#define COMET_DEFAULT_SPIN_MS 600000  // developer builds may shorten it (-DCOMET_DEFAULT_SPIN_MS=10000)
#endif
constexpr int kOptDefaults[COMET_OPT_COUNT] = {
    /*FUSED*/ 1, /*KSPLIT_MAX*/ 8, /*SPLIT_TAIL0*/ 1, /*SPLIT1*/ -1, /*DEDUP*/ -1, /*PULL_LOCAL*/ 1,
    /*FOLD_ORDER*/ 0, /*GROUP1*/ 0, /*CHUNK_ROWS*/ 0, /*PDL*/ 14, /*GRID*/ 0, /*FUSE1*/ 0,
    /*SPIN_TIMEOUT_MS*/ COMET_DEFAULT_SPIN_MS, /*ZC_DEDUP*/ 1, /*ZC_INTERLEAVE*/ 1, /*ZC_DOWNLOAD*/ 8, /*ZC_ORDER*/ 0,
    /*ZC_FOLD_ORDER*/ 0, /*STREAM_FUSE*/ 0, /*SEQUENTIAL*/ 0, /*STREAMK*/ 0, /*FOLD_STRIDE*/ 0};

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous one drains; it calls griddepcontrol.wait before touching
// the previous kernel's results.  `pdl` is the context's PDL bitmask
// (COMET_OPT_PDL): 1 dispatch_local, 2 layer kernel, 4 combine kernels, 8 index build.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(int pdl, int bit, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = (pdl & bit) ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kernel, std::forward<Args>(args)...);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D bf16 row-major [rows, cols] map, 128-byte swizzle, box {64, box_rows}.
int make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(COMET_ECUDA, "cuTensorMapEncodeTiled unavailable");
  if ((cols * 2) % 16 != 0) return fail(COMET_EINVAL, "row pitch %llu B not 16-byte aligned", (unsigned long long)(cols * 2));
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(COMET_ECUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r,
                                     (unsigned long long)rows, (unsigned long long)cols);
  return COMET_OK;
}

struct MapCache {
  const void* ptr = nullptr;
  uint64_t rows = 0, cols = 0;
  CUtensorMap map;
};

}  // namespace

struct comet_ctx {
  comet_config cfg;
  int opt[COMET_OPT_COUNT];  // COMET_OPT_* values (kOptDefaults until set)
  int e_lo = 0, E_r = 0, k_local = 0, n_sm = 0, max_clusters = 0;
  int nb0 = 0, nb1 = 0, kb0 = 0, kb1 = 0;
  uint32_t epoch = 0;
  int M = 0;  // tokens of the current forward

  // index
  IndexDev ix{};
  void* index_mem = nullptr;
  size_t index_bytes = 0;
  int cap_rows = 0, cap_rows_pad = 0, cap_tiles0 = 0, cap_tiles1 = 0, cap_pairs = 0;
  int32_t* tiles_mem = nullptr;  // tiles0 + tiles1 + chunks (re-sized by tile knobs)
  int cap_chunks = 0;

  // symmetric region
  void* symm = nullptr;
  size_t symm_bytes = 0;
  __nv_bfloat16* xs = nullptr;
  uint32_t* tok_ready = nullptr;
  uint32_t* x_ready = nullptr;
  __nv_bfloat16* cb = nullptr;
  uint32_t* cb_flag = nullptr;
  int mloc_cap = 0;
  std::vector<void*> opened;  // IPC-mapped peer bases

  // device peer tables: [xs_peer | cb_peer | cb_flag_peer | x_ready_peer] x world
  void** peer_tab = nullptr;

  // work buffers
  __nv_bfloat16* H = nullptr;
  __nv_bfloat16* yrows = nullptr;
  __nv_bfloat16* xg = nullptr;      // dispatched (expert-sorted) layer0 rows
  uint32_t* xg_ready = nullptr;     // per 128-row tile epoch
  uint32_t* counters = nullptr;   // nb_done[nb1] | nb_sent[nb1]
  uint32_t* tile_done = nullptr;  // [Rpad/128 + 1][nb1] fused-combine tile epochs
  int32_t* routing = nullptr;

  CUtensorMap tm_xs, tm_H, tm_y, tm_xg;
  CUtensorMap tm_Hs, tm_ys;  // epilogue TMA stores: box {64 cols, 32 rows} (one epilogue warp's block)
  unsigned long long* timeline = nullptr;
  int timeline_cap = 0;
  void* last_y = nullptr;
  const float* last_combine_w = nullptr;
  MapCache w0c, w1c;
  uint32_t* sched = nullptr;  // [2] unit claim / CTA exit counters of the layer kernel (self-resetting)
  uint32_t* h_cnt = nullptr;  // [(cap_rows_pad / 128 + 1) * nb0] fused-launch H half counts (self-resetting)
  // host-streamed forward: upload / download streams, per-chunk upload epochs
  cudaStream_t up_stream = nullptr, down_stream = nullptr;
  cudaEvent_t ev_start = nullptr, ev_index = nullptr, ev_down = nullptr;
  uint32_t* chunk_ready = nullptr;
  float* cw_dev = nullptr;                 // uploaded combine weights
  __nv_bfloat16* y_stream = nullptr;       // [m_cap, N] output of the streamed forward
  float* part = nullptr;       // split-K partials: 2 layers x (pairs x 2 CTA tiles) x 128 x 512 fp32
  uint32_t* split_cnt = nullptr;  // 2 layers x 1024 slice counters: [tile] arrived / finished, [256 + tile]
                                  // landed, [512 + 2 tile + half] finished chunks (reset by their last user)
  int n_h = 0;
  // layer-kernel launch timing (comet_kernel_timing_*): an event pair around
  // each moe_layer_kernel launch, on the launch stream, in a ring of slots
  std::vector<cudaEvent_t> kt_ev;
  int kt_slots = 0, kt_next = 0;
};

cudaError_t set_abort_flag_index(const volatile uint32_t* p);
cudaError_t set_abort_flag_layers(const volatile uint32_t* p);

namespace {

uint32_t* g_abort_host = nullptr;  // pinned, mapped (comet_abort_waits)

// Device flag-wait timeout of this context's device (ptx::Spin; both
// translation units hold their own copy of the timeout and abort pointer).
int apply_spin_timeout(comet_ctx* x) {
  const unsigned long long ms = static_cast<unsigned long long>(std::max(1, x->opt[COMET_OPT_SPIN_TIMEOUT_MS]));
  CK(cudaSetDevice(x->cfg.device));
  CK(set_spin_timeout_index(ms * 1000000ull));
  CK(set_spin_timeout_layers(ms * 1000000ull));
  // process-wide host abort word (comet_abort_waits), mapped into every device
  if (!g_abort_host) {
    CK(cudaHostAlloc(&g_abort_host, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    *g_abort_host = 0;
  }
  uint32_t* dev = nullptr;
  CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), g_abort_host, 0));
  CK(set_abort_flag_index(dev));
  CK(set_abort_flag_layers(dev));
  return COMET_OK;
}

// DEDUP -1 (automatic): off -- measured slower in single-GPU emulation for
// every BASELINE shape; 1 forces it on.
bool dedup_on(const comet_ctx* x) { return x->opt[COMET_OPT_DEDUP] > 0; }

int group1(const comet_ctx* x, int group0) { return x->opt[COMET_OPT_GROUP1] > 0 ? x->opt[COMET_OPT_GROUP1] : group0; }

}  // namespace

extern "C" {

int comet_set_option(comet_ctx* x, int opt, int value) {
  if (!x) return fail(COMET_EINVAL, "null context");
  if (opt < 0 || opt >= COMET_OPT_COUNT) return fail(COMET_EINVAL, "unknown option %d", opt);
  if (value == COMET_OPT_DEFAULT) value = kOptDefaults[opt];
  if (opt == COMET_OPT_CHUNK_ROWS && (value < 0 || value > 32))
    return fail(COMET_EINVAL, "CHUNK_ROWS must be 0 (auto) or in [1, 32], got %d", value);
  if (opt == COMET_OPT_FOLD_STRIDE && (value < 0 || value == 1 || value > 8))
    return fail(COMET_EINVAL, "FOLD_STRIDE must be 0 or in [2, 8], got %d", value);
  if (opt == COMET_OPT_KSPLIT_MAX && (value < 0 || value > 8))
    return fail(COMET_EINVAL, "KSPLIT_MAX must be in [0, 8], got %d", value);
  if (opt == COMET_OPT_GRID && (value < 0 || value == 1 || (value & 1)))
    return fail(COMET_EINVAL, "GRID must be 0 or an even CTA count >= 2, got %d", value);
  if (opt == COMET_OPT_SPIN_TIMEOUT_MS && value < 1)
    return fail(COMET_EINVAL, "SPIN_TIMEOUT_MS must be >= 1, got %d", value);
  const int old = x->opt[opt];
  x->opt[opt] = value;
  if (opt == COMET_OPT_SPIN_TIMEOUT_MS && old != value) return apply_spin_timeout(x);
  return COMET_OK;
}

int comet_get_option(comet_ctx* x, int opt, int* value) {
  if (!x || !value) return fail(COMET_EINVAL, "null argument");
  if (opt < 0 || opt >= COMET_OPT_COUNT) return fail(COMET_EINVAL, "unknown option %d", opt);
  *value = x->opt[opt];
  return COMET_OK;
}

int comet_abort_waits(int value) {
  if (!g_abort_host) return fail(COMET_EINVAL, "no context created yet");
  *reinterpret_cast<volatile uint32_t*>(g_abort_host) = static_cast<uint32_t>(value);
  return COMET_OK;
}

const char* comet_last_error(void) { return g_err.c_str(); }
int comet_version(void) { return 1; }

int comet_device_info(int device, int32_t out[4]) {
  CK(cudaSetDevice(device));
  int n_sm = 0, major = 0, minor = 0;
  CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  CK(cudaFuncSetAttribute(moe_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLayerSmem));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(n_sm);
  lc.blockDim = dim3(kLayerThreads);
  lc.dynamicSmemBytes = kLayerSmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int clusters = 0;
  CK(cudaOccupancyMaxActiveClusters(&clusters, moe_layer_kernel, &lc));
  out[0] = n_sm;
  out[1] = clusters;
  out[2] = major * 10 + minor;
  out[3] = (int)kLayerSmem;
  return COMET_OK;
}

int comet_router_topk(const void* d_logits, int logits_dtype, int M, int E, int topk, int norm,
                      int32_t* d_experts, float* d_weights, void* stream) {
  if (M < 0 || E < 1 || E > 512) return fail(COMET_EINVAL, "router: need M >= 0 and 1 <= E <= 512 (M=%d, E=%d)", M, E);
  if (topk < 1 || topk > E || topk > 32)
    return fail(COMET_EINVAL, "router: topk=%d must be in [1, min(E=%d, 32)]", topk, E);
  if (logits_dtype != 0 && logits_dtype != 1) return fail(COMET_EINVAL, "router: logits_dtype %d (0 fp32, 1 bf16)", logits_dtype);
  if (norm < 0 || norm > 2) return fail(COMET_EINVAL, "router: norm %d (0 none, 1 top-k softmax, 2 full softmax)", norm);
  if (M > 0 && norm != 0 && d_weights == nullptr) return fail(COMET_EINVAL, "router: norm %d needs a weights buffer", norm);
  if (M > 0 && (d_logits == nullptr || d_experts == nullptr)) return fail(COMET_EINVAL, "router: null buffer");
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  }
  CK(router_topk_launch(d_logits, logits_dtype, M, E, topk, norm, d_experts, norm ? d_weights : nullptr, n_sm,
                        static_cast<cudaStream_t>(stream)));
  return COMET_OK;
}

int comet_ctx_create(const comet_config* cfg, comet_ctx** out) {
  const comet_config& c = *cfg;
  if (c.world != c.tp * c.ep || c.world < 1 || c.world > kMaxWorld)
    return fail(COMET_EINVAL, "world=%d must equal tp*ep=%d and be in [1, %d]", c.world, c.tp * c.ep, kMaxWorld);
  if (c.rank < 0 || c.rank >= c.world) return fail(COMET_EINVAL, "rank %d out of range", c.rank);
  if (c.E % c.ep) return fail(COMET_EINVAL, "E=%d is not divisible by ep=%d", c.E, c.ep);
  if (c.K % c.tp) return fail(COMET_EINVAL, "K=%d is not divisible by tp=%d", c.K, c.tp);
  if (c.E > 1024) return fail(COMET_EINVAL, "E=%d > 1024 unsupported", c.E);
  if (c.topk < 1 || c.topk > c.E) return fail(COMET_EINVAL, "bad topk %d", c.topk);
  if (c.m_cap < 1 || c.m_cap > 65536) return fail(COMET_EINVAL, "m_cap must be in [1, 65536]");

  comet_ctx* x = new comet_ctx();
  x->cfg = c;
  CK(cudaSetDevice(c.device));
  std::copy(kOptDefaults, kOptDefaults + COMET_OPT_COUNT, x->opt);
  if (int rc = apply_spin_timeout(x)) { delete x; return rc; }
  // per device: the dynamic shared-memory opt-in of the index kernel
  CK(cudaFuncSetAttribute(index_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kIndexSmem));
  int32_t info[4];
  if (int rc = comet_device_info(c.device, info)) { delete x; return rc; }
  x->n_sm = info[0];
  x->max_clusters = info[1];
  x->E_r = c.E / c.ep;
  x->e_lo = (c.rank / c.tp) * x->E_r;
  x->k_local = c.K / c.tp;
  x->nb0 = (x->k_local + kBlockN - 1) / kBlockN;
  x->nb1 = (c.N + kBlockN - 1) / kBlockN;
  x->kb0 = c.N / 64;
  x->kb1 = x->k_local / 64;

  // ---- index arrays ----
  const long long rows = (long long)c.m_cap * std::min(c.topk, x->E_r);
  x->cap_rows = (int)rows;
  x->cap_rows_pad = (int)align_up(rows + (long long)x->E_r * (kPairRows - 1), kPairRows);
  x->cap_pairs = x->cap_rows_pad / kPairRows;
  const int W = c.world;
  struct Part { int32_t** dst; size_t n; };
  IndexDev& ix = x->ix;
  std::vector<Part> parts = {
      {&ix.counts, (size_t)c.E},
      {&ix.transfer, (size_t)W * W},
      {&ix.row_off, (size_t)x->E_r + 1},
      {&ix.pad_off, (size_t)x->E_r + 1},
      {&ix.n_local, (size_t)x->E_r},
      {&ix.row_token, (size_t)x->cap_rows},
      {&ix.row_src, (size_t)x->cap_rows},
      {&ix.gather_row, (size_t)x->cap_rows_pad},
      {&ix.tok_pos, (size_t)c.m_cap * c.topk},
      {&ix.pairs0, (size_t)x->cap_pairs * 4},
      {&ix.pairs1, (size_t)x->cap_pairs * 4},
      {&ix.claim_of_tile, (size_t)x->cap_rows_pad / kTileRows + 1},
      {&ix.pull_token, (size_t)c.m_cap},
      {&ix.pull_src, (size_t)c.m_cap},
      {&ix.combine_tok, (size_t)c.m_cap},
      {&ix.row_dst, (size_t)x->cap_rows_pad},
      {&ix.row_widx, (size_t)x->cap_rows_pad},
      {&ix.meta, (size_t)kMetaSlots},
      {&ix.chunk_cnt, (size_t)x->E_r * kIndexMaxChunks},
      {&ix.chunk_loc, (size_t)x->E_r * kIndexMaxChunks},
      {reinterpret_cast<int32_t**>(&ix.chunk_flag), (size_t)x->E_r * kIndexMaxChunks},
      {&ix.pair_key, (size_t)x->cap_pairs},
      {reinterpret_cast<int32_t**>(&ix.fold_part), (size_t)2 * 160 * std::min(x->E_r, 64)},
  };
  size_t total = 0;
  for (auto& p : parts) total += align_up(p.n * 4, 256);
  total += 256;  // done counter
  CK(cudaMalloc(&x->index_mem, total));
  CK(cudaMemset(x->index_mem, 0, total));
  x->index_bytes = total;
  {
    char* b = static_cast<char*>(x->index_mem);
    for (auto& p : parts) {
      *p.dst = reinterpret_cast<int32_t*>(b);
      b += align_up(p.n * 4, 256);
    }
    ix.done = reinterpret_cast<uint32_t*>(b);
    ix.p1_done = reinterpret_cast<uint32_t*>(b + 128);
  }
  ix.cap_rows = x->cap_rows;
  ix.cap_rows_pad = x->cap_rows_pad;
  ix.cap_pairs = x->cap_pairs;

  // ---- symmetric region ----
  x->mloc_cap = c.m_cap / W + W;
  ix.mloc_cap = x->mloc_cap;
  const size_t xs_b = align_up((size_t)c.m_cap * c.N * 2, 4096);
  const size_t tr_b = align_up((size_t)c.m_cap * 4, 4096);
  const size_t xr_b = 4096;
  const size_t cb_b = align_up((size_t)W * x->mloc_cap * c.N * 2, 4096);
  const size_t cf_b = align_up((size_t)W * x->nb1 * 4, 4096);
  x->symm_bytes = xs_b + tr_b + xr_b + cb_b + cf_b;
  CK(cudaMalloc(&x->symm, x->symm_bytes));
  CK(cudaMemset(x->symm, 0, x->symm_bytes));
  {
    char* b = static_cast<char*>(x->symm);
    x->xs = reinterpret_cast<__nv_bfloat16*>(b);
    b += xs_b;
    x->tok_ready = reinterpret_cast<uint32_t*>(b);
    b += tr_b;
    x->x_ready = reinterpret_cast<uint32_t*>(b);
    b += xr_b;
    x->cb = reinterpret_cast<__nv_bfloat16*>(b);
    b += cb_b;
    x->cb_flag = reinterpret_cast<uint32_t*>(b);
  }
  CK(cudaMalloc(&x->peer_tab, sizeof(void*) * 4 * W));
  x->opened.assign(W, nullptr);

  // ---- counters (work buffers H / yrows are allocated on the first layer call) ----
  // layer1 per-n-block counters + streamed-forward output chunk counters,
  // all zeroed by every index build
  CK(cudaMalloc(&x->counters, sizeof(uint32_t) * (2 * x->nb1 + kMaxStreamChunks)));
  CK(cudaMemset(x->counters, 0, sizeof(uint32_t) * (2 * x->nb1 + kMaxStreamChunks)));
  CK(cudaMalloc(&x->routing, sizeof(int32_t) * (size_t)c.m_cap * c.topk));
  ix.zero_words = x->counters;
  ix.n_zero_words = 2 * x->nb1 + kMaxStreamChunks;

  if (W == 1) {
    comet_ctx* self = x;
    if (int r2 = comet_link_local(&self, 1)) { comet_ctx_destroy(x); return r2; }
  }
  *out = x;
  return COMET_OK;
}

int comet_ctx_destroy(comet_ctx* x) {
  if (!x) return COMET_OK;
  cudaSetDevice(x->cfg.device);
  for (void* p : x->opened)
    if (p) cudaIpcCloseMemHandle(p);
  cudaFree(x->index_mem);
  cudaFree(x->tiles_mem);
  cudaFree(x->symm);
  cudaFree(x->peer_tab);
  cudaFree(x->H);
  cudaFree(x->yrows);
  cudaFree(x->xg);
  cudaFree(x->xg_ready);
  cudaFree(x->tile_done);
  cudaFree(x->sched);
  cudaFree(x->h_cnt);
  cudaFree(x->chunk_ready);
  cudaFree(x->cw_dev);
  cudaFree(x->y_stream);
  if (x->up_stream) cudaStreamDestroy(x->up_stream);
  if (x->down_stream) cudaStreamDestroy(x->down_stream);
  if (x->ev_start) cudaEventDestroy(x->ev_start);
  if (x->ev_index) cudaEventDestroy(x->ev_index);
  if (x->ev_down) cudaEventDestroy(x->ev_down);
  for (cudaEvent_t e : x->kt_ev) cudaEventDestroy(e);
  cudaFree(x->part);
  cudaFree(x->split_cnt);
  cudaFree(x->timeline);
  cudaFree(x->counters);
  cudaFree(x->routing);
  delete x;
  return COMET_OK;
}

static int upload_peer_table(comet_ctx* x, const std::vector<char*>& bases) {
  const int W = x->cfg.world;
  std::vector<void*> tab(4 * W);
  const size_t off_tr = reinterpret_cast<char*>(x->tok_ready) - static_cast<char*>(x->symm);
  (void)off_tr;
  const size_t off_xr = reinterpret_cast<char*>(x->x_ready) - static_cast<char*>(x->symm);
  const size_t off_cb = reinterpret_cast<char*>(x->cb) - static_cast<char*>(x->symm);
  const size_t off_cf = reinterpret_cast<char*>(x->cb_flag) - static_cast<char*>(x->symm);
  for (int r = 0; r < W; ++r) {
    tab[r] = bases[r];
    tab[W + r] = bases[r] + off_cb;
    tab[2 * W + r] = bases[r] + off_cf;
    tab[3 * W + r] = bases[r] + off_xr;
  }
  CK(cudaSetDevice(x->cfg.device));
  CK(cudaMemcpy(x->peer_tab, tab.data(), sizeof(void*) * 4 * W, cudaMemcpyHostToDevice));
  return COMET_OK;
}

int comet_symm_export(comet_ctx* x, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  CK(cudaSetDevice(x->cfg.device));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, x->symm));
  memcpy(handle64, &h, 64);
  return COMET_OK;
}

int comet_symm_import(comet_ctx* x, const void* handles) {
  const int W = x->cfg.world;
  CK(cudaSetDevice(x->cfg.device));
  std::vector<char*> bases(W);
  for (int r = 0; r < W; ++r) {
    if (r == x->cfg.rank) {
      bases[r] = static_cast<char*>(x->symm);
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + 64 * r, 64);
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    x->opened[r] = p;
    bases[r] = static_cast<char*>(p);
  }
  return upload_peer_table(x, bases);
}

int comet_link_local(comet_ctx** ctxs, int n) {
  for (int i = 0; i < n; ++i) {
    comet_ctx* x = ctxs[i];
    if (x->cfg.world != n || x->cfg.rank != i)
      return fail(COMET_EINVAL, "link_local: ctx %d has rank %d world %d", i, x->cfg.rank, x->cfg.world);
    if (ctxs[0]->symm_bytes != x->symm_bytes) return fail(COMET_EINVAL, "link_local: asymmetric heaps");
  }
  std::vector<char*> bases(n);
  for (int i = 0; i < n; ++i) bases[i] = static_cast<char*>(ctxs[i]->symm);
  for (int i = 0; i < n; ++i) {
    // peer access between devices when the group spans several GPUs
    for (int j = 0; j < n; ++j) {
      if (ctxs[j]->cfg.device != ctxs[i]->cfg.device) {
        cudaSetDevice(ctxs[i]->cfg.device);
        cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[j]->cfg.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(COMET_ECUDA, "peer access %d->%d: %s", ctxs[i]->cfg.device, ctxs[j]->cfg.device,
                      cudaGetErrorString(e));
        cudaGetLastError();
      }
    }
    if (int rc = upload_peer_table(ctxs[i], bases)) return rc;
  }
  return COMET_OK;
}

void* comet_token_buffer(comet_ctx* x) { return x->xs; }
void* comet_routing_buffer(comet_ctx* x) { return x->routing; }
void* comet_hidden_buffer(comet_ctx* x) { return x->H; }
void* comet_yrows_buffer(comet_ctx* x) { return x->yrows; }
int32_t comet_hidden_rows_cap(comet_ctx* x) { return x->cap_rows_pad; }

static int ensure_tiles(comet_ctx* x, int tile_rows, int tile_cols) {
  const auto& c = x->cfg;
  const long long t0 = (long long)x->cap_rows / tile_rows + x->E_r + 1;
  const long long ch = (c.N + tile_cols - 1) / tile_cols;
  const long long t1 = t0 * ch;
  if (t0 <= x->cap_tiles0 && t1 <= x->cap_tiles1 && ch <= x->cap_chunks && x->tiles_mem) return COMET_OK;
  if (t1 > (1ll << 28)) return fail(COMET_EINVAL, "tile list too large (tile_rows=%d tile_cols=%d)", tile_rows, tile_cols);
  cudaFree(x->tiles_mem);
  x->tiles_mem = nullptr;
  const size_t n = align_up(t0 * 4, 64) + align_up(t1 * 6, 64) + align_up(ch * 4, 64);
  CK(cudaMalloc(&x->tiles_mem, n * 4));
  x->cap_tiles0 = (int)t0;
  x->cap_tiles1 = (int)t1;
  x->cap_chunks = (int)ch;
  x->ix.tiles0 = x->tiles_mem;
  x->ix.tiles1 = x->tiles_mem + align_up(t0 * 4, 64);
  x->ix.chunks = x->ix.tiles1 + align_up(t1 * 6, 64);
  x->ix.cap_tiles0 = (int)t0;
  x->ix.cap_tiles1 = (int)t1;
  return COMET_OK;
}

int comet_index_build_ex(comet_ctx* x, const int32_t* d_experts, int M, int tile_rows, int tile_cols, int flags,
                         void* stream);

int comet_index_build(comet_ctx* x, const int32_t* d_experts, int M, int tile_rows, int tile_cols, void* stream) {
  return comet_index_build_ex(x, d_experts, M, tile_rows, tile_cols, kIndexRefLists | kIndexCombineList, stream);
}

// Layer1 pair-order bit of comet_forward's index build: world > 1 with fold
// chains (several hosted experts per token) orders the layer1 pairs by fold
// level when COMET_OPT_FOLD_ORDER is set.
static int forward_order_flags(const comet_ctx* x) {
  const bool fold_order = x->cfg.world > 1 && x->E_r > 1 && x->E_r <= 64 && x->cfg.topk > 1 &&
                          x->opt[COMET_OPT_FOLD_ORDER] != 0;
  return fold_order ? kIndexFoldOrder : 0;
}

int comet_index_build_ex(comet_ctx* x, const int32_t* d_experts, int M, int tile_rows, int tile_cols, int flags,
                         void* stream) {
  const auto& c = x->cfg;
  if (flags & kIndexForwardOrder) flags = (flags & ~kIndexForwardOrder) | forward_order_flags(x);
  if (M < 0 || M > c.m_cap) return fail(COMET_EINVAL, "M=%d outside [0, m_cap=%d]", M, c.m_cap);
  if (tile_rows < 1) return fail(COMET_EINVAL, "tile_rows must be >= 1, got %d", tile_rows);
  if (tile_cols < 1 || tile_cols > c.N) return fail(COMET_EINVAL, "tile_cols must be in [1, %d], got %d", c.N, tile_cols);
  if (c.world * c.world > 4096) return fail(COMET_EINVAL, "world too large");
  if (int rc = ensure_tiles(x, tile_rows, tile_cols)) return rc;
  CK(cudaSetDevice(c.device));
  x->M = M;
  x->epoch += 1;
  IndexDev ix = x->ix;
  ix.experts = d_experts;
  ix.M = M;
  ix.E = c.E;
  ix.topk = c.topk;
  ix.tp = c.tp;
  ix.ep = c.ep;
  ix.rank = c.rank;
  ix.world = c.world;
  ix.e_lo = x->e_lo;
  ix.E_r = x->E_r;
  ix.tile_rows = tile_rows;
  ix.tile_cols = tile_cols;
  ix.n_embed = c.N;
  ix.flags = flags;
  ix.epoch = x->epoch;
  ix.x_ready_peer = reinterpret_cast<uint32_t* const*>(x->peer_tab + 3 * c.world);
  ix.tpt = std::max(1, (M + 16 * kIndexThreads - 1) / (16 * kIndexThreads));
  const int chunks = (M + kIndexThreads * ix.tpt - 1) / (kIndexThreads * ix.tpt);
  if (chunks > kIndexMaxChunks) return fail(COMET_EINVAL, "M=%d too large for the index build", M);
  // item CTAs [0, grid - 1) + the table CTA (grid - 1, no items)
  const int grid = std::min(x->n_sm, std::max(32, x->E_r * chunks + 1));
  // global histogram + transfer matrix accumulate by atomics: zero both (adjacent)
  const size_t zbytes = reinterpret_cast<char*>(x->ix.transfer + c.world * c.world) - reinterpret_cast<char*>(x->ix.counts);
  if (flags & kIndexRefLists) CK(cudaMemsetAsync(x->ix.counts, 0, zbytes, static_cast<cudaStream_t>(stream)));
  CK(launch_pdl(x->opt[COMET_OPT_PDL], 8, index_build_kernel, dim3(grid), dim3(kIndexThreads), kIndexSmem,
                static_cast<cudaStream_t>(stream), ix));
  CK(cudaGetLastError());
  x->ix.experts = d_experts;  // the layer1 finish kernel reads the global routing
  return COMET_OK;
}

int comet_index_sizes(comet_ctx* x, int32_t meta_out[16], void* stream) {
  CK(cudaSetDevice(x->cfg.device));
  CK(cudaMemcpyAsync(meta_out, x->ix.meta, 16 * 4, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  if (meta_out[kMetaSlots - 1]) return fail(COMET_ECAP, "index capacity exceeded (flags %d)", meta_out[kMetaSlots - 1]);
  return COMET_OK;
}

int comet_index_download(comet_ctx* x, comet_index_host* h, void* stream) {
  if (int rc = comet_index_sizes(x, h->meta, stream)) return rc;
  const auto& c = x->cfg;
  const int32_t* m = h->meta;
  auto cp = [&](int32_t* dst, const int32_t* src, size_t n) -> int {
    if (dst && n) CK(cudaMemcpy(dst, src, n * 4, cudaMemcpyDeviceToHost));
    return COMET_OK;
  };
  int rc = 0;
  rc |= cp(h->counts, x->ix.counts, c.E);
  rc |= cp(h->transfer, x->ix.transfer, (size_t)c.world * c.world);
  rc |= cp(h->row_off, x->ix.row_off, x->E_r + 1);
  rc |= cp(h->n_local, x->ix.n_local, x->E_r);
  rc |= cp(h->row_token, x->ix.row_token, m[kMetaRows]);
  rc |= cp(h->row_src, x->ix.row_src, m[kMetaRows]);
  rc |= cp(h->tiles0, x->ix.tiles0, (size_t)m[kMetaTiles0] * 4);
  rc |= cp(h->tiles1, x->ix.tiles1, (size_t)m[kMetaTiles1] * 6);
  rc |= cp(h->chunks, x->ix.chunks, (size_t)m[kMetaChunks] * 4);
  rc |= cp(h->pairs0, x->ix.pairs0, (size_t)m[kMetaPairs] * 4);
  rc |= cp(h->pull_token, x->ix.pull_token, m[kMetaPull]);
  rc |= cp(h->pull_src, x->ix.pull_src, m[kMetaPull]);
  return rc ? COMET_ECUDA : COMET_OK;
}

int comet_signal_tokens_ready(comet_ctx* x, void* stream) {
  CK(cudaSetDevice(x->cfg.device));
  const int W = x->cfg.world;
  signal_x_ready_kernel<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint32_t* const*>(x->peer_tab + 3 * W), x->cfg.rank, W, x->epoch);
  CK(cudaGetLastError());
  return COMET_OK;
}

// Layer work buffers + their TMA maps, allocated once on first use (an
// index-only context -- resolver API -- never pays for them).
static int ensure_work(comet_ctx* x) {
  if (x->H) return COMET_OK;
  const auto& c = x->cfg;
  if (c.N * 2 > 20480) return fail(COMET_EINVAL, "N=%d too large for the dispatch ring (N <= 10240)", c.N);
  if (c.topk > 8) return fail(COMET_EINVAL, "topk=%d > 8 unsupported by the combine engine", c.topk);
  if (c.N % 64 || x->k_local % 64)
    return fail(COMET_EINVAL, "N=%d and K/tp=%d must be multiples of 64 for the GPU layer (pad on the host)", c.N,
                x->k_local);
  CK(cudaSetDevice(c.device));
  CK(cudaMalloc(&x->H, (size_t)x->cap_rows_pad * x->k_local * 2));
  CK(cudaMalloc(&x->yrows, (size_t)x->cap_rows_pad * c.N * 2));
  CK(cudaMalloc(&x->xg, (size_t)x->cap_rows_pad * c.N * 2));
  CK(cudaMalloc(&x->xg_ready, 2 * sizeof(uint32_t) * (x->cap_rows_pad / kTileRows + 1)));
  CK(cudaMemset(x->xg_ready, 0, 2 * sizeof(uint32_t) * (x->cap_rows_pad / kTileRows + 1)));
  const size_t td = sizeof(uint32_t) * (x->cap_rows_pad / kTileRows + 1) * x->nb1 * 2;
  CK(cudaMalloc(&x->tile_done, td));
  CK(cudaMemset(x->tile_done, 0, td));
  x->n_h = (x->cap_rows_pad / kTileRows + 1) * x->nb0;  // per (128-row H tile, layer0 n-block)
  CK(cudaMalloc(&x->sched, sizeof(uint32_t) * 2));
  CK(cudaMemset(x->sched, 0, sizeof(uint32_t) * 2));
  CK(cudaMalloc(&x->h_cnt, sizeof(uint32_t) * x->n_h));
  CK(cudaMemset(x->h_cnt, 0, sizeof(uint32_t) * x->n_h));
  // split-K only runs when a layer's output tiles x slices <= pairs: each
  // layer needs at most (grid/2 pairs) x 2 CTA tiles of 128 x 512 fp32;
  // layer1 also holds the stream-K tail's partials: two per range, ranges <= pairs
  CK(cudaMalloc(&x->part, (size_t)3 * x->n_sm * kTileRows * kBlockN * sizeof(float)));
  CK(cudaMalloc(&x->split_cnt, sizeof(uint32_t) * 2 * 1024));
  CK(cudaMemset(x->split_cnt, 0, sizeof(uint32_t) * 2 * 1024));
  int rc = make_map(&x->tm_xs, x->xs, c.m_cap, c.N, 1);
  if (!rc) rc = make_map(&x->tm_xg, x->xg, x->cap_rows_pad, c.N, 128);
  if (!rc) rc = make_map(&x->tm_H, x->H, x->cap_rows_pad, x->k_local, 128);
  if (!rc) rc = make_map(&x->tm_y, x->yrows, x->cap_rows_pad, c.N, 128);
  if (!rc) rc = make_map(&x->tm_Hs, x->H, x->cap_rows_pad, x->k_local, 32);
  if (!rc) rc = make_map(&x->tm_ys, x->yrows, x->cap_rows_pad, c.N, 32);
  return rc;
}

static int get_weight_map(comet_ctx* x, MapCache& mc, const void* w, uint64_t rows, uint64_t cols) {
  if (mc.ptr == w && mc.rows == rows && mc.cols == cols) return COMET_OK;
  if (int rc = make_map(&mc.map, w, rows, cols, 128)) return rc;
  mc.ptr = w;
  mc.rows = rows;
  mc.cols = cols;
  return COMET_OK;
}

static LayerArgs base_args(comet_ctx* x) {
  const auto& c = x->cfg;
  LayerArgs a{};
#ifdef COMET_TIMING_EXPERIMENTS
  // timing-experiment bits (layers.cuh LayerArgs::debug): a separate build
  // only, never the shipped library -- they skip work and give wrong results
  if (const char* d = getenv("COMET_DEBUG")) a.debug = atoi(d);
#endif
  a.rank = c.rank;
  a.world = c.world;
  a.tp = c.tp;
  a.ep = c.ep;
  a.M = x->M;
  a.topk = c.topk;
  a.n_embed = c.N;
  a.k_local = x->k_local;
  a.e_lo = x->e_lo;
  a.experts_per_group = x->E_r;
  a.epoch = x->epoch;
  a.meta = x->ix.meta;
  a.gather_row = x->ix.gather_row;
  a.pad_off = x->ix.pad_off;
  a.n_local = x->ix.n_local;
  a.xg = x->xg;
  a.xg_ready = x->xg_ready;
  a.xg_cnt = x->xg_ready + (x->cap_rows_pad / kTileRows + 1);
  a.pull_token = x->ix.pull_token;
  a.pull_src = x->ix.pull_src;
  a.tok_pos = x->ix.tok_pos;
  a.combine_tok = x->ix.combine_tok;
  a.row_dst = x->ix.row_dst;
  a.row_widx = x->ix.row_widx;
  const int W = c.world;
  a.xs_local = x->xs;
  a.xs_peer = reinterpret_cast<const __nv_bfloat16* const*>(x->peer_tab);
  a.cb_peer = reinterpret_cast<__nv_bfloat16* const*>(x->peer_tab + W);
  a.cb_flag_peer = reinterpret_cast<uint32_t* const*>(x->peer_tab + 2 * W);
  a.tok_ready = x->tok_ready;
  a.x_ready = x->x_ready;
  a.yrows = x->yrows;
  a.nb_done = x->counters;
  a.nb_sent = x->counters + x->nb1;
  a.mloc_cap = x->mloc_cap;
  a.ksplit_max = std::max(0, std::min(8, x->opt[COMET_OPT_KSPLIT_MAX]));  // measured: EP=8 M=1K-4K 10-20% faster
  a.timeline = x->timeline;
  a.timeline_cap = x->timeline_cap;
  return a;
}

static int layer_grid(comet_ctx* x) {
  int grid = std::min(x->n_sm, 2 * x->max_clusters);
  if (x->opt[COMET_OPT_GRID] > 0) grid = std::min(grid, x->opt[COMET_OPT_GRID]);
  return grid & ~1;
}


static int launch_kernel(comet_ctx* x, KernelArgs& f, const CUtensorMap& a0, const CUtensorMap& b0,
                         const CUtensorMap& a1, const CUtensorMap& b1, cudaStream_t st) {
  f.sched = x->sched;
  f.h_cnt = x->h_cnt;
  f.n_h = x->n_h;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(layer_grid(x));
  lc.blockDim = dim3(kLayerThreads);
  lc.dynamicSmemBytes = kLayerSmem;
  lc.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = (x->opt[COMET_OPT_PDL] & 2) ? 2 : 1;
  const bool timed = x->kt_slots > 0 && x->kt_next < x->kt_slots;
  if (timed) CK(cudaEventRecord(x->kt_ev[2 * x->kt_next], st));
  CK(cudaLaunchKernelEx(&lc, moe_layer_kernel, a0, b0, a1, b1, x->tm_Hs, x->tm_ys, f));
  if (timed) CK(cudaEventRecord(x->kt_ev[2 * x->kt_next++ + 1], st));
  return COMET_OK;
}

// Dispatch item rows (COMET_OPT_CHUNK_ROWS, 0 = auto): about one item per
// dispatch CTA for the expected rows of this rank (M * topk / ep at balanced
// routing), 4..32.  Each CTA streams its item at ~20 GB/s (one load/store
// ring), and every item of the first round lands at about the same time, so
// fewer rows per item publish the first tiles sooner when the rows are few
// (Mixtral EP=8, M=2K: 512 rows on 96 CTAs, 32-row items kept 80 CTAs idle
// and landed the first tile after ~12 us; 4-6 rows: -6..8% per forward);
// with many rows per CTA, 32-row items keep the per-item walk cheap (QW EP=8:
// 16 rows +1%, 4 rows +10%).
static int chunk_rows_for(const comet_ctx* x, int n_comm) {
  const int v = x->opt[COMET_OPT_CHUNK_ROWS];
  if (v > 0) return std::min(32, v);
  const auto& c = x->cfg;
  const long long rows = static_cast<long long>(x->M) * c.topk / std::max(1, c.ep);
  const long long per = n_comm > 0 ? (rows + n_comm - 1) / n_comm : 32;
  return static_cast<int>(std::max(4LL, std::min(32LL, per)));
}

// Layer0 arguments (dispatch + FC1 + activation); n_comm dispatch CTAs.
static int layer0_args(comet_ctx* x, const void* w0t, int activation, int n_comm, int group, LayerArgs* out) {
  const auto& c = x->cfg;
  if (activation < 0 || activation > COMET_ACT_TANH) return fail(COMET_EINVAL, "bad activation %d", activation);
  if (group < 1) return fail(COMET_EINVAL, "group must be >= 1");
  if (c.world > 1 && n_comm < 2) return fail(COMET_EINVAL, "world > 1: layer0 needs n_comm >= 2 (NVLink dispatch CTAs)");
  if (c.world == 1) n_comm = 0;  // no remote rows: every row is placed by the local dispatch
  if (n_comm < 0 || (n_comm & 1)) return fail(COMET_EINVAL, "n_comm=%d must be even and >= 0", n_comm);
  const int grid = layer_grid(x);
  if (grid - n_comm < 2) return fail(COMET_EINVAL, "n_comm=%d leaves no compute pair (grid %d)", n_comm, grid);
  if (int rc = ensure_work(x)) return rc;
  if (int rc = get_weight_map(x, x->w0c, w0t, (uint64_t)x->E_r * x->k_local, c.N)) return rc;
  LayerArgs a = base_args(x);
  a.layer = 0;
  a.part = x->part;
  a.split_cnt = x->split_cnt;
  a.n_compute = grid - n_comm;
  a.n_blocks = x->nb0;
  a.k_blocks = x->kb0;
  a.b_rows = x->k_local;
  a.order_group = group;
  a.raster = 0;
  a.activation = activation;
  a.split_tail = x->opt[COMET_OPT_SPLIT_TAIL0] != 0;
  a.sequential = x->opt[COMET_OPT_SEQUENTIAL] != 0;
  a.chunk_rows = chunk_rows_for(x, n_comm);
  a.dedup = 0;
  a.claim_of_tile = x->ix.claim_of_tile;
  a.pairs = x->ix.pairs0;
  a.out = x->H;
  a.out_ld = x->k_local;
  *out = a;
  return COMET_OK;
}

// Layer1 arguments (FC2 + top-k combine); n_comm combine CTAs (world 1 only).
static int layer1_args(comet_ctx* x, const void* w1t, const float* combine_w, void* y_local, int n_comm, int wave,
                       bool alone, LayerArgs* out) {
  const auto& c = x->cfg;
  if (wave < 1) return fail(COMET_EINVAL, "wave must be >= 1");
  if (n_comm < 0 || (n_comm & 1)) return fail(COMET_EINVAL, "n_comm=%d must be even and >= 0", n_comm);
  if (int rc = ensure_work(x)) return rc;
  if (int rc = get_weight_map(x, x->w1c, w1t, (uint64_t)x->E_r * c.N, x->k_local)) return rc;
  LayerArgs a = base_args(x);
  a.layer = 1;
  a.part = x->part + (size_t)x->n_sm * kTileRows * kBlockN;
  a.split_cnt = x->split_cnt + 1024;
  a.streamk = x->opt[COMET_OPT_STREAMK] != 0;
  a.n_blocks = x->nb1;
  a.k_blocks = x->kb1;
  a.b_rows = c.N;
  a.order_group = wave;
  a.order_group2 = 8;
  a.raster = 1;
  a.pairs = x->ix.pairs1;
  a.out = x->yrows;
  a.out_ld = c.N;
  a.combine_w = combine_w;
  a.y_local = static_cast<__nv_bfloat16*>(y_local);
  // Fused combine (world > 1 always; world 1 when no combine CTAs are asked
  // for and COMET_OPT_FUSE1 is set): the epilogue of each token's last hosted row
  // folds the earlier rows in and writes / pushes the result, so layer1 runs
  // without communication CTAs.  Otherwise combine CTAs (n_comm > 0) or the
  // local combine kernel reduce yrows.  At world 1 the fold's tile waits cost
  // what the local combine kernel saves (A/B in DESIGN.md), so it is opt-in.
  a.fuse_combine = c.world > 1 || (n_comm == 0 && x->opt[COMET_OPT_FUSE1] != 0);
  a.fold_stride = x->opt[COMET_OPT_FOLD_STRIDE];
  a.tile_done = x->tile_done;
  if (c.world > 1 || !alone) n_comm = 0;  // combine CTAs only in a layer1-alone launch at world 1
  const int grid = layer_grid(x);
  if (grid - n_comm < 2) return fail(COMET_EINVAL, "n_comm=%d leaves no compute pair (grid %d)", n_comm, grid);
  a.n_compute = grid - n_comm;
  // the last layer1 units may run as 256-column halves (finer tail; off by
  // default: a half moves 64 B/cycle/SM for its MMAs instead of 48 and ran
  // ~35% slower per FLOP, tools/fused_timeline.py)
  // Default: long fold chains (top-k >= 4 with >= 4 hosted experts: the last
  // units are folders reading up to k-1 rows each, 55-66 us epilogues at QW
  // EP=8) end layer1 in 256-column halves over 3/4 of the pairs, so the
  // folder epilogues split over twice the CTAs (QW EP=8 0.42 -> 0.40 ms;
  // MX: halves only cost, 0.44 -> 0.47 ms at EP=8 -- off).
  const int split1 = x->opt[COMET_OPT_SPLIT1];
  a.split_units = split1 >= 0 ? split1
                  : (a.fuse_combine && c.topk >= 4 && x->E_r >= 4) ? 3 * (layer_grid(x) / 2) / 4
                  : -1;  // -1: sched.cuh picks by the round count
  *out = a;
  return COMET_OK;
}

static int local_combine(comet_ctx* x, const LayerArgs& a, const float* combine_w, void* y_local, cudaStream_t st) {
  const auto& c = x->cfg;
  if (a.n_compute < layer_grid(x) || a.fuse_combine) return COMET_OK;  // combine CTAs / epilogue did it
  const int t0 = token_start_of(c.rank, x->M, c.world);
  const int n_tok = token_stop_of(c.rank, x->M, c.world) - t0;
  CK(launch_pdl(x->opt[COMET_OPT_PDL], 4, combine_local_kernel, dim3(x->n_sm * 8), dim3(256), 0, st, (const int32_t*)x->ix.tok_pos, combine_w,
                (const __nv_bfloat16*)x->yrows, static_cast<__nv_bfloat16*>(y_local), t0, n_tok, c.topk, c.N));
  return COMET_OK;
}

static int dispatch_local(comet_ctx* x, cudaStream_t st) {
  const auto& c = x->cfg;
  // HBM-local rows first (whole GPU, bandwidth-bound); dispatch CTAs pull only remote rows.
  CK(launch_pdl(x->opt[COMET_OPT_PDL], 1, dispatch_local_kernel, dim3(x->n_sm * 4), dim3(256), 0, st, (const int32_t*)x->ix.gather_row,
                (const int32_t*)x->ix.meta, (const __nv_bfloat16*)x->xs, x->xg, c.N, x->M, c.world, c.rank));
  return COMET_OK;
}

int comet_layer0(comet_ctx* x, const void* w0t, int activation, int n_comm, int group, void* stream) {
  CK(cudaSetDevice(x->cfg.device));
  KernelArgs f{};
  if (int rc = layer0_args(x, w0t, activation, n_comm, group, &f.l[0])) return rc;
  f.mode = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = dispatch_local(x, st)) return rc;
  return launch_kernel(x, f, x->tm_xg, x->w0c.map, x->tm_xg, x->w0c.map, st);
}

int comet_layer1(comet_ctx* x, const void* w1t, const float* combine_w, void* y_local, int n_comm, int wave,
                 void* stream) {
  CK(cudaSetDevice(x->cfg.device));
  KernelArgs f{};
  if (int rc = layer1_args(x, w1t, combine_w, y_local, n_comm, wave, true, &f.l[1])) return rc;
  f.mode = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = launch_kernel(x, f, x->tm_H, x->w1c.map, x->tm_H, x->w1c.map, st)) return rc;
  if (int rc = local_combine(x, f.l[1], combine_w, y_local, st)) return rc;
  x->last_y = y_local;
  x->last_combine_w = combine_w;
  return COMET_OK;
}

int comet_layers(comet_ctx* x, const void* w0t, const void* w1t, const float* combine_w, void* y_local,
                 int activation, int n_comm0, int group0, int wave1, void* stream) {
  CK(cudaSetDevice(x->cfg.device));
  KernelArgs f{};
  if (int rc = layer0_args(x, w0t, activation, n_comm0, group0, &f.l[0])) return rc;
  if (int rc = layer1_args(x, w1t, combine_w, y_local, 0, wave1, false, &f.l[1])) return rc;
  f.mode = 2;
  // layer1 in the layer0 pair groups (a group's layer1 units become ready
  // together).  Without fold chains (no fused combine, or one hosted expert
  // per token) layer1 walks the layer0 claim-ordered pair table itself, so
  // its first group is the group layer0 finished first; with fold chains it
  // keeps the expert-ascending table (a token's earlier hosted rows must sit
  // in earlier units of the same columns).
  f.l[1].raster = 2;
  f.l[1].order_group2 = group1(x, f.l[0].order_group);
  // layer0's last partial round in halves too: the layer1 units of its pairs
  // wait for it (critical path = last layer0 unit + one layer1 unit)
  if (!f.l[1].fuse_combine || x->E_r == 1 || x->cfg.topk == 1) f.l[1].pairs = x->ix.pairs0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // world > 1: the dispatch CTAs place the local rows too (locality-first:
  // they are the first tiles claimed), saving the local-dispatch launch
  f.l[0].pull_local = x->cfg.world > 1 && x->opt[COMET_OPT_PULL_LOCAL] != 0;
  // per-token dedup of the NVLink pulls (dispatch_rows_dedup; one read per
  // (token, rank), fanned out to the token's hosted rows)
  f.l[0].dedup = f.l[0].pull_local && x->cfg.topk <= 8 && dedup_on(x);
  if (!f.l[0].pull_local)
    if (int rc = dispatch_local(x, st)) return rc;
  if (int rc = launch_kernel(x, f, x->tm_xg, x->w0c.map, x->tm_H, x->w1c.map, st)) return rc;
  if (int rc = local_combine(x, f.l[1], combine_w, y_local, st)) return rc;
  x->last_y = y_local;
  x->last_combine_w = combine_w;
  return COMET_OK;
}

int comet_kernel_timing_enable(comet_ctx* x, int slots) {
  if (slots < 0) return fail(COMET_EINVAL, "slots=%d must be >= 0", slots);
  CK(cudaSetDevice(x->cfg.device));
  for (cudaEvent_t e : x->kt_ev) cudaEventDestroy(e);
  x->kt_ev.assign(2 * (size_t)slots, nullptr);
  for (auto& e : x->kt_ev) CK(cudaEventCreate(&e));
  x->kt_slots = slots;
  x->kt_next = 0;
  return COMET_OK;
}

int comet_kernel_timing_read(comet_ctx* x, float* ms_out, int cap, int* n_out) {
  CK(cudaSetDevice(x->cfg.device));
  const int n = std::min(cap, x->kt_next);
  for (int i = 0; i < n; ++i) {
    CK(cudaEventSynchronize(x->kt_ev[2 * i + 1]));
    CK(cudaEventElapsedTime(&ms_out[i], x->kt_ev[2 * i], x->kt_ev[2 * i + 1]));
  }
  if (n_out) *n_out = n;
  x->kt_next = 0;  // re-arm
  return COMET_OK;
}

int comet_timeline_enable(comet_ctx* x, int cap) {
  CK(cudaSetDevice(x->cfg.device));
  cudaFree(x->timeline);
  x->timeline = nullptr;
  x->timeline_cap = 0;
  if (cap <= 0) return COMET_OK;
  const size_t bytes = (size_t)x->n_sm * kRoles * cap * 2 * sizeof(unsigned long long);
  CK(cudaMalloc(&x->timeline, bytes));
  CK(cudaMemset(x->timeline, 0, bytes));
  x->timeline_cap = cap;
  return COMET_OK;
}

int comet_timeline_dump(comet_ctx* x, void* host_buf, size_t cap_bytes) {
  if (!x->timeline) return fail(COMET_EINVAL, "timeline not enabled");
  const size_t bytes = (size_t)x->n_sm * kRoles * x->timeline_cap * 2 * sizeof(unsigned long long);
  if (cap_bytes < bytes) return fail(COMET_EINVAL, "timeline buffer too small (%zu < %zu)", cap_bytes, bytes);
  CK(cudaSetDevice(x->cfg.device));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(host_buf, x->timeline, bytes, cudaMemcpyDeviceToHost));
  CK(cudaMemset(x->timeline, 0, bytes));
  return COMET_OK;
}

int comet_combine_finish(comet_ctx* x, void* y_local, void* stream) {
  const auto& c = x->cfg;
  if (c.world == 1) return COMET_OK;
  CK(cudaSetDevice(c.device));
  LayerArgs a = base_args(x);
  a.layer = 1;
  a.n_blocks = x->nb1;
  a.y_local = static_cast<__nv_bfloat16*>(y_local ? y_local : x->last_y);
  const int n_own = token_stop_of(c.rank, x->M, c.world) - token_start_of(c.rank, x->M, c.world);
  const int items = n_own * ((c.N / 8 + 127) / 128);  // one warp per (token, 1024-column segment)
  const int blocks = std::max(1, std::min(x->n_sm * 8, (items + 7) / 8));
  CK(launch_pdl(x->opt[COMET_OPT_PDL], 4, combine_finish_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), a,
                (const __nv_bfloat16*)x->cb, (const uint32_t*)x->cb_flag, (const int32_t*)x->ix.experts));
  CK(cudaGetLastError());
  return COMET_OK;
}

int comet_forward(comet_ctx* x, const int32_t* d_experts, int M, const void* w0t, const void* w1t,
                  const float* combine_w, void* y_local, int activation, int n_comm0, int n_comm1, int group0,
                  int wave1, void* stream) {
  // hot path: no reference-format tile lists; combine list only for comm-CTA combine
  // (the combine list only feeds world-1 combine CTAs; world > 1 fuses the combine)
  const int flags = (x->cfg.world == 1 && n_comm1 > 0 ? kIndexCombineList : 0) |
                    (x->cfg.world > 1 ? kIndexSignal : 0) | forward_order_flags(x);
  if (int rc = comet_index_build_ex(x, d_experts, M, 128, x->cfg.N >= 512 ? 128 : std::max(1, x->cfg.N / 4), flags,
                                    stream))
    return rc;
  // One launch for both layers (layer1 tiles start as their H rows land),
  // unless world-1 combine CTAs are asked for or COMET_OPT_FUSED is 0.
  const bool fused = x->opt[COMET_OPT_FUSED] != 0 && !(x->cfg.world == 1 && n_comm1 > 0);
  if (fused) {
    if (int rc = comet_layers(x, w0t, w1t, combine_w, y_local, activation, n_comm0, group0, wave1, stream)) return rc;
  } else {
    if (int rc = comet_layer0(x, w0t, activation, n_comm0, group0, stream)) return rc;
    if (int rc = comet_layer1(x, w1t, combine_w, y_local, n_comm1, wave1, stream)) return rc;
  }
  return comet_combine_finish(x, y_local, stream);
}

// Driver stream memory operations (flag writes / waits on the copy streams).
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_streamValue32 stream_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_streamValue32>(p);
}

int comet_forward_host(comet_ctx* x, const void* h_x, const int32_t* h_experts, const float* h_combine_w,
                       void* h_y, int M, const void* w0t, const void* w1t, int activation, int n_comm0, int group0,
                       int wave1, int chunks, void* stream) {
  const auto& c = x->cfg;
  if (c.world != 1) return fail(COMET_EINVAL, "comet_forward_host streams a single-GPU forward (world=%d)", c.world);
  if (M < 1 || M > c.m_cap) return fail(COMET_EINVAL, "M=%d outside [1, m_cap=%d]", M, c.m_cap);
  if (chunks < 1 || chunks > kMaxStreamChunks) return fail(COMET_EINVAL, "chunks=%d outside [1, %d]", chunks, kMaxStreamChunks);
  if (n_comm0 < 2 || (n_comm0 & 1)) return fail(COMET_EINVAL, "streamed forward needs n_comm0 >= 2, even");
  static PFN_streamValue32 write32 = stream_fn("cuStreamWriteValue32");
  static PFN_streamValue32 wait32 = stream_fn("cuStreamWaitValue32");
  if (!write32 || !wait32) return fail(COMET_ECUDA, "cuStreamWriteValue32 / cuStreamWaitValue32 unavailable");
  CK(cudaSetDevice(c.device));
  if (int rc = ensure_work(x)) return rc;
  if (!x->up_stream) {
    CK(cudaStreamCreateWithFlags(&x->up_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&x->down_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&x->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&x->ev_index, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&x->ev_down, cudaEventDisableTiming));
    CK(cudaMalloc(&x->chunk_ready, sizeof(uint32_t) * kMaxStreamChunks));
    if (!x->y_stream) CK(cudaMalloc(&x->y_stream, (size_t)c.m_cap * c.N * 2));
    CK(cudaMemset(x->chunk_ready, 0, sizeof(uint32_t) * kMaxStreamChunks));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int ct = (M + chunks - 1) / chunks;  // tokens per upload / download chunk
  const int n_ch = (M + ct - 1) / ct;
  const size_t row_b = (size_t)c.N * 2;
  // router output (+ weights) first: the index build needs only these
  CK(cudaMemcpyAsync(x->routing, h_experts, sizeof(int32_t) * (size_t)M * c.topk, cudaMemcpyHostToDevice, st));
  const float* cw = nullptr;
  if (h_combine_w) {
    if (!x->cw_dev) CK(cudaMalloc(&x->cw_dev, sizeof(float) * (size_t)c.m_cap * c.topk));
    CK(cudaMemcpyAsync(x->cw_dev, h_combine_w, sizeof(float) * (size_t)M * c.topk, cudaMemcpyHostToDevice, st));
    cw = x->cw_dev;
  }
  // the token upload may start once this call's prior work on `stream` is
  // done (the previous forward read the token buffer)
  CK(cudaEventRecord(x->ev_start, st));
  CK(cudaStreamWaitEvent(x->up_stream, x->ev_start, 0));
  if (int rc = comet_index_build_ex(x, x->routing, M, 128, c.N >= 512 ? 128 : std::max(1, c.N / 4), kIndexStream,
                                    stream))
    return rc;
  const uint32_t epoch = x->epoch;
  CK(cudaEventRecord(x->ev_index, st));  // output counters zeroed by this build
  for (int k = 0; k < n_ch; ++k) {
    const int t0 = k * ct, n = std::min(ct, M - t0);
    CK(cudaMemcpyAsync(static_cast<char*>(static_cast<void*>(x->xs)) + t0 * row_b,
                       static_cast<const char*>(h_x) + t0 * row_b, n * row_b, cudaMemcpyHostToDevice, x->up_stream));
    if (write32(x->up_stream, reinterpret_cast<CUdeviceptr>(x->chunk_ready + k), epoch, 0) != CUDA_SUCCESS)
      return fail(COMET_ECUDA, "cuStreamWriteValue32 failed");
  }
  // one launch: dispatch CTAs pull rows as their chunks land, layer1's
  // fused combine writes y rows and counts them per chunk
  KernelArgs f{};
  if (int rc = layer0_args(x, w0t, activation, 0, group0, &f.l[0])) return rc;
  if (int rc = layer1_args(x, w1t, cw, x->y_stream, 0, wave1, false, &f.l[1])) return rc;
  const int grid = layer_grid(x);
  f.mode = 2;
  f.l[0].n_compute = grid - n_comm0;
  f.l[0].stream = 1;
  f.l[0].pull_local = 1;
  f.l[0].chunk_ready = x->chunk_ready;
  f.l[0].chunk_tokens = ct;
  f.l[0].split_tail = 0;
  f.l[1].raster = 2;
  f.l[1].order_group2 = group1(x, f.l[0].order_group);
  f.l[1].pairs = x->ix.pairs0;  // (row tile, expert) order
  // the dispatch CTAs reduce finished token chunks (no layer1 unit waits for
  // another); COMET_STREAM_FUSE=1: the epilogue fold (folder claimed last)
  const bool fold = x->opt[COMET_OPT_STREAM_FUSE] != 0;
  f.l[0].stream_combine = fold ? 0 : 1;
  f.l[1].fuse_combine = fold ? 1 : 0;
  f.l[1].fold_stride = 0;  // the folder is the row claimed last, not the last slot: fold everything there
  f.l[1].publish_tiles = 1;
  f.l[1].y_local = x->y_stream;
  f.l[1].out_cnt = x->counters + 2 * x->nb1;
  f.l[1].chunk_tokens = ct;
  if (int rc = launch_kernel(x, f, x->tm_xg, x->w0c.map, x->tm_H, x->w1c.map, st)) return rc;
  // downloads: chunk k once its tokens' output halves are all final
  CK(cudaStreamWaitEvent(x->down_stream, x->ev_index, 0));
  const uint32_t halves = 2u * x->nb1 - ((c.N % kBlockN) && (c.N % kBlockN) <= kBlockN / 2 ? 1u : 0u);
  for (int k = 0; k < n_ch; ++k) {
    const int t0 = k * ct, n = std::min(ct, M - t0);
    if (wait32(x->down_stream, reinterpret_cast<CUdeviceptr>(x->counters + 2 * x->nb1 + k), (uint32_t)n * halves,
               0 /* CU_STREAM_WAIT_VALUE_GEQ */) != CUDA_SUCCESS)
      return fail(COMET_ECUDA, "cuStreamWaitValue32 failed");
    CK(cudaMemcpyAsync(static_cast<char*>(h_y) + t0 * row_b, static_cast<char*>(static_cast<void*>(x->y_stream)) + t0 * row_b,
                       n * row_b, cudaMemcpyDeviceToHost, x->down_stream));
  }
  CK(cudaEventRecord(x->ev_down, x->down_stream));
  CK(cudaStreamWaitEvent(st, x->ev_down, 0));  // the caller's stream covers the whole step
  x->last_y = x->y_stream;
  return COMET_OK;
}

// Zero-copy single-GPU forward: the host is the source "peer".  The dispatch
// CTAs read each token row once straight from pinned host memory over PCIe
// (deduplicated per token, fanned out to its hosted rows) in the compute
// claim order, then join the GEMMs; layer1's fused combine writes each
// token's output row straight into pinned host memory.  No staging copies:
// PCIe traffic is M*N*2 bytes each way, overlapped with the GEMMs.
int comet_forward_zerocopy(comet_ctx* x, const void* h_x, const int32_t* h_experts, const float* h_combine_w,
                           void* h_y, int M, const void* w0t, const void* w1t, int activation, int n_comm0, int group0,
                           int wave1, void* stream) {
  const auto& c = x->cfg;
  if (c.world != 1) return fail(COMET_EINVAL, "comet_forward_zerocopy is a single-GPU forward (world=%d)", c.world);
  if (M < 1 || M > c.m_cap) return fail(COMET_EINVAL, "M=%d outside [1, m_cap=%d]", M, c.m_cap);
  if (n_comm0 < 2 || (n_comm0 & 1)) return fail(COMET_EINVAL, "zero-copy forward needs n_comm0 >= 2, even");
  if (c.topk > 8) return fail(COMET_EINVAL, "zero-copy forward fans a token out to <= 8 rows (topk=%d)", c.topk);
  if (c.N % kBlockN) return fail(COMET_EINVAL, "zero-copy forward needs N %% %d == 0 (N=%d)", kBlockN, c.N);
  if (!h_x || !h_y || !h_experts) return fail(COMET_EINVAL, "null host buffer");
  CK(cudaSetDevice(c.device));
  if (int rc = ensure_work(x)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(cudaMemcpyAsync(x->routing, h_experts, sizeof(int32_t) * (size_t)M * c.topk, cudaMemcpyHostToDevice, st));
  const float* cw = nullptr;
  if (h_combine_w) {
    if (!x->cw_dev) CK(cudaMalloc(&x->cw_dev, sizeof(float) * (size_t)c.m_cap * c.topk));
    CK(cudaMemcpyAsync(x->cw_dev, h_combine_w, sizeof(float) * (size_t)M * c.topk, cudaMemcpyHostToDevice, st));
    cw = x->cw_dev;
  }
  // expert-ascending layer1 (fold-level order would put every folder row --
  // every host write -- into the second half of layer1; expert order spreads
  // the PCIe writes: 3.49 vs 3.84 ms, tools/stream_probe.py MODE=zc)
  // COMET_ZC_ORDER=1: pairs in (row tile, expert) order -- a pair's tokens
  // were mostly pulled for the same row tile of the previous experts, so the
  // PCIe bytes per tile are uniform instead of front-loaded (measured slower:
  // 3.7 vs 3.4 ms, consecutive units cycle through the experts' weights)
  const bool tile_order = x->opt[COMET_OPT_ZC_ORDER] != 0;
  const bool fold_order = !tile_order && x->E_r > 1 && x->E_r <= 64 && c.topk > 1 &&
                          x->opt[COMET_OPT_ZC_FOLD_ORDER] != 0;
  if (int rc = comet_index_build_ex(x, x->routing, M, 128, c.N >= 512 ? 128 : std::max(1, c.N / 4),
                                    (fold_order ? kIndexFoldOrder : 0) | (tile_order ? kIndexStream : 0), stream))
    return rc;
  // n_dl of the dispatch CTAs download the output afterwards (the fused
  // combine writes a device copy); n_dl = 0: the epilogues write h_y directly
  const int n_dl = std::min(n_comm0, std::max(0, x->opt[COMET_OPT_ZC_DOWNLOAD])) & ~1;
  if (n_dl > 0 && !x->y_stream) CK(cudaMalloc(&x->y_stream, (size_t)c.m_cap * c.N * 2));
  KernelArgs f{};
  if (int rc = layer0_args(x, w0t, activation, 0, group0, &f.l[0])) return rc;
  if (int rc = layer1_args(x, w1t, cw, n_dl > 0 ? static_cast<void*>(x->y_stream) : h_y, 0, wave1, false, &f.l[1]))
    return rc;
  f.mode = 2;
  f.n_dl = n_dl;
  f.y_host = static_cast<__nv_bfloat16*>(h_y);
  f.l[0].n_compute = layer_grid(x) - n_comm0;
  f.l[0].pull_local = 1;
  f.l[0].dedup = x->opt[COMET_OPT_ZC_DEDUP] != 0;
  f.l[0].host_src = static_cast<const __nv_bfloat16*>(h_x);
  f.l[1].raster = 2;
  f.l[1].order_group2 = group1(x, f.l[0].order_group);
  f.l[1].fuse_combine = 1;
  if (x->E_r == 1 || c.topk == 1 || tile_order) f.l[1].pairs = x->ix.pairs0;
  // Interleave the layers (COMET_OPT_ZC_INTERLEAVE groups of lag, default 1 with the
  // 16-pair groups the host layer passes; 0 = layer1 after all
  // of layer0): the dispatch is PCIe-paced, so layer0 alone leaves the
  // tensor cores waiting; layer1 groups of finished pairs fill the gaps and
  // start the host writes early.  Needs one pair order for both layers: at
  // world 1 the claim order is expert-ascending like pairs1 (no fold-level
  // order), and no split tails / split-K.
  f.interleave = fold_order ? 0 : std::max(0, x->opt[COMET_OPT_ZC_INTERLEAVE]);
  if (f.interleave > 0) {
    f.l[1].pairs = x->ix.pairs0;
    f.l[1].order_group2 = f.l[0].order_group;
    f.l[0].split_tail = 0;
    f.l[0].ksplit_max = 0;
    f.l[1].ksplit_max = 0;
    f.l[1].split_units = 0;
  }
  if (int rc = launch_kernel(x, f, x->tm_xg, x->w0c.map, x->tm_H, x->w1c.map, st)) return rc;
  x->last_y = h_y;
  x->last_combine_w = cw;
  return COMET_OK;
}

}  // extern "C"
