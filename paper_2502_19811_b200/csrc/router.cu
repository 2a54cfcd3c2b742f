// GPU router front-end: gate logits [M, E] -> the
// reference's router output, top-k expert ids stored ascending per token
// (RoutingTable.experts_per_token, routing.py:146-163, the layout
// moe_index_build consumes), plus the combine weights in the same
// ascending-expert slot order (_combine's combine_weights[t, slot],
// executor.py:102-120).
//
// Selection order = (logit descending, expert id ascending): a stable
// descending argsort, so ties go to the smaller id.  -0.0 ties +0.0; NaN
// ranks below -inf.  Bit-exact against oracle/moe_oracle.router_topk.
//
// Weights (fp32): kNormTopk  softmax over the k selected logits (Mixtral);
//                 kNormAll   softmax over all E logits, selected entries
//                            (Qwen2-MoE, norm_topk_prob = False).
//
// One warp per token; lane l holds logits l, l+32, ... (coalesced row read).
// Integer/latency-bound: M*E*4 bytes in, M*k*8 bytes out.
#include <cuda_bf16.h>
#include <cstdint>

namespace comet {

enum RouterNorm : int { kNormNone = 0, kNormTopk = 1, kNormAll = 2 };

namespace {

__device__ __forceinline__ uint32_t order_key(float f) {
  if (f != f) return 0u;          // NaN: below every number
  if (f == 0.f) f = 0.f;          // -0.0 == +0.0
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // -inf -> 0x007FFFFF > 0
}

template <int EPL>
__device__ __forceinline__ void route_token(const float (&v)[EPL], int E, int topk, int norm, int lane,
                                            int32_t* out_e, float* out_w) {
  // 64-bit keys: (order key << 32) | ~id  -> max = largest logit, then smallest id.
  unsigned long long key[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    key[j] = e < E ? (static_cast<unsigned long long>(order_key(v[j])) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(e))
                   : 0ull;
  }
  int my_id = 0x7FFFFFFF;  // lane s < topk keeps the s-th selected expert
  float my_logit = 0.f;
  for (int s = 0; s < topk; ++s) {
    unsigned long long best = 0ull;
#pragma unroll
    for (int j = 0; j < EPL; ++j) best = key[j] > best ? key[j] : best;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other > best ? other : best;
    }
    const int id = static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(best & 0xFFFFFFFFull));
    float lg = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (lane + 32 * j == id) { key[j] = 0ull; lg = v[j]; }
    lg = __shfl_sync(0xffffffffu, lg, id & 31);
    if (lane == s) { my_id = id; my_logit = lg; }
  }
  // weights
  float w = 0.f;
  if (norm == kNormTopk) {
    const float mx = __shfl_sync(0xffffffffu, my_logit, 0);  // slot 0 holds the largest logit
    const float ex = lane < topk ? expf(my_logit - mx) : 0.f;
    float sum = ex;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    w = ex / sum;
  } else if (norm == kNormAll) {
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (lane + 32 * j < E) mx = fmaxf(mx, v[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (lane + 32 * j < E) sum += expf(v[j] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    w = expf(my_logit - mx) / sum;
  }
  // ascending id order: slot of lane s = number of selected ids below its id
  int pos = 0;
  for (int s = 0; s < topk; ++s) {
    const int other = __shfl_sync(0xffffffffu, my_id, s);
    pos += other < my_id;
  }
  if (lane < topk) {
    out_e[pos] = my_id;
    if (out_w) out_w[pos] = w;
  }
}

template <int EPL, typename T>
__global__ void __launch_bounds__(256) router_topk_kernel(const T* __restrict__ logits, int M, int E, int topk,
                                                          int norm, int32_t* __restrict__ experts,
                                                          float* __restrict__ weights) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < M; t += warps) {
    const T* row = logits + static_cast<long long>(t) * E;
    float v[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = lane + 32 * j;
      if constexpr (sizeof(T) == 4) v[j] = e < E ? __ldg(reinterpret_cast<const float*>(row) + e) : 0.f;
      else v[j] = e < E ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(row)[e]) : 0.f;
    }
    route_token<EPL>(v, E, topk, norm, lane, experts + static_cast<long long>(t) * topk,
                     weights ? weights + static_cast<long long>(t) * topk : nullptr);
  }
}

template <typename T>
cudaError_t launch_typed(const void* logits, int M, int E, int topk, int norm, int32_t* experts, float* weights,
                         int n_sm, cudaStream_t stream) {
  const int blocks = max(1, min((M + 7) / 8, n_sm * 8));
  const T* lg = static_cast<const T*>(logits);
  if (E <= 32) router_topk_kernel<1, T><<<blocks, 256, 0, stream>>>(lg, M, E, topk, norm, experts, weights);
  else if (E <= 64) router_topk_kernel<2, T><<<blocks, 256, 0, stream>>>(lg, M, E, topk, norm, experts, weights);
  else if (E <= 128) router_topk_kernel<4, T><<<blocks, 256, 0, stream>>>(lg, M, E, topk, norm, experts, weights);
  else if (E <= 256) router_topk_kernel<8, T><<<blocks, 256, 0, stream>>>(lg, M, E, topk, norm, experts, weights);
  else router_topk_kernel<16, T><<<blocks, 256, 0, stream>>>(lg, M, E, topk, norm, experts, weights);
  return cudaGetLastError();
}

}  // namespace

// logits_dtype: 0 = fp32, 1 = bf16.  E <= 512, 1 <= topk <= min(E, 32).
cudaError_t router_topk_launch(const void* logits, int logits_dtype, int M, int E, int topk, int norm,
                               int32_t* experts, float* weights, int n_sm, cudaStream_t stream) {
  if (M == 0) return cudaSuccess;
  return logits_dtype == 1 ? launch_typed<__nv_bfloat16>(logits, M, E, topk, norm, experts, weights, n_sm, stream)
                           : launch_typed<float>(logits, M, E, topk, norm, experts, weights, n_sm, stream);
}

}  // namespace comet
