// Decode-step glue kernels for the tensor-parallel driver (decode.py).
//
// The quantized linears, their RMSNorm / SwiGLU prologues and the residual adds
// live in gemv.cu; what remains per layer is RoPE + KV-cache append (this file),
// the attention itself, and the final RMSNorm before the fp16 lm_head.
#include <cuda_fp16.h>

#include "common.cuh"

namespace qigen {

// qkv: f32 [B, 3, H, hd] (the fused QKV GEMV output).  Rotates q and k at
// position `pos` (rotate-half convention, cos/sin [hd/2] of that position),
// writes q as f16 [B, H, hd] and appends k, v (f16) to the layer's caches
// [B, H, ctx, hd] at `pos`.  One thread per (b, h, pair i < hd/2).
__global__ void rope_kv_kernel(const float* __restrict__ qkv, int B, int H, int hd,
                               const float* __restrict__ cosv, const float* __restrict__ sinv,
                               __half* __restrict__ q_out, __half* __restrict__ kc,
                               __half* __restrict__ vc, int ctx, int pos) {
  const int half = hd / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * H * half) return;
  const int i = idx % half, bh = idx / half;
  const int b = bh / H, h = bh % H;
  const float c = cosv[i], s = sinv[i];
  const float* q = qkv + ((size_t)(b * 3 + 0) * H + h) * hd;
  const float* k = qkv + ((size_t)(b * 3 + 1) * H + h) * hd;
  const float* v = qkv + ((size_t)(b * 3 + 2) * H + h) * hd;
  __half* qo = q_out + (size_t)bh * hd;
  qo[i] = __float2half_rn(q[i] * c - q[i + half] * s);
  qo[i + half] = __float2half_rn(q[i + half] * c + q[i] * s);
  const size_t co = ((size_t)bh * ctx + pos) * hd;
  kc[co + i] = __float2half_rn(k[i] * c - k[i + half] * s);
  kc[co + i + half] = __float2half_rn(k[i + half] * c + k[i] * s);
  vc[co + i] = __float2half_rn(v[i]);
  vc[co + i + half] = __float2half_rn(v[i + half]);
}

// out[b] = f16(h[b] * rsqrt(mean(h[b]^2) + eps) * w); one CTA per row.
__global__ void __launch_bounds__(1024) rmsnorm_f16_kernel(const float* __restrict__ h,
                                                          const float* __restrict__ w, int d,
                                                          float eps, __half* __restrict__ out) {
  // one CTA per row; 4 independent loads in flight per thread (a row of d <= 16K
  // floats is one L2 round trip, not d / blockDim dependent ones)
  constexpr int U = 4;
  const float* row = h + (size_t)blockIdx.x * d;
  float ss = 0.f;
  for (int k0 = threadIdx.x; k0 < d; k0 += blockDim.x * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * blockDim.x;
      v[u] = k < d ? row[k] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) ss += v[u] * v[u];
  }
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    ss = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (threadIdx.x == 0) red[0] = rsqrtf(ss / (float)d + eps);
  }
  __syncthreads();
  const float inv = red[0];
  for (int k = threadIdx.x; k < d; k += blockDim.x)
    out[(size_t)blockIdx.x * d + k] = __float2half_rn(row[k] * inv * w[k]);
}

}  // namespace qigen

using namespace qigen;

extern "C" int qigen_rope_kv(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                             const float* cos_pos, const float* sin_pos, void* q_out,
                             void* k_cache, void* v_cache, int64_t ctx, int64_t pos,
                             void* stream) {
  QIGEN_CHECK_ARG(qkv && cos_pos && sin_pos && q_out && k_cache && v_cache, QIGEN_ERR_ARG,
                  "null pointer");
  QIGEN_CHECK_ARG(head_dim % 2 == 0 && pos >= 0 && pos < ctx, QIGEN_ERR_ARG,
                  "bad head_dim / position");
  const int64_t n = batch * heads * (head_dim / 2);
  rope_kv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      qkv, (int)batch, (int)heads, (int)head_dim, cos_pos, sin_pos, (__half*)q_out,
      (__half*)k_cache, (__half*)v_cache, (int)ctx, (int)pos);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_rmsnorm_f16(const float* h, const float* w, int64_t rows, int64_t d,
                                 float eps, void* out, void* stream) {
  QIGEN_CHECK_ARG(h && w && out && rows > 0 && d > 0, QIGEN_ERR_ARG, "bad arguments");
  rmsnorm_f16_kernel<<<(unsigned)rows, 1024, 0, (cudaStream_t)stream>>>(h, w, (int)d, eps,
                                                                       (__half*)out);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}
