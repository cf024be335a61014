// Vocab-parallel LM head of the decode driver with the greedy argmax fused
// (local argmax + a (max, index) reduce instead of gathering the
// logits).  No reference counterpart (the reference has no model path,
// SPEC.md:13); it replaces the fp16 cuBLAS GEMV + torch argmax of the driver.
//
//   xn[b]       = fp16( h[b] * rsqrt(mean(h[b]^2) + eps) * norm_w )   (LLaMA final RMSNorm)
//   logits[b,v] = sum_k xn[b,k] W[v,k]                                 (W fp16 [V, d], f32 accumulate)
//   out[b]      = (max_v logits[b,v], v0 + argmax_v)                   (lowest index on ties)
//
// HBM-bound: the algorithmic bytes are the fp16 weight matrix (V d 2).  One
// persistent CTA (16 warps) per SM works on 16-row tiles of W; the 16 warps of a
// CTA split the tile's K range, each streaming 16 B per lane per row pair (two
// full rows of a 64 B segment per quad) straight into m16n8k16 f16 MMA
// fragments: swap-AB, the vocabulary rows are the M=16 side and the (<= 8)
// tokens the N=8 side.  The fragments use a permuted k order (lane quad t owns
// the contiguous k range 8t..8t+7 of each 32-k chunk) and the activations in
// shared memory are read in the same permuted order, so the dot products are
// exact re-associations of the same sums.  Small vocab shards (TP) also split
// the K range across CTAs; the last CTA to finish a tile adds the partials in
// slice order and the last tile reduces the per-tile best values in tile order:
// deterministic for any grid size.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"

namespace qigen {

constexpr int kLmWarps = 16;
constexpr int kLmThreads = kLmWarps * 32;
constexpr int kLmMaxB = 8;

struct LmArgs {
  const float* h;
  const float* nw;
  const __half* W;
  float* logits;      // [B, V] (may be null)
  float* part;        // [ntiles * S][16][8] partial logits (S > 1)
  float2* tbest;      // [ntiles][B] (max, local index as float bits)
  unsigned* cnt;      // [ntiles + 1] arrival counters (left zeroed after every launch)
  float* out_max;     // [B]
  int64_t* out_idx;   // [B]
  int64_t V, d, v0;
  int B, S, ntiles;
  float eps;
};

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

__global__ void __launch_bounds__(kLmThreads, 1) lm_head_kernel(const LmArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t xstr = a.d + 32;                                  // row stride (+64 B: banks)
  __half* xs = (__half*)smem;                                     // [B][xstr]
  float* red = (float*)(smem + (size_t)a.B * xstr * 2);           // [16 warps][16 rows][8 tokens]
  float* ssq = red + kLmWarps * 128;                              // [16 warps][8 tokens]
  float* inv = ssq + kLmWarps * kLmMaxB;                          // [8]
  float2* best = (float2*)(inv + kLmMaxB);                        // [4 row quads][8 tokens]
  int* flag = (int*)(best + 4 * kLmMaxB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int items = a.ntiles * a.S;
  const int64_t dk = a.d / a.S, dw = dk / kLmWarps;  // K per slice, per warp (multiples of 32)

  // the first item's weight rows into L2 before the programmatic-launch wait
  // (independent of the previous kernel)
  if (blockIdx.x < items) {
    const int t0 = blockIdx.x / a.S, ks = blockIdx.x % a.S;
    const int64_t lines = 16 * dk * 2 / 128;
    for (int64_t i = threadIdx.x; i < lines; i += kLmThreads) {
      const int64_t r = t0 * 16 + i / (dk * 2 / 128);
      if (r < a.V)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(
            (const char*)(a.W + r * a.d + ks * dk) + (i % (dk * 2 / 128)) * 128));
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");

  // ---- RMSNorm of the B rows of h -> fp16 activations in shared memory -------
  for (int b = 0; b < a.B; ++b) {
    float s = 0.f;
    for (int64_t k = 4 * threadIdx.x; k < a.d; k += 4 * kLmThreads) {
      const float4 v = *(const float4*)(a.h + b * a.d + k);
      s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ssq[warp * kLmMaxB + b] = s;
  }
  __syncthreads();
  if (threadIdx.x < a.B) {
    float s = 0.f;
    for (int w = 0; w < kLmWarps; ++w) s += ssq[w * kLmMaxB + threadIdx.x];
    inv[threadIdx.x] = rsqrtf(s / (float)a.d + a.eps);
  }
  __syncthreads();
  for (int b = 0; b < a.B; ++b) {
    const float r = inv[b];
    for (int64_t k = 4 * threadIdx.x; k < a.d; k += 4 * kLmThreads) {
      const float4 v = *(const float4*)(a.h + b * a.d + k);
      const float4 w = *(const float4*)(a.nw + k);
      __half2* dst = (__half2*)(xs + b * xstr + k);
      dst[0] = __floats2half2_rn(v.x * r * w.x, v.y * r * w.y);
      dst[1] = __floats2half2_rn(v.z * r * w.z, v.w * r * w.w);
    }
  }
  if (threadIdx.x < 4 * kLmMaxB) best[threadIdx.x] = make_float2(-INFINITY, __int_as_float(0x7fffffff));
  __syncthreads();

  const bool xon = gq < a.B;
  const __half* xrow = xs + (xon ? gq : 0) * xstr;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int tile = it / a.S, ks = it % a.S;
    const int64_t row0 = (int64_t)tile * 16;
    const int64_t ra = min(row0 + gq, a.V - 1), rb = min(row0 + gq + 8, a.V - 1);
    const int64_t k0 = ks * dk + warp * dw;
    const uint4* pa = (const uint4*)(a.W + ra * a.d + k0) + t;
    const uint4* pb = (const uint4*)(a.W + rb * a.d + k0) + t;
    const uint4* px = (const uint4*)(xrow + k0) + t;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    const int nch = (int)(dw / 32);
    int ch = 0;
    for (; ch + 4 <= nch; ch += 4) {  // 8 x 16 B loads in flight per lane
      uint4 wa[4], wb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wa[u] = __ldcs(pa + (ch + u) * 4);
        wb[u] = __ldcs(pb + (ch + u) * 4);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 xv = xon ? px[(ch + u) * 4] : make_uint4(0u, 0u, 0u, 0u);
        const uint32_t a1[4] = {wa[u].x, wb[u].x, wa[u].y, wb[u].y};
        const uint32_t a2[4] = {wa[u].z, wb[u].z, wa[u].w, wb[u].w};
        mma_f16(c, a1, xv.x, xv.y);
        mma_f16(c, a2, xv.z, xv.w);
      }
    }
    for (; ch < nch; ++ch) {
      const uint4 wa = __ldcs(pa + ch * 4), wb = __ldcs(pb + ch * 4);
      const uint4 xv = xon ? px[ch * 4] : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t a1[4] = {wa.x, wb.x, wa.y, wb.y};
      const uint32_t a2[4] = {wa.z, wb.z, wa.w, wb.w};
      mma_f16(c, a1, xv.x, xv.y);
      mma_f16(c, a2, xv.z, xv.w);
    }
    // warp partials [row][token] -> fixed-order sum over the 16 warps
    red[(warp * 16 + gq) * 8 + 2 * t] = c[0];
    red[(warp * 16 + gq) * 8 + 2 * t + 1] = c[1];
    red[(warp * 16 + gq + 8) * 8 + 2 * t] = c[2];
    red[(warp * 16 + gq + 8) * 8 + 2 * t + 1] = c[3];
    __syncthreads();
    float v = 0.f;
    const int e = threadIdx.x;  // e < 128: (row e / 8, token e % 8)
    if (e < 128) {
#pragma unroll
      for (int w = 0; w < kLmWarps; ++w) v += red[w * 128 + e];
    }
    bool final_ = a.S == 1;
    if (a.S > 1) {
      if (e < 128) a.part[(size_t)it * 128 + e] = v;
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) *flag = atomicAdd(&a.cnt[tile], 1u) == (unsigned)(a.S - 1);
      __syncthreads();
      final_ = *flag;
      if (final_) {
        __threadfence();
        if (e < 128) {
          v = 0.f;
          for (int q = 0; q < a.S; ++q) v += __ldcg(a.part + ((size_t)tile * a.S + q) * 128 + e);
        }
        if (threadIdx.x == 0) a.cnt[tile] = 0u;  // re-armed for the next launch
      }
    }
    if (final_ && e < 128) {
      const int r = e >> 3, b = e & 7;
      const int64_t vrow = row0 + r;
      const bool live = vrow < a.V && b < a.B;
      if (live && a.logits) a.logits[b * a.V + vrow] = v;
      float bv = live ? v : -INFINITY;
      int bi = live ? (int)vrow : 0x7fffffff;
#pragma unroll
      for (int o = 8; o < 32; o <<= 1) {  // the 4 rows of this warp, same token
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
      }
      if (lane < 8) {
        const float2 cur = best[warp * 8 + lane];
        if (better(bv, bi, cur.x, __float_as_int(cur.y)))
          best[warp * 8 + lane] = make_float2(bv, __int_as_float(bi));
      }
    }
    __syncthreads();
    if (final_) {  // (CTA-uniform)
      if (threadIdx.x < a.B) {  // this tile's best per token, reduced in tile order below
        float2 bb = best[threadIdx.x];
        for (int q = 1; q < 4; ++q) {
          const float2 o = best[q * 8 + threadIdx.x];
          if (better(o.x, __float_as_int(o.y), bb.x, __float_as_int(bb.y))) bb = o;
        }
        a.tbest[(size_t)tile * a.B + threadIdx.x] = bb;
      }
      __syncthreads();
      if (threadIdx.x < 4 * kLmMaxB)
        best[threadIdx.x] = make_float2(-INFINITY, __int_as_float(0x7fffffff));
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        *flag = atomicAdd(&a.cnt[a.ntiles], 1u) == (unsigned)(a.ntiles - 1) ? 2 : 0;
      __syncthreads();
      if (*flag == 2) {  // every tile is final: reduce the tile bests in tile order
        __threadfence();
        if (threadIdx.x < a.B) {
          float bv = -INFINITY;
          int bi = 0x7fffffff;
          for (int q = 0; q < a.ntiles; ++q) {
            const float2 o = __ldcg(&a.tbest[(size_t)q * a.B + threadIdx.x]);
            if (better(o.x, __float_as_int(o.y), bv, bi)) { bv = o.x; bi = __float_as_int(o.y); }
          }
          a.out_max[threadIdx.x] = bv;
          a.out_idx[threadIdx.x] = a.v0 + bi;
        }
        if (threadIdx.x == 0) a.cnt[a.ntiles] = 0u;
      }
      __syncthreads();
    }
  }
}

}  // namespace qigen

using namespace qigen;

static int lm_slices(int64_t V, int64_t d, int sms) {
  const int64_t ntiles = (V + 15) / 16;
  int S = 1;
  while (ntiles * S < 2 * sms && d % (S * 2 * kLmWarps * 32) == 0 && S < 16) S *= 2;
  return S;
}

extern "C" int64_t qigen_lm_head_workspace_size(int64_t vocab, int64_t d, int64_t batch) {
  const int64_t ntiles = (vocab + 15) / 16;
  const int64_t S = 16;  // upper bound of lm_slices
  return ntiles * S * 128 * 4 + ntiles * std::max<int64_t>(batch, 1) * 8 + (ntiles + 1) * 4 + 256;
}

extern "C" int qigen_lm_head(const float* h, const float* norm_w, float eps, const void* w_f16,
                             int64_t vocab, int64_t d, int64_t batch, int64_t vocab_offset,
                             float* logits, float* out_max, int64_t* out_idx, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  QIGEN_CHECK_ARG(h && norm_w && w_f16 && out_max && out_idx && workspace, QIGEN_ERR_ARG,
                  "null pointer");
  QIGEN_CHECK_ARG(batch >= 1 && batch <= kLmMaxB, QIGEN_ERR_UNSUPPORTED,
                  "LM head takes 1..%d tokens", kLmMaxB);
  QIGEN_CHECK_ARG(vocab >= 1 && vocab < (1ll << 30), QIGEN_ERR_ARG, "bad vocabulary size");
  QIGEN_CHECK_ARG(d >= 512 && d % 512 == 0, QIGEN_ERR_UNSUPPORTED,
                  "LM head: d_model must be a multiple of 512, got %lld", (long long)d);
  QIGEN_CHECK_ARG(workspace_bytes >= qigen_lm_head_workspace_size(vocab, d, batch), QIGEN_ERR_ARG,
                  "LM head workspace too small");
  const size_t smem = (size_t)batch * (d + 32) * 2 + kLmWarps * 128 * 4 + kLmWarps * kLmMaxB * 4 +
                      kLmMaxB * 4 + 4 * kLmMaxB * 8 + 16;
  QIGEN_CHECK_ARG(smem <= 227 * 1024, QIGEN_ERR_UNSUPPORTED, "LM head: batch x d too large");
  int dev = 0, sms = 148;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static OncePerDevice once;
  const int cst = once.run([]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
    return QIGEN_OK;
  });
  if (cst) return cst;
  LmArgs a;
  a.h = h;
  a.nw = norm_w;
  a.W = (const __half*)w_f16;
  a.logits = logits;
  a.V = vocab;
  a.d = d;
  a.v0 = vocab_offset;
  a.B = (int)batch;
  a.eps = eps;
  a.ntiles = (int)((vocab + 15) / 16);
  a.S = lm_slices(vocab, d, sms);
  char* ws = (char*)workspace;
  a.part = (float*)ws;
  ws += (size_t)a.ntiles * 16 * 128 * 4;
  a.tbest = (float2*)ws;
  ws += (size_t)a.ntiles * batch * 8;
  a.cnt = (unsigned*)ws;
  a.out_max = out_max;
  a.out_idx = out_idx;
  const int items = a.ntiles * a.S;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min(items, sms), 1, 1);
  cfg.blockDim = dim3(kLmThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, lm_head_kernel, a));
  return QIGEN_OK;
}
