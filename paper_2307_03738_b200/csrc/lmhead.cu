// Vocab-parallel LM head of the decode driver with the greedy argmax fused
// (local argmax + a (max, index) reduce instead of gathering the
// logits).  No reference counterpart (the reference has no model path,
// SPEC.md:13); it replaces the fp16 cuBLAS GEMV + torch argmax of the driver.
//
//   xn[b]       = fp16( h[b] * rsqrt(mean(h[b]^2) + eps) * norm_w )   (LLaMA final RMSNorm)
//   logits[b,v] = sum_k xn[b,k] W[v,k]                                 (W fp16 [V, d], f32 accumulate)
//   out[b]      = (max_v logits[b,v], v0 + argmax_v)                   (lowest index on ties)
//
// HBM-bound: the algorithmic bytes are the fp16 weight matrix (V d 2).  A warp
// owns a 16-row tile of W over a K slice and streams it with 16 B loads (16 in
// flight per lane) straight into m16n8k16 f16 MMA fragments: swap-AB, the
// vocabulary rows are the M=16 side and the (<= 8) tokens the N=8 side.  The
// fragments use a permuted k order (lane quad t owns the contiguous k range
// 8t..8t+7 of each 32-k chunk) and the activations in shared memory are read in
// the same permuted order, so each dot product is a re-association of the same
// sum.  Large vocabularies give every warp whole rows (no reduction, no CTA
// barrier in the stream); small vocab shards (TP) split each tile's K range over
// up to 16 warps of one CTA, reduced in warp order through shared memory.  The
// argmax is a running (max, lowest index) per warp, then per CTA in warp order,
// then across CTAs in CTA order by the last CTA to finish: deterministic.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"

namespace qigen {

constexpr int kLmWarps = 16;
constexpr int kLmThreads = kLmWarps * 32;
constexpr int kLmMaxB = 8;
// Streaming: a warp's chunks (32 k of its 16 rows) go in batches of U through
// a per-warp shared-memory ring of kLmDepth batches filled with cp.async (16 B
// per lane and row, each lane reads back only its own bytes): kLmDepth - 1
// batches stay in flight (U KB each per warp), and the first ones are issued
// before the programmatic-launch wait (the weights do not depend on the
// previous kernel), so they overlap the RMSNorm prologue.
constexpr int kLmDepth = 3;

struct LmArgs {
  const float* h;
  const float* nw;
  const __half* W;
  float* logits;      // [B, V] (may be null)
  float2* cbest;      // [grid][B] (max, local index as float bits) per CTA
  unsigned* cnt;      // arrival counter (left zeroed after every launch)
  float* out_max;     // [B]
  int64_t* out_idx;   // [B]
  int64_t V, d, v0;
  int B, SK, ntiles;  // SK: warps per tile (K slices), 1..16
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

__device__ __forceinline__ void mma_chunk(float (&c)[4], uint4 wa, uint4 wb, uint4 xv) {
  const uint32_t a1[4] = {wa.x, wb.x, wa.y, wb.y};
  const uint32_t a2[4] = {wa.z, wb.z, wa.w, wb.w};
  mma_f16(c, a1, xv.x, xv.y);
  mma_f16(c, a2, xv.z, xv.w);
}

template <int U>
__global__ void __launch_bounds__(kLmThreads, 1) lm_head_kernel(const LmArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t xstr = a.d + 32;                                  // row stride (+64 B: banks)
  __half* xs = (__half*)smem;                                     // [B][xstr]
  float* red = (float*)(smem + (size_t)a.B * xstr * 2);           // [16 warps][16 rows][8 tokens]
  float* ssq = red + kLmWarps * 128;                              // [16 warps][8 tokens]
  float* inv = ssq + kLmWarps * kLmMaxB;                          // [8]
  float2* wbest = (float2*)(inv + kLmMaxB);                       // [16 warps][8 tokens]
  int* flag = (int*)(wbest + kLmWarps * kLmMaxB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int SK = a.SK, TPC = kLmWarps / SK;                       // tiles per CTA iteration
  const int64_t dw = a.d / SK;                                    // K per warp (multiple of 32 U)
  const int my_tile = warp / SK, my_ks = warp % SK;
  const int nb = (int)(dw / (32 * U));                            // batches per tile
  const int iters = (a.ntiles + TPC * gridDim.x - 1) / (TPC * gridDim.x);
  const int total = iters * nb;                                   // CTA-uniform

  auto tile_of = [&](int q) { return ((int64_t)(q / nb) * gridDim.x + blockIdx.x) * TPC + my_tile; };
  // this warp's ring: kLmDepth slots of U x 2 rows x 32 lanes x 16 B, after the
  // activations / reduction scratch
  unsigned char* ring = smem + (((size_t)a.B * xstr * 2 + kLmWarps * 128 * 4 +
                                 kLmWarps * kLmMaxB * 4 + kLmMaxB * 4 + kLmWarps * kLmMaxB * 8 +
                                 16 + 127) & ~(size_t)127) +
                        (size_t)warp * kLmDepth * U * 1024;
  auto issue = [&](int q) {  // batch q -> slot q % kLmDepth (one commit group, maybe empty)
    const int64_t tile = tile_of(q);
    if (q < total && tile < a.ntiles) {
      const int64_t row0 = tile * 16;
      const int64_t ra = min(row0 + gq, a.V - 1), rb = min(row0 + gq + 8, a.V - 1);
      const int64_t k0 = my_ks * dw + (int64_t)(q % nb) * 32 * U;
      const uint4* pa = (const uint4*)(a.W + ra * a.d + k0) + t;
      const uint4* pb = (const uint4*)(a.W + rb * a.d + k0) + t;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (q % kLmDepth) * U * 1024) +
                           lane * 16;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (2 * u) * 512),
                     "l"(pa + u * 4) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (2 * u + 1) * 512),
                     "l"(pb + u * 4) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int q = 0; q < kLmDepth - 1; ++q) issue(q);
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
  __syncthreads();

  const bool xon = gq < a.B;
  const __half* xrow = xs + (xon ? gq : 0) * xstr;
  // running best of this lane's tokens 2t, 2t+1 (valid in lanes gq == 0 after reduction)
  float bv[2] = {-INFINITY, -INFINITY};
  int bi[2] = {0x7fffffff, 0x7fffffff};
  float c[4] = {0.f, 0.f, 0.f, 0.f};

  // batch q of this warp from its ring slot; at a tile's last batch: reduce its
  // K slices (fixed warp order) and fold its rows into the running argmax
  auto consume = [&](int q) {
    const int64_t tile = tile_of(q);
    const bool live_tile = tile < a.ntiles;
    if (live_tile) {
      const uint4* src = (const uint4*)(ring + (q % kLmDepth) * U * 1024) + lane;
      const uint4* px = (const uint4*)(xrow + my_ks * dw + (int64_t)(q % nb) * 32 * U) + t;
#pragma unroll
      for (int u = 0; u < U; ++u)
        mma_chunk(c, src[(2 * u) * 32], src[(2 * u + 1) * 32],
                  xon ? px[u * 4] : make_uint4(0u, 0u, 0u, 0u));
    }
    if (q % nb != nb - 1) return;
    bool owner = true;  // this warp holds the tile's final values
    if (SK > 1) {       // K slices of a tile: fixed-order sum over its SK warps
      red[(warp * 16 + gq) * 8 + 2 * t] = c[0];
      red[(warp * 16 + gq) * 8 + 2 * t + 1] = c[1];
      red[(warp * 16 + gq + 8) * 8 + 2 * t] = c[2];
      red[(warp * 16 + gq + 8) * 8 + 2 * t + 1] = c[3];
      __syncthreads();
      owner = my_ks == 0;
      if (owner) {
        c[0] = c[1] = c[2] = c[3] = 0.f;
        for (int s = 0; s < SK; ++s) {
          const float* r = red + (warp + s) * 128;
          c[0] += r[gq * 8 + 2 * t];
          c[1] += r[gq * 8 + 2 * t + 1];
          c[2] += r[(gq + 8) * 8 + 2 * t];
          c[3] += r[(gq + 8) * 8 + 2 * t + 1];
        }
      }
      __syncthreads();  // red is rewritten at the next tile
    }
    if (owner && live_tile) {
      const int64_t row0 = tile * 16;
#pragma unroll
      for (int h = 0; h < 2; ++h) {    // rows gq, gq + 8
#pragma unroll
        for (int j = 0; j < 2; ++j) {  // tokens 2t, 2t + 1
          const int64_t v = row0 + gq + 8 * h;
          const int b = 2 * t + j;
          const float val = c[2 * h + j];
          if (v < a.V && b < a.B) {
            if (a.logits) a.logits[b * a.V + v] = val;
            if (better(val, (int)v, bv[j], bi[j])) { bv[j] = val; bi[j] = (int)v; }
          }
        }
      }
    }
    c[0] = c[1] = c[2] = c[3] = 0.f;
  };
  for (int q = 0; q < total; ++q) {
    issue(q + kLmDepth - 1);  // (slot (q - 1) % depth: consumed in the previous iteration)
    asm volatile("cp.async.wait_group %0;" ::"n"(kLmDepth - 1) : "memory");
    consume(q);
  }
  // warp: reduce over the 8 row groups (lanes with the same t), then CTA, then grid
#pragma unroll
  for (int j = 0; j < 2; ++j) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv[j], o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi[j], o);
      if (better(ov, oi, bv[j], bi[j])) { bv[j] = ov; bi[j] = oi; }
    }
  }
  if (gq == 0)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      wbest[warp * kLmMaxB + 2 * t + j] = make_float2(bv[j], __int_as_float(bi[j]));
  __syncthreads();
  if (threadIdx.x < a.B) {
    float2 cb = wbest[threadIdx.x];
    for (int w = 1; w < kLmWarps; ++w) {
      const float2 o = wbest[w * kLmMaxB + threadIdx.x];
      if (better(o.x, __float_as_int(o.y), cb.x, __float_as_int(cb.y))) cb = o;
    }
    a.cbest[(size_t)blockIdx.x * a.B + threadIdx.x] = cb;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *flag = atomicAdd(a.cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (*flag) {  // the last CTA: reduce the CTAs' bests in CTA order
    __threadfence();
    if (threadIdx.x < a.B) {
      float v = -INFINITY;
      int i = 0x7fffffff;
      for (int q = 0; q < (int)gridDim.x; ++q) {
        const float2 o = __ldcg(&a.cbest[(size_t)q * a.B + threadIdx.x]);
        if (better(o.x, __float_as_int(o.y), v, i)) { v = o.x; i = __float_as_int(o.y); }
      }
      a.out_max[threadIdx.x] = v;
      a.out_idx[threadIdx.x] = a.v0 + i;
    }
    if (threadIdx.x == 0) *a.cnt = 0u;  // re-armed for the next launch
  }
}

}  // namespace qigen

using namespace qigen;

// Warps per 16-row tile (K slices): the split that minimises the longest
// warp's stream, ceil(tiles / (tiles per CTA iteration x grid)) x d / SK
// (ties: fewer slices, i.e. fewer CTA barriers); K per warp a multiple of 32.
static int lm_slices(int64_t V, int64_t d, int sms) {
  const int64_t ntiles = (V + 15) / 16;
  int best = 1;
  double best_cost = 1e30;
  for (int SK = 1; SK <= kLmWarps && d % (SK * 32) == 0; SK *= 2) {
    const int64_t tpc = kLmWarps / SK;
    const int64_t grid = std::min<int64_t>(sms, (ntiles + tpc - 1) / tpc);
    const int64_t iters = (ntiles + tpc * grid - 1) / (tpc * grid);
    const double cost = (double)iters / SK;
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = SK;
    }
  }
  return best;
}

extern "C" int64_t qigen_lm_head_workspace_size(int64_t vocab, int64_t d, int64_t batch) {
  (void)vocab; (void)d;
  return 1024 * std::max<int64_t>(batch, 1) * 8 + 256;  // per-CTA bests (<= 1024 CTAs) + counter
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
  const size_t smem0 = ((size_t)batch * (d + 32) * 2 + kLmWarps * 128 * 4 + kLmWarps * kLmMaxB * 4 +
                        kLmMaxB * 4 + kLmWarps * kLmMaxB * 8 + 16 + 127) & ~(size_t)127;
  QIGEN_CHECK_ARG(smem0 + kLmWarps * kLmDepth * 1024 <= 227 * 1024, QIGEN_ERR_UNSUPPORTED,
                  "LM head: batch x d too large");
  int dev = 0, sms = 148;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  static OncePerDevice once;
  const int cst = once.run([]() -> int {
    for (auto kf : {lm_head_kernel<4>, lm_head_kernel<2>, lm_head_kernel<1>})
      QIGEN_CUDA_RET(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  a.SK = lm_slices(vocab, d, sms);
  const int tpc = kLmWarps / a.SK;
  const int grid = (int)std::min<int64_t>(sms, (a.ntiles + tpc - 1) / tpc);
  a.cbest = (float2*)workspace;
  a.cnt = (unsigned*)((char*)workspace + 1024 * batch * 8);
  a.out_max = out_max;
  a.out_idx = out_idx;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(kLmThreads, 1, 1);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  // batch size U: the largest of 4 / 2 / 1 chunks that divides a warp's chunks
  // and whose ring fits next to the activations
  const int64_t nch = d / a.SK / 32;  // 32-k chunks per warp and tile
  int U = 1;
  for (int u : {4, 2})
    if (nch % u == 0 && smem0 + (size_t)kLmWarps * kLmDepth * u * 1024 <= 227 * 1024) {
      U = u;
      break;
    }
  cfg.dynamicSmemBytes = smem0 + (size_t)kLmWarps * kLmDepth * U * 1024;
  auto kern = U == 4 ? lm_head_kernel<4> : U == 2 ? lm_head_kernel<2> : lm_head_kernel<1>;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, kern, a));
  return QIGEN_OK;
}
