// Decode-step glue kernels for the tensor-parallel driver (decode.py).
//
// The quantized linears, their RMSNorm / SwiGLU prologues and the residual adds
// live in gemv.cu; what remains per layer is RoPE + KV-cache append (this file),
// the attention itself, and the final RMSNorm before the fp16 lm_head.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "gemv_common.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

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

// ---- fused decode attention ---------------------------------------------------
// One new token per sequence attends over its KV cache (flash-decoding split
// over positions).  Per CTA: one (sequence, head) and a chunk of positions; the
// nsplit CTAs of a head form a thread-block cluster (nsplit <= 16).  The
// chunk's cached K/V rows (written by earlier decode steps, not by the
// preceding kernel) are bulk-copied into shared memory BEFORE the PDL wait, so
// they stream while the QKV GEMV finishes; after the wait the CTA applies RoPE
// to q (and, in the chunk holding `pos`, to the new k, appending k/v to the
// cache) and computes its partial softmax state (m, l, acc), which it writes
// into the rank-0 CTA's shared memory (DSMEM); after one cluster barrier rank 0
// combines the partials in split order (deterministic, no global round trip).
constexpr int kAttnMaxSplit = 16;
constexpr int kAttnThreads = 256;  // 8 warps (measured best: 128 and 512 slower, tools/attn_exp.py)

struct AttnArgs {
  const float* qkv;  // [B, 3, H, HD] f32 (the fused QKV GEMV output)
  const float* cosv;
  const float* sinv;  // [HD/2] at pos
  __half* kc;
  __half* vc;  // [B, H, ctx, HD]
  float* out;  // [B, H * HD]
  int B, H, ctx, pos, nsplit, chunk;
  float scale;
  unsigned long long* trace;  // optional per-CTA %globaltimer: entry, after wait, exit
  // decode chain: the head's output also written as the o_proj GEMV's prepared
  // activation digits (qigen_gemv_chain layout: K = H * HD, dout_ipu items per
  // exponent unit, dout_tp padded tokens, dout_ks supersteps of K)
  unsigned char* dout;
  int dout_tp, dout_ks, dout_ipu;
};

__device__ __forceinline__ void attn_trace(const AttnArgs& a, int i) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 4 + i] = t;
  }
}

// dynamic shared memory: K chunk | V chunk (f16 [chunk][HD] each) | scores
// [chunk] | inbox [kAttnMaxSplit][HD + 2] (rank 0: every split's acc, m, l)
template <int HD>
__global__ void __launch_bounds__(kAttnThreads) attn_decode_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) unsigned char sm[];
  __half* ks = (__half*)sm;
  __half* vs = ks + a.chunk * HD;
  float* ps = (float*)(vs + a.chunk * HD);
  float* inbox = ps + a.chunk;
  __shared__ float qs[HD];
  __shared__ float red[2];
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cluster = cg::this_cluster();
  const int split = blockIdx.x, bh = blockIdx.y;  // cluster rank == split
  const int b = bh / a.H, h = bh % a.H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int p0 = split * a.chunk;
  const int p1 = min(p0 + a.chunk, a.pos + 1);  // positions [p0, p1)
  const int pe = min(p1, a.pos);                // cached rows [p0, pe)
  attn_trace(a, 0);
  asm volatile("griddepcontrol.launch_dependents;");
  const size_t row0 = ((size_t)bh * a.ctx + p0) * HD;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (pe > p0) {
      const uint32_t bytes = (uint32_t)((pe - p0) * HD * 2);
      mbar_expect_tx(&bar, 2 * bytes);
      bulk_g2s(ks, a.kc + row0, bytes, &bar);
      bulk_g2s(vs, a.vc + row0, bytes, &bar);
    }
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  asm volatile("griddepcontrol.wait;" ::: "memory");  // q, k, v of the new token
  attn_trace(a, 1);
  const float* q = a.qkv + ((size_t)(b * 3 + 0) * a.H + h) * HD;
  const float* k = a.qkv + ((size_t)(b * 3 + 1) * a.H + h) * HD;
  const float* v = a.qkv + ((size_t)(b * 3 + 2) * a.H + h) * HD;
  constexpr int half = HD / 2;
  const bool mine = a.pos >= p0 && a.pos < p0 + a.chunk;  // this chunk holds the new token
  for (int i = tid; i < half; i += blockDim.x) {
    const float c = a.cosv[i], s = a.sinv[i];
    // rotate-half with separately rounded products (no FMA contraction: the
    // same f32 results as an elementwise implementation); q rounded through
    // f16 like the cache (the attention inputs are f16)
    auto rot_lo = [&](float x0, float x1) { return __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s)); };
    auto rot_hi = [&](float x0, float x1) { return __fadd_rn(__fmul_rn(x1, c), __fmul_rn(x0, s)); };
    qs[i] = __half2float(__float2half_rn(rot_lo(q[i], q[i + half])));
    qs[i + half] = __half2float(__float2half_rn(rot_hi(q[i], q[i + half])));
    if (mine) {
      const __half k0 = __float2half_rn(rot_lo(k[i], k[i + half]));
      const __half k1 = __float2half_rn(rot_hi(k[i], k[i + half]));
      const __half v0 = __float2half_rn(v[i]), v1 = __float2half_rn(v[i + half]);
      const int r = (a.pos - p0) * HD;
      ks[r + i] = k0;
      ks[r + i + half] = k1;
      vs[r + i] = v0;
      vs[r + i + half] = v1;
      const size_t g = ((size_t)bh * a.ctx + a.pos) * HD;
      a.kc[g + i] = k0;
      a.kc[g + i + half] = k1;
      a.vc[g + i] = v0;
      a.vc[g + i + half] = v1;
    }
  }
  if (pe > p0) mbar_wait(&bar, 0);
  __syncthreads();
  // scores: a warp per position (4 positions per pass for ILP), lanes over
  // the head dimension with vector loads of K
  const int n = p1 - p0;
  constexpr int DPL = HD / 32;  // dims per lane (4 or 2)
  float qv[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) qv[e] = qs[lane * DPL + e];
  for (int j0 = warp * 4; j0 < n; j0 += (blockDim.x / 32) * 4) {
    float acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc[u] = 0.f;
      const int j = j0 + u;
      if (j < n) {
        const __half* kr = ks + j * HD + lane * DPL;
        if constexpr (DPL == 4) {
          const uint2 raw = *(const uint2*)kr;
          const float2 k01 = __half22float2(*(const __half2*)&raw.x);
          const float2 k23 = __half22float2(*(const __half2*)&raw.y);
          acc[u] = qv[0] * k01.x + qv[1] * k01.y + qv[2] * k23.x + qv[3] * k23.y;
        } else {
          const float2 k01 = __half22float2(*(const __half2*)kr);
          acc[u] = qv[0] * k01.x + qv[1] * k01.y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (lane < 4 && j0 + lane < n) ps[j0 + lane] = (lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3]) * a.scale;
  }
  __syncthreads();
  if (warp == 0) {
    float m = -INFINITY;
    for (int j = lane; j < n; j += 32) m = fmaxf(m, ps[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int j = lane; j < n; j += 32) {
      const float e = __expf(ps[j] - m);
      ps[j] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      red[0] = m;
      red[1] = l;
    }
  }
  __syncthreads();
  // P V: thread = (dim pair, position residue class); half2 loads of V, the
  // NPH classes summed in fixed order; the partial state goes into the rank-0
  // CTA's inbox (distributed shared memory)
  constexpr int NPAIR = HD / 2, NPH = kAttnThreads / NPAIR;  // dim pairs x residue classes
  __shared__ float2 pv[kAttnThreads];
  {
    const int dp = tid % NPAIR, ph = tid / NPAIR;
    float2 acc = make_float2(0.f, 0.f);
    for (int j = ph; j < n; j += NPH) {
      const float2 vv = __half22float2(*(const __half2*)(vs + j * HD + 2 * dp));
      const float w = ps[j];
      acc.x = fmaf(w, vv.x, acc.x);
      acc.y = fmaf(w, vv.y, acc.y);
    }
    pv[tid] = acc;
  }
  __syncthreads();
  float* dst = cluster.map_shared_rank(inbox, 0) + split * (HD + 2);
  if (tid < NPAIR) {
    float2 t = pv[tid];
#pragma unroll
    for (int q = 1; q < NPH; ++q) {
      t.x += pv[q * NPAIR + tid].x;
      t.y += pv[q * NPAIR + tid].y;
    }
    dst[2 * tid] = t.x;
    dst[2 * tid + 1] = t.y;
  }
  if (tid == 0) {
    dst[HD] = red[0];
    dst[HD + 1] = red[1];
  }
  attn_trace(a, 2);
  cluster.sync();  // release the partials / acquire them in rank 0
  if (split != 0) return;
  // rank 0: combine in split order
  if (warp == 0) {
    float M = -INFINITY;
    for (int s = lane; s < a.nsplit; s += 32) M = fmaxf(M, inbox[s * (HD + 2) + HD]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.f;
    for (int s = lane; s < a.nsplit; s += 32) {
      const float e = __expf(inbox[s * (HD + 2) + HD] - M);
      ps[s] = e;  // the weights of the splits (rank 0's scores are no longer needed)
      L += e * inbox[s * (HD + 2) + HD + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) red[1] = 1.f / L;
  }
  __syncthreads();
  const float inv = red[1];
  for (int d = tid; d < HD; d += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < a.nsplit; ++s) acc += ps[s] * inbox[s * (HD + 2) + d];
    a.out[(size_t)b * a.H * HD + h * HD + d] = acc * inv;
    if (a.dout) qs[d] = acc * inv;  // (q is no longer needed)
  }
  if constexpr (HD == 128) {
    if (a.dout) {
      // this head's 128 outputs are rows [h HD, (h + 1) HD) of o_proj's K: one
      // warp digitises them (act_prep layout, item = 4 rows)
      __syncthreads();
      if (warp == 0) {
        const int kl = 32 * (lane >> 3) + 16 * ((lane & 7) >> 2) + 4 * (lane & 3);
        const float v4[4] = {qs[kl], qs[kl + 1], qs[kl + 2], qs[kl + 3]};
        const Digits d = a.dout_ipu == 32 ? digitize<32>(v4, 0xffffffffu)
                                          : digitize<16>(v4, 0xffffu << (lane & 16));
        const int it = h * (HD / 4) + lane;
        store_digits((uint32_t*)a.dout, it >> 3, b, a.dout_tp, it & 7, d);
        if ((it % a.dout_ipu) == 0)
          ((float2*)(a.dout + (size_t)a.dout_ks * 8 * a.dout_tp * 128))[(it / a.dout_ipu) * a.dout_tp + b] =
              make_float2(d.xsum, d.scale);
      }
    }
  }
  attn_trace(a, 3);
}

}  // namespace qigen

using namespace qigen;

// tuning aids: per calling thread (a knob set by one thread never changes
// another thread's launches)
static thread_local unsigned long long* g_attn_trace = nullptr;
static thread_local int g_attn_splits = 12;  // splits (cluster size) cap per head: 12 measured best at ctx 1025 (tools/attn_exp.py)
extern "C" int qigen_debug_attn_splits(int n) {
  g_attn_splits = n < 1 ? 1 : (n > kAttnMaxSplit ? kAttnMaxSplit : n);
  return QIGEN_OK;
}
extern "C" int qigen_debug_attn_trace(void* buf) {
  g_attn_trace = (unsigned long long*)buf;
  return QIGEN_OK;
}

extern "C" int64_t qigen_attn_decode_workspace_size(int64_t batch, int64_t heads, int64_t head_dim,
                                                    int64_t ctx) {
  (void)batch; (void)heads; (void)head_dim; (void)ctx;
  return 0;  // the split partials are combined on chip (cluster shared memory)
}

static int attn_decode_impl(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                            const float* cos_pos, const float* sin_pos, void* k_cache,
                            void* v_cache, int64_t ctx, int64_t pos, float scale, float* out,
                            void* workspace, int64_t workspace_bytes, void* o_digits,
                            int64_t o_group, void* stream) {
  (void)workspace; (void)workspace_bytes;
  QIGEN_CHECK_ARG(qkv && cos_pos && sin_pos && k_cache && v_cache && out, QIGEN_ERR_ARG,
                  "null pointer");
  QIGEN_CHECK_ARG(head_dim == 64 || head_dim == 128, QIGEN_ERR_UNSUPPORTED,
                  "decode attention takes head_dim 64 or 128, got %lld", (long long)head_dim);
  QIGEN_CHECK_ARG(pos >= 0 && pos < ctx && batch > 0 && heads > 0 && batch * heads < 65536,
                  QIGEN_ERR_ARG, "bad position / shape");
  // chunk: >= 64 positions (a multiple of 8), at most kAttnMaxSplit chunks (one
  // cluster); long contexts get just enough positions per CTA to fit
  const int64_t npos = pos + 1;
  int64_t chunk = std::max<int64_t>(64, ((npos + g_attn_splits - 1) / g_attn_splits + 7) / 8 * 8);
  const size_t smem = (size_t)chunk * head_dim * 2 * 2 + chunk * 4 +
                      (size_t)kAttnMaxSplit * (head_dim + 2) * 4;
  QIGEN_CHECK_ARG(smem <= 200 * 1024, QIGEN_ERR_UNSUPPORTED,
                  "decode attention: %lld positions do not fit one cluster", (long long)npos);
  AttnArgs a;
  a.qkv = qkv;
  a.cosv = cos_pos;
  a.sinv = sin_pos;
  a.kc = (__half*)k_cache;
  a.vc = (__half*)v_cache;
  a.B = (int)batch;
  a.H = (int)heads;
  a.ctx = (int)ctx;
  a.pos = (int)pos;
  a.chunk = (int)chunk;
  a.nsplit = (int)((npos + chunk - 1) / chunk);
  a.scale = scale;
  a.out = out;
  a.trace = g_attn_trace;
  a.dout = (unsigned char*)o_digits;
  if (o_digits) {
    QIGEN_CHECK_ARG(head_dim == 128 && batch <= 16 && (o_group == 64 || o_group == 128 ||
                                                       o_group == 0 || o_group % 256 == 0),
                    QIGEN_ERR_UNSUPPORTED,
                    "attention digit output: head_dim 128, <= 16 tokens, o_proj group >= 64");
    const int nb = (int)(batch + 1) / 2;
    a.dout_tp = 2 * (nb <= 1 ? 1 : nb <= 2 ? 2 : nb <= 4 ? 4 : 8);
    a.dout_ks = (int)supersteps(heads * head_dim);
    a.dout_ipu = o_group == 64 ? 16 : 32;
  }
  auto kern = head_dim == 128 ? attn_decode_kernel<128> : attn_decode_kernel<64>;
  static OncePerDevice once;
  const int cst = once.run([]() -> int {
    for (auto kf : {attn_decode_kernel<128>, attn_decode_kernel<64>}) {
      QIGEN_CUDA_RET(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024));
      QIGEN_CUDA_RET(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    return QIGEN_OK;
  });
  if (cst) return cst;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.nsplit, (unsigned)(batch * heads), 1);
  cfg.blockDim = dim3(kAttnThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = (unsigned)a.nsplit;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, kern, a));
  return QIGEN_OK;
}

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

extern "C" int qigen_attn_decode(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                                 const float* cos_pos, const float* sin_pos, void* k_cache,
                                 void* v_cache, int64_t ctx, int64_t pos, float scale, float* out,
                                 void* workspace, int64_t workspace_bytes, void* stream) {
  return attn_decode_impl(qkv, batch, heads, head_dim, cos_pos, sin_pos, k_cache, v_cache, ctx,
                          pos, scale, out, workspace, workspace_bytes, nullptr, 0, stream);
}

extern "C" int qigen_attn_decode_chain(const float* qkv, int64_t batch, int64_t heads,
                                       int64_t head_dim, const float* cos_pos,
                                       const float* sin_pos, void* k_cache, void* v_cache,
                                       int64_t ctx, int64_t pos, float scale, float* out,
                                       void* workspace, int64_t workspace_bytes, void* o_digits,
                                       int64_t o_group, void* stream) {
  QIGEN_CHECK_ARG(o_digits, QIGEN_ERR_ARG, "null digit buffer");
  return attn_decode_impl(qkv, batch, heads, head_dim, cos_pos, sin_pos, k_cache, v_cache, ctx,
                          pos, scale, out, workspace, workspace_bytes, o_digits, o_group, stream);
}
