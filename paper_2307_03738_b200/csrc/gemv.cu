// Batch-1 / small-batch quantized GEMV for sm_100a — the hot path.
//
// Replaces the reference's generated qGEMV (kernelgen.py:371-423) behind
// qgemv(pm, x, sums, threads).  Same factorisation as the
// reference (kernelgen.py:227-240, PAPER Eq. 2):
//     y_j = sum_g s_gj * ( sum_{i in g} x_i c_ij  -  z_gj * X_g )
// but the inner product sum x_i c_ij is computed EXACTLY on the integer tensor
// cores (IMMA, mma.sync.m16n8k32.u8.s8):
//   * codes c (0..2^b-1) are the u8 A operand, unpacked from the panel layout
//     with one or two shift/LOP3 per 4 codes (no int->float conversion);
//   * each activation row x (f32/f16/bf16) is converted per CTA K-chunk to a
//     fixed-point integer m = rint(x * 2^(30-E)), |m| < 2^30, split into four
//     balanced signed bytes d0..d3 (m = d0 2^24 + d1 2^16 + d2 2^8 + d3); the
//     digits are the s8 B operand, one n8 column per (token, digit);
//   * the int32 accumulators are exact; at every quantisation-group boundary
//     they are folded into f32 with the scale/zero correction (the flush).
// One warp owns a 16-column panel over the CTA's K-chunk; CTAs that share a
// panel group but own different K-chunks form a thread-block cluster and reduce
// their partial outputs through distributed shared memory in a fixed order
// (deterministic, no atomics, no workspace).  Programmatic dependent launch:
// weights are prefetched before griddepcontrol.wait, activations after it.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace qigen {

struct GemvArgs {
  const uint4* qw;
  const float2* qsz;
  const void* x;
  float* y;
  int64_t n, m, ldx, ldy;
  int KS, P, Gp, g;  // g = group size; 0 = full column
  int M;             // tokens
  int x_dtype;
  int accumulate;
  int max_steps;     // max K-steps of any chunk (smem sizing)
  int max_ranges;    // max flush ranges of any chunk
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void imma(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t idx) {
  if (dtype == QIGEN_F32) return __ldg((const float*)x + idx);
  if (dtype == QIGEN_F16) return __half2float(((const __half*)x)[idx]);
  return __bfloat162float(((const __nv_bfloat16*)x)[idx]);
}

// Fragment registers of local step sl (0..7) from the lane's superstep words.
template <int BITS>
__device__ __forceinline__ void extract(const uint4 (&w)[BITS], int sl, uint32_t (&a)[4]);

template <>
__device__ __forceinline__ void extract<4>(const uint4 (&w)[4], int sl, uint32_t (&a)[4]) {
  const uint4 u = w[sl >> 1];
  const uint32_t A = (sl & 1) ? u.z : u.x, B = (sl & 1) ? u.w : u.y;
  a[0] = A & 0x0F0F0F0Fu;
  a[1] = (A >> 4) & 0x0F0F0F0Fu;
  a[2] = B & 0x0F0F0F0Fu;
  a[3] = (B >> 4) & 0x0F0F0F0Fu;
}

template <>
__device__ __forceinline__ void extract<2>(const uint4 (&w)[2], int sl, uint32_t (&a)[4]) {
  const uint4 u = w[sl >> 2];
  const int q = sl & 3;
  const uint32_t W = q == 0 ? u.x : q == 1 ? u.y : q == 2 ? u.z : u.w;
  a[0] = W & 0x03030303u;
  a[1] = (W >> 2) & 0x03030303u;
  a[2] = (W >> 4) & 0x03030303u;
  a[3] = (W >> 6) & 0x03030303u;
}

__device__ __forceinline__ uint32_t word_of(const uint4 (&w)[3], int q) {
  const uint4 u = w[q >> 2];
  const int c = q & 3;
  return c == 0 ? u.x : c == 1 ? u.y : c == 2 ? u.z : u.w;
}

template <>
__device__ __forceinline__ void extract<3>(const uint4 (&w)[3], int sl, uint32_t (&a)[4]) {
  const int pi = sl >> 1;
  const uint32_t A = word_of(w, 3 * pi), B = word_of(w, 3 * pi + 1), C = word_of(w, 3 * pi + 2);
  if ((sl & 1) == 0) {
    a[0] = A & 0x07070707u;
    a[1] = (A >> 3) & 0x07070707u;
    a[2] = B & 0x07070707u;
    a[3] = (B >> 3) & 0x07070707u;
  } else {
    a[0] = C & 0x07070707u;
    a[1] = (C >> 3) & 0x07070707u;
    a[2] = ((A >> 6) & 0x03030303u) | ((C >> 4) & 0x04040404u);
    a[3] = ((B >> 6) & 0x03030303u) | ((C >> 5) & 0x04040404u);
  }
}

__device__ __forceinline__ int sbyte(int v) { return (int)(int8_t)(v & 0xFF); }

// Shared-memory carve-up (bytes), identical on host and device.
struct SmemLayout {
  int bfrag, xstep, xr, yp, expo, red, total;
  __host__ __device__ SmemLayout(int max_steps, int NB, int M, int max_ranges, int WPC) {
    int off = 0;
    bfrag = off; off += max_steps * NB * 32 * 8;
    xstep = off; off += max_steps * M * 8;
    xr = off;    off += max_ranges * M * 4;
    yp = off;    off += WPC * 16 * M * 4;
    expo = off;  off += 16 * 4;
    red = off;   off += 32 * 16 * 4;
    total = off;
  }
};

template <int BITS, int NB, int WPC, int D>
__global__ void __launch_bounds__(WPC * 32) gemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int T = WPC * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int S = gridDim.y, ys = blockIdx.y;
  const int ks0 = (int)((int64_t)a.KS * ys / S), ks1 = (int)((int64_t)a.KS * (ys + 1) / S);
  const int nks = ks1 - ks0;
  const int p = blockIdx.x * WPC + warp;
  const bool active = p < a.P;
  const int M = a.M;
  SmemLayout L(a.max_steps, NB, M, a.max_ranges, WPC);
  uint2* bfrag = (uint2*)(smem + L.bfrag);
  double* xstep = (double*)(smem + L.xstep);
  float* xr = (float*)(smem + L.xr);
  float* yp = (float*)(smem + L.yp);
  int* expo = (int*)(smem + L.expo);
  float* red = (float*)(smem + L.red);

  // ---- 1. weight prefetch (independent of the previous kernel) -------------
  const uint4* wp = a.qw + ((int64_t)(active ? p : 0) * a.KS + ks0) * BITS * 32 + lane;
  uint4 buf[D][BITS];
#pragma unroll
  for (int d = 0; d < D; ++d)
#pragma unroll
    for (int v = 0; v < BITS; ++v)
      buf[d][v] = (active && d < nks) ? ldg_stream(wp + (d * BITS + v) * 32) : make_uint4(0, 0, 0, 0);

  // ---- 2. PDL: wait for the producer of x; let our successor start early ---
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");

  // ---- 3. activation prologue: fixed-point digits + range sums -------------
  const int64_t k0 = (int64_t)ks0 * kSuper;
  const int nsteps = nks * 8;
  const int64_t kend = min((int64_t)ks1 * kSuper, a.n);
  {
    float mx[2 * NB];
#pragma unroll
    for (int tk = 0; tk < 2 * NB; ++tk) mx[tk] = 0.f;
    for (int64_t k = k0 + threadIdx.x; k < kend; k += T)
#pragma unroll
      for (int tk = 0; tk < 2 * NB; ++tk)
        if (tk < M) mx[tk] = fmaxf(mx[tk], fabsf(load_x(a.x, a.x_dtype, tk * a.ldx + k)));
#pragma unroll
    for (int tk = 0; tk < 2 * NB; ++tk) {
      float v = mx[tk];
      for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) red[tk * 32 + warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * NB) {
      float v = 0.f;
      for (int w = 0; w < WPC; ++w) v = fmaxf(v, red[threadIdx.x * 32 + w]);
      int e = 0;
      if (v > 0.f) frexpf(v, &e);  // v < 2^e
      expo[threadIdx.x] = e;
    }
    __syncthreads();
    // items: (token, step, half, t) -> 4 consecutive k; 8 items of a step are
    // 8 consecutive lanes so their X partial sums reduce with shuffles.
    const int items = 2 * NB * nsteps * 8;
    for (int it0 = 0; it0 < items; it0 += T) {
      const int it = it0 + threadIdx.x;
      const bool live = it < items;
      const int sub = it & 7, hh = sub >> 2, tt = sub & 3;
      const int st = (it >> 3) % nsteps, tk = (it >> 3) / nsteps;
      const int64_t kb = k0 + 32 * st + 16 * hh + 4 * tt;
      long long xsum = 0;
      uint32_t dw[4] = {0u, 0u, 0u, 0u};
      if (live && tk < M) {
        const int sh = 30 - expo[tk];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t k = kb + i;
          const float xv = (k < a.n) ? load_x(a.x, a.x_dtype, tk * a.ldx + k) : 0.f;
          const int mv = __double2int_rn(scalbn((double)xv, sh));
          xsum += mv;
          const int d3 = sbyte(mv);
          const int m1 = (mv - d3) >> 8;
          const int d2 = sbyte(m1);
          const int m2 = (m1 - d2) >> 8;
          const int d1 = sbyte(m2);
          const int d0 = (m2 - d1) >> 8;
          dw[0] |= (uint32_t)(d0 & 0xFF) << (8 * i);
          dw[1] |= (uint32_t)(d1 & 0xFF) << (8 * i);
          dw[2] |= (uint32_t)(d2 & 0xFF) << (8 * i);
          dw[3] |= (uint32_t)(d3 & 0xFF) << (8 * i);
        }
      }
      if (live) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = tk * 4 + j;
          uint32_t* dst = (uint32_t*)&bfrag[(st * NB + (col >> 3)) * 32 + (col & 7) * 4 + tt];
          dst[hh] = dw[j];
        }
      }
      for (int o = 1; o < 8; o <<= 1) xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
      if (live && sub == 0 && tk < M) xstep[st * M + tk] = (double)xsum;
    }
    __syncthreads();
    // X over each flush range (group ∩ chunk), in units of 2^(E-30)
    const int64_t ge = a.g ? a.g : (int64_t)a.KS * kSuper;
    const int gi0 = (int)(k0 / ge);
    const int gi1 = (int)(((int64_t)ks1 * kSuper - 1) / ge);
    const int nr = gi1 - gi0 + 1;
    for (int e = threadIdx.x; e < nr * M; e += T) {
      const int r = e / M, tk = e % M;
      const int64_t lo = max((int64_t)(gi0 + r) * ge, k0), hi = min((int64_t)(gi0 + r + 1) * ge, (int64_t)ks1 * kSuper);
      double s = 0.0;
      for (int st = (int)((lo - k0) / 32); st < (int)((hi - k0) / 32); ++st) s += xstep[st * M + tk];
      xr[r * M + tk] = (float)s;
    }
    __syncthreads();
  }

  // ---- 4. main loop ---------------------------------------------------------
  const int64_t ge = a.g ? a.g : (int64_t)a.KS * kSuper;
  const int steps_per_group = (int)(ge / kStep);
  const int gi0 = (int)(k0 / ge);
  int acc[NB][4];
  float yv[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    yv[nb][0] = yv[nb][1] = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[nb][q] = 0;
  }
  const float2* szp = a.qsz + (int64_t)(active ? p : 0) * a.Gp * 16;
  float2 sz0 = szp[gi0 * 16 + gq], sz1 = szp[gi0 * 16 + gq + 8];
  const float wscale = (t & 1) ? 1.f : 65536.f;
  int gcur = gi0;
  const int sg0 = ks0 * 8;  // global step index of the chunk start

  for (int s0 = 0; s0 < nks; s0 += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int s = s0 + d;
      if (s < nks) {
#pragma unroll
        for (int sl = 0; sl < 8; ++sl) {
          uint32_t af[4];
          extract<BITS>(buf[d], sl, af);
          const int st = s * 8 + sl;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) imma(acc[nb], af, bfrag[(st * NB + nb) * 32 + lane]);
          const int gstep = sg0 + st + 1;
          if ((gstep % steps_per_group) == 0 || st + 1 == nsteps) {
            // flush: y += s * (A - z * X) for range (gcur ∩ chunk)
            const int r = gcur - gi0;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              const int tk = 2 * nb + (t >> 1);
              const float X = ((t & 1) == 0 && tk < M) ? xr[r * M + tk] : 0.f;
              // digit pair (d_2h, d_2h+1) of this lane: value = (acc_hi*256 + acc_lo)*w
              const float a0 = fmaf((float)acc[nb][0], 256.f * wscale, (float)acc[nb][1] * wscale);
              const float a1 = fmaf((float)acc[nb][2], 256.f * wscale, (float)acc[nb][3] * wscale);
              const float f0 = fmaf(-sz0.y, X, a0);
              const float f1 = fmaf(-sz1.y, X, a1);
              yv[nb][0] = fmaf(sz0.x, f0, yv[nb][0]);
              yv[nb][1] = fmaf(sz1.x, f1, yv[nb][1]);
              acc[nb][0] = acc[nb][1] = acc[nb][2] = acc[nb][3] = 0;
            }
            ++gcur;
            if (gcur < a.Gp) {
              sz0 = szp[gcur * 16 + gq];
              sz1 = szp[gcur * 16 + gq + 8];
            }
          }
        }
        if (s + D < nks && active) {
#pragma unroll
          for (int v = 0; v < BITS; ++v) buf[d][v] = ldg_stream(wp + ((s + D) * BITS + v) * 32);
        }
      }
    }
  }

  // ---- 5. combine digit-pair lanes, undo the fixed-point scale -------------
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    float v0 = yv[nb][0] + __shfl_xor_sync(0xffffffffu, yv[nb][0], 1);
    float v1 = yv[nb][1] + __shfl_xor_sync(0xffffffffu, yv[nb][1], 1);
    const int tk = 2 * nb + (t >> 1);
    if ((t & 1) == 0 && tk < M) {
      const int sh = expo[tk] - 30;
      yp[(warp * 16 + gq) * M + tk] = scalbnf(v0, sh);
      yp[(warp * 16 + gq + 8) * M + tk] = scalbnf(v1, sh);
    }
  }

  // ---- 6. deterministic split-K reduction across the cluster ---------------
  const int R = WPC * 16 * M;
  const int64_t col0 = (int64_t)blockIdx.x * WPC * 16;
  if (S == 1) {
    __syncthreads();
    for (int e = threadIdx.x; e < R; e += T) {
      const int64_t col = col0 + e / M;
      const int tk = e % M;
      if (col < a.m) {
        float* dst = a.y + tk * a.ldy + col;
        *dst = a.accumulate ? *dst + yp[e] : yp[e];
      }
    }
  } else {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    const int rank = (int)cluster.block_rank();
    const int e0 = (int)((int64_t)R * rank / S), e1 = (int)((int64_t)R * (rank + 1) / S);
    for (int e = e0 + threadIdx.x; e < e1; e += T) {
      float v = 0.f;
      for (int q = 0; q < S; ++q) v += cluster.map_shared_rank(yp, q)[e];
      const int64_t col = col0 + e / M;
      const int tk = e % M;
      if (col < a.m) {
        float* dst = a.y + tk * a.ldy + col;
        *dst = a.accumulate ? *dst + v : v;
      }
    }
    cluster.sync();
  }
}

// ---------------------------------------------------------------------------
constexpr int kWPC = 4;

template <int BITS, int NB>
static int launch_nb(const GemvArgs& a, int S, cudaStream_t stream) {
  constexpr int D = BITS == 2 ? 4 : (BITS == 3 ? 3 : 2);
  auto kern = gemv_kernel<BITS, NB, kWPC, D>;
  SmemLayout L(a.max_steps, NB, a.M, a.max_ranges, kWPC);
  static int configured_bytes = 0;
  if (L.total > 48 * 1024 && L.total > configured_bytes) {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total));
    configured_bytes = L.total;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.P + kWPC - 1) / kWPC), (unsigned)S, 1);
  cfg.blockDim = dim3(kWPC * 32, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  if (S > 1) {
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = (unsigned)S;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, kern, a));
  return QIGEN_OK;
}

template <int BITS>
static int launch_bits(const GemvArgs& a, int S, cudaStream_t stream) {
  const int nb = (a.M + 1) / 2;
  if (nb <= 1) return launch_nb<BITS, 1>(a, S, stream);
  if (nb <= 2) return launch_nb<BITS, 2>(a, S, stream);
  if (nb <= 4) return launch_nb<BITS, 4>(a, S, stream);
  return launch_nb<BITS, 8>(a, S, stream);
}

static int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// K split: enough warps to cover DRAM latency (~16 per SM), at most 8 CTAs
// per cluster, at least one superstep per chunk.
int choose_splits(int64_t P, int KS, int M) {
  const int64_t target = (int64_t)sm_count() * 16;
  int64_t S = (target + P - 1) / P;
  S = std::max<int64_t>(1, std::min<int64_t>({S, 8, (int64_t)KS}));
  (void)M;
  return (int)S;
}

}  // namespace qigen

using namespace qigen;

extern "C" int qigen_gemv(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                          int64_t group, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                          float* y, int64_t ldy, int accumulate, int k_splits, void* stream) {
  QIGEN_CHECK_ARG(bits == 2 || bits == 3 || bits == 4, QIGEN_ERR_CONFIG,
                  "bits must be one of (2, 3, 4), got %d", bits);
  QIGEN_CHECK_ARG(qw && qsz && x && y, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(n > 0 && m > 0, QIGEN_ERR_ARG, "empty matrix");
  QIGEN_CHECK_ARG(group == 0 || (n % group == 0), QIGEN_ERR_CONFIG,
                  "group size %lld does not divide row count %lld", (long long)group, (long long)n);
  QIGEN_CHECK_ARG(group == 0 || group % kStep == 0, QIGEN_ERR_UNSUPPORTED,
                  "group size %lld: the GEMV needs a multiple of 32", (long long)group);
  QIGEN_CHECK_ARG(tokens >= 1 && tokens <= 16, QIGEN_ERR_UNSUPPORTED,
                  "the GEMV path takes 1..16 activation rows, got %lld", (long long)tokens);
  QIGEN_CHECK_ARG(x_dtype >= 0 && x_dtype <= 2, QIGEN_ERR_ARG, "bad x dtype %d", x_dtype);
  QIGEN_CHECK_ARG(ldx >= n && ldy >= m, QIGEN_ERR_ARG, "leading dimensions too small");
  GemvArgs a;
  a.qw = (const uint4*)qw;
  a.qsz = (const float2*)qsz;
  a.x = x;
  a.y = y;
  a.n = n;
  a.m = m;
  a.ldx = ldx;
  a.ldy = ldy;
  a.KS = (int)supersteps(n);
  a.P = (int)panels(m);
  a.Gp = (int)groups_padded(n, group);
  a.g = (int)group;
  a.M = (int)tokens;
  a.x_dtype = x_dtype;
  a.accumulate = accumulate;
  int S = k_splits > 0 ? k_splits : choose_splits(a.P, a.KS, a.M);
  QIGEN_CHECK_ARG(S >= 1 && S <= 8 && S <= a.KS, QIGEN_ERR_ARG, "k_splits %d out of range", S);
  const int max_ks = (a.KS + S - 1) / S;
  a.max_steps = max_ks * 8;
  const int64_t ge = group ? group : (int64_t)a.KS * kSuper;
  a.max_ranges = (int)((int64_t)max_ks * kSuper / ge) + 2;
  cudaStream_t s = (cudaStream_t)stream;
  switch (bits) {
    case 2: return launch_bits<2>(a, S, s);
    case 3: return launch_bits<3>(a, S, s);
    default: return launch_bits<4>(a, S, s);
  }
}
