// Small-batch (M >= 16 tokens) quantized GEMM on the 5th-generation tensor
// cores: tcgen05.mma kind::f16 with the accumulator in TMEM.
//
// north_star (c): "tensor cores (dequant to bf16 feeding mma) only at M >= 16,
// where the op really becomes a dense contraction".  We dequantize to fp16
// rather than bf16 (11-bit mantissa: w = s (c - z) keeps ~2^-11 relative error,
// activations of LLM range fit fp16), accumulate in f32 in TMEM.
//
// Swap-AB mapping: MMA M = 128 output columns (8 panels of the GPU layout), MMA
// N = NT padded tokens, K in 64-row k-blocks (4 instructions of K = 16).
//   * warps 0..7 ("dequant"): warp w streams panel w of the tile through its
//     own TMA bulk-copy ring (same stages as the GEMV: codes + (s, z)), and
//     writes w = s (c - z) as fp16 into a shared A tile in the canonical K-major
//     no-swizzle UMMA layout (8x16-byte core matrices), 4 codes per PRMT/LOP3
//     magic-number pair + HSUB2 + HFMA2;
//   * warp 8 lane 0: bulk-copies the prepared fp16 activation tile of each
//     superstep (tc_prep_kernel, same canonical layout) and issues the MMAs;
//     tcgen05.commit frees A buffers / activation stages through mbarriers;
//   * epilogue: tcgen05.ld 32x32b from TMEM, split-K partials pushed to the
//     cluster's rank-0 CTA with st.async (deterministic order), y written.
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace qigen {
namespace tc {

struct TcArgs {
  const uint4* qw;
  const float2* qsz;
  const __half* xt;  // prepared activations: [KS][NT/8][32][8 rows][8] fp16
  float* y;
  int64_t n, m, ldy;
  int KS, P, Gp, g, M, NT, accumulate, D;
};

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t mapa(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}

// UMMA shared-memory descriptor, K-major, no swizzle (canonical layout
// ((8,n),2):((16B,SBO),LBO)), sm_100 version bits = 1.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // base offset 0, layout type 0 (SWIZZLE_NONE)
}

// Instruction descriptor kind::f16: D f32, A/B f16, both K-major, M = 128.
__host__ __device__ constexpr uint32_t instr_desc(int n) {
  return (1u << 4)                        // c_format = F32
         | (0u << 7) | (0u << 10)         // a_format = b_format = F16
         | ((uint32_t)(n >> 3) << 17)     // N >> 3
         | ((uint32_t)(128 >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   saddr(bar))
               : "memory");
}

// ---- activation prep: x (f32 / f16 / bf16) -> fp16 canonical tiles -----------
// out[s][rg][c8][r][e] = x[token 8 rg + r][256 s + 8 c8 + e]; tokens >= M -> 0.
__global__ void tc_prep_kernel(const void* x, int dtype, int64_t ldx, int64_t n, int M, int NT,
                               int KS, __half* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one 8-element chunk
  const int64_t total = (int64_t)KS * NT * 32;
  if (idx >= total) return;
  const int c8 = idx % 32, tok = (idx / 32) % NT;
  const int64_t s = idx / (32 * NT);
  const int rg = tok / 8, r = tok % 8;
  const int64_t k0 = s * 256 + c8 * 8;
  __align__(16) __half v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float f = 0.f;
    if (tok < M && k0 + e < n) {
      const int64_t off = tok * ldx + k0 + e;
      f = dtype == QIGEN_F32 ? ((const float*)x)[off]
          : dtype == QIGEN_F16 ? __half2float(((const __half*)x)[off])
                               : __bfloat162float(((const __nv_bfloat16*)x)[off]);
    }
    v[e] = __float2half_rn(f);
  }
  __half* dst = out + (((s * (NT / 8) + rg) * 32 + c8) * 8 + r) * 8;
  *(uint4*)dst = *(const uint4*)v;
}

// ---- the GEMM ----------------------------------------------------------------
constexpr int kDequantWarps = 8;          // one per panel of the 128-column tile
constexpr int kThreads = (kDequantWarps + 1) * 32;
constexpr int kNA = 3;                    // A-tile buffers (64-row k-blocks)
constexpr int kATile = 128 * 64 * 2;      // bytes per A tile
constexpr int kXS = 2;                    // activation stages (supersteps)

struct TcSmem {
  int ring, a, x, bars, abars, xbars, misc, yp, total, stage, xstage;
  __host__ __device__ TcSmem(int D, int NT, int GPS, int S) {
    stage = 4 * 512 + GPS * 128;
    xstage = NT * 512;
    int off = 0;
    a = off;     off += kNA * kATile;
    x = off;     off += kXS * xstage;
    ring = off;  off += kDequantWarps * D * stage;
    bars = off;  off += kDequantWarps * D * 8;
    abars = off; off += 2 * kNA * 8;
    xbars = off; off += 2 * kXS * 8;
    misc = off;  off += 64;  // accdone, rbar, tmem base
    yp = off;    off += (S - 1) * 128 * NT * 4 + 16;
    total = off;
  }
};

template <int GPS, int NT>
__global__ void __launch_bounds__(kThreads, 1) qgemm_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int SZB = GPS * 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.y, ys = blockIdx.y;
  const int ks0 = (int)((int64_t)a.KS * ys / S), ks1 = (int)((int64_t)a.KS * (ys + 1) / S);
  const int nks = ks1 - ks0;
  const int D = a.D;
  TcSmem L(D, NT, GPS, S);
  uint64_t* abar_full = (uint64_t*)(smem + L.abars);
  uint64_t* abar_empty = abar_full + kNA;
  uint64_t* xbar_full = (uint64_t*)(smem + L.xbars);
  uint64_t* xbar_empty = xbar_full + kXS;
  uint64_t* accdone = (uint64_t*)(smem + L.misc);
  uint64_t* rbar = accdone + 1;
  uint32_t* tmem_slot = (uint32_t*)(accdone + 2);
  float* yp = (float*)(smem + L.yp);
  const int R = 128 * NT;

  // ---- setup ------------------------------------------------------------------
  const int p = blockIdx.x * kDequantWarps + warp;  // panel of a dequant warp
  const bool active = warp < kDequantWarps && p < a.P;
  unsigned char* ring = smem + L.ring + warp * D * L.stage;
  uint64_t* wbars = (uint64_t*)(smem + L.bars) + warp * D;
  const char* wsrc = (const char*)(a.qw + (int64_t)(active ? p : 0) * a.KS * 4 * 32);
  const char* zsrc = (const char*)(a.qsz + (int64_t)(active ? p : 0) * a.Gp * 16);
  auto issue_w = [&](int s) {
    const int slot = s % D;
    unsigned char* dst = ring + slot * L.stage;
    mbar_expect_tx(&wbars[slot], (uint32_t)L.stage);
    bulk_g2s(dst, wsrc + (int64_t)(ks0 + s) * 4 * 512, 4 * 512, &wbars[slot]);
    if (SZB) bulk_g2s(dst + 4 * 512, zsrc + (int64_t)(ks0 + s) * SZB, SZB, &wbars[slot]);
  };
  if (warp < kDequantWarps && lane == 0) {
    for (int i = 0; i < D; ++i) mbar_init(&wbars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (active)
      for (int s = 0; s < min(D, nks); ++s) issue_w(s);
  }
  if (warp == kDequantWarps) {
    if (lane == 0) {
      for (int i = 0; i < kNA; ++i) {
        mbar_init(&abar_full[i], kDequantWarps);
        mbar_init(&abar_empty[i], 1);
      }
      for (int i = 0; i < kXS; ++i) {
        mbar_init(&xbar_full[i], 1);
        mbar_init(&xbar_empty[i], 1);
      }
      mbar_init(accdone, 1);
      if (S > 1) {
        mbar_init(rbar, 1);
        mbar_expect_tx(rbar, (uint32_t)((S - 1) * 128 * a.M * 4));  // real tokens only
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t cols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  asm volatile("griddepcontrol.wait;" ::: "memory");  // activations come from the prep kernel

  const int nkb = nks * 4;  // 64-row k-blocks in this chunk
  if (warp == kDequantWarps) {
    // ---- activation producer + MMA issuer (one thread) -------------------------
    if (lane == 0) {
      const uint32_t idesc = instr_desc(NT);
      auto issue_x = [&](int s) {
        const int slot = s % kXS;
        mbar_expect_tx(&xbar_full[slot], (uint32_t)L.xstage);
        bulk_g2s(smem + L.x + slot * L.xstage, a.xt + (size_t)(ks0 + s) * NT * 256, L.xstage,
                 &xbar_full[slot]);
      };
      for (int s = 0; s < min(kXS, nks); ++s) issue_x(s);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb >> 2, buf = kb % kNA, xs = s % kXS;
        if ((kb & 3) == 0) mbar_wait(&xbar_full[xs], (uint32_t)((s / kXS) & 1));
        mbar_wait(&abar_full[buf], (uint32_t)((kb / kNA) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_base = saddr(smem + L.a + buf * kATile);
        const uint32_t x_base = saddr(smem + L.x + xs * L.xstage) + (kb & 3) * 8 * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // A: core (rg, c8) at (rg*8 + c8)*128; B: core (rg, c8) at (rg*32 + c8)*128
          const uint64_t ad = smem_desc(a_base + 2 * q * 128, 128, 8 * 128);
          const uint64_t bd = smem_desc(x_base + 2 * q * 128, 128, 32 * 128);
          mma_f16(tmem, ad, bd, idesc, (kb | q) ? 1u : 0u);
        }
        mma_commit(&abar_empty[buf]);
        if ((kb & 3) == 3) {
          mma_commit(&xbar_empty[xs]);
          if (s + kXS < nks) {
            mbar_wait(&xbar_empty[xs], (uint32_t)((s / kXS) & 1));
            issue_x(s + kXS);
          }
        }
      }
      mma_commit(accdone);
    }
    __syncwarp();
  } else {
    // ---- dequant warps: panel `warp` of the tile, 16 rows x 64 k per k-block ---
    const int gq = lane >> 2, t = lane & 3;
    const __half2 k1024 = __half2half2(__float2half(1024.f));
    int slot = 0;
    uint32_t phase = 0;
    for (int s = 0; s < nks; ++s) {
      uint4 w[4] = {};
      const float2* szs = nullptr;
      if (active) {
        mbar_wait(&wbars[slot], phase);
        const unsigned char* stg = ring + slot * L.stage;
#pragma unroll
        for (int v = 0; v < 4; ++v) w[v] = ((const uint4*)stg)[v * 32 + lane];
        szs = (const float2*)(stg + 4 * 512);
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int kb = s * 4 + kk, buf = kb % kNA;
        if (kb >= kNA) mbar_wait(&abar_empty[buf], (uint32_t)(((kb / kNA) - 1) & 1));
        unsigned char* at = smem + L.a + buf * kATile;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // the two 32-row steps of the k-block
          const int sl = 2 * kk + h;
          const uint4 u = w[sl >> 1];
          const uint32_t A = (sl & 1) ? u.z : u.x, B = (sl & 1) ? u.w : u.y;
          const int gi = GPS > 0 ? (32 * sl) / (256 / GPS) : 0;  // group within superstep
          float2 sz0 = make_float2(0.f, 0.f), sz1 = sz0;
          if (active && GPS > 0) {
            sz0 = szs[gi * 16 + gq];
            sz1 = szs[gi * 16 + gq + 8];
          }
          // rows gq (low nibbles) and gq + 8 (high nibbles, codes x16)
          const __half2 s0 = __half2half2(__float2half_rn(sz0.x));
          const __half2 n0 = __half2half2(__float2half_rn(-sz0.x * sz0.y));
          const __half2 s1 = __half2half2(__float2half_rn(sz1.x * (1.f / 16.f)));
          const __half2 n1 = __half2half2(__float2half_rn(-sz1.x * sz1.y));
#pragma unroll
          for (int half_k = 0; half_k < 2; ++half_k) {  // word A: k 4t.., word B: k 16+4t..
            const uint32_t W = half_k ? B : A;
            const uint32_t p01 = __byte_perm(W, 0, 0x4140), p23 = __byte_perm(W, 0, 0x4342);
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
              const uint32_t msk = hi ? 0x00F000F0u : 0x000F000Fu;
              uint32_t q01 = (p01 & msk) | 0x64006400u, q23 = (p23 & msk) | 0x64006400u;
              __half2 c01 = __hsub2(*(__half2*)&q01, k1024), c23 = __hsub2(*(__half2*)&q23, k1024);
              c01 = __hfma2(c01, hi ? s1 : s0, hi ? n1 : n0);
              c23 = __hfma2(c23, hi ? s1 : s0, hi ? n1 : n0);
              const int row = warp * 16 + gq + 8 * hi;
              const int kl = 32 * h + 16 * half_k + 4 * t;  // k within the 64-row block
              const int off = ((row >> 3) * 8 + (kl >> 3)) * 128 + (row & 7) * 16 + (kl & 7) * 2;
              uint2 v2;
              v2.x = *(uint32_t*)&c01;
              v2.y = *(uint32_t*)&c23;
              *(uint2*)(at + off) = v2;
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&abar_full[buf]);
      }
      __syncwarp();
      if (active && lane == 0 && s + D < nks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_w(s + D);
      }
      if (++slot == D) {
        slot = 0;
        phase ^= 1u;
      }
    }
  }

  // ---- epilogue: TMEM -> registers -> split-K reduction -> y ---------------------
  asm volatile("griddepcontrol.launch_dependents;");
  const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
  if (S > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp < 4) {
    mbar_wait(accdone, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (rank == 0 && S > 1) mbar_wait(rbar, 0);
    const int row = warp * 32 + lane;  // output column within the tile
    const int64_t col = (int64_t)blockIdx.x * 128 + row;
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 8) {
      uint32_t r[8];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int tok = c0 + j;
        if (tok >= a.M) continue;
        float v = __uint_as_float(r[j]);
        const int e = tok * 128 + row;
        if (rank > 0) {
          st_async(mapa(yp + (rank - 1) * R + e, 0), v, mapa(rbar, 0));
        } else {
          for (int q = 1; q < S; ++q) v += yp[(q - 1) * R + e];
          if (col < a.m) {
            float* dst = a.y + tok * a.ldy + col;
            *dst = a.accumulate ? *dst + v : v;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kDequantWarps) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t cols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}

int sm_count_tc() {
  static int c = 0;
  if (!c) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d);
  }
  return c;
}

template <int GPS, int NT>
static int launch(TcArgs& a, int req_S, void* ws, cudaStream_t stream, const void* x, int dtype,
                  int64_t ldx) {
  auto kern = qgemm_tc_kernel<GPS, NT>;
  static bool configured = false;
  if (!configured) {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  const int cols = (a.P + kDequantWarps - 1) / kDequantWarps;
  int S = req_S;
  if (S <= 0) {  // about one CTA per SM, at most 8 per cluster
    S = std::max(1, std::min({sm_count_tc() / std::max(cols, 1), 8, a.KS}));
  }
  auto plan = [&](int s_) {
    const int max_ks = (a.KS + s_ - 1) / s_;
    TcSmem L0(0, NT, GPS, s_);
    const int per = 4 * 512 + GPS * 128;
    a.D = std::max(1, std::min(max_ks, (220 * 1024 - L0.total) / (kDequantWarps * per)));
    a.D = std::min(a.D, 3);
    return TcSmem(a.D, NT, GPS, s_);
  };
  TcSmem L = plan(S);
  while (L.total > 227 * 1024 && S > 1) L = plan(--S);
  QIGEN_CHECK_ARG(L.total <= 227 * 1024, QIGEN_ERR_UNSUPPORTED,
                  "tensor-core GEMM needs %d bytes of shared memory", L.total);
  // prep: activations -> fp16 canonical tiles in the workspace
  a.xt = (const __half*)ws;
  {
    const int64_t total = (int64_t)a.KS * NT * 32;
    cudaLaunchConfig_t pc = {};
    pc.gridDim = dim3((unsigned)((total + 255) / 256), 1, 1);
    pc.blockDim = dim3(256, 1, 1);
    pc.stream = stream;
    cudaLaunchAttribute pa;
    pa.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pa.val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = &pa;
    pc.numAttrs = 1;
    QIGEN_CUDA_RET(cudaLaunchKernelEx(&pc, tc_prep_kernel, x, dtype, ldx, a.n, a.M, NT, a.KS,
                                      (__half*)ws));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cols, (unsigned)S, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
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

template <int GPS>
static int launch_nt(TcArgs& a, int S, void* ws, cudaStream_t st, const void* x, int dt, int64_t ldx) {
  if (a.NT <= 16) return launch<GPS, 16>(a, S, ws, st, x, dt, ldx);
  if (a.NT <= 32) return launch<GPS, 32>(a, S, ws, st, x, dt, ldx);
  if (a.NT <= 64) return launch<GPS, 64>(a, S, ws, st, x, dt, ldx);
  if (a.NT <= 128) return launch<GPS, 128>(a, S, ws, st, x, dt, ldx);
  return launch<GPS, 256>(a, S, ws, st, x, dt, ldx);
}

}  // namespace tc
}  // namespace qigen

using namespace qigen;

extern "C" int64_t qigen_gemm_tc_workspace_size(int64_t n, int64_t tokens) {
  const int64_t nt = tokens <= 16 ? 16 : tokens <= 32 ? 32 : tokens <= 64 ? 64 : tokens <= 128 ? 128 : 256;
  return supersteps(n) * nt * 256 * 2;
}

extern "C" int qigen_gemm_tc(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                             int64_t group, const void* x, int x_dtype, int64_t tokens,
                             int64_t ldx, float* y, int64_t ldy, int accumulate, int k_splits,
                             void* workspace, int64_t workspace_bytes, void* stream) {
  QIGEN_CHECK_ARG(bits == 4, QIGEN_ERR_UNSUPPORTED, "tensor-core path: 4-bit weights only (got %d)",
                  bits);
  QIGEN_CHECK_ARG(group == 32 || group == 64 || group == 128 || group == 256,
                  QIGEN_ERR_UNSUPPORTED, "tensor-core path: group size 32..256 dividing 256");
  QIGEN_CHECK_ARG(n % group == 0, QIGEN_ERR_CONFIG, "group size does not divide n");
  QIGEN_CHECK_ARG(tokens >= 1 && tokens <= 256, QIGEN_ERR_UNSUPPORTED, "1..256 tokens");
  QIGEN_CHECK_ARG(qw && qsz && x && y && workspace, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(workspace_bytes >= qigen_gemm_tc_workspace_size(n, tokens), QIGEN_ERR_ARG,
                  "workspace too small");
  QIGEN_CHECK_ARG(ldx >= n && ldy >= m, QIGEN_ERR_ARG, "leading dimensions too small");
  tc::TcArgs a = {};
  a.qw = (const uint4*)qw;
  a.qsz = (const float2*)qsz;
  a.y = y;
  a.n = n;
  a.m = m;
  a.ldy = ldy;
  a.KS = (int)supersteps(n);
  a.P = (int)panels(m);
  a.Gp = (int)groups_padded(n, group);
  a.g = (int)group;
  a.M = (int)tokens;
  a.NT = tokens <= 16 ? 16 : tokens <= 32 ? 32 : tokens <= 64 ? 64 : tokens <= 128 ? 128 : 256;
  a.accumulate = accumulate;
  cudaStream_t s = (cudaStream_t)stream;
  switch (group) {
    case 32: return tc::launch_nt<8>(a, k_splits, workspace, s, x, x_dtype, ldx);
    case 64: return tc::launch_nt<4>(a, k_splits, workspace, s, x, x_dtype, ldx);
    case 128: return tc::launch_nt<2>(a, k_splits, workspace, s, x, x_dtype, ldx);
    default: return tc::launch_nt<1>(a, k_splits, workspace, s, x, x_dtype, ldx);
  }
}
