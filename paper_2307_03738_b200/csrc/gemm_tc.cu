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
//   * warps 0..15 ("dequant", two per panel: even / odd k-blocks): read the
//     panel's superstep stage (codes + (s, z)) from a TMA bulk-copy ring and
//     write w = s (c - z) as fp16 straight into TMEM (tcgen05.st 16x256b: the
//     panel layout's lane fragments are exactly that shape's thread fragments),
//     4 codes per PRMT/LOP3 magic-number pair + HSUB2 + HFMA2.  The A operand
//     never touches shared memory: TMEM holds 8 A tiles of 32 columns;
//   * warp 16 lane 0: issues tcgen05.mma (A from TMEM, activations from smem);
//     tcgen05.commit frees A tiles / activation stages through mbarriers;
//   * warp 17 lane 0: bulk-copies the prepared fp16 activation tile of each
//     k-block (tc_prep_kernel, canonical K-major no-swizzle layout);
//   * warp 18 lane 0: keeps every panel's weight ring full;
//   * epilogue: tcgen05.ld 32x32b from TMEM, split-K partials pushed to the
//     cluster's rank-0 CTA with one bulk DSMEM copy each, y written.
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace qigen {
extern thread_local unsigned long long* g_trace;
static thread_local int g_tc_dbg = 0;  // tuning aid, per calling thread
namespace tc {

struct TcArgs {
  const uint4* qw;
  const float2* qsz;
  const __half* xt;  // prepared activations: [KS][NT/8][32][8 rows][8] fp16
  float* y;
  int64_t n, m, ldy;
  int KS, P, Gp, g, M, NT, accumulate, D;
  unsigned long long* trace;
  int dbg;  // tuning: 1 = no A-tile stores, 2 = no MMAs, 3 = no activation tiles (+2),
            // 4 = MMA does not wait for the dequant warps (+2)
};

__device__ __forceinline__ void tpoint(const TcArgs& a, int i) {
  if (a.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + i] = t;
  }
}

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
// Wait, and (tuning builds, -DQIGEN_TC_WAIT_TRACE) accumulate the cycles spent.
__device__ __forceinline__ void mbar_wait_t(uint64_t* b, uint32_t parity, long long& acc) {
#ifdef QIGEN_TC_WAIT_TRACE
  const long long t0 = clock64();
  mbar_wait(b, parity);
  acc += clock64() - t0;
#else
  (void)acc;
  mbar_wait(b, parity);
#endif
}
// (a & b) | c in one LOP3: ptxas folds at most one immediate per LOP3, so the two
// constants arrive as registers
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// One lane of a converged warp.  tcgen05.mma issued from a divergent single
// thread (if (lane == 0)) costs ~370 cycles per instruction on B200 vs 25-128
// converged (tools/ubench/umma_rate.cu), so every issuing loop runs warp-wide.
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e != 0;
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

// D[tmem] (+)= A[tmem_a] (TMEM, 128 lanes x 16 fp16 of K) * B[smem descriptor]
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem, uint32_t ta, uint64_t bd, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
      "r"(ta), "l"(bd), "r"(idesc), "r"(acc));
}
// 16 TMEM lanes x 32 columns: thread (gq, t) holds lanes gq / gq + 8, columns 8 i + 2 t + {0, 1}
__device__ __forceinline__ void tmem_st_16x256b_x4(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   saddr(bar))
               : "memory");
}

// ---- activation prep: x (f32 / f16 / bf16) -> fp16 canonical tiles -----------
// Per 64-row k-block kb: out[kb][rg][c8][r][e] = x[token 8 rg + r][64 kb + 8 c8 + e]
// (canonical K-major core matrices, one contiguous NT x 128-byte tile per k-block);
// tokens >= M and rows >= n are zero.
__global__ void tc_prep_kernel(const void* x, int dtype, int64_t ldx, int64_t n, int M, int NT,
                               int KB, __half* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // one 8-element chunk
  const int64_t total = (int64_t)KB * NT * 8;
  if (idx >= total) return;
  const int c8 = idx % 8, tok = (idx / 8) % NT;
  const int64_t kb = idx / (8 * NT);
  const int rg = tok / 8, r = tok % 8;
  const int64_t k0 = kb * 64 + c8 * 8;
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
  __half* dst = out + (((kb * (NT / 8) + rg) * 8 + c8) * 8 + r) * 8;
  *(uint4*)dst = *(const uint4*)v;
}

// ---- the GEMM ----------------------------------------------------------------
constexpr int kPanels = 8;                 // 16-column panels per 128-column tile
constexpr int kDequantWarps = 16;          // two per panel (even / odd k-blocks)
constexpr int kMmaWarp = kDequantWarps;    // + TMEM allocation
constexpr int kXWarp = kDequantWarps + 1;  // activation producer
constexpr int kWWarp = kDequantWarps + 2;  // weight producer
constexpr int kThreads = (kDequantWarps + 3) * 32;
// The MMA warp works in groups of G 64-row k-blocks (one wait pair + 4 G MMAs +
// one commit per group; per-k-block handshakes left the MMA warp latency-bound).
// TMEM: accumulator in columns [0, acc_cols), then NGS A-group slots of 32 G columns.
__host__ __device__ constexpr int tc_group(int NT) { return NT <= 64 ? 4 : 2; }
__host__ __device__ constexpr int tc_acc_cols(int NT) { return NT <= 128 ? 128 : 256; }
__host__ __device__ constexpr int tc_slots(int NT) {
  return (512 - tc_acc_cols(NT)) / (32 * tc_group(NT));
}

struct TcSmem {
  int x, ring, wfull, wempty, abars, xbars, misc, inbox, total, stage, xstage, XS;
  __host__ __device__ TcSmem(int D, int NT, int GPS, int S, int M) {
    stage = 4 * 512 + GPS * 128;
    xstage = tc_group(NT) * NT * 128;  // activation tiles of one MMA group
    // XS <= NGS: an activation stage is released by the same tcgen05.commit as the
    // A slot of its group (abar_empty), at most one phase ahead of its waiter
    XS = 96 * 1024 / xstage;
    if (XS > tc_slots(NT)) XS = tc_slots(NT);
    if (XS < 2) XS = 2;
    int off = 0;
    x = off;      off += XS * xstage;           // x ring + weight ring double as the
    ring = off;   off += kPanels * D * stage;   // epilogue staging (M x 128 f32)
    if (off < M * 512) off = M * 512;
    off = (off + 15) & ~15;
    wfull = off;  off += kPanels * D * 8;
    wempty = off; off += D * 8;
    abars = off;  off += 2 * tc_slots(NT) * 8;
    xbars = off;  off += XS * 8;
    off = (off + 15) & ~15;
    misc = off;   off += 64;  // accdone, rbar, tmem base
    off = (off + 127) & ~127;  // bulk-copy destination
    inbox = off;  off += (S - 1) * 128 * M * 4;
    total = off;
  }
};

template <int GPS, int NT>
__global__ void __launch_bounds__(kThreads, 1) qgemm_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int SZB = GPS * 128;
  constexpr int G = tc_group(NT), NGS = tc_slots(NT), KPW = G / 2;  // KPW: k-blocks per warp
  constexpr uint32_t kACol = tc_acc_cols(NT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = gridDim.y, ys = blockIdx.y;
  const int ks0 = (int)((int64_t)a.KS * ys / S), ks1 = (int)((int64_t)a.KS * (ys + 1) / S);
  const int nks = ks1 - ks0;
  const int D = a.D, M = a.M;
  TcSmem L(D, NT, GPS, S, M);
  const int XS = L.XS;
  uint64_t* abar_full = (uint64_t*)(smem + L.abars);
  uint64_t* abar_empty = abar_full + NGS;
  uint64_t* xbar_full = (uint64_t*)(smem + L.xbars);
  uint64_t* accdone = (uint64_t*)(smem + L.misc);
  uint64_t* rbar = accdone + 1;
  uint32_t* tmem_slot = (uint32_t*)(accdone + 2);
  const int R = 128 * M;  // partial outputs of this CTA (real tokens only)

  // ---- setup ------------------------------------------------------------------
  // dequant warp w may only touch TMEM lanes 32 (w % 4) ..: panel 2 (w % 4) + (w / 4) % 2
  const int pn = 2 * (warp & 3) + ((warp >> 2) & 1), par = (warp >> 3) & 1;
  const int p = blockIdx.x * kPanels + pn;
  const bool active = warp < kDequantWarps && p < a.P;
  unsigned char* ring = smem + L.ring + pn * D * L.stage;
  uint64_t* wfull = (uint64_t*)(smem + L.wfull) + pn * D;
  uint64_t* wempty = (uint64_t*)(smem + L.wempty);  // per slot, all 16 dequant warps release
  auto issue_w = [&](int pp, int s) {  // weight producer: superstep s of panel pp
    const int slot = s % D;
    const bool act = blockIdx.x * kPanels + pp < a.P;
    unsigned char* dst = smem + L.ring + (pp * D + slot) * L.stage;
    uint64_t* full = (uint64_t*)(smem + L.wfull) + pp * D + slot;
    const int64_t pg = act ? blockIdx.x * kPanels + pp : 0;
    const char* ws = (const char*)(a.qw + pg * a.KS * 4 * 32);
    const char* zs = (const char*)(a.qsz + pg * a.Gp * 16);
    mbar_expect_tx(full, (uint32_t)L.stage);
    bulk_g2s(dst, ws + (int64_t)(ks0 + s) * 4 * 512, 4 * 512, full);
    if (SZB) bulk_g2s(dst + 4 * 512, zs + (int64_t)(ks0 + s) * SZB, SZB, full);
  };
  if (warp == kWWarp && lane == 0) {
    for (int i = 0; i < kPanels * D; ++i) mbar_init((uint64_t*)(smem + L.wfull) + i, 1);
    for (int i = 0; i < D; ++i) mbar_init((uint64_t*)(smem + L.wempty) + i, kDequantWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < min(D, nks); ++s)
      for (int pp = 0; pp < kPanels; ++pp) issue_w(pp, s);
  }
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int i = 0; i < NGS; ++i) {
        mbar_init(&abar_full[i], kDequantWarps);  // every dequant warp writes into a group
        mbar_init(&abar_empty[i], 1);
      }
      for (int i = 0; i < XS; ++i) mbar_init(&xbar_full[i], 1);
      mbar_init(accdone, 1);
      if (S > 1) {
        mbar_init(rbar, 1);
        mbar_expect_tx(rbar, (uint32_t)((S - 1) * R * 4));
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     saddr(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) tpoint(a, 0);

  asm volatile("griddepcontrol.wait;" ::: "memory");  // activations come from the prep kernel
  if (threadIdx.x == 0) tpoint(a, 1);

  const int ngr = nks * 4 / G;  // MMA groups in this chunk
  long long wt0 = 0, wt1 = 0, wt2 = 0;  // cycles in mbarrier waits (-DQIGEN_TC_WAIT_TRACE)
  (void)wt2;
#ifdef QIGEN_TC_WAIT_TRACE
  long long tloop = clock64();
#endif
  if (warp == kWWarp) {
    // ---- weight stages: one wait per superstep, lane pp refills panel pp ---------
    // (a serial per-panel wait + issue loop in one warp costs ~170 ns per
    // iteration and capped the weight stream at ~2 TB/s: tools/ubench/bulk_bw.cu)
    for (int s = D; s < nks; ++s) {
      mbar_wait_t(wempty + s % D, (uint32_t)(((s / D) - 1) & 1), wt0);
      if (lane < kPanels) issue_w(lane, s);
      __syncwarp();
    }
  } else if (warp == kXWarp) {
    // ---- activation tiles, one stage per MMA group -----------------------------------
    for (int gi = 0; gi < (a.dbg == 3 ? 0 : ngr); ++gi) {
      const int slot = gi % XS;
      if (gi >= XS) {  // the MMAs of group gi - XS are done with this stage
        const int pg = gi - XS;
        mbar_wait_t(&abar_empty[pg % NGS], (uint32_t)((pg / NGS) & 1), wt0);
      }
      if (elect_one()) {
        mbar_expect_tx(&xbar_full[slot], (uint32_t)L.xstage);
        bulk_g2s(smem + L.x + slot * L.xstage, a.xt + ((size_t)ks0 * 4 + (size_t)gi * G) * NT * 64,
                 (uint32_t)L.xstage, &xbar_full[slot]);
      }
      __syncwarp();
    }
  } else if (warp == kMmaWarp) {
    // ---- MMA issue: the whole warp waits, one elected lane issues ----------------
    const uint32_t idesc = instr_desc(NT);
    for (int gi = 0; gi < ngr; ++gi) {
      const int buf = gi % NGS, xs = gi % XS;
      if (a.dbg != 3) mbar_wait_t(&xbar_full[xs], (uint32_t)((gi / XS) & 1), wt0);
      if (a.dbg != 4) mbar_wait_t(&abar_full[buf], (uint32_t)((gi / NGS) & 1), wt1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ta = tmem + kACol + 32 * G * buf;
      const uint32_t x_base = saddr(smem + L.x + xs * L.xstage);
#ifdef QIGEN_TC_WAIT_TRACE
      const long long ti0 = clock64();
#endif
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < G; ++kk)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (a.dbg == 2) break;
            // activation tile kk: core matrix (rg, c8) at (rg * 8 + c8) * 128 bytes
            const uint64_t bd = smem_desc(x_base + kk * NT * 128 + 2 * q * 128, 128, 8 * 128);
            mma_f16_ts(tmem, ta + 32 * kk + 8 * q, bd, idesc, (gi | kk | q) ? 1u : 0u);
          }
        mma_commit(&abar_empty[buf]);  // frees A slot gi and activation stage gi % XS
      }
      __syncwarp();
#ifdef QIGEN_TC_WAIT_TRACE
      wt2 += clock64() - ti0;
#endif
    }
    if (elect_one()) mma_commit(accdone);
    __syncwarp();
    if (lane == 0) tpoint(a, 3);
  } else {
    // ---- dequant warps: 16 rows x 64 k of panel pn for k-blocks of parity par ---
    const int gq = lane >> 2;
    const __half2 k1024 = __half2half2(__float2half(1024.f));
    // opaque to the constant folder so that and_or keeps them in registers
    uint32_t mlo = 0x000F000Fu, mhi = 0x00F000F0u, magic = 0x64006400u;
    asm volatile("" : "+r"(mlo), "+r"(mhi), "+r"(magic));
    int slot = 0;
    uint32_t phase = 0;
    for (int s = 0; s < nks; ++s) {
      uint4 w[2] = {};
      float2 szr[4][2];
      if (active) {
        mbar_wait_t(&wfull[slot], phase, wt0);
        const unsigned char* stg = ring + slot * L.stage;
        // k-block kk = steps 2 kk, 2 kk + 1 = uint4 kk of the stage; this warp: kk = par, par + 2
        w[0] = ((const uint4*)stg)[par * 32 + lane];
        w[1] = ((const uint4*)stg)[(par + 2) * 32 + lane];
        const float2* szs = (const float2*)(stg + 4 * 512);
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {  // the two steps of each of this warp's k-blocks
          const int step = 4 * (sl >> 1) + 2 * par + (sl & 1);
          const int gi = GPS > 0 ? (32 * step) / (256 / GPS) : 0;
          szr[sl][0] = GPS > 0 ? szs[gi * 16 + gq] : make_float2(0.f, 0.f);
          szr[sl][1] = GPS > 0 ? szs[gi * 16 + gq + 8] : make_float2(0.f, 0.f);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&wempty[slot]);
      } else {
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) szr[sl][0] = szr[sl][1] = make_float2(0.f, 0.f);
        if (lane == 0) mbar_arrive(&wempty[slot]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int kk = par + 2 * j, kb = s * 4 + kk, gi = kb / G, buf = gi % NGS;
        uint32_t r[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // the two 32-row steps of the k-block
          const uint32_t A = h ? w[j].z : w[j].x, B = h ? w[j].w : w[j].y;
          const float2 sz0 = szr[2 * j + h][0], sz1 = szr[2 * j + h][1];
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
              const uint32_t msk = hi ? mhi : mlo;
              uint32_t q01 = and_or(p01, msk, magic), q23 = and_or(p23, msk, magic);
              __half2 c01 = __hsub2(*(__half2*)&q01, k1024), c23 = __hsub2(*(__half2*)&q23, k1024);
              c01 = __hfma2(c01, hi ? s1 : s0, hi ? n1 : n0);
              c23 = __hfma2(c23, hi ? s1 : s0, hi ? n1 : n0);
              // 16-k slab 2 h + half_k -> TMEM columns 8 (2 h + half_k) + 2 t + {0, 1}
              r[4 * (2 * h + half_k) + 2 * hi] = *(uint32_t*)&c01;
              r[4 * (2 * h + half_k) + 2 * hi + 1] = *(uint32_t*)&c23;
            }
          }
        }
        if (j % KPW == 0 && gi >= NGS) {  // first k-block of this warp in group gi
          mbar_wait_t(&abar_empty[buf], (uint32_t)(((gi / NGS) - 1) & 1), wt1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        if (a.dbg != 1)
          tmem_st_16x256b_x4(
              tmem + ((uint32_t)(16 * pn) << 16) + kACol + 32 * (G * buf + kb % G), r);
        if (j % KPW == KPW - 1) {  // last one: publish to the MMA warp
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(&abar_full[buf]);
        }
      }
      if (++slot == D) {
        slot = 0;
        phase ^= 1u;
      }
    }
    if (threadIdx.x == 0) tpoint(a, 2);
  }

#ifdef QIGEN_TC_WAIT_TRACE
  if (a.trace && lane == 0) {
    tloop = clock64() - tloop;
    const size_t base = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16;
    int sl = -1;
    if (warp == 0) sl = 6;
    else if (warp == kPanels) sl = 8;
    else if (warp == kMmaWarp) sl = 10;
    else if (warp == kWWarp) sl = 12;
    else if (warp == kXWarp) sl = 13;
    if (sl >= 0) {
      a.trace[base + sl] = wt0;
      if (sl <= 10) a.trace[base + sl + 1] = wt1;
      if (warp == 0) a.trace[base + 14] = tloop;
      if (warp == kMmaWarp) a.trace[base + 15] = wt2;
    }
  }
#endif
  // ---- epilogue: TMEM -> staging (smem) -> split-K reduction -> y ----------------
  asm volatile("griddepcontrol.launch_dependents;");
  const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
  float* stg = (float*)(smem + L.x);  // [token][128 rows], the rings are drained now
  if (warp < kDequantWarps) {
    mbar_wait(accdone, 0);
    if (threadIdx.x == 0) tpoint(a, 4);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = (warp & 3) * 32 + lane;
    const int cq = NT / 4;  // token columns per quarter
    const int c_lo = (warp >> 2) * cq;
#pragma unroll 1
    for (int c0 = c_lo; c0 < c_lo + cq; c0 += 4) {
      uint32_t r[4];
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c0 + j < M) stg[(c0 + j) * 128 + row] = __uint_as_float(r[j]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (S > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank > 0) {
    if (threadIdx.x == 0) {  // one bulk copy of the partial tile into rank 0's inbox
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(mapa(smem + L.inbox + (size_t)(rank - 1) * R * 4, 0)),
          "r"(saddr(stg)), "r"((uint32_t)(R * 4)), "r"(mapa(rbar, 0))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  } else {
    if (S > 1) mbar_wait(rbar, 0);
    const float* inbox = (const float*)(smem + L.inbox);
    const int64_t col0 = (int64_t)blockIdx.x * 128;
    for (int e = threadIdx.x; e < R; e += kThreads) {
      float v = stg[e];
      for (int q = 1; q < S; ++q) v += inbox[(q - 1) * R + e];
      const int tok = e / 128, row = e % 128;
      const int64_t col = col0 + row;
      if (col < a.m) {
        float* dst = a.y + tok * a.ldy + col;
        *dst = a.accumulate ? *dst + v : v;
      }
    }
  }
  if (threadIdx.x == 0) tpoint(a, 5);
  __syncthreads();
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int sm_count_tc() {
  int d = 0, c = 148;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, d);
  return c;
}

template <int GPS, int NT>
static int launch(TcArgs& a, int req_S, void* ws, cudaStream_t stream, const void* x, int dtype,
                  int64_t ldx) {
  auto kern = qgemm_tc_kernel<GPS, NT>;
  static OncePerDevice once;
  const int cst = once.run([&]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return QIGEN_OK;
  });
  if (cst) return cst;
  const int cols = (a.P + kPanels - 1) / kPanels;
  int S = req_S;
  if (S <= 0) {  // about one CTA per SM, at most 8 per cluster
    S = std::max(1, std::min({sm_count_tc() / std::max(cols, 1), 8, a.KS}));
  }
  auto plan = [&](int s_) {
    const int max_ks = (a.KS + s_ - 1) / s_;
    a.D = std::max(2, std::min(max_ks, 6));
    while (a.D > 2 && TcSmem(a.D, NT, GPS, s_, a.M).total > 220 * 1024) --a.D;
    return TcSmem(a.D, NT, GPS, s_, a.M);
  };
  TcSmem L = plan(S);
  while (L.total > 227 * 1024 && S > 1) L = plan(--S);
  QIGEN_CHECK_ARG(L.total <= 227 * 1024, QIGEN_ERR_UNSUPPORTED,
                  "tensor-core GEMM needs %d bytes of shared memory", L.total);
  // prep: activations -> fp16 canonical tiles in the workspace
  a.xt = (const __half*)ws;
  {
    const int64_t total = (int64_t)a.KS * 4 * NT * 8;
    cudaLaunchConfig_t pc = {};
    pc.gridDim = dim3((unsigned)((total + 255) / 256), 1, 1);
    pc.blockDim = dim3(256, 1, 1);
    pc.stream = stream;
    cudaLaunchAttribute pa;
    pa.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pa.val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = &pa;
    pc.numAttrs = 1;
    QIGEN_CUDA_RET(cudaLaunchKernelEx(&pc, tc_prep_kernel, x, dtype, ldx, a.n, a.M, NT, a.KS * 4,
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

extern "C" int qigen_debug_tc_mode(int mode) {
  g_tc_dbg = mode;
  return QIGEN_OK;
}

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
  a.trace = g_trace;
  a.dbg = g_tc_dbg;
  cudaStream_t s = (cudaStream_t)stream;
  switch (group) {
    case 32: return tc::launch_nt<8>(a, k_splits, workspace, s, x, x_dtype, ldx);
    case 64: return tc::launch_nt<4>(a, k_splits, workspace, s, x, x_dtype, ldx);
    case 128: return tc::launch_nt<2>(a, k_splits, workspace, s, x, x_dtype, ldx);
    default: return tc::launch_nt<1>(a, k_splits, workspace, s, x, x_dtype, ldx);
  }
}
