// Batch-1 / small-batch quantized GEMV for sm_100a — the hot path.
//
// Replaces the reference's generated qGEMV (kernelgen.py:371-423) behind
// qgemv(pm, x, sums, threads).  Same factorisation as the
// reference (kernelgen.py:227-240, PAPER Eq. 2):
//     y_j = sum_g s_gj * ( sum_{i in g} x_i c_ij  -  z_gj * X_g )
// but the inner product sum x_i c_ij is computed EXACTLY on the integer tensor
// cores (IMMA, mma.sync.m16n8k32.u8.s8):
//   * codes c (0..2^b-1) are the u8 A operand, rebuilt from the panel layout
//     with one or two shift/LOP3 per 4 codes (no int->float conversion);
//   * each activation row x (f32/f16/bf16) is converted per CTA K-chunk to a
//     fixed-point integer m = rint(x * 2^(30-E)), |m| < 2^30, split into four
//     balanced signed bytes d0..d3 (m = d0 2^24 + d1 2^16 + d2 2^8 + d3); the
//     digits are the s8 B operand, one n8 column per (token, digit);
//   * the int32 accumulators are exact; at every quantisation-group boundary
//     they are folded into f32 with the scale/zero correction (the flush).
//
// Data movement: one warp owns a 16-column panel over the CTA's
// K-chunk and streams it through its own ring of shared-memory stages filled
// by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx); a stage is
// one 256-row superstep of codes plus, for g | 256, the (s, z) pairs of the
// groups it closes.  The first ring fill is issued BEFORE griddepcontrol.wait,
// so under programmatic dependent launch the weight stream of this GEMV
// overlaps the tail of the previous kernel.  CTAs sharing panels but owning
// different K-chunks form a thread-block cluster and reduce their partial
// outputs through distributed shared memory in a fixed order (deterministic,
// no atomics, no workspace).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <unordered_map>
#include <utility>

#include "common.cuh"
#include "gemv_common.cuh"
#include "tp.cuh"

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
  int x_vec;         // x rows 16-byte aligned -> vector loads
  int accumulate;
  int x_ready;       // x is not written by the preceding kernel: read it before the PDL wait
  int max_steps;     // max K-steps (32 rows) of any chunk
  int D;             // ring stages per warp
  int pre;           // stages per warp issued before griddepcontrol.wait
  int xmode;         // activation prologue: 0 plain, 1 RMSNorm(x) * w, 2 SwiGLU(x[:n], x[n:]),
                     // 3 RMSNorm with the weight folded into W: y = rsqrt(mean(x^2) + eps) (x W)
  const float* xw;   // RMSNorm weight [n]
  float eps;         // RMSNorm epsilon
  unsigned char* dig;         // prepared activation digits (act_prep_kernel) or null
  unsigned char* ws;          // caller workspace for `dig` (may be null)
  size_t ws_bytes;
  unsigned long long* trace;  // optional per-CTA timestamps (qigen_debug_trace)
  unsigned long long* trace_clk;  // optional per-CTA SM clocks at the same points
  int early;                  // trigger dependents at kernel entry
  int policy;                 // 1: weight bulk copies carry an L2 evict_first hint
  int push_on;                // TP push epilogue: y goes to every rank's inbox (tp.cuh)
  TpPush push;
  // decode chains (qigen_gemv_chain): the producer's epilogue writes its final
  // output columns (after the residual add) also as the NEXT GEMV's prepared
  // activation digits, scaled per column by dout_w (that GEMV's RMSNorm weight),
  // plus per-CTA sums of squares; the consumer bulk-copies the digits (no prep
  // kernel, no prologue) and applies 1 / rms from the sums in its epilogue.
  unsigned char* dout;        // consumer's digit buffer (act_prep layout) or null
  const float* dout_w;        // per-column multiplier or null
  int dout_tp, dout_ks, dout_ipu;  // consumer's token padding, supersteps, items per unit
  float* ss_out;              // [M][gridDim.x] sums of squares of the output (or null)
  const float* ss_in;         // consumer: [M][ss_n] partial sums of squares of its x (or null)
  int ss_n;
  int prepared;               // x is already digits at `dig` (skip prep / prologue)
};

__device__ __forceinline__ void trace_point(const GemvArgs& a, int i) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + i] = t;
    if (a.trace_clk) a.trace_clk[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 + i] = clock64();
  }
}


// Four consecutive raw activations (row element offset `base`, `k` = column) as
// f32, zero beyond n.
__device__ __forceinline__ void load_raw4(const GemvArgs& a, int64_t base, int64_t k, float (&v)[4]) {
  if (a.x_vec && k + 3 < a.n) {
    if (a.x_dtype == QIGEN_F32) {
      const float4 f = __ldg((const float4*)((const float*)a.x + base));
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    } else {
      const uint2 u = __ldg((const uint2*)((const uint16_t*)a.x + base));
      if (a.x_dtype == QIGEN_F16) {
        const float2 lo = __half22float2(*(const __half2*)&u.x), hi = __half22float2(*(const __half2*)&u.y);
        v[0] = lo.x; v[1] = lo.y; v[2] = hi.x; v[3] = hi.y;
      } else {
        const float2 lo = __bfloat1622float2(*(const __nv_bfloat162*)&u.x);
        const float2 hi = __bfloat1622float2(*(const __nv_bfloat162*)&u.y);
        v[0] = lo.x; v[1] = lo.y; v[2] = hi.x; v[3] = hi.y;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float f = 0.f;
    if (k + i < a.n) {
      if (a.x_dtype == QIGEN_F32) f = __ldg((const float*)a.x + base + i);
      else if (a.x_dtype == QIGEN_F16) f = __half2float(((const __half*)a.x)[base + i]);
      else f = __bfloat162float(((const __nv_bfloat16*)a.x)[base + i]);
    }
    v[i] = f;
  }
}

// Four consecutive GEMV inputs after the fused prologue transform:
//   xmode 0: x;  1: x * inv_rms(token) * w (RMSNorm);  2: silu(x[k]) * x[n + k] (SwiGLU)
__device__ __forceinline__ void load_x4(const GemvArgs& a, int tk, int64_t k, float (&v)[4],
                                        const float* inv_rms) {
  load_raw4(a, tk * a.ldx + k, k, v);
  if (a.xmode == 1) {
    const float inv = inv_rms[tk];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (k + i < a.n) ? v[i] * inv * __ldg(a.xw + k + i) : 0.f;
  } else if (a.xmode == 2) {
    float u[4];
    load_raw4(a, tk * a.ldx + a.n + k, k, u);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = v[i] / (1.f + __expf(-v[i])) * u[i];
  }
}


// 1/rms over the full rows of tokens [t0, t0 + ntok) (RMSNorm prologue),
// block-wide; inv[tk - t0].
template <int T>
__device__ __forceinline__ void row_inv_rms(const GemvArgs& a, int t0, int ntok, float* red,
                                            float* inv) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 0; j < ntok; ++j) {
    float ss = 0.f;
    for (int64_t k = 4 * threadIdx.x; k < a.n; k += 4 * T) {
      float v[4];
      load_raw4(a, (t0 + j) * a.ldx + k, k, v);
      ss += v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[j * (T / 32) + warp] = ss;
  }
  __syncthreads();
  if (threadIdx.x < ntok) {
    float ss = 0.f;
    for (int w = 0; w < T / 32; ++w) ss += red[threadIdx.x * (T / 32) + w];
    inv[threadIdx.x] = rsqrtf(ss / (float)a.n + a.eps);
  }
  __syncthreads();
}

// Activation prep kernel (used when a CTA's chunk x tokens is too long for the
// in-kernel prologue): digits for all rows of all (padded) tokens, once per
// GEMV, into a global buffer [step][TP][16 x uint2] + [unit][TP] (xsum, scale).
// grid = (ceil(KS*64 / 256), TP); tokens >= M are written as zeros.
template <int IPU>
__global__ void __launch_bounds__(256) act_prep_kernel(const GemvArgs a, int TP, int UPS) {
  __shared__ float red[16 * 8];
  __shared__ float inv[16];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int tk = blockIdx.y;
  const int lane = threadIdx.x & 31;
  if (a.xmode == 1 && tk < a.M) row_inv_rms<256>(a, tk, 1, red, inv);  // this CTA's token
  const int it = blockIdx.x * 256 + threadIdx.x;  // item within the token
  const int nitems = a.KS * 64;
  const bool live = it < nitems && tk < a.M;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  const int st = it >> 3, sub = it & 7;
  if (live) load_x4(a, tk, (int64_t)32 * st + 16 * (sub >> 2) + 4 * (sub & 3), v, inv - tk);
  // (load_x4 reads inv_rms[tk]; this CTA's single value sits at inv[0])
  const uint32_t umask = IPU == 32 ? 0xffffffffu : ((1u << IPU) - 1u) << (lane & ~(IPU - 1));
  Digits d = digitize<IPU>(v, umask);
  if (it < nitems) {
    uint32_t* dig = (uint32_t*)a.dig;
    store_digits(dig, st, tk, TP, sub, d);
    if ((it % IPU) == 0) {
      const int u = it / IPU;
      ((float2*)(a.dig + (size_t)a.KS * 8 * TP * 128))[u * TP + tk] =
          live ? make_float2(d.xsum, d.scale) : make_float2(0.f, 0.f);
    }
  }
}

// Prep kernel for the RMSNorm prologue: one 1024-thread CTA per token holds the
// whole row in registers (item it = x[4it .. 4it+3]), so the row is read once:
// sum of squares -> block reduction -> normalise -> digitise.
constexpr int kNormPrepThreads = 1024;
constexpr int kNormPrepMaxR = 8;  // items per thread: K <= 32768
template <int IPU>
__global__ void __launch_bounds__(kNormPrepThreads) act_prep_norm_kernel(const GemvArgs a, int TP,
                                                                         int UPS) {
  __shared__ float red[kNormPrepThreads / 32];
  __shared__ float inv_s;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int tk = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nitems = a.KS * 64;
  const int R = (nitems + kNormPrepThreads - 1) / kNormPrepThreads;
  uint32_t* dig = (uint32_t*)a.dig;
  float2* xsp = (float2*)(a.dig + (size_t)a.KS * 8 * TP * 128);
  if (tk >= a.M) {  // padding token: zero digits and unit parameters
    for (int r = 0; r < R; ++r) {
      const int it = r * kNormPrepThreads + threadIdx.x;
      if (it >= nitems) continue;
      store_digits(dig, it >> 3, tk, TP, it & 7, Digits{{0u, 0u, 0u, 0u}, 0.f, 0.f});
      if ((it % IPU) == 0) xsp[(it / IPU) * TP + tk] = make_float2(0.f, 0.f);
    }
    return;
  }
  float v[kNormPrepMaxR][4];
  float ss = 0.f;
#pragma unroll
  for (int r = 0; r < kNormPrepMaxR; ++r) {
    v[r][0] = v[r][1] = v[r][2] = v[r][3] = 0.f;
    const int it = r * kNormPrepThreads + threadIdx.x;
    if (r < R && it < nitems) {
      load_raw4(a, tk * a.ldx + 4 * (int64_t)it, 4 * (int64_t)it, v[r]);
      ss += v[r][0] * v[r][0] + v[r][1] * v[r][1] + v[r][2] * v[r][2] + v[r][3] * v[r][3];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (warp == 0) {
    ss = red[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) inv_s = rsqrtf(ss / (float)a.n + a.eps);
  }
  __syncthreads();
  const float inv = inv_s;
  const uint32_t umask = IPU == 32 ? 0xffffffffu : ((1u << IPU) - 1u) << (lane & ~(IPU - 1));
#pragma unroll
  for (int r = 0; r < kNormPrepMaxR; ++r) {
    if (r >= R) break;  // CTA-uniform
    const int it = r * kNormPrepThreads + threadIdx.x;
    const int64_t k = 4 * (int64_t)it;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[r][i] = (k + i < a.n) ? v[r][i] * inv * __ldg(a.xw + k + i) : 0.f;
    const Digits d = digitize<IPU>(v[r], umask);
    if (it < nitems) {
      store_digits(dig, it >> 3, tk, TP, it & 7, d);
      if ((it % IPU) == 0) xsp[(it / IPU) * TP + tk] = make_float2(d.xsum, d.scale);
    }
  }
}

constexpr int kMaxRounds3 = 16;  // xmode 3: prologue rounds of the block per chunk (smem slots)

// Shared-memory carve-up (bytes), identical on host and device.
struct SmemLayout {
  int ring, bars, bfrag, xs, zero, rbar, pbar, inv, ssw, yp, ep, total, stage;
  __host__ __device__ SmemLayout(int bits, int szb, int D, int max_steps, int TP, int M, int WPC,
                                 int S, int epi = 0) {
    stage = bits * 512 + szb;
    // units are >= 32 rows, except g = 16 (szb 2048: 16 groups per superstep)
    const int max_units = szb == 16 * 128 ? 2 * max_steps : max_steps;
    int off = 0;
    ring = off;  off += WPC * D * stage;
    bars = off;  off += WPC * D * 8;
    bfrag = off; off += max_steps * TP * 128;   // [step][TP][digit j][t] (b0, b1)
    xs = off;    off += max_units * TP * 8;     // [unit][TP] (sum of m, 2^(E-30))
    zero = off;  off += 8;
    rbar = off;  off += 8;
    pbar = off;  off += 8;
    inv = off;   off += 16 * 4;
    ssw = off;   off += kMaxRounds3 * WPC * 8;            // xmode 3: (sum x^2, token) per round x warp
    yp = off;    off += (S - 1) * (WPC * 16 * M + M) * 4 + 16;  // owner's inbox (+ sum x^2 per rank)
    ep = off;    off += epi ? (2 * M + 1) * WPC * 16 * 4 : 0;  // epilogue: final / old y / scale
    total = off;
  }
};

// GPS = quantisation groups closed per superstep: 16, 8, 4, 2, 1 for g = 16,
// 32, 64, 128, 256 (their (s, z) ride in the stage), 0 for longer groups (g a
// multiple of 256 or full column; (s, z) prefetched from global one group
// ahead).  Exponent/flush unit U = min(g, 128) rows: the activations of one unit
// share a fixed-point exponent (found with one REDUX, no CTA barrier), and the
// integer accumulators are folded into f32 once per unit.  g = 16 (
// the reference unrolls groups inside a packing unit, kernelgen.py:289-310): a
// group is half an m16n8k32 step, so each step issues two m16n8k16 IMMAs (the
// A fragment's k halves, the B digit words' halves) and flushes after each.
template <int BITS, int NB, int WPC, int GPS>
__global__ void __launch_bounds__(WPC * 32, 2) gemv_kernel(const GemvArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int T = WPC * 32;
  constexpr int TP = 2 * NB;                // tokens in the fragment layout (padded)
  constexpr int SZB = GPS * 128;
  constexpr int UPS = GPS > 2 ? GPS : 2;   // flush units per superstep
  constexpr int SPU = GPS == 16 ? 1 : 8 / UPS;  // steps per unit (g = 16: half a step)
  constexpr int IPU = GPS == 16 ? 4 : SPU * 8;  // prologue items (4 rows) per unit
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, t = lane & 3;
  const int S = gridDim.y, ys = blockIdx.y;
  const int ks0 = (int)((int64_t)a.KS * ys / S), ks1 = (int)((int64_t)a.KS * (ys + 1) / S);
  const int nks = ks1 - ks0;
  const int p = blockIdx.x * WPC + warp;
  const bool active = p < a.P;
  const int M = a.M, D = a.D;
  const int nsteps = nks * 8;
  const int nunits = nks * UPS;
  SmemLayout L(BITS, SZB, D, a.max_steps, TP, M, WPC, S, a.dout != nullptr || a.accumulate);
  unsigned char* ring = smem + L.ring + warp * D * L.stage;
  uint64_t* bars = (uint64_t*)(smem + L.bars) + warp * D;
  float2* xs = (float2*)(smem + L.xs);
  float* yp = (float*)(smem + L.yp);

  const char* wsrc = (const char*)(a.qw + ((int64_t)(active ? p : 0) * a.KS) * BITS * 32);
  const char* zsrc = (const char*)(a.qsz + (int64_t)(active ? p : 0) * a.Gp * 16);
  uint64_t pol = 0;
  if (a.policy) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int s) {  // lane 0: superstep s of the chunk into slot s % D
    const int slot = s % D;
    unsigned char* dst = ring + slot * L.stage;
    mbar_expect_tx(&bars[slot], (uint32_t)L.stage);
    if (a.policy) {
      bulk_g2s_hint(dst, wsrc + (int64_t)(ks0 + s) * BITS * 512, BITS * 512, &bars[slot], pol);
      if (SZB) bulk_g2s_hint(dst + BITS * 512, zsrc + (int64_t)(ks0 + s) * SZB, SZB, &bars[slot], pol);
    } else {
      bulk_g2s(dst, wsrc + (int64_t)(ks0 + s) * BITS * 512, BITS * 512, &bars[slot]);
      if (SZB) bulk_g2s(dst + BITS * 512, zsrc + (int64_t)(ks0 + s) * SZB, SZB, &bars[slot]);
    }
  };
  trace_point(a, 0);
  if (a.early) asm volatile("griddepcontrol.launch_dependents;");

  // ---- 1. ring setup + weight prefetch (independent of the previous kernel) --
  const int n_first = active ? min(D, nks) : 0;
  const int n_pre = min(a.pre, n_first);
  if (lane == 0) {
    for (int i = 0; i < D; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < n_pre; ++s) issue(s);
  }
  if (threadIdx.x < 2) ((uint32_t*)(smem + L.zero))[threadIdx.x] = 0u;
  uint64_t* rbar = (uint64_t*)(smem + L.rbar);
  uint64_t* pbar = (uint64_t*)(smem + L.pbar);
  if (threadIdx.x == 0) {
    if (S > 1) {
      // split-K inbox of the cluster's rank-0 CTA: (S-1) partials of R floats
      mbar_init(rbar, 1);
      mbar_expect_tx(rbar, (uint32_t)((S - 1) * (WPC * 16 * M + (a.xmode == 3 ? M : 0)) * 4));
    }
    if (a.dig) mbar_init(pbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (S > 1)  // arrive now, wait only before pushing: every inbox is initialised by then
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (!a.dig) {
    // pull this chunk's activations into L2 now (safe before the PDL wait: L2
    // is the point of coherence, and nothing is read into registers or L1 here)
    const int esz = a.x_dtype == QIGEN_F32 ? 4 : 2;
    const int64_t kb = a.xmode == 1 ? 0 : (int64_t)ks0 * kSuper * esz;
    const int64_t ke = (a.xmode == 1 ? a.n : min((int64_t)ks1 * kSuper, a.n)) * esz;
    const int lines = (int)((ke - kb + 127) / 128);
    const int halves = a.xmode == 2 ? 2 : 1;
    for (int i = threadIdx.x; i < lines * M * halves; i += T) {
      const int li = i % lines, rest = i / lines;
      const char* pa = (const char*)a.x + ((rest % M) * a.ldx + (rest / M) * a.n) * esz + kb +
                       (int64_t)li * 128;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
    }
  }
  __syncthreads();

  // ---- 2. PDL: everything below may read what the previous kernel wrote -----
  // (with x_ready the inputs are known not to come from the preceding kernel:
  // only the y write below waits, so this GEMV overlaps its predecessor fully)
  const bool early_x = a.x_ready && !a.dig;
  trace_point(a, 9);
  if (!early_x) asm volatile("griddepcontrol.wait;" ::: "memory");
  trace_point(a, 1);
  // the epilogue's inputs that are not computed here (the y it accumulates
  // into, the next GEMV's per-column scale), staged now so the epilogue of the
  // owning CTA does no dependent global loads
  constexpr int C = WPC * 16;
  float* ep_fin = (float*)(smem + L.ep);
  float* ep_old = ep_fin + M * C;
  float* ep_w = ep_old + M * C;
  const bool ep_stage = ys == 0 && !early_x && (a.dout || a.accumulate);
  if (ep_stage) {
    const int64_t c0 = (int64_t)blockIdx.x * C;
    for (int i = threadIdx.x; i < M * C; i += T) {
      const int64_t col = c0 + i % C;
      ep_old[i] = a.accumulate && col < a.m ? a.y[(i / C) * a.ldy + col] : 0.f;
    }
    if (a.dout)
      for (int i = threadIdx.x; i < C; i += T)
        ep_w[i] = a.dout_w && c0 + i < a.m ? __ldg(a.dout_w + c0 + i) : 1.f;
  }
  if (a.ss_in && ys == 0 && threadIdx.x < M) {
    // RMSNorm of x folded into the epilogue: 1 / rms from the producer's per-CTA
    // sums of squares, fixed order (read now: no dependent load at the end)
    float ss = 0.f;
    for (int c = 0; c < a.ss_n; ++c) ss += a.ss_in[threadIdx.x * a.ss_n + c];
    ((float*)(smem + L.inv))[threadIdx.x] = rsqrtf(ss / (float)a.n + a.eps);
  }

  // ---- 3. activation digits for this chunk into shared memory ----------------
  if (a.dig) {
    // prepared by act_prep_kernel: two bulk copies
    if (threadIdx.x == 0) {
      const uint32_t db = (uint32_t)(nsteps * TP * 128), xb = (uint32_t)(nunits * TP * 8);
      mbar_expect_tx(pbar, db + xb);
      bulk_g2s(smem + L.bfrag, a.dig + (size_t)ks0 * 8 * TP * 128, db, pbar);
      bulk_g2s(smem + L.xs, a.dig + (size_t)a.KS * 8 * TP * 128 + (size_t)ks0 * UPS * TP * 8, xb,
               pbar);
      trace_point(a, 8);
      if (lane == 0)
        for (int s = n_pre; s < n_first; ++s) issue(s);
    } else if (lane == 0) {
      for (int s = n_pre; s < n_first; ++s) issue(s);
    }
    mbar_wait(pbar, 0);
  } else {
    // fused prologue: every CTA digitises its own chunk (short chunks only)
    float* inv_rms = (float*)(smem + L.inv);
    if (a.xmode == 1) row_inv_rms<T>(a, 0, M, (float*)(smem + L.xs), inv_rms);
    const int64_t k0 = (int64_t)ks0 * kSuper;
    const int items = M * nsteps * 8;  // item = (token, step, half, t): 4 consecutive k
    uint32_t* bw = (uint32_t*)(smem + L.bfrag);
    const uint32_t umask = IPU == 32 ? 0xffffffffu : ((1u << IPU) - 1u) << (lane & ~(IPU - 1));
    bool first = true;
    for (int it0 = 0; it0 < items; it0 += T) {  // CTA-uniform trip count
      const int it = it0 + threadIdx.x;
      const bool live = it < items;
      const int sub = it & 7, st = (it >> 3) % nsteps, tk = live ? (it >> 3) / nsteps : 0;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (live) load_x4(a, tk, k0 + 32 * st + 16 * (sub >> 2) + 4 * (sub & 3), v, inv_rms);
      if (first) {  // the rest of the first ring fill goes out behind the x loads
        trace_point(a, 8);
        first = false;
        if (lane == 0)
          for (int s = n_pre; s < n_first; ++s) issue(s);
      }
      const Digits d = digitize<IPU>(v, umask);
      if (it0 == 0) trace_point(a, 11);
      if (live) {
        store_digits(bw, st, tk, TP, sub, d);
        if ((it % IPU) == 0) xs[((it % (nsteps * 8)) / IPU) * TP + tk] = make_float2(d.xsum, d.scale);
      }
      if (a.xmode == 3) {
        // sum of squares of this chunk: a warp's 32 items belong to one token
        // (a token has nsteps * 8 items, a multiple of 64); fixed-order warp
        // reduction, one slot per (round, warp)
        float ss = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0)
          ((float2*)(smem + L.ssw))[(it0 / T) * WPC + warp] =
              make_float2(ss, __int_as_float(live ? tk : -1));
      }
    }
    // zero fragments / unit params of the padding tokens M..TP-1
    for (int e = threadIdx.x; e < nsteps * (TP - M) * 16; e += T) {
      const int st = e / ((TP - M) * 16), r = e % ((TP - M) * 16);
      ((uint2*)bw)[(st * TP + M) * 16 + r] = make_uint2(0u, 0u);
    }
    for (int e = threadIdx.x; e < nunits * (TP - M); e += T)
      xs[(e / (TP - M)) * TP + M + e % (TP - M)] = make_float2(0.f, 0.f);
    if (first && lane == 0)  // no activation items (cannot happen for n > 0)
      for (int s = n_pre; s < n_first; ++s) issue(s);
    trace_point(a, 10);
    __syncthreads();
    if (a.xmode == 3 && threadIdx.x < M) {  // this chunk's sum of squares per token, fixed order
      const float2* sw = (const float2*)(smem + L.ssw);
      const int nr = (items + T - 1) / T;
      float ss = 0.f;
      for (int i = 0; i < nr * WPC; ++i)
        if (__float_as_int(sw[i].y) == (int)threadIdx.x) ss += sw[i].x;
      inv_rms[threadIdx.x] = ss;  // (the chunk's partial; the row total is formed in the epilogue)
    }
  }
  if (!a.early) asm volatile("griddepcontrol.launch_dependents;");
  trace_point(a, 2);

  // ---- 4. main loop ------------------------------------------------------------
  // AC accumulator sets alternate over steps: AC independent IMMA chains (2-bit
  // always uses two: odd steps carry an extra x16)
  constexpr int AC = (NB <= 2 || BITS == 2) ? 2 : 1;
  int acc[AC][NB][4];
  float yv[NB][2];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    yv[nb][0] = yv[nb][1] = 0.f;
#pragma unroll
    for (int c = 0; c < AC; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[c][nb][q] = 0;
  }
  // digit-pair weight of this lane: columns (d0, d1) -> 2^16, (d2, d3) -> 1
  const float w_lo = (t & 1) ? 1.f : 65536.f;
  const float w_hi = w_lo * RowScale<BITS>::inv_hi;
  // B fragment of n8 block nb: token 2nb + (gq >> 2), digit gq & 3; per step the
  // fragments of all TP tokens are 2 NB x 128 bytes apart (compile-time stride)
  const uint2* bbase = (const uint2*)(smem + L.bfrag) + (gq >> 2) * 16 + (gq & 3) * 4 + t;
  const bool xon = (t & 1) == 0;  // lanes holding digits (d0, d1) carry the z X term
  const int tcol = t >> 1;        // token offset of this lane's accumulator columns
  const float2* szg = (const float2*)zsrc;
  const int spg = GPS == 0 ? (a.g ? a.g / kStep : a.KS * 8) : 1;  // steps per (long) group
  int gcur = ks0 * 8 / spg;
  float2 szr0 = make_float2(0.f, 0.f), szr1 = szr0;
  if (GPS == 0) {
    szr0 = szg[gcur * 16 + gq];
    szr1 = szg[gcur * 16 + gq + 8];
  }
  auto flush = [&](int u, float2 sz0, float2 sz1) {
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const float2 xv = xs[u * TP + 2 * nb + tcol];
      const float X = xon ? xv.x : 0.f, sc = xv.y;
      int c0 = acc[0][nb][0], c1 = acc[0][nb][1], c2 = acc[0][nb][2], c3 = acc[0][nb][3];
#pragma unroll
      for (int c = 1; c < AC; ++c) {
        // 2-bit odd steps: both rows carry an extra exact x16
        const int sh = BITS == 2 ? 4 : 0;
        c0 += acc[c][nb][0] >> sh; c1 += acc[c][nb][1] >> sh;
        c2 += acc[c][nb][2] >> sh; c3 += acc[c][nb][3] >> sh;
      }
      // digit pair -> one exact int32 (|.| < 2^31 for units <= 128 rows)
      const float q0 = (float)(c0 * 256 + c1), q1 = (float)(c2 * 256 + c3);
      yv[nb][0] = fmaf(sz0.x * sc, fmaf(-sz0.y, X, q0 * w_lo), yv[nb][0]);
      yv[nb][1] = fmaf(sz1.x * sc, fmaf(-sz1.y, X, q1 * w_hi), yv[nb][1]);
#pragma unroll
      for (int c = 0; c < AC; ++c) acc[c][nb][0] = acc[c][nb][1] = acc[c][nb][2] = acc[c][nb][3] = 0;
    }
  };

  int slot = 0;
  uint32_t phase = 0;
  const int my_nks = active ? nks : 0;  // idle warps never wait on their ring
  for (int s = 0; s < my_nks; ++s) {
    mbar_wait(&bars[slot], phase);
    if (s == 0) trace_point(a, 5);
    const unsigned char* stg = ring + slot * L.stage;
    uint4 w[BITS];
#pragma unroll
    for (int v = 0; v < BITS; ++v) w[v] = ((const uint4*)stg)[v * 32 + lane];
    const float2* szs = (const float2*)(stg + BITS * 512);
    const uint2* bs = bbase + s * 8 * TP * 16;
#pragma unroll
    for (int sl = 0; sl < 8; ++sl) {
      uint32_t af[4];
      extract<BITS>(w, sl, af);
      if constexpr (GPS == 16) {
        // two groups per step: k16 IMMA on each half, flush each
        constexpr int sh = BITS == 2 ? 4 : 0;  // 2-bit odd steps carry an extra x16
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int c16[NB][4];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const uint2 b = bs[(sl * TP + 2 * nb) * 16];
            imma16(c16[nb], af[2 * h], af[2 * h + 1], h ? b.y : b.x);
          }
          const int u = s * 16 + 2 * sl + h;
          const float2 sz0 = szs[(2 * sl + h) * 16 + gq], sz1 = szs[(2 * sl + h) * 16 + gq + 8];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const float2 xv = xs[u * TP + 2 * nb + tcol];
            const float X = xon ? xv.x : 0.f, sc = xv.y;
            const int k = (sl & 1) ? sh : 0;
            const float q0 = (float)((c16[nb][0] >> k) * 256 + (c16[nb][1] >> k));
            const float q1 = (float)((c16[nb][2] >> k) * 256 + (c16[nb][3] >> k));
            yv[nb][0] = fmaf(sz0.x * sc, fmaf(-sz0.y, X, q0 * w_lo), yv[nb][0]);
            yv[nb][1] = fmaf(sz1.x * sc, fmaf(-sz1.y, X, q1 * w_hi), yv[nb][1]);
          }
        }
      } else {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) imma(acc[sl % AC][nb], af, bs[(sl * TP + 2 * nb) * 16]);
        if ((sl + 1) % SPU == 0) {
          const int uj = (sl + 1) / SPU - 1;  // unit within the superstep
          const int u = s * UPS + uj;
          if (GPS > 0) {
            const int gi = GPS >= UPS ? uj : 0;  // g = 256: both units use group 0
            flush(u, szs[gi * 16 + gq], szs[gi * 16 + gq + 8]);
          } else {
            flush(u, szr0, szr1);
          }
        }
      }
    }
    if (GPS == 0 && ((ks0 + s + 1) * 8) % spg == 0) {  // long group closed
      ++gcur;
      if (gcur < a.Gp) {
        szr0 = szg[gcur * 16 + gq];
        szr1 = szg[gcur * 16 + gq + 8];
      }
    }
    __syncwarp();
    if (lane == 0 && s + D < nks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s + D);
    }
    if (++slot == D) {
      slot = 0;
      phase ^= 1u;
    }
  }
  trace_point(a, 3);

  // ---- 5. combine digit-pair lanes; deterministic split-K reduction ---------
  // Element e = (warp*16 + row)*M + token of this CTA column.  With S > 1 the
  // CTAs of ranks 1..S-1 push their partials into the rank-0 CTA's inbox with
  // st.async (completing bytes on its mbarrier) and exit; rank 0 adds them to
  // its own in rank order (deterministic) and writes y.
  const int R = WPC * 16 * M;
  const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
  if (S > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  trace_point(a, 6);
  const int64_t col0 = (int64_t)blockIdx.x * WPC * 16;
  float* ssl = (float*)(smem + L.inv);  // xmode 3: this CTA's chunk sum of squares per token
  if (a.xmode == 3 && rank > 0 && threadIdx.x < M)
    st_async(mapa(yp + (S - 1) * R + (rank - 1) * M + threadIdx.x, 0), ssl[threadIdx.x],
             mapa(rbar, 0));
  if (rank == 0 && S > 1) mbar_wait(rbar, 0);
  if (a.xmode == 3 && rank == 0) {  // row totals in rank order -> 1 / rms
    if (threadIdx.x < M) {
      float ss = ssl[threadIdx.x];
      for (int q = 1; q < S; ++q) ss += yp[(S - 1) * R + (q - 1) * M + threadIdx.x];
      ssl[threadIdx.x] = rsqrtf(ss / (float)a.n + a.eps);
    }
    __syncthreads();
  }
  if (early_x && rank == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // before y
  trace_point(a, 7);
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const float v0 = yv[nb][0] + __shfl_xor_sync(0xffffffffu, yv[nb][0], 1);
    const float v1 = yv[nb][1] + __shfl_xor_sync(0xffffffffu, yv[nb][1], 1);
    const int tk = 2 * nb + (t >> 1);
    if ((t & 1) == 0 && tk < M) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = warp * 16 + gq + 8 * h;
        const int e = row * M + tk;
        float v = h ? v1 : v0;
        if (rank > 0) {
          st_async(mapa(yp + (rank - 1) * R + e, 0), v, mapa(rbar, 0));
        } else {
          for (int q = 1; q < S; ++q) v += yp[(q - 1) * R + e];
          if (a.xmode == 3) v *= ssl[tk];
          if (a.ss_in) v *= ((const float*)(smem + L.inv))[tk];
          const int64_t col = col0 + row;
          const float fin = ep_stage ? ep_old[tk * C + row] + v : v;  // (ep_old 0 unless accumulate)
          if (a.dout) ep_fin[tk * C + row] = col < a.m ? fin : 0.f;
          if (col < a.m) {
            if (a.push_on) {  // this rank's partial into every rank's inbox (NVLink stores)
              const TpPush& pp = a.push;
              const size_t off = ((size_t)(pp.slot * pp.world + pp.rank) * pp.bmax + tk) * pp.d + col;
              for (int q = 0; q < pp.world; ++q) pp.inbox[q][off] = v;
            } else {
              float* dst = a.y + tk * a.ldy + col;
              *dst = ep_stage ? fin : (a.accumulate ? *dst + v : v);
            }
          }
        }
      }
    }
  }
  if (a.dout && rank == 0) {
    // The CTA's WPC * 16 final columns are rows [col0, col0 + WPC * 16) of the
    // next GEMV's K: digitise them in the act_prep layout (item it = 4 rows:
    // step it >> 3, sub-item it & 7), dout_ipu items per exponent unit, and
    // publish this CTA's sum of squares per token.
    trace_point(a, 12);
    __syncthreads();
    trace_point(a, 13);
    const float* ev = ep_fin;
    for (int tk = warp; tk < M; tk += WPC) {  // (WPC = 8: one warp-wide unit set per token)
      const int it_l = lane;
      const int kl = 32 * (it_l >> 3) + 16 * ((it_l & 7) >> 2) + 4 * (it_l & 3);
      float v4[4], ss = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float f = ev[tk * C + kl + i];
        ss += f * f;
        v4[i] = f * ep_w[kl + i];
      }
      Digits d;
      if (a.dout_ipu == 32) {
        d = digitize<32>(v4, 0xffffffffu);
      } else if (a.dout_ipu == 16) {
        d = digitize<16>(v4, 0xffffu << (lane & 16));
      } else {
        d = digitize<8>(v4, 0xffu << (lane & 24));
      }
      const int it = (int)(col0 / 4) + it_l;
      store_digits((uint32_t*)a.dout, it >> 3, tk, a.dout_tp, it & 7, d);
      if ((it % a.dout_ipu) == 0)
        ((float2*)(a.dout + (size_t)a.dout_ks * 8 * a.dout_tp * 128))[(it / a.dout_ipu) * a.dout_tp + tk] =
            make_float2(d.xsum, d.scale);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (a.ss_out && lane == 0) a.ss_out[tk * gridDim.x + blockIdx.x] = ss;
    }
  }
  if (a.push_on && rank == 0) {
    // release the pushed columns: every thread's stores are ordered before the
    // arrival counts (system scope), one count per rank
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const TpPush& pp = a.push;
      const unsigned ncols = (unsigned)min((int64_t)WPC * 16, a.m - col0);
      for (int q = 0; q < pp.world; ++q) atomicAdd_system(pp.flags[q] + pp.slot * 8 + pp.rank, ncols);
    }
  }
  trace_point(a, 4);
}

// ---------------------------------------------------------------------------
// Tuning / debugging aids (qigen_debug_*): per calling thread, so a knob set by
// one thread never changes another thread's launches.  The product defaults
// are the initial values.
thread_local unsigned long long* g_trace = nullptr;  // shared with gemm_tc.cu, gemv_grouped.cu
static thread_local unsigned long long* g_trace_clk = nullptr;
constexpr int kMaxSplits = 16;  // cluster size along K (non-portable above 8)
static thread_local int g_pre = -1;  // stages issued before the PDL wait (-1: all of the first fill)
static thread_local int g_force_prep = 0;  // always digitise activations in act_prep_kernel
static thread_local int g_early = 0;       // trigger the dependent launch at kernel entry
static thread_local int g_policy = 0;      // L2 evict_first hint on weight copies
static thread_local int g_wpc = 8;         // warps per CTA for <= 4 tokens (8 or 16)
static thread_local int g_ring_kb = 0;     // ring bytes per CTA (KB; 0 = 10 KB per warp)
static thread_local int g_max_ctas = 0;    // cap on the grid (0 = rule below)
static thread_local int g_max_split = kMaxSplits;  // cap on the automatic K split (cluster size)
static thread_local int g_norm_prep = 1;  // RMSNorm prologues via act_prep_norm_kernel (measured: -1 us per 7B layer)

static int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Scratch for prepared activation digits when the caller passes no workspace:
// allocated stream-ordered for this call and freed stream-ordered behind its
// kernels, so concurrent calls on different streams (or threads) never share
// it.  Outside capture it comes from a per-device pool that keeps its memory
// (no cudaMalloc after warm-up); inside stream capture it becomes a graph
// memory node.  Callers on a hot path pass a workspace instead
// (qigen_gemv_workspace_size): the free is a full stream dependency, which
// ends the programmatic-launch overlap with the next kernel.
int scratch_alloc(cudaStream_t stream, size_t bytes, unsigned char** out) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  QIGEN_CUDA_RET(cudaStreamIsCapturing(stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    QIGEN_CUDA_RET(cudaMallocAsync((void**)out, bytes, stream));
    return QIGEN_OK;
  }
  static std::once_flag flag[kMaxDevices];
  static cudaMemPool_t pool[kMaxDevices];
  static int pst[kMaxDevices];
  int dev = 0;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CHECK_ARG(dev >= 0 && dev < kMaxDevices, QIGEN_ERR_CUDA, "device index %d", dev);
  std::call_once(flag[dev], [&] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    uint64_t keep = ~0ull;
    if (cudaMemPoolCreate(&pool[dev], &props) != cudaSuccess ||
        cudaMemPoolSetAttribute(pool[dev], cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess)
      pst[dev] = QIGEN_ERR_CUDA;
  });
  QIGEN_CHECK_ARG(!pst[dev], QIGEN_ERR_CUDA, "could not create the GEMV scratch pool");
  QIGEN_CUDA_RET(cudaMallocFromPoolAsync((void**)out, bytes, pool[dev], stream));
  return QIGEN_OK;
}

template <int BITS, int NB, int WPC, int GPS>
static int launch_cfg(GemvArgs& a, int req_S, cudaStream_t stream) {
  auto kern = gemv_kernel<BITS, NB, WPC, GPS>;
  constexpr int TP = 2 * NB;
  constexpr int UPS = GPS > 2 ? GPS : 2;
  constexpr int IPU = GPS == 16 ? 4 : (8 / UPS) * 8;
  static OncePerDevice once;
  const int cst = once.run([&]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
    QIGEN_CUDA_RET(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return QIGEN_OK;
  });
  if (cst) return cst;
  const int stage = BITS * 512 + GPS * 128;
  auto shape = [&](int S) {  // smem plan for S chunks: ring of <= 80 KB per CTA
    const int max_ks = (a.KS + S - 1) / S;
    a.max_steps = max_ks * 8;
    const int epi = a.dout != nullptr || a.accumulate;
    SmemLayout L0(BITS, GPS * 128, 0, a.max_steps, TP, a.M, WPC, S, epi);
    const int budget = std::min(g_ring_kb ? g_ring_kb * 1024 : WPC * 10 * 1024,
                                224 * 1024 - L0.total - WPC * 16);
    a.D = std::max(2, std::min(max_ks, budget / (WPC * stage)));
    return SmemLayout(BITS, GPS * 128, a.D, a.max_steps, TP, a.M, WPC, S, epi);
  };
  const int cols = (a.P + WPC - 1) / WPC;
  int S = req_S;
  const int sms = sm_count();
  if (S <= 0 && a.M >= 4) {
    // 4+ tokens: the loop is issue-bound (NB n8 blocks per step), so fewer,
    // longer chunks win; 2 splits unless the fragments need more shared memory
    // (measured on the 65B B=8 shapes: 8192x24576 63 vs 75 us, 8192x44032 103 vs
    // 122 us; tools/microbench.py --tokens 8 --splits ...)
    S = std::min(2, a.KS);
  }
  if (S <= 0 && (int64_t)cols * a.KS >= (int64_t)sms * 24) {
    // Large matrices are streaming-bound: pick the split whose grid fills whole
    // waves of SMs best (an SM holding one CTA more than its neighbours sets the
    // kernel time), each extra split charged 2% (reduction, shorter chunks).
    // 8192x24576 (192 column tiles): S = 1 -> 38.8 us, S = 3 -> 32.7 us;
    // 8192x44032: S = 1 58 us, S = 3 47 us; 22016x8192: S = 2 27 us, S = 3 36 us.
    double best = -1.0;
    for (int c = 1; c <= std::min(8, a.KS); ++c) {
      if ((a.KS + c - 1) / c < 4) break;  // keep >= 4 supersteps per chunk
      const int64_t ctas = (int64_t)cols * c;
      const double eff = (double)ctas / ((double)sms * (double)((ctas + sms - 1) / sms));
      if (eff - 0.02 * c > best) {
        best = eff - 0.02 * c;
        S = c;
      }
    }
  }
  if (S <= 0) {
    // Empirical rule (tools/tune_splits.py, dependent chains of launches under
    // PDL on B200): grids above ~1.55 CTAs per SM lose more to the next kernel
    // not fitting beside this one than they gain from shorter chunks; below
    // that, the shortest longest-chunk wins (ties: fewer CTAs).  Never more
    // CTAs than fit at once.
    S = 1;
    int best = a.KS;
    for (int c = 2; c <= std::min(kMaxSplits, a.KS); ++c) {
      int occ = 2;  // resident CTAs per SM for this shape's shared memory
      QIGEN_CUDA_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, WPC * 32,
                                                                   shape(c).total));
      const int max_ctas = (sm_count() * std::min(155, 100 * std::max(occ, 1) - 10)) / 100;
      if (cols * c > max_ctas) break;
      const int chunk = (a.KS + c - 1) / c;
      if (chunk < best) {
        best = chunk;
        S = c;
      }
    }
  }
  if (req_S <= 0 && g_max_ctas > 0) {
    // tuning: the largest split whose grid stays within the cap
    S = 1;
    for (int c = 2; c <= std::min(kMaxSplits, a.KS); ++c)
      if (cols * c <= g_max_ctas && (a.KS + c - 1) / c >= 2) S = c;
  }
  if (req_S <= 0) S = std::min(S, g_max_split);
  QIGEN_CHECK_ARG(S >= 1 && S <= a.KS && S <= kMaxSplits, QIGEN_ERR_ARG, "k_splits %d out of range", S);
  // many tokens x long chunks: split K further until the fragments fit in smem
  while (req_S <= 0 && shape(S).total > 224 * 1024 && S < std::min(kMaxSplits, a.KS)) ++S;
  // (the smem-fit rule above may exceed g_max_split: fitting wins)
  // xmode 3 (RMSNorm folded into W) needs the chunk's own x in every CTA: it
  // never uses the prep kernels; K is split further until a chunk is <= 4
  // rounds of the block
  auto nrounds = [&](int s_) {
    return (a.M * ((a.KS + s_ - 1) / s_) * 64 + WPC * 32 - 1) / (WPC * 32);
  };
  if (a.xmode == 3)
    while (req_S <= 0 && S < std::min(kMaxSplits, a.KS) && nrounds(S) > 4) ++S;
  QIGEN_CHECK_ARG(a.xmode != 3 || nrounds(S) <= kMaxRounds3, QIGEN_ERR_UNSUPPORTED,
                  "folded-RMSNorm GEMV: K chunk too long for %d tokens", a.M);
  const SmemLayout L = shape(S);
  a.pre = g_pre < 0 ? a.D : g_pre;
  QIGEN_CHECK_ARG(L.total <= 227 * 1024, QIGEN_ERR_UNSUPPORTED,
                  "GEMV needs %d bytes of shared memory (K chunk too long; raise k_splits)",
                  L.total);
  // activation digits: in each CTA when its chunk takes <= 2 rounds of the
  // block, else once per GEMV in act_prep_kernel
  const int rounds = (a.M * a.max_steps * 8 + WPC * 32 - 1) / (WPC * 32);
  a.dig = nullptr;
  unsigned char* scratch = nullptr;  // stream-ordered, freed behind this call's kernels
  // RMSNorm prologue for 1-2 tokens: one prep CTA per token (measured faster
  // than every CTA re-reading the row on the 7B chain; slower at 8 tokens)
  const bool norm_prep = a.xmode == 1 && a.M <= 2 && a.KS * 64 <= kNormPrepThreads * kNormPrepMaxR &&
                         (rounds > 2 || g_force_prep || g_norm_prep);
  if (a.prepared) {
    a.dig = a.ws;  // digits written by the producer's epilogue (qigen_gemv_chain)
  } else if (a.xmode != 3 && (rounds > 2 || g_force_prep || norm_prep)) {
    const size_t bytes = (size_t)a.KS * 8 * TP * 128 + (size_t)a.KS * UPS * TP * 8;
    if (a.ws && a.ws_bytes >= bytes) {
      a.dig = a.ws;
    } else {
      int st = scratch_alloc(stream, bytes, &scratch);
      if (st) return st;
      a.dig = scratch;
    }
    cudaLaunchConfig_t pc = {};
    pc.gridDim = dim3((unsigned)((a.KS * 64 + 255) / 256), (unsigned)TP, 1);
    pc.blockDim = dim3(256, 1, 1);
    pc.stream = stream;
    cudaLaunchAttribute pa;
    pa.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pa.val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = &pa;
    pc.numAttrs = 1;
    cudaError_t pe;
    if (norm_prep) {
      pc.gridDim = dim3(1, (unsigned)TP, 1);
      pc.blockDim = dim3(kNormPrepThreads, 1, 1);
      pe = cudaLaunchKernelEx(&pc, act_prep_norm_kernel<IPU>, a, (int)TP, (int)UPS);
    } else {
      pe = cudaLaunchKernelEx(&pc, act_prep_kernel<IPU>, a, (int)TP, (int)UPS);
    }
    if (pe != cudaSuccess && scratch) cudaFreeAsync(scratch, stream);
    QIGEN_CUDA_RET(pe);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cols, (unsigned)S, 1);
  cfg.blockDim = dim3(WPC * 32, 1, 1);
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
  const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, a);
  if (scratch) QIGEN_CUDA_RET(cudaFreeAsync(scratch, stream));
  QIGEN_CUDA_RET(le);
  return QIGEN_OK;
}

template <int BITS, int NB, int WPC>
static int launch_gps(GemvArgs& a, int S, cudaStream_t stream) {
  switch (a.g) {
    case 16: return launch_cfg<BITS, NB, WPC, 16>(a, S, stream);
    case 32: return launch_cfg<BITS, NB, WPC, 8>(a, S, stream);
    case 64: return launch_cfg<BITS, NB, WPC, 4>(a, S, stream);
    case 128: return launch_cfg<BITS, NB, WPC, 2>(a, S, stream);
    case 256: return launch_cfg<BITS, NB, WPC, 1>(a, S, stream);
    default: return launch_cfg<BITS, NB, WPC, 0>(a, S, stream);
  }
}

template <int BITS, int WPC>
static int launch_nb(GemvArgs& a, int S, cudaStream_t stream) {
  const int nb = (a.M + 1) / 2;
  if (nb <= 1) return launch_gps<BITS, 1, WPC>(a, S, stream);
  if (nb <= 2) return launch_gps<BITS, 2, WPC>(a, S, stream);
  if constexpr (WPC > 8) {
    return QIGEN_ERR_ARG;
  } else {
    if (nb <= 4) return launch_gps<BITS, 4, WPC>(a, S, stream);
    return launch_gps<BITS, 8, WPC>(a, S, stream);
  }
}

}  // namespace qigen

using namespace qigen;

extern "C" int qigen_debug_trace(void* buf) {
  g_trace = (unsigned long long*)buf;
  return QIGEN_OK;
}

extern "C" int qigen_debug_prefetch(int stages_before_wait) {
  g_pre = stages_before_wait;
  return QIGEN_OK;
}

extern "C" int qigen_debug_norm_prep(int on) {
  g_norm_prep = on;
  return QIGEN_OK;
}

extern "C" int qigen_debug_max_split(int s) {
  g_max_split = s < 1 ? 1 : (s > kMaxSplits ? kMaxSplits : s);
  return QIGEN_OK;
}

extern "C" int qigen_debug_trace_clk(void* buf) {
  g_trace_clk = (unsigned long long*)buf;
  return QIGEN_OK;
}

extern "C" int qigen_debug_early_trigger(int on) {
  g_early = on;
  return QIGEN_OK;
}

extern "C" int qigen_debug_gemv_tuning(int policy, int wpc, int ring_kb, int max_ctas) {
  g_policy = policy;
  g_wpc = wpc;
  g_ring_kb = ring_kb;
  g_max_ctas = max_ctas;
  return QIGEN_OK;
}

extern "C" int qigen_debug_force_prep(int on) {
  g_force_prep = on;
  return QIGEN_OK;
}
extern "C" int64_t qigen_gemv_workspace_size(int64_t n, int64_t tokens) {
  const int64_t tp = tokens <= 2 ? 2 : tokens <= 4 ? 4 : tokens <= 8 ? 8 : 16;
  return supersteps(n) * 8 * tp * (128 + 16);  // digits + unit factors (g = 16: 2 units per step)
}

static int gemv_entry(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                      int64_t group, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                      float* y, int64_t ldy, int accumulate, int k_splits, int prologue,
                      const float* prologue_w, float eps, void* workspace,
                      int64_t workspace_bytes, void* stream, const TpPush* push,
                      const qigen_gemv_chain_opts* ch = nullptr) {
  QIGEN_CHECK_ARG(bits == 2 || bits == 3 || bits == 4, QIGEN_ERR_CONFIG,
                  "bits must be one of (2, 3, 4), got %d", bits);
  const bool prepared = ch && ch->x_digits;
  QIGEN_CHECK_ARG(qw && qsz && (x || prepared) && (y || push), QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(n > 0 && m > 0, QIGEN_ERR_ARG, "empty matrix");
  QIGEN_CHECK_ARG(group == 0 || (n % group == 0), QIGEN_ERR_CONFIG,
                  "group size %lld does not divide row count %lld", (long long)group, (long long)n);
  QIGEN_CHECK_ARG(group == 0 || group == 16 || group == 32 || group == 64 || group == 128 ||
                      group % kSuper == 0,
                  QIGEN_ERR_UNSUPPORTED,
                  "group size %lld: the GEMV takes 16, 32, 64, 128 or a multiple of 256 (or full "
                  "column)", (long long)group);
  QIGEN_CHECK_ARG(tokens >= 1 && tokens <= 16, QIGEN_ERR_UNSUPPORTED,
                  "the GEMV path takes 1..16 activation rows, got %lld", (long long)tokens);
  QIGEN_CHECK_ARG(x_dtype >= 0 && x_dtype <= 2, QIGEN_ERR_ARG, "bad x dtype %d", x_dtype);
  QIGEN_CHECK_ARG(prologue >= 0 && prologue <= 3, QIGEN_ERR_ARG, "bad prologue %d", prologue);
  QIGEN_CHECK_ARG(prologue != 1 || prologue_w, QIGEN_ERR_ARG, "RMSNorm prologue needs a weight");
  QIGEN_CHECK_ARG(ldx >= (prologue == 2 ? 2 * n : n) && ldy >= m, QIGEN_ERR_ARG,
                  "leading dimensions too small");
  QIGEN_CHECK_ARG(k_splits >= 0 && k_splits <= kMaxSplits, QIGEN_ERR_ARG,
                  "k_splits %d out of range", k_splits);
  GemvArgs a = {};
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
  const int esz = x_dtype == QIGEN_F32 ? 4 : 2;
  a.x_vec = ((uintptr_t)x % 16 == 0) && ((ldx * esz) % 16 == 0) && ((n * esz) % 16 == 0 || prologue != 2);
  a.xmode = prologue;
  a.ws = (unsigned char*)workspace;
  a.ws_bytes = workspace ? (size_t)workspace_bytes : 0;
  a.xw = prologue_w;
  a.eps = eps;
  a.accumulate = accumulate & QIGEN_GEMV_ACCUMULATE;
  a.x_ready = (accumulate & QIGEN_GEMV_X_READY) ? 1 : 0;
  a.trace = g_trace;
  a.trace_clk = g_trace_clk;
  a.early = g_early || a.x_ready;  // independent x: overlap the predecessor fully
  a.policy = g_policy;
  if (push) {
    a.push_on = 1;
    a.push = *push;
  }
  if (ch) {
    if (prepared) {
      QIGEN_CHECK_ARG(prologue == 0, QIGEN_ERR_ARG, "prepared digits take no prologue");
      QIGEN_CHECK_ARG(group != 16, QIGEN_ERR_UNSUPPORTED, "prepared digits: group size 16");
      a.prepared = 1;
      a.ws = (unsigned char*)ch->x_digits;
      a.ws_bytes = (size_t)qigen_gemv_workspace_size(n, tokens);
      a.x = ch->x_digits;
      a.x_ready = 0;
      a.early = g_early;
    }
    if (ch->ss_in) {
      QIGEN_CHECK_ARG(prologue != 3 && ch->ss_count > 0, QIGEN_ERR_ARG, "bad ss_in");
      a.ss_in = ch->ss_in;
      a.ss_n = ch->ss_count;
      a.eps = ch->eps;
    }
    if (ch->y_digits) {
      const int64_t og = ch->out_group;
      QIGEN_CHECK_ARG(og == 0 || og == 32 || og == 64 || og == 128 || og % kSuper == 0,
                      QIGEN_ERR_UNSUPPORTED, "digit epilogue: consumer group size %lld",
                      (long long)og);
      QIGEN_CHECK_ARG(!push, QIGEN_ERR_ARG, "digit epilogue and TP push are exclusive");
      const int nb = (int)(tokens + 1) / 2;
      a.dout = (unsigned char*)ch->y_digits;
      a.dout_w = ch->out_scale;
      a.dout_tp = 2 * (nb <= 1 ? 1 : nb <= 2 ? 2 : nb <= 4 ? 4 : 8);
      a.dout_ks = (int)supersteps(m);
      a.dout_ipu = (og == 32 ? 32 : og == 64 ? 64 : 128) / 4;
      a.ss_out = ch->ss_out;
    }
  }
  const int S = k_splits;  // 0: chosen per launch shape in launch_cfg
  cudaStream_t s = (cudaStream_t)stream;
#define QIGEN_LAUNCH(B)                                                              \
  return (g_wpc == 16 && tokens <= 4 && !a.dout) ? launch_nb<B, 16>(a, S, s)       \
                                                 : launch_nb<B, 8>(a, S, s)
  switch (bits) {
    case 2: QIGEN_LAUNCH(2);
    case 3: QIGEN_LAUNCH(3);
    default: QIGEN_LAUNCH(4);
  }
#undef QIGEN_LAUNCH
}

extern "C" int qigen_gemv_ex(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                             int64_t group, const void* x, int x_dtype, int64_t tokens,
                             int64_t ldx, float* y, int64_t ldy, int accumulate, int k_splits,
                             int prologue, const float* prologue_w, float eps, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  return gemv_entry(qw, qsz, n, m, bits, group, x, x_dtype, tokens, ldx, y, ldy, accumulate,
                    k_splits, prologue, prologue_w, eps, workspace, workspace_bytes, stream,
                    nullptr);
}

extern "C" int64_t qigen_gemv_ss_count(int64_t m) { return (panels(m) + 7) / 8; }

extern "C" int qigen_gemv_chain(const uint32_t* qw, const float* qsz, int64_t n, int64_t m,
                                int bits, int64_t group, const void* x, int x_dtype,
                                int64_t tokens, int64_t ldx, float* y, int64_t ldy, int accumulate,
                                int prologue, const float* prologue_w, float eps, void* workspace,
                                int64_t workspace_bytes, const qigen_gemv_chain_opts* opts,
                                void* stream) {
  return gemv_entry(qw, qsz, n, m, bits, group, x, x_dtype, tokens, ldx, y, ldy, accumulate, 0,
                    prologue, prologue_w, eps, workspace, workspace_bytes, stream, nullptr, opts);
}

extern "C" int qigen_gemv_tp_push(const qigen_tp_comm* comm, int slot, const uint32_t* qw,
                                  const float* qsz, int64_t n, int64_t m, int bits,
                                  int64_t group, const void* x, int x_dtype, int64_t tokens,
                                  int64_t ldx, int prologue, const float* prologue_w, float eps,
                                  void* workspace, int64_t workspace_bytes, void* stream) {
  QIGEN_CHECK_ARG(comm, QIGEN_ERR_ARG, "null comm");
  QIGEN_CHECK_ARG(slot == 0 || slot == 1, QIGEN_ERR_ARG, "slot must be 0 or 1");
  QIGEN_CHECK_ARG(m == comm->d && tokens <= comm->bmax, QIGEN_ERR_ARG,
                  "push GEMV: m must equal the comm's d and tokens <= its max");
  TpPush p = {};
  for (int q = 0; q < comm->world; ++q) {
    p.flags[q] = (unsigned*)comm->base[q];
    p.inbox[q] = (float*)((char*)comm->base[q] + kTpHeader);
  }
  p.rank = comm->rank;
  p.world = comm->world;
  p.slot = slot;
  p.bmax = comm->bmax;
  p.d = comm->d;
  return gemv_entry(qw, qsz, n, m, bits, group, x, x_dtype, tokens, ldx, nullptr, m, 0, 0,
                    prologue, prologue_w, eps, workspace, workspace_bytes, stream, &p);
}

extern "C" int qigen_gemv(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                          int64_t group, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                          float* y, int64_t ldy, int accumulate, int k_splits, void* stream) {
  return qigen_gemv_ex(qw, qsz, n, m, bits, group, x, x_dtype, tokens, ldx, y, ldy, accumulate,
                       k_splits, 0, nullptr, 0.f, nullptr, 0, stream);
}
