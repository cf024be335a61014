// Persistent multi-token GEMV (3..8 activation rows): the schedule of the
// decode stack (decode_stack.cu) applied to ONE quantized GEMV.
//
// The split-K GEMV (gemv.cu) at 4-8 tokens runs one 8-warp CTA per SM (its
// activation fragments fill shared memory), 2.6 waves of CTAs on the 65B decode
// shapes, and every CTA re-loads the fragments of its whole K chunk: 1.3-1.6
// TB/s (profiles/r02/gemv8_ncu.txt).  Here one 16-warp CTA per SM is resident
// (cooperative launch):
//   * the CTAs form ksl K-slab groups x G / ksl panel ranges; within a group
//     the (panel, superstep-of-the-slab) units, panel-major, are cut into equal
//     contiguous ranges, one per warp (host-built table, cached per shape);
//   * a CTA bulk-copies the activation digit records of its slab ONCE (written
//     by gemv.cu's act_prep kernels, which also apply the RMSNorm / SwiGLU
//     prologues) and streams its warps' weight ranges through per-warp TMA
//     rings;
//   * same arithmetic as gemv.cu (exact IMMA partials per exponent unit, f32
//     flush; kernelgen.py:227-240), NB n8 blocks of (token, digit) columns;
//   * the CTA adds its warps' segments of a panel in warp order and stores one
//     partial per (CTA, panel) (slot 2 slab, or 2 slab + 1 for the second CTA of
//     a panel; the CTA that covers a panel alone also zeroes the other slot);
//     after one grid barrier every CTA adds the 2 ksl slots of its share of y
//     in slot order.  Deterministic, no atomics.
#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "gemv_common.cuh"

namespace qigen {
namespace {

constexpr int kMW = 16;          // warps per CTA
constexpr int kMT = kMW * 32;
constexpr int kMSeg = 4;         // panel segments per warp
constexpr int kMRow = 36;        // table row: lo[17], first panel[16], panels, slab start, slab length

struct MtArgs {
  const char* qw;
  const char* qsz;
  const unsigned char* dig;  // act_prep layout: [KS * 8 steps][TP][16 uint2] | [KS * UPS units][TP] (xsum, scale)
  float* y;
  int64_t ldy, m;
  int KS, P, M, accumulate;
  int G, ksl, depth, sss;
  uint32_t slot_bytes, rec_dig, rec_fac;  // ring slot; record bytes per superstep: digits, factors
  uint32_t pstride;          // floats per partial slot (P * 16 * M)
  const uint32_t* ctab;      // [G][kMRow]
  float* part;               // [2 ksl][P * 16][M]
  unsigned int* bar;         // grid barrier counter (zero at launch)
};

__device__ __forceinline__ bool mt_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
#pragma unroll 1
  for (int i = 0; i < 300; ++i) {  // x 10 ms suspend hint
    uint32_t done = 0;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x989680u)
        : "memory");
    if (done) return true;
  }
  return false;
}

template <int BITS, int NB, int GPS>
__global__ void __launch_bounds__(kMT, 1) gemv_mt_kernel(const MtArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int TP = 2 * NB;
  constexpr int WB = BITS * 512, ZB = GPS * 128;
  constexpr int UPS = GPS > 2 ? GPS : 2, SPU = 8 / UPS;
  constexpr int AC = (NB <= 2 || BITS == 2) ? 2 : 1;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t cta = blockIdx.x, G = (uint32_t)a.G;
  const int depth = a.depth, sss = a.sss, M = a.M;
  const uint32_t slot_bytes = a.slot_bytes;

  uint32_t* row = (uint32_t*)smem;                                     // [kMRow]
  uint64_t* fullb = (uint64_t*)(smem + 256);                           // [warp][depth], then the record barrier
  unsigned char* rec = smem + 256 + (kMW * 8 + 1) * 8;                 // (depth <= 8)
  rec = (unsigned char*)(((uintptr_t)rec + 127) & ~(uintptr_t)127);
  for (int i = tid; i < kMRow; i += kMT) row[i] = a.ctab[(size_t)cta * kMRow + i];
  __syncthreads();
  const uint32_t s0 = row[34], Sk = row[35];
  const uint32_t dig_bytes = Sk * a.rec_dig, fac_bytes = Sk * a.rec_fac;
  unsigned char* facs = rec + ((dig_bytes + 127) & ~127u);
  unsigned char* rings = facs + ((fac_bytes + 127) & ~127u);           // [warp][depth][slot]
  float* wpart = (float*)(rings + (size_t)kMW * depth * slot_bytes);   // [warp][kMSeg][16][M]
  uint64_t* rbar = fullb + kMW * 8;
  if (tid == 0) {
    for (int i = 0; i < kMW * depth; ++i) mbar_init(&fullb[i], 1);
    mbar_init(rbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // this CTA's slab of the activation records
    mbar_expect_tx(rbar, dig_bytes + fac_bytes);
    const unsigned char* dsrc = a.dig + (size_t)s0 * a.rec_dig;
    for (uint32_t off = 0; off < dig_bytes; off += 32768)
      bulk_g2s(rec + off, dsrc + off, min(32768u, dig_bytes - off), rbar);
    bulk_g2s(facs, a.dig + (size_t)a.KS * a.rec_dig + (size_t)s0 * a.rec_fac, fac_bytes, rbar);
  }
  __syncthreads();

  unsigned char* ring = rings + (size_t)warp * depth * slot_bytes;
  uint64_t* full = fullb + warp * depth;
  // issue cursor (warp-uniform): stages of the warp's unit range
  const uint32_t lo = row[warp], hi = row[warp + 1];
  uint32_t c_u = lo, c_segend = (row[17 + warp] + 1) * Sk;
  const uint32_t jump = (uint32_t)a.KS - Sk;
  int islot = 0;
  const char *c_w, *c_z;
  {
    const uint32_t p = row[17 + warp];
    const size_t first = (size_t)p * a.KS + s0 + (lo - p * Sk);
    c_w = a.qw + first * WB;
    c_z = a.qsz + first * ZB;
  }
  auto issue_one = [&]() {
    if (c_u >= hi) return;
    const uint32_t nss = min((uint32_t)sss, min(hi, c_segend) - c_u);
    unsigned char* dst = ring + (size_t)islot * slot_bytes;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&full[islot], nss * (WB + ZB));
      bulk_g2s(dst, c_w, nss * WB, &full[islot]);
      bulk_g2s(dst + sss * WB, c_z, nss * ZB, &full[islot]);
    }
    if (++islot == depth) islot = 0;
    c_u += nss;
    c_w += nss * WB;
    c_z += nss * ZB;
    if (c_u == c_segend) {
      c_segend += Sk;
      c_w += (size_t)jump * WB;
      c_z += (size_t)jump * ZB;
    }
  };
  for (int i = 0; i < depth; ++i) issue_one();
  __syncwarp();
  if (!mt_wait(rbar, 0)) return;  // (records never arrived: give up rather than hang)

  // ---- main loop -----------------------------------------------------------------
  const int gq = lane >> 2, t = lane & 3;
  const float w_lo = (t & 1) ? 1.f : 65536.f;
  const float w_hi = w_lo * RowScale<BITS>::inv_hi;
  const bool xon = (t & 1) == 0;
  const int tcol = t >> 1;
  const uint2* bbase = (const uint2*)rec + (gq >> 2) * 16 + (gq & 3) * 4 + t;
  const float2* xs = (const float2*)facs;
  int wslot = 0, seg = 0;
  uint32_t wph = 0, u = lo, p = row[17 + warp];
  while (u < hi) {
    uint32_t s = u - p * Sk;
    const uint32_t seg_end = min(hi, (p + 1) * Sk);
    float yv[NB][2];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) yv[nb][0] = yv[nb][1] = 0.f;
    while (u < seg_end) {
      const uint32_t nss = min((uint32_t)sss, seg_end - u);
      if (!mt_wait(&full[wslot], wph)) return;
      const unsigned char* stg = ring + (size_t)wslot * slot_bytes;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j < (int)nss) {
          uint4 w[BITS];
#pragma unroll
          for (int v = 0; v < BITS; ++v) w[v] = ((const uint4*)(stg + j * WB))[v * 32 + lane];
          const float2* szs = (const float2*)(stg + sss * WB + j * ZB);
          const uint2* bs = bbase + (size_t)(s + j) * 8 * TP * 16;
          int acc[AC][NB][4];
#pragma unroll
          for (int c = 0; c < AC; ++c)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) acc[c][nb][0] = acc[c][nb][1] = acc[c][nb][2] = acc[c][nb][3] = 0;
#pragma unroll
          for (int sl = 0; sl < 8; ++sl) {
            uint32_t af[4];
            extract<BITS>(w, sl, af);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) imma(acc[sl % AC][nb], af, bs[(sl * TP + 2 * nb) * 16]);
            if ((sl + 1) % SPU == 0) {
              const int uj = (sl + 1) / SPU - 1;
              const int gi = GPS >= UPS ? uj : 0;
              const float2 sz0 = szs[gi * 16 + gq], sz1 = szs[gi * 16 + gq + 8];
              const uint32_t uu = (s + j) * UPS + uj;  // unit within the slab
#pragma unroll
              for (int nb = 0; nb < NB; ++nb) {
                const float2 xv = xs[uu * TP + 2 * nb + tcol];
                const float X = xon ? xv.x : 0.f, sc = xv.y;
                int c0 = acc[0][nb][0], c1 = acc[0][nb][1], c2 = acc[0][nb][2], c3 = acc[0][nb][3];
#pragma unroll
                for (int c = 1; c < AC; ++c) {
                  constexpr int sh = BITS == 2 ? 4 : 0;  // 2-bit odd steps carry an extra x16
                  c0 += acc[c][nb][0] >> sh; c1 += acc[c][nb][1] >> sh;
                  c2 += acc[c][nb][2] >> sh; c3 += acc[c][nb][3] >> sh;
                }
                const float q0 = (float)(c0 * 256 + c1), q1 = (float)(c2 * 256 + c3);
                yv[nb][0] = fmaf(sz0.x * sc, fmaf(-sz0.y, X, q0 * w_lo), yv[nb][0]);
                yv[nb][1] = fmaf(sz1.x * sc, fmaf(-sz1.y, X, q1 * w_hi), yv[nb][1]);
#pragma unroll
                for (int c = 0; c < AC; ++c)
                  acc[c][nb][0] = acc[c][nb][1] = acc[c][nb][2] = acc[c][nb][3] = 0;
              }
            }
          }
        }
      }
      __syncwarp();
      issue_one();
      if (++wslot == depth) {
        wslot = 0;
        wph ^= 1u;
      }
      u += nss;
      s += nss;
    }
    // digit-pair lanes combined; lane (gq, t even) holds token 2 nb + (t >> 1), rows gq, gq + 8
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const float v0 = yv[nb][0] + __shfl_xor_sync(0xffffffffu, yv[nb][0], 1);
      const float v1 = yv[nb][1] + __shfl_xor_sync(0xffffffffu, yv[nb][1], 1);
      const int tk = 2 * nb + (t >> 1);
      if ((t & 1) == 0 && tk < M && seg < kMSeg) {
        float* dst = wpart + ((size_t)(warp * kMSeg + seg) * 16) * M;
        dst[gq * M + tk] = v0;
        dst[(gq + 8) * M + tk] = v1;
      }
    }
    ++seg;
    ++p;
  }
  __syncthreads();
  // ---- the CTA's partial of every panel it touched ------------------------------------
  {
    const uint32_t LO = row[0], HI = row[16], pf = row[17], npan = row[33];
    const uint32_t slab = cta / (G / (uint32_t)a.ksl);
    const uint32_t per = 16u * (uint32_t)M;
    for (uint32_t idx = tid; idx < npan * per; idx += kMT) {
      const uint32_t pp = pf + idx / per, e = idx % per;  // e = row * M + token
      const uint32_t ua = max(LO, pp * Sk), ub = min(HI, (pp + 1) * Sk) - 1;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kMW; ++w) {
        const uint32_t lw = row[w], hw = row[w + 1];
        if (hw > lw && hw > ua && lw <= ub)
          acc += wpart[((size_t)(w * kMSeg + (pp - row[17 + w])) * 16) * M + e];
      }
      const bool second = pp * Sk < LO;                       // the panel started in the previous CTA
      const bool alone = !second && (pp + 1) * Sk <= HI;      // this CTA covers it alone
      float* dst = a.part + (size_t)(2 * slab) * a.pstride + (size_t)pp * per + e;
      if (second) {
        dst[a.pstride] = acc;
      } else {
        dst[0] = acc;
        if (alone) dst[a.pstride] = 0.f;
      }
    }
  }
  // ---- grid barrier -------------------------------------------------------------------
  __syncthreads();
  if (tid == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned int spins = 0;
    for (;;) {
      unsigned int v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
      if (v >= G) break;
      if ((++spins & 1023u) == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 2000000000ull) break;  // never hang the GPU
      }
    }
  }
  __syncthreads();
  // ---- y = sum of the slots, in slot order -------------------------------------------------
  {
    const int64_t n = a.m * M;  // elements (column, token): index col * M + token
    for (int64_t i = (int64_t)cta * kMT + tid; i < n; i += (int64_t)G * kMT) {
      float v = 0.f;
      for (int sl = 0; sl < 2 * a.ksl; ++sl) v += __ldcg(a.part + (size_t)sl * a.pstride + i);
      const int64_t col = i / M, tk = i % M;
      float* dst = a.y + tk * a.ldy + col;
      *dst = a.accumulate ? *dst + v : v;
    }
  }
}

// The static partition of one shape on this device (table on the device).
struct MtPlan {
  int G = 0, ksl = 0, depth = 0, sss = 0;
  uint32_t slot_bytes = 0, smem = 0;
  uint32_t* ctab = nullptr;
};

using MtKey = std::tuple<int, int, int, int, int, int, int>;  // device, KS, P, bits, gps, TP, M
std::mutex g_mt_mutex;
std::map<MtKey, MtPlan> g_mt_plans;

uint32_t lo_of(uint32_t gw, uint32_t T, uint32_t GW) { return (uint32_t)((uint64_t)gw * T / GW); }
uint32_t warp_of(uint32_t u, uint32_t T, uint32_t GW) { return (uint32_t)((((uint64_t)u + 1) * GW - 1) / T); }

// ksl = 0 in the result: the shape does not fit (caller keeps the split-K GEMV).
MtPlan mt_plan(int dev, int sms, int KS, int P, int bits, int gps, int TP, int M) {
  const MtKey key{dev, KS, P, bits, gps, TP, M};
  std::lock_guard<std::mutex> lock(g_mt_mutex);
  auto it = g_mt_plans.find(key);
  if (it != g_mt_plans.end()) return it->second;
  MtPlan pl;
  const int ups = gps > 2 ? gps : 2;
  const uint32_t rec_dig = 8u * TP * 128, rec_fac = (uint32_t)ups * TP * 8;
  const size_t budget = 227 * 1024;
  const int G0 = std::min(sms, P);
  for (int ksl : {4, 2, 1}) {
    if (G0 % ksl || KS < ksl || P < G0 / ksl) continue;
    const int GJ = G0 / ksl;
    const uint32_t GWJ = (uint32_t)GJ * kMW;
    const uint32_t skmax = (uint32_t)((KS + ksl - 1) / ksl);
    const size_t recb = ((size_t)skmax * rec_dig + 127) / 128 * 128 + ((size_t)skmax * rec_fac + 127) / 128 * 128;
    const size_t fixed = 256 + (kMW * 8 + 1) * 8 + 128 + recb + (size_t)kMW * kMSeg * 16 * M * 4;
    int sss = 2, depth = 0;
    size_t slot = 0;
    for (; sss >= 1; --sss) {
      slot = (size_t)sss * (bits * 512 + gps * 128);
      for (int dd = 4; dd >= 2; --dd)
        if (fixed + (size_t)kMW * dd * slot <= budget) {
          depth = dd;
          break;
        }
      if (depth >= 2) break;
    }
    if (depth < 2) continue;
    // the partition: every panel of a slab within at most two CTAs, few segments per warp
    std::vector<uint32_t> ctab((size_t)G0 * kMRow, 0u);
    bool fits = true;
    for (int k = 0; k < ksl && fits; ++k) {
      const uint32_t s0 = (uint32_t)((uint64_t)k * KS / ksl), s1 = (uint32_t)((uint64_t)(k + 1) * KS / ksl);
      const uint32_t Sk = s1 - s0, T = (uint32_t)P * Sk;
      for (uint32_t p = 0; fits && p < (uint32_t)P; ++p)
        if (warp_of(p * Sk + Sk - 1, T, GWJ) / kMW - warp_of(p * Sk, T, GWJ) / kMW > 1) fits = false;
      for (int j = 0; fits && j < GJ; ++j) {
        uint32_t* row = &ctab[(size_t)(k * GJ + j) * kMRow];
        for (int w = 0; w <= kMW; ++w) row[w] = lo_of((uint32_t)j * kMW + w, T, GWJ);
        for (int w = 0; w < kMW; ++w) {
          row[17 + w] = row[w] / Sk;
          if (row[w + 1] > row[w] && (row[w + 1] - 1) / Sk - row[17 + w] + 1 > (uint32_t)kMSeg) fits = false;
        }
        row[33] = row[16] > row[0] ? (row[16] - 1) / Sk - row[17] + 1 : 0u;
        row[34] = s0;
        row[35] = Sk;
      }
    }
    if (!fits) continue;
    if (cudaMalloc((void**)&pl.ctab, ctab.size() * 4) != cudaSuccess ||
        cudaMemcpy(pl.ctab, ctab.data(), ctab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      pl.ctab = nullptr;
      break;
    }
    pl.G = G0;
    pl.ksl = ksl;
    pl.depth = depth;
    pl.sss = sss;
    pl.slot_bytes = (uint32_t)slot;
    pl.smem = (uint32_t)(fixed + (size_t)kMW * depth * slot);
    break;
  }
  g_mt_plans[key] = pl;
  return pl;
}

}  // namespace

// Tuning aid: 0 disables the persistent multi-token GEMV (per calling thread).
thread_local int g_mt_on = 1;

// The multi-token GEMV on prepared activation records (gemv.cu launch_cfg).
// Returns -1 when the shape is left to the split-K kernel.
template <int BITS, int NB, int GPS>
int launch_gemv_mt(const char* qw, const char* qsz, const unsigned char* dig, float* y, int64_t ldy,
                   int64_t m, int KS, int P, int M, int accumulate, cudaStream_t stream) {
  if (!g_mt_on) return -1;
  int dev = 0, sms = 0;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  constexpr int TP = 2 * NB;
  const MtPlan pl = mt_plan(dev, sms, KS, P, BITS, GPS, TP, M);
  if (pl.ksl == 0 || !pl.ctab) return -1;
  static OncePerDevice once;
  const int rc = once.run([]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(gemv_mt_kernel<BITS, NB, GPS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    return QIGEN_OK;
  });
  if (rc) return rc;
  constexpr int UPS = GPS > 2 ? GPS : 2;
  MtArgs a{};
  a.qw = qw;
  a.qsz = qsz;
  a.dig = dig;
  a.y = y;
  a.ldy = ldy;
  a.m = m;
  a.KS = KS;
  a.P = P;
  a.M = M;
  a.accumulate = accumulate;
  a.G = pl.G;
  a.ksl = pl.ksl;
  a.depth = pl.depth;
  a.sss = pl.sss;
  a.slot_bytes = pl.slot_bytes;
  a.rec_dig = 8u * TP * 128;
  a.rec_fac = (uint32_t)UPS * TP * 8;
  a.pstride = (uint32_t)P * 16u * (uint32_t)M;
  a.ctab = pl.ctab;
  // partial slots + the barrier word: stream-ordered scratch, freed behind the kernel
  const size_t part_bytes = (size_t)2 * pl.ksl * a.pstride * 4;
  unsigned char* scratch = nullptr;
  int st = scratch_alloc(stream, part_bytes + 256, &scratch);
  if (st) return st;
  a.part = (float*)scratch;
  a.bar = (unsigned int*)(scratch + part_bytes);
  cudaError_t e = cudaMemsetAsync(a.bar, 0, 4, stream);
  if (e == cudaSuccess) {
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeCooperative;
    at.val.cooperative = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.G, 1, 1);
    cfg.blockDim = dim3(kMT, 1, 1);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, gemv_mt_kernel<BITS, NB, GPS>, a);
  }
  const cudaError_t f = cudaFreeAsync(scratch, stream);
  QIGEN_CUDA_RET(e);
  QIGEN_CUDA_RET(f);
  return QIGEN_OK;
}

#define QIGEN_MT_INST(B, N, G)                                                                   \
  template int launch_gemv_mt<B, N, G>(const char*, const char*, const unsigned char*, float*,    \
                                       int64_t, int64_t, int, int, int, int, cudaStream_t);
QIGEN_MT_INST(2, 2, 2) QIGEN_MT_INST(2, 2, 4) QIGEN_MT_INST(2, 2, 8)
QIGEN_MT_INST(2, 4, 2) QIGEN_MT_INST(2, 4, 4) QIGEN_MT_INST(2, 4, 8)
QIGEN_MT_INST(3, 2, 2) QIGEN_MT_INST(3, 2, 4) QIGEN_MT_INST(3, 2, 8)
QIGEN_MT_INST(3, 4, 2) QIGEN_MT_INST(3, 4, 4) QIGEN_MT_INST(3, 4, 8)
QIGEN_MT_INST(4, 2, 2) QIGEN_MT_INST(4, 2, 4) QIGEN_MT_INST(4, 2, 8)
QIGEN_MT_INST(4, 4, 2) QIGEN_MT_INST(4, 4, 4) QIGEN_MT_INST(4, 4, 8)
#undef QIGEN_MT_INST

}  // namespace qigen

extern "C" int qigen_debug_gemv_mt(int on) {
  qigen::g_mt_on = on;
  return QIGEN_OK;
}
