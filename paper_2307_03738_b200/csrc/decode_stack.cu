// Persistent decode stack: every layer of a LLaMA-architecture decode step
// (batch 1, one GPU) as ONE launch.
//
// The per-op chain of the decode driver (decode.py) is latency-bound: each of
// the five kernels of a layer pays its launch boundary, its activation
// prologue and its split-K tail on the critical path.  Here one
// CTA (16 warps) per SM stays resident for the whole step (cooperative launch):
//   * the four quantized linears of every layer (fused QKV, o_proj, fused
//     gate|up, down_proj; same arithmetic as gemv.cu / gemv_grouped.cu: the
//     reference factorisation kernelgen.py:227-240 with exact IMMA partials)
//     and the attention in between are PHASES;
//   * per GEMV phase the CTAs form ksl groups (K slabs) x G / ksl panel ranges:
//     group k owns the k-th slab of the phase's K supersteps, and within a group
//     the (panel, superstep-of-the-slab) units, in panel-major order, are cut
//     into equal contiguous ranges, one per warp (host-built tables).  So a CTA
//     needs only 1 / ksl of each activation vector (its prologue work and its
//     shared-memory records shrink by ksl), and every warp streams its range
//     through its own ring of TMA bulk-copy stages.  The schedule is static, so
//     a warp's issue cursor simply runs ahead into the NEXT phases (and
//     layers): the first stages of a phase are in shared memory before its
//     inputs exist, and the rings never drain;
//   * a warp's partial sums of a panel are reduced inside the CTA in warp
//     order and stored as one partial per (CTA, panel) ("slot": 2 per slab, a
//     panel of a slab spans at most two CTAs); the consumer of the vector adds
//     the slots in a fixed order.  No atomics: deterministic;
//   * the consumer side of each phase ("prologue") is computed by every CTA
//     for its slab straight into shared memory: residual add, RMSNorm weight,
//     SwiGLU or the attention combine, then the fixed-point digit records
//     (1152 B per 256 rows).  The residual rows of the slab stay in the CTA's
//     shared memory.  The 1/rms of an RMSNorm is applied to the GEMV's OUTPUT
//     by its consumer (the GEMV is linear), from the per-slab sums of squares
//     the groups publish;
//   * attention: a head's cached positions are split over cph CTAs; a warp
//     keeps an online-softmax state over its positions, the CTA combines its
//     warps and stores one partial per (head, chunk); the o_proj prologue
//     combines them;
//   * NO grid barrier between phases (1.3-1.7 us each on 148 CTAs): every value
//     that crosses CTAs travels as an 8-byte {value, flag} pair, polled by its
//     reader ("flag in data", see below).
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "gemv_common.cuh"

namespace qigen {

extern thread_local unsigned long long* g_trace;  // gemv.cu (qigen_debug_trace)

namespace {

constexpr int kSWarps = 16;
constexpr int kSThreads = kSWarps * 32;
constexpr int kSRecDig = 1024;              // digit bytes per superstep record (1 token)
constexpr int kSRec = kSRecDig + 8 * 16;    // + up to 8 units x {A, B, scale, 0}
constexpr int kMaxSeg = 8;                  // panel segments per warp and phase
constexpr int kMaxKsl = 4;                  // K slabs (CTA groups)
constexpr int kMaxSlot = 2;                 // partials per output column and slab
constexpr int kAttRow = 264;                // floats per attention partial: {value, flag} pairs of
                                            // acc[128], m, l (+ pad); also the warps' smem rows
constexpr int kHD = 128;                    // head dimension
constexpr int kMaxCph = 4;                  // position chunks (CTAs) per head
constexpr int kAttSm = 132;                 // floats per warp partial in shared memory: acc[128], m, l
constexpr int kAttScratch = (4 * kHD + kSWarps * kAttSm) * 4;
constexpr int kLtab = 12;                   // pointers per layer in the shared-memory table
constexpr int kCrow = 38;  // per phase: lo[17], first panel[16], panels, slab start, slab length,
                           // slab index, CTA index within the slab group
constexpr int kCtab = 4 * kCrow;

struct SLayer {          // device table entry
  const char* qw[4];     // qkv, o, gate|up, down: panel words
  const char* qsz[4];    // their (s, z)
  const float* n1;
  const float* n2;       // RMSNorm weights
  __half* kc;
  __half* vc;            // [H][ctx][128]
};

struct SPlan {
  const SLayer* layers;
  int L, d, H, ffn, ctx, cph, G;
  int ksl[4];                  // K slabs (CTA groups) of each GEMV phase
  uint32_t P[4], S[4], T[4];   // panels, supersteps, units of the four GEMV phases
  uint32_t pstride[4];         // floats per partial slot (P * 16)
  float* part[4];              // [3 buffer sets][2 ksl slots][P * 16] {value, flag}
  float* attp;                 // [3][H][cph][kAttRow]
  const uint32_t* ctab;        // [G][kCtab]: per CTA and phase, lo[17] | first panel[16] | panels
  const uint32_t* two;         // bit p of phase ph (word offset two_off[ph]): panel spans two CTAs
  uint32_t two_off[4], two_wp[4], two_words;  // per phase: word offset, words per slab
  float* ssq;                  // [3][2][kMaxKsl] {value, flag}: per-slab sums of squares (norm1, norm2 input)
  uint32_t own_q[4];           // residual items (4 floats) each CTA of a slab group stores
  uint32_t pf_units[4];        // units of a phase each warp prefetches into L2 one phase ahead
  unsigned int* bar;           // [0] layers finished (all CTAs), [1] error word, [2] exit counter,
                               // [3] launch epoch
  const float* h_in;
  float* h_out;
  const float* cosv;
  const float* sinv;
  int pos;
  float scale, eps;
  int depth, sss;              // ring stages per warp, supersteps per stage
  int mode;                    // tuning: 1 = stream the weights without the math
  uint32_t slot_bytes, xrec_bytes, hp_bytes;
  unsigned long long* trace;   // optional: per barrier and CTA (arrive, pass) in ns
};

__device__ __forceinline__ void imma_z(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y), "r"(0));
}

// One 256-row superstep of one panel against the single token's digit record
// (gemv_grouped.cu group_superstep with a one-token record: the n8 columns 4-7
// repeat the token's digits and are ignored).
template <int BITS, int GPS>
__device__ __forceinline__ void stack_superstep(const uint4 (&w)[BITS], const float2* szs,
                                                const unsigned char* rec, float (&yv)[2]) {
  constexpr int UPS = GPS > 2 ? GPS : 2;
  constexpr int SPU = 8 / UPS;
  const int lane = threadIdx.x & 31, gq = lane >> 2, t = lane & 3;
  const uint2* bs = (const uint2*)rec + (gq & 3) * 4 + t;
  const float2* ab = (const float2*)(rec + kSRecDig) + (t & 1);
  int acc[2][4];
#pragma unroll
  for (int sl = 0; sl < 8; ++sl) {
    uint32_t af[4];
    extract<BITS>(w, sl, af);
    if (sl % SPU < 2) imma_z(acc[sl & 1], af, bs[sl * 16]);
    else imma(acc[sl & 1], af, bs[sl * 16]);
    if ((sl + 1) % SPU == 0) {
      const int uj = (sl + 1) / SPU - 1;
      const int gi = GPS >= UPS ? uj : 0;
      const float2 sz0 = szs[gi * 16 + gq], sz1 = szs[gi * 16 + gq + 8];
      const float2 f = ab[uj * 2];
      constexpr int sh = BITS == 2 ? 4 : 0;  // 2-bit odd steps carry an extra x16
      int c0, c1, c2, c3;
      if (SPU == 1) {
        const int k = sl & 1, shk = k ? sh : 0;
        c0 = acc[k][0] >> shk; c1 = acc[k][1] >> shk; c2 = acc[k][2] >> shk; c3 = acc[k][3] >> shk;
      } else {
        c0 = acc[0][0] + (acc[1][0] >> sh); c1 = acc[0][1] + (acc[1][1] >> sh);
        c2 = acc[0][2] + (acc[1][2] >> sh); c3 = acc[0][3] + (acc[1][3] >> sh);
      }
      const float q0 = (float)(c0 * 256 + c1), q1 = (float)(c2 * 256 + c3);
      yv[0] = fmaf(sz0.x, fmaf(-sz0.y, f.y, f.x * q0), yv[0]);
      yv[1] = fmaf(sz1.x, fmaf(-sz1.y, f.y, (f.x * RowScale<BITS>::inv_hi) * q1), yv[1]);
    }
  }
}

// Unit ranges: warp gw of GW owns [lo(gw), lo(gw + 1)) of T units.
__host__ __device__ __forceinline__ uint32_t lo_of(uint32_t gw, uint32_t T, uint32_t GW) {
  return (uint32_t)((uint64_t)gw * T / GW);
}
// (host guarantees (T + 1) * GW < 2^32)
__host__ __device__ __forceinline__ uint32_t warp_of(uint32_t u, uint32_t T, uint32_t GW) {
  return ((u + 1) * GW - 1) / T;
}

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg((const float4*)p); }
__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}

__device__ __forceinline__ bool mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
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

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- flagged data ("flag in data"): every value crossing CTAs travels as an
// 8-byte {value, flag} pair written with ONE store; the reader polls the pair
// itself until the flag is the one of the current (launch, layer).  No fence, no
// separate signal, no grid barrier: the hand-off costs one store plus one load
// round trip (a grid barrier costs 1.3-1.7 us on 148 CTAs, tools/ubench/gridbar.cu).
__device__ __forceinline__ float4 ld_pair2(const float* p) {  // two pairs: {v0, f0, v1, f1}
  float4 v;
  asm volatile("ld.volatile.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_pair(const float* p) {
  float2 v;
  asm volatile("ld.volatile.global.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_pair(float* p, float v, uint32_t flag) {
  asm volatile("st.volatile.global.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(v), "f"(__uint_as_float(flag))
               : "memory");
}
__device__ __forceinline__ bool flags_ok(const float4& a, uint32_t fl) {
  return __float_as_uint(a.y) == fl && __float_as_uint(a.w) == fl;
}

template <int BITS, int GPS>
__global__ void __launch_bounds__(kSThreads, 1) decode_stack_kernel(const SPlan pl) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int WB = BITS * 512, ZB = GPS * 128;
  constexpr int UPS = GPS > 2 ? GPS : 2, IPU = 64 / UPS;
  const int tid = threadIdx.x, lane = tid & 31;
  // (the shuffle tells the compiler the warp index is warp-uniform: the issue
  // cursor below then lives in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t cta = blockIdx.x, G = (uint32_t)pl.G;
  const int depth = pl.depth, sss = pl.sss;
  const uint32_t slot_bytes = pl.slot_bytes;

  unsigned char* xrec = smem;                                          // digit records / attention scratch
  unsigned char* rings = smem + pl.xrec_bytes;                         // [warp][depth][slot]
  float* wpart = (float*)(rings + (size_t)kSWarps * depth * slot_bytes);  // [warp][kMaxSeg][16]
  float* red = wpart + kSWarps * kMaxSeg * 16;                         // [32]
  uint64_t* fullb = (uint64_t*)(red + 32);                             // [warp][depth]
  const char** ltab = (const char**)(fullb + kSWarps * depth);  // [L][12]: qw[4], qsz[4], n1, n2, kc, vc
  uint32_t* ctab = (uint32_t*)(ltab + pl.L * kLtab);            // this CTA's unit ranges
  uint32_t* twob = ctab + kCtab;                                // two-CTA panel bits
  float* hp = (float*)(twob + ((pl.two_words + 3) & ~3u));      // the residual rows of this CTA's slab

  static_assert(sizeof(SLayer) == kLtab * sizeof(void*), "layer table entry");
  for (int i = tid; i < pl.L * kLtab; i += kSThreads)
    ltab[i] = ((const char* const*)pl.layers)[i];
  for (int i = tid; i < kCtab; i += kSThreads) ctab[i] = pl.ctab[(size_t)cta * kCtab + i];
  for (uint32_t i = tid; i < pl.two_words; i += kSThreads) twob[i] = pl.two[i];
  if (tid == 0) {
    for (int i = 0; i < kSWarps * depth; ++i) mbar_init(&fullb[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // flags of this launch: epoch * L + layer + 1 (the epoch advances at kernel exit)
  const uint32_t fl0 = __ldcg(pl.bar + 3) * (uint32_t)pl.L + 1u;
  __syncthreads();

  unsigned char* ring = rings + (size_t)warp * depth * slot_bytes;
  uint64_t* full = fullb + warp * depth;

  // ---- issue cursor: the warp's static stream of weight stages over all phases
  // of all layers, kept identically by every lane (warp-uniform state); one
  // elected lane issues the copies.  Units are slab-local: unit u = (panel p,
  // local superstep u - p Sk); the weights of panel p start S supersteps apart.
  int c_l = 0, c_ph = -1, islot = 0;
  uint32_t c_u = 0, c_hi = 0, c_segend = 0, c_sk = 0, c_jump = 0;
  bool c_done = false;
  const char *c_w = nullptr, *c_z = nullptr;
  auto next_phase = [&]() {
    for (;;) {
      if (++c_ph == 4) {
        c_ph = 0;
        if (++c_l == pl.L) {
          c_done = true;
          return;
        }
      }
      const uint32_t* row = ctab + c_ph * kCrow;
      c_u = row[warp];
      c_hi = row[warp + 1];
      if (c_hi > c_u) {
        const uint32_t p = row[17 + warp], s0 = row[34];
        c_sk = row[35];
        c_segend = (p + 1) * c_sk;
        c_jump = pl.S[c_ph] - c_sk;  // supersteps of other slabs between two panels
        const size_t first = (size_t)p * pl.S[c_ph] + s0 + (c_u - p * c_sk);
        c_w = ltab[c_l * kLtab + c_ph] + first * WB;
        c_z = ltab[c_l * kLtab + 4 + c_ph] + first * ZB;
        return;
      }
    }
  };
  auto issue_one = [&]() {
    if (c_done) return;
    const uint32_t nss = min((uint32_t)sss, min(c_hi, c_segend) - c_u);
    unsigned char* dst = ring + (size_t)islot * slot_bytes;
    uint64_t* bar = &full[islot];
    if (lane == 0) {
      // (the slot's last readers are behind a __syncwarp: order their generic
      // reads before the async-proxy writes)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(bar, nss * (WB + ZB));
      bulk_g2s(dst, c_w, nss * WB, bar);
      bulk_g2s(dst + sss * WB, c_z, nss * ZB, bar);
    }
    if (++islot == depth) islot = 0;
    c_u += nss;
    c_w += nss * WB;
    c_z += nss * ZB;
    if (c_u == c_hi) {
      next_phase();
    } else if (c_u == c_segend) {
      c_segend += c_sk;
      c_w += (size_t)c_jump * WB;
      c_z += (size_t)c_jump * ZB;
    }
  };
  next_phase();
  for (int i = 0; i < depth; ++i) issue_one();
  __syncwarp();

  // ---- trace / waiting ----------------------------------------------------------
  unsigned int nph = 0;  // phases done (5 per layer)
  if (pl.trace && tid == 0) {  // trace slot 1 of phase 0: the SM this CTA runs on
    unsigned int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    pl.trace[(size_t)cta * 4 + 1] = smid;
  }
  auto stamp = [&](int i) {  // trace point i of the current phase
    if (pl.trace && tid == 0) pl.trace[((size_t)nph * G + cta) * 4 + i] = gtime();
  };
  // a poll loop gives up after 2 s (error word bit 0) instead of hanging the GPU
  auto spin_guard = [&](uint32_t& spins, unsigned long long& t0) {
    if ((++spins & 255u) != 0) return false;
    if (t0 == 0) {
      t0 = gtime();
      return false;
    }
    if (gtime() - t0 < 2000000000ull) return false;
    atomicOr(pl.bar + 1, 1u);
    return true;
  };

  // A column block c .. c + 3 of a phase's output lies in one panel; each K slab
  // contributed one partial (slot 2k) or two (2k + 1 too, when the panel spans
  // two CTAs of group k; host-built bit table), as {value, flag} pairs in the
  // buffer set `bs` (layer % 3).  Polls until every pair carries flag fl; the
  // slots are added in a fixed order.  Called by whole warps.
  auto slot_sum4 = [&](int ph, uint32_t c, uint32_t fl, int bs) {
    const uint32_t p = c >> 4;
    const size_t st = (size_t)pl.pstride[ph] * 2;
    const uint32_t* tb = twob + pl.two_off[ph] + (p >> 5);
    const int ksl = pl.ksl[ph];
    const float* src = pl.part[ph] + (size_t)bs * (2 * ksl) * st + (size_t)c * 2;
    float4 r;
    uint32_t spins = 0;
    unsigned long long t0 = 0;
    for (;;) {
      bool ok = true;
      r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int k = 0; k < kMaxKsl; ++k) {
        if (k < ksl) {
          const bool two = (tb[k * pl.two_wp[ph]] >> (p & 31)) & 1u;
          const float4 x0 = ld_pair2(src + (size_t)(2 * k) * st), x1 = ld_pair2(src + (size_t)(2 * k) * st + 4);
          float4 y0 = make_float4(0.f, __uint_as_float(fl), 0.f, __uint_as_float(fl)), y1 = y0;
          if (two) {
            y0 = ld_pair2(src + (size_t)(2 * k + 1) * st);
            y1 = ld_pair2(src + (size_t)(2 * k + 1) * st + 4);
          }
          ok = ok && flags_ok(x0, fl) && flags_ok(x1, fl) && flags_ok(y0, fl) && flags_ok(y1, fl);
          r.x += x0.x; r.y += x0.z; r.z += x1.x; r.w += x1.z;
          r.x += y0.x; r.y += y0.z; r.z += y1.x; r.w += y1.z;
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
      if (spin_guard(spins, t0)) break;
    }
    return r;
  };
  auto slot_sum1 = [&](int ph, uint32_t c, uint32_t fl, int bs) {  // one column
    const uint32_t p = c >> 4;
    const size_t st = (size_t)pl.pstride[ph] * 2;
    const uint32_t* tb = twob + pl.two_off[ph] + (p >> 5);
    const int ksl = pl.ksl[ph];
    const float* src = pl.part[ph] + (size_t)bs * (2 * ksl) * st + (size_t)c * 2;
    float r;
    uint32_t spins = 0;
    unsigned long long t0 = 0;
    for (;;) {
      bool ok = true;
      r = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxKsl; ++k) {
        if (k < ksl) {
          const bool two = (tb[k * pl.two_wp[ph]] >> (p & 31)) & 1u;
          const float2 x = ld_pair(src + (size_t)(2 * k) * st);
          float2 y = make_float2(0.f, __uint_as_float(fl));
          if (two) y = ld_pair(src + (size_t)(2 * k + 1) * st);
          ok = ok && __float_as_uint(x.y) == fl && __float_as_uint(y.y) == fl;
          r += x.x;
          r += y.x;
        }
      }
      if (__all_sync(0xffffffffu, ok)) break;
      if (spin_guard(spins, t0)) break;
    }
    return r;
  };
  // 1 / rms of a residual from the per-slab sums of squares its prologue (of
  // phase 0: norm1, phase 2: norm2) published for this layer.  Whole warps.
  auto rinv_of = [&](int which, uint32_t fl, int bs) {
    const float* src = pl.ssq + ((size_t)bs * 2 + which) * kMaxKsl * 2;
    float ssum;
    uint32_t spins = 0;
    unsigned long long t0 = 0;
    for (;;) {
      bool ok = true;
      ssum = 0.f;
#pragma unroll
      for (int k = 0; k < kMaxKsl; ++k)
        if (k < pl.ksl[2 * which]) {
          const float2 x = ld_pair(src + 2 * k);
          ok = ok && __float_as_uint(x.y) == fl;
          ssum += x.x;
        }
      if (__all_sync(0xffffffffu, ok)) break;
      if (spin_guard(spins, t0)) break;
    }
    return rsqrtf(ssum / (float)pl.d + pl.eps);
  };

  // Digitise this CTA's K slab of a phase's input into the shared-memory
  // records: item it = rows 4 it .. 4 it + 3 (absolute), record of local
  // superstep (it >> 6) - s0.  load(it) fetches the item's inputs (addresses
  // clamped into the vector; it may poll), finish(it, raw, v) turns them into
  // the four values (zeros beyond K).
  auto digitize_rows = [&](int ph, auto&& load, auto&& finish) {
    const uint32_t umask = IPU == 32 ? 0xffffffffu : ((1u << IPU) - 1u) << (lane & ~(IPU - 1));
    const int s0 = (int)ctab[ph * kCrow + 34], sk = (int)ctab[ph * kCrow + 35];
    const int itb = s0 * 64, nit = itb + sk * 64;
    for (int it0 = itb + warp * 32; it0 < nit; it0 += kSThreads) {
      const int it = it0 + lane;
      const auto r = load(it);
      float v[4];
      finish(it, r, v);
      const Digits dg = digitize<IPU>(v, umask);
      unsigned char* rec = xrec + (size_t)((it >> 6) - s0) * kSRec;
      store_digits((uint32_t*)rec, (it >> 3) & 7, 0, 1, it & 7, dg);
      if ((it % IPU) == 0)
        ((float4*)(rec + kSRecDig))[(it & 63) / IPU] =
            make_float4(dg.scale * 65536.f, dg.xsum * dg.scale, dg.scale, 0.f);
    }
  };
  // block sum of a per-thread value (ends with a CTA barrier: also publishes
  // the records written before it)
  auto block_sum = [&](float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < kSWarps; ++w) s += red[w];
    return s;
  };

  // L2 prefetch of this warp's unit range of GEMV phase (l, ph), at most
  // pl.pf_units[ph] units: issued one phase ahead, so HBM keeps streaming through
  // the hand-offs between phases and the ring copies of that phase hit L2.
  auto prefetch_phase = [&](int l, int ph) {
    if (l >= pl.L || lane != 0) return;
    const uint32_t* row = ctab + ph * kCrow;
    const uint32_t Sk = row[35], S = pl.S[ph];
    // (the ring already holds / has requested the first depth * sss units)
    uint32_t u = row[warp] + (uint32_t)(depth * sss);
    const uint32_t hi = min(row[warp + 1], u + pl.pf_units[ph]);
    if (u >= hi) return;
    uint32_t p = u / Sk;
    const char* w = ltab[l * kLtab + ph];
    const char* z = ltab[l * kLtab + 4 + ph];
    while (u < hi) {
      const uint32_t seg_end = min(hi, (p + 1) * Sk), n = seg_end - u;
      const size_t first = (size_t)p * S + row[34] + (u - p * Sk);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w + first * WB), "r"(n * WB) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(z + first * ZB), "r"(n * ZB) : "memory");
      u = seg_end;
      ++p;
    }
  };

  // ---- one GEMV phase: consume this warp's unit range ----------------------------
  int wslot = 0;
  uint32_t wph = 0;
  auto gemv_phase = [&](int ph, uint32_t fl, int bs, int nl) {
    const uint32_t* row = ctab + ph * kCrow;
    const uint32_t Sk = row[35];
    const uint32_t lo = row[warp], hi = row[warp + 1];
    uint32_t u = lo, p = row[17 + warp];
    int seg = 0;
    while (u < hi) {
      uint32_t s = u - p * Sk;  // local superstep = record index
      const uint32_t seg_end = min(hi, (p + 1) * Sk);
      float yv[2] = {0.f, 0.f};
      while (u < seg_end) {
        const uint32_t nss = min((uint32_t)sss, seg_end - u);
        if (!mbar_wait_bounded(&full[wslot], wph)) atomicOr(pl.bar + 1, 2u);
        const unsigned char* stg = ring + (size_t)wslot * slot_bytes;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j < (int)nss && pl.mode != 1) {  // (mode 1: the copies alone)
            uint4 w[BITS];
#pragma unroll
            for (int v = 0; v < BITS; ++v) w[v] = ((const uint4*)(stg + j * WB))[v * 32 + lane];
            stack_superstep<BITS, GPS>(w, (const float2*)(stg + sss * WB + j * ZB),
                                       xrec + (size_t)(s + j) * kSRec, yv);
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
      const float v0 = yv[0] + __shfl_xor_sync(0xffffffffu, yv[0], 1);
      const float v1 = yv[1] + __shfl_xor_sync(0xffffffffu, yv[1], 1);
      if ((lane & 3) == 0 && seg < kMaxSeg) {
        wpart[(warp * kMaxSeg + seg) * 16 + (lane >> 2)] = v0;
        wpart[(warp * kMaxSeg + seg) * 16 + (lane >> 2) + 8] = v1;
      }
      ++seg;
      ++p;
    }
    // this warp's range is done: pull the next part of its next range into L2
    // while the phase drains and the next one's inputs are handed over
    if (pl.mode != 2) prefetch_phase(ph == 3 ? nl + 1 : nl, (ph + 1) & 3);
    __syncthreads();
    stamp(3);
    // the CTA's partial of every panel it touched: its warps' segments in warp
    // order; slot 2 slab (+ 1 when the panel started in the previous CTA)
    const uint32_t LO = row[0], HI = row[16], pf = row[17], npan = row[33];
    float* dst = pl.part[ph] + (size_t)bs * (2 * pl.ksl[ph]) * pl.pstride[ph] * 2;
    for (uint32_t idx = tid; idx < npan * 16; idx += kSThreads) {
      const uint32_t pp = pf + idx / 16, col = idx % 16;
      const uint32_t ua = max(LO, pp * Sk), ub = min(HI, (pp + 1) * Sk) - 1;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kSWarps; ++w) {
        const uint32_t lw = row[w], hw = row[w + 1];
        if (hw > lw && hw > ua && lw <= ub)
          acc += wpart[((uint32_t)w * kMaxSeg + (pp - row[17 + w])) * 16 + col];
      }
      const uint32_t sl = 2 * row[36] + (pp * Sk < LO ? 1u : 0u);
      st_pair(dst + ((size_t)sl * pl.pstride[ph] + pp * 16 + col) * 2, acc, fl);
    }
    stamp(0);
    ++nph;
  };

  // The cached K / V rows this CTA will read in the attention phase of layer l
  // (written by earlier steps): pulled into L2 while the QKV phase runs.
  auto prefetch_kv = [&](int l) {
    const int cph = pl.cph, ngroups = (int)G / cph;
    const int gi = (int)cta / cph, j = (int)cta % cph;
    const int Lc = (pl.pos + cph - 1) / cph;
    const int p0 = j * Lc, p1 = min(p0 + Lc, pl.pos);  // cached rows of this chunk
    if (gi >= ngroups || p1 <= p0 || tid >= 2) return;
    const char* base = ltab[l * kLtab + 10 + tid];
    for (int hh = gi; hh < pl.H; hh += ngroups) {
      const char* src = base + ((size_t)hh * pl.ctx + p0) * kHD * 2;
      const uint32_t bytes = (uint32_t)(p1 - p0) * kHD * 2;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  };

  // ---- attention of layer l (reads the QKV partials x 1 / rms) --------------------
  // A head's CACHED positions 0 .. pos - 1 are split over its cph CTAs, a CTA's
  // chunk over its warps (position p0 + warp + 16 i); the new token is one more
  // position, taken from shared memory by warp 0 of the last chunk's CTA (which
  // also appends it to the cache).  The first batch of cached K / V rows of each
  // warp (first head of the CTA) and the RoPE factors are loaded into registers
  // before the QKV outputs are awaited.
  constexpr int NB = 8;
  auto attention = [&](int l, uint32_t fl, int bs) {
    float* qs = (float*)xrec;       // rotated q (through f16)
    float* raw = qs + kHD;          // [3][128]: q, k, v of the new token (k, v: as cached)
    float* wsm = raw + 3 * kHD;     // [warp][kAttSm]
    __half* const kc = (__half*)ltab[l * kLtab + 10];
    __half* const vc = (__half*)ltab[l * kLtab + 11];
    const int cph = pl.cph, ngroups = (int)G / cph;
    const int gi = (int)cta / cph, j = (int)cta % cph;
    const int Lc = (pl.pos + cph - 1) / cph;
    const int p0 = j * Lc, p1 = min(p0 + Lc, pl.pos);  // cached rows of this chunk
    const bool mine = j == cph - 1;                    // this CTA takes the new token
    float* const attp = pl.attp + (size_t)bs * pl.H * cph * kAttRow;
    if (gi < ngroups && gi < pl.H) {
      uint2 kr0[NB], vr0[NB];
      float rope_c = 0.f, rope_s = 0.f;
      if (tid < kHD / 2) {
        rope_c = pl.cosv[tid];
        rope_s = pl.sinv[tid];
      }
      {
        const __half* kb = kc + (size_t)gi * pl.ctx * kHD + 4 * lane;
        const __half* vb = vc + (size_t)gi * pl.ctx * kHD + 4 * lane;
#pragma unroll
        for (int u = 0; u < NB; ++u) {
          const int pu = p0 + warp + kSWarps * u;
          if (pu < p1) {
            kr0[u] = __ldcg((const uint2*)(kb + (size_t)pu * kHD));
            vr0[u] = __ldcg((const uint2*)(vb + (size_t)pu * kHD));
          }
        }
      }
      const float rinv = rinv_of(0, fl, bs);
      for (int hh = gi; hh < pl.H; hh += ngroups) {
        if (tid < 3 * kHD && (tid < kHD || mine))
          raw[tid] = slot_sum1(0, (uint32_t)(tid >> 7) * pl.d + (uint32_t)hh * kHD + (tid & 127), fl, bs) * rinv;
        __syncthreads();
        float k0 = 0.f, k1 = 0.f, v0 = 0.f, v1 = 0.f;
        if (tid < kHD / 2) {
          const int i = tid;
          const float c = rope_c, s = rope_s;
          // rotate-half with separately rounded products, q / k rounded through
          // f16 (decode_ops.cu attn_decode_kernel)
          auto rot_lo = [&](float x0, float x1) { return __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s)); };
          auto rot_hi = [&](float x0, float x1) { return __fadd_rn(__fmul_rn(x1, c), __fmul_rn(x0, s)); };
          const float q0 = raw[i], q1 = raw[i + kHD / 2];
          qs[i] = __half2float(__float2half_rn(rot_lo(q0, q1)));
          qs[i + kHD / 2] = __half2float(__float2half_rn(rot_hi(q0, q1)));
          if (mine) {  // append k, v
            const float x0 = raw[kHD + i], x1 = raw[kHD + i + kHD / 2];
            const __half hk0 = __float2half_rn(rot_lo(x0, x1)), hk1 = __float2half_rn(rot_hi(x0, x1));
            const __half hv0 = __float2half_rn(raw[2 * kHD + i]);
            const __half hv1 = __float2half_rn(raw[2 * kHD + i + kHD / 2]);
            const size_t g = ((size_t)hh * pl.ctx + pl.pos) * kHD;
            kc[g + i] = hk0;
            kc[g + i + kHD / 2] = hk1;
            vc[g + i] = hv0;
            vc[g + i + kHD / 2] = hv1;
            k0 = __half2float(hk0); k1 = __half2float(hk1);
            v0 = __half2float(hv0); v1 = __half2float(hv1);
          }
        }
        __syncthreads();  // every thread has read raw: k, v of the new token replace it
        if (mine && tid < kHD / 2) {
          raw[kHD + tid] = k0;
          raw[kHD + tid + kHD / 2] = k1;
          raw[2 * kHD + tid] = v0;
          raw[2 * kHD + tid + kHD / 2] = v1;
        }
        stamp(2);
        const float4 q = *(const float4*)(qs + 4 * lane);
        float m = -INFINITY, ls = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
        const __half* kb = kc + (size_t)hh * pl.ctx * kHD + 4 * lane;
        const __half* vb = vc + (size_t)hh * pl.ctx * kHD + 4 * lane;
        for (int pp = p0 + warp; pp < p1; pp += kSWarps * NB) {
          uint2 kr[NB], vr[NB];
          float sc[NB];
          const bool pre = hh == gi && pp == p0 + warp;  // the preloaded batch
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            if (pre) {
              kr[u] = kr0[u];
              vr[u] = vr0[u];
            } else {
              const int pu = min(pp + kSWarps * u, p1 - 1);
              kr[u] = __ldcg((const uint2*)(kb + (size_t)pu * kHD));
              vr[u] = __ldcg((const uint2*)(vb + (size_t)pu * kHD));
            }
          }
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            const float2 k01 = __half22float2(*(const __half2*)&kr[u].x);
            const float2 k23 = __half22float2(*(const __half2*)&kr[u].y);
            sc[u] = q.x * k01.x + q.y * k01.y + q.z * k23.x + q.w * k23.y;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < NB; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], o);
          float mb = m;
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            sc[u] = pp + kSWarps * u < p1 ? sc[u] * pl.scale : -INFINITY;
            mb = fmaxf(mb, sc[u]);
          }
          const float corr = m == -INFINITY ? 0.f : __expf(m - mb);
          ls *= corr;
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] *= corr;
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            // masked tail: weight 0 (its registers may hold anything)
            const float e = pp + kSWarps * u < p1 ? __expf(sc[u] - mb) : 0.f;
            const float2 v01 = __half22float2(*(const __half2*)&vr[u].x);
            const float2 v23 = __half22float2(*(const __half2*)&vr[u].y);
            ls += e;
            acc[0] = e != 0.f ? fmaf(e, v01.x, acc[0]) : acc[0];
            acc[1] = e != 0.f ? fmaf(e, v01.y, acc[1]) : acc[1];
            acc[2] = e != 0.f ? fmaf(e, v23.x, acc[2]) : acc[2];
            acc[3] = e != 0.f ? fmaf(e, v23.y, acc[3]) : acc[3];
          }
          m = mb;
        }
        stamp(1);
        __syncthreads();  // the new token's k, v are in raw
        if (mine && warp == 0) {  // the new token: one more position
          const float4 kn = *(const float4*)(raw + kHD + 4 * lane);
          const float4 vn = *(const float4*)(raw + 2 * kHD + 4 * lane);
          float sc = q.x * kn.x + q.y * kn.y + q.z * kn.z + q.w * kn.w;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
          sc *= pl.scale;
          const float mb = fmaxf(m, sc);
          const float corr = m == -INFINITY ? 0.f : __expf(m - mb);
          const float e = __expf(sc - mb);
          ls = ls * corr + e;
          acc[0] = fmaf(e, vn.x, acc[0] * corr);
          acc[1] = fmaf(e, vn.y, acc[1] * corr);
          acc[2] = fmaf(e, vn.z, acc[2] * corr);
          acc[3] = fmaf(e, vn.w, acc[3] * corr);
          m = mb;
        }
        stamp(3);
        *(float4*)(wsm + warp * kAttSm + 4 * lane) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        if (lane == 0) {
          wsm[warp * kAttSm + kHD] = m;
          wsm[warp * kAttSm + kHD + 1] = ls;
        }
        __syncthreads();
        if (tid < kHD) {  // combine the warps in warp order
          float M = -INFINITY;
#pragma unroll
          for (int w = 0; w < kSWarps; ++w) M = fmaxf(M, wsm[w * kAttSm + kHD]);
          float o = 0.f, Ls = 0.f;
#pragma unroll
          for (int w = 0; w < kSWarps; ++w) {
            const float mw = wsm[w * kAttSm + kHD];
            const float wt = mw == -INFINITY ? 0.f : __expf(mw - M);
            o = fmaf(wt, wsm[w * kAttSm + tid], o);
            Ls = fmaf(wt, wsm[w * kAttSm + kHD + 1], Ls);
          }
          // partial of (head, chunk) as {value, flag} pairs: acc[128], m, l
          float* dst = attp + ((size_t)hh * cph + j) * kAttRow;
          st_pair(dst + 2 * tid, o, fl);
          if (tid == 0) {
            st_pair(dst + 2 * kHD, M, fl);
            st_pair(dst + 2 * kHD + 2, Ls, fl);
          }
        }
        __syncthreads();
      }
    }
    stamp(0);
    ++nph;
  };

  // ---- the step ------------------------------------------------------------------------
  const int d = pl.d;
  // Residual prologue of an RMSNorm'd GEMV over this CTA's slab of rows (the
  // same slab in phases 0 and 2; the CTA keeps those rows of the residual in
  // shared memory, hp): hp += the partial slots of phase pph (flag pfl, buffer
  // set pbs); hp * nw is digitised; the slab's sum of squares is published as
  // ssq[which] (applied as 1 / rms by the GEMV's consumer).
  struct ResRaw {
    float4 h, w, p;
  };
  auto residual_prologue = [&](int ph, int pph, uint32_t pfl, int pbs, const float* nw, int which,
                               uint32_t fl, int bs) {
    float ss = 0.f;
    const int itb = (int)ctab[ph * kCrow + 34] * 64;
    digitize_rows(
        ph,
        [&](int it) {
          ResRaw r;
          const uint32_t c = min(4u * it, (uint32_t)d - 4u);
          r.h = pph >= 0 ? *(const float4*)(hp + 4 * (it - itb)) : ldcg4(pl.h_in + c);
          r.w = __ldg((const float4*)(nw + c));
          r.p = pph >= 0 ? slot_sum4(pph, c, pfl, pbs) : make_float4(0.f, 0.f, 0.f, 0.f);
          return r;
        },
        [&](int it, const ResRaw& r, float (&v)[4]) {
          float4 a = r.h;
          add4(a, r.p);
          if (4 * it >= d) a = make_float4(0.f, 0.f, 0.f, 0.f);
          *(float4*)(hp + 4 * (it - itb)) = a;
          ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
          v[0] = a.x * r.w.x; v[1] = a.y * r.w.y; v[2] = a.z * r.w.z; v[3] = a.w * r.w.w;
        });
    ss = block_sum(ss);
    if (ctab[ph * kCrow + 37] == 0 && tid == 0)
      st_pair(pl.ssq + (((size_t)bs * 2 + which) * kMaxKsl + ctab[ph * kCrow + 36]) * 2, ss, fl);
  };
  struct AttRaw {
    float4 a[kMaxCph];
    float2 ml[kMaxCph];
  };
  struct GuRaw {
    float4 g, u;
  };
  for (int l = 0; l < pl.L; ++l) {
    const float* const n1 = (const float*)ltab[l * kLtab + 8];
    const float* const n2 = (const float*)ltab[l * kLtab + 9];
    const uint32_t fl = fl0 + (uint32_t)l;  // this layer's flag
    const int bs = l % 3;                   // and buffer set
#pragma unroll 1
    for (int st = 0; st < 4; ++st) {  // one call site of the GEMV loop (code size)
      if (st == 0) {
        // QKV: h (layer input) = h' of the previous layer + its down_proj partials
        residual_prologue(0, l == 0 ? -1 : 3, fl - 1u, (l + 2) % 3, n1, 0, fl, bs);
        prefetch_kv(l);
      } else if (st == 1) {
        // o_proj: combine the attention partials of each head
        const int cph = pl.cph;
        const float* const attp = pl.attp + (size_t)bs * pl.H * cph * kAttRow;
        digitize_rows(
            1,
            [&](int it) {
              AttRaw r;
              const uint32_t c = min(4u * it, (uint32_t)d - 4u);
              const float* src = attp + (size_t)(c / kHD) * cph * kAttRow;
              uint32_t spins = 0;
              unsigned long long t0 = 0;
              for (;;) {
                bool ok = true;
#pragma unroll
                for (int j = 0; j < kMaxCph; ++j) {
                  const int jj = min(j, cph - 1);
                  const float4 x0 = ld_pair2(src + jj * kAttRow + 2 * (c % kHD));
                  const float4 x1 = ld_pair2(src + jj * kAttRow + 2 * (c % kHD) + 4);
                  const float4 z = ld_pair2(src + jj * kAttRow + 2 * kHD);
                  ok = ok && flags_ok(x0, fl) && flags_ok(x1, fl) && flags_ok(z, fl);
                  r.a[j] = make_float4(x0.x, x0.z, x1.x, x1.z);
                  r.ml[j] = make_float2(z.x, z.z);
                }
                if (__all_sync(0xffffffffu, ok)) break;
                if (spin_guard(spins, t0)) break;
              }
              return r;
            },
            [&](int it, const AttRaw& r, float (&v)[4]) {
              float M = -INFINITY;
#pragma unroll
              for (int j = 0; j < kMaxCph; ++j)
                if (j < cph) M = fmaxf(M, r.ml[j].x);
              float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
              float Ls = 0.f;
#pragma unroll
              for (int j = 0; j < kMaxCph; ++j) {
                if (j < cph) {
                  const float wt = r.ml[j].x == -INFINITY ? 0.f : __expf(r.ml[j].x - M);
                  o.x = fmaf(wt, r.a[j].x, o.x); o.y = fmaf(wt, r.a[j].y, o.y);
                  o.z = fmaf(wt, r.a[j].z, o.z); o.w = fmaf(wt, r.a[j].w, o.w);
                  Ls = fmaf(wt, r.ml[j].y, Ls);
                }
              }
              const float il = 4 * it < d ? 1.f / Ls : 0.f;
              v[0] = o.x * il; v[1] = o.y * il; v[2] = o.z * il; v[3] = o.w * il;
            });
        __syncthreads();
      } else if (st == 2) {
        // gate|up: h' = h + o_proj partials
        residual_prologue(2, 1, fl, bs, n2, 1, fl, bs);
      } else {
        // down_proj: SwiGLU of the gate|up partials (x 1 / rms)
        const int ffn = pl.ffn;
        const float rinv2 = rinv_of(1, fl, bs);
        digitize_rows(
            3,
            [&](int it) {
              GuRaw r;
              const uint32_t c = min(4u * it, (uint32_t)ffn - 4u);
              r.g = slot_sum4(2, c, fl, bs);
              r.u = slot_sum4(2, (uint32_t)ffn + c, fl, bs);
              return r;
            },
            [&](int it, const GuRaw& r, float (&v)[4]) {
              if (4 * it < ffn) {
                const float gg[4] = {r.g.x * rinv2, r.g.y * rinv2, r.g.z * rinv2, r.g.w * rinv2};
                const float uu[4] = {r.u.x * rinv2, r.u.y * rinv2, r.u.z * rinv2, r.u.w * rinv2};
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = __fdividef(gg[i], 1.f + __expf(-gg[i])) * uu[i];
              } else {
                v[0] = v[1] = v[2] = v[3] = 0.f;
              }
            });
        __syncthreads();
      }
      stamp(2);
      gemv_phase(st, fl, bs, l);
      if (st == 0) attention(l, fl, bs);
    }
    // Skew bound for the three buffer sets: this CTA enters layer l + 1 (whose
    // writes reuse the buffers of layer l - 2, last read early in layer l - 1)
    // only after every CTA has finished layer l - 1.  Normally long satisfied.
    if (tid == 0) {
      asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(pl.bar) : "memory");
      if (l >= 1) {
        const unsigned int target = (unsigned int)l * G;
        uint32_t spins = 0;
        unsigned long long t0 = 0;
        for (;;) {
          unsigned int v;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pl.bar) : "memory");
          if (v >= target) break;
          if (spin_guard(spins, t0)) break;
        }
      }
    }
  }
  // the step's output: the residual + the last layer's down_proj partials (each
  // CTA its share of its slab's rows)
  {
    const uint32_t itb = ctab[34] * 64, nit = min((ctab[34] + ctab[35]) * 64, (uint32_t)d / 4);
    const uint32_t own0 = itb + ctab[37] * pl.own_q[0];
    const uint32_t own1 = min(own0 + pl.own_q[0], nit);
    const uint32_t fl = fl0 + (uint32_t)pl.L - 1u;
    for (uint32_t it0 = own0 + warp * 32; it0 < own1; it0 += kSThreads) {  // whole warps poll
      const uint32_t it = min(it0 + lane, nit - 1);
      float4 a = *(const float4*)(hp + 4 * (it - itb));
      add4(a, slot_sum4(3, 4 * it, fl, (pl.L - 1) % 3));
      if (it0 + lane < own1) *(float4*)(pl.h_out + 4 * it) = a;
    }
  }
  // the last CTA to leave re-arms the counters and advances the launch epoch
  __syncthreads();
  if (tid == 0) {
    if (atomicAdd(pl.bar + 2, 1u) == G - 1) {
      pl.bar[0] = 0u;
      pl.bar[2] = 0u;
      pl.bar[3] = pl.bar[3] + 1u;
      __threadfence();
    }
  }
}

}  // namespace
}  // namespace qigen

using namespace qigen;

struct qigen_decode_stack {
  SPlan plan{};
  void* blob = nullptr;   // layer table | partial buffers | residuals | barrier words
  size_t smem = 0;
  int bits = 0, gps = 0;
};

// tuning aids (per calling thread): supersteps per weight stage (1 or 2), ring
// depth cap
static thread_local int g_stack_sss = 2;
static thread_local int g_stack_depth = 8;
static thread_local int g_stack_mode = 0;
static thread_local int g_stack_cph = kMaxCph;  // cap on the position chunks (CTAs) per head
// MB of L2 prefetch per phase hand-off ((MB + 1) << 8 in qigen_debug_stack_mode).  Off:
// measured slower at every size (7B layer 36.4 us -> 37.6 / 38.8 / 39.6 us at 8 / 16 / 40 MB):
// the extra traffic delays the latency-critical flagged loads of the hand-off.
static thread_local int g_stack_pf = 0;
extern "C" int qigen_debug_stack_mode(int mode) {
  g_stack_mode = mode & 3;
  g_stack_cph = (mode >> 2) & 7 ? std::min(kMaxCph, (mode >> 2) & 7) : kMaxCph;
  if (mode >> 8) g_stack_pf = (mode >> 8) - 1;
  return QIGEN_OK;
}
static thread_local int g_stack_ksl = 2424;  // K slabs wanted for qkv, o, gate|up, down (digits)
extern "C" int qigen_debug_stack_tuning(int sss, int depth, int ksl) {
  g_stack_sss = sss == 1 ? 1 : 2;
  g_stack_depth = depth < 2 ? 2 : depth;
  g_stack_ksl = ksl < 1111 ? 1111 : ksl;
  return QIGEN_OK;
}

template <int B, int G>
static int stack_launch(const qigen_decode_stack* s, const SPlan& pl, cudaStream_t st) {
  static OncePerDevice once;
  const int rc = once.run([]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(decode_stack_kernel<B, G>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    return QIGEN_OK;
  });
  if (rc) return rc;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeCooperative;
  at.val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.G, 1, 1);
  cfg.blockDim = dim3(kSThreads, 1, 1);
  cfg.dynamicSmemBytes = s->smem;
  cfg.stream = st;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, decode_stack_kernel<B, G>, pl));
  return QIGEN_OK;
}

extern "C" int qigen_decode_stack_create(const qigen_stack_desc* desc,
                                         const qigen_stack_layer* layers,
                                         qigen_decode_stack** out) {
  QIGEN_CHECK_ARG(desc && layers && out, QIGEN_ERR_ARG, "null pointer");
  const qigen_stack_desc& e = *desc;
  QIGEN_CHECK_ARG(e.bits == 2 || e.bits == 3 || e.bits == 4, QIGEN_ERR_CONFIG,
                  "bits must be one of (2, 3, 4), got %d", e.bits);
  QIGEN_CHECK_ARG(e.group_size == 32 || e.group_size == 64 || e.group_size == 128,
                  QIGEN_ERR_UNSUPPORTED, "decode stack: group size must be 32, 64 or 128");
  QIGEN_CHECK_ARG(e.layers > 0 && e.d_model > 0 && e.heads > 0 && e.ffn > 0 && e.ctx > 0,
                  QIGEN_ERR_ARG, "decode stack: empty model");
  QIGEN_CHECK_ARG(e.head_dim == kHD && (int64_t)e.heads * kHD == e.d_model, QIGEN_ERR_UNSUPPORTED,
                  "decode stack: head_dim must be 128 and heads * 128 == d_model");
  QIGEN_CHECK_ARG(e.d_model % 16 == 0 && e.ffn % 16 == 0 && e.d_model % e.group_size == 0 &&
                      e.ffn % e.group_size == 0,
                  QIGEN_ERR_UNSUPPORTED, "decode stack: d_model / ffn alignment");
  for (int l = 0; l < e.layers; ++l)
    for (int ph = 0; ph < 4; ++ph)
      QIGEN_CHECK_ARG(layers[l].qw[ph] && layers[l].qsz[ph] && layers[l].norm1 &&
                          layers[l].norm2 && layers[l].k_cache && layers[l].v_cache,
                      QIGEN_ERR_ARG, "decode stack: layer %d has a null pointer", l);
  int dev = 0, sms = 0;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t Kd[4] = {e.d_model, e.d_model, e.d_model, e.ffn};
  const int64_t Nd[4] = {3 * (int64_t)e.d_model, e.d_model, 2 * (int64_t)e.ffn, e.d_model};
  SPlan pl{};
  for (int ph = 0; ph < 4; ++ph) {
    pl.P[ph] = (uint32_t)panels(Nd[ph]);
    pl.S[ph] = (uint32_t)supersteps(Kd[ph]);
    pl.pstride[ph] = pl.P[ph] * 16;
  }
  // CTAs: at most the panels of the narrowest phase divided by its slab count,
  // so that within a slab group a panel spans at most two CTAs (two slots per
  // slab).  K slabs per phase: g_stack_ksl digits (qkv, o, gate|up, down), each
  // reduced to a divisor of the grid that leaves every slab a superstep.
  int G = sms;
  for (int ph = 0; ph < 4; ++ph) G = (int)std::min<uint32_t>((uint32_t)G, pl.P[ph]);
  G = std::max(1, G);
  pl.L = e.layers;
  pl.d = e.d_model;
  pl.H = e.heads;
  pl.ffn = e.ffn;
  pl.ctx = (int)e.ctx;
  pl.G = G;
  pl.eps = e.eps;
  pl.cph = std::max(1, std::min(g_stack_cph, G / e.heads));
  // per-CTA unit ranges and the two-CTA panel bits of the static partition
  std::vector<uint32_t> ctab((size_t)G * kCtab, 0u), two;
  uint32_t skmax = 0;
  bool fits = true;
  const int want[4] = {g_stack_ksl / 1000 % 10, g_stack_ksl / 100 % 10, g_stack_ksl / 10 % 10,
                       g_stack_ksl % 10};
  for (int ph = 0; ph < 4; ++ph) {
    pl.ksl[ph] = 1;
    for (int k : {4, 2})
      if (k <= want[ph] && G % k == 0 && pl.S[ph] >= (uint32_t)k && pl.P[ph] >= (uint32_t)(G / k)) {
        pl.ksl[ph] = k;
        break;
      }
  }
  // QKV and gate|up read the same residual rows: one slab split for both (the
  // CTA keeps its slab of the residual in shared memory)
  pl.ksl[0] = pl.ksl[2] = std::min(pl.ksl[0], pl.ksl[2]);
  for (int ph = 0; ph < 4; ++ph) {
    const uint32_t P = pl.P[ph], S = pl.S[ph];
    const int ksl = pl.ksl[ph];
    const int GJ = G / ksl;
    const uint32_t GWJ = (uint32_t)GJ * kSWarps;  // warps per slab group
    pl.own_q[ph] = (uint32_t)(((S + ksl - 1) / ksl * 64 + GJ - 1) / GJ);
    pl.two_off[ph] = (uint32_t)two.size();
    pl.two_wp[ph] = (P + 31) / 32;
    two.resize(two.size() + (size_t)ksl * pl.two_wp[ph], 0u);
    for (int k = 0; k < ksl; ++k) {
      const uint32_t s0 = (uint32_t)((uint64_t)k * S / ksl), s1 = (uint32_t)((uint64_t)(k + 1) * S / ksl);
      const uint32_t Sk = s1 - s0, T = P * Sk;
      skmax = std::max(skmax, Sk);
      if ((uint64_t)(T + 1) * GWJ >= (1ull << 32)) fits = false;
      for (uint32_t p = 0; fits && p < P; ++p) {
        const uint32_t c0 = warp_of(p * Sk, T, GWJ) / kSWarps;
        const uint32_t c1 = warp_of(p * Sk + Sk - 1, T, GWJ) / kSWarps;
        if (c1 - c0 + 1 > kMaxSlot) fits = false;
        if (c1 != c0) two[pl.two_off[ph] + (size_t)k * pl.two_wp[ph] + p / 32] |= 1u << (p % 32);
      }
      for (int j = 0; fits && j < GJ; ++j) {
        uint32_t* row = &ctab[(size_t)(k * GJ + j) * kCtab + ph * kCrow];
        for (int w = 0; w <= kSWarps; ++w) row[w] = lo_of((uint32_t)j * kSWarps + w, T, GWJ);
        for (int w = 0; w < kSWarps; ++w) {
          row[17 + w] = row[w] / Sk;
          // panel segments of warp w
          if (row[w + 1] > row[w] && (row[w + 1] - 1) / Sk - row[17 + w] + 1 > (uint32_t)kMaxSeg)
            fits = false;
        }
        row[33] = row[16] > row[0] ? (row[16] - 1) / Sk - row[17] + 1 : 0u;
        row[34] = s0;
        row[35] = Sk;
        row[36] = (uint32_t)k;
        row[37] = (uint32_t)j;
      }
    }
  }
  QIGEN_CHECK_ARG(fits, QIGEN_ERR_UNSUPPORTED,
                  "decode stack: shape outside the static partition's limits");
  pl.two_words = (uint32_t)two.size();
  // optional L2 prefetch behind the ring's lookahead, issued by a warp when it
  // finishes a phase (tuning aid, off by default: see g_stack_pf)
  for (int ph = 0; ph < 4; ++ph) {
    const double unit_bytes = e.bits * 512 + (256 / e.group_size) * 128;
    const double cap = (double)g_stack_pf * 1e6 / ((double)G * kSWarps * unit_bytes);
    pl.pf_units[ph] = (uint32_t)(cap + 0.5);
  }
  // shared memory: records | rings | warp partials | red | barriers | tables
  const size_t xrec = std::max<size_t>((size_t)skmax * kSRec, kAttScratch);
  const size_t xrec_al = (xrec + 127) / 128 * 128;
  const int gps = (int)(256 / e.group_size);
  int sss = g_stack_sss, depth = 0;
  size_t slot = 0;
  const size_t hp_bytes = (size_t)((pl.S[0] + pl.ksl[0] - 1) / pl.ksl[0]) * kSuper * 4;
  pl.hp_bytes = (uint32_t)hp_bytes;
  const size_t fixed = xrec_al + kSWarps * kMaxSeg * 16 * 4 + 32 * 4 +
                       (size_t)e.layers * kLtab * sizeof(void*) + kCtab * 4 +
                       ((two.size() + 3) & ~(size_t)3) * 4 + hp_bytes;
  const size_t budget = 227 * 1024;
  for (; sss >= 1; --sss) {  // 2-superstep stages unless only 1-superstep ones fit
    slot = (size_t)sss * (e.bits * 512 + gps * 128);
    for (int dd = std::min(g_stack_depth, 16); dd >= 2; --dd)
      if (fixed + (size_t)kSWarps * dd * (slot + 8) <= budget) {
        depth = dd;
        break;
      }
    if (depth >= 2) break;
  }
  QIGEN_CHECK_ARG(depth >= 2, QIGEN_ERR_UNSUPPORTED, "decode stack: shared memory does not fit");
  pl.depth = depth;
  pl.sss = sss;
  pl.slot_bytes = (uint32_t)slot;
  pl.xrec_bytes = (uint32_t)xrec_al;
  // device blob
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_lay = take((size_t)e.layers * sizeof(SLayer));
  size_t o_part[4];
  for (int ph = 0; ph < 4; ++ph)
    o_part[ph] = take((size_t)3 * 2 * pl.ksl[ph] * pl.pstride[ph] * 2 * 4);
  const size_t o_att = take((size_t)3 * e.heads * pl.cph * kAttRow * 4);
  const size_t o_bar = take(256), o_ssq = take((size_t)3 * 2 * kMaxKsl * 2 * 4);
  const size_t o_ctab = take(ctab.size() * 4), o_two = take(two.size() * 4);
  std::vector<SLayer> tab(e.layers);
  for (int l = 0; l < e.layers; ++l) {
    for (int ph = 0; ph < 4; ++ph) {
      tab[l].qw[ph] = (const char*)layers[l].qw[ph];
      tab[l].qsz[ph] = (const char*)layers[l].qsz[ph];
    }
    tab[l].n1 = layers[l].norm1;
    tab[l].n2 = layers[l].norm2;
    tab[l].kc = (__half*)layers[l].k_cache;
    tab[l].vc = (__half*)layers[l].v_cache;
  }
  auto* s = new qigen_decode_stack();
  cudaError_t ce = cudaMalloc(&s->blob, off);
  char* b = (char*)s->blob;
  if (ce == cudaSuccess) ce = cudaMemset(b, 0, off);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(b + o_lay, tab.data(), tab.size() * sizeof(SLayer), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(b + o_ctab, ctab.data(), ctab.size() * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(b + o_two, two.data(), two.size() * 4, cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) {
    if (s->blob) cudaFree(s->blob);
    delete s;
    QIGEN_CUDA_RET(ce);
  }
  pl.layers = (const SLayer*)(b + o_lay);
  for (int ph = 0; ph < 4; ++ph) pl.part[ph] = (float*)(b + o_part[ph]);
  pl.attp = (float*)(b + o_att);
  pl.bar = (unsigned int*)(b + o_bar);
  pl.ssq = (float*)(b + o_ssq);
  pl.ctab = (const uint32_t*)(b + o_ctab);
  pl.two = (const uint32_t*)(b + o_two);
  s->plan = pl;
  s->bits = e.bits;
  s->gps = gps;
  s->smem = fixed + (size_t)kSWarps * depth * (slot + 8);
  *out = s;
  return QIGEN_OK;
}

extern "C" int qigen_decode_stack_run(const qigen_decode_stack* s, const float* h_in, float* h_out,
                                      const float* cosv, const float* sinv, int64_t pos,
                                      float scale, void* stream) {
  QIGEN_CHECK_ARG(s && h_in && h_out && cosv && sinv, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(pos >= 0 && pos < s->plan.ctx, QIGEN_ERR_ARG, "position outside the KV cache");
  SPlan pl = s->plan;
  pl.h_in = h_in;
  pl.h_out = h_out;
  pl.cosv = cosv;
  pl.sinv = sinv;
  pl.pos = (int)pos;
  pl.scale = scale;
  pl.trace = g_trace;
  pl.mode = g_stack_mode;
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->bits * 16 + s->gps) {
#define QS_CASE(B, G) \
  case B * 16 + G: return stack_launch<B, G>(s, pl, st);
    QS_CASE(2, 2) QS_CASE(2, 4) QS_CASE(2, 8)
    QS_CASE(3, 2) QS_CASE(3, 4) QS_CASE(3, 8)
    QS_CASE(4, 2) QS_CASE(4, 4) QS_CASE(4, 8)
#undef QS_CASE
    default: break;
  }
  set_error("decode stack: unsupported configuration");
  return QIGEN_ERR_UNSUPPORTED;
}

extern "C" int qigen_decode_stack_error(const qigen_decode_stack* s, int* out) {
  QIGEN_CHECK_ARG(s && out, QIGEN_ERR_ARG, "null pointer");
  unsigned int w[4] = {};
  QIGEN_CUDA_RET(cudaMemcpy(w, s->plan.bar, sizeof(w), cudaMemcpyDeviceToHost));
  *out = (int)w[1];
  if (w[1]) {  // a wait timed out: re-arm the counters
    QIGEN_CUDA_RET(cudaMemset(s->plan.bar, 0, 16));
  }
  return QIGEN_OK;
}

extern "C" int qigen_decode_stack_info(const qigen_decode_stack* s, int* grid, int* depth,
                                       int* smem_bytes) {
  QIGEN_CHECK_ARG(s, QIGEN_ERR_ARG, "null pointer");
  if (grid) *grid = s->plan.G;
  if (depth)
    *depth = s->plan.depth * 100000 + s->plan.sss * 10000 + s->plan.ksl[0] * 1000 +
             s->plan.ksl[1] * 100 + s->plan.ksl[2] * 10 + s->plan.ksl[3];
  if (smem_bytes) *smem_bytes = (int)s->smem;
  return QIGEN_OK;
}

extern "C" int qigen_decode_stack_destroy(qigen_decode_stack* s) {
  if (!s) return QIGEN_OK;
  if (s->blob) cudaFree(s->blob);
  delete s;
  return QIGEN_OK;
}
