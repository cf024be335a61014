// Grouped batch-1 GEMV: many INDEPENDENT quantized GEMVs (mixed bits / group
// sizes / shapes) in one persistent launch.
//
// Same arithmetic as the split-K GEMV (gemv.cu; the reference factorisation
// kernelgen.py:227-240 with exact IMMA partials), different schedule.  A chain
// of single GEMVs pays, per launch, the programmatic-launch release, the
// activation prologue and the split-K reduction on the critical path (DESIGN.md
// §4).  When the GEMVs are independent (the reference runtime's per-matrix
// qgemv calls of a sweep; the BASELINE configs[1] workload) a
// persistent schedule hides all of it:
//   * one CTA per SM: 16 consumer warps + 1 activation-record producer warp;
//   * a work item is one GEMV x 16 panels (256 output columns) x its K range
//     (the full K by default), so every output column is reduced by one warp
//     in a fixed order: deterministic, no atomics, no cross-CTA traffic;
//   * group_prep_kernel digitises the activations of all GEMVs into
//     per-superstep records (digits + unit flush factors); the grouped kernel
//     streams its first weight stages meanwhile and waits for it (PDL) before
//     reading records or claiming items;
//   * items are ordered by a cost model (bytes vs issue time) and scheduled
//     greedily: CTA c starts with item c, then claims the next unclaimed item
//     from a global counter - list scheduling in decreasing-cost order, robust
//     to the model's errors; the claimer stages the item's geometry in shared
//     memory, normally a few stages before it is needed;
//   * each consumer warp streams its panel of every item through its own ring
//     of TMA bulk-copy stages (2 supersteps of weights + their (s, z); 4 for
//     2-bit weights, whose per-stage issue cost would otherwise dominate), refilled
//     by its lane 0 ahead ACROSS item boundaries, so the weight stream never
//     drains between GEMVs and a slow copy stalls only its own panel;
//   * the producer warp streams the activation records through a CTA-shared
//     ring.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <queue>
#include <utility>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "gemv_common.cuh"

namespace qigen {

extern thread_local unsigned long long* g_trace;  // gemv.cu (qigen_debug_trace)

constexpr int kGWarps = 16;            // consumer warps per CTA (panels per item)
constexpr int kGTP = 2;                // tokens in the fragment layout (M <= 2)
constexpr int kRecDig = 8 * kGTP * 128;  // digit bytes per superstep record
// + per unit and token {2^(E-30) * 2^16, X * 2^(E-30), 2^(E-30), 0}: the flush
// factors of the even (digits d0 d1) and odd (d2 d3) lanes, one LDS.64 each
constexpr int kRecBytes = kRecDig + 8 * kGTP * 16;
constexpr int kGSS = 2;                // supersteps per activation-record stage
constexpr int kGSlot = kGSS * (4 * 512 + 8 * 128);  // largest weight stage (4-bit, g = 32)
// Supersteps per WEIGHT stage: 4 where they fit a slot (2-bit weights with at
// most 4 groups per superstep), else kGSS.  Each stage costs the issuing lane
// a fixed overhead while its warp waits, so small-bit stages are made longer.
__host__ __device__ constexpr int wss_for(int bits, int gps) {
  return bits == 2 && gps <= 4 ? 2 * kGSS : kGSS;
}
constexpr int kGDepth = 2;             // weight stages per consumer warp
constexpr int kRecSlot = kGSS * kRecBytes;
constexpr int kGRecDepth = 4;          // activation-record stages in the CTA ring
constexpr int kMaxSeq = 2048;          // items one CTA may claim (dynamic schedule)
constexpr double kSplitPct = 20.0;     // K-split GEMVs with items below this % of the largest

struct GDesc {
  const uint4* qw;
  const float2* qsz;
  const void* x;
  float* y;
  int64_t ldx, ldy, n, m;
  int KS, P, Gp, g, bits, gps, M, x_dtype;
  int split;     // 1: K is split in two items whose partials are atomically added to
                 // a zeroed y (two addends: commutative, so still deterministic)
  int64_t rec0;  // index of this GEMV's first superstep record in the workspace
};
struct GItem {
  int d, p0, k0, k1;  // GEMV, first panel, superstep range
};
struct GPlan {
  const GDesc* desc;
  const GItem* items;
  const int* cta_start;  // [grid + 1] (static schedule)
  unsigned char* rec;    // activation records
  int* counter;          // dynamic schedule: next unclaimed item (re-armed in phase 1)
  int nitems, first_dyn, dynamic;
  int64_t total_items;   // activation items (4 rows) of all GEMVs
  int count;
  int mode;              // tuning: &15 == 1 stream only (no compute); &32 early trigger
  int64_t ydelta;        // bytes added to every y pointer (run_rebased: a fresh output block)
  unsigned long long* trace;  // optional per-CTA %globaltimer (entry, exit)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Four consecutive activations of token tk (zero beyond n / for padding tokens).
__device__ __forceinline__ void gload4(const GDesc& d, int tk, int64_t k, float (&v)[4]) {
  const int64_t o = tk * d.ldx + k;
  if (d.x_dtype == QIGEN_F32 && k + 3 < d.n && ((uintptr_t)((const float*)d.x + o) & 15) == 0) {
    const float4 f = __ldg((const float4*)((const float*)d.x + o));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float f = 0.f;
    if (k + i < d.n) {
      if (d.x_dtype == QIGEN_F32) f = __ldg((const float*)d.x + o + i);
      else if (d.x_dtype == QIGEN_F16) f = __half2float(((const __half*)d.x)[o + i]);
      else f = __bfloat162float(((const __nv_bfloat16*)d.x)[o + i]);
    }
    v[i] = f;
  }
}

template <int IPU>
__device__ __forceinline__ void group_prep_item(const GPlan& pl, const GDesc& d, int it) {
  const int lane = threadIdx.x & 31;
  const uint32_t umask = IPU == 32 ? 0xffffffffu : ((1u << IPU) - 1u) << (lane & ~(IPU - 1));
  const bool live = it < d.KS * 64;
  const int st = it >> 3, sub = it & 7;
  const int sup = st >> 3, sl = st & 7;
  unsigned char* rec = pl.rec + (size_t)(d.rec0 + (live ? sup : 0)) * kRecBytes;
#pragma unroll
  for (int tk = 0; tk < kGTP; ++tk) {
    if (tk >= d.M) {  // padding token (CTA-uniform): zero digits and flush factors
      if (live) {
        store_digits((uint32_t*)rec, sl, tk, kGTP, sub, Digits{{0u, 0u, 0u, 0u}, 0.f, 0.f});
        if ((it % IPU) == 0)
          ((float4*)(rec + kRecDig))[((it % 64) / IPU) * kGTP + tk] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (live) gload4(d, tk, (int64_t)32 * st + 16 * (sub >> 2) + 4 * (sub & 3), v);
    const Digits dg = digitize<IPU>(v, umask);
    if (live) {
      store_digits((uint32_t*)rec, sl, tk, kGTP, sub, dg);
      if ((it % IPU) == 0) {
        const int uj = (it % 64) / IPU;
        // dg.scale is a power of two: both products are exact
        ((float4*)(rec + kRecDig))[uj * kGTP + tk] =
            make_float4(dg.scale * 65536.f, dg.xsum * dg.scale, dg.scale, 0.f);
      }
    }
  }
}

// Exponent units of 256 rows (group sizes >= 256 and full-column: ONE flush per
// superstep in the consumer): 64 items = two warps agree on the exponent and
// add their sums through shared memory.  Called by whole 256-thread blocks.
__device__ __forceinline__ void group_prep_item64(const GPlan& pl, const GDesc& d, int it) {
  __shared__ uint32_t s_max[8];
  __shared__ int s_lo[8], s_hi[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool live = it < d.KS * 64;
  const int st = it >> 3, sub = it & 7;
  const int sup = st >> 3, sl = st & 7;
  unsigned char* rec = pl.rec + (size_t)(d.rec0 + (live ? sup : 0)) * kRecBytes;
#pragma unroll
  for (int tk = 0; tk < kGTP; ++tk) {
    if (tk >= d.M) {  // padding token (CTA-uniform): zero digits and flush factors
      if (live) {
        store_digits((uint32_t*)rec, sl, tk, kGTP, sub, Digits{{0u, 0u, 0u, 0u}, 0.f, 0.f});
        if ((it % 64) == 0) ((float4*)(rec + kRecDig))[tk] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (live) gload4(d, tk, (int64_t)32 * st + 16 * (sub >> 2) + 4 * (sub & 3), v);
    const float m4 = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
    const uint32_t wmx = __reduce_max_sync(0xffffffffu, __float_as_uint(m4));
    __syncthreads();  // (the previous token's exchange is over)
    if (lane == 0) s_max[warp] = wmx;
    __syncthreads();
    const uint32_t umx = max(s_max[warp & ~1], s_max[warp | 1]);
    // as digitize<> (gemv_common.cuh) from here on, with the unit = this warp pair
    const int e = umx ? (int)((umx >> 23) & 0xFF) - 126 : 0;
    const int k = 30 - e, k1 = k >> 1, k2 = k - k1;
    const float f1 = __int_as_float((127 + k1) << 23), f2 = __int_as_float((127 + k2) << 23);
    int mv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) mv[i] = __float2int_rn(__fmul_rn(__fmul_rn(v[i], f1), f2));
    uint32_t tt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) tt[i] = (uint32_t)(mv[i] + 0x808080);
    const uint32_t lo01 = __byte_perm(tt[0], tt[1], 0x5140), lo23 = __byte_perm(tt[2], tt[3], 0x5140);
    const uint32_t hi01 = __byte_perm(tt[0], tt[1], 0x7362), hi23 = __byte_perm(tt[2], tt[3], 0x7362);
    Digits dg;
    dg.dw[3] = __byte_perm(lo01, lo23, 0x5410) ^ 0x80808080u;
    dg.dw[2] = __byte_perm(lo01, lo23, 0x7632) ^ 0x80808080u;
    dg.dw[1] = __byte_perm(hi01, hi23, 0x5410) ^ 0x80808080u;
    dg.dw[0] = __byte_perm(hi01, hi23, 0x7632);
    int slo = 0, shi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      slo += mv[i] & 0xFFFF;
      shi += mv[i] >> 16;
    }
    slo = __reduce_add_sync(0xffffffffu, slo);
    shi = __reduce_add_sync(0xffffffffu, shi);
    if (lane == 0) {
      s_lo[warp] = slo;
      s_hi[warp] = shi;
    }
    __syncthreads();
    slo = s_lo[warp & ~1] + s_lo[warp | 1];
    shi = s_hi[warp & ~1] + s_hi[warp | 1];
    dg.xsum = fmaf((float)shi, 65536.f, (float)slo);
    dg.scale = umx ? __int_as_float((127 + e - 30) << 23) : 0.f;
    if (umx && e - 30 < -126) dg.scale = scalbnf(1.f, e - 30);
    if (live) {
      store_digits((uint32_t*)rec, sl, tk, kGTP, sub, dg);
      if ((it % 64) == 0)
        ((float4*)(rec + kRecDig))[tk] =
            make_float4(dg.scale * 65536.f, dg.xsum * dg.scale, dg.scale, 0.f);
    }
  }
}

// Activation records of every GEMV of the group; grid (ceil(max KS*64/256),
// count), launched just before the grouped kernel (which prefetches weights
// meanwhile and waits for it before reading records or claiming items).
__global__ void __launch_bounds__(256) group_prep_kernel(const GPlan pl) {
  // mode & 32: trigger the grouped launch before waiting, so its CTAs take SMs
  // (and start their weight prefetch) as the previous launch's CTAs leave
  if (pl.mode & 32) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  // the previous grouped launch has completed: re-arm the dynamic schedule
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && pl.dynamic)
    *pl.counter = pl.first_dyn;
  const GDesc& d = pl.desc[blockIdx.y];
  if (d.split)  // the two K halves add into a zeroed y
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < (int64_t)d.M * d.m; i += gridDim.x * 256)
      ((float*)((char*)d.y + pl.ydelta))[(i / d.m) * d.ldy + i % d.m] = 0.f;
  if ((int)blockIdx.x * 256 >= d.KS * 64) return;
  const int it = blockIdx.x * 256 + threadIdx.x;
  // exponent unit (rows): the group, 256 for groups of >= 256 rows / full column
  if (d.g == 32) group_prep_item<8>(pl, d, it);
  else if (d.g == 64) group_prep_item<16>(pl, d, it);
  else if (d.g == 128) group_prep_item<32>(pl, d, it);
  else group_prep_item64(pl, d, it);
}

// IMMA with a zero accumulator input (first step of a chain in a unit).
__device__ __forceinline__ void imma0(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y), "r"(0));
}

// Accumulate one 256-row superstep of one panel: 8 IMMA steps + unit flushes.
// w: the lane's weight words; szs: (s, z) of the groups of this superstep;
// rec: the activation record of this superstep.  Flush of unit u, row r:
//   y_r += s_r * (A q_r - z_r B),  q_r the exact digit-pair partial,
//   (A, B) = (2^(E-30) 2^16, X 2^(E-30)) on even lanes, (2^(E-30), 0) on odd.
template <int BITS, int GPS>
__device__ __forceinline__ void group_superstep(const uint4 (&w)[BITS], const float2* szs,
                                                const unsigned char* rec, float (&yv)[2]) {
  // exponent units per superstep: the groups, one for groups of >= 256 rows / full
  // column (the digit-pair partial c * 256 + c' of 256 rows still fits an int32:
  // |c| <= 256 * 240 * 128, see the flush)
  constexpr int UPS = GPS >= 2 ? GPS : 1;
  constexpr int SPU = 8 / UPS;
  const int lane = threadIdx.x & 31, gq = lane >> 2, t = lane & 3;
  const uint2* bs = (const uint2*)rec + (gq >> 2) * 16 + (gq & 3) * 4 + t;
  const float2* ab = (const float2*)(rec + kRecDig) + (t >> 1) * 2 + (t & 1);
  int acc[2][4];
#pragma unroll
  for (int sl = 0; sl < 8; ++sl) {
    uint32_t af[4];
    extract<BITS>(w, sl, af);
    // a chain starts from zero at its first step in the unit (no reset moves)
    if (sl % SPU < 2) imma0(acc[sl & 1], af, bs[sl * kGTP * 16]);
    else imma(acc[sl & 1], af, bs[sl * kGTP * 16]);
    if ((sl + 1) % SPU == 0) {
      const int uj = (sl + 1) / SPU - 1;
      const int gi = GPS >= UPS ? uj : 0;
      const float2 sz0 = szs[gi * 16 + gq], sz1 = szs[gi * 16 + gq + 8];
      const float2 f = ab[uj * kGTP * 2];
      constexpr int sh = BITS == 2 ? 4 : 0;  // 2-bit odd steps carry an extra x16
      int c0, c1, c2, c3;
      if (SPU == 1) {  // one step per unit: only its chain holds data
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

__device__ __forceinline__ int gcombo(const GDesc& d) { return (d.bits - 2) * 5 + d.gps; }

// Everything a warp needs about one item, staged in shared memory by the
// thread that claims the item (so no warp stalls on global loads at an item
// boundary).  Ring of kInfo entries indexed by sequence position.
struct GInfo {
  const char* w;            // weights of the item's first panel
  const char* z;            // (s, z) of the item's first panel
  float* y;
  const unsigned char* rec; // the GEMV's first activation record
  int64_t wstride, zstride, ldy;
  int p0, k0, k1, P, gps, g, wb, M, m, split, combo;
};
constexpr int kInfo = 8;

__device__ __forceinline__ void fill_info(GInfo* inf, const GPlan& pl, int id) {
  const GItem itm = pl.items[id];
  const GDesc& d = pl.desc[itm.d];
  const int wb = d.bits * 512;
  inf->wstride = (int64_t)d.KS * wb;
  inf->zstride = (int64_t)d.Gp * 16 * 8;
  inf->w = (const char*)d.qw + itm.p0 * inf->wstride;
  inf->z = (const char*)d.qsz + itm.p0 * inf->zstride;
  inf->y = d.y;
  inf->rec = pl.rec + (size_t)d.rec0 * kRecBytes;
  inf->ldy = d.ldy;
  inf->p0 = itm.p0;
  inf->k0 = itm.k0;
  inf->k1 = itm.k1;
  inf->P = d.P;
  inf->gps = d.gps;
  inf->g = d.g;
  inf->wb = wb;
  inf->M = d.M;
  inf->m = (int)d.m;
  inf->split = d.split;
  inf->combo = gcombo(d);
}

// Item k of this CTA's sequence (-1: done); info[k % kInfo] is valid after it
// returns >= 0.  Static schedule: the host's LPT list.  Dynamic schedule: item
// 0 is the CTA's static first item (so its weights stream before the PDL
// wait); later items are claimed from a global counter in decreasing-cost
// order by whichever thread of the CTA needs them first (normally the record
// producer, a few stages ahead), which also stages their info.
__device__ __forceinline__ int seq_get(volatile int* seq, GInfo* info, int k, const GPlan& pl) {
  if (k >= kMaxSeq) return -1;  // (host guarantees the sequence fits)
  int v = seq[k];
  if (v == -2 && atomicCAS((int*)&seq[k], -2, -3) == -2) {
    if (!pl.dynamic) {
      const int i = pl.cta_start[blockIdx.x] + k;
      v = i < pl.cta_start[blockIdx.x + 1] ? i : -1;
    } else {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // counter re-armed by the prep kernel
      const int c = atomicAdd(pl.counter, 1);
      v = c < pl.nitems ? c : -1;
    }
    if (v >= 0) fill_info(&info[k % kInfo], pl, v);
    __threadfence_block();
    seq[k] = v;
    return v;
  }
  while ((v = seq[k]) < -1) {
  }
  __threadfence_block();
  return v;
}

__global__ void __launch_bounds__((kGWarps + 1) * 32, 1) gemv_group_kernel(const GPlan pl) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* rring = smem + kGWarps * kGDepth * kGSlot;           // [DD][kGSS records]
  uint64_t* wfull = (uint64_t*)(rring + kGRecDepth * kRecSlot);       // [warp][D]
  uint64_t* rfull = wfull + kGWarps * kGDepth;                        // [DD]
  uint64_t* rempty = rfull + kGRecDepth;
  GInfo* info = (GInfo*)(rempty + kGRecDepth);                        // [kInfo]
  volatile int* seq = (volatile int*)(info + kInfo);                  // [kMaxSeq]
  asm volatile("griddepcontrol.launch_dependents;");
  if (pl.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    pl.trace[blockIdx.x * 4] = t;
  }
  for (int i = threadIdx.x; i < kMaxSeq; i += blockDim.x) seq[i] = -2;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kGWarps * kGDepth; ++i) mbar_init(&wfull[i], 1);
    for (int i = 0; i < kGRecDepth; ++i) {
      mbar_init(&rfull[i], 1);
      mbar_init(&rempty[i], kGWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // item 0: static (dynamic schedule: item blockIdx.x), needs no PDL wait
    const int i0 = pl.dynamic ? (int)blockIdx.x : pl.cta_start[blockIdx.x];
    const bool any = pl.dynamic ? true : i0 < pl.cta_start[blockIdx.x + 1];
    if (any) fill_info(&info[0], pl, i0);
    seq[0] = any ? i0 : -1;
  }
  __syncthreads();

  // ---- weight prefetch of item 0 (independent of every other kernel) --------
  unsigned char* ring = smem + warp * kGDepth * kGSlot;
  uint64_t* full = wfull + warp * kGDepth;
  // Issue cursor (lane 0) over this warp's stream of stages (wss_for supersteps
  // of its panel: weights, then the (s, z) of their groups at offset wss * wb),
  // skipping items in which the warp has no panel (ragged last item of a
  // GEMV); the current item's geometry is cached in registers.
  int ck = 0, cs = 0, islot = 0;  // cursor: sequence index, superstep, ring slot
  bool cdone = false;
  int c_k1 = 0, c_gps = 0, c_g = 0, c_wss = kGSS;
  uint32_t c_wb = 0;
  const char *c_w = nullptr, *c_z = nullptr;
  auto load_item = [&]() {
    for (;; ++ck) {
      if (seq_get(seq, info, ck, pl) < 0) {
        cdone = true;
        return;
      }
      const GInfo& f = info[ck % kInfo];
      if (f.p0 + warp < f.P) {
        c_k1 = f.k1;
        cs = f.k0;
        c_gps = f.gps;
        c_g = f.g;
        c_wb = f.wb;
        c_wss = wss_for(f.wb / 512, f.gps);
        c_w = f.w + warp * f.wstride;
        c_z = f.z + warp * f.zstride;
        return;
      }
    }
  };
  // next stage of the stream into slot islot; false at the end of an item
  // when `advance` is off (the first ring fill stays inside item 0: claiming a
  // later item waits for the prep kernel)
  auto issue_one = [&](bool advance) {
    const int nss = min(c_wss, c_k1 - cs);
    unsigned char* dst = ring + islot * kGSlot;
    uint64_t* bar = &full[islot];
    const uint32_t zb = (uint32_t)((c_gps > 0 ? nss * c_gps : c_g ? nss : 1) * 128);
    mbar_expect_tx(bar, nss * c_wb + zb);
    bulk_g2s(dst, c_w + (int64_t)cs * c_wb, nss * c_wb, bar);
    if (c_gps > 0) {
      bulk_g2s(dst + c_wss * c_wb, c_z + (int64_t)cs * c_gps * 128, zb, bar);
    } else if (c_g == 0) {  // full column: one group for the whole stage
      bulk_g2s(dst + c_wss * c_wb, c_z, 128, bar);
    } else {  // one group per superstep: the one containing it
      for (int j = 0; j < nss; ++j) {
        const int64_t gi = c_g ? (int64_t)(cs + j) * kSuper / c_g : 0;
        bulk_g2s(dst + c_wss * c_wb + j * 128, c_z + gi * 128, 128, bar);
      }
    }
    if (++islot == kGDepth) islot = 0;
    cs += nss;
    if (cs == c_k1) {
      ++ck;
      if (!advance) return false;
      load_item();
    }
    return true;
  };
  bool pend = false;  // the cursor stopped at the end of item 0: advance later
  int npre = 0;       // stages issued before the barrier
  if (warp < kGWarps && lane == 0) {
    if (seq[0] >= 0 && info[0].p0 + warp < info[0].P) {
      load_item();  // item 0 (staged by thread 0, no claim)
      while (npre < kGDepth) {
        ++npre;
        if (!issue_one(false)) {
          pend = true;
          break;
        }
      }
    } else {
      pend = true;  // no panel in item 0: start from item 1 after the barrier
      ck = 1;
    }
  }

  if (warp == kGWarps) {
    // ---- activation-record producer (after the PDL wait on the prep kernel)
    if (lane == 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int slot = 0;
      uint32_t ph = 0;
      for (int k = 0;; ++k) {
        if (seq_get(seq, info, k, pl) < 0) break;
        const GInfo& f = info[k % kInfo];
        // fields in registers: the asm memory clobbers below would otherwise
        // force a reload per stage
        const int K1 = f.k1;
        const unsigned char* src = f.rec;
        bool claimed = false;
        for (int s = f.k0; s < K1; s += kGSS) {
          // claim (and stage) the next item a few stages before the issue
          // cursors need it, hiding the global atomic's latency
          if (!claimed && s + 3 * kGSS >= K1) {
            seq_get(seq, info, k + 1, pl);
            claimed = true;
          }
          const uint32_t bytes = (uint32_t)(min(kGSS, K1 - s) * kRecBytes);
          mbar_wait(&rempty[slot], ph ^ 1u);
          mbar_expect_tx(&rfull[slot], bytes);
          bulk_g2s(rring + slot * kRecSlot, src + (size_t)s * kRecBytes, bytes, &rfull[slot]);
          if (++slot == kGRecDepth) {
            slot = 0;
            ph ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---- consumer warp: panel p0 + warp of every item of this CTA ---------------
  if (lane == 0 && pend) {  // top the ring up from the items after item 0
    // (a claim waits on the prep kernel; the rest of the CTA is not held)
    load_item();
    for (; npre < kGDepth && !cdone; ++npre) issue_one(true);
  }
  __syncwarp();

  int wslot = 0, rslot = 0;
  uint32_t wph = 0, rph = 0;
  bool waited = false;
  for (int k = 0;; ++k) {
    int it = 0;
    if (lane == 0) it = seq_get(seq, info, k, pl);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it < 0) break;
    __threadfence_block();
    const GInfo& f = info[k % kInfo];
    const int p = f.p0 + warp;
    const bool active = p < f.P;
    const int combo = f.combo;
    const int K0 = f.k0, K1 = f.k1;  // registers (see the producer)
    float* const yg = (float*)((char*)f.y + pl.ydelta);
    const int64_t ldy = f.ldy;
    const int M = f.M, m = f.m, split = f.split;
    float yv[2] = {0.f, 0.f};
    // the item's stage loop, specialised per (bits, groups per superstep): no
    // dispatch inside the loop, compile-time stage geometry
    auto stage_loop = [&](auto bits_c, auto gps_c) {
      constexpr int B = decltype(bits_c)::value, G = decltype(gps_c)::value;
      constexpr int WB = B * 512, ZPJ = (G > 0 ? G : 1) * 128, WSS = wss_for(B, G);
      const int zpj = G > 0 || f.g ? ZPJ : 0;  // full column: one (s, z) block per stage
      int sub = 0;
      for (int s = K0; s < K1; s += kGSS) {
        const int nss = min(kGSS, K1 - s);
        mbar_wait(&rfull[rslot], rph);
        if (active) {
          // a weight stage spans WSS / kGSS record stages (sub = the part done)
          if (sub == 0) mbar_wait(&full[wslot], wph);
          const unsigned char* stg = ring + wslot * kGSlot;
          const unsigned char* rec = rring + rslot * kRecSlot;
          if ((pl.mode & 15) != 1) {
#pragma unroll
            for (int j = 0; j < kGSS; ++j) {
              if (j < nss) {
                uint4 w[B];
                const int js = sub + j;
#pragma unroll
                for (int v = 0; v < B; ++v) w[v] = ((const uint4*)(stg + js * WB))[v * 32 + lane];
                group_superstep<B, G>(w, (const float2*)(stg + WSS * WB + js * zpj),
                                      rec + j * kRecBytes, yv);
              }
            }
          }
          sub += kGSS;
          if (sub == WSS || s + kGSS >= K1) {
            sub = 0;
            __syncwarp();
            if (lane == 0 && !cdone) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue_one(true);
            }
            if (++wslot == kGDepth) {
              wslot = 0;
              wph ^= 1u;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[rslot]);
        if (++rslot == kGRecDepth) {
          rslot = 0;
          rph ^= 1u;
        }
      }
    };
    using std::integral_constant;
    switch (combo) {
#define QG_CASE(B, G) \
  case (B - 2) * 5 + G: stage_loop(integral_constant<int, B>{}, integral_constant<int, G>{}); break;
      QG_CASE(2, 0) QG_CASE(2, 1) QG_CASE(2, 2) QG_CASE(2, 4) QG_CASE(2, 8)
      QG_CASE(3, 0) QG_CASE(3, 1) QG_CASE(3, 2) QG_CASE(3, 4) QG_CASE(3, 8)
      QG_CASE(4, 0) QG_CASE(4, 1) QG_CASE(4, 2) QG_CASE(4, 4) QG_CASE(4, 8)
#undef QG_CASE
      default: break;
    }
    if (active) {
      const int gq = lane >> 2, t = lane & 3;
      const float v0 = yv[0] + __shfl_xor_sync(0xffffffffu, yv[0], 1);
      const float v1 = yv[1] + __shfl_xor_sync(0xffffffffu, yv[1], 1);
      const int tk = t >> 1;
      if (!waited) {  // y may be read or written by the preceding kernel
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
      }
      if ((t & 1) == 0 && tk < M) {
        const int64_t c0 = (int64_t)p * 16 + gq;
        float* yr = yg + tk * ldy;
        if (split) {
          if (c0 < m) atomicAdd(yr + c0, v0);
          if (c0 + 8 < m) atomicAdd(yr + c0 + 8, v1);
        } else {
          if (c0 < m) yr[c0] = v0;
          if (c0 + 8 < m) yr[c0 + 8] = v1;
        }
      }
    }
  }
  if (pl.trace && lane == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&pl.trace[blockIdx.x * 4 + 3], t);
  }
}

constexpr int kGSmem = kGWarps * kGDepth * kGSlot + kGRecDepth * kRecSlot +
                       (kGWarps * kGDepth + 2 * kGRecDepth) * 8 + kInfo * sizeof(GInfo) +
                       kMaxSeq * 4;

}  // namespace qigen

using namespace qigen;

// tuning aid (per calling thread): 1 stream only; at create: 16 split every K
// in two, (pct+1) << 8 sets the split threshold (1 << 8: never split)
static thread_local int g_group_mode = 0;

struct qigen_gemv_group {
  void* blob = nullptr;  // device: descs | items | cta_start
  unsigned char* rec = nullptr;
  GPlan plan{};
  int grid = 0, max_ks = 0;
  bool any_split = false;  // some GEMV adds two K halves into y with atomics
};

// Kind of memory behind p: device (or managed), page-locked host, or -1 for
// memory the GPU cannot address (pageable host).
static int mem_kind(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return 0;
  if (a.type == cudaMemoryTypeHost) return 1;
  return -1;
}

extern "C" int qigen_gemv_group_create(int count, const qigen_gemv_desc* descs,
                                       qigen_gemv_group** out) {
  QIGEN_CHECK_ARG(out && descs && count > 0, QIGEN_ERR_ARG, "bad group arguments");
  std::vector<GDesc> ds(count);
  int64_t recs = 0;
  int max_ks = 0;
  for (int i = 0; i < count; ++i) {
    const qigen_gemv_desc& e = descs[i];
    QIGEN_CHECK_ARG(e.bits == 2 || e.bits == 3 || e.bits == 4, QIGEN_ERR_CONFIG,
                    "gemv %d: bits must be one of (2, 3, 4), got %d", i, e.bits);
    QIGEN_CHECK_ARG(e.qw && e.qsz && e.x && e.y && e.n > 0 && e.m > 0, QIGEN_ERR_ARG,
                    "gemv %d: null pointer or empty matrix", i);
    QIGEN_CHECK_ARG(e.group_size == 0 || e.n % e.group_size == 0, QIGEN_ERR_CONFIG,
                    "gemv %d: group size %lld does not divide row count %lld", i,
                    (long long)e.group_size, (long long)e.n);
    QIGEN_CHECK_ARG(e.group_size == 0 || e.group_size == 32 || e.group_size == 64 ||
                        e.group_size == 128 || e.group_size % kSuper == 0,
                    QIGEN_ERR_UNSUPPORTED, "gemv %d: unsupported group size %lld", i,
                    (long long)e.group_size);
    QIGEN_CHECK_ARG(e.tokens >= 1 && e.tokens <= kGTP, QIGEN_ERR_UNSUPPORTED,
                    "gemv %d: the grouped GEMV takes 1 or 2 activation rows", i);
    QIGEN_CHECK_ARG(e.x_dtype >= 0 && e.x_dtype <= 2, QIGEN_ERR_ARG, "gemv %d: bad x dtype", i);
    QIGEN_CHECK_ARG(e.ldx >= e.n && e.ldy >= e.m, QIGEN_ERR_ARG, "gemv %d: leading dimensions", i);
    // x and y may be device or page-locked host memory (zero-copy over PCIe);
    // pageable host memory would fault inside the kernel
    QIGEN_CHECK_ARG(mem_kind(e.x) >= 0 && mem_kind(e.y) >= 0, QIGEN_ERR_ARG,
                    "gemv %d: x and y must be device or page-locked host memory", i);
    GDesc& d = ds[i];
    d.qw = (const uint4*)e.qw;
    d.qsz = (const float2*)e.qsz;
    d.x = e.x;
    d.y = e.y;
    d.ldx = e.ldx;
    d.ldy = e.ldy;
    d.n = e.n;
    d.m = e.m;
    d.KS = (int)supersteps(e.n);
    d.P = (int)panels(e.m);
    d.Gp = (int)groups_padded(e.n, e.group_size);
    d.g = (int)e.group_size;
    d.bits = e.bits;
    d.gps = e.group_size == 32 ? 8 : e.group_size == 64 ? 4 : e.group_size == 128 ? 2
            : e.group_size == 256 ? 1 : 0;
    d.M = (int)e.tokens;
    d.x_dtype = e.x_dtype;
    d.split = 0;  // decided below, once every GEMV's item cost is known
    d.rec0 = recs;
    recs += d.KS;
    max_ks = std::max(max_ks, d.KS);
  }
  // time model of an item per SM: max(stream at ~44 GB/s, issue at ~4.5
  // instr/ns); ~110 warp instructions per panel superstep + ~17 per flush unit
  auto item_cost = [](const GDesc& d, int act, int nks) {
    const int zb = (d.gps > 0 ? d.gps : 1) * 128;
    const int ups = d.gps >= 2 ? d.gps : 1;
    const double bytes = (double)nks * (act * (d.bits * 512 + zb) + kRecBytes);
    const double instr = (double)nks * act * (110.0 + 17.0 * ups);
    return std::max(bytes / 44.0, instr / 4.5);
  };
  // The greedy schedule's tail is about one of the last (cheapest) items: the
  // GEMVs whose full-K items cost < kSplitPct % of the largest get their K
  // split in two halves (each >= 4 supersteps); splitting everything costs
  // more per-item overhead than it saves (measured).
  {
    double mx = 0.0;
    for (const GDesc& d : ds) mx = std::max(mx, item_cost(d, kGWarps, d.KS));
    const int pct_knob = (g_group_mode >> 8) & 0xff;
    const double pct = (g_group_mode & 16) ? 101.0 : pct_knob ? pct_knob - 1 : kSplitPct;
    for (GDesc& d : ds) d.split = (d.KS >= 8 && item_cost(d, kGWarps, d.KS) < mx * pct / 100.0);
    // y in host memory (zero-copy output): plain stores only, never split atomics
    for (GDesc& d : ds)
      if (d.split && mem_kind(d.y) != 0) d.split = 0;
  }
  // items (GEMV x 16 panels x K range) and their cost
  std::vector<GItem> items;
  std::vector<double> cost;
  for (int i = 0; i < count; ++i) {
    const GDesc& d = ds[i];
    const int halves = d.split ? 2 : 1;
    for (int p0 = 0; p0 < d.P; p0 += kGWarps)
    for (int hf = 0; hf < halves; ++hf) {
      const int act = std::min(kGWarps, d.P - p0);
      const int k0 = hf * (d.KS / 2), k1 = halves == 1 || hf == 1 ? d.KS : d.KS / 2;
      items.push_back({i, p0, k0, k1});
      cost.push_back(item_cost(d, act, k1 - k0));
    }
  }
  int dev = 0, sms = 148;
  QIGEN_CUDA_RET(cudaGetDevice(&dev));
  QIGEN_CUDA_RET(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::max(1, std::min<int>(sms, (int)items.size()));
  // longest-processing-time-first greedy: biggest item to the least-loaded CTA
  std::vector<int> order(items.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  using Load = std::pair<double, int>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int c = 0; c < grid; ++c) heap.push({0.0, c});
  std::vector<std::vector<int>> per(grid);
  for (int i : order) {
    Load l = heap.top();
    heap.pop();
    per[l.second].push_back(i);
    heap.push({l.first + cost[i], l.second});
  }
  // Dynamic schedule (default): items in decreasing-cost order, CTA c starts
  // with item c and then claims the next unclaimed one (greedy list
  // scheduling, which absorbs the model's errors).  Static LPT lists when a
  // CTA's claim sequence could overflow its shared-memory table.
  const bool dynamic = (int)items.size() - grid < kMaxSeq;
  QIGEN_CHECK_ARG(dynamic || (int)items.size() / grid + 2 < kMaxSeq, QIGEN_ERR_UNSUPPORTED,
                  "grouped GEMV: too many work items (%d)", (int)items.size());
  std::vector<GItem> flat;
  std::vector<int> start(grid + 1, 0);
  if (dynamic) {
    for (int i : order) flat.push_back(items[i]);
    for (int c = 0; c <= grid; ++c) start[c] = c;
  } else {
    for (int c = 0; c < grid; ++c) {
      start[c] = (int)flat.size();
      for (int i : per[c]) flat.push_back(items[i]);
    }
    start[grid] = (int)flat.size();
  }

  auto* g = new qigen_gemv_group();
  const size_t db = ds.size() * sizeof(GDesc), ib = flat.size() * sizeof(GItem),
               sb = start.size() * sizeof(int);
  const size_t ib_off = (db + 255) / 256 * 256, sb_off = ib_off + (ib + 255) / 256 * 256;
  const size_t cnt_off = sb_off + (sb + 255) / 256 * 256;
  cudaError_t e1 = cudaMalloc(&g->blob, cnt_off + 256);
  cudaError_t e2 = e1 == cudaSuccess ? cudaMalloc((void**)&g->rec, (size_t)recs * kRecBytes) : e1;
  if (e2 != cudaSuccess) {
    if (g->blob) cudaFree(g->blob);
    delete g;
    QIGEN_CUDA_RET(e2);
  }
  char* b = (char*)g->blob;
  QIGEN_CUDA_RET(cudaMemcpy(b, ds.data(), db, cudaMemcpyHostToDevice));
  QIGEN_CUDA_RET(cudaMemcpy(b + ib_off, flat.data(), ib, cudaMemcpyHostToDevice));
  QIGEN_CUDA_RET(cudaMemcpy(b + sb_off, start.data(), sb, cudaMemcpyHostToDevice));
  QIGEN_CUDA_RET(cudaMemset(b + cnt_off, 0, 256));
  QIGEN_CUDA_RET(cudaMemcpy(b + cnt_off, &grid, sizeof(int), cudaMemcpyHostToDevice));
  g->plan.desc = (const GDesc*)b;
  g->plan.items = (const GItem*)(b + ib_off);
  g->plan.cta_start = (const int*)(b + sb_off);
  g->plan.rec = g->rec;
  g->plan.counter = (int*)(b + cnt_off);
  g->plan.nitems = (int)flat.size();
  g->plan.first_dyn = grid;
  g->plan.dynamic = dynamic ? 1 : 0;
  g->plan.total_items = recs * 64;
  g->plan.count = count;
  g->plan.mode = 0;
  g->plan.ydelta = 0;
  g->plan.trace = nullptr;
  g->grid = grid;
  g->max_ks = max_ks;
  for (const GDesc& d : ds) g->any_split = g->any_split || d.split;
  static OncePerDevice once;
  const int cst = once.run([]() -> int {
    QIGEN_CUDA_RET(cudaFuncSetAttribute(gemv_group_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, kGSmem));
    return QIGEN_OK;
  });
  if (cst) {
    qigen_gemv_group_destroy(g);
    return cst;
  }
  *out = g;
  return QIGEN_OK;
}

extern "C" int qigen_debug_group_mode(int mode) {
  g_group_mode = mode;
  return QIGEN_OK;
}

extern "C" int qigen_gemv_group_run(const qigen_gemv_group* g, void* stream) {
  QIGEN_CHECK_ARG(g, QIGEN_ERR_ARG, "null group");
  GPlan plan = g->plan;
  plan.mode = g_group_mode & 47;
  plan.trace = g_trace;
  cudaLaunchAttribute pa;
  pa.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pa.val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t pc = {};
  pc.gridDim = dim3((unsigned)((g->max_ks * 64 + 255) / 256), (unsigned)g->plan.count, 1);
  pc.blockDim = dim3(256, 1, 1);
  pc.stream = (cudaStream_t)stream;
  pc.attrs = &pa;
  pc.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&pc, group_prep_kernel, plan));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)g->grid, 1, 1);
  cfg.blockDim = dim3((kGWarps + 1) * 32, 1, 1);
  cfg.dynamicSmemBytes = kGSmem;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = &pa;
  cfg.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, gemv_group_kernel, plan));
  return QIGEN_OK;
}

extern "C" int qigen_gemv_group_run_rebased(const qigen_gemv_group* g, const void* y_plan_base,
                                            void* y_base, void* stream) {
  QIGEN_CHECK_ARG(g && y_plan_base && y_base, QIGEN_ERR_ARG, "null pointer");
  // the outputs move to y_base's memory: it must be GPU-addressable, and a plan
  // whose K-split GEMVs add into y with atomics must not be moved to host memory
  const int kind = mem_kind(y_base);
  QIGEN_CHECK_ARG(kind >= 0, QIGEN_ERR_ARG,
                  "y_base must be device or page-locked host memory");
  QIGEN_CHECK_ARG(kind == 0 || !g->any_split, QIGEN_ERR_ARG,
                  "this plan K-splits some GEMVs (atomic adds into y): y_base must be device "
                  "memory; create the plan with host y to run it on host blocks");
  qigen_gemv_group h = *g;
  h.plan.ydelta = (int64_t)((const char*)y_base - (const char*)y_plan_base);
  return qigen_gemv_group_run(&h, stream);
}

extern "C" int qigen_gemv_group_run_host(const qigen_gemv_group* g, const void* x_host,
                                         void* x_dev, size_t x_bytes, const void* y_dev,
                                         void* y_host, size_t y_bytes, void* stream) {
  QIGEN_CHECK_ARG(g && x_host && x_dev && y_dev && y_host, QIGEN_ERR_ARG, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  QIGEN_CUDA_RET(cudaMemcpyAsync(x_dev, x_host, x_bytes, cudaMemcpyHostToDevice, st));
  const int rc = qigen_gemv_group_run(g, stream);
  if (rc != QIGEN_OK) return rc;
  QIGEN_CUDA_RET(cudaMemcpyAsync(y_host, y_dev, y_bytes, cudaMemcpyDeviceToHost, st));
  QIGEN_CUDA_RET(cudaStreamSynchronize(st));
  return QIGEN_OK;
}

extern "C" int qigen_gemv_group_destroy(qigen_gemv_group* g) {
  if (!g) return QIGEN_OK;
  if (g->blob) cudaFree(g->blob);
  if (g->rec) cudaFree(g->rec);
  delete g;
  return QIGEN_OK;
}
