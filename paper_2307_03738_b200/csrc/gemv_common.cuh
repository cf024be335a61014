// Device helpers shared by the split-K GEMV (gemv.cu) and the grouped GEMV
// (gemv_grouped.cu): PTX wrappers for mbarriers / bulk copies / cluster stores,
// the u8 x s8 IMMA, code extraction from the panel layout and
// the fixed-point activation digitiser.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace qigen {

// ---- PTX helpers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t done = 0;
  // with a suspend-time hint the waiting warp sleeps until the phase
  // completes (or the hint expires) instead of spinning on issue slots
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x989680u)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// Cluster address of the same shared-memory offset in CTA `rank`.
__device__ __forceinline__ uint32_t mapa(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
// 4-byte store into another CTA's shared memory, completing tx on its mbarrier.
__device__ __forceinline__ void st_async(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   addr),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void imma(int (&c)[4], const uint32_t (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// m16n8k16 IMMA (zero accumulator input): A = one k half of the k32 fragment
// (a0: rows gq, a1: rows gq+8), B = the matching digit word.
__device__ __forceinline__ void imma16(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%7,%7,%7,%7};"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
      : "r"(a0), "r"(a1), "r"(b), "r"(0));
}

// Fragment registers of local step sl (0..7) from the lane's superstep words.
// Codes stay in place (one AND each); every accumulator row then carries a
// power-of-two scale: RowScale<BITS>::hi for rows gq+8 (rows gq: 1), and for
// 2-bit odd steps a further x16 on both rows (kept in the odd accumulator set).
template <int BITS>
__device__ __forceinline__ void extract(const uint4 (&w)[BITS], int sl, uint32_t (&a)[4]);

template <>
__device__ __forceinline__ void extract<4>(const uint4 (&w)[4], int sl, uint32_t (&a)[4]) {
  const uint4 u = w[sl >> 1];
  const uint32_t A = (sl & 1) ? u.z : u.x, B = (sl & 1) ? u.w : u.y;
  a[0] = A & 0x0F0F0F0Fu;  // rows gq,   k 4t..      x1
  a[1] = A & 0xF0F0F0F0u;  // rows gq+8, k 4t..      x16
  a[2] = B & 0x0F0F0F0Fu;  // rows gq,   k 16+4t..   x1
  a[3] = B & 0xF0F0F0F0u;  // rows gq+8, k 16+4t..   x16
}

template <>
__device__ __forceinline__ void extract<2>(const uint4 (&w)[2], int sl, uint32_t (&a)[4]) {
  const uint4 u = w[sl >> 2];
  const int q = sl & 2;  // word pair of this step pair
  const uint32_t X = q == 0 ? u.x : u.z, Y = q == 0 ? u.y : u.w;
  const uint32_t m0 = (sl & 1) ? 0x30303030u : 0x03030303u;  // x1  (odd: x16)
  const uint32_t m1 = (sl & 1) ? 0xC0C0C0C0u : 0x0C0C0C0Cu;  // x4  (odd: x64)
  a[0] = X & m0;
  a[1] = X & m1;
  a[2] = Y & m0;
  a[3] = Y & m1;
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
    a[0] = A & 0x07070707u;  // x1
    a[1] = A & 0x38383838u;  // x8
    a[2] = B & 0x07070707u;
    a[3] = B & 0x38383838u;
  } else {
    a[0] = C & 0x07070707u;
    a[1] = C & 0x38383838u;
    a[2] = ((A >> 6) & 0x03030303u) | ((C >> 4) & 0x04040404u);  // x1
    a[3] = ((B >> 3) & 0x18181818u) | ((C >> 2) & 0x20202020u);  // x8
  }
}

template <int BITS>
struct RowScale {  // scale of the rows gq+8 accumulators relative to rows gq
  static constexpr float inv_hi = BITS == 4 ? 1.f / 16.f : BITS == 3 ? 1.f / 8.f : 1.f / 4.f;
};

__device__ __forceinline__ int sbyte(int v) { return (int)(int8_t)(v & 0xFF); }

// ---- activation digitisation (shared by the fused prologue and the prep kernel)
// An "item" is 4 consecutive rows of one token.  IPU consecutive lanes hold one
// exponent unit (U = min(g, 128) rows); they agree on E (max |x| < 2^E) with one
// REDUX, split m = rint(x 2^(30-E)) into balanced signed bytes, and reduce the
// exact unit sum of m.  Returns the four digit words (d0..d3 of the 4 rows).
struct Digits {
  uint32_t dw[4];
  float xsum;   // sum of m over the unit (valid in every lane of the unit)
  float scale;  // 2^(E-30)
};

template <int IPU>
__device__ __forceinline__ Digits digitize(const float (&v)[4], uint32_t umask) {
  Digits d;
  const float m4 = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
  const uint32_t umx = __reduce_max_sync(umask, __float_as_uint(m4));
  // max < 2^e; e from the biased exponent (denormal max: 2^-126 still bounds it)
  const int e = umx ? (int)((umx >> 23) & 0xFF) - 126 : 0;
  const int k = 30 - e, k1 = k >> 1, k2 = k - k1;  // 2^k may leave the f32 range
  const float f1 = __int_as_float((127 + k1) << 23), f2 = __int_as_float((127 + k2) << 23);
  int mv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) mv[i] = __float2int_rn(__fmul_rn(__fmul_rn(v[i], f1), f2));
  // balanced base-256 digits: with t = m + 0x808080, digit j < 3 is byte j of t
  // minus 128 (i.e. byte ^ 0x80 as s8) and the top digit is t >> 24 (|.| <= 64)
  uint32_t tt[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) tt[i] = (uint32_t)(mv[i] + 0x808080);
  const uint32_t lo01 = __byte_perm(tt[0], tt[1], 0x5140), lo23 = __byte_perm(tt[2], tt[3], 0x5140);
  const uint32_t hi01 = __byte_perm(tt[0], tt[1], 0x7362), hi23 = __byte_perm(tt[2], tt[3], 0x7362);
  d.dw[3] = __byte_perm(lo01, lo23, 0x5410) ^ 0x80808080u;  // byte 0 of each
  d.dw[2] = __byte_perm(lo01, lo23, 0x7632) ^ 0x80808080u;  // byte 1
  d.dw[1] = __byte_perm(hi01, hi23, 0x5410) ^ 0x80808080u;  // byte 2
  d.dw[0] = __byte_perm(hi01, hi23, 0x7632);                // byte 3 = t >> 24
  // exact unit sum of m, split 16/16 so each half fits an int32 REDUX
  int slo = 0, shi = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    slo += mv[i] & 0xFFFF;
    shi += mv[i] >> 16;
  }
  slo = __reduce_add_sync(umask, slo);
  shi = __reduce_add_sync(umask, shi);
  d.xsum = fmaf((float)shi, 65536.f, (float)slo);
  d.scale = umx ? __int_as_float((127 + e - 30) << 23) : 0.f;  // e - 30 >= -156: see below
  if (umx && e - 30 < -126) d.scale = scalbnf(1.f, e - 30);
  return d;
}

// Digit store: B-fragment words of (step st, token tk) at [st][TP][j][t] x (b0, b1).
__device__ __forceinline__ void store_digits(uint32_t* base, int st, int tk, int TP, int sub,
                                             const Digits& d) {
  uint32_t* dst = base + ((st * TP + tk) * 16 + (sub & 3)) * 2 + (sub >> 2);
  dst[0] = d.dw[0];
  dst[8] = d.dw[1];
  dst[16] = d.dw[2];
  dst[24] = d.dw[3];
}

}  // namespace qigen
