// Bit-exact quantization and packing on the GPU, plus the panel re-tiling.
//
// Compiled with -fmad=false: the parameter math of quant.py:74-94 rounds every
// fp64 operation separately and the codes must match the reference bit for
// bit.  None of these kernels is on the per-token hot path; they
// run once per weight matrix (setup), so they favour clarity over speed.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace qigen {

// ---------------------------------------------------------------------------
// quant.py:70-71 round half away from zero; np.clip keeps a value equal to a
// bound unchanged (so -0.0 survives clip(.., 0, max)).
__device__ __forceinline__ double rha(double v) { return copysign(floor(fabs(v) + 0.5), v); }
__device__ __forceinline__ double clip_keep(double v, double lo, double hi) {
  double o = v < lo ? lo : v;
  return o > hi ? hi : o;
}

// One thread per (group, column).  Rows of a group are visited in order and
// min/max keep the LAST of equal values (numpy's strided minimum.reduce), which
// decides the sign of a zero minimum and hence of z.
__global__ void quantize_kernel(const float* __restrict__ w, int64_t n, int64_t m, int bits,
                                int64_t g, int zero_mode, uint8_t* __restrict__ codes,
                                float* __restrict__ scales, float* __restrict__ zeros) {
  const int64_t G = n / g;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= G * m) return;
  const int64_t gi = idx / m, col = idx % m;
  const float* src = w + gi * g * m + col;
  double mn = (double)src[0], mx = mn;
  for (int64_t r = 1; r < g; ++r) {
    const double v = (double)src[r * m];
    mn = (mn < v) ? mn : v;
    mx = (mx > v) ? mx : v;
  }
  const double max_code = (double)((1 << bits) - 1);
  const double span = mx - mn;
  const double s = (span == 0.0) ? 1.0 : span / max_code;
  const float s32 = (float)s;  // round to nearest
  const double s64 = (double)s32;
  const double z = -mn / s64;
  float z32;
  if (zero_mode == QIGEN_ZERO_QUANTIZED)
    z32 = (float)clip_keep(rha(z), 0.0, max_code);
  else
    z32 = (float)z;
  const double z64 = (double)z32;
  scales[gi * m + col] = s32;
  zeros[gi * m + col] = z32;
  uint8_t* dst = codes + gi * g * m + col;
  for (int64_t r = 0; r < g; ++r) {
    const double v = (double)src[r * m] / s64 + z64;
    dst[r * m] = (uint8_t)clip_keep(rha(v), 0.0, max_code);
  }
}

__global__ void dequantize_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ s,
                                  const float* __restrict__ z, int64_t n, int64_t m, int64_t g,
                                  float* __restrict__ out) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * m) return;
  const int64_t r = idx / m, col = idx % m;
  const int64_t gi = r / g;
  out[idx] = s[gi * m + col] * ((float)codes[idx] - z[gi * m + col]);
}

// ---------------------------------------------------------------------------
// packing.py:42-70 + :204-214.  Thread per (word-row r, column c).
__global__ void pack_rowseq_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t m,
                                   int bits, uint32_t* __restrict__ words) {
  const int unit = unit_codes(bits), kw = unit_words(bits);
  const int64_t wr = n / unit;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= wr * m) return;
  const int64_t r = idx / m, c = idx % m;
  const uint8_t* src = codes + r * unit * m + c;
  if (bits != 3) {
    uint32_t wv = 0;
    for (int j = 0; j < unit; ++j) wv |= (uint32_t)src[j * m] << (j * bits);
    words[r * m + c] = wv;
  } else {
    uint32_t wv[3] = {0u, 0u, 0u};
    for (int j = 0; j < 32; ++j) {  // 96-bit little-endian stream, bit 3j+t
      const uint32_t v = src[j * m];
      const int bit = 3 * j, k = bit >> 5, off = bit & 31;
      wv[k] |= v << off;
      if (off > 29) wv[k + 1] |= v >> (32 - off);  // straddles into the next word
    }
    for (int k = 0; k < 3; ++k) words[(r * 3 + k) * m + c] = wv[k];
  }
}

__global__ void unpack_rowseq_kernel(const uint32_t* __restrict__ words, int64_t n, int64_t m,
                                     int bits, uint8_t* __restrict__ codes) {
  const int unit = unit_codes(bits);
  const int64_t wr = n / unit;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= wr * m) return;
  const int64_t r = idx / m, c = idx % m;
  uint8_t* dst = codes + r * unit * m + c;
  const uint32_t mask = (1u << bits) - 1u;
  if (bits != 3) {
    const uint32_t wv = words[r * m + c];
    for (int j = 0; j < unit; ++j) dst[j * m] = (uint8_t)((wv >> (j * bits)) & mask);
  } else {
    uint32_t wv[3];
    for (int k = 0; k < 3; ++k) wv[k] = words[(r * 3 + k) * m + c];
    for (int j = 0; j < 32; ++j) {  // kernelgen.py:116-124 straddle rule
      const int bit = 3 * j, k = bit >> 5, off = bit & 31;
      uint32_t v = wv[k] >> off;
      if (off > 29) v |= (wv[k + 1] & ((1u << (3 - (32 - off))) - 1u)) << (32 - off);
      dst[j * m] = (uint8_t)(v & mask);
    }
  }
}

// packing.py:175-201.  One CUDA block per Morton block; its storage offset is
// the sum of the compact sizes of all earlier blocks (ragged edges unpadded).
__global__ void permute_zcurve_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                      int64_t n, int64_t m, int bits, int64_t m_b, int64_t t_b,
                                      const int32_t* __restrict__ blk_rc, int to_zcurve) {
  const int unit = unit_codes(bits), kw = unit_words(bits);
  const int64_t wr = n / unit, wgb = m_b / unit;
  __shared__ int64_t s_off;
  const int bi = blockIdx.x;
  if (threadIdx.x == 0) {
    int64_t off = 0;
    for (int b = 0; b < bi; ++b) {
      const int64_t rb = blk_rc[2 * b], cb = blk_rc[2 * b + 1];
      const int64_t rows = min(wgb, wr - rb * wgb), cols = min(t_b, m - cb * t_b);
      off += rows * kw * cols;
    }
    s_off = off;
  }
  __syncthreads();
  const int64_t rb = blk_rc[2 * bi], cb = blk_rc[2 * bi + 1];
  const int64_t r0 = rb * wgb, c0 = cb * t_b;
  const int64_t rows = min(wgb, wr - r0), cols = min(t_b, m - c0);
  const int64_t total = rows * kw * cols;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t rr = e / (kw * cols), rem = e % (kw * cols);
    const int64_t k = rem / cols, cc = rem % cols;
    const int64_t rs = ((r0 + rr) * kw + k) * m + c0 + cc;
    const int64_t st = s_off + e;
    if (to_zcurve) dst[st] = src[rs];
    else dst[rs] = src[st];
  }
}

// ---------------------------------------------------------------------------
// Panel layout.  For panel p, superstep s, lane l = 4*gq + t,
// the lane owns 4*bits words; element (local step sl in 0..7, fragment
// register j in 0..3, byte i in 0..3) is
//     column = 16p + gq + 8*(j & 1),  k = 256s + 32*sl + 16*(j >> 1) + 4t + i
// i.e. exactly the u8 A-fragment of mma.m16n8k32 for step sl.  The bit
// positions are chosen so that the GEMV rebuilds fragment registers with a
// single AND mask each (codes left in place, scaled by a power of two that is
// uniform per accumulator row and undone at the flush; gemv.cu: extract<>):
//   4-bit: word pair per step; low nibbles = rows gq, high nibbles = rows gq+8.
//   2-bit: word pair per step pair; 2-bit field 2*(sl&1) + (j&1) of byte i.
//   3-bit: word triple (A, B, C) per step pair; fields 0-2 / 3-5 of each byte,
//          the two last registers of the odd step spread over bits 6-7.
__device__ __forceinline__ void place_code(int bits, uint32_t* wv, int sl, int j, int i,
                                           uint32_t c) {
  if (bits == 4) {
    wv[2 * sl + (j >> 1)] |= c << (8 * i + 4 * (j & 1));
  } else if (bits == 2) {  // step pair -> words (X, Y); X: a0,a1  Y: a2,a3; odd step in fields 2,3
    wv[2 * (sl >> 1) + (j >> 1)] |= c << (8 * i + 2 * (2 * (sl & 1) + (j & 1)));
  } else {  // 3-bit: step pair -> words (A, B, C), fragment regs R0..R7
    const int q = 3 * (sl >> 1), R = 4 * (sl & 1) + j;
    if (R < 6) {
      wv[q + (R >> 1)] |= c << (8 * i + 3 * (R & 1));
    } else {
      wv[q + (R - 6)] |= (c & 3u) << (8 * i + 6);          // A (R6) / B (R7): bits 6-7
      wv[q + 2] |= ((c >> 2) & 1u) << (8 * i + 6 + (R - 6));  // C: bit 6 (R6) / 7 (R7)
    }
  }
}

__device__ __forceinline__ uint32_t read_code(int bits, const uint32_t* wv, int sl, int j, int i) {
  if (bits == 4) return (wv[2 * sl + (j >> 1)] >> (8 * i + 4 * (j & 1))) & 15u;
  if (bits == 2) return (wv[2 * (sl >> 1) + (j >> 1)] >> (8 * i + 2 * (2 * (sl & 1) + (j & 1)))) & 3u;
  const int q = 3 * (sl >> 1), R = 4 * (sl & 1) + j;
  if (R < 6) return (wv[q + (R >> 1)] >> (8 * i + 3 * (R & 1))) & 7u;
  return ((wv[q + (R - 6)] >> (8 * i + 6)) & 3u) | (((wv[q + 2] >> (8 * i + 6 + (R - 6))) & 1u) << 2);
}

// Thread per (panel, superstep, lane): writes the lane's 4*bits words as
// `bits` uint4 at ((p*KS + s)*bits + v)*32 + lane.
__global__ void panels_from_codes_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t m,
                                         int bits, uint4* __restrict__ qw) {
  const int64_t KS = supersteps(n), P = panels(m);
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * KS * 32) return;
  const int lane = idx & 31;
  const int64_t ps = idx >> 5;
  const int64_t p = ps / KS, s = ps % KS;
  const int gq = lane >> 2, t = lane & 3;
  uint32_t wv[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) wv[q] = 0u;
  for (int sl = 0; sl < 8; ++sl)
    for (int j = 0; j < 4; ++j) {
      const int64_t col = 16 * p + gq + 8 * (j & 1);
      for (int i = 0; i < 4; ++i) {
        const int64_t k = 256 * s + 32 * sl + 16 * (j >> 1) + 4 * t + i;
        const uint32_t c = (col < m && k < n) ? codes[k * m + col] : 0u;
        place_code(bits, wv, sl, j, i, c);
      }
    }
  for (int v = 0; v < bits; ++v)
    qw[((p * KS + s) * bits + v) * 32 + lane] =
        make_uint4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]);
}

__global__ void panels_to_codes_kernel(const uint4* __restrict__ qw, int64_t n, int64_t m,
                                       int bits, uint8_t* __restrict__ codes) {
  const int64_t KS = supersteps(n), P = panels(m);
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * KS * 32) return;
  const int lane = idx & 31;
  const int64_t ps = idx >> 5;
  const int64_t p = ps / KS, s = ps % KS;
  const int gq = lane >> 2, t = lane & 3;
  uint32_t wv[16];
  for (int v = 0; v < bits; ++v) {
    const uint4 u = qw[((p * KS + s) * bits + v) * 32 + lane];
    wv[4 * v] = u.x; wv[4 * v + 1] = u.y; wv[4 * v + 2] = u.z; wv[4 * v + 3] = u.w;
  }
  for (int sl = 0; sl < 8; ++sl)
    for (int j = 0; j < 4; ++j) {
      const int64_t col = 16 * p + gq + 8 * (j & 1);
      for (int i = 0; i < 4; ++i) {
        const int64_t k = 256 * s + 32 * sl + 16 * (j >> 1) + 4 * t + i;
        if (col < m && k < n) codes[k * m + col] = (uint8_t)read_code(bits, wv, sl, j, i);
      }
    }
}

// (s, z) float2 per (panel, padded group, panel column); ghosts are (0, 0).
__global__ void panel_params_kernel(const float* __restrict__ scales, const float* __restrict__ zeros,
                                    int64_t n, int64_t m, int64_t g, float2* __restrict__ qsz) {
  const int64_t P = panels(m), Gp = groups_padded(n, g);
  const int64_t G = (g == 0) ? 1 : n / g;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= P * Gp * 16) return;
  const int r = idx & 15;
  const int64_t pg = idx >> 4;
  const int64_t p = pg / Gp, gi = pg % Gp;
  const int64_t col = 16 * p + r;
  float2 v = make_float2(0.f, 0.f);
  if (col < m && gi < G) v = make_float2(scales[gi * m + col], zeros[gi * m + col]);
  qsz[idx] = v;
}

// per-group sums, fp64 accumulation, one rounding.
__global__ void input_sums_kernel(const float* __restrict__ x, int64_t n, int64_t g,
                                  float* __restrict__ out) {
  const int64_t gi = blockIdx.x;
  const int64_t len = (g == 0) ? n : g;
  const float* src = x + gi * len;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) acc += (double)src[i];
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) out[gi] = (float)acc;
  }
}

static inline unsigned blocks_for(int64_t total, int threads) {
  return (unsigned)((total + threads - 1) / threads);
}

}  // namespace qigen

using namespace qigen;

// ---------------------------------------------------------------------------
// Validation mirrors config.py: bits in {2,3,4} (:54-55), group divides n
// (:73-74), rows fill whole packing units (:108-113).
static int check_config(int64_t n, int64_t m, int bits, int64_t group) {
  QIGEN_CHECK_ARG(bits == 2 || bits == 3 || bits == 4, QIGEN_ERR_CONFIG,
                  "bits must be one of (2, 3, 4), got %d", bits);
  QIGEN_CHECK_ARG(n > 0 && m > 0, QIGEN_ERR_CONFIG, "matrix must be non-empty (%lld x %lld)",
                  (long long)n, (long long)m);
  QIGEN_CHECK_ARG(group >= 0, QIGEN_ERR_CONFIG, "group_size must be positive or 0 (FULL_COLUMN)");
  QIGEN_CHECK_ARG(group == 0 || n % group == 0, QIGEN_ERR_CONFIG,
                  "group size %lld does not divide row count %lld", (long long)group,
                  (long long)n);
  return QIGEN_OK;
}

extern "C" int qigen_quantize(const float* w, int64_t n, int64_t m, int bits, int64_t group,
                              int zero_mode, uint8_t* codes, float* scales, float* zeros,
                              void* stream) {
  int st = check_config(n, m, bits, group);
  if (st) return st;
  QIGEN_CHECK_ARG(w && codes && scales && zeros, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(zero_mode == 0 || zero_mode == 1, QIGEN_ERR_CONFIG, "unknown zero mode %d",
                  zero_mode);
  const int64_t g = group ? group : n;
  const int64_t total = (n / g) * m;
  quantize_kernel<<<blocks_for(total, 128), 128, 0, (cudaStream_t)stream>>>(
      w, n, m, bits, g, zero_mode, codes, scales, zeros);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_dequantize(const uint8_t* codes, const float* scales, const float* zeros,
                                int64_t n, int64_t m, int64_t group, float* out, void* stream) {
  QIGEN_CHECK_ARG(codes && scales && zeros && out, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(n > 0 && m > 0 && (group == 0 || n % group == 0), QIGEN_ERR_CONFIG,
                  "bad shape / group");
  dequantize_kernel<<<blocks_for(n * m, 256), 256, 0, (cudaStream_t)stream>>>(
      codes, scales, zeros, n, m, group ? group : n, out);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_pack_rowseq(const uint8_t* codes, int64_t n, int64_t m, int bits,
                                 uint32_t* words, void* stream) {
  int st = check_config(n, m, bits, 0);
  if (st) return st;
  QIGEN_CHECK_ARG(n % unit_codes(bits) == 0, QIGEN_ERR_CONFIG,
                  "row count %lld must be a multiple of %d for %d-bit packing", (long long)n,
                  unit_codes(bits), bits);
  QIGEN_CHECK_ARG(codes && words, QIGEN_ERR_ARG, "null pointer");
  const int64_t total = n / unit_codes(bits) * m;
  pack_rowseq_kernel<<<blocks_for(total, 128), 128, 0, (cudaStream_t)stream>>>(codes, n, m, bits,
                                                                                words);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_unpack_rowseq(const uint32_t* words, int64_t n, int64_t m, int bits,
                                   uint8_t* codes, void* stream) {
  int st = check_config(n, m, bits, 0);
  if (st) return st;
  QIGEN_CHECK_ARG(n % unit_codes(bits) == 0, QIGEN_ERR_PACK, "word count is not whole units");
  QIGEN_CHECK_ARG(codes && words, QIGEN_ERR_ARG, "null pointer");
  const int64_t total = n / unit_codes(bits) * m;
  unpack_rowseq_kernel<<<blocks_for(total, 128), 128, 0, (cudaStream_t)stream>>>(words, n, m, bits,
                                                                                  codes);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_permute_zcurve(const uint32_t* src, uint32_t* dst, int64_t n, int64_t m,
                                    int bits, int64_t m_b, int64_t t_b, const int32_t* blk_rc,
                                    int64_t nblk, int to_zcurve, void* stream) {
  int st = check_config(n, m, bits, 0);
  if (st) return st;
  QIGEN_CHECK_ARG(src && dst && blk_rc, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(m_b > 0 && t_b > 0 && m_b % unit_codes(bits) == 0, QIGEN_ERR_PACK,
                  "plan m_b=%lld does not cover whole %d-bit packed words", (long long)m_b, bits);
  const int64_t rbs = (n + m_b - 1) / m_b, cbs = (m + t_b - 1) / t_b;
  QIGEN_CHECK_ARG(nblk == rbs * cbs, QIGEN_ERR_PACK, "block table has %lld blocks, grid needs %lld",
                  (long long)nblk, (long long)(rbs * cbs));
  if (nblk == 0) return QIGEN_OK;
  permute_zcurve_kernel<<<(unsigned)nblk, 256, 0, (cudaStream_t)stream>>>(src, dst, n, m, bits, m_b,
                                                                          t_b, blk_rc, to_zcurve);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int64_t qigen_panel_words(int64_t n, int64_t m, int bits) {
  return tile_words(n, m, bits);
}
extern "C" int64_t qigen_panel_params(int64_t n, int64_t m, int64_t group) {
  return panels(m) * groups_padded(n, group) * 16;
}

extern "C" int qigen_panels_from_codes(const uint8_t* codes, const float* scales,
                                       const float* zeros, int64_t n, int64_t m, int bits,
                                       int64_t group, uint32_t* qw, float* qsz, void* stream) {
  int st = check_config(n, m, bits, group);
  if (st) return st;
  QIGEN_CHECK_ARG(codes && qw, QIGEN_ERR_ARG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t lanes = panels(m) * supersteps(n) * 32;
  panels_from_codes_kernel<<<blocks_for(lanes, 128), 128, 0, s>>>(codes, n, m, bits, (uint4*)qw);
  QIGEN_CUDA_RET(cudaGetLastError());
  if (qsz) {
    QIGEN_CHECK_ARG(scales && zeros, QIGEN_ERR_ARG, "null scales/zeros");
    const int64_t np = qigen_panel_params(n, m, group);
    panel_params_kernel<<<blocks_for(np, 256), 256, 0, s>>>(scales, zeros, n, m, group,
                                                            (float2*)qsz);
    QIGEN_CUDA_RET(cudaGetLastError());
  }
  return QIGEN_OK;
}

extern "C" int qigen_panels_to_codes(const uint32_t* qw, int64_t n, int64_t m, int bits,
                                     uint8_t* codes, void* stream) {
  int st = check_config(n, m, bits, 0);
  if (st) return st;
  QIGEN_CHECK_ARG(codes && qw, QIGEN_ERR_ARG, "null pointer");
  const int64_t lanes = panels(m) * supersteps(n) * 32;
  panels_to_codes_kernel<<<blocks_for(lanes, 128), 128, 0, (cudaStream_t)stream>>>(
      (const uint4*)qw, n, m, bits, codes);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}

extern "C" int qigen_panels_from_rowseq(const uint32_t* words, const float* scales,
                                        const float* zeros, int64_t n, int64_t m, int bits,
                                        int64_t group, uint32_t* qw, float* qsz, void* stream) {
  int st = check_config(n, m, bits, group);
  if (st) return st;
  QIGEN_CHECK_ARG(n % unit_codes(bits) == 0, QIGEN_ERR_PACK, "rows do not fill packing units");
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* tmp = nullptr;
  QIGEN_CUDA_RET(cudaMallocAsync((void**)&tmp, (size_t)(n * m), s));
  st = qigen_unpack_rowseq(words, n, m, bits, tmp, stream);
  if (!st) st = qigen_panels_from_codes(tmp, scales, zeros, n, m, bits, group, qw, qsz, stream);
  cudaFreeAsync(tmp, s);
  return st;
}

extern "C" int qigen_input_sums(const float* x, int64_t n, int64_t group, float* out,
                                void* stream) {
  QIGEN_CHECK_ARG(x && out, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(n > 0 && (group == 0 || n % group == 0), QIGEN_ERR_CONFIG,
                  "group size %lld does not divide %lld", (long long)group, (long long)n);
  const int64_t G = group ? n / group : 1;
  input_sums_kernel<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>(x, n, group, out);
  QIGEN_CUDA_RET(cudaGetLastError());
  return QIGEN_OK;
}
