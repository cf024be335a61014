/* C port of the reference's generated qGEMV kernel — TEST/BASELINE ONLY.
 *
 * Restates the arithmetic of the kernels that qigen's kernelgen.py emits and
 * numba compiles (reference: /root/reference/pkg/src/qigen/kernelgen.py), over
 * the same execution layout and with the same calling convention
 * (kernelgen.py:399-401: words, scales, zeros, x, xsums, y, blk_off, blk_rb,
 * blk_cb, nblk, cb_lo, cb_hi, cb_count) plus the descriptor fields the
 * generated source bakes in as constants (bits, group, m_b, t_b, stripe).
 *
 *  grouped (kernelgen.py:264-313, flush :227-240), per output column:
 *      ya = y;  for each group:  ia = 0;  for each row r:  ia = x[r]*f32(code) + ia
 *               tv = z*(-xsum_g) + ia;  ya = s*tv + ya
 *  full column (kernelgen.py:243-261 raw accumulation with the x index fixed
 *      per SURVEY F4, then the epilogue :316-330):
 *      acc = y; acc = x[r]*f32(code) + acc ...;  y = s*(z*(-xhat) + y) + 0
 *
 * Multiply and add are rounded separately (numba emits fmul/fadd without
 * contraction), so this file is compiled with -ffp-contract=off;
 * columns are independent, so vectorising across columns keeps every column's
 * operation sequence — and therefore its bits — identical to the reference.
 * Threads own disjoint contiguous column-block ranges.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SW 24 /* stripe width t_u * lanes = 3 * 8 for the default plan */

static inline void word_group_rows(const uint32_t *wp, int t_b, int bits, int u0, int u1,
                                   const float *xr, float *acc) {
  const uint32_t mask = (1u << bits) - 1u;
  for (int u = u0; u < u1; ++u) {
    const float xv = xr[u];
    if (bits != 3) {
      const int sh = u * bits;
      for (int c = 0; c < SW; ++c) {
        const float cf = (float)((wp[c] >> sh) & mask);
        acc[c] = xv * cf + acc[c];
      }
    } else {
      const int bit = 3 * u, k = bit >> 5, off = bit & 31;
      const uint32_t *w0 = wp + (size_t)k * t_b;
      if (off <= 29) {
        for (int c = 0; c < SW; ++c) {
          const float cf = (float)((w0[c] >> off) & mask);
          acc[c] = xv * cf + acc[c];
        }
      } else { /* straddle: kernelgen.py:120-124 */
        const int lo = 32 - off;
        const uint32_t hm = (1u << (3 - lo)) - 1u;
        const uint32_t *w1 = w0 + t_b;
        for (int c = 0; c < SW; ++c) {
          const uint32_t v = (w0[c] >> off) | ((w1[c] & hm) << lo);
          const float cf = (float)(v & mask);
          acc[c] = xv * cf + acc[c];
        }
      }
    }
  }
}

static void run_blocks(const uint32_t *words, const float *scales, const float *zeros,
                       const float *x, const float *xsums, float *y, int bits, int group,
                       int m_b, int t_b, const int64_t *blk_off, const int64_t *blk_rb,
                       const int64_t *blk_cb, int64_t nblk, int64_t cb_lo, int64_t cb_hi,
                       int64_t cb_count) {
  const int unit = bits == 3 ? 32 : 32 / bits;
  const int kw = bits == 3 ? 3 : 1;
  const int64_t mpad = cb_count * t_b;
  const int stripes = t_b / SW;
  for (int64_t bi = 0; bi < nblk; ++bi) {
    const int64_t cb = blk_cb[bi];
    if (cb < cb_lo || cb >= cb_hi) continue;
    const int64_t rb = blk_rb[bi];
    const uint32_t *wb = words + blk_off[bi];
    const float *xb = x + rb * m_b;
    for (int st = 0; st < stripes; ++st) {
      const int coff = st * SW;
      float *yv = y + cb * t_b + coff;
      if (group == 0) {
        float acc[SW];
        memcpy(acc, yv, sizeof acc);
        for (int wg = 0; wg < m_b / unit; ++wg)
          word_group_rows(wb + (size_t)wg * kw * t_b + coff, t_b, bits, 0, unit,
                          xb + wg * unit, acc);
        memcpy(yv, acc, sizeof acc);
      } else {
        float ya[SW], ia[SW];
        memcpy(ya, yv, sizeof ya);
        const int gpb = m_b / group;
        for (int gs = 0; gs < gpb; ++gs) {
          for (int c = 0; c < SW; ++c) ia[c] = 0.0f;
          /* rows [gs*group, (gs+1)*group) walked word-group by word-group */
          int r = gs * group;
          const int r_end = r + group;
          while (r < r_end) {
            const int wg = r / unit, u0 = r % unit;
            int u1 = unit;
            if (wg * unit + u1 > r_end) u1 = r_end - wg * unit;
            word_group_rows(wb + (size_t)wg * kw * t_b + coff, t_b, bits, u0, u1,
                            xb + wg * unit, ia);
            r = wg * unit + u1;
          }
          const int64_t gi = rb * gpb + gs;
          const float nxg = -xsums[gi];
          const float *sv = scales + gi * mpad + cb * t_b + coff;
          const float *zv = zeros + gi * mpad + cb * t_b + coff;
          for (int c = 0; c < SW; ++c) {
            const float tv = zv[c] * nxg + ia[c];
            ya[c] = sv[c] * tv + ya[c];
          }
        }
        memcpy(yv, ya, sizeof ya);
      }
    }
  }
  if (group == 0) { /* FC epilogue, kernelgen.py:316-330 */
    const float nxh = -xsums[0];
    for (int64_t c = cb_lo * t_b; c < cb_hi * t_b; ++c) {
      const float tv = zeros[c] * nxh + y[c];
      y[c] = scales[c] * tv + 0.0f;
    }
  }
}

void qgemv_port_blocks(const uint32_t *words, const float *scales, const float *zeros,
                       const float *x, const float *xsums, float *y, int bits, int group,
                       int m_b, int t_b, int stripe, const int64_t *blk_off,
                       const int64_t *blk_rb, const int64_t *blk_cb, int64_t nblk,
                       int64_t cb_lo, int64_t cb_hi, int64_t cb_count) {
  (void)stripe;
  run_blocks(words, scales, zeros, x, xsums, y, bits, group, m_b, t_b, blk_off, blk_rb,
             blk_cb, nblk, cb_lo, cb_hi, cb_count);
}

/* Reference runtime threading: thread i owns column blocks
 * [CB*i/T, CB*(i+1)/T). */
void qgemv_port_threads(const uint32_t *words, const float *scales, const float *zeros,
                        const float *x, const float *xsums, float *y, int bits, int group,
                        int m_b, int t_b, int stripe, const int64_t *blk_off,
                        const int64_t *blk_rb, const int64_t *blk_cb, int64_t nblk,
                        int64_t cb_count, int threads) {
  (void)stripe;
  if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static, 1)
  for (int i = 0; i < threads; ++i) {
    const int64_t lo = cb_count * i / threads, hi = cb_count * (i + 1) / threads;
    run_blocks(words, scales, zeros, x, xsums, y, bits, group, m_b, t_b, blk_off, blk_rb,
               blk_cb, nblk, lo, hi, cb_count);
  }
}

int qgemv_port_max_threads(void) {
#ifdef _OPENMP
  return omp_get_num_procs();
#else
  return 1;
#endif
}
