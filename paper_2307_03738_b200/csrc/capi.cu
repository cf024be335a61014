// C-ABI plumbing: error reporting, version, and the owning weight handle.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace qigen {
static thread_local char g_err[512] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}
}  // namespace qigen

using namespace qigen;

extern "C" int qigen_version(void) { return 100; }
extern "C" const char* qigen_last_error(void) { return g_err; }

struct qigen_weights {
  int64_t n, m, group;
  int bits;
  uint32_t* qw;
  float* qsz;
};

extern "C" int qigen_weights_create(const uint32_t* words, int layout, int64_t n, int64_t m,
                                    int bits, int64_t group, int64_t m_b, int64_t t_b,
                                    const int32_t* blk_rc, int64_t nblk, const float* scales,
                                    const float* zeros, void* stream, qigen_weights** out) {
  QIGEN_CHECK_ARG(out && words && scales && zeros, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(layout == QIGEN_LAYOUT_ROW_SEQUENTIAL || layout == QIGEN_LAYOUT_ZCURVE,
                  QIGEN_ERR_ARG, "unknown layout %d", layout);
  // config.py:54-55,73-74,108-113 (ConfigError) before any allocation
  QIGEN_CHECK_ARG(bits == 2 || bits == 3 || bits == 4, QIGEN_ERR_CONFIG,
                  "bits must be one of (2, 3, 4), got %d", bits);
  QIGEN_CHECK_ARG(n > 0 && m > 0, QIGEN_ERR_CONFIG, "matrix must be non-empty");
  QIGEN_CHECK_ARG(group >= 0 && (group == 0 || n % group == 0), QIGEN_ERR_CONFIG,
                  "group size %lld does not divide row count %lld", (long long)group,
                  (long long)n);
  QIGEN_CHECK_ARG(n % unit_codes(bits) == 0, QIGEN_ERR_CONFIG,
                  "row count %lld is not a multiple of %d for %d-bit packing", (long long)n,
                  unit_codes(bits), bits);
  QIGEN_CHECK_ARG(layout != QIGEN_LAYOUT_ZCURVE || (blk_rc && nblk > 0 && m_b > 0 && t_b > 0),
                  QIGEN_ERR_PACK, "ZCURVE words need the block table and the plan's (m_b, t_b)");
  cudaStream_t s = (cudaStream_t)stream;
  qigen_weights* w = (qigen_weights*)calloc(1, sizeof(qigen_weights));
  QIGEN_CHECK_ARG(w, QIGEN_ERR_ARG, "out of host memory");
  w->n = n; w->m = m; w->bits = bits; w->group = group;
  int st = QIGEN_OK;
  const uint32_t* rowseq = words;
  uint32_t* tmp = nullptr;
  if (cudaMalloc((void**)&w->qw, qigen_panel_words(n, m, bits) * 4) != cudaSuccess ||
      cudaMalloc((void**)&w->qsz, qigen_panel_params(n, m, group) * 8) != cudaSuccess) {
    set_error("cudaMalloc failed for weight handle");
    st = QIGEN_ERR_CUDA;
  }
  if (!st && layout == QIGEN_LAYOUT_ZCURVE) {
    const int64_t nw = n * m * bits / 32;
    if (cudaMalloc((void**)&tmp, nw * 4) != cudaSuccess) {
      set_error("cudaMalloc failed");
      st = QIGEN_ERR_CUDA;
    } else {
      st = qigen_permute_zcurve(words, tmp, n, m, bits, m_b, t_b, blk_rc, nblk, 0, stream);
      rowseq = tmp;
    }
  }
  if (!st) st = qigen_panels_from_rowseq(rowseq, scales, zeros, n, m, bits, group, w->qw, w->qsz, stream);
  if (!st && cudaStreamSynchronize(s) != cudaSuccess) {
    set_error("stream sync failed while building weights");
    st = QIGEN_ERR_CUDA;
  }
  if (tmp) cudaFree(tmp);
  if (st) {
    qigen_weights_destroy(w);
    return st;
  }
  *out = w;
  return QIGEN_OK;
}

extern "C" int qigen_weights_destroy(qigen_weights* w) {
  if (!w) return QIGEN_OK;
  if (w->qw) cudaFree(w->qw);
  if (w->qsz) cudaFree(w->qsz);
  free(w);
  return QIGEN_OK;
}

extern "C" int qigen_weights_gemv(const qigen_weights* w, const void* x, int x_dtype,
                                  int64_t tokens, float* y, int accumulate, void* stream) {
  QIGEN_CHECK_ARG(w, QIGEN_ERR_ARG, "null handle");
  return qigen_gemv(w->qw, w->qsz, w->n, w->m, w->bits, w->group, x, x_dtype, tokens, w->n, y,
                    w->m, accumulate, 0, stream);
}

extern "C" int qigen_weights_gemv_host(const qigen_weights* w, const float* x_host,
                                       int64_t tokens, float* y_host, void* stream) {
  QIGEN_CHECK_ARG(w && x_host && y_host, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(tokens >= 1, QIGEN_ERR_ARG, "tokens must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  // device staging is stream-ordered scratch (not owned by the handle), so one
  // handle may serve several host threads / streams at once (read-only weights)
  const size_t xb = (size_t)tokens * w->n * 4, yb = (size_t)tokens * w->m * 4;
  unsigned char* io = nullptr;
  int st = scratch_alloc(s, (xb + 255) / 256 * 256 + yb, &io);
  if (st) return st;
  float* x_dev = (float*)io;
  float* y_dev = (float*)(io + (xb + 255) / 256 * 256);
  cudaError_t e = cudaMemcpyAsync(x_dev, x_host, xb, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    st = qigen_gemv(w->qw, w->qsz, w->n, w->m, w->bits, w->group, x_dev, QIGEN_F32, tokens,
                    w->n, y_dev, w->m, 0, 0, stream);
    if (!st) e = cudaMemcpyAsync(y_host, y_dev, yb, cudaMemcpyDeviceToHost, s);
  }
  cudaFreeAsync(io, s);
  if (st) return st;
  QIGEN_CUDA_RET(e);
  QIGEN_CUDA_RET(cudaStreamSynchronize(s));
  return QIGEN_OK;
}
