// Shared helpers for the qigen-b200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/qigen_b200.h"

namespace qigen {

// Set by every C-ABI entry point that fails; read with qigen_last_error().
void set_error(const char* fmt, ...);

// Stream-ordered scratch (gemv.cu): released with cudaFreeAsync on the same
// stream behind the kernels that use it; safe for concurrent streams.
int scratch_alloc(cudaStream_t stream, size_t bytes, unsigned char** out);

// Lazy per-device setup (kernel attributes) that is safe when several host
// threads make their first call at once: fn runs exactly once per device, and
// every caller sees its status.
constexpr int kMaxDevices = 64;
struct OncePerDevice {
  std::once_flag flag[kMaxDevices];
  int status[kMaxDevices] = {};
  template <class F>
  int run(F&& fn) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
      set_error("no current CUDA device");
      return QIGEN_ERR_CUDA;
    }
    std::call_once(flag[dev], [&] { status[dev] = fn(); });
    return status[dev];
  }
};

#define QIGEN_CHECK_ARG(cond, code, ...)   \
  do {                                     \
    if (!(cond)) {                         \
      ::qigen::set_error(__VA_ARGS__);     \
      return (code);                       \
    }                                      \
  } while (0)

#define QIGEN_CUDA_RET(expr)                                                 \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::qigen::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), \
                         __FILE__, __LINE__, cudaGetErrorString(_e));        \
      return QIGEN_ERR_CUDA;                                                 \
    }                                                                        \
  } while (0)

__host__ __device__ inline int unit_codes(int bits) { return bits == 3 ? 32 : 32 / bits; }
__host__ __device__ inline int unit_words(int bits) { return bits == 3 ? 3 : 1; }

// GPU ("panel") layout geometry, see DESIGN.md §3.
constexpr int kPanel = 16;       // output columns per panel (mma M)
constexpr int kStep = 32;        // K per mma step (m16n8k32)
constexpr int kSuper = 256;      // K per superstep = 8 steps; a lane loads `bits` uint4
__host__ __device__ inline int64_t panels(int64_t m) { return (m + kPanel - 1) / kPanel; }
__host__ __device__ inline int64_t supersteps(int64_t n) { return (n + kSuper - 1) / kSuper; }
// groups per column in the padded layout (FC: one group spanning the padded K)
__host__ __device__ inline int64_t groups_padded(int64_t n, int64_t group) {
  if (group == 0) return 1;
  return (supersteps(n) * kSuper + group - 1) / group;
}
__host__ __device__ inline int64_t tile_words(int64_t n, int64_t m, int bits) {
  return panels(m) * supersteps(n) * (int64_t)bits * 32 * 4;  // uint32 words
}

}  // namespace qigen
