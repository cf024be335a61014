// Tensor-parallel one-shot all-reduce: buffers (CUDA IPC), the per-step epoch
// and the reduce kernel.  Protocol: tp.cuh.  The push half lives in the GEMV
// epilogue (gemv.cu, qigen_gemv_tp_push).
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tp.cuh"

namespace qigen {

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void tp_step_begin_kernel(unsigned* epoch) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  *epoch += 1u;
}

// h[b, k] += sum_r inbox[slot][r][b][k], r = 0..world-1 in order, once every
// source's columns of this use have arrived.
__global__ void __launch_bounds__(256) tp_reduce_kernel(char* base, int world, int slot, int layer,
                                                        int layers, int bmax, int64_t d, float* h,
                                                        int B) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // this rank's own push is complete
  unsigned* flags = (unsigned*)base;
  if (threadIdx.x == 0) {
    const unsigned epoch = *(volatile unsigned*)(base + 64);
    const unsigned target = ((epoch - 1u) * (unsigned)layers + (unsigned)layer + 1u) * (unsigned)d;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // (after a timeout every later reduce of the step fails fast instead of
    // waiting 4 s again)
    bool good = *(volatile unsigned*)(base + 68) == 0u;
    for (int q = 0; q < world && good; ++q) {
      while ((int)(ld_acquire_sys(&flags[slot * 8 + q]) - target) < 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 4000000000ull) {  // 4 s: a peer never arrived; flag it, never hang
          atomicExch((unsigned*)(base + 68), 1u);
          good = false;
          break;
        }
        __nanosleep(64);
      }
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  const float* inbox = (const float*)(base + kTpHeader) + (size_t)slot * world * bmax * d;
  const int64_t n = (int64_t)B * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / d, k = i % d;
    float v = h[i];
    for (int q = 0; q < world; ++q) v += __ldcg(inbox + ((size_t)q * bmax + b) * d + k);
    h[i] = v;
  }
}

}  // namespace qigen

using namespace qigen;

extern "C" int64_t qigen_tp_buffer_size(int world, int64_t d, int64_t max_tokens) {
  return kTpHeader + 2ll * world * max_tokens * d * 4;
}

extern "C" int qigen_tp_alloc(int64_t bytes, void** ptr, void* ipc_handle_out) {
  QIGEN_CHECK_ARG(ptr && bytes > 0, QIGEN_ERR_ARG, "bad arguments");
  QIGEN_CUDA_RET(cudaMalloc(ptr, (size_t)bytes));
  QIGEN_CUDA_RET(cudaMemset(*ptr, 0, (size_t)bytes));
  QIGEN_CUDA_RET(cudaDeviceSynchronize());
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    QIGEN_CUDA_RET(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(ipc_handle_out, &h, sizeof h);
  }
  return QIGEN_OK;
}

extern "C" int qigen_tp_free(void* ptr) {
  if (ptr) QIGEN_CUDA_RET(cudaFree(ptr));
  return QIGEN_OK;
}

extern "C" int qigen_tp_open_peer(const void* ipc_handle, void** ptr) {
  QIGEN_CHECK_ARG(ipc_handle && ptr, QIGEN_ERR_ARG, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof h);
  QIGEN_CUDA_RET(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return QIGEN_OK;
}

extern "C" int qigen_tp_close_peer(void* ptr) {
  if (ptr) QIGEN_CUDA_RET(cudaIpcCloseMemHandle(ptr));
  return QIGEN_OK;
}

extern "C" int qigen_tp_create(int rank, int world, int64_t d, int64_t max_tokens, int layers,
                               void* const* bases, qigen_tp_comm** out) {
  QIGEN_CHECK_ARG(out && bases, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(world >= 1 && world <= kTpMaxWorld && rank >= 0 && rank < world, QIGEN_ERR_ARG,
                  "rank %d / world %d (world <= %d)", rank, world, kTpMaxWorld);
  QIGEN_CHECK_ARG(d > 0 && max_tokens >= 1 && layers >= 1, QIGEN_ERR_ARG, "bad shape");
  for (int q = 0; q < world; ++q) QIGEN_CHECK_ARG(bases[q], QIGEN_ERR_ARG, "null buffer of rank %d", q);
  auto* c = (qigen_tp_comm*)calloc(1, sizeof(qigen_tp_comm));
  QIGEN_CHECK_ARG(c, QIGEN_ERR_ARG, "out of host memory");
  for (int q = 0; q < world; ++q) c->base[q] = bases[q];
  c->rank = rank;
  c->world = world;
  c->d = d;
  c->bmax = (int)max_tokens;
  c->layers = layers;
  *out = c;
  return QIGEN_OK;
}

extern "C" int qigen_tp_destroy(qigen_tp_comm* c) {
  free(c);
  return QIGEN_OK;
}

extern "C" int qigen_tp_step_begin(const qigen_tp_comm* c, void* stream) {
  QIGEN_CHECK_ARG(c, QIGEN_ERR_ARG, "null comm");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1, 1, 1);
  cfg.blockDim = dim3(1, 1, 1);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, tp_step_begin_kernel,
                                    (unsigned*)((char*)c->base[c->rank] + 64)));
  return QIGEN_OK;
}

extern "C" int qigen_tp_reduce(const qigen_tp_comm* c, int slot, int layer, float* h,
                               int64_t tokens, void* stream) {
  QIGEN_CHECK_ARG(c && h, QIGEN_ERR_ARG, "null pointer");
  QIGEN_CHECK_ARG(slot == 0 || slot == 1, QIGEN_ERR_ARG, "slot must be 0 or 1");
  QIGEN_CHECK_ARG(layer >= 0 && layer < c->layers, QIGEN_ERR_ARG, "layer out of range");
  QIGEN_CHECK_ARG(tokens >= 1 && tokens <= c->bmax, QIGEN_ERR_ARG, "tokens out of range");
  const int64_t n = tokens * c->d;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::min<int64_t>((n + 1023) / 1024, 148), 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  QIGEN_CUDA_RET(cudaLaunchKernelEx(&cfg, tp_reduce_kernel, (char*)c->base[c->rank], c->world,
                                    slot, layer, c->layers, c->bmax, c->d, h, (int)tokens));
  return QIGEN_OK;
}

// Nonzero when a reduce on this rank gave up waiting for a peer (then reset).
extern "C" int qigen_tp_error(const qigen_tp_comm* c, int* out) {
  QIGEN_CHECK_ARG(c && out, QIGEN_ERR_ARG, "null pointer");
  unsigned v = 0;
  char* p = (char*)c->base[c->rank] + 68;
  QIGEN_CUDA_RET(cudaMemcpy(&v, p, 4, cudaMemcpyDeviceToHost));
  if (v) QIGEN_CUDA_RET(cudaMemset(p, 0, 4));
  *out = (int)v;
  return QIGEN_OK;
}
