// Grid-barrier latency on one CTA per SM (the decode stack's barrier), variants:
//   0: one counter, red.release.gpu arrive + ld.acquire.gpu poll by thread 0
//   1: NC counters on separate 128 B lines (arrive on counter cta % NC; the poller's
//      lanes read all of them)
//   2: flag array, no atomics: CTA c stores the epoch to flags[c] (st.release.gpu);
//      warps 0..4 poll 32 flags each (ld.acquire.gpu), then __syncthreads
//   3: like 2 with ld.relaxed + one fence.acq_rel.gpu after the poll
// each with global stores before the arrive and ld.cg loads after the pass.
//   nvcc -arch=sm_100a -O3 -o gridbar gridbar.cu && ./gridbar
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NC = 16;

__global__ void __launch_bounds__(512, 1) bar_kernel(unsigned* bar, float* buf, int iters, int variant,
                                                     int* err) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x, cta = blockIdx.x;
  unsigned nbar = 0;
  for (int it = 0; it < iters; ++it) {
    buf[(size_t)cta * 512 + tid] = (float)it;  // stores before the arrive
    __syncthreads();
    ++nbar;
    if (variant == 0) {
      if (tid == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned target = nbar * G;
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
      }
    } else if (variant == 1) {
      if (warp == 0) {
        if (lane == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + (cta % NC) * 32) : "memory");
        const unsigned target = nbar * G;
        unsigned sum;
        do {
          unsigned v = 0;
          if (lane < NC)
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + lane * 32) : "memory");
          sum = __reduce_add_sync(0xffffffffu, v);
        } while (sum < target);
      }
    } else {
      if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + cta), "r"(nbar) : "memory");
      if (warp < (G + 31) / 32) {
        const unsigned i = warp * 32 + lane;
        bool ok;
        do {
          unsigned v = nbar;
          if (i < G) {
            if (variant == 2)
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + i) : "memory");
            else
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + i) : "memory");
          }
          ok = __all_sync(0xffffffffu, (int)(v - nbar) >= 0);
        } while (!ok);
        if (variant == 3) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
    // loads after the pass: the neighbour's stores of this iteration must be visible
    // (it may already have stored the next iteration's value)
    const float v = __ldcg(buf + (size_t)((cta + 1) % G) * 512 + tid);
    if (v < (float)it) atomicAdd(err, 1);
    __syncthreads();
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  float* buf;
  int* err;
  cudaMalloc(&bar, 4096);
  cudaMalloc(&buf, (size_t)sms * 512 * 4);
  cudaMalloc(&err, 4);
  const int iters = 2000;
  for (int variant = 0; variant < 4; ++variant) {
    cudaMemset(bar, 0, 4096);
    cudaMemset(err, 0, 4);
    void* args[] = {&bar, &buf, (void*)&iters, &variant, &err};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel, dim3(sms), dim3(512), args, 0, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    int herr = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
    printf("variant %d: %s, %.0f ns per iteration (store + barrier + load), %d stale loads (%d SMs)\n",
           variant, cudaGetErrorString(e), ms * 1e6 / iters, herr, sms);
  }
  return 0;
}
