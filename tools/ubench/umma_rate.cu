// tcgen05.mma issue / completion cost on sm_100a for the small-N shapes of the
// quantized GEMM: M = 128, N = NT, K = 16 (kind::f16), A from TMEM ("ts") or
// shared memory ("ss"), one tcgen05.commit every C instructions.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(saddr(b)), "r"(ph) : "memory");
}

template <int NT, bool TS, int NACC>
__global__ void __launch_bounds__(128, 1) umma(int iters, int C, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    long long t0 = clock64(), tiss = 0;
    for (int i = 0; i < iters; ++i) {
      const uint32_t bofs = saddr(sm) + (uint32_t)((i & 7) * 2 * 128);
      if (TS) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                     ::"r"(tm + (uint32_t)((i % NACC) * (256 / NACC))), "r"(tm + 256 + (uint32_t)(i & 31) * 8), "l"(desc(bofs)), "r"(idesc), "r"(i));
      } else {
        const uint32_t aofs = saddr(sm) + 32768 + (uint32_t)((i & 7) * 2 * 128);
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     ::"r"(tm + (uint32_t)((i % NACC) * (256 / NACC))), "l"(desc(aofs)), "l"(desc(bofs)), "r"(idesc), "r"(i));
      }
      if ((i + 1) % C == 0) {
        const int j = (i + 1) / C - 1;  // commit group index
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar[j & 1])) : "memory");
        if (j >= 1) wait(&bar[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
      }
    }
    tiss = clock64() - t0;
    const int groups = iters / C;
    if (groups >= 1) wait(&bar[(groups - 1) & 1], (uint32_t)(((groups - 1) >> 1) & 1));
    long long tall = clock64() - t0;
    if (blockIdx.x == 0) { out[0] = tiss; out[1] = tall; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int NT, bool TS, int NACC = 1>
void run(int C, long long* d) {
  auto k = umma<NT, TS, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148, 128, 65536>>>(iters, C, d);
  cudaEventRecord(e0);
  k<<<148, 128, 65536>>>(iters, C, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * NT * 16 * iters * 148;
  printf("%s NACC=%d NT=%3d commit/%2d: issue %6.1f cyc/mma, total %6.1f cyc/mma, %7.1f TFLOP/s  err=%s\n",
         TS ? "ts" : "ss", NACC, NT, C, (double)h[0] / iters, (double)h[1] / iters, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}


// Warp-converged variant: warp 0 runs the loop, one elected lane issues; 16 MMAs
// per commit, unrolled; ACC = 0 disables accumulation (no D dependency).
template <int NT, int ACC>
__global__ void __launch_bounds__(128, 1) umma2(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t slot;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (threadIdx.x < 32) {
    const long long t0 = clock64();
    const int groups = iters / 16;
    for (int j = 0; j < groups; ++j) {
      uint32_t e;
      asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t bofs = saddr(sm) + (uint32_t)((q & 7) * 2 * 128);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                       ::"r"(tm), "r"(tm + 256 + (uint32_t)(q * 8)), "l"(desc(bofs)), "r"(idesc), "r"(ACC ? (j | q) : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar[j & 1])) : "memory");
      }
      __syncwarp();
      if (j >= 1) wait(&bar[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
    }
    wait(&bar[(groups - 1) & 1], (uint32_t)(((groups - 1) >> 1) & 1));
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = clock64() - t0; out[1] = out[0]; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
  }
}

template <int NT, int ACC>
void run2(long long* d) {
  auto k = umma2<NT, ACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148, 128, 65536>>>(iters, d);
  cudaEventRecord(e0);
  k<<<148, 128, 65536>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double flops = 2.0 * 128 * NT * 16 * iters * 148;
  printf("warp-elect ACC=%d NT=%3d: %6.1f cyc/mma, %7.1f TFLOP/s  err=%s\n", ACC, NT,
         (double)h[0] / iters, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  long long* d; cudaMalloc(&d, 64);
  run2<16, 1>(d); run2<16, 0>(d); run2<64, 1>(d); run2<256, 1>(d); run2<256, 0>(d);
  for (int C : {16}) {
    run<16, true>(C, d); run<16, true, 4>(C, d); run<16, false, 4>(C, d);
    run<64, true>(C, d); run<64, true, 4>(C, d);
    run<256, true>(C, d); run<256, false>(C, d);
  }
  return 0;
}
