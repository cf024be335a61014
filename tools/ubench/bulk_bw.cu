// HBM streaming bandwidth through cp.async.bulk (global -> shared, mbarrier
// complete_tx) on sm_100a as a function of stage size and ring depth: one
// producer warp (elected lane issues), one consumer warp (waits full, frees).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw bulk_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(saddr(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void spin(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(saddr(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ bool elect() {
  uint32_t e;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(e));
  return e;
}

// NP producer "streams" (panels), each with its own ring of D stages of B bytes.
template <int SPIN>
__global__ void __launch_bounds__(64, 1) stream(const char* src, int64_t per_cta, int B, int D, int NP,
                                                unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)NP * D * B);
  uint64_t* empty = full + NP * D;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NP * D; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  const int nst = (int)(per_cta / ((int64_t)B * NP));  // stages per stream
  if (warp == 0) {
    for (int s = 0; s < nst; ++s)
      for (int p = 0; p < NP; ++p) {
        const int slot = p * D + s % D;
        if (s >= D) { if (SPIN) spin(&empty[slot], ((s / D) - 1) & 1); else wait(&empty[slot], ((s / D) - 1) & 1); }
        if (elect()) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[slot])), "r"(B) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(saddr(sm + (size_t)slot * B)), "l"(base + ((int64_t)s * NP + p) * B), "r"(B), "r"(saddr(&full[slot])) : "memory");
        }
        __syncwarp();
      }
  } else {
    unsigned acc = 0;
    for (int s = 0; s < nst; ++s)
      for (int p = 0; p < NP; ++p) {
        const int slot = p * D + s % D;
        if (SPIN) spin(&full[slot], (s / D) & 1); else wait(&full[slot], (s / D) & 1);
        acc += ((const unsigned*)(sm + (size_t)slot * B))[threadIdx.x & 31];
        __syncwarp();
        if (elect()) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[slot])) : "memory");
        __syncwarp();
      }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}


// NW independent producer/consumer warp pairs per CTA (ring of D stages of B bytes each)
template <int LANE0>
__global__ void __launch_bounds__(1024, 1) multi(const char* src, int64_t per_cta, int B, int D, int NW,
                                                 unsigned* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)NW * D * B);
  uint64_t* empty = full + NW * D;
  const int warp = threadIdx.x >> 5, pair = warp >> 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NW * D; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t per_w = per_cta / NW / B * B;
  const char* base = src + blockIdx.x * per_cta + pair * per_w;
  const int nst = (int)(per_w / B);
  if (pair >= NW) return;
  if ((warp & 1) == 0) {
    for (int s = 0; s < nst; ++s) {
      const int slot = pair * D + s % D;
      if (LANE0) {
        if ((threadIdx.x & 31) == 0) {
          if (s >= D) wait(&empty[slot], ((s / D) - 1) & 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[slot])), "r"(B) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(saddr(sm + (size_t)slot * B)), "l"(base + (int64_t)s * B), "r"(B), "r"(saddr(&full[slot])) : "memory");
        }
      } else {
      if (s >= D) wait(&empty[slot], ((s / D) - 1) & 1);
      if (elect()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[slot])), "r"(B) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(saddr(sm + (size_t)slot * B)), "l"(base + (int64_t)s * B), "r"(B), "r"(saddr(&full[slot])) : "memory");
      }
      __syncwarp();
      }
    }
  } else {
    unsigned acc = 0;
    for (int s = 0; s < nst; ++s) {
      const int slot = pair * D + s % D;
      wait(&full[slot], (s / D) & 1);
      acc += ((const unsigned*)(sm + (size_t)slot * B))[threadIdx.x & 31];
      __syncwarp();
      if (elect()) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[slot])) : "memory");
      __syncwarp();
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
}
// plain vector loads: every thread streams uint4 with U loads in flight
template <int U>
__global__ void __launch_bounds__(512) ldg(const uint4* src, int64_t n16, unsigned* sink) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (i + u * stride < n16) ? __ldg(src + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 2ll << 30;
  char* src; unsigned* sink;
  cudaMalloc(&src, total); cudaMalloc(&sink, 64);
  cudaMemset(src, 1, total);
  cudaFuncSetAttribute(stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int B, D, NP; } cfgs[] = {
      {2560, 4, 8}, {2560, 6, 8}, {2560, 10, 8}, {2048, 6, 8}, {4096, 6, 8}, {8192, 4, 4},
      {8192, 8, 2}, {16384, 6, 1}, {32768, 4, 1}, {32768, 6, 1}, {2048, 32, 1}, {2048, 64, 1}};
  cudaFuncSetAttribute(multi<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(multi<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct M { int B, D, NW; } ms_[] = {{2048, 6, 1}, {2048, 6, 4}, {2048, 6, 8}, {2048, 6, 16}, {4096, 4, 8}, {8192, 3, 8}};
  for (int l0 = 0; l0 < 2; ++l0)
  for (auto c : ms_) {
    const int64_t per_cta = (total / sms) / ((int64_t)c.B * c.NW) * ((int64_t)c.B * c.NW);
    const size_t smem = (size_t)c.NW * c.D * c.B + 2 * c.NW * c.D * 8;
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      if (l0) multi<1><<<sms, 64 * c.NW, smem>>>(src, per_cta, c.B, c.D, c.NW, sink);
      else multi<0><<<sms, 64 * c.NW, smem>>>(src, per_cta, c.B, c.D, c.NW, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("multi %s B=%6d D=%d NW=%2d: %7.1f GB/s err=%s\n", l0 ? "lane0" : "elect", c.B, c.D, c.NW, (double)(per_cta / c.NW / c.B * c.B * c.NW) * sms / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int u : {4, 8}) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      if (u == 4) ldg<4><<<sms * 4, 512>>>((const uint4*)src, total / 16, sink);
      else ldg<8><<<sms * 4, 512>>>((const uint4*)src, total / 16, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("ldg U=%d: %7.1f GB/s\n", u, (double)total / best / 1e6);
  }
  for (int spin_ = 0; spin_ < 0; ++spin_)
  for (auto c : cfgs) {
    const int64_t per_cta = (total / sms) / ((int64_t)c.B * c.NP) * ((int64_t)c.B * c.NP);
    const size_t smem = (size_t)c.NP * c.D * c.B + 2 * c.NP * c.D * 8;
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      if (spin_) stream<1><<<sms, 64, smem>>>(src, per_cta, c.B, c.D, c.NP, sink);
      else stream<0><<<sms, 64, smem>>>(src, per_cta, c.B, c.D, c.NP, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%s B=%6d D=%3d NP=%d in-flight/SM=%6zu B: %7.1f GB/s  err=%s\n", spin_ ? "test_wait" : "try_wait ", c.B, c.D, c.NP, smem,
           (double)per_cta * sms / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
