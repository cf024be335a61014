// Throughput of legacy mma.sync on sm_100a: IMMA m16n8k32 u8.s8 and HMMA m16n8k16 bf16.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void imma_loop(int* out, int iters) {
  int c[8][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 17;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void hmma_loop(float* out, int iters) {
  float c[8][4] = {};
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 17;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void imma_chain(int* out, int iters, long long* cyc) {
  int c[4] = {};
  uint32_t a0 = threadIdx.x, b0 = a0 ^ 9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3]) : "r"(a0), "r"(b0));
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* oi; float* of; long long* cy;
  cudaMalloc(&oi, 1 << 24); cudaMalloc(&of, 1 << 24); cudaMalloc(&cy, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, threads = 256, blocks = sms * 4;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); imma_loop<<<blocks, threads>>>(oi, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * blocks * (threads / 32);
    printf("IMMA m16n8k32 u8.s8: %.1f TOPS (%.2f ms)\n", ops / ms / 1e9, ms);
    cudaEventRecord(e0); hmma_loop<<<blocks, threads>>>(of, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ops = 2.0 * 16 * 8 * 16 * 8.0 * iters * blocks * (threads / 32);
    printf("HMMA m16n8k16 bf16: %.1f TFLOPS (%.2f ms)\n", ops / ms / 1e9, ms);
  }
  imma_chain<<<1, 32>>>(oi, 1000, cy);
  long long c; cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
  printf("IMMA dependent-chain latency: %.1f cycles\n", c / 1000.0);
  return 0;
}
