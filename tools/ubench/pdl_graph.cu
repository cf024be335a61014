// Per-kernel period of a chain of small kernels in a CUDA graph (stream capture),
// with and without programmatic dependent launch, and with an early trigger.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_graph.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(float* buf, int early, int smem_kb) {
  extern __shared__ float sm[];
  if (early) asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float v = buf[blockIdx.x * blockDim.x + threadIdx.x];
  if (smem_kb) sm[threadIdx.x] = v;
  __syncthreads();
  if (smem_kb) v += sm[(threadIdx.x + 1) % blockDim.x];
  buf[blockIdx.x * blockDim.x + threadIdx.x] = v + 1.f;
}

int main() {
  float* buf;
  cudaMalloc(&buf, 4 << 20);
  cudaMemset(buf, 0, 4 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int N = 200;
  for (int mode = 0; mode < 6; ++mode) {
    const int pdl = mode % 3 != 0, early = mode % 3 == 2, smem = mode >= 3 ? 64 : 0;
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t c = {};
      c.gridDim = 148; c.blockDim = 256; c.stream = s; c.dynamicSmemBytes = smem * 1024;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
      a.val.programmaticStreamSerializationAllowed = 1;
      c.attrs = &a; c.numAttrs = pdl;
      cudaLaunchKernelEx(&c, k, buf, early, smem);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d early=%d smem=%dKB: %.2f us per kernel\n", pdl, early, smem, ms * 1e3 / (10 * N));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
