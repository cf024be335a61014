// PDL in CUDA graphs: chains that alternate two kernels, with / without
// thread-block clusters and with an early trigger, timed per kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_graph2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(float* buf, int early) {
  extern __shared__ float sm[];
  if (early) asm volatile("griddepcontrol.launch_dependents;");
  // ~2 us of independent work before the wait (weight prefetch stand-in)
  float acc = 0.f;
  for (int i = 0; i < 400; ++i) acc = acc * 0.999f + (float)i;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int idx = (blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
  sm[threadIdx.x] = buf[idx] + acc * 1e-30f;
  __syncthreads();
  buf[idx] = sm[(threadIdx.x + V) % blockDim.x] + 1.f;
  if (!early) asm volatile("griddepcontrol.launch_dependents;");
}

int main() {
  float* buf;
  cudaMalloc(&buf, 16 << 20);
  cudaMemset(buf, 0, 16 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int N = 100;
  for (int mode = 0; mode < 16; ++mode) {
    const int pdl = mode & 1, early = (mode >> 1) & 1, cl = (mode >> 2);  // cl: 0 none, 1 = 2, 2 = 7, 3 = alternate 9 / 6
    const int csz0 = cl == 0 ? 1 : cl == 1 ? 2 : cl == 2 ? 7 : 9;
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      const int csz = (cl == 3 && (i & 1)) ? 6 : csz0;
      cudaLaunchConfig_t c = {};
      c.gridDim = dim3(32, csz == 1 ? 6 : csz, 1);
      c.blockDim = 256; c.stream = s;
      c.dynamicSmemBytes = (i & 1 ? 64 : 96) * 1024;
      cudaLaunchAttribute a[2];
      int na = 0;
      if (pdl) {
        a[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      if (csz > 1) {
        a[na].id = cudaLaunchAttributeClusterDimension;
        a[na].val.clusterDim.x = 1; a[na].val.clusterDim.y = csz; a[na].val.clusterDim.z = 1;
        ++na;
      }
      c.attrs = a; c.numAttrs = na;
      if (i & 1) cudaLaunchKernelEx(&c, k<1>, buf, early);
      else cudaLaunchKernelEx(&c, k<2>, buf, early);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("inst fail %d\n", mode); continue; }
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("pdl=%d early=%d cluster=%d%s: %.2f us per kernel\n", pdl, early, csz0, cl == 3 ? "/6 alternating" : "", ms * 1e3 / (10 * N));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
