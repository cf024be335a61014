// Latency of the first global load after griddepcontrol.wait in a PDL chain,
// versus the same load without PDL.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_lat.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k(const float* __restrict__ x, float* out, long long* tr, int use_wait, int nld) {
  asm volatile("griddepcontrol.launch_dependents;");
  if (use_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  long long t0 = clock64();
  float acc = 0.f;
  const float* p = x + blockIdx.x * 1024 + threadIdx.x;
  for (int i = 0; i < nld; ++i) {  // dependent chain of loads
    float v;
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    acc += v;
    p += (int)(v * 0.f) + 32;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) tr[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  float *x, *out;
  long long* tr;
  const int nb = 148, chain = 64;
  cudaMalloc(&x, 148 * 1024 * 4 * 64);
  cudaMemset(x, 0, 148 * 1024 * 4 * 64);
  cudaMalloc(&out, 4);
  cudaMalloc(&tr, sizeof(long long) * nb * chain);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int mode = 0; mode < 4; ++mode) {
    const int use_pdl = mode & 1, nld = (mode & 2) ? 4 : 1;
    for (int rep = 0; rep < 2; ++rep)
      for (int i = 0; i < chain; ++i) {
        cudaLaunchConfig_t c = {};
        c.gridDim = nb; c.blockDim = 128; c.stream = s;
        cudaLaunchAttribute a;
        a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a.val.programmaticStreamSerializationAllowed = 1;
        c.attrs = &a; c.numAttrs = use_pdl;
        cudaLaunchKernelEx(&c, k, (const float*)x, out, tr + i * nb, use_pdl, nld);
      }
    cudaStreamSynchronize(s);
    std::vector<long long> h(nb * chain);
    cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    printf("pdl=%d loads=%d: cycles median %lld p10 %lld p90 %lld\n", use_pdl, nld, h[h.size() / 2],
           h[h.size() / 10], h[h.size() * 9 / 10]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
