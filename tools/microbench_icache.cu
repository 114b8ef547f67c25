// Cost of executing straight-line code once per launch (cold instruction
// cache) versus a second pass over the same code (warm), with and without a
// concurrent HBM stream (another kernel on a second stream).  One CTA per SM,
// 16 warps, each running ~2000 independent integer instructions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbicache tools/microbench_icache.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define R8(X) X X X X X X X X
#define BODY                                                    \
  a = a * 1664525u + 1013904223u; b = (b ^ a) * 2246822519u;    \
  c = c + (a >> 7) + (b << 3); d = (d ^ c) + 0x9e3779b9u;

__device__ __noinline__ uint32_t straight(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  R8(R8(R8(BODY)))  // 512 x BODY ~ 2500 instructions
  return a ^ b ^ c ^ d;
}

__global__ void __launch_bounds__(512, 1) probe(unsigned long long* out, int passes) {
  uint32_t x = threadIdx.x;
  unsigned long long t[3];
  for (int p = 0; p < passes; ++p) {
    const long long t0 = clock64();
    x = straight(x, x + 1, x + 2, x + 3);
    t[p] = clock64() - t0;
  }
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = t[0];
    out[blockIdx.x * 4 + 1] = passes > 1 ? t[1] : 0;
  }
  if (x == 0x12345) out[2047] = x;
}

__global__ void stream_kernel(const uint4* src, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x1234567u) sink[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, 2048 * 8);
  const size_t big = 2ull << 30;
  uint4* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  uint32_t* sink;
  cudaMalloc(&sink, 64);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  unsigned long long h[1024];
  for (int load = 0; load < 2; ++load) {
    for (int rep = 0; rep < 3; ++rep) {
      if (load) stream_kernel<<<sms * 4, 256, 0, s2>>>(buf, big / 16, sink);
      probe<<<sms, 512, 0, s1>>>(out, 2);  // grid of sms CTAs (may share SMs with the stream kernel)
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, sms * 4 * 8, cudaMemcpyDeviceToHost);
      double a0 = 0, a1 = 0;
      for (int i = 0; i < sms; ++i) {
        a0 += h[i * 4];
        a1 += h[i * 4 + 1];
      }
      printf("  launch %d (stream %s): first pass %.0f, second pass %.0f cycles\n", rep, load ? "on" : "off", a0 / sms,
             a1 / sms);
    }
    double c0 = 0, c1 = 0;
    for (int i = 0; i < sms; ++i) {
      c0 += h[i * 4];
      c1 += h[i * 4 + 1];
    }
    printf("HBM stream %s: first pass %.0f cycles, second pass %.0f cycles (~2500 instructions)  %s\n", load ? "on " : "off",
           c0 / sms, c1 / sms, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
