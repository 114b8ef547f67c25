// Latencies of the decode main loop's building blocks on one warp (sm_100a):
// dependent IMMA m16n8k32 chain, IMMA -> integer use, mbarrier try_wait on a
// completed phase, dependent LDS.128, shared atomicAdd.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mblat tools/microbench_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void lat(unsigned long long* out, int n, uint32_t seed) {
  __shared__ __align__(16) uint32_t sm[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t cnt[32];
  const int lane = threadIdx.x;
  for (int i = lane; i < 4096; i += 32) sm[i] = (i * 4 + 16) & 4095;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
  cnt[lane] = 0;
  __syncwarp();
  if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&bar)) : "memory");
  __syncwarp();
  int d[4] = {1, 2, 3, 4};
  long long t0, t1;
  // (a) dependent IMMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) imma(d, seed, seed + 1, seed + 2, seed + 3, seed ^ i, seed);
  t1 = clock64();
  out[0] = (t1 - t0) / n;
  // (b) IMMA then integer use of the result feeding the next IMMA's A operand
  uint32_t a = seed;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    int e[4] = {0, 0, 0, 0};
    imma(e, a, a, a, a, seed, seed);
    a = (uint32_t)e[0] >> 3;
  }
  t1 = clock64();
  out[1] = (t1 - t0) / n;
  // (c) try_wait on a completed phase (parity 0)
  uint32_t acc = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    uint32_t p;
    asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                 : "=r"(p) : "r"(saddr(&bar)) : "memory");
    acc += p;
  }
  t1 = clock64();
  out[2] = (t1 - t0) / n;
  // (d) dependent LDS.128 chain
  uint32_t idx = lane * 4;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr(sm) + (idx & 4095) * 4));
    idx = v.x + (v.y & 0);
  }
  t1 = clock64();
  out[3] = (t1 - t0) / n;
  // (e) shared atomicAdd (return value used)
  uint32_t r = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) r = atomicAdd(&cnt[(lane + r) & 31], 1u);
  t1 = clock64();
  out[4] = (t1 - t0) / n;
  // (f) 8 independent IMMA chains (throughput for one warp)
  int e0[4] = {0}, e1[4] = {0}, e2[4] = {0}, e3[4] = {0}, e4[4] = {0}, e5[4] = {0}, e6[4] = {0}, e7[4] = {0};
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    imma(e0, seed, i, seed, i, seed, i); imma(e1, seed, i, seed, i, seed, i);
    imma(e2, seed, i, seed, i, seed, i); imma(e3, seed, i, seed, i, seed, i);
    imma(e4, seed, i, seed, i, seed, i); imma(e5, seed, i, seed, i, seed, i);
    imma(e6, seed, i, seed, i, seed, i); imma(e7, seed, i, seed, i, seed, i);
  }
  t1 = clock64();
  out[5] = (t1 - t0) / n;
  // (g) FP64 division latency
  double x = 1.0 + seed * 1e-9;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = (x + 3.0) / 7.000001;
  t1 = clock64();
  out[6] = (t1 - t0) / n;
  out[7] = d[0] + d[1] + a + acc + idx + r + e0[0] + e1[1] + e2[2] + e3[3] + e4[0] + e5[1] + e6[2] + e7[3] + (long long)x;
}

int main() {
  unsigned long long* o;
  cudaMalloc(&o, 64 * 8);
  lat<<<1, 32>>>(o, 1000, 12345u);
  cudaDeviceSynchronize();
  unsigned long long h[8];
  cudaMemcpy(h, o, 64, cudaMemcpyDeviceToHost);
  printf("dependent IMMA.16832 chain      %llu clk\n", h[0]);
  printf("IMMA -> int use -> IMMA         %llu clk\n", h[1]);
  printf("mbarrier try_wait (complete)    %llu clk\n", h[2]);
  printf("dependent LDS.128               %llu clk\n", h[3]);
  printf("shared atomicAdd (used)         %llu clk\n", h[4]);
  printf("8 independent IMMA (per 8)      %llu clk\n", h[5]);
  printf("FP64 (x+3)/c dependent          %llu clk\n", h[6]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
