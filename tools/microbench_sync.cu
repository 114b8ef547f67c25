// Latency of the per-slot primitives of the decode GEMV consumer loop, one
// warp, in SM clocks: mbarrier try_wait / test_wait on a completed phase,
// mbarrier arrive, a dependent LDS.128 chain, S2R of the thread index,
// __syncwarp, and legacy IMMA m16n8k32 (dependent chain).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbsync tools/microbench_sync.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(unsigned long long* out, int reps) {
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(16) uint4 buf[64];
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(sa(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    // complete phase 0 of bar[0]
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[0])));
  }
  for (int i = lane; i < 64; i += 32) buf[i] = make_uint4(i, i, i, i);
  __syncwarp();
  unsigned long long t0, t1;
  uint32_t sink = 0;
  // (a) try_wait.parity on the completed phase 0
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sa(&bar[0])) : "memory");
    sink += ok;
  }
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / reps;
  // (b) test_wait.parity
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(sa(&bar[0])) : "memory");
    sink += ok;
  }
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0) / reps;
  // (c) arrive (lane 0) on a barrier with a huge count + syncwarp
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar[1])) : "memory");
    __syncwarp();
  }
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0) / reps;
  // (d) dependent LDS.128 chain
  uint32_t idx = lane;
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint4 v = buf[idx & 63];
    idx = v.x + 1;
  }
  t1 = clock64();
  sink += idx;
  if (lane == 0) out[3] = (t1 - t0) / reps;
  // (e) S2R tid chain
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    uint32_t t;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
    sink += t;
  }
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0) / reps;
  // (f) dependent IMMA chain
  int acc[4] = {0, 0, 0, 0};
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3])
                 : "r"(idx), "r"(idx), "r"(idx), "r"(idx), "r"(sink), "r"(sink));
  }
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0) / reps;
  // (g) four independent IMMA chains
  int a2[4][4] = {};
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(a2[c][0]), "+r"(a2[c][1]), "+r"(a2[c][2]), "+r"(a2[c][3])
                   : "r"(idx), "r"(idx), "r"(idx), "r"(idx), "r"(sink), "r"(sink));
  }
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0) / reps;
  // (h) globaltimer read + store
  t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    sink += (uint32_t)g;
  }
  t1 = clock64();
  if (lane == 0) out[7] = (t1 - t0) / reps;
  if (sink == 0x12345 && acc[0] == 7 && a2[1][2] == 9) out[8] = sink;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16 * 8);
  probe<<<1, 32>>>(d, 1000);
  probe<<<1, 32>>>(d, 1000);
  unsigned long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"mbarrier.try_wait (phase complete)", "mbarrier.test_wait (phase complete)",
                         "mbarrier.arrive + __syncwarp", "dependent LDS.128", "S2R tid",
                         "dependent IMMA.16832.U8", "4 independent IMMA chains (per round of 4)", "globaltimer read"};
  for (int i = 0; i < 8; ++i) printf("%-45s %6llu cycles\n", names[i], h[i]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
