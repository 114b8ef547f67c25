// Pipe-rate microbenchmarks for sm_100a: POPC, LOP3, IADD3, IMAD, IDP4A,
// legacy IMMA (mma.sync u8), emulated b1 mma.sync (and.popc). Decides the
// decode-GEMV / prefill-GEMM designs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c * 77 + 1);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = __popc(v[c]) ^ (v[c] + 0x9e3779b9u);
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= v[c];
  if (s == 0x12345) out[0] = s;
}
// pure POPC feeding xor: each iter 1 POPC + 1 IADD3/LOP3 pair -> test ratio
__global__ void k_popc_acc(uint32_t* out, uint32_t seed) {
  uint32_t w[CH], acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { w[c] = seed * (threadIdx.x + c * 77 + 1); acc[c] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) { acc[c] += __popc(w[c] & (acc[c] | i)); }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH], c2[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = seed * (threadIdx.x + c); b[c] = a[c] * 3; c2[c] = a[c] ^ 0x5555; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t t;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(t) : "r"(a[c]), "r"(b[c]), "r"(c2[c]));
      asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(c2[c]) : "r"(a[c]), "r"(b[c]), "r"(c2[c]));
      a[c] = t;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c] ^ c2[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_dp4a(uint32_t* out, uint32_t seed) {
  int a[CH], b[CH], acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = seed * (threadIdx.x + c); b[c] = a[c] * 7; acc[c] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __dp4a((unsigned)a[c], (unsigned)b[c], (unsigned)acc[c]);
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = __dp4a((unsigned)b[c], (unsigned)a[c], (unsigned)acc[c]);
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= acc[c];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_imma(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed * threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int d[4][4] = {};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s ^= d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_bmma(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed * threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int d[4][4] = {};
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s ^= d[c][0] ^ d[c][1] ^ d[c][2] ^ d[c][3];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_ddiv(double* out, double seed) {
  double v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed + threadIdx.x + c;
  double st = seed * 0.37 + 1.1;
  for (int i = 0; i < ITERS / 16; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) v[c] = round(v[c] / st) + 1.0;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 0.123) out[0] = s;
}

template <typename K, typename T>
void run(const char* name, K kern, T* buf, double ops_per_thread_iter, int iters, int blocks_per_sm, int threads) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * blocks_per_sm;
  kern<<<grid, threads>>>(buf, (T)3);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<grid, threads>>>(buf, (T)3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double sec = ms * 1e-3 / 5;
  double total = ops_per_thread_iter * iters * (double)grid * threads;
  double per_sec = total / sec;
  // report per SM per clock at max clock and per-second
  printf("%-10s %10.3f Gop/s  %8.2f ops/clk/SM @max(%d MHz)  (%.1f us)\n", name, per_sec * 1e-9,
         per_sec / sms / (clk * 1e3), clk / 1000, sec * 1e6);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("  error %s\n", cudaGetErrorString(err));
}

int main() {
  uint32_t* b; cudaMalloc(&b, 64);
  double* d; cudaMalloc(&d, 64);
  for (int bps : {4, 8}) {
    printf("--- %d blocks/SM x 256 threads ---\n", bps);
    run("popc+xor", k_popc, b, CH * 1.0, ITERS, bps, 256);          // count POPCs
    run("popc_acc", k_popc_acc, b, CH * 1.0, ITERS, bps, 256);      // count POPCs (with and+add)
    run("lop3", k_lop3, b, CH * 2.0, ITERS, bps, 256);              // count LOP3s
    run("dp4a", k_dp4a, b, CH * 2.0, ITERS, bps, 256);              // count IDP4A
    run("imma_mac", k_imma, b, 4.0 * 16 * 8 * 32 / 32, ITERS, bps, 256);  // MACs per thread
    run("bmma_mac", k_bmma, b, 4.0 * 16 * 8 * 256 / 32, ITERS / 8, bps, 256);  // 1-bit MACs
    run("ddiv+rnd", k_ddiv, d, CH * 1.0, ITERS / 16, bps, 256);
  }
  return 0;
}
