// Issue rate of the FP64 / conversion instructions the exact dequant epilogue
// uses (y = RN16(RN64(RN64(s_a * s_b) * corr))), sm_100a, per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbd tools/microbench_fp64.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k(int iters, double seed, long long iseed, float* out) {
  double a[4], b = seed * 1.0000001;
  long long c[4];
  float f[4];
  unsigned short h[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[j] = seed + threadIdx.x + j;
    c[j] = iseed + threadIdx.x * 7 + j;
    f[j] = 0.f;
    h[j] = 0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (OP == 0) a[j] = __dmul_rn(a[j], b);                               // DMUL
      if (OP == 1) { a[j] += static_cast<double>(c[j]); c[j] += 3; }        // I2F.F64.S64 (+DADD)
      if (OP == 2) { h[j] ^= __half_as_ushort(__double2half(a[j])); a[j] += 1.0; }  // F2F.F16.F64
      if (OP == 3) { f[j] += __double2float_rn(a[j]); a[j] += 1.0; }        // F2F.F32.F64
      if (OP == 4) { a[j] = __dadd_rn(a[j], b); }                           // DADD
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += static_cast<float>(a[j]) + f[j] + h[j];
  if (s == 1234.5f) out[0] = s;
}

template <int OP>
void run(const char* name, float* out) {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, blocks = sms * 8;
  k<OP><<<blocks, 256>>>(iters, 1.5, 3, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, 256>>>(iters, 1.5, 3, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = double(blocks) * 256 * iters * 4;
  printf("%-22s %8.2f ops/clk/SM\n", name, ops / (ms * 1e-3 * clk * 1e3) / sms);
}

// dependent-chain latency (one warp): cycles per instruction
template <int OP>
__global__ void lat(int iters, double seed, long long* out, double* sink) {
  double a = seed;
  float f = static_cast<float>(seed);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) a = __fma_rn(a, 1.0000001, 1e-9);
    if (OP == 1) a = 1.0 / a;
    if (OP == 2) f = __fmaf_rn(f, 1.0000001f, 1e-9f);
    if (OP == 3) a = static_cast<double>(static_cast<float>(a) + 1.0f);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    sink[0] = a + f;
  }
}

template <int OP>
void run_lat(const char* name, long long* o, double* sink) {
  const int iters = 4096;
  lat<OP><<<1, 32>>>(iters, 1.5, o, sink);
  lat<OP><<<1, 32>>>(iters, 1.5, o, sink);
  long long c;
  cudaMemcpy(&c, o, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %8.1f cycles latency\n", name, double(c) / iters);
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  run<0>("DMUL", out);
  run<4>("DADD", out);
  run<1>("I2F.F64.S64 + DADD", out);
  run<2>("F2F.F16.F64 + DADD", out);
  run<3>("F2F.F32.F64 + DADD", out);
  long long* o;
  double* sink;
  cudaMalloc(&o, 8);
  cudaMalloc(&sink, 8);
  run_lat<0>("DFMA chain", o, sink);
  run_lat<1>("FP64 1/x chain", o, sink);
  run_lat<2>("FFMA chain", o, sink);
  run_lat<3>("F2F.F32.F64+FADD+F2F", o, sink);
  return 0;
}
