// Latency (SM clocks, one warp, warm) of the fused-ReQuant prologue pieces:
// group_params (FP64 step / zero point), f32_reciprocal, quant_codes8_f16 on
// one 16-byte vector, a REDUX + shared atomic, and a 512-thread bar.sync.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_08554_b200/csrc -I include \
//        --expt-relaxed-constexpr -o tools/mbquant tools/microbench_quant.cu
#include <cstdio>
#include "quant_dev.cuh"

using namespace abq_dev;

__global__ void probe(const uint4* x, QuantParams qp, unsigned long long* out, float lo_in, float hi_in) {
  __shared__ unsigned long long s;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  unsigned long long acc = 0;
  for (int rep = 0; rep < 3; ++rep) {  // rep 0 cold i-cache, reps 1-2 warm
    const long long t0 = clock64();
    double step = 0.0;
    int z = 0;
    float inv = 0.f;
    if (lane == 0) {
      group_params(qp, lo_in + rep * 1e-7f, hi_in, &step, &z);
    }
    step = __shfl_sync(0xffffffffu, step, 0);
    z = __shfl_sync(0xffffffffu, z, 0);
    const long long t1 = clock64();
    if (lane == 0) inv = f32_reciprocal(step);
    inv = __shfl_sync(0xffffffffu, inv, 0);
    const long long t2 = clock64();
    uint32_t w0, w1;
    int sum = quant_codes8_f16(x[threadIdx.x], step, inv, z, 15, &w0, &w1);
    acc += w0 ^ w1;
    const long long t3 = clock64();
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (lane == 0) atomicAdd(&s, (unsigned long long)sum);
    const long long t4 = clock64();
    __syncthreads();
    const long long t5 = clock64();
    if (threadIdx.x == 0) {
      out[rep * 8 + 0] = t1 - t0;
      out[rep * 8 + 1] = t2 - t1;
      out[rep * 8 + 2] = t3 - t2;
      out[rep * 8 + 3] = t4 - t3;
      out[rep * 8 + 4] = t5 - t4;
    }
  }
  if (acc == 12345) out[63] = acc + s;
}

int main() {
  uint4* x;
  cudaMalloc(&x, 512 * 16);
  cudaMemset(x, 0x3c, 512 * 16);
  unsigned long long* out;
  cudaMalloc(&out, 64 * 8);
  QuantParams qp{4, ABQ_ASYMMETRIC, 0, 1.0, 1.0, 16};
  for (int threads : {32, 512}) {
    probe<<<1, threads>>>(x, qp, out, -3.1f, 2.7f);
    unsigned long long h[64];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[] = {"group_params + 2 shfl", "f32_reciprocal + shfl", "quant_codes8_f16 (8 codes)",
                           "REDUX add + shared atomic", "bar.sync"};
    printf("block of %d threads (%s)\n", threads, cudaGetErrorString(cudaGetLastError()));
    for (int i = 0; i < 5; ++i) printf("  %-28s cold %5llu  warm %5llu %5llu cycles\n", names[i], h[i], h[8 + i], h[16 + i]);
  }
  return 0;
}
