// Issue-to-completion throughput of tcgen05.mma kind::i8 (u8 x u8 -> s32,
// M = 128, K = 32, K-major no-swizzle operands resident in shared memory) on
// sm_100a: one elected thread issues back-to-back UMMAs into one TMEM
// accumulator, commits, waits.  Reports cycles per UMMA and MAC/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbu tools/microbench_umma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int N, int C = 0, int TA = 0>
__global__ void __launch_bounds__(128, 1) umma_loop(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar, cbar[8];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 * 128 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&cbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tbase)), "r"(TA ? 2 * N : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
    const uint32_t a0 = sa(sm), b0 = sa(sm + 128 * 128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int j = it & 3;
      const uint64_t ad = desc(a0 + j * 2 * 2048, 2048, 128);
      const uint64_t bd = desc(b0 + j * 2 * 128, 128, 1024);
      if (TA)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
            "r"(tm + N + j * 8), "l"(bd), "r"(idesc), "r"(it));
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(ad), "l"(bd), "r"(idesc), "r"(it));
      if (C > 0 && (it % (C > 0 ? C : 1)) == C - 1)  // commit (never waited on) every C UMMAs
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         sa(&cbar[(it / (C > 0 ? C : 1)) & 7]))
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
            sa(&bar))
        : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(TA ? 2 * N : N));
}

template <int N, int C = 0, int TA = 0>
void run(int sms, long long* out) {
  const int iters = 8192;
  const int smem = 128 * 128 + N * 128;
  cudaFuncSetAttribute(umma_loop<N, C, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_loop<N, C, TA><<<sms, 128, smem>>>(iters, out);
  umma_loop<N, C, TA><<<sms, 128, smem>>>(iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d error %s\n", N, cudaGetErrorString(e));
    return;
  }
  long long h[256];
  cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  printf("UMMA kind::i8 M=128 N=%3d K=32 A in %s, commit every %d: %6.1f cycles/UMMA  %7.0f MAC/clk/SM\n", N,
         TA ? "TMEM" : "smem", C, c / iters,
         128.0 * N * 32 * iters / c);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, 256 * 8);
  run<64>(sms, out);
  run<128>(sms, out);
  run<256>(sms, out);
  run<128, 4>(sms, out);
  run<128, 8>(sms, out);
  run<128, 1>(sms, out);
  run<128, 0, 1>(sms, out);
  run<128, 4, 1>(sms, out);
  run<128, 8, 1>(sms, out);
  return 0;
}
