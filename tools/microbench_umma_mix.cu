// UMMA (kind::i8, M = N = 128, K = 32, A in TMEM, commit every 4) throughput
// while other warps of the CTA keep the SM busy: X = 1 four warps stream
// tcgen05.st x32 into other TMEM columns, X = 2 four warps stream LDS.128,
// X = 4 four warps stream STS.128, X = 8 the MMA thread polls an mbarrier
// (try_wait) between groups of 4 UMMAs.  Cycles per UMMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbumix tools/microbench_umma_mix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int X>
__global__ void __launch_bounds__(256, 1) mix(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar, cbar[8];
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&cbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  uint32_t sink = 0;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | (128u >> 3 << 17) | (128u >> 4 << 24);
    const uint32_t b0 = sa(sm);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int j = it & 3;
      const uint64_t bd = desc(b0 + j * 2 * 128 + ((it >> 2) & 3) * 16384, 128, 1024);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
          "r"(tm + 128 + ((it >> 2) & 7) * 32 + j * 8), "l"(bd), "r"(idesc), "r"(it));
      if (j == 3) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         sa(&cbar[(it >> 2) & 7]))
                     : "memory");
        if (X & 32) {  // poll a shared-memory word instead (LDS)
          sink += stop;
        }
        if ((X & 64) && (it & 15) == 15) {  // a try_wait every 16 UMMAs (4 k-blocks)
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(sa(&bar)) : "memory");
          sink += ok;
        }
        if ((X & 128) && (it & 7) == 7) {  // ... every 8 UMMAs, two back-to-back
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(sa(&bar)) : "memory");
          sink += ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(sa(&cbar[7])) : "memory");
          sink += ok;
        }
        if (X & 8) {  // poll a barrier that is never pending (phase 1 of bar completed = false -> try once)
          uint32_t ok;
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(sa(&bar)) : "memory");
          sink += ok;
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
            sa(&bar))
        : "memory");
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (warp >= 4) {
    const int w = warp - 4, lane = tid & 31;
    if ((X & 1)) {
      const uint32_t ta = tm + (static_cast<uint32_t>(w * 32) << 16) + 384;
      uint32_t v = tid;
      while (!stop) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
            "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(ta), "r"(v) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        ++v;
      }
    }
    if ((X & 16) && w == 0 && lane == 0) {  // another warp spinning on try_wait
      while (!stop) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(sa(&bar)) : "memory");
        sink += ok;
      }
    }
    if (X & 2) {
      const uint32_t base = sa(sm + 65536) + (w * 32 + lane) * 16;
      while (!stop) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t a, b, c, d;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(base + i * 2048));
          sink ^= a ^ b ^ c ^ d;
        }
      }
    }
    if (X & 4) {
      const uint32_t base = sa(sm + 65536) + (w * 32 + lane) * 16;
      while (!stop) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" ::"r"(base + i * 2048), "r"(sink + i) : "memory");
        ++sink;
      }
    }
  }
  if (sink == 0x12345678u) out[1023] = sink;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int X>
void run(int sms, long long* out) {
  const int iters = 8192, smem = 128 * 1024;
  cudaFuncSetAttribute(mix<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mix<X><<<sms, 256, smem>>>(iters, out);
  mix<X><<<sms, 256, smem>>>(iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("X=%d error %s\n", X, cudaGetErrorString(e));
    return;
  }
  long long h[256];
  cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < sms; ++i) c += h[i];
  c /= sms;
  printf("X=%2d (%s%s%s%s): %6.1f cycles/UMMA\n", X, X & 1 ? "STTM " : "", X & 2 ? "LDS " : "", X & 4 ? "STS " : "",
         X & 8 ? "poll " : "", c / iters);
  if (X & 48) printf("   (16: other warp spins on try_wait, 32: MMA thread polls a shared word)\n");
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMalloc(&out, 1024 * 8);
  run<0>(sms, out);
  run<1>(sms, out);
  run<2>(sms, out);
  run<4>(sms, out);
  run<8>(sms, out);
  run<3>(sms, out);
  run<16>(sms, out);
  run<32>(sms, out);
  run<64>(sms, out);
  run<128>(sms, out);
  return 0;
}
