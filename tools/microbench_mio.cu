// Does a TMA weight stream into shared memory slow the other warps' shared-
// memory instructions?  One CTA per SM: warp 8 streams a 640 MB buffer through
// a ring (1-D bulk copies, 16 KB chunks, `inflight` KB in flight) while warps
// 0..7 run a fixed loop of (a) independent LDS.128, (b) ALU-only work, or
// (c) mbarrier try_wait on a completed phase; reports cycles per loop
// iteration with the stream on and off.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbmio tools/microbench_mio.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(288, 1) kern(const uint8_t* src, size_t per_cta, int slots, int mode, int iters,
                                               int stream, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ int stop;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunk = 16384;
  if (tid == 0) {
    for (int s = 0; s < 16; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&done_bar)));
    stop = 0;
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0 && stream) {
      const uint8_t* base = src + blockIdx.x * per_cta;
      const int n = (int)(per_cta / chunk);
      uint32_t ph[16] = {};
      for (int i = 0; i < n && !*(volatile int*)&stop; ++i) {
        const int s = i % slots;
        if (i >= slots) {
          asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(&full[s])), "r"(ph[s]) : "memory");
          ph[s] ^= 1;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(sm + s * chunk)),
                     "l"(base + (size_t)i * chunk), "r"(chunk), "r"(sa(&full[s])) : "memory");
      }
    }
    return;
  }
  // workers: wait until the stream is running (~2 us), then time their loop
  const long long t_start = clock64();
  while (clock64() - t_start < 4000) {
  }
  uint32_t acc = lane;
  const long long t0 = clock64();
  if (mode == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(sm + 16384 * 8 + warp * 2048) + lane;  // outside the ring
    for (int r = 0; r < iters; ++r) {
      uint4 v0 = p[0], v1 = p[32], v2 = p[64], v3 = p[96];
      acc += v0.x ^ v1.y ^ v2.z ^ v3.w;
    }
  } else if (mode == 1) {
    for (int r = 0; r < iters; ++r) {
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = (acc << 1) ^ (acc >> 3) ^ u;
    }
  } else {
    for (int r = 0; r < iters; ++r) {
      uint32_t ok;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(sa(&done_bar)) : "memory");
      acc += ok;
    }
  }
  const long long t1 = clock64();
  if (tid == 0) stop = 1;
  if (lane == 0) out[blockIdx.x * 8 + warp] = (t1 - t0) / iters;
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = 640ull << 20;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* out;
  cudaMalloc(&out, sms * 8 * 8);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"4 x LDS.128 (independent)", "16 dependent ALU ops", "mbarrier try_wait (complete)"};
  unsigned long long* h = new unsigned long long[sms * 8];
  for (int mode = 0; mode < 3; ++mode)
    for (int stream = 0; stream < 2; ++stream) {
      kern<<<sms, 288, 160 * 1024>>>(buf, total / sms / 16384 * 16384, 8, mode, 2000, stream, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, sms * 8 * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (int i = 0; i < sms * 8; ++i) m += h[i];
      printf("%-32s stream=%d : %7.1f cycles / iteration (8 warps per SM)  %s\n", names[mode], stream, m / (sms * 8),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
