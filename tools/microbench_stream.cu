// Streaming-read microbenchmark for the decode GEMV design (sm_100a):
// HBM -> SM bandwidth with (a) 1-D TMA bulk copies (cp.async.bulk) of CHUNK
// bytes into a per-warp shared-memory ring, (b) plain 16-byte LDG per lane
// with U loads in flight.  Buffer >> L2 so every byte comes from HBM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbs tools/microbench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int WARPS, int SLOTS, int CHUNK>
__global__ void __launch_bounds__(WARPS * 32, 1) tma_stream(const uint8_t* src, size_t chunks_per_warp, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[WARPS][SLOTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t gw = (size_t)blockIdx.x * WARPS + warp;
  const uint8_t* base = src + gw * chunks_per_warp * CHUNK;
  uint8_t* ring = sm + warp * SLOTS * CHUNK;
  if (lane == 0) {
    for (int s = 0; s < SLOTS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (int s = 0; s < SLOTS && s < (int)chunks_per_warp; ++s) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[warp][s])), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + s * CHUNK)),
                   "l"(base + s * CHUNK), "r"(CHUNK), "r"(sa(&bars[warp][s])) : "memory");
    }
  }
  __syncwarp();
  uint32_t acc = 0;
  int slot = 0; uint32_t phase = 0;
  for (size_t c = 0; c < chunks_per_warp; ++c) {
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(sa(&bars[warp][slot])), "r"(phase) : "memory");
    acc ^= reinterpret_cast<const uint32_t*>(ring + slot * CHUNK)[lane];
    __syncwarp();
    if (lane == 0 && c + SLOTS < chunks_per_warp) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[warp][slot])), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + slot * CHUNK)),
                   "l"(base + (c + SLOTS) * CHUNK), "r"(CHUNK), "r"(sa(&bars[warp][slot])) : "memory");
    }
    if (++slot == SLOTS) { slot = 0; phase ^= 1; }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int WARPS, int U>
__global__ void __launch_bounds__(WARPS * 32) ldg_stream(const uint4* src, size_t iters, uint32_t* sink) {
  const size_t gw = (size_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint4* base = src + gw * iters * U * 32;
  uint32_t acc = 0;
  for (size_t i = 0; i < iters; ++i) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint4* p = base + (i * U + u) * 32 + lane;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <typename F>
double time_it(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5 * 1e-3;
}

template <int WARPS, int SLOTS, int CHUNK>
void run_tma(const uint8_t* buf, size_t bytes, uint32_t* sink, int sms) {
  const size_t warps = (size_t)sms * WARPS;
  const size_t cpw = bytes / CHUNK / warps;
  const size_t smem = (size_t)WARPS * SLOTS * CHUNK;
  cudaFuncSetAttribute(tma_stream<WARPS, SLOTS, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double t = time_it([&] { tma_stream<WARPS, SLOTS, CHUNK><<<sms, WARPS * 32, smem>>>(buf, cpw, sink); });
  printf("TMA  warps=%2d slots=%d chunk=%5d  in-flight/SM=%6zu B : %7.1f GB/s  (%s)\n", WARPS, SLOTS, CHUNK, smem,
         cpw * CHUNK * warps / t * 1e-9, cudaGetErrorString(cudaGetLastError()));
}
template <int WARPS, int U, int BPS>
void run_ldg(const uint8_t* buf, size_t bytes, uint32_t* sink, int sms) {
  const size_t warps = (size_t)sms * BPS * WARPS;
  const size_t iters = bytes / (U * 512) / warps;
  double t = time_it([&] { ldg_stream<WARPS, U><<<sms * BPS, WARPS * 32>>>((const uint4*)buf, iters, sink); });
  printf("LDG  warps/SM=%2d U=%d                               : %7.1f GB/s\n", WARPS * BPS, U, iters * U * 512.0 * warps / t * 1e-9);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 2ull << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  uint32_t* sink; cudaMalloc(&sink, 64);
  run_tma<16, 5, 2048>(buf, bytes, sink, sms);
  run_tma<32, 2, 2048>(buf, bytes, sink, sms);
  run_tma<16, 2, 4096>(buf, bytes, sink, sms);
  run_tma<8, 4, 4096>(buf, bytes, sink, sms);
  run_tma<4, 4, 8192>(buf, bytes, sink, sms);
  run_tma<4, 6, 8192>(buf, bytes, sink, sms);
  run_tma<2, 4, 16384>(buf, bytes, sink, sms);
  run_tma<1, 6, 32768>(buf, bytes, sink, sms);
  run_ldg<16, 4, 1>(buf, bytes, sink, sms);
  run_ldg<16, 8, 1>(buf, bytes, sink, sms);
  run_ldg<8, 4, 4>(buf, bytes, sink, sms);
  run_ldg<8, 8, 4>(buf, bytes, sink, sms);
  run_ldg<32, 4, 1>(buf, bytes, sink, sms);
  return 0;
}
