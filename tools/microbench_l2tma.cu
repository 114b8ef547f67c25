// L2 -> shared-memory ingest rate of 1-D TMA bulk copies on sm_100a, one CTA
// per SM, data resident in L2.  Question it answers: what bounds the tcgen05
// GEMM's per-stage operand loads (profiles/r01_microbench_l2tma.txt).
//   shared : every CTA copies the same 64 KB region (activation tile pattern)
//   private: every CTA copies its own 64 KB region
//   mcastC : clusters of C CTAs; each CTA copies 1/C of a 16 KB chunk and
//            multicasts it to the whole cluster (.multicast::cluster)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbt tools/microbench_l2tma.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b)));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          sa(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(n), "r"(sa(b))
               : "memory");
}
__device__ __forceinline__ void bulk_mc(void* dst, const void* src, uint32_t n, uint64_t* b, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          sa(dst)),
      "l"(src), "r"(n), "r"(sa(b)), "h"(mask)
      : "memory");
}

constexpr int kChunk = 16384, kSlots = 4;

template <int MODE, int C>  // MODE 0 shared, 1 private, 2 multicast (cluster C)
__global__ void __launch_bounds__(32, 1) ingest(const unsigned char* src, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[kSlots];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < kSlots; ++s) bar_init(&bars[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (C > 1) cg::this_cluster().sync();
  __syncwarp();
  const unsigned char* base = MODE == 1 ? src + static_cast<size_t>(blockIdx.x) * kSlots * kChunk : src;
  const unsigned rank = C > 1 ? cg::this_cluster().block_rank() : 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it % kSlots;
    if (it >= kSlots) wait_par(&bars[s], ((it / kSlots) - 1) & 1);  // slot consumed
    if (MODE == 2 && C > 1 && it >= kSlots) {
      // nobody refills slot s until every CTA of the cluster is done with it
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (lane == 0) {
      expect_tx(&bars[s], kChunk);
      if (MODE == 2) {
        const uint32_t piece = kChunk / C;  // my piece, delivered to every CTA of the cluster
        bulk_mc(sm + s * kChunk + rank * piece, base + s * kChunk + rank * piece, piece, &bars[s],
                static_cast<uint16_t>((1u << C) - 1));
      } else {
        bulk(sm + s * kChunk, base + s * kChunk, kChunk, &bars[s]);
      }
    }
    __syncwarp();
  }
  for (int it = iters; it < iters + kSlots; ++it) wait_par(&bars[it % kSlots], ((it / kSlots) - 1) & 1);
  __syncwarp();
  long long t1 = clock64();
  if (C > 1) cg::this_cluster().sync();
  if (lane == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE, int C>
void run(const char* name, const unsigned char* src, long long* out, int sms) {
  const int iters = 4000;
  const int grid = (sms / C) * C;
  auto k = ingest<MODE, C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * kChunk);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = kSlots * kChunk;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, src, iters, out);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, src, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    printf("%-10s error %s\n", name, cudaGetErrorString(e));
    return;
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[1024];
  cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < grid; ++i) cyc += h[i];
  cyc /= grid;
  const double bytes_per_cta = double(iters) * kChunk;  // bytes landing in each CTA's smem
  printf("%-10s CTAs=%3d  %.1f B/clk/SM into smem  (%.2f TB/s delivered, %.2f TB/s read from L2)\n", name, grid,
         bytes_per_cta / cyc, bytes_per_cta * grid / (ms * 1e-3) / 1e12,
         bytes_per_cta * grid / C / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned char* src;
  cudaMalloc(&src, static_cast<size_t>(sms) * kSlots * kChunk);
  cudaMemset(src, 1, static_cast<size_t>(sms) * kSlots * kChunk);
  long long* out;
  cudaMalloc(&out, 1024 * 8);
  run<0, 1>("shared", src, out, sms);
  run<1, 1>("private", src, out, sms);
  run<2, 2>("mcast2", src, out, sms);
  run<2, 4>("mcast4", src, out, sms);
  return 0;
}
