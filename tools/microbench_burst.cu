// Short-burst streaming microbenchmark: the shape of one decode GEMV launch.
// Every CTA (one per SM) streams its share B of a weight copy through a TMA
// ring with F bytes in flight; launches are back to back in a CUDA graph over
// rotating copies (> 4x L2).  Reports per-launch time and the latency of a
// dependent chain of L2-hit loads issued while the ring is in flight (what a
// prologue pays for every memory access made after the ring starts).
// Also: empty-kernel floor, with and without programmatic dependent launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbb tools/microbench_burst.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Args {
  const uint8_t* src;   // this launch's copy
  size_t per_cta;       // bytes per CTA
  int chunk, slots;     // ring geometry (single warp producer/consumer)
  const uint32_t* probe;  // L2-resident pointer-chase array (or null)
  int probe_len;
  unsigned long long* out;  // [grid][4]
  int pdl;
};

__global__ void __launch_bounds__(128, 1) burst(Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint8_t* base = a.src + blockIdx.x * a.per_cta;
  const int nchunks = (int)(a.per_cta / a.chunk);
  unsigned long long t0 = gt();
  if (a.pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < a.slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[s])));
      asm volatile("fence.mbarrier_init.release.cluster;");
      for (int s = 0; s < a.slots && s < nchunks; ++s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])), "r"(a.chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + s * a.chunk)), "l"(base + (size_t)s * a.chunk), "r"(a.chunk), "r"(sa(&bars[s]))
                     : "memory");
      }
    }
    __syncwarp();
    uint32_t acc = 0;
    int slot = 0;
    uint32_t phase = 0;
    for (int c = 0; c < nchunks; ++c) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
              sa(&bars[slot])), "r"(phase)
          : "memory");
      acc ^= reinterpret_cast<const uint32_t*>(sm + slot * a.chunk)[lane];
      __syncwarp();
      if (lane == 0 && c + a.slots < nchunks) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[slot])), "r"(a.chunk));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + slot * a.chunk)), "l"(base + (size_t)(c + a.slots) * a.chunk), "r"(a.chunk), "r"(sa(&bars[slot]))
                     : "memory");
      }
      if (++slot == a.slots) {
        slot = 0;
        phase ^= 1;
      }
    }
    if (acc == 0x12345678u && a.out) a.out[0] = acc;
  } else if (warp == 1 && lane == 0 && a.probe) {
    // dependent pointer chase through an L2-resident array, started a little after the ring
    unsigned long long p0 = gt();
    uint32_t i = blockIdx.x & 63;
    for (int r = 0; r < a.probe_len; ++r) i = __ldcg(a.probe + i * 32);  // 128 B apart
    unsigned long long p1 = gt();
    if (a.out) {
      a.out[blockIdx.x * 4 + 1] = (p1 - p0) / a.probe_len;
      a.out[blockIdx.x * 4 + 3] = i;
    }
  }
  __syncthreads();
  if (a.out && tid == 0) {
    a.out[blockIdx.x * 4 + 0] = gt() - t0;
  }
}

__global__ void empty_kernel(int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

static void launch(Args a, int grid, size_t smem, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  a.pdl = pdl;
  cudaLaunchKernelEx(&cfg, burst, a);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = 640ull << 20;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  uint32_t* probe;
  cudaMalloc(&probe, 64 * 32 * 4);
  std::vector<uint32_t> hp(64 * 32);
  for (int i = 0; i < 64; ++i) hp[i * 32] = (i * 17 + 5) & 63;
  cudaMemcpy(probe, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, sms * 4 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);

  // empty-kernel floor
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms);
      cfg.blockDim = dim3(128);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl;
      cudaLaunchKernelEx(&cfg, empty_kernel, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel grid=%d pdl=%d: %.3f us/launch\n", sms, pdl, ms * 1e3 / 2000);
  }

  const size_t per_cta_list[] = {28 * 1024, 152 * 1024, 304 * 1024};
  const int inflight_kb[] = {16, 32, 48, 64, 96, 128, 192};
  for (size_t per_cta : per_cta_list) {
    const size_t copy = per_cta * sms;
    const int copies = (int)(total / copy);
    for (int pdl = 0; pdl < 2; ++pdl)
      for (int fk : inflight_kb) {
        const int chunk = fk >= 64 ? 16384 : 4096;
        const int slots = fk * 1024 / chunk;
        const size_t smem = (size_t)fk * 1024;
        Args a{};
        a.per_cta = per_cta;
        a.chunk = chunk;
        a.slots = slots;
        a.probe = nullptr;
        a.out = nullptr;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        const int L = copies * 4;
        for (int i = 0; i < L; ++i) {
          a.src = buf + (size_t)(i % copies) * copy;
          launch(a, sms, smem, s, pdl);
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / (5 * L);
        // probe run (single launches, traced) right after a warm graph
        a.probe = probe;
        a.probe_len = 8;
        a.out = out;
        a.src = buf;
        cudaGraphLaunch(ge, s);
        launch(a, sms, smem, s, 0);
        cudaStreamSynchronize(s);
        std::vector<unsigned long long> h(sms * 4);
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        double lat = 0, dur = 0;
        for (int b = 0; b < sms; ++b) {
          lat += h[b * 4 + 1];
          dur += h[b * 4 + 0];
        }
        printf("per-CTA %6zu B  in-flight %3d KB  pdl=%d : %7.3f us/launch  %7.1f GB/s   probe L2-hit lat %6.0f ns  CTA span %6.0f ns  (%s)\n",
               per_cta, fk, pdl, us, copy / us * 1e-3, lat / sms, dur / sms, cudaGetErrorString(cudaGetLastError()));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
      }
  }
  return 0;
}
