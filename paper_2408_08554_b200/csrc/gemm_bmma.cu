// gemm_bmma.cu -- the binary-tensor-core (BTC) alternative for the prefill
// GEMM: the reference's plane decomposition (include/abq/gemm.hpp:94-146,
// paper Eq. 11) on the b1 tensor-core path that sm_100a still exposes,
// mma.sync.m16n8k256.row.col.s32.b1.b1.s32.and.popc, straight from the ABQP
// planes.  Kept as the measured comparator for the tcgen05 recombination
// GEMM (gemm_tc.cu): on sm_100a the b1 MMA is not a native tensor-core
// datapath (profiles/r01_microbench_pipes.txt: ~700 bit-MAC/clk/SM against
// ~8192 u8 MAC/clk/SM for tcgen05, and p x q plane pairs per code product), so
// the recombination kernel is the one the engine dispatches to.
//
// One warp computes a 16-channel x 8-token output tile over all p x q plane
// pairs: per 256-bit k step it loads the q weight-plane A fragments and the p
// activation-plane B fragments (32-bit words straight from the planes) and
// issues p x q BMMAs into accumulators grouped by s + t, combined at the end
// as sum_d 2^d acc_d.
#include "common.cuh"

namespace abq_dev {

__device__ __forceinline__ void bmma_16_8_256(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                              uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int P, int Q>
__global__ void __launch_bounds__(128) gemm_bmma_kernel(const uint64_t* __restrict__ a, int m,
                                                        const uint64_t* __restrict__ w, int n, int k,
                                                        int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int ntile_ch = (n + 15) / 16;
  const long long wt = static_cast<long long>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  const int ct = static_cast<int>(wt % ntile_ch), tt = static_cast<int>(wt / ntile_ch);
  if (tt * 8 >= m) return;
  const int wpr = (k + 63) / 64;
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(a);
  const uint32_t* w32 = reinterpret_cast<const uint32_t*>(w);
  const int r0 = ct * 16 + g, r1 = r0 + 8, tok = tt * 8 + g;
  int acc[P + Q - 1][4];
#pragma unroll
  for (int d = 0; d < P + Q - 1; ++d) acc[d][0] = acc[d][1] = acc[d][2] = acc[d][3] = 0;
  // 32-bit word of plane row `row` covering k = 32 * word32 .. +31 (0 past the end)
  auto word = [&](const uint32_t* base, int plane, int rows, int row, int w32i) -> uint32_t {
    if (row >= rows || w32i >= 2 * wpr) return 0u;
    return __ldg(base + (static_cast<size_t>(plane) * rows + row) * (2 * wpr) + w32i);
  };
  for (int k0 = 0; k0 < k; k0 += 256) {
    const int w0 = k0 / 32 + tig, w1 = w0 + 4;
    uint32_t fa[Q][4], fb[P][2];
#pragma unroll
    for (int t = 0; t < Q; ++t) {
      fa[t][0] = word(w32, t, n, r0, w0);
      fa[t][1] = word(w32, t, n, r1, w0);
      fa[t][2] = word(w32, t, n, r0, w1);
      fa[t][3] = word(w32, t, n, r1, w1);
    }
#pragma unroll
    for (int s = 0; s < P; ++s) {
      fb[s][0] = word(a32, s, m, tok, w0);
      fb[s][1] = word(a32, s, m, tok, w1);
    }
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int t = 0; t < Q; ++t) bmma_16_8_256(acc[s + t], fa[t][0], fa[t][1], fa[t][2], fa[t][3], fb[s][0], fb[s][1]);
  }
  // C fragment: c0,c1 -> row g, cols 2 tig, 2 tig + 1; c2,c3 -> row g + 8
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    long long v = 0;
#pragma unroll
    for (int d = 0; d < P + Q - 1; ++d) v += static_cast<long long>(acc[d][r]) << d;
    const int ch = ct * 16 + g + 8 * (r >> 1), tk = tt * 8 + 2 * tig + (r & 1);
    if (ch < n && tk < m) out[static_cast<size_t>(tk) * n + ch] = static_cast<int32_t>(v);
  }
}

template <int P, int Q>
static int launch_bmma(const uint64_t* a, size_t m, const uint64_t* w, size_t n, size_t k, int32_t* out,
                       cudaStream_t st) {
  const long long warps = static_cast<long long>((n + 15) / 16) * ((m + 7) / 8);
  gemm_bmma_kernel<P, Q><<<static_cast<unsigned>((warps + 3) / 4), 128, 0, st>>>(
      a, static_cast<int>(m), w, static_cast<int>(n), static_cast<int>(k), out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

// acc[m][n] (int32) = sum_{s,t} 2^(s+t) popc(A_s & W_t); the (p, q) pairs of
// the BASELINE configs are instantiated (2x8, 4x4, 8x8, 4x8, 8x4, 2x2).
int run_gemm_bmma(const uint64_t* a, unsigned p, size_t m, const uint64_t* w, unsigned q, size_t n, size_t k,
                  int32_t* out, cudaStream_t st) {
  if (m == 0 || n == 0) return ABQ_OK;
#define ABQ_BMMA_CASE(PP, QQ) \
  if (p == PP && q == QQ) return launch_bmma<PP, QQ>(a, m, w, n, k, out, st);
  ABQ_BMMA_CASE(4, 4)
  ABQ_BMMA_CASE(8, 8)
  ABQ_BMMA_CASE(8, 2)
  ABQ_BMMA_CASE(8, 4)
  ABQ_BMMA_CASE(4, 8)
  ABQ_BMMA_CASE(2, 2)
#undef ABQ_BMMA_CASE
  return fail(ABQ_ERR_VALUE, "gemm_bmma: plane counts (%u, %u) not instantiated", p, q);
}

}  // namespace abq_dev
