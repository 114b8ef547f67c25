// gemv_popc.cu -- K2: bit-serial AND + popcount plane GEMV/GEMM on CUDA cores
// with the fused K4 epilogue, sm_100a.
//
// Computes acc[i][j] = sum_{s<p} sum_{t<q} 2^(s+t) * sum_w popc(A_s[i][w] & W_t[j][w])
// -- the reference's gemm_plane_rows / gemm_naive sum (include/abq/gemm.hpp:94-146,
// 213-231, paper Eq. 11) -- then zero-point correction and dequant in the
// epilogue (gemm.hpp:235-254, 292-306).
//
// Layout / mapping (B200-first, decode-shaped):
//   * activation planes of MT tokens are staged once per CTA in shared memory
//     ([p][MT][wpr2] u64);
//   * each warp owns R consecutive weight rows (output channels) at a time and
//     its 32 lanes stride the K words with 16-byte loads (two u64 words per
//     lane, 512 B per warp per plane row: fully coalesced, L1-bypassing
//     streaming loads of the ABQP planes, which are read exactly once);
//   * per lane: R*q weight vectors in registers, p*MT activation vectors from
//     shared memory (reused R*q times), AND + POPC + shift-add;
//   * warp-shuffle butterfly reduction, then the epilogue is spread over lanes.
// Exact integer arithmetic: u32 lane accumulators whenever fits_int32 holds
// (every lane partial is bounded by the total), u64 for the _wide path.
#include <type_traits>

#include "common.cuh"

namespace abq_dev {

__device__ __forceinline__ uint4 ld_stream_u4(const uint64_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream_u2(const uint64_t* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

template <int PT, int QT, int MT, int R, bool WIDE, bool VEC>
__global__ void __launch_bounds__(256)
    gemv_popc_kernel(const uint64_t* __restrict__ A, int p_rt, int m,
                     const uint64_t* __restrict__ W, int q_rt, int n, int wpr, EpiParams e) {
  constexpr int PMAX = PT > 0 ? PT : 8;
  constexpr int QMAX = QT > 0 ? QT : 8;
  constexpr int NW = VEC ? 4 : 2;  // u32 words per lane per load
  using Acc = typename std::conditional<WIDE, unsigned long long, unsigned>::type;
  const int p = PT > 0 ? PT : p_rt;
  const int q = QT > 0 ? QT : q_rt;

  extern __shared__ __align__(16) uint64_t smA[];
  const int wpr2 = (wpr + 1) & ~1;
  const int m0 = blockIdx.y * MT;
  for (int idx = threadIdx.x; idx < p * MT * wpr2; idx += blockDim.x) {
    const int w = idx % wpr2, r = idx / wpr2, i = r % MT, s = r / MT;
    uint64_t v = 0;
    if (w < wpr && m0 + i < m) v = A[(static_cast<size_t>(s) * m + m0 + i) * wpr + w];
    smA[idx] = v;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lane_words = VEC ? 2 : 1;
  const int step_words = 32 * lane_words;
  const uint32_t* smA32 = reinterpret_cast<const uint32_t*>(smA);

  for (long long row0 = (static_cast<long long>(blockIdx.x) * nwarps + warp) * R; row0 < n;
       row0 += static_cast<long long>(gridDim.x) * nwarps * R) {
    Acc acc[MT][R];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][r] = 0;

    for (int w0 = lane * lane_words; w0 < wpr; w0 += step_words) {
      uint32_t wv[QMAX][R][NW];
#pragma unroll
      for (int t = 0; t < QMAX; ++t)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const long long row = row0 + r;
          if (t < q && row < n) {
            const uint64_t* src = W + (static_cast<size_t>(t) * n + row) * wpr + w0;
            if (VEC) {
              const uint4 v = ld_stream_u4(src);
              wv[t][r][0] = v.x;
              wv[t][r][1] = v.y;
              if (NW == 4) {
                wv[t][r][NW - 2] = v.z;
                wv[t][r][NW - 1] = v.w;
              }
            } else {
              const uint2 v = ld_stream_u2(src);
              wv[t][r][0] = v.x;
              wv[t][r][1] = v.y;
            }
          } else {
#pragma unroll
            for (int u = 0; u < NW; ++u) wv[t][r][u] = 0u;
          }
        }
#pragma unroll
      for (int s = 0; s < PMAX; ++s) {
        if (s < p) {
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            uint32_t av[NW];
            const uint32_t* ap = smA32 + 2 * ((static_cast<size_t>(s) * MT + i) * wpr2 + w0);
            if (VEC) {
              const uint4 v = *reinterpret_cast<const uint4*>(ap);
              av[0] = v.x;
              av[1] = v.y;
              if (NW == 4) {
                av[NW - 2] = v.z;
                av[NW - 1] = v.w;
              }
            } else {
              const uint2 v = *reinterpret_cast<const uint2*>(ap);
              av[0] = v.x;
              av[1] = v.y;
            }
#pragma unroll
            for (int t = 0; t < QMAX; ++t) {
              if (t < q) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  unsigned c = 0;
#pragma unroll
                  for (int u = 0; u < NW; ++u) c += __popc(av[u] & wv[t][r][u]);
                  acc[i][r] += static_cast<Acc>(c) << (s + t);
                }
              }
            }
          }
        }
      }
    }
    // warp reduction (xor butterfly: every lane ends with the full sums)
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        Acc v = acc[i][r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[i][r] = v;
      }
    // epilogue: element (i, r) handled by lane (i*R + r) % 32
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (lane == ((i * R + r) & 31)) {
          const long long row = row0 + r;
          const int tok = m0 + i;
          if (row < n && tok < m) epi_store(e, tok, row, static_cast<long long>(acc[i][r]));
        }
      }
  }
}

// ============================================================================
// dispatch
// ============================================================================
template <int PT, int QT, int MT, bool WIDE, bool VEC>
static int launch_one(const uint64_t* A, int p, int m, const uint64_t* W, int q, int n, int wpr,
                      const EpiParams& e, cudaStream_t st) {
  constexpr int QQ = QT > 0 ? QT : 8;
  constexpr int R = QT == 0 ? 2 : (QQ <= 2 ? 4 : (QQ <= 4 ? 2 : 1));
  const int wpr2 = (wpr + 1) & ~1;
  const size_t smem = static_cast<size_t>(p) * MT * wpr2 * sizeof(uint64_t);
  auto kern = gemv_popc_kernel<PT, QT, MT, R, WIDE, VEC>;
  if (smem > 48 * 1024) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
    if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv: smem attribute: %s", cudaGetErrorString(err));
  }
  const int threads = 256;
  const long long rows_per_cta = (threads / 32) * R;
  long long gx = (n + rows_per_cta - 1) / rows_per_cta;
  const long long cap = static_cast<long long>(num_sms()) * 4;
  if (gx > cap) gx = cap;
  if (gx < 1) gx = 1;
  const int gy = (m + MT - 1) / MT;
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
  kern<<<grid, threads, smem, st>>>(A, p, m, W, q, n, wpr, e);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int PT, int QT, bool WIDE, bool VEC>
static int launch_mt(const uint64_t* A, int p, int m, const uint64_t* W, int q, int n, int wpr,
                     const EpiParams& e, int mt, cudaStream_t st) {
  switch (mt) {
    case 1: return launch_one<PT, QT, 1, WIDE, VEC>(A, p, m, W, q, n, wpr, e, st);
    case 2: return launch_one<PT, QT, 2, WIDE, VEC>(A, p, m, W, q, n, wpr, e, st);
    case 4: return launch_one<PT, QT, 4, WIDE, VEC>(A, p, m, W, q, n, wpr, e, st);
    default: return launch_one<PT, QT, 8, WIDE, VEC>(A, p, m, W, q, n, wpr, e, st);
  }
}

// Token block: m=1,2 exact; 3-4 -> 4; >4 -> 8, shrunk until the staged
// activation planes fit in 200 KB of shared memory.
static int pick_mt(int m, int p, int wpr) {
  const int wpr2 = (wpr + 1) & ~1;
  int mt = m >= 5 ? 8 : (m >= 3 ? 4 : m);
  while (mt > 1 && static_cast<size_t>(p) * mt * wpr2 * 8 > 200 * 1024) mt >>= 1;
  return mt;
}

int run_gemm_popc(const uint64_t* A, unsigned p, size_t m, const uint64_t* W, unsigned q, size_t n,
                  size_t k, bool wide, const EpiParams& e, cudaStream_t st, int token_tile) {
  if (m == 0 || n == 0) return ABQ_OK;
  const int wpr = static_cast<int>(wpr_of(k));
  const int ip = static_cast<int>(p), iq = static_cast<int>(q);
  const int im = static_cast<int>(m), in = static_cast<int>(n);
  if (static_cast<size_t>(p) * 1 * ((wpr + 1) & ~1) * 8 > 200 * 1024)
    return fail(ABQ_ERR_VALUE, "gemm: K=%zu too large for the staged activation planes", k);
  int mt = pick_mt(im, ip, wpr);
  while (token_tile > 0 && mt > 1 && mt > token_tile) mt >>= 1;  // TileConfig BM cap (abi.cu plan_of)
  const bool vec = (wpr % 2) == 0;
  if (wide) {
    if (vec) return launch_mt<0, 0, true, true>(A, ip, im, W, iq, in, wpr, e, mt, st);
    return launch_mt<0, 0, true, false>(A, ip, im, W, iq, in, wpr, e, mt, st);
  }
  if (!vec) return launch_mt<0, 0, false, false>(A, ip, im, W, iq, in, wpr, e, mt, st);
#define ABQ_PQ(P, Q) \
  if (ip == P && iq == Q) return launch_mt<P, Q, false, true>(A, ip, im, W, iq, in, wpr, e, mt, st)
  ABQ_PQ(8, 2);
  ABQ_PQ(4, 4);
  ABQ_PQ(8, 8);
  ABQ_PQ(4, 2);
  ABQ_PQ(8, 3);
  ABQ_PQ(8, 4);
  ABQ_PQ(6, 6);
  ABQ_PQ(4, 3);
#undef ABQ_PQ
  return launch_mt<0, 0, false, true>(A, ip, im, W, iq, in, wpr, e, mt, st);
}

}  // namespace abq_dev
