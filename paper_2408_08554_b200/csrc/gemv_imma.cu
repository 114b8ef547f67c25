// gemv_imma.cu -- K2 "recombination" variant: decode GEMV (M <= 8 tokens per
// token block) that feeds the weight BIT PLANES to the int8 tensor pipe, one
// plane at a time, against u8 activation codes.  sm_100a.
//
// Why (measured in profiles/r01_microbench_pipes.txt): on
// sm_100a POPC issues at 16/clk/SM, so the AND+popcount decomposition of a
// p-bit activation x q-bit weight product needs p POPCs per 32 weight-plane
// bits -- 36% of HBM at p=8.  The int8 tensor pipe (legacy IMMA m16n8k32,
// ~1950 MAC/clk/SM) is idle in that kernel.  Here each 32-bit weight-plane
// word is expanded to 0/128 bytes with one shift + one AND (fma and alu pipes)
// and multiplied on the tensor pipe against the activation codes:
//
//   acc = sum_t 2^t * sum_k a_k * W_t[k]        (paper Eq. 11 with the
//                                                 activation planes recombined)
//
// which is the same exact unsigned code product as the reference's
// gemm_plane_rows (include/abq/gemm.hpp:94-146).  Accumulation is exact:
// every IMMA partial is an integer < 2^31 and planes are combined after the
// 2^-7 scale is divided out exactly.
//
// Weight layout ("fragment-major planes", built once by prepack_frag_kernel
// from the ABQP planes): [row-tile of 16][k-block of 256][plane][lane][4 x u32].
// Lane l = (g = l/4, tig = l%4) holds exactly the bits its IMMA A fragments
// need for the 8 k32 chunks of the block; bit (8b + c) of word u is element
// (row g + 8*(u&1), k = 32c + 16*(u>>1) + 4*tig + b), so chunk c's register
// is (w << (7 - c)) & 0x80808080.  Same byte count as ABQP; each (tile, block)
// is q x 512 contiguous bytes: one coalesced 16-byte load per lane per plane.
//
// Work split (persistent, stream-K): the (row-tile, k-block) units are split
// evenly over all CTAs and warps; partial row-tile sums meet in shared memory
// (64-bit atomics) and, for row-tiles cut between CTAs, in a self-cleaning
// global accumulator where the last contributing CTA runs the epilogue.
// The prologue ReQuantizes the fp16 activations (or recombines given planes)
// into shared memory while the first weight loads are in flight.
#include "common.cuh"
#include "quant_dev.cuh"

namespace abq_dev {

constexpr int kRowTile = 16;
constexpr int kKBlock = 256;
constexpr int kImmaThreads = 512;

// ---------------------------------------------------------------------------
// prepack: ABQP [q][n][wpr] -> fragment-major [rt][kb][q][lane][4]
// ---------------------------------------------------------------------------
__global__ void prepack_frag_kernel(const uint64_t* __restrict__ planes, int q, int n, int k, int wpr,
                                    int rowtiles, int kblocks, uint32_t* __restrict__ frag) {
  const size_t total = static_cast<size_t>(rowtiles) * kblocks * q * 128;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int u = static_cast<int>(idx & 3);
    const int lane = static_cast<int>((idx >> 2) & 31);
    size_t rest = idx >> 7;
    const int t = static_cast<int>(rest % q);
    rest /= q;
    const int kb = static_cast<int>(rest % kblocks);
    const int rt = static_cast<int>(rest / kblocks);
    const int g = lane >> 2, tig = lane & 3;
    const int row = rt * kRowTile + g + 8 * (u & 1);
    const int kbase = kb * kKBlock + 16 * (u >> 1) + 4 * tig;
    uint32_t w = 0;
    if (row < n) {
      const uint64_t* src = planes + (static_cast<size_t>(t) * n + row) * wpr;
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kk = kbase + 32 * c + b;
          if (kk < k) w |= static_cast<uint32_t>((src[kk >> 6] >> (kk & 63)) & 1ull) << (8 * b + c);
        }
    }
    frag[idx] = w;
  }
}

// ---------------------------------------------------------------------------
// main kernel
// ---------------------------------------------------------------------------
struct ImmaParams {
  const uint32_t* frag;
  int q, n, k, rowtiles, kblocks;
  int m;  // total tokens
  // activations: either float x (+ quant params) or packed planes
  const void* x;
  QuantParams qp;
  const uint64_t* a_planes;
  int p;
  int wpr_a;
  EpiParams e;
  long long* gacc;  // [tokblocks][rowtiles][16][8] int64, zero on entry and exit
  unsigned* gcnt;   // [tokblocks][rowtiles], zero on entry and exit
  unsigned long long* bad;
};

__device__ __forceinline__ void imma_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ld_frag(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// CTA that owns unit u under the even split (c*U)/G
__device__ __forceinline__ int cta_of_unit(long long u, long long U, int G) {
  return static_cast<int>(((u + 1) * G - 1) / U);
}

// SRC: 0 = activation planes, 1 = fp16 x, 2 = fp32 x, 3 = fp64 x
template <int QT, int MT, int SRC, int PF>
__global__ void __launch_bounds__(kImmaThreads, 1) gemv_imma_kernel(ImmaParams P) {
  constexpr int QMAX = QT > 0 ? QT : 8;
  const int q = QT > 0 ? QT : P.q;
  extern __shared__ __align__(16) unsigned char smem[];
  const int kpad = P.kblocks * kKBlock;
  uint32_t* act = reinterpret_cast<uint32_t*>(smem);  // MT * kpad bytes
  const int G = gridDim.x;
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  const bool stream_k = P.gacc != nullptr;
  // CTA unit range
  long long U0, U1;
  if (stream_k) {
    U0 = blockIdx.x * U / G;
    U1 = (blockIdx.x + 1) * U / G;
  } else {  // row-tile granular split: no row-tile shared between CTAs
    U0 = static_cast<long long>(blockIdx.x * static_cast<long long>(P.rowtiles) / G) * P.kblocks;
    U1 = static_cast<long long>((blockIdx.x + 1) * static_cast<long long>(P.rowtiles) / G) * P.kblocks;
  }
  const int rt_first = static_cast<int>(U0 / P.kblocks);
  const int rt_last = U1 > U0 ? static_cast<int>((U1 - 1) / P.kblocks) : rt_first - 1;
  const int nlrt = rt_last - rt_first + 1;
  long long* accs = reinterpret_cast<long long*>(smem + static_cast<size_t>(MT) * kpad);  // [nlrt][16][MT]
  double* s_sa = reinterpret_cast<double*>(accs + static_cast<size_t>(max(nlrt, 0)) * 16 * MT);
  long long* s_za = reinterpret_cast<long long*>(s_sa + MT);
  long long* s_ra = s_za + MT;
  double* s_lo = reinterpret_cast<double*>(s_ra + MT);  // [16 warps][MT]
  double* s_hi = s_lo + 16 * MT;
  long long* s_sum = reinterpret_cast<long long*>(s_hi + 16 * MT);  // [16][MT]
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int tok0 = blockIdx.y * MT;
  const int mb = min(MT, P.m - tok0);

  // ---- warp unit range and the first weight loads (in flight during the prologue)
  const long long wu0 = U0 + (U1 - U0) * warp / 16;
  const long long wu1 = U0 + (U1 - U0) * (warp + 1) / 16;
  const size_t unit_words = static_cast<size_t>(q) * 128;
  uint4 ring[PF + 1][QMAX];
#pragma unroll
  for (int s = 0; s < PF; ++s) {
    const long long uu = wu0 + s;
#pragma unroll
    for (int t = 0; t < QMAX; ++t)
      if (t < q && uu < wu1) ring[s][t] = ld_frag(P.frag + uu * unit_words + t * 128 + lane * 4);
  }

  // ---- prologue: activations -> u8 codes in smem, fragment layout
  // u32 index of (kb, c, h, tok i, tig): (((kb*8 + c)*MT + i)*4 + tig)*2 + h
  for (int idx = tid; idx < MT * kpad / 4; idx += kImmaThreads) act[idx] = 0u;
  for (int idx = tid; idx < nlrt * 16 * MT; idx += kImmaThreads) accs[idx] = 0;
  // only CTA (0, y=0) reports non-finite inputs; it owns the status word
  if (SRC != 0 && P.bad && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *P.bad = ~0ull;
  __syncthreads();
  const int ngroups = (P.k + 3) / 4;
  if (SRC == 0) {
    for (int idx = tid; idx < mb * ngroups; idx += kImmaThreads) {
      const int i = idx / ngroups, v = idx % ngroups;
      const int tok = tok0 + i;
      uint32_t word = 0;
      for (int s = 0; s < P.p; ++s) {
        const uint64_t pw = P.a_planes[(static_cast<size_t>(s) * P.m + tok) * P.wpr_a + (v >> 4)];
        const uint32_t nib = static_cast<uint32_t>(pw >> ((v & 15) * 4)) & 0xFu;
        word |= ((nib * 0x00204081u) & 0x01010101u) << s;
      }
      const int kb = v >> 6, rem = v & 63;
      act[((((kb * 8 + (rem >> 3)) * MT + i) * 4 + (rem & 3)) * 2) + ((rem >> 2) & 1)] = word;
    }
  } else {
    // ReQuant (quantizer.hpp:146-213), per-token (or per-tensor) asymmetric/symmetric/balanced
    double lo[MT], hi[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      lo[i] = CUDART_INF;
      hi[i] = -CUDART_INF;
    }
    auto scan = [&](int tok, double& l, double& h) {
      for (int j = tid; j < P.k; j += kImmaThreads) {
        double v;
        if (SRC == 1) v = load_as_double(static_cast<const __half*>(P.x), static_cast<size_t>(tok) * P.k + j);
        else if (SRC == 2) v = load_as_double(static_cast<const float*>(P.x), static_cast<size_t>(tok) * P.k + j);
        else v = load_as_double(static_cast<const double*>(P.x), static_cast<size_t>(tok) * P.k + j);
        if (!isfinite(v) && blockIdx.x == 0 && blockIdx.y == 0 && P.bad)
          atomicMin(P.bad, static_cast<unsigned long long>(tok) * P.k + j);
        l = fmin(l, v);
        h = fmax(h, v);
      }
    };
    if (P.qp.per_tensor) {  // one range over every token (quantizer.hpp:116-129)
      for (int tok = 0; tok < P.m; ++tok) scan(tok, lo[0], hi[0]);
    } else {
#pragma unroll
      for (int i = 0; i < MT; ++i)
        if (i < mb) scan(tok0 + i, lo[i], hi[i]);
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const double l = warp_min(lo[i]), h = warp_max(hi[i]);
      if (lane == 0) {
        s_lo[warp * MT + i] = l;
        s_hi[warp * MT + i] = h;
      }
    }
    __syncthreads();
    if (tid < MT) {
      const int i = P.qp.per_tensor ? 0 : tid;
      double l = CUDART_INF, h = -CUDART_INF;
      for (int w = 0; w < 16; ++w) {
        l = fmin(l, s_lo[w * MT + i]);
        h = fmax(h, s_hi[w * MT + i]);
      }
      double step;
      int z;
      group_params(P.qp, l, h, &step, &z);
      s_sa[tid] = step;
      s_za[tid] = z;
    }
    __syncthreads();
    long long rsum[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) rsum[i] = 0;
    const double top = static_cast<double>(P.qp.levels - 1);
    for (int idx = tid; idx < mb * ngroups; idx += kImmaThreads) {
      const int i = idx / ngroups, v = idx % ngroups;
      const int tok = tok0 + i;
      const double step = s_sa[i], zd = static_cast<double>(s_za[i]);
      const double inv = 1.0 / step;
      uint32_t word = 0;
      unsigned sum = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = 4 * v + b;
        if (j < P.k) {
          double x;
          if (SRC == 1) x = load_as_double(static_cast<const __half*>(P.x), static_cast<size_t>(tok) * P.k + j);
          else if (SRC == 2) x = load_as_double(static_cast<const float*>(P.x), static_cast<size_t>(tok) * P.k + j);
          else x = load_as_double(static_cast<const double*>(P.x), static_cast<size_t>(tok) * P.k + j);
          const unsigned c = quant_code_fast(x, step, inv, zd, top);
          sum += c;
          word |= c << (8 * b);
        }
      }
#pragma unroll
      for (int ii = 0; ii < MT; ++ii)
        if (ii == i) rsum[ii] += sum;
      const int kb = v >> 6, rem = v & 63;
      act[((((kb * 8 + (rem >> 3)) * MT + i) * 4 + (rem & 3)) * 2) + ((rem >> 2) & 1)] = word;
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const long long r = warp_sum(rsum[i]);
      if (lane == 0) s_sum[warp * MT + i] = r;
    }
    __syncthreads();
    if (tid < MT) {
      long long r = 0;
      for (int w = 0; w < 16; ++w) r += s_sum[w * MT + tid];
      s_ra[tid] = r;
    }
  }
  __syncthreads();

  // ---- main loop over this warp's (row-tile, k-block) units
  int acc[QMAX][4];
#pragma unroll
  for (int t = 0; t < QMAX; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;
  int cur_rt = wu0 < wu1 ? static_cast<int>(wu0 / P.kblocks) : -1;
  const uint2* act2 = reinterpret_cast<const uint2*>(act);

  auto flush = [&](int rt) {
    const int lrt = rt - rt_first;
    long long v[4] = {0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < QMAX; ++t)
      if (t < q) {
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] += static_cast<long long>(acc[t][r] >> 7) << t;
      }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = g + 8 * (r >> 1), tok = 2 * tig + (r & 1);
      if (tok < mb) atomicAdd(reinterpret_cast<unsigned long long*>(&accs[(lrt * 16 + row) * MT + tok]),
                              static_cast<unsigned long long>(v[r]));
    }
#pragma unroll
    for (int t = 0; t < QMAX; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;
  };

  for (long long u = wu0; u < wu1; u += PF + 1) {
#pragma unroll
    for (int s = 0; s <= PF; ++s) {
      const long long uu = u + s;
      if (uu < wu1) {
        // issue the load PF units ahead into the slot freed last iteration
        const long long un = uu + PF;
        const int slot_n = (s + PF) % (PF + 1);
        if (un < wu1) {
#pragma unroll
          for (int t = 0; t < QMAX; ++t)
            if (t < q) ring[slot_n][t] = ld_frag(P.frag + un * unit_words + t * 128 + lane * 4);
        }
        const int rt = static_cast<int>(uu / P.kblocks);
        const int kb = static_cast<int>(uu % P.kblocks);
        if (rt != cur_rt) {
          flush(cur_rt);
          cur_rt = rt;
        }
        const uint2* ab = act2 + static_cast<size_t>(kb) * 8 * MT * 4;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint2 b = make_uint2(0u, 0u);
          if (g < MT) b = ab[(c * MT + g) * 4 + tig];
#pragma unroll
          for (int t = 0; t < QMAX; ++t) {
            if (t < q) {
              const uint4 w = ring[s][t];
              const uint32_t a0 = (w.x << (7 - c)) & 0x80808080u;
              const uint32_t a1 = (w.y << (7 - c)) & 0x80808080u;
              const uint32_t a2 = (w.z << (7 - c)) & 0x80808080u;
              const uint32_t a3 = (w.w << (7 - c)) & 0x80808080u;
              imma_16832(acc[t], a0, a1, a2, a3, b.x, b.y);
            }
          }
        }
      }
    }
  }
  if (cur_rt >= 0) flush(cur_rt);
  __syncthreads();

  // ---- epilogue per local row-tile
  const int base_blk = blockIdx.y * P.rowtiles;
  for (int lrt = 0; lrt < nlrt; ++lrt) {
    const int rt = rt_first + lrt;
    const long long ufirst = static_cast<long long>(rt) * P.kblocks;
    const long long ulast = ufirst + P.kblocks - 1;
    const int contributors = stream_k ? cta_of_unit(ulast, U, G) - cta_of_unit(ufirst, U, G) + 1 : 1;
    if (contributors == 1) {
      for (int idx = tid; idx < 16 * mb; idx += kImmaThreads) {
        const int row = idx / mb, i = idx % mb;
        const int j = rt * kRowTile + row;
        if (j < P.n) {
          const long long a = accs[(lrt * 16 + row) * MT + i];
          if (SRC == 0) epi_store(P.e, tok0 + i, j, a);
          else epi_store_v(P.e, tok0 + i, j, a, s_sa[P.qp.per_tensor ? 0 : i],
                           s_za[P.qp.per_tensor ? 0 : i], s_ra[i]);
        }
      }
    } else {
      long long* gslot = P.gacc + (static_cast<size_t>(base_blk) + rt) * 16 * 8;
      for (int idx = tid; idx < 16 * mb; idx += kImmaThreads) {
        const int row = idx / mb, i = idx % mb;
        atomicAdd(reinterpret_cast<unsigned long long*>(&gslot[row * 8 + i]),
                  static_cast<unsigned long long>(accs[(lrt * 16 + row) * MT + i]));
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const unsigned old = atomicAdd(&P.gcnt[base_blk + rt], 1u);
        s_last = old == static_cast<unsigned>(contributors - 1);
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int idx = tid; idx < 16 * mb; idx += kImmaThreads) {
          const int row = idx / mb, i = idx % mb;
          const long long a = static_cast<long long>(
              atomicExch(reinterpret_cast<unsigned long long*>(&gslot[row * 8 + i]), 0ull));
          const int j = rt * kRowTile + row;
          if (j < P.n) {
            if (SRC == 0) epi_store(P.e, tok0 + i, j, a);
            else epi_store_v(P.e, tok0 + i, j, a, s_sa[P.qp.per_tensor ? 0 : i],
                             s_za[P.qp.per_tensor ? 0 : i], s_ra[i]);
          }
        }
        if (tid == 0) P.gcnt[base_blk + rt] = 0u;
      }
      __syncthreads();
    }
  }
}

// ============================================================================
// host side
// ============================================================================
size_t frag_words(unsigned q, size_t n, size_t k) {
  const size_t rowtiles = (n + kRowTile - 1) / kRowTile, kblocks = (k + kKBlock - 1) / kKBlock;
  return rowtiles * kblocks * q * 128;
}

size_t imma_gacc_bytes(size_t m, size_t n) {
  const size_t rowtiles = (n + kRowTile - 1) / kRowTile, tokblocks = (m + 7) / 8;
  return tokblocks * rowtiles * (16 * 8 * sizeof(long long) + sizeof(unsigned));
}

int run_prepack_frag(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* frag,
                     cudaStream_t st) {
  const size_t total = frag_words(q, n, k);
  if (total == 0) return ABQ_OK;
  const int rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  const int kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  size_t grid = (total + 255) / 256;
  if (grid > static_cast<size_t>(num_sms()) * 32) grid = num_sms() * 32;
  prepack_frag_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
      planes, static_cast<int>(q), static_cast<int>(n), static_cast<int>(k),
      static_cast<int>(wpr_of(k)), rowtiles, kblocks, frag);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int QT, int MT, int SRC>
static int launch_imma(ImmaParams P, int grid_x, int grid_y, cudaStream_t st) {
  constexpr int QQ = QT > 0 ? QT : 8;
  constexpr int PF = QQ <= 2 ? 3 : (QQ <= 4 ? 2 : 1);
  auto kern = gemv_imma_kernel<QT, MT, SRC, PF>;
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  const long long per_cta_units = (U + grid_x - 1) / grid_x + P.kblocks;
  const int nlrt_max = static_cast<int>(per_cta_units / P.kblocks + 2);
  const size_t smem = static_cast<size_t>(MT) * P.kblocks * kKBlock +
                      static_cast<size_t>(nlrt_max) * 16 * MT * 8 + MT * (8 + 8 + 8) +
                      2 * 16 * MT * 8 + 16 * MT * 8;
  if (smem > 227 * 1024) return fail(ABQ_ERR_VALUE, "gemv_imma: shared memory plan too large (%zu B)", smem);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_imma: smem attribute: %s", cudaGetErrorString(err));
  kern<<<dim3(grid_x, grid_y), kImmaThreads, smem, st>>>(P);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int MT, int SRC>
static int launch_q(ImmaParams P, int gx, int gy, cudaStream_t st) {
  switch (P.q) {
    case 1: return launch_imma<1, MT, SRC>(P, gx, gy, st);
    case 2: return launch_imma<2, MT, SRC>(P, gx, gy, st);
    case 3: return launch_imma<3, MT, SRC>(P, gx, gy, st);
    case 4: return launch_imma<4, MT, SRC>(P, gx, gy, st);
    case 8: return launch_imma<8, MT, SRC>(P, gx, gy, st);
    default: return launch_imma<0, MT, SRC>(P, gx, gy, st);
  }
}

template <int SRC>
static int launch_mt(ImmaParams P, int mt, int gx, int gy, cudaStream_t st) {
  switch (mt) {
    case 1: return launch_q<1, SRC>(P, gx, gy, st);
    case 2: return launch_q<2, SRC>(P, gx, gy, st);
    case 4: return launch_q<4, SRC>(P, gx, gy, st);
    default: return launch_q<8, SRC>(P, gx, gy, st);
  }
}

static int pick_imma_mt(int m, int kblocks) {
  int mt = m >= 5 ? 8 : (m >= 3 ? 4 : m);
  while (mt > 1 && static_cast<size_t>(mt) * kblocks * kKBlock > 160 * 1024) mt >>= 1;
  return mt;
}

// K supported by the activation smem plan (mt=1): up to 160 KB of codes
bool imma_supported(size_t m, size_t k) {
  (void)m;
  return k > 0 && ((k + kKBlock - 1) / kKBlock) * kKBlock <= 160 * 1024;
}

// x_dtype < 0: activations come from planes (a_planes/p), else from float x.
int run_gemv_imma(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const void* x,
                  int x_dtype, const QuantParams* qp, const uint64_t* a_planes, unsigned p,
                  const EpiParams& e, long long* gacc, unsigned* gcnt, unsigned long long* bad,
                  cudaStream_t st) {
  if (m == 0 || n == 0) return ABQ_OK;
  ImmaParams P{};
  P.frag = frag;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  P.kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  P.m = static_cast<int>(m);
  P.x = x;
  if (qp) P.qp = *qp;
  P.a_planes = a_planes;
  P.p = static_cast<int>(p);
  P.wpr_a = static_cast<int>(wpr_of(k));
  P.e = e;
  P.gacc = reinterpret_cast<long long*>(gacc);
  P.gcnt = gcnt;
  P.bad = bad;
  const int mt = pick_imma_mt(static_cast<int>(m), P.kblocks);
  const int gy = static_cast<int>((m + mt - 1) / mt);
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  int gx;
  if (gacc) {
    // stream-K over units; keep >= 16 units (one per warp) per CTA
    gx = static_cast<int>(std::min<long long>(num_sms(), std::max<long long>(1, U / 16)));
  } else {
    gx = std::min(num_sms(), P.rowtiles);
  }
  if (gacc && mt != 8 && gy > 1) return fail(ABQ_ERR_VALUE, "gemv_imma: token blocking needs mt=8");
  if (x_dtype < 0) return launch_mt<0>(P, mt, gx, gy, st);
  if (x_dtype == ABQ_F16) return launch_mt<1>(P, mt, gx, gy, st);
  if (x_dtype == ABQ_F32) return launch_mt<2>(P, mt, gx, gy, st);
  return launch_mt<3>(P, mt, gx, gy, st);
}

}  // namespace abq_dev
