// gemm_tc.cu -- K3: prefill GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), sm_100a.
//
// The reference's plane GEMM (include/abq/gemm.hpp:94-146) sums 2^(s+t) x
// popc(A_s & W_t) over p x q binary plane pairs.  sm_100a has no binary
// tensor-core instruction (b1 mma.sync is emulated with 8 IMMA + ~100 ALU
// ops per m16n8k256; measured 700 bit-MAC/clk/SM vs ~8192
// int8 MAC/clk/SM for tcgen05), so the q weight bits are recombined into u8
// codes and one exact u8 x u8 -> s32 UMMA is issued per 32-k step:
//     acc[j][i] = sum_k (sum_t 2^t W_t[j][k]) * a_ik.
//
// Per CTA: 128 output channels (UMMA M) x TT tokens (UMMA N); K streamed in
// 128-wide stages through an S-deep shared-memory ring.  Warp roles:
//   * warp 0 (one thread): TMA producer -- per stage one 1-D bulk copy of the
//     packed weight codes (q x 2 KB) and one of the activation tile (TT x 128
//     bytes, already in the UMMA operand layout, see tc_act_offset); weights
//     of the first S stages are requested before griddepcontrol.wait, i.e.
//     while the ReQuant kernel is still running;
//   * warps 4-7 (q < 8): widen the packed code slices (common.cuh) of one
//     weight row each to u8 codes (q = 4: 1.5 ALU ops per 4 codes) and store
//     them as the UMMA A operand; q = 8 weights are copied by TMA straight
//     into the operand buffer;
//   * warp 1 (one thread): waits for a stage, issues 4 x tcgen05.mma (K = 32)
//     into the TMEM accumulator, tcgen05.commit's the stage back to the
//     producer;
//   * epilogue, all warps: tcgen05.ld (32x32b) -> fused zero-point correction
//     + dequant (gemm.hpp:235-254, 292-306) -> global.
//
// Weight layout ("tc code slices", prepack_tc_kernel): [row-tile 128][k-block
// 128][q][row 128][4 x u32]: row r's 4q words hold its 128 codes of the block
// as code slices; widened register o = 4 kc + u holds k = 16 kc + 4 u + b in
// byte b, stored to the operand at (kc * 128 + r) * 16 (core matrices 8 rows x
// 16 B: LBO 2048 B along K, SBO 128 B along M).  For q = 8 the packed words
// ARE that operand.
#include <cstdlib>

#include "common.cuh"

namespace abq_dev {

unsigned long long*& trace_buffer();

constexpr int kTcM = 128;
constexpr int kTcK = 128;
constexpr int kTcThreads = 512;  // warps 8-15 only join the epilogue
constexpr int kTcColGroups = kTcThreads / 128;  // epilogue: token-column groups per TMEM lane quarter

// ---------------------------------------------------------------------------
// prepack: ABQP [q][n][wpr] -> tc code slices
// ---------------------------------------------------------------------------
__global__ void prepack_tc_kernel(const uint64_t* __restrict__ planes, int q, int n, int k, int wpr,
                                  int rowtiles, int kblocks, uint32_t* __restrict__ out) {
  const size_t total = static_cast<size_t>(rowtiles) * kblocks * q * kTcM * 4;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>((idx >> 2) & (kTcM - 1));
    size_t rest = idx >> 9;
    const int J = static_cast<int>(rest % q) * 4 + static_cast<int>(idx & 3);
    rest /= q;
    const int kb = static_cast<int>(rest % kblocks);
    const int rt = static_cast<int>(rest / kblocks);
    const int grow = rt * kTcM + row;
    const int si = slice_of_bit(q, J >> 2), sw = slice_width(q, si), so = slice_off(q, si);
    const int j = J - 4 * so;
    uint32_t w = 0;
    if (grow < n) {
      for (int s = 0; s < 8 / sw; ++s) {
        const int o = s * 4 * sw + j;  // widened register: k = 16 (o >> 2) + 4 (o & 3) + b
        for (int b = 0; b < 4; ++b) {
          const int kk = kb * kTcK + 16 * (o >> 2) + 4 * (o & 3) + b;
          if (kk >= k) continue;
          for (int e = 0; e < sw; ++e) {
            const uint64_t* src = planes + (static_cast<size_t>(so + e) * n + grow) * wpr;
            w |= static_cast<uint32_t>((src[kk >> 6] >> (kk & 63)) & 1ull) << (8 * b + sw * s + e);
          }
        }
      }
    }
    out[idx] = w;
  }
}

// row-major u8 codes [m][k] (k % 16 == 0, 16-B aligned rows) -> tiled operand
// layout; zero codes past k.  One thread per 16-byte run.
__global__ void tile_codes_kernel(const uint8_t* __restrict__ src, int m, int k, int groups,
                                  uint8_t* __restrict__ dst) {
  const int kp = (k + kTcK - 1) / kTcK * kTcK;
  const size_t runs = static_cast<size_t>(m) * (kp / 16);
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < runs;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int tok = static_cast<int>(idx / (kp / 16)), kk = static_cast<int>(idx % (kp / 16)) * 16;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (kk < k) v = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(tok) * k + kk);
    *reinterpret_cast<uint4*>(dst + tc_act_offset(tok, kk, groups)) = v;
  }
}

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows
// x 16 B, LBO = byte step between core matrices along K, SBO = along M/N;
// version 1 (bit 46) for sm_100.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  const uint32_t mask0 = 0, mask1 = 0, mask2 = 0, mask3 = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(mask0), "r"(mask1), "r"(mask2),
      "r"(mask3));
}

// u8 code register o (k = 16 (o >> 2) + 4 (o & 3) + b in byte b) of one row
// from its 4Q code-slice words: one shift + one mask-merge per slice.
template <int Q>
__device__ __forceinline__ uint32_t widen_row(const uint4 (&w)[Q], int o) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < slice_count(Q); ++i) {
    const int sw = slice_width(Q, i), so = slice_off(Q, i);
    const int J = 4 * so + o % (4 * sw), sh = sw * (o / (4 * sw));
    const uint4 v = w[J >> 2];
    const uint32_t x = (J & 3) == 0 ? v.x : (J & 3) == 1 ? v.y : (J & 3) == 2 ? v.z : v.w;
    const uint32_t m = static_cast<uint32_t>((1u << sw) - 1u) * 0x01010101u;
    r |= so >= sh ? (x << (so - sh)) & (m << so) : (x >> (sh - so)) & (m << so);
  }
  return r;
}

// Epilogue of one CTA tile, one output channel (TMEM lane) and half of the
// token columns per thread, specialised per output mode so the loop body is
// branch-free: 8 accumulators per tcgen05.ld, zero-point correction in
// unsigned 32x32 -> 64-bit products, exact int64 -> double by the 1.5 * 2^52
// magic add (|corr| < 2^51; keeps the conversion unit for the final F2F),
// dequant as RN64(RN64(s_a * s_b) * corr) like gemm.hpp:292-306; all 8 values
// are computed before the (token-bounded) stores.  fp16 results go to a
// [token][channel] shared-memory tile first (written out with 16-byte stores
// by tc_store_f16).
template <int MODE, int TT>
__device__ __forceinline__ void tc_epilogue(const EpiParams& E, uint32_t taddr, int half, int tok0, int m, int ch,
                                            int n, const double* t_sa, const unsigned* t_za, const unsigned* t_kz,
                                            const unsigned* t_ra, __half* stage, int lch, const double* c_sb,
                                            const int* c_zb, const int* c_cs, bool k32) {
  constexpr bool kRaw = MODE == EPI_ACC_I32 || MODE == EPI_ACC_I64;
  const bool chan_ok = ch < n;
  // per-channel values, staged in shared memory during the k-loop (loaded here
  // from global they cost two dependent memory round trips on the tail);
  // |colsum_b|, |u| <= 255 K < 2^31 for K <= 65536
  const double sb = c_sb[lch];
  const int zb = c_zb[lch], cs = c_cs[lch];
  // up to 16 columns per tcgen05.ld; a thread covers TT / kTcColGroups columns
  constexpr int TC = TT / kTcColGroups;
  constexpr int CW = TC >= 16 ? 16 : TC;
#pragma unroll 1
  for (int c0 = half * TC; c0 < (half + 1) * TC; c0 += CW) {
    uint32_t v[CW];
    if constexpr (CW == 4)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                   : "r"(taddr + static_cast<uint32_t>(c0)));
    else if constexpr (CW == 16)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr + static_cast<uint32_t>(c0)));
    else
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
          : "r"(taddr + static_cast<uint32_t>(c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!chan_ok) continue;
    const bool full = tok0 + c0 + CW <= m;  // uniform: no per-token bound in the common case
    const long long o0 = static_cast<long long>(tok0 + c0) * E.ldo + ch;
    if constexpr (kRaw) {
#pragma unroll
      for (int i = 0; i < CW; ++i) {
        // the true sum is < 2^32 (K <= 65536, codes <= 255): exact as unsigned
        if (full || tok0 + c0 + i < m) {
          if constexpr (MODE == EPI_ACC_I32) static_cast<int32_t*>(E.out)[o0 + i * E.ldo] = static_cast<int32_t>(v[i]);
          else static_cast<int64_t*>(E.out)[o0 + i * E.ldo] = static_cast<long long>(v[i]);
        }
      }
    } else {
      // corrected = acc + (K z_a - rowsum_a) z_b - z_a colsum_b.  With K <= 32768
      // the true value is |corr| <= 255^2 K < 2^31, so the sum is computed in
      // wrapping 32-bit arithmetic (two IMADs; exact modulo 2^32, hence exactly);
      // larger K takes the 64-bit products.
      long long corr[CW];
      if (k32) {
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int ti = c0 + i;
          const uint32_t c = v[i] + (t_kz[ti] - t_ra[ti]) * static_cast<uint32_t>(zb) - t_za[ti] * static_cast<uint32_t>(cs);
          corr[i] = static_cast<int>(c);
        }
      } else {
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int ti = c0 + i;
          const unsigned long long plus = static_cast<unsigned long long>(v[i]) +
                                          static_cast<unsigned long long>(t_kz[ti]) * static_cast<unsigned>(zb);
          const unsigned long long minus = static_cast<unsigned long long>(t_za[ti]) * static_cast<unsigned>(cs) +
                                           static_cast<unsigned long long>(t_ra[ti]) * static_cast<unsigned>(zb);
          corr[i] = static_cast<long long>(plus - minus);
        }
      }
      if constexpr (MODE == EPI_CORR_I64) {
#pragma unroll
        for (int i = 0; i < CW; ++i)
          if (full || tok0 + c0 + i < m) static_cast<int64_t*>(E.out)[o0 + i * E.ldo] = corr[i];
      } else {
        double y[CW];
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          // exact int64 -> double (|corr| < 2^51) by the 1.5 * 2^52 magic add
          const double cd = __dsub_rn(__longlong_as_double(0x4338000000000000LL + corr[i]), 6755399441055744.0);
          // (for k32 the compiler sees corr[i] as a sign-extended int32)
          y[i] = __dmul_rn(__dmul_rn(t_sa[c0 + i], sb), cd);
        }
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          if (full || tok0 + c0 + i < m) {
            const long long o = o0 + i * E.ldo;
            if constexpr (MODE == EPI_F64) static_cast<double*>(E.out)[o] = y[i];
            else if constexpr (MODE == EPI_F16) stage[(c0 + i) * kTcM + lch] = __double2half(y[i]);
            else static_cast<float*>(E.out)[o] = __double2float_rn(y[i]);
          }
        }
      }
    }
  }
}

struct TcParams {
  const uint32_t* wtc;  // tc code slices
  const uint8_t* act;   // tiled u8 activation codes (tc_act_offset)
  int q, n, k, m, groups, rowtiles, kblocks;
  EpiParams e;
  unsigned long long* bad_word;  // ReQuant status (~index, 0 = none), published to bad_out
  unsigned long long* bad_out;
  unsigned long long* trace;  // optional [grid][64] clock64 / globaltimer stamps (profiling)
  int dbg;                    // experiments (ABQ_TC_DBG): 2 MMA skips the A wait, 4 no UMMA
};

// Shared memory: an input ring of kS stages -- the packed weights of a
// 128-k block (or, q = 8, the A operand itself) + the activation tile -- that
// the TMA producer keeps full, and (q < 8) a separate 2-deep ring of widened
// u8 A operands.  Keeping the 16 KB widened operand out of the input stage
// makes the input ring ~1.7x deeper for the same shared memory, which is what
// bounds the k-loop (each stage's L2/HBM latency is covered by the stages in
// flight behind it).
template <int Q, int TT>
struct TcShape {
  static constexpr bool kExpand = Q < 8;
  static constexpr int kA = kTcM * kTcK;          // u8 operand A (weights), 16 KB
  static constexpr int kB = TT * kTcK;            // u8 operand B (activations)
  static constexpr int kW = kExpand ? Q * kTcM * 16 : kA;  // packed slices (or A itself)
  static constexpr int kStage = kW + kB;          // one input stage
  static constexpr int kSA = kExpand ? 4 : 0;     // widened-A ring depth (2 k-blocks per widening pass)
  static constexpr int kBudget = 208 * 1024 - kSA * kA;
  static constexpr int kS = kBudget / kStage > 12 ? 12 : kBudget / kStage;
  static constexpr int kSmem = kS * kStage + kSA * kA + 1024;  // + alignment slack
};

template <int Q, int TT>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(const __grid_constant__ TcParams P) {
  using Sh = TcShape<Q, TT>;
  constexpr int S = Sh::kS;
  constexpr int TMEM_COLS = TT <= 32 ? 32 : (TT <= 64 ? 64 : (TT <= 128 ? 128 : 256));
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SA = Sh::kSA > 0 ? Sh::kSA : 1;
  // wbar/abar: stage s weights / activations landed; ebar: MMA done with input
  // stage s; rbar/xbar: widened A slot a filled / free again
  __shared__ __align__(8) uint64_t wbar[S], abar[S], ebar[S], rbar[SA], xbar[SA], done_bar;
  __shared__ uint32_t tmem_base_s;
  // per-token epilogue values, loaded by the otherwise idle warps 2-3:
  // s_a, z_a, K z_a, rowsum_a (all non-negative, < 2^32 for K <= 65536)
  __shared__ double t_sa[TT];
  __shared__ unsigned t_za[TT], t_kz[TT], t_ra[TT];
  __shared__ double c_sb[kTcM];  // per-channel epilogue values (warps 8-11, during the k-loop)
  __shared__ int c_zb[kTcM], c_cs[kTcM];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 7) warm_param_block(P, lane);
  const int rt = blockIdx.x, tok0 = blockIdx.y * TT;
  const int nkb = P.kblocks;
  unsigned long long* trace = P.trace ? P.trace + 64 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (trace && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    trace[0] = clock64();
    trace[8] = g;
  }
  auto w_of = [&](int s) { return smem + s * Sh::kStage; };                  // packed W (q = 8: A)
  auto b_of = [&](int s) { return smem + s * Sh::kStage + Sh::kW; };         // activations
  auto x_of = [&](int a) { return smem + S * Sh::kStage + a * Sh::kA; };     // widened A (q < 8)

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&wbar[s], 1);
      mbar_init(&abar[s], 1);
      mbar_init(&ebar[s], 1);
    }
    for (int a = 0; a < SA; ++a) {
      mbar_init(&rbar[a], 4);  // one arrival per widening warp
      mbar_init(&xbar[a], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_d = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      constexpr uint32_t WB = Sh::kW;
      const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(P.wtc) +
                                  static_cast<size_t>(rt) * nkb * WB;
      const unsigned char* asrc = P.act + static_cast<size_t>(tok0 / 8) * 1024;
      auto issue_w = [&](int kb) {
        const int s = kb % S;
        mbar_expect_tx(&wbar[s], WB);
        bulk_g2s(w_of(s), wsrc + static_cast<size_t>(kb) * WB, WB, &wbar[s]);
      };
      auto issue_a = [&](int kb) {
        const int s = kb % S;
        mbar_expect_tx(&abar[s], Sh::kB);
        bulk_g2s(b_of(s), asrc + static_cast<size_t>(kb) * P.groups * 1024, Sh::kB, &abar[s]);
      };
      const int pre = nkb < S ? nkb : S;
      for (int kb = 0; kb < pre; ++kb) issue_w(kb);
      {  // the rest of this CTA's weights: L2 bulk prefetch, so the ring's later
         // weight copies hit L2 instead of waiting on HBM latency
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        const size_t total = static_cast<size_t>(nkb) * WB;
        for (size_t off = static_cast<size_t>(pre) * WB; off < total; off += 32768)
          asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(wsrc + off),
                       "r"(static_cast<uint32_t>(total - off < 32768 ? total - off : 32768)), "l"(pol)
                       : "memory");
      }
      // the weights do not depend on the preceding ReQuant kernel; its codes do
      // (programmatic dependent launch; a no-op otherwise)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (P.bad_out && blockIdx.x == 0 && blockIdx.y == 0) {
        const unsigned long long w = *P.bad_word;
        *P.bad_out = w ? ~w : ~0ull;
        *P.bad_word = 0ull;
      }
      for (int kb = 0; kb < pre; ++kb) issue_a(kb);
      for (int kb = S; kb < nkb; ++kb) {
        mbar_wait(&ebar[kb % S], ((kb / S) - 1) & 1);  // MMA of kb - S done with the stage
        if (trace && kb < S + 16) trace[48 + kb - S] = clock64();
        issue_w(kb);
        issue_a(kb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: D=s32, A=B=u8, both K-major, N=TT, M=128
      const uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(TT >> 3) << 17) |
                             (static_cast<uint32_t>(kTcM >> 4) << 24);
      // descriptors: the start-address field is the low 14 bits of (addr >> 4)
      // and every operand lies below 256 KB, so a descriptor advances by a
      // plain add of (byte offset >> 4) -- precomputed, the issue loop is a
      // handful of uniform ops per UMMA
      const uint64_t a_base = umma_desc(smem_u32(Sh::kExpand ? x_of(0) : w_of(0)), kTcM * 16, 128);
      const uint64_t b_base = umma_desc(smem_u32(b_of(0)), 128, 1024);
      constexpr uint64_t a_stride = (Sh::kExpand ? Sh::kA : Sh::kStage) >> 4;  // per ring slot
      constexpr uint64_t b_stride = Sh::kStage >> 4;
      constexpr uint64_t a_j = (2 * kTcM * 16) >> 4, b_j = (2 * 128) >> 4;  // per K = 32 step
      int s = 0, a = 0;
      uint32_t ph = 0, pha = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        if (!(P.dbg & 2)) {
          if (Sh::kExpand) mbar_wait(&rbar[a], pha);
          else mbar_wait(&wbar[s], ph);
        }
        mbar_wait(&abar[s], ph);
        tc_fence_after();
        if (trace && kb < 16) trace[32 + kb] = clock64();
        const uint64_t ad = a_base + (Sh::kExpand ? a : s) * a_stride, bd = b_base + s * b_stride;
#pragma unroll
        for (int j = 0; j < kTcK / 32; ++j)
          if (!(P.dbg & 4)) umma_i8(tmem_d, ad + j * a_j, bd + j * b_j, idesc, (kb | j) != 0 ? 1u : 0u);
        tc_commit(&ebar[s]);
        if (Sh::kExpand) tc_commit(&xbar[a]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
        if (++a == SA) {
          a = 0;
          pha ^= 1u;
        }
      }
      tc_commit(&done_bar);
      if (trace) trace[3] = clock64();
    }
  } else if (warp == 2 || warp == 3) {
    const EpiParams& E = P.e;
    if (E.mode != EPI_ACC_I32 && E.mode != EPI_ACC_I64) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // ReQuant results visible
      for (int i = tid - 64; i < TT; i += 64) {
        const int tk = tok0 + i;
        if (tk < P.m) {
          const int za = E.z_a[tk * E.za_stride];
          t_sa[i] = E.s_a[tk * E.sa_stride];
          t_za[i] = static_cast<unsigned>(za);
          t_kz[i] = static_cast<unsigned>(E.k * za);
          t_ra[i] = static_cast<unsigned>(E.rowsum_a[tk]);
        }
      }
    }
  } else if (Sh::kExpand && warp >= 4 && warp < 8) {
    // ---- widen packed code slices of row r into the A operand, two k-blocks
    // per pass (their loads, widening and stores interleave: one k-block per
    // pass left each warp a ~600-cycle dependent chain per k-block, which
    // paced the whole k-loop)
    const int r = tid - 128;
    auto widen_one = [&](int kb, const uint4 (&w)[Q > 0 ? Q : 1]) {
      const int a = kb % SA;
      if (kb >= SA) mbar_wait(&xbar[a], static_cast<uint32_t>(kb / SA - 1) & 1u);  // MMA of kb - SA done
      uint4* adst = reinterpret_cast<uint4*>(x_of(a)) + r;
#pragma unroll
      for (int kc = 0; kc < 8; ++kc)
        adst[kc * kTcM] = make_uint4(widen_row<Q>(w, 4 * kc), widen_row<Q>(w, 4 * kc + 1),
                                     widen_row<Q>(w, 4 * kc + 2), widen_row<Q>(w, 4 * kc + 3));
    };
    auto load_one = [&](int kb, uint4 (&w)[Q > 0 ? Q : 1]) {
      const int s = kb % S;
      mbar_wait(&wbar[s], static_cast<uint32_t>(kb / S) & 1u);
      const uint4* wsl = reinterpret_cast<const uint4*>(w_of(s)) + r;
#pragma unroll
      for (int t = 0; t < Q; ++t) w[t] = wsl[t * kTcM];
    };
    for (int kb = 0; kb < nkb; kb += 2) {
      const bool two = kb + 1 < nkb;
      uint4 w0[Q > 0 ? Q : 1], w1[Q > 0 ? Q : 1];
      load_one(kb, w0);
      if (two) load_one(kb + 1, w1);
      widen_one(kb, w0);
      if (two) widen_one(kb + 1, w1);
      fence_async_smem();  // generic-proxy stores -> visible to the tensor core
      __syncwarp();
      if (trace && tid == 128 && kb < 16) trace[16 + kb] = clock64();
      if (lane == 0) {
        mbar_arrive(&rbar[kb % SA]);
        if (two) mbar_arrive(&rbar[(kb + 1) % SA]);
      }
    }
  }
  if (warp >= 8 && warp < 12) {  // idle during the k-loop: this tile's channel parameters
    const int c = tid - 256, j = rt * kTcM + c;
    const EpiParams& E = P.e;
    const bool ok = j < P.n && E.mode != EPI_ACC_I32 && E.mode != EPI_ACC_I64;
    c_sb[c] = ok ? E.s_b[j * E.sb_stride] : 0.0;
    c_zb[c] = ok ? E.z_b[j * E.zb_stride] : 0;
    c_cs[c] = ok ? static_cast<int>(E.colsum_b[j]) : 0;
  }
  __syncthreads();  // per-token and per-channel values in shared memory

  // ---- epilogue: TMEM -> registers -> zero-point correction + dequant.  A
  // thread owns one output channel (TMEM lane) and half of the token columns,
  // so the per-channel parameters are loaded once.
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  if (trace && tid == 0) trace[4] = clock64();
  const int quarter = warp & 3, half = warp >> 2;
  const int lch = quarter * 32 + lane, ch = rt * kTcM + lch;
  __half* stage = reinterpret_cast<__half*>(smem);  // the operand ring is idle now
  const uint32_t taddr = tmem_d + (static_cast<uint32_t>(quarter * 32) << 16);
  switch (P.e.mode) {
    case EPI_ACC_I32: tc_epilogue<EPI_ACC_I32, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
    case EPI_ACC_I64: tc_epilogue<EPI_ACC_I64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
    case EPI_F64: tc_epilogue<EPI_F64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
    case EPI_F16: tc_epilogue<EPI_F16, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
    case EPI_F32: tc_epilogue<EPI_F32, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
    default: tc_epilogue<EPI_CORR_I64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, P.k <= 32768); break;
  }
  if (trace && tid == 0) trace[6] = clock64();
  if (P.e.mode == EPI_F16) {
    // staged fp16 tile -> global, 8 channels (16 B) per store where aligned
    __syncthreads();
    if (trace && tid == 0) trace[7] = clock64();
    const int rows = min(TT, P.m - tok0), cols = min(kTcM, P.n - rt * kTcM);
    __half* out = static_cast<__half*>(P.e.out);
    const bool vec = (P.e.ldo & 7) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    for (int idx = tid; idx < rows * (kTcM / 8); idx += kTcThreads) {
      const int r = idx / (kTcM / 8), c8 = (idx % (kTcM / 8)) * 8;
      if (c8 >= cols) continue;
      const __half* src = stage + r * kTcM + c8;
      __half* dst = out + static_cast<long long>(tok0 + r) * P.e.ldo + rt * kTcM + c8;
      if (vec && c8 + 8 <= cols) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      } else {
        for (int j = 0; j < 8 && c8 + j < cols; ++j) dst[j] = src[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (trace && tid == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    trace[5] = clock64();
    trace[9] = g;
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(TMEM_COLS));
}

// ============================================================================
// host side
// ============================================================================
size_t tc_words(unsigned q, size_t n, size_t k) {
  const size_t rowtiles = (n + kTcM - 1) / kTcM, kblocks = (k + kTcK - 1) / kTcK;
  return rowtiles * kblocks * q * kTcM * 4;
}

int run_prepack_tc(const uint64_t* planes, unsigned q, size_t n, size_t k, uint32_t* out,
                   cudaStream_t st) {
  const size_t total = tc_words(q, n, k);
  if (total == 0) return ABQ_OK;
  size_t grid = (total + 255) / 256;
  if (grid > static_cast<size_t>(num_sms()) * 32) grid = num_sms() * 32;
  prepack_tc_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(
      planes, static_cast<int>(q), static_cast<int>(n), static_cast<int>(k), static_cast<int>(wpr_of(k)),
      static_cast<int>((n + kTcM - 1) / kTcM), static_cast<int>((k + kTcK - 1) / kTcK), out);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

// row-major codes [m][k] -> tiled operand layout (tc_act_bytes(m, k) bytes)
int run_tile_codes(const uint8_t* src, size_t m, size_t k, uint8_t* dst, cudaStream_t st) {
  if (m == 0) return ABQ_OK;
  const size_t runs = m * ((k + kTcK - 1) / kTcK) * (kTcK / 16);
  size_t grid = (runs + 255) / 256;
  if (grid > static_cast<size_t>(num_sms()) * 16) grid = num_sms() * 16;
  tile_codes_kernel<<<static_cast<unsigned>(grid), 256, 0, st>>>(src, static_cast<int>(m), static_cast<int>(k),
                                                                  tc_act_groups(static_cast<long long>(m)), dst);
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int Q, int TT>
static int launch_tc(const TcParams& P, bool pdl, cudaStream_t st) {
  using Sh = TcShape<Q, TT>;
  auto kern = gemm_tc_kernel<Q, TT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::kSmem);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: smem attribute: %s", cudaGetErrorString(err));
  dim3 grid(static_cast<unsigned>(P.rowtiles), static_cast<unsigned>((P.m + TT - 1) / TT));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = Sh::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  err = cudaLaunchKernelEx(&cfg, kern, P);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int Q>
static int launch_tt(const TcParams& P, bool pdl, cudaStream_t st) {
  if (P.m <= 16) return launch_tc<Q, 16>(P, pdl, st);
  if (P.m <= 32) return launch_tc<Q, 32>(P, pdl, st);
  if (P.m <= 64) return launch_tc<Q, 64>(P, pdl, st);
  if (P.m <= 128) return launch_tc<Q, 128>(P, pdl, st);
  return launch_tc<Q, 256>(P, pdl, st);
}

// k % 16 == 0 (16-byte code runs); the unsigned accumulator is exact to K = 65536
bool gemm_tc_supported(size_t k) { return k > 0 && k <= 65536 && k % 16 == 0; }

// act: tiled u8 codes (tc_act_offset, groups = tc_act_groups(m)), 16-B aligned
int run_gemm_tc(const uint32_t* wtc, unsigned q, size_t n, size_t k, const uint8_t* act, size_t m,
                const EpiParams& e, cudaStream_t st, unsigned long long* bad_word,
                unsigned long long* bad_out, bool pdl) {
  if (m == 0 || n == 0) return ABQ_OK;
  TcParams P{};
  P.bad_word = bad_word;
  P.bad_out = bad_out;
  P.wtc = wtc;
  P.act = act;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.m = static_cast<int>(m);
  P.groups = tc_act_groups(static_cast<long long>(m));
  P.rowtiles = static_cast<int>((n + kTcM - 1) / kTcM);
  P.kblocks = static_cast<int>((k + kTcK - 1) / kTcK);
  P.e = e;
  P.trace = trace_buffer();
  if (const char* env = std::getenv("ABQ_TC_DBG")) P.dbg = std::atoi(env);
  switch (q) {
    case 1: return launch_tt<1>(P, pdl, st);
    case 2: return launch_tt<2>(P, pdl, st);
    case 3: return launch_tt<3>(P, pdl, st);
    case 4: return launch_tt<4>(P, pdl, st);
    case 5: return launch_tt<5>(P, pdl, st);
    case 6: return launch_tt<6>(P, pdl, st);
    case 7: return launch_tt<7>(P, pdl, st);
    default: return launch_tt<8>(P, pdl, st);
  }
}

}  // namespace abq_dev
