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
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace abq_dev {

unsigned long long*& trace_buffer();

constexpr int kTcM = 128;
constexpr int kTcK = 128;
constexpr int kTcThreads = 512;  // warps 8-15 only join the epilogue
constexpr int kTcColGroups = kTcThreads / 128;
constexpr int kTcIssuers = 3;  // MMA-issuing threads (lane 0 of warps 1 .. kTcIssuers)
// ABQ_GEMM_AUTO picks stream-K when the one-CTA-per-row-tile grid leaves at
// least half the SMs idle (2 x row-tiles <= SMs): measured with
// abq.autotune_linear (profiles/r01_tune_sweep.csv), stream-K is 17-18 %
// faster at N <= 4096 with K = 11008 or M = 256 and ties at K = 4096, while
// at N = 11008 (86 row-tiles) the partial-tile hand-off costs more than the
// 62 idle SMs.
inline bool tc_stream_k_auto(int rowtiles) { return 2 * rowtiles <= num_sms(); }  // epilogue: token-column groups per TMEM lane quarter

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

// same with A in tensor memory ([a_tmem]: 128 lanes = rows, K = 32 u8 in 8 columns)
__device__ __forceinline__ void umma_i8_tmem_a(uint32_t tmem_d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  const uint32_t mask0 = 0, mask1 = 0, mask2 = 0, mask3 = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(mask0), "r"(mask1), "r"(mask2),
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
                                            const int* c_zb, const int* c_cs, bool k32, const uint32_t* part,
                                            int npart, int dbg) {
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
    if (dbg & 128) {  // timing experiment (results invalid): the accumulator loads dropped
#pragma unroll
      for (int i = 0; i < CW; ++i) v[i] = static_cast<uint32_t>(i);
    }
    if (dbg & 64) {  // timing experiment (results invalid): no correction / dequant math
      if (chan_ok && MODE == EPI_F16)
#pragma unroll
        for (int i = 0; i < CW; ++i) stage[(c0 + i) * kTcM + lch] = __ushort_as_half(static_cast<unsigned short>(v[i]));
      continue;
    }
    // stream-K: the k-ranges of this tile other CTAs accumulated (exact
    // modulo 2^32 like the accumulator itself)
    for (int c = 0; c < npart; ++c)
#pragma unroll
      for (int i = 0; i < CW; ++i) v[i] += __ldcg(part + (c * TT + c0 + i) * kTcM + lch);
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

// stream-K contributor: this CTA's partial accumulator of a tile -> global
// [column][channel] (coalesced along the TMEM lanes), read back by the tile's
// finisher CTA.
template <int TT>
__device__ __forceinline__ void tc_store_partial(uint32_t taddr, int half, int lch, uint32_t* part) {
  constexpr int TC = TT / kTcColGroups;
  constexpr int CW = TC >= 16 ? 16 : (TC >= 8 ? 8 : 4);
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
#pragma unroll
    for (int i = 0; i < CW; ++i) __stcg(part + (c0 + i) * kTcM + lch, v[i]);
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
  int pre_w;                  // weight stages requested before griddepcontrol.wait (the rest behind the activations)
  int dbg;                    // experiments (abq_set_tuning "tc_dbg"): 2 MMA skips the A wait, 4 no UMMA,
                              // 8 no activation TMA, 16 no weight TMA, 32 no widening (results invalid)
  // stream-K (one token tile, grid < rowtiles x kblocks units): CTA b owns the
  // units [b T / G, (b + 1) T / G) of the (row-tile, k-block) sequence; a
  // tile's finisher is the CTA holding its last k-block, its contributors
  // (at most 2) publish partial accumulators + a flag.  Flags are zero
  // between launches (the finisher resets them).
  int sk;
  unsigned* sk_flags;  // [rowtiles][sk_slots]
  uint32_t* sk_part;   // [rowtiles][sk_slots][TT][128]
  int sk_slots;        // CTAs that can share one tile (tc_sk_slots)
};

// stream-K workspace: flags (zero-filled once by the caller, at an offset that
// does not depend on m) and partial tiles (no initial value needed)
// abq_set_gemm_schedule (ABQ_GEMM_AUTO / CLASSIC / STREAM_K)
int& gemm_schedule() {
  static int s = 0;
  return s;
}

// Stream-K grid: G = min(SMs, c x rowtiles, T) CTAs for T = rowtiles x kblocks
// units, c = tc_sk_ctas (abq_set_tuning "tc_sk_ctas", default 2).  G >= rowtiles
// keeps every CTA's range <= kblocks: <= 2 segments, the first finishing a
// tile, the last contributing to one.  A tile is shared by at most
// ceil(kblocks / floor(T / G)) + 1 CTAs: its slots in the flag and
// partial-tile arrays.  Measured (profiles/r02_gemm_n4096.txt): every SM
// (c = 5 at N = 4096) halves the k-loop but the finisher then sums 4-5
// partial tiles from L2 on its tail (o_proj M=128 17.7 -> 21.7 us), so c = 2.
constexpr size_t kSkMaxRowtiles = 160;
int tc_sk_grid(long long rowtiles, long long kblocks) {
  const long long c = std::max(2, dec_tuning().tc_sk_ctas);
  return static_cast<int>(std::min<long long>(std::min<long long>(num_sms(), c * rowtiles), rowtiles * kblocks));
}
int tc_sk_slots(size_t n, size_t k) {
  const long long rt = static_cast<long long>((n + kTcM - 1) / kTcM), kb = static_cast<long long>((k + kTcK - 1) / kTcK);
  const long long T = rt * kb, G = tc_sk_grid(rt, kb);
  if (G <= 0) return 2;
  const long long per = std::max<long long>(1, T / G);
  return static_cast<int>(std::max<long long>(2, (kb + per - 1) / per + 1));
}
size_t tc_sk_flag_bytes(size_t n, size_t k) { return (n + kTcM - 1) / kTcM * tc_sk_slots(n, k) * 4; }
// stream-K only runs with fewer row-tiles than SMs; layers wider than this
// never need partial tiles (keeps the per-layer workspace small)
size_t tc_sk_part_bytes(size_t m, size_t n, size_t k) {
  if (m == 0 || m > 256 || (n + kTcM - 1) / kTcM > kSkMaxRowtiles) return 0;
  const size_t tt = m <= 16 ? 16 : m <= 32 ? 32 : m <= 64 ? 64 : m <= 128 ? 128 : 256;
  return (n + kTcM - 1) / kTcM * tc_sk_slots(n, k) * tt * kTcM * 4;
}

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
  // widened A in tensor memory (tcgen05.st from the widening warps, UMMA
  // reads A from TMEM): takes the 16 KB store + 16 KB UMMA read per k-block
  // off the 128 B/clk shared-memory port that bounds the k-loop.  Needs
  // 2 TT accumulator + 4 x 32 operand columns <= 512.
  static constexpr bool kTmemA = kExpand && TT <= 128;
  static constexpr int kXA = kExpand ? (kTmemA ? 8 : 4) : 0;  // widened-A ring depth (2 k-blocks per widening pass)
  static constexpr int kWG = kTmemA ? 2 : 1;                  // widening warp groups (4 warps = 128 rows each)
  static constexpr int kSA = kTmemA ? 0 : kXA;               // ... of it in shared memory
  static constexpr int kBudget = 208 * 1024 - kSA * kA;
  static constexpr int kS = kBudget / kStage > 12 ? 12 : kBudget / kStage;
  static constexpr int kSmem = kS * kStage + kSA * kA + 1024;  // + alignment slack
};

template <int Q, int TT>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(const __grid_constant__ TcParams P) {
  using Sh = TcShape<Q, TT>;
  constexpr int S = Sh::kS;
  // two accumulators (a stream-K CTA's range touches at most two tiles)
  constexpr int TMEM_NEED = 2 * TT + (Sh::kTmemA ? Sh::kXA * 32 : 0);
  constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : (TMEM_NEED <= 64 ? 64 : (TMEM_NEED <= 128 ? 128 : (TMEM_NEED <= 256 ? 256 : 512)));
  constexpr uint32_t TMEM_A = 2 * TT;  // first column of the widened-A ring (kTmemA)
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int SA = Sh::kXA > 0 ? Sh::kXA : 1;
  // wbar/abar: stage s weights / activations landed; ebar: MMA done with input
  // stage s; rbar/xbar: widened A slot a filled / free again
  __shared__ __align__(8) uint64_t wbar[S], abar[S], ebar[S], rbar[SA], xbar[SA], done_bar;
  __shared__ uint32_t tmem_base_s;
  // per-token epilogue values, loaded by the otherwise idle warps 12-15:
  // s_a, z_a, K z_a, rowsum_a (all non-negative, < 2^32 for K <= 65536)
  __shared__ double t_sa[TT];
  __shared__ unsigned t_za[TT], t_kz[TT], t_ra[TT];
  __shared__ double c_sb[kTcM];  // per-channel epilogue values (warps 8-11, during the k-loop)
  __shared__ int c_zb[kTcM], c_cs[kTcM];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 7) warm_param_block(P, lane);
  const int tok0 = blockIdx.y * TT;
  const int nkb = P.kblocks;
  // this CTA's units u = row-tile x nkb + k-block: [U0, U0 + nU), split into
  // <= 2 segments at a row-tile boundary (seg0 = [U0, U0 + n0))
  int U0, nU;
  if (P.sk) {
    const long long T = static_cast<long long>(P.rowtiles) * nkb, G = gridDim.x;
    U0 = static_cast<int>(blockIdx.x * T / G);
    nU = static_cast<int>((blockIdx.x + 1) * T / G) - U0;
  } else {
    U0 = blockIdx.x * nkb;
    nU = nkb;
  }
  const int t0 = U0 / nkb, n0 = min(nU, (t0 + 1) * nkb - U0);
  const int nseg = n0 < nU ? 2 : 1;
  // the (single) tile this CTA finishes, -1 if none
  const int fin_seg = U0 + n0 == (t0 + 1) * nkb ? 0 : (nseg == 2 && U0 + nU == (t0 + 2) * nkb ? 1 : -1);
  const int rt = fin_seg < 0 ? -1 : t0 + fin_seg;
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
    mbar_init(&done_bar, kTcIssuers);  // one commit per MMA-issuing thread
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
  if (warp >= 12) {
    // zero both accumulators (the two MMA-issuing threads always accumulate,
    // so neither has to go first)
    const uint32_t tz = tmem_d + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    const uint32_t z = 0u;
#pragma unroll 1
    for (int c = 0; c < 2 * TT; c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tz + c),
          "r"(z)
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      constexpr uint32_t WB = Sh::kW;
      const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(P.wtc) +
                                  static_cast<size_t>(U0) * WB;
      const unsigned char* asrc = P.act + static_cast<size_t>(tok0 / 8) * 1024;
      auto issue_w = [&](int kb) {
        const int s = kb % S;
        if (P.dbg & 16) {
          mbar_arrive(&wbar[s]);
          return;
        }
        mbar_expect_tx(&wbar[s], WB);
        bulk_g2s(w_of(s), wsrc + static_cast<size_t>(kb) * WB, WB, &wbar[s]);
      };
      auto issue_a = [&](int kb) {
        const int s = kb % S, kk = (U0 + kb) % nkb;
        if (P.dbg & 8) {
          mbar_arrive(&abar[s]);
          return;
        }
        mbar_expect_tx(&abar[s], Sh::kB);
        bulk_g2s(b_of(s), asrc + static_cast<size_t>(kk) * P.groups * 1024, Sh::kB, &abar[s]);
      };
      const int pre = nU < S ? nU : S;
      const int pre_w = P.pre_w > 0 && P.pre_w < pre ? P.pre_w : pre;
      for (int kb = 0; kb < pre_w; ++kb) issue_w(kb);
      {  // the rest of this CTA's weights: L2 bulk prefetch, so the ring's later
         // weight copies hit L2 instead of waiting on HBM latency
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        const size_t total = static_cast<size_t>(nU) * WB;
        for (size_t off = static_cast<size_t>(pre_w) * WB; off < total; off += 32768)
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
      // the activation tiles first (they queue behind whatever this SM has
      // requested), then the weight stages not requested yet
      for (int kb = 0; kb < pre; ++kb) {
        issue_a(kb);
        if (kb + pre_w < pre) issue_w(kb + pre_w);
      }
      for (int kb = S; kb < nU; ++kb) {
        mbar_wait(&ebar[kb % S], ((kb / S) - 1) & 1);  // MMA of kb - S done with the stage
        if (trace && kb < S + 16) trace[48 + kb - S] = clock64();
        issue_w(kb);
        issue_a(kb);
      }
    }
  } else if (warp >= 1 && warp <= kTcIssuers) {
    if (lane == 0) {
      // ---- MMA issuers: D=s32, A=B=u8, both K-major, N=TT, M=128.
      // kTcIssuers threads (lane 0 of warps 1..) take k-blocks round robin: an mbarrier wait in
      // the issuing thread stalls that thread's instruction stream for ~40
      // cycles per UMMA in flight (microbench_umma_mix), so while one waits
      // the other's UMMAs keep the tensor pipe busy.  Both accumulate into
      // the (pre-zeroed) accumulator; integer sums commute.
      const int t = warp - 1;
      const uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(TT >> 3) << 17) |
                             (static_cast<uint32_t>(kTcM >> 4) << 24);
      // descriptors: the start-address field is the low 14 bits of (addr >> 4)
      // and every operand lies below 256 KB, so a descriptor advances by a
      // plain add of (byte offset >> 4) -- precomputed, the issue loop is a
      // handful of uniform ops per UMMA
      const uint64_t a_base = umma_desc(smem_u32(Sh::kTmemA ? smem : (Sh::kExpand ? x_of(0) : w_of(0))), kTcM * 16, 128);
      const uint64_t b_base = umma_desc(smem_u32(b_of(0)), 128, 1024);
      constexpr uint64_t a_stride = (Sh::kExpand ? Sh::kA : Sh::kStage) >> 4;  // per ring slot
      constexpr uint64_t b_stride = Sh::kStage >> 4;
      constexpr uint64_t a_j = (2 * kTcM * 16) >> 4, b_j = (2 * 128) >> 4;  // per K = 32 step
      for (int kb = t; kb < nU; kb += kTcIssuers) {
        const int s = kb % S, a = kb % SA;
        const uint32_t ph = static_cast<uint32_t>(kb / S) & 1u, pha = static_cast<uint32_t>(kb / SA) & 1u;
        // a new segment (row tile) accumulates into the second TMEM buffer
        const uint32_t td = tmem_d + (kb >= n0 ? static_cast<uint32_t>(TT) : 0u);
        if (!(P.dbg & 2)) {
          if (Sh::kExpand) mbar_wait(&rbar[a], pha);
          else mbar_wait(&wbar[s], ph);
        }
        mbar_wait(&abar[s], ph);
        tc_fence_after();
        if (trace && kb < 16) trace[32 + kb] = clock64();
        const uint64_t ad = a_base + (Sh::kExpand ? a : s) * a_stride, bd = b_base + s * b_stride;
#pragma unroll
        for (int j = 0; j < kTcK / 32; ++j) {
          if (P.dbg & 4) continue;
          if constexpr (Sh::kTmemA) umma_i8_tmem_a(td, tmem_d + TMEM_A + a * 32 + j * 8, bd + j * b_j, idesc, 1u);
          else umma_i8(td, ad + j * a_j, bd + j * b_j, idesc, 1u);
        }
        tc_commit(&ebar[s]);
        if (Sh::kExpand) tc_commit(&xbar[a]);
      }
      tc_commit(&done_bar);
      if (trace) trace[3] = clock64();
    }
  } else if (Sh::kExpand && warp >= 4 && warp < 4 + 4 * Sh::kWG) {
    // ---- widen packed code slices of row r into the A operand, two k-blocks
    // per pass (their loads, widening and stores interleave: one k-block per
    // pass left each warp a ~600-cycle dependent chain per k-block, which
    // paced the whole k-loop)
    // kWG groups of 4 warps take alternate k-block pairs (TMEM lane quarter = warp % 4)
    const int r = (tid - 128) & (kTcM - 1), grp = (warp - 4) >> 2;
    auto widen_one = [&](int kb, const uint4 (&w)[Q > 0 ? Q : 1]) {
      const int a = kb % SA;
      if (kb >= SA) mbar_wait(&xbar[a], static_cast<uint32_t>(kb / SA - 1) & 1u);  // MMA of kb - SA done
      if constexpr (Sh::kTmemA) {
        // row r = TMEM lane r (warp w owns lanes 32 (w % 4) ..), register o -> column o
        tc_fence_after();
        uint32_t v[32];
#pragma unroll
        for (int o = 0; o < 32; ++o) v[o] = widen_row<Q>(w, o);
        const uint32_t ta = tmem_d + (static_cast<uint32_t>((warp & 3) * 32) << 16) + TMEM_A + a * 32;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
            "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
            "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
            : "memory");
      } else {
        uint4* adst = reinterpret_cast<uint4*>(x_of(a)) + r;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc)
          adst[kc * kTcM] = make_uint4(widen_row<Q>(w, 4 * kc), widen_row<Q>(w, 4 * kc + 1),
                                       widen_row<Q>(w, 4 * kc + 2), widen_row<Q>(w, 4 * kc + 3));
      }
    };
    auto load_one = [&](int kb, uint4 (&w)[Q > 0 ? Q : 1]) {
      const int s = kb % S;
      mbar_wait(&wbar[s], static_cast<uint32_t>(kb / S) & 1u);
      const uint32_t wsl = smem_u32(w_of(s)) + r * 16;
#pragma unroll
      for (int t = 0; t < Q; ++t)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w)
                     : "r"(wsl + t * kTcM * 16));
    };
    for (int kb = 2 * grp; kb < nU; kb += 2 * Sh::kWG) {
      const bool two = kb + 1 < nU;
      uint4 w0[Q > 0 ? Q : 1], w1[Q > 0 ? Q : 1];
      if (!(P.dbg & 32)) {
        load_one(kb, w0);
        if (two) load_one(kb + 1, w1);
        widen_one(kb, w0);
        if (two) widen_one(kb + 1, w1);
      }
      if constexpr (Sh::kTmemA) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
      } else {
        fence_async_smem();  // generic-proxy stores -> visible to the tensor core
      }
      __syncwarp();
      if (trace && tid == 128 && kb < 16) trace[16 + kb] = clock64();
      if (lane == 0) {
        mbar_arrive(&rbar[kb % SA]);
        if (two) mbar_arrive(&rbar[(kb + 1) % SA]);
      }
    }
  }
  if (warp >= 12) {  // idle during the k-loop: per-token epilogue values (after the ReQuant kernel)
    const EpiParams& E = P.e;
    if (E.mode != EPI_ACC_I32 && E.mode != EPI_ACC_I64) {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // ReQuant results visible
      for (int i = tid - 384; i < TT; i += 128) {
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
  }
  if (warp >= 12 && rt >= 0) {  // ... and the finished tile's channel parameters
    const int c = tid - 384, j = rt * kTcM + c;
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
  const int lch = quarter * 32 + lane;
  const uint32_t tlane = tmem_d + (static_cast<uint32_t>(quarter * 32) << 16);
  const uint32_t* part = nullptr;
  int npart = 0;
  if (P.sk) {
    // stream-K hand-off.  Contributions are published before any finisher
    // waits (a CTA's contributed segment is always its last one, its finished
    // segment its first), so no chain of CTAs serialises.
    const long long T = static_cast<long long>(P.rowtiles) * nkb, G = gridDim.x;
    auto cta_of = [&](long long u) { return static_cast<int>(((u + 1) * G - 1) / T); };
    const int con_seg = nseg == 2 ? 1 : (fin_seg < 0 ? 0 : -1);
    if (con_seg >= 0) {
      const int tcon = t0 + con_seg, slot = static_cast<int>(blockIdx.x) - cta_of(static_cast<long long>(tcon) * nkb);
      tc_store_partial<TT>(tlane + (con_seg ? static_cast<uint32_t>(TT) : 0u), half, lch,
                           P.sk_part + (static_cast<size_t>(tcon) * P.sk_slots + slot) * TT * kTcM);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.sk_flags + tcon * P.sk_slots + slot), "r"(1u) : "memory");
        if (trace) trace[10] = clock64();
      }
    }
    if (rt >= 0) {
      npart = static_cast<int>(blockIdx.x) - cta_of(static_cast<long long>(rt) * nkb);
      part = P.sk_part + static_cast<size_t>(rt) * P.sk_slots * TT * kTcM;
      if (tid == 0) {
        for (int c = 0; c < npart; ++c) {
          unsigned f = 0;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(P.sk_flags + rt * P.sk_slots + c) : "memory");
            if (f) break;
            __nanosleep(64);
          }
          P.sk_flags[rt * P.sk_slots + c] = 0u;  // consumed: zero for the next launch
        }
        if (trace) {
          trace[11] = clock64();
          trace[12] = (static_cast<unsigned long long>(nU) << 32) | (static_cast<unsigned>(npart) << 8) |
                      static_cast<unsigned>(nseg);
        }
      }
      __syncthreads();
    }
  }
  if (rt >= 0) {
    const int ch = rt * kTcM + lch;
    __half* stage = reinterpret_cast<__half*>(smem);  // the operand ring is idle now
    const uint32_t taddr = tlane + (fin_seg == 1 ? static_cast<uint32_t>(TT) : 0u);
    const bool k32 = P.k <= 32768;
    switch (P.e.mode) {
      case EPI_ACC_I32: tc_epilogue<EPI_ACC_I32, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
      case EPI_ACC_I64: tc_epilogue<EPI_ACC_I64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
      case EPI_F64: tc_epilogue<EPI_F64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
      case EPI_F16: tc_epilogue<EPI_F16, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
      case EPI_F32: tc_epilogue<EPI_F32, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
      default: tc_epilogue<EPI_CORR_I64, TT>(P.e, taddr, half, tok0, P.m, ch, P.n, t_sa, t_za, t_kz, t_ra, stage, lch, c_sb, c_zb, c_cs, k32, part, npart, P.dbg); break;
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
  static bool attr_set[64] = {false};  // once per instantiation and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    const cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::kSmem);
    if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: smem attribute: %s", cudaGetErrorString(err));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaError_t err = cudaSuccess;
  TcParams L = P;
  const int gy = (P.m + TT - 1) / TT;
  int gx = P.rowtiles;
  // stream-K when one token tile leaves SMs idle: G = min(SMs, units) CTAs
  // (tc_sk_grid) share the (row-tile, k-block) units, tc_sk_slots CTAs per tile
  // at most.  Finishers spin on their contributors, so every CTA must become
  // resident: G <= SMs with one CTA per SM, and this kernel never triggers its
  // dependents early (no griddepcontrol.launch_dependents: a dependent grid
  // waiting on this one cannot hold an SM a contributor needs).
  if (L.sk && gy == 1 && P.kblocks >= 2 && P.rowtiles < num_sms() &&
      static_cast<size_t>(P.rowtiles) <= kSkMaxRowtiles) {
    gx = tc_sk_grid(P.rowtiles, P.kblocks);
    L.sk_slots = tc_sk_slots(static_cast<size_t>(P.n), static_cast<size_t>(P.k));
  } else {
    L.sk = 0;
  }
  dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
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
  err = cudaLaunchKernelEx(&cfg, kern, L);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int Q>
static int launch_tt(const TcParams& P, bool pdl, cudaStream_t st, int tt_cap) {
  // Narrow layers with short K (LLaMA-7B o_proj N = K = 4096 at M = 128): 32-token
  // tiles fill one wave of SMs (32 row-tiles x 4 token tiles) where one
  // 128-token tile per row-tile leaves 116 SMs idle or hands partial tiles
  // around (stream-K): 17.0 -> 15.5 us (profiles/r02_gemm_tt_sweep.txt).  Longer
  // K (down_proj) and wide N lose with it (each CTA widens the whole weight tile).
  if (tt_cap <= 0 && P.m > 32 && P.kblocks <= 32 &&
      static_cast<long long>(P.rowtiles) * ((P.m + 31) / 32) <= num_sms())
    tt_cap = 32;
  const int cap = tt_cap > 0 ? std::max(16, tt_cap) : 256;  // TileConfig BM cap (abi.cu plan_of)
  if (P.m <= 16 || cap <= 16) return launch_tc<Q, 16>(P, pdl, st);
  if (P.m <= 32 || cap <= 32) return launch_tc<Q, 32>(P, pdl, st);
  if (P.m <= 64 || cap <= 64) return launch_tc<Q, 64>(P, pdl, st);
  if (P.m <= 128 || cap <= 128) return launch_tc<Q, 128>(P, pdl, st);
  return launch_tc<Q, 256>(P, pdl, st);
}

// k % 16 == 0 (16-byte code runs); the unsigned accumulator is exact to K = 65536
bool gemm_tc_supported(size_t k) { return k > 0 && k <= 65536 && k % 16 == 0; }

// act: tiled u8 codes (tc_act_offset, groups = tc_act_groups(m)), 16-B aligned
int run_gemm_tc(const uint32_t* wtc, unsigned q, size_t n, size_t k, const uint8_t* act, size_t m,
                const EpiParams& e, cudaStream_t st, unsigned long long* bad_word,
                unsigned long long* bad_out, bool pdl, unsigned* sk_flags, uint32_t* sk_part, EnginePlan plan) {
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
  P.dbg = dec_tuning().tc_dbg;
  P.pre_w = dec_tuning().tc_pre;
  if (plan.token_tile == 0 && dec_tuning().tc_tt > 0) plan.token_tile = dec_tuning().tc_tt;
  // a TileConfig's schedule (abi.cu plan_of) wins, then an explicit
  // abq_set_gemm_schedule; else the default
  const int sched = plan.schedule != ABQ_GEMM_AUTO ? plan.schedule : gemm_schedule();
  const bool sk_on = sched == ABQ_GEMM_STREAM_K ? true
                     : sched == ABQ_GEMM_CLASSIC ? false
                     : tc_stream_k_auto(P.rowtiles);
  if (sk_flags && sk_part && m <= 256 && sk_on) {
    P.sk = 1;
    P.sk_flags = sk_flags;
    P.sk_part = sk_part;
  }
  switch (q) {
    case 1: return launch_tt<1>(P, pdl, st, plan.token_tile);
    case 2: return launch_tt<2>(P, pdl, st, plan.token_tile);
    case 3: return launch_tt<3>(P, pdl, st, plan.token_tile);
    case 4: return launch_tt<4>(P, pdl, st, plan.token_tile);
    case 5: return launch_tt<5>(P, pdl, st, plan.token_tile);
    case 6: return launch_tt<6>(P, pdl, st, plan.token_tile);
    case 7: return launch_tt<7>(P, pdl, st, plan.token_tile);
    default: return launch_tt<8>(P, pdl, st, plan.token_tile);
  }
}

}  // namespace abq_dev
