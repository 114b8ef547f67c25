// gemm_tc.cu -- K3: prefill GEMM on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM), sm_100a.
//
// The reference's plane GEMM (include/abq/gemm.hpp:94-146) sums 2^(s+t) x
// popc(A_s & W_t) over p x q binary plane pairs.  sm_100a has no binary
// tensor-core instruction (b1 mma.sync is emulated with 8 IMMA + ~100 ALU
// ops per m16n8k256; measured 700 bit-MAC/clk/SM vs ~8192
// int8 MAC/clk/SM for tcgen05), so this kernel recombines the q weight planes
// into u8 codes on the fly in shared memory and issues one exact u8 x u8 ->
// s32 UMMA per 32-k step:   acc[i][j] = sum_k a_ik * (sum_t 2^t W_t[j][k]).
//
// Per CTA: 128 output channels (UMMA M) x TT tokens (UMMA N), K streamed in
// 128-wide stages through a 3-4 deep shared-memory ring:
//   * all 256 threads: load this stage's packed weight planes (one coalesced
//     8-byte load per plane per thread), rebuild 64 u8 codes per thread with
//     shift / mask / merge, store them in the UMMA canonical K-major
//     (no-swizzle) layout; cp.async the u8 activation codes of the stage;
//   * thread 0: waits for the stage, issues 4 x tcgen05.mma (K = 32 each) into
//     the TMEM accumulator and tcgen05.commit's the stage back to the
//     producers;
//   * epilogue: tcgen05.ld (32x32b) -> registers -> fused zero-point
//     correction + dequant (gemm.hpp:235-254, 292-306) -> global.
// Weight layout ("tc planes", prepack_tc_kernel): [row-tile 128][k-block 128]
// [plane][row][4 x u32]; word j of a (row, plane) holds k = 32j..32j+31 of the
// block with bit (8b + c) <-> k = 32j + 4c + b, so code register c is
// sum_t ((w_t >> c) & 0x01010101) << t.  Same bits as ABQP, rows padded to
// 128 and K to 128 with zeros.
#include "common.cuh"

namespace abq_dev {

constexpr int kTcM = 128;
constexpr int kTcK = 128;
constexpr int kTcThreads = 256;

// ---------------------------------------------------------------------------
// prepack: ABQP [q][n][wpr] -> tc planes
// ---------------------------------------------------------------------------
__global__ void prepack_tc_kernel(const uint64_t* __restrict__ planes, int q, int n, int k, int wpr,
                                  int rowtiles, int kblocks, uint32_t* __restrict__ out) {
  const size_t total = static_cast<size_t>(rowtiles) * kblocks * q * kTcM * 4;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(idx & 3);
    const int row = static_cast<int>((idx >> 2) & (kTcM - 1));
    size_t rest = idx >> 9;
    const int t = static_cast<int>(rest % q);
    rest /= q;
    const int kb = static_cast<int>(rest % kblocks);
    const int rt = static_cast<int>(rest / kblocks);
    const int grow = rt * kTcM + row;
    const int kbase = kb * kTcK + 32 * j;
    uint32_t w = 0;
    if (grow < n) {
      const uint64_t* src = planes + (static_cast<size_t>(t) * n + grow) * wpr;
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kk = kbase + 4 * c + b;
          if (kk < k) w |= static_cast<uint32_t>((src[kk >> 6] >> (kk & 63)) & 1ull) << (8 * b + c);
        }
    }
    out[idx] = w;
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
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
// UMMA shared-memory descriptor, K-major, no swizzle (canonical layout
// ((8,m),2):((16B,SBO),LBO)), version 1 for sm_100.
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
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ uint2 ld_nc_u2(const uint32_t* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

template <int T, int C>
__device__ __forceinline__ uint32_t plane_to_codes(uint32_t w) {
  uint32_t x;
  if constexpr (T >= C)
    x = w << (T - C);
  else
    x = w >> (C - T);
  return x & (0x01010101u << T);
}

// 8 code registers (32 codes, k = 4c..4c+3 in register c) from the q plane words
template <int Q>
__device__ __forceinline__ void rebuild32(const uint32_t (&w)[Q], uint32_t (&r)[8]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) r[c] = 0u;
  // plane t lands on bit (8 - Q + t): the code scaled by 2^(8-Q), so that most
  // bit moves are left shifts (IMAD.SHL on the fma pipe) next to the LOP3 merges
  // on the alu pipe; the accumulator is divided back exactly in the epilogue.
#define ABQ_PLACE(T)                                                 \
  if constexpr (Q > T) {                                             \
    r[0] |= plane_to_codes<8 - Q + T, 0>(w[T]);                      \
    r[1] |= plane_to_codes<8 - Q + T, 1>(w[T]);                      \
    r[2] |= plane_to_codes<8 - Q + T, 2>(w[T]);                      \
    r[3] |= plane_to_codes<8 - Q + T, 3>(w[T]);                      \
    r[4] |= plane_to_codes<8 - Q + T, 4>(w[T]);                      \
    r[5] |= plane_to_codes<8 - Q + T, 5>(w[T]);                      \
    r[6] |= plane_to_codes<8 - Q + T, 6>(w[T]);                      \
    r[7] |= plane_to_codes<8 - Q + T, 7>(w[T]);                      \
  }
  ABQ_PLACE(0)
  ABQ_PLACE(1)
  ABQ_PLACE(2)
  ABQ_PLACE(3)
  ABQ_PLACE(4)
  ABQ_PLACE(5)
  ABQ_PLACE(6)
  ABQ_PLACE(7)
#undef ABQ_PLACE
}

struct TcParams {
  const uint32_t* wtc;  // tc planes
  const uint8_t* act;   // u8 activation codes, row stride ldk (multiple of 16, 16B aligned)
  int q, n, k, m, ldk, rowtiles, kblocks;
  EpiParams e;
  unsigned long long* bad_word;  // ReQuant status (~index, 0 = none), published to bad_out
  unsigned long long* bad_out;
  int pdl;                       // launched as a programmatic dependent of the ReQuant kernel
};

template <int Q, int TT, int S>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(TcParams P) {
  constexpr int A_BYTES = kTcM * kTcK;  // 16 KB
  constexpr int B_BYTES = TT * kTcK;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = TT <= 32 ? 32 : (TT <= 64 ? 64 : (TT <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t full_bar[S], empty_bar[S], done_bar;
  __shared__ uint32_t tmem_base_s;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rt = blockIdx.x, tok0 = blockIdx.y * TT;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], kTcThreads);
      mbar_init(&empty_bar[s], 1);
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

  // instruction descriptor: D=s32, A=B=u8, K-major both, N=TT, M=128
  const uint32_t idesc = (2u << 4) | (static_cast<uint32_t>(TT >> 3) << 17) | (static_cast<uint32_t>(kTcM >> 4) << 24);
  const int prow = tid >> 1, phalf = tid & 1;  // producer: weight row, 64-k half
  const size_t stage_words = static_cast<size_t>(Q) * kTcM * 4;

  // Software pipeline (per thread): the packed weight words of stage kb + DW
  // and the activation tile of stage kb + DA are requested while stage kb is
  // rebuilt, so every thread keeps several HBM / L2 round trips in flight.
  constexpr int DW = 3;                    // weight-word prefetch distance (registers)
  constexpr int DA = S >= 3 ? S - 2 : 1;   // activation cp.async distance (smem stages)
  auto issue_act = [&](int j) {            // cp.async of stage j's activations, one group
    if (j < P.kblocks) {
      const int sj = j % S;
      if (j >= S) mbar_wait(&empty_bar[sj], ((j / S) + 1) & 1);
      unsigned char* b_st = smem + sj * STAGE + A_BYTES;
      for (int piece = tid; piece < TT * 8; piece += kTcThreads) {
        const int token = piece >> 3, kc = piece & 7;
        const int tk = tok0 + token;
        const int kk = j * kTcK + kc * 16;
        const bool ok = tk < P.m && kk < P.k;
        const uint8_t* src = ok ? P.act + static_cast<size_t>(tk) * P.ldk + kk : P.act;
        cp_async16(smem_u32(b_st + (kc * (TT / 8) + (token >> 3)) * 128 + (token & 7) * 16), src,
                   ok ? 16u : 0u);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  uint32_t wring[DW + 1][2][Q];
  auto issue_w = [&](int j, uint32_t (&dst)[2][Q]) {
    if (j < P.kblocks) {
      const uint32_t* wsrc = P.wtc + (static_cast<size_t>(rt) * P.kblocks + j) * stage_words;
#pragma unroll
      for (int t = 0; t < Q; ++t) {
        const uint2 v = ld_nc_u2(wsrc + (t * kTcM + prow) * 4 + 2 * phalf);
        dst[0][t] = v.x;
        dst[1][t] = v.y;
      }
    }
  };
  // weights do not depend on the preceding ReQuant kernel: start them first,
  // then wait for its codes (programmatic dependent launch; a no-op otherwise)
#pragma unroll
  for (int j = 0; j < DW; ++j) issue_w(j, wring[j]);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (P.bad_out && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
    const unsigned long long w = *P.bad_word;
    *P.bad_out = w ? ~w : ~0ull;
    *P.bad_word = 0ull;
  }
#pragma unroll
  for (int j = 0; j < DA; ++j) issue_act(j);

  // one copy of the stage body (compact hot loop); the weight ring shifts by one stage
  for (int kb = 0; kb < P.kblocks; ++kb) {
    const int s = kb % S;
    const uint32_t use = static_cast<uint32_t>(kb / S);
    issue_act(kb + DA);  // also guarantees stage s is free (waited DA stages ago)
    uint32_t wn[2][Q];
    issue_w(kb + DW, wn);
    unsigned char* a_st = smem + s * STAGE;
    unsigned char* b_st = a_st + A_BYTES;
    {
      uint32_t r0[8], r1[8];
      rebuild32<Q>(wring[0][0], r0);
      rebuild32<Q>(wring[0][1], r1);
      const int kc0 = 4 * phalf;  // 16-byte k chunk index of r0[0..3]
      auto sts = [&](int kc, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
        *reinterpret_cast<uint4*>(a_st + (kc * (kTcM / 8) + (prow >> 3)) * 128 + (prow & 7) * 16) =
            make_uint4(x, y, z, w);
      };
      sts(kc0 + 0, r0[0], r0[1], r0[2], r0[3]);
      sts(kc0 + 1, r0[4], r0[5], r0[6], r0[7]);
      sts(kc0 + 2, r1[0], r1[1], r1[2], r1[3]);
      sts(kc0 + 3, r1[4], r1[5], r1[6], r1[7]);
    }
#pragma unroll
    for (int d = 0; d < DW; ++d)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < Q; ++t) wring[d][h][t] = d + 1 < DW ? wring[d + 1][h][t] : wn[h][t];
    // this thread's activation pieces of stage kb have landed (DA newer groups may still fly)
    asm volatile("cp.async.wait_group %0;" ::"n"(DA) : "memory");
    fence_async_smem();
    mbar_arrive(&full_bar[s]);
    if (tid == 0) {
      mbar_wait(&full_bar[s], use & 1);
      tc_fence_after();
      const uint32_t a_addr = smem_u32(a_st), b_addr = smem_u32(b_st);
#pragma unroll
      for (int j = 0; j < kTcK / 32; ++j) {
        const uint64_t ad = umma_desc(a_addr + j * 2 * (kTcM / 8) * 128, (kTcM / 8) * 128, 128);
        const uint64_t bd = umma_desc(b_addr + j * 2 * (TT / 8) * 128, (TT / 8) * 128, 128);
        umma_i8(tmem_d, ad, bd, idesc, (kb | j) != 0 ? 1u : 0u);
      }
      tc_commit(&empty_bar[s]);
      if (kb == P.kblocks - 1) tc_commit(&done_bar);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  // ---- epilogue: TMEM -> registers -> zero-point correction + dequant.  A
  // thread owns one output channel (TMEM lane) and half of the token columns,
  // so the per-channel parameters are loaded once.
  mbar_wait(&done_bar, 0);
  tc_fence_after();
  const int quarter = warp & 3, half = warp >> 2;
  const int ch = rt * kTcM + quarter * 32 + lane;
  const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
  const EpiParams& E = P.e;
  const bool raw = E.mode == EPI_ACC_I32 || E.mode == EPI_ACC_I64;
  const bool chan_ok = ch < P.n;
  double sb = 0.0;
  long long zb = 0, cs = 0;
  if (!raw && chan_ok) {
    sb = E.s_b[ch * E.sb_stride];
    zb = E.z_b[ch * E.zb_stride];
    cs = E.colsum_b[ch];
  }
#pragma unroll 1
  for (int c0 = half * (TT / 2); c0 < (half + 1) * (TT / 2); c0 += 8) {
    uint32_t v[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
        : "r"(tmem_d + lane_base + static_cast<uint32_t>(c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!chan_ok) continue;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int tk = tok0 + c0 + i;
      if (tk >= P.m) continue;
      const long long acc = static_cast<long long>(static_cast<int32_t>(v[i]) >> (8 - Q));
      const long long o = static_cast<long long>(tk) * E.ldo + ch;
      if (raw) {
        if (E.mode == EPI_ACC_I32) static_cast<int32_t*>(E.out)[o] = static_cast<int32_t>(acc);
        else static_cast<int64_t*>(E.out)[o] = acc;
        continue;
      }
      const long long za = E.z_a[tk * E.za_stride];
      const long long corr = acc - za * cs - zb * E.rowsum_a[tk] + E.k * za * zb;
      if (E.mode == EPI_CORR_I64) {
        static_cast<int64_t*>(E.out)[o] = corr;
        continue;
      }
      const double y = __dmul_rn(__dmul_rn(E.s_a[tk * E.sa_stride], sb), static_cast<double>(corr));
      if (E.mode == EPI_F64) static_cast<double*>(E.out)[o] = y;
      else if (E.mode == EPI_F16) static_cast<__half*>(E.out)[o] = __double2half(y);
      else static_cast<float*>(E.out)[o] = __double2float_rn(y);
    }
  }
  tc_fence_before();
  __syncthreads();
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

template <int Q, int TT>
static int launch_tc(const TcParams& P, cudaStream_t st) {
  constexpr int STAGE = kTcM * kTcK + TT * kTcK;
  constexpr int S = (200 * 1024) / STAGE >= 4 ? 4 : ((200 * 1024) / STAGE >= 3 ? 3 : 2);
  auto kern = gemm_tc_kernel<Q, TT, S>;
  const size_t smem = static_cast<size_t>(S) * STAGE;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: smem attribute: %s", cudaGetErrorString(err));
  dim3 grid(static_cast<unsigned>(P.rowtiles), static_cast<unsigned>((P.m + TT - 1) / TT));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = P.pdl ? 1 : 0;
  err = cudaLaunchKernelEx(&cfg, kern, P);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemm_tc: launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int Q>
static int launch_tt(const TcParams& P, cudaStream_t st) {
  if (P.m <= 16) return launch_tc<Q, 16>(P, st);
  if (P.m <= 32) return launch_tc<Q, 32>(P, st);
  if (P.m <= 64) return launch_tc<Q, 64>(P, st);
  if (P.m <= 128) return launch_tc<Q, 128>(P, st);
  return launch_tc<Q, 256>(P, st);
}

// act: u8 codes [m][ldk]; requires k % 16 == 0, ldk % 16 == 0 and a 16-B aligned act.
// K <= 32768 keeps the scaled-code accumulator (255 * 255 * K) inside s32
bool gemm_tc_supported(size_t k, size_t ldk) {
  return k > 0 && k <= 32768 && k % 16 == 0 && ldk % 16 == 0;
}

int run_gemm_tc(const uint32_t* wtc, unsigned q, size_t n, size_t k, const uint8_t* act, size_t ldk,
                size_t m, const EpiParams& e, cudaStream_t st, unsigned long long* bad_word,
                unsigned long long* bad_out, bool pdl) {
  if (m == 0 || n == 0) return ABQ_OK;
  TcParams P{};
  P.bad_word = bad_word;
  P.bad_out = bad_out;
  P.pdl = pdl ? 1 : 0;
  P.wtc = wtc;
  P.act = act;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.m = static_cast<int>(m);
  P.ldk = static_cast<int>(ldk);
  P.rowtiles = static_cast<int>((n + kTcM - 1) / kTcM);
  P.kblocks = static_cast<int>((k + kTcK - 1) / kTcK);
  P.e = e;
  switch (q) {
    case 1: return launch_tt<1>(P, st);
    case 2: return launch_tt<2>(P, st);
    case 3: return launch_tt<3>(P, st);
    case 4: return launch_tt<4>(P, st);
    case 5: return launch_tt<5>(P, st);
    case 6: return launch_tt<6>(P, st);
    case 7: return launch_tt<7>(P, st);
    default: return launch_tt<8>(P, st);
  }
}

}  // namespace abq_dev
