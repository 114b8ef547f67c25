// gemv_imma.cu -- K2 "recombination" variant: decode GEMV (M <= 8 tokens per
// token block) that feeds the q-bit weight codes to the int8 tensor pipe
// against u8 activation codes.  sm_100a.
//
// Why (measured in profiles/r01_microbench_pipes.txt): on
// sm_100a POPC issues at 16/clk/SM, so the AND+popcount decomposition of a
// p-bit activation x q-bit weight product needs p POPCs per 32 weight-plane
// bits -- 36% of HBM at p=8.  The int8 tensor pipe (legacy IMMA m16n8k32,
// ~1950 MAC/clk/SM) is idle in that kernel.  Here the weight bit planes are
// recombined into u8 codes and multiplied on the tensor pipe:
//
//   acc = sum_k a_k * (sum_t 2^t W_t[k])       (paper Eq. 11 with both sides'
//                                                planes recombined)
//
// which is the same exact unsigned code product as the reference's
// gemm_plane_rows (include/abq/gemm.hpp:94-146).  Accumulation is exact: the
// per-row-tile sum is < 2^32 for K <= 65536 and read back as unsigned.
//
// Weight layout (built once by prepack_frag_kernel from the ABQP planes):
// [row-tile of 16][k-block of 256][q][lane][4 x u32] holding the codes as
// "code slices" (common.cuh): the binary decomposition of q into slices of
// width 8/4/2/1, each packing its code bits in byte lanes so that widening
// to the u8 A register o = 4c + u (chunk c, register u: element row g + 8*(u&1),
// k = 32c + 16*(u>>1) + 4*tig + b in byte b) is one shift + one mask per slice
// (q = 4: 1.5 ALU ops per register; q = 8: none).  Same byte count as ABQP;
// each (tile, block) "unit" is q x 512 contiguous bytes.
// (profiles/r01_microbench_gemv_body.txt: the earlier per-plane merge needed
// 8 ALU ops per register and capped the loop at ~19 B/clk/SM.)
//
// Pipeline (one persistent CTA of 16 warps per SM):
//   * work split, stream-K: the (row-tile, k-block) units are divided evenly
//     over CTAs and warps; a warp's units are one contiguous global range;
//   * each warp streams its units through a private ring of shared-memory
//     slots with 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx),
//     issued at kernel start -- before the activations exist;
//   * the activations are ReQuantized by the small act_quant_kernel launched
//     just before this kernel with programmatic dependent launch: this kernel
//     starts immediately, fills its weight ring, prefetches its per-channel
//     epilogue parameters, and only then waits (griddepcontrol.wait) for the
//     u8 codes (written by act_quant_kernel already in the B-fragment order);
//   * partial row-tile sums meet in shared memory (64-bit atomics) and, for the
//     row-tiles cut between CTAs, in a self-cleaning global accumulator where
//     the last contributing CTA runs the fused zero-point/dequant epilogue.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "quant_dev.cuh"
#include "gemv_frag.cuh"

namespace abq_dev {


// ---------------------------------------------------------------------------
// prepack: ABQP [q][n][wpr] -> fragment-major code slices [rt][kb][q][lane][4]
// (the lane's 4q words; word J belongs to the slice holding code bit J / 4)
// ---------------------------------------------------------------------------
__global__ void prepack_frag_kernel(const uint64_t* __restrict__ planes, int q, int n, int k, int wpr,
                                    int rowtiles, int kblocks, uint32_t* __restrict__ frag) {
  const size_t total = static_cast<size_t>(rowtiles) * kblocks * q * 128;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    // word J (0..4q-1) of this lane; J / 4 is a code bit of slice `si`
    const int lane = static_cast<int>((idx >> 2) & 31);
    size_t rest = idx >> 7;
    const int J = static_cast<int>(rest % q) * 4 + static_cast<int>(idx & 3);
    rest /= q;
    const int kb = static_cast<int>(rest % kblocks);
    const int rt = static_cast<int>(rest / kblocks);
    const int si = slice_of_bit(q, J >> 2), sw = slice_width(q, si), so = slice_off(q, si);
    const int j = J - 4 * so;  // word within the slice (0..4w-1)
    const int g = lane >> 2, tig = lane & 3;
    uint32_t w = 0;
    for (int s = 0; s < 8 / sw; ++s) {
      // output register o = 4c + u of the lane's A fragments
      const int o = s * 4 * sw + j, c = o >> 2, u = o & 3;
      const int row = rt * kRowTile + g + 8 * (u & 1);
      if (row >= n) continue;
      for (int b = 0; b < 4; ++b) {
        const int kk = kb * kKBlock + 32 * c + 16 * (u >> 1) + 4 * tig + b;
        if (kk >= k) continue;
        for (int e = 0; e < sw; ++e) {
          const uint64_t* src = planes + (static_cast<size_t>(so + e) * n + row) * wpr;
          w |= static_cast<uint32_t>((src[kk >> 6] >> (kk & 63)) & 1ull) << (8 * b + sw * s + e);
        }
      }
    }
    frag[idx] = w;
  }
}

// ---------------------------------------------------------------------------
// K1 for the fused decode path: per-token ReQuant of the float activations
// into u8 codes already in the GEMV's B-fragment order (one CTA per token)
// plus scale / zero point / code row sum.  Non-finite inputs are reported as
// atomicMax(~flat_index) into a zero-initialised word (0 = none).
// ---------------------------------------------------------------------------
constexpr int kActThreads = 256;

// non-finite fp16 inputs of one thread's vectors -> atomicMax(~flat index);
// out of line: it only runs when one was seen
static __device__ __noinline__ void act_report_nonfinite(const __half* row, int tok, int k, int tid, int nvec,
                                                         unsigned long long* bad_word) {
  for (int v = tid; v < nvec; v += kActThreads) {
    const uint4 q = reinterpret_cast<const uint4*>(row)[v];
    const __half* h = reinterpret_cast<const __half*>(&q);
    for (int e = 0; e < 8; ++e)
      if (!isfinite(__half2float(h[e])))
        atomicMax(bad_word, ~(static_cast<unsigned long long>(tok) * k + static_cast<unsigned long long>(v) * 8 + e));
  }
}

// ROW: write the tcgen05 GEMM's tiled u8 operand (tc_act_offset, `row_ld` =
// token groups) instead of the GEMV's B-fragment order.
// VR: 16-byte fp16 vectors per thread of the register-resident fast path
// (4: K <= 8192; 8: K <= 16384, e.g. LLaMA-7B/13B down_proj K = 11008 / 13824;
// 16: K <= 32768, LLaMA-70B down_proj K = 28672), which otherwise took the
// generic per-element FP64 path: ~12 us per launch at K = 11008, M = 128.
template <typename T, bool ROW, int VR>
__global__ void __launch_bounds__(kActThreads) act_quant_kernel(const T* __restrict__ x, int m, int k, int mt,
                                                                QuantParams qp, uint32_t* __restrict__ act_frag,
                                                                int row_ld, double* __restrict__ s_a,
                                                                int32_t* __restrict__ z_a,
                                                                long long* __restrict__ rowsum,
                                                                unsigned long long* __restrict__ bad_word) {
  __shared__ double s_lo[kActThreads / 32], s_hi[kActThreads / 32];
  __shared__ long long s_sum[kActThreads / 32];
  __shared__ double s_step;
  __shared__ int s_z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tok = blockIdx.x;
  const int tb = tok / mt, i = tok % mt;
  const int kpad = ((k + kKBlock - 1) / kKBlock) * kKBlock;
  uint32_t* dst = ROW ? act_frag : act_frag + static_cast<size_t>(tb) * mt * kpad / 4;
  // u32 slot of the codes of elements 4v..4v+3
  auto slot_of = [&](int v) {
    return ROW ? static_cast<int>(tc_act_offset(tok, 4 * v, row_ld) >> 2) : act_frag_index(v, i, mt);
  };
  // codes past k are zero: to the 256-block (GEMV) / 128-block (GEMM)
  const int kzero = ROW ? (k + 127) / 128 * 128 : kpad;
  const T* row = x + static_cast<size_t>(tok) * k;
  if constexpr (sizeof(T) == 2) {
    // fp16 rows, per token, K % 8 == 0, K <= 8 * VR * kActThreads: the row is read
    // once with 16-byte loads and kept in registers (min/max in fp32 is exact
    // for fp16 inputs); codes and sums as in the generic path below.
    if (!qp.per_tensor && (k & 7) == 0 && k <= 8 * VR * kActThreads) {
      const int nvec = k >> 3;
      uint4 v[VR];
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        const int idx = tid + r * kActThreads;
        v[r] = idx < nvec ? __ldg(reinterpret_cast<const uint4*>(row) + idx) : make_uint4(0u, 0u, 0u, 0u);
      }
      // the row is requested: let the dependent GEMV / GEMM start streaming its
      // weights now (issued after our loads, so they do not queue behind them)
      griddep_launch();
      // range in the order-preserving integer image of fp32 (exact for fp16):
      // one REDUX per warp; non-finite inputs by exponent test, reported out of line
      auto ord = [](float f) {
        const int b = __float_as_int(f);
        return b >= 0 ? b : b ^ 0x7FFFFFFF;
      };
      auto unord = [](int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); };
      int lo = 0x7FFFFFFF, hi = static_cast<int>(0x80000000u);
      uint32_t bad = 0;
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        if (tid + r * kActThreads >= nvec) break;
        bad |= f16x8_nonfinite(v[r]);
        const __half2* h2 = reinterpret_cast<const __half2*>(&v[r]);
        __half2 mn = h2[0], mx = h2[0];
#pragma unroll
        for (int e = 1; e < 4; ++e) {
          mn = __hmin2(mn, h2[e]);
          mx = __hmax2(mx, h2[e]);
        }
        lo = min(lo, min(ord(__low2float(mn)), ord(__high2float(mn))));
        hi = max(hi, max(ord(__low2float(mx)), ord(__high2float(mx))));
      }
      if (bad) act_report_nonfinite(row, tok, k, tid, nvec, bad_word);
      lo = __reduce_min_sync(0xffffffffu, lo);
      hi = __reduce_max_sync(0xffffffffu, hi);
      if (lane == 0) {
        s_lo[warp] = __int_as_float(lo);  // raw bits, decoded below
        s_hi[warp] = __int_as_float(hi);
      }
      if (tid == 0) s_sum[0] = 0;
      __syncthreads();
      // every warp derives step / zero point itself (lanes 0 and 1 in parallel)
      int l2 = lane < kActThreads / 32 ? __float_as_int(s_lo[lane]) : 0x7FFFFFFF;
      int h2 = lane < kActThreads / 32 ? __float_as_int(s_hi[lane]) : static_cast<int>(0x80000000u);
      l2 = __reduce_min_sync(0xffffffffu, l2);
      h2 = __reduce_max_sync(0xffffffffu, h2);
      double step = 0.0;
      int z = 0;
      float inv32 = 0.0f;
      // every lane (same inputs, same results): one FP64 division, no broadcast
      group_params_fast(qp, unord(l2), unord(h2), &step, &z, &inv32);
      if (tid == 0) {
        s_a[tok] = step;
        z_a[tok] = z;
      }
      const int topi = static_cast<int>(qp.levels - 1);
      int rsum = 0;
#pragma unroll
      for (int r = 0; r < VR; ++r) {
        const int idx = tid + r * kActThreads;
        if (idx >= nvec) break;
        uint32_t w0, w1;
        rsum += quant_codes8_f16(v[r], step, inv32, z, topi, &w0, &w1);
        dst[slot_of(2 * idx)] = w0;
        dst[slot_of(2 * idx + 1)] = w1;
      }
      // zero codes in the k padding of the last block
      for (int v4 = k / 4 + tid; v4 < kzero / 4; v4 += kActThreads) dst[slot_of(v4)] = 0u;
      rsum = __reduce_add_sync(0xffffffffu, rsum);  // < 2^31: <= 255 * 65536
      if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_sum[0]), static_cast<unsigned long long>(rsum));
      __syncthreads();
      if (tid == 0) rowsum[tok] = s_sum[0];
      return;
    }
  }
  griddep_launch();
  double lo = CUDART_INF, hi = -CUDART_INF;
  if (qp.per_tensor) {
    for (int t = 0; t < m; ++t)
      for (int j = tid; j < k; j += kActThreads) {
        const double v = load_as_double(x, static_cast<size_t>(t) * k + j);
        if (!isfinite(v)) atomicMax(bad_word, ~(static_cast<unsigned long long>(t) * k + j));
        lo = fmin(lo, v);
        hi = fmax(hi, v);
      }
  } else {
    for (int j = tid; j < k; j += kActThreads) {
      const double v = load_as_double(row, j);
      if (!isfinite(v)) atomicMax(bad_word, ~(static_cast<unsigned long long>(tok) * k + j));
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
  }
  lo = warp_min(lo);
  hi = warp_max(hi);
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kActThreads / 32; ++w) {
      lo = fmin(lo, s_lo[w]);
      hi = fmax(hi, s_hi[w]);
    }
    double step;
    int z;
    group_params(qp, lo, hi, &step, &z);
    s_step = step;
    s_z = z;
    s_a[tok] = step;
    z_a[tok] = z;
  }
  __syncthreads();
  const double step = s_step, zd = static_cast<double>(s_z), inv = 1.0 / step;
  const double top = static_cast<double>(qp.levels - 1);
  long long rsum = 0;
  const int ngroups = kzero / 4;  // zero codes past k
  for (int v = tid; v < ngroups; v += kActThreads) {
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = 4 * v + b;
      if (j < k) {
        const unsigned c = quant_code_fast(load_as_double(row, j), step, inv, zd, top);
        rsum += c;
        word |= c << (8 * b);
      }
    }
    dst[slot_of(v)] = word;
  }
  rsum = warp_sum(rsum);
  if (lane == 0) s_sum[warp] = rsum;
  __syncthreads();
  if (tid == 0) {
    long long r = 0;
    for (int w = 0; w < kActThreads / 32; ++w) r += s_sum[w];
    rowsum[tok] = r;
  }
}

// ---------------------------------------------------------------------------
// main kernel
// ---------------------------------------------------------------------------
struct ImmaParams {
  const uint32_t* frag;
  int q, n, k, rowtiles, kblocks;
  int m;  // total tokens
  // activations: codes from act_quant_kernel (act_frag + stats) or packed planes
  const uint32_t* act_frag;
  const double* s_a;
  const int32_t* z_a;
  const long long* rowsum;
  const uint64_t* a_planes;
  int p;
  int wpr_a;
  EpiParams e;
  long long* gacc;  // [rowtiles][16][8] int64, zero on entry and exit (stream-K)
  unsigned* gcnt;   // [rowtiles], zero on entry and exit
  unsigned long long* bad_word;  // written by act_quant_kernel (~index, 0 = none)
  unsigned long long* bad_out;   // published here: first bad index or ~0
  unsigned long long* trace;     // optional [grid][4] globaltimer stamps (profiling)
  const __half* x16;             // fused path: fp16 activations quantized in the prologue
  QuantParams qp;
  int slots;                     // TMA ring slots per warp
  int late_ring;                 // experiment: start the whole ring after the prologue
  int upc;                       // units per TMA chunk (chunks of ~4 KB stream at full HBM rate)
};

// FROM_PLANES: activations are given as ABQP planes (API path) instead of
// codes from act_quant_kernel.
template <int QT, int MT, bool FROM_PLANES, int NWARP>
__global__ void __launch_bounds__(NWARP * 32, 1) gemv_imma_kernel(const __grid_constant__ ImmaParams P) {
  constexpr int q = QT;
  extern __shared__ __align__(128) unsigned char smem[];
  const int kpad = P.kblocks * kKBlock;
  const int G = gridDim.x;
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  const bool stream_k = P.gacc != nullptr;
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
  const int unit_bytes = q * 512;

  // shared memory carve-up
  const int chunk_bytes = P.upc * unit_bytes;
  unsigned char* wring = smem;                                                         // [warps][slots][chunk]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wring + NWARP * P.slots * chunk_bytes);  // [warps][slots]
  uint32_t* act = reinterpret_cast<uint32_t*>(bars + NWARP * P.slots);           // MT * kpad bytes
  long long* accs = reinterpret_cast<long long*>(reinterpret_cast<unsigned char*>(act) + MT * kpad);
  double* c_sb = reinterpret_cast<double*>(accs + nlrt * 16 * MT);  // per-channel epilogue params
  long long* c_zb = reinterpret_cast<long long*>(c_sb + nlrt * 16);
  long long* c_cs = c_zb + nlrt * 16;
  double* s_sa = reinterpret_cast<double*>(c_cs + nlrt * 16);
  long long* s_za = reinterpret_cast<long long*>(s_sa + MT);
  long long* s_ra = s_za + MT;
  __shared__ int s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const int tok0 = blockIdx.y * MT;
  const int mb = min(MT, P.m - tok0);
  if (warp == NWARP - 1) warm_param_block(P, lane);
  unsigned long long* trace = P.trace ? P.trace + 16 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (trace && tid == 0) {
    trace[0] = clock64();
    trace[8] = gtimer();
  }

  // ring barriers first: the release fence that publishes their init would
  // otherwise wait for the loads below to complete
  const long long wu0 = U0 + (U1 - U0) * warp / NWARP;
  const long long wu1 = U0 + (U1 - U0) * (warp + 1) / NWARP;
  unsigned char* my_ring = wring + warp * P.slots * chunk_bytes;
  uint64_t* my_bars = bars + warp * P.slots;
  if (lane == 0) {
    for (int s = 0; s < P.slots; ++s) mbar_init1(&my_bars[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // ---- 0. global reads of the prologue are REQUESTED before the weight ring
  // is started: every SM queues ~200 KB of TMA traffic next, and a load issued
  // behind it waits for that queue to drain (~4 us at the per-SM share of HBM).
  // (a) fused ReQuant: the activation rows (registers)
  constexpr int XT = MT < 2 ? MT : 2;
  uint4 xv[XT][4];
  if (!FROM_PLANES && P.x16) {
#pragma unroll
    for (int i = 0; i < XT; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int idx = tid + r * NWARP * 32;
        xv[i][r] = make_uint4(0u, 0u, 0u, 0u);
        if (i < mb && idx < (P.k >> 3))
          xv[i][r] = __ldg(reinterpret_cast<const uint4*>(P.x16 + static_cast<size_t>(tok0 + i) * P.k) + idx);
      }
  }
  // (b) per-channel epilogue parameters of this CTA's row-tiles (<= 1 channel
  // per thread; stored to shared memory after the ring is started)
  const bool dequant = P.e.mode != EPI_ACC_I32 && P.e.mode != EPI_ACC_I64;
  const int pj = rt_first * kRowTile + tid;
  const bool has_param = dequant && tid < nlrt * 16 && pj < P.n;
  double p_sb = 0.0;
  long long p_zb = 0, p_cs = 0;
  if (has_param) {
    p_sb = P.e.s_b[pj * P.e.sb_stride];
    p_zb = P.e.z_b[pj * P.e.zb_stride];
    p_cs = P.e.colsum_b[pj];
  }

  // ---- 1. this warp's units; start its TMA weight ring.  Paths that still
  // read activations from global memory after this point (ReQuant kernel
  // codes, packed planes) start one slot per warp now (64 KB per SM, enough to
  // keep HBM busy) and the rest once those reads are issued.
  const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(P.frag);
  auto start_slots = [&](int s0, int s1) {  // lane 0 only
    for (int s = s0; s < s1; ++s) {
      const long long un = wu0 + static_cast<long long>(s) * P.upc;
      if (un >= wu1) break;
      const long long un1 = un + P.upc < wu1 ? un + P.upc : wu1;
      const uint32_t bytes = static_cast<uint32_t>((un1 - un) * unit_bytes);
      mbar_expect_tx(&my_bars[s], bytes);
      tma_bulk_g2s(my_ring + s * chunk_bytes, wsrc + un * unit_bytes, bytes, &my_bars[s]);
    }
  };
  const bool late_act = FROM_PLANES || P.x16 == nullptr;
  const int first_slots = P.late_ring ? 0 : (late_act ? 1 : P.slots);
  if (lane == 0) start_slots(0, first_slots);

  // ---- 2. epilogue parameters to shared memory, zero accumulators.  The
  // epilogue's scalar parameters are copied to shared memory too, so their
  // constant-bank loads happen now instead of after the main loop.
  __shared__ EpiParams s_e;
  if (trace && tid == 0) trace[7] = clock64();
  if (tid == 0) s_e = P.e;
  if (has_param) {
    c_sb[tid] = p_sb;
    c_zb[tid] = p_zb;
    c_cs[tid] = p_cs;
  }
  for (int idx = tid + NWARP * 32; dequant && idx < nlrt * 16; idx += NWARP * 32) {  // > 32 row-tiles per CTA
    const int j = rt_first * kRowTile + idx;
    if (j < P.n) {
      c_sb[idx] = P.e.s_b[j * P.e.sb_stride];
      c_zb[idx] = P.e.z_b[j * P.e.zb_stride];
      c_cs[idx] = P.e.colsum_b[j];
    }
  }
  for (int idx = tid; idx < nlrt * 16 * MT; idx += NWARP * 32) accs[idx] = 0;

  // ---- 3. activations (u8 codes, B-fragment order) into shared memory
  if (FROM_PLANES) {
    for (int idx = tid; idx < MT * kpad / 4; idx += NWARP * 32) act[idx] = 0u;
    __syncthreads();
    const int ngroups = (P.k + 3) / 4;
    for (int idx = tid; idx < mb * ngroups; idx += NWARP * 32) {
      const int i = idx / ngroups, v = idx % ngroups;
      const int tok = tok0 + i;
      uint32_t word = 0;
      for (int s = 0; s < P.p; ++s) {
        const uint64_t pw = P.a_planes[(static_cast<size_t>(s) * P.m + tok) * P.wpr_a + (v >> 4)];
        const uint32_t nib = static_cast<uint32_t>(pw >> ((v & 15) * 4)) & 0xFu;
        word |= ((nib * 0x00204081u) & 0x01010101u) << s;
      }
      act[act_frag_index(v, i, MT)] = word;
    }
    if (lane == 0) start_slots(first_slots, P.slots);
  } else if (P.x16) {
    // Fused ReQuant (decode, m <= 2, fp16, per token): every CTA quantizes the
    // activation rows itself while its TMA weight ring fills -- no extra launch.
    // Row held in registers (<= 4 x 16 B per thread), min/max in fp32 (exact for
    // fp16), step / zero point in FP64 as quantizer.hpp:169-201, codes on the
    // fp32 pipe with the exact FP64 decision near ties (quant_code_f32, :205-210).
    for (int idx = tid; idx < MT * kpad / 4; idx += NWARP * 32) act[idx] = 0u;
    const int nvec = P.k >> 3;
#pragma unroll
    for (int i = 0; i < XT; ++i) {
      if (i >= mb) break;  // uniform across the CTA
      uint4 (&v)[4] = xv[i];
      float lo = CUDART_INF_F, hi = -CUDART_INF_F;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int idx = tid + r * NWARP * 32;
        if (idx < nvec) {
          const __half2* h2 = reinterpret_cast<const __half2*>(&v[r]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __half22float2(h2[e]);
            if (blockIdx.x == 0 && P.bad_out) {
              if (!isfinite(f.x)) atomicMax(P.bad_word, ~(static_cast<unsigned long long>(tok0 + i) * P.k + idx * 8 + 2 * e));
              if (!isfinite(f.y)) atomicMax(P.bad_word, ~(static_cast<unsigned long long>(tok0 + i) * P.k + idx * 8 + 2 * e + 1));
            }
            lo = fminf(lo, fminf(f.x, f.y));
            hi = fmaxf(hi, fmaxf(f.x, f.y));
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      __shared__ float q_lo[NWARP], q_hi[NWARP], q_inv;
      __shared__ int q_sum[NWARP];
      if (lane == 0) {
        q_lo[warp] = lo;
        q_hi[warp] = hi;
      }
      __syncthreads();
      if (trace && tid == 0 && i == 0) trace[10] = clock64();
      if (warp == 0) {  // row range -> step, zero point, fp32 reciprocal (one thread)
        // every lane loads (lane % NWARP): no divergence before the shuffles
        float l = q_lo[lane & (NWARP - 1)], h = q_hi[lane & (NWARP - 1)];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          l = fminf(l, __shfl_xor_sync(0xffffffffu, l, o));
          h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, o));
        }
        if (lane == 0) {
          double step;
          int z;
          group_params(P.qp, l, h, &step, &z);
          s_sa[i] = step;
          s_za[i] = z;
          q_inv = f32_reciprocal(step);
        }
      }
      __syncthreads();
      if (trace && tid == 0 && i == 0) trace[11] = clock64();
      const double step = s_sa[i];
      const float inv32 = q_inv;
      const int zi = static_cast<int>(s_za[i]), topi = static_cast<int>(P.qp.levels - 1);
      int rsum = 0;  // <= 255 K
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int idx = tid + r * NWARP * 32;
        if (idx < nvec) {
          const __half* hv = reinterpret_cast<const __half*>(&v[r]);
          uint32_t w0 = 0, w1 = 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const unsigned c = quant_code_f32(__half2float(hv[e]), step, inv32, zi, topi);
            rsum += c;
            if (e < 4) w0 |= c << (8 * e);
            else w1 |= c << (8 * (e - 4));
          }
          act[act_frag_index(2 * idx, i, MT)] = w0;
          act[act_frag_index(2 * idx + 1, i, MT)] = w1;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
      if (lane == 0) q_sum[warp] = rsum;
      __syncthreads();
      if (trace && tid == 0 && i == 0) trace[12] = clock64();
      if (warp == 0) {
        int rr = q_sum[lane & (NWARP - 1)] * (lane < NWARP ? 1 : 0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
        if (lane == 0) s_ra[i] = rr;
      }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && P.bad_out) {  // only CTA 0 reports
      const unsigned long long w = atomicExch(P.bad_word, 0ull);
      *P.bad_out = w ? ~w : ~0ull;
    }
  } else {
    griddep_wait();  // act_quant_kernel done and its writes visible
    // codes (<= 64 KB: <= 8 x 16 B per thread) and stats requested into
    // registers, then the rest of the weight ring, then the shared-memory stores
    const uint4* src = reinterpret_cast<const uint4*>(P.act_frag + static_cast<size_t>(blockIdx.y) * MT * kpad / 4);
    uint4* dst = reinterpret_cast<uint4*>(act);
    constexpr int AR = 8;
    const int nv = MT * kpad / 16;
    uint4 av[AR];
#pragma unroll
    for (int r = 0; r < AR; ++r) {
      const int idx = tid + r * NWARP * 32;
      if (idx < nv) av[r] = __ldcg(src + idx);
    }
    double t_sa = 0.0;
    long long t_za = 0, t_ra = 0;
    if (tid < mb) {
      t_sa = P.s_a[tok0 + tid];
      t_za = P.z_a[tok0 + tid];
      t_ra = P.rowsum[tok0 + tid];
    }
    if (lane == 0) start_slots(first_slots, P.slots);
#pragma unroll
    for (int r = 0; r < AR; ++r) {
      const int idx = tid + r * NWARP * 32;
      if (idx < nv) dst[idx] = av[r];
    }
    if (tid < mb) {
      s_sa[tid] = t_sa;
      s_za[tid] = t_za;
      s_ra[tid] = t_ra;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && P.bad_out) {
      const unsigned long long w = *P.bad_word;
      *P.bad_out = w ? ~w : ~0ull;
      *P.bad_word = 0ull;
    }
  }
  __syncthreads();
  if (P.late_ring && !late_act && lane == 0) start_slots(0, P.slots);
  if (trace && tid == 0) trace[1] = clock64();

  // ---- 4. main loop over this warp's units (one body, TMA ring slots)
  // one accumulator fragment: the code slices of a chunk are widened into one
  // A register set of u8 codes, so each k32 chunk costs one IMMA.
  int acc[4] = {0, 0, 0, 0};
  int cur_rt = wu0 < wu1 ? static_cast<int>(wu0 / P.kblocks) : -1;
  const uint2* act2 = reinterpret_cast<const uint2*>(act);

  auto flush = [&](int rt) {
    const int lrt = rt - rt_first;
    long long v[4];
#pragma unroll
    // the true sum is < 2^32 (K <= 65536, codes <= 255): exact as unsigned
    for (int r = 0; r < 4; ++r) v[r] = static_cast<long long>(static_cast<uint32_t>(acc[r]));
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = g + 8 * (r >> 1), tok = 2 * tig + (r & 1);
      if (tok < mb) atomicAdd(reinterpret_cast<unsigned long long*>(&accs[(lrt * 16 + row) * MT + tok]),
                              static_cast<unsigned long long>(v[r]));
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[r] = 0;
  };

  // incremental (row-tile, k-block, chunk) counters: no divisions in the loop
  int slot = 0;
  uint32_t phase = 0;
  const int uend = static_cast<int>(wu1);
  int rt = cur_rt, kb = wu0 < wu1 ? static_cast<int>(wu0 - static_cast<long long>(cur_rt) * P.kblocks) : 0;
  int ui = 0, cidx = 0;  // unit within the chunk, chunk index
  for (int uu = static_cast<int>(wu0); uu < uend; ++uu) {
    if (ui == 0) mbar_wait_parity(&my_bars[slot], phase);
    const uint4* wv = reinterpret_cast<const uint4*>(my_ring + slot * chunk_bytes + ui * unit_bytes) + lane;
    uint4 w[QT];
#pragma unroll
    for (int t = 0; t < QT; ++t) w[t] = wv[t * 32];
    const uint2* ab = act2 + static_cast<size_t>(kb) * 8 * MT * 4;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint2 b = make_uint2(0u, 0u);
      if (g < MT) b = ab[(c * MT + g) * 4 + tig];
      uint32_t a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = widen_slices<QT>(w, 4 * c + u);
      imma_16832(acc, a[0], a[1], a[2], a[3], b.x, b.y);
    }
    // chunk finished: refill its slot with the chunk `slots` ahead (the whole
    // warp has read it)
    if (++ui == P.upc || uu + 1 == uend) {
      __syncwarp();
      const int un = static_cast<int>(wu0) + (cidx + P.slots) * P.upc;  // first unit to load next
      if (lane == 0 && un < uend) {
        const int un1 = un + P.upc < uend ? un + P.upc : uend;
        const uint32_t bytes = static_cast<uint32_t>(un1 - un) * static_cast<uint32_t>(unit_bytes);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&my_bars[slot], bytes);
        tma_bulk_g2s(my_ring + slot * chunk_bytes, wsrc + static_cast<size_t>(un) * unit_bytes, bytes,
                     &my_bars[slot]);
      }
      ui = 0;
      ++cidx;
      if (++slot == P.slots) {
        slot = 0;
        phase ^= 1u;
      }
    }
    // row-tile finished: fold its plane accumulators into the CTA's sums
    if (++kb == P.kblocks) {
      flush(rt);
      kb = 0;
      ++rt;
    }
  }
  if (wu0 < wu1 && kb != 0) flush(rt);  // last row-tile was cut inside this warp's range
  __shared__ long long s_wend[NWARP];
  if (trace && lane == 0) s_wend[warp] = clock64();
  __syncthreads();
  if (trace && tid == 0) {  // earliest / latest warp finishing the main loop
    long long lo = s_wend[0], hi = s_wend[0];
    for (int w = 1; w < NWARP; ++w) {
      lo = min(lo, s_wend[w]);
      hi = max(hi, s_wend[w]);
    }
    trace[2] = lo;
    trace[6] = hi;
  }

  // ---- 5. epilogue.  Row-tiles owned by this CTA alone are stored straight
  // from shared memory; only the first / last row-tile can be cut between CTAs
  // (stream-K): their partial sums meet in the global accumulator and the last
  // arriving CTA (counter) stores them and re-zeroes the slot.
  // a row-tile is owned by this CTA alone iff all its units lie in [U0, U1)
  auto owned = [&](int rt) {
    const long long ufirst = static_cast<long long>(rt) * P.kblocks;
    return ufirst >= U0 && ufirst + P.kblocks <= U1;
  };
  auto contributors_of = [&](int rt) {  // thread 0 only: 64-bit divisions
    if (!stream_k) return 1;
    const long long ufirst = static_cast<long long>(rt) * P.kblocks;
    return cta_of_unit(ufirst + P.kblocks - 1, U, G) - cta_of_unit(ufirst, U, G) + 1;
  };
  auto store = [&](int lrt, int row, int i, long long a) {
    const int j = (rt_first + lrt) * kRowTile + row;
    if (j >= P.n) return;
    const int c = lrt * 16 + row;
    const EpiParams& E = s_e;
    if (E.mode == EPI_ACC_I32 || E.mode == EPI_ACC_I64) {
      epi_store_v(E, tok0 + i, j, a, 0.0, 0, 0);
      return;
    }
    // fused zero-point correction + dequant from the prefetched parameters
    double sa;
    long long za, ra;
    if (FROM_PLANES) {
      sa = E.s_a[(tok0 + i) * E.sa_stride];
      za = E.z_a[(tok0 + i) * E.za_stride];
      ra = E.rowsum_a[tok0 + i];
    } else {
      sa = s_sa[i];
      za = s_za[i];
      ra = s_ra[i];
    }
    const long long zb = c_zb[c];
    const long long corr = a - za * c_cs[c] - zb * ra + E.k * za * zb;
    const long long o = static_cast<long long>(tok0 + i) * E.ldo + j;
    if (E.mode == EPI_CORR_I64) {
      static_cast<int64_t*>(E.out)[o] = corr;
      return;
    }
    const double y = __dmul_rn(__dmul_rn(sa, c_sb[c]), static_cast<double>(corr));
    if (E.mode == EPI_F64)
      static_cast<double*>(E.out)[o] = y;
    else if (E.mode == EPI_F16)
      static_cast<__half*>(E.out)[o] = __double2half(y);
    else
      static_cast<float*>(E.out)[o] = __double2float_rn(y);
  };
  int nsplit = 0;
  if (trace && tid == 0) trace[4] = nlrt;
  for (int idx = tid; idx < nlrt * 16 * mb; idx += NWARP * 32) {
    const int lrt = idx / (16 * mb), rem = idx % (16 * mb), row = rem / mb, i = rem % mb;
    if (!stream_k || owned(rt_first + lrt)) store(lrt, row, i, accs[(lrt * 16 + row) * MT + i]);
  }
  if (trace && tid == 0) trace[5] = clock64();
  for (int lrt = 0; lrt < nlrt; ++lrt) {
    if (!stream_k || owned(rt_first + lrt)) continue;
    ++nsplit;
    long long* gslot = P.gacc + static_cast<size_t>(rt_first + lrt) * 16 * 8;
    for (int idx = tid; idx < 16 * mb; idx += NWARP * 32)
      atomicAdd(reinterpret_cast<unsigned long long*>(&gslot[(idx / mb) * 8 + idx % mb]),
                static_cast<unsigned long long>(accs[(lrt * 16 + idx / mb) * MT + idx % mb]));
  }
  if (trace && tid == 0) {
    trace[3] = clock64();
    trace[9] = gtimer();
  }
  if (nsplit == 0) return;  // uniform across the CTA
  __syncthreads();
  // release: one gpu-scope fence by thread 0 after the CTA barrier orders every
  // thread's partial-sum atomics before the arrival counter (fence cumulativity)
  if (tid == 0) {
    __threadfence();
    int mask = 0;
    for (int e = 0; e < 2; ++e) {  // only the first / last local row-tile can be shared
      const int lrt = e == 0 ? 0 : nlrt - 1;
      if (e == 1 && lrt == 0) break;
      const int rt = rt_first + lrt;
      const int c = contributors_of(rt);
      if (c > 1 && atomicAdd(&P.gcnt[rt], 1u) == static_cast<unsigned>(c - 1)) mask |= 1 << e;
    }
    if (mask) __threadfence();  // acquire side for the slot reads below
    s_last = mask;
  }
  __syncthreads();
  const int mask = s_last;
  for (int e = 0; e < 2; ++e) {
    if (!(mask & (1 << e))) continue;
    const int lrt = e == 0 ? 0 : nlrt - 1;
    long long* gslot = P.gacc + static_cast<size_t>(rt_first + lrt) * 16 * 8;
    for (int idx = tid; idx < 16 * mb; idx += NWARP * 32) {
      const long long a = static_cast<long long>(
          atomicExch(reinterpret_cast<unsigned long long*>(&gslot[(idx / mb) * 8 + idx % mb]), 0ull));
      store(lrt, idx / mb, idx % mb, a);
    }
    if (tid == 0) P.gcnt[rt_first + lrt] = 0u;
  }
}

// ============================================================================
// host side
// ============================================================================
size_t frag_words(unsigned q, size_t n, size_t k) {
  const size_t rowtiles = (n + kRowTile - 1) / kRowTile, kblocks = (k + kKBlock - 1) / kKBlock;
  return rowtiles * kblocks * q * 128;
}

// stream-K accumulators + counters + act codes (8 tokens) + stats + status word
size_t imma_ws_bytes(size_t n, size_t k) {
  const size_t rowtiles = (n + kRowTile - 1) / kRowTile;
  const size_t kpad = ((k + kKBlock - 1) / kKBlock) * kKBlock;
  return rowtiles * 16 * 8 * 8 + ((rowtiles * 4 + 255) & ~size_t(255)) + 8 * kpad + 8 * 24 + 256;
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

unsigned long long*& trace_buffer() {
  static unsigned long long* buf = nullptr;
  return buf;
}

static size_t imma_smem_bytes(const ImmaParams& P, int mt, int grid_x, int nwarp) {
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  const long long per_cta_units = (U + grid_x - 1) / grid_x + P.kblocks;
  const int nlrt_max = static_cast<int>(per_cta_units / P.kblocks + 2);
  return static_cast<size_t>(nwarp) * P.slots * P.upc * P.q * 512 + nwarp * P.slots * 8 +
         static_cast<size_t>(mt) * P.kblocks * kKBlock + static_cast<size_t>(nlrt_max) * 16 * mt * 8 +
         static_cast<size_t>(nlrt_max) * 16 * 24 + mt * 24 + 128;
}

// warps per CTA: 16 (512 threads) -- leaves room on every SM for the
// act_quant_kernel CTA that runs concurrently under programmatic dependent
// launch, and gives each warp a 3-deep ring of ~4 KB TMA chunks
// (profiles/r01_microbench_stream.txt: >= 4 KB bulk copies stream at ~7.2 TB/s,
// 2 KB copies at ~5 TB/s).
static int imma_warps(int q) {
  (void)q;
  return 16;
}

template <int QT, int MT, bool FROM_PLANES, int NWARP>
static int launch_imma_w(ImmaParams P, int grid_x, int grid_y, bool pdl, cudaStream_t st) {
  auto kern = gemv_imma_kernel<QT, MT, FROM_PLANES, NWARP>;
  const size_t smem = imma_smem_bytes(P, MT, grid_x, NWARP);
  if (smem > 227 * 1024) return fail(ABQ_ERR_VALUE, "gemv_imma: shared memory plan too large (%zu B)", smem);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_imma: smem attribute: %s", cudaGetErrorString(err));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid_x, grid_y);
  cfg.blockDim = dim3(NWARP * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  err = cudaLaunchKernelEx(&cfg, kern, P);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_imma: launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int QT, int MT, bool FROM_PLANES>
static int launch_imma(ImmaParams P, int grid_x, int grid_y, bool pdl, cudaStream_t st) {
  return launch_imma_w<QT, MT, FROM_PLANES, 16>(P, grid_x, grid_y, pdl, st);
}

template <int MT, bool FP>
static int launch_q(ImmaParams P, int gx, int gy, bool pdl, cudaStream_t st) {
  switch (P.q) {
    case 1: return launch_imma<1, MT, FP>(P, gx, gy, pdl, st);
    case 2: return launch_imma<2, MT, FP>(P, gx, gy, pdl, st);
    case 3: return launch_imma<3, MT, FP>(P, gx, gy, pdl, st);
    case 4: return launch_imma<4, MT, FP>(P, gx, gy, pdl, st);
    case 5: return launch_imma<5, MT, FP>(P, gx, gy, pdl, st);
    case 6: return launch_imma<6, MT, FP>(P, gx, gy, pdl, st);
    case 7: return launch_imma<7, MT, FP>(P, gx, gy, pdl, st);
    default: return launch_imma<8, MT, FP>(P, gx, gy, pdl, st);
  }
}

template <bool FP>
static int launch_mt(ImmaParams P, int mt, int gx, int gy, bool pdl, cudaStream_t st) {
  switch (mt) {
    case 1: return launch_q<1, FP>(P, gx, gy, pdl, st);
    case 2: return launch_q<2, FP>(P, gx, gy, pdl, st);
    case 4: return launch_q<4, FP>(P, gx, gy, pdl, st);
    default: return launch_q<8, FP>(P, gx, gy, pdl, st);
  }
}

static int pick_imma_mt(int m) { return m >= 5 ? 8 : (m >= 3 ? 4 : m); }

// activations + stats for 8 tokens must fit next to a minimal weight ring
bool imma_supported(size_t m, size_t k) {
  (void)m;
  const size_t kpad = ((k + kKBlock - 1) / kKBlock) * kKBlock;
  return k > 0 && k <= 65536 && 8 * kpad <= 64 * 1024;
}

static void plan_grid(ImmaParams& P, int mt, bool stream_k, int* gx) {
  const int nwarp = imma_warps(P.q);
  const long long U = static_cast<long long>(P.rowtiles) * P.kblocks;
  if (stream_k)  // stream-K over units; keep >= one unit per warp per CTA
    *gx = static_cast<int>(std::min<long long>(num_sms(), std::max<long long>(1, U / nwarp)));
  else
    *gx = std::min(num_sms(), P.rowtiles);
  // TMA chunks of ~4 KB (whole units), ring as deep as shared memory allows (<= 4)
  const int unit = P.q * 512;
  P.upc = unit >= 4096 ? 1 : 4096 / unit;
  P.slots = 1;
  for (int s = 4; s >= 2; --s) {
    P.slots = s;
    if (imma_smem_bytes(P, mt, *gx, nwarp) <= 220 * 1024) break;
  }
}

static ImmaParams base_params(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m,
                              const EpiParams& e) {
  ImmaParams P{};
  P.frag = frag;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  P.kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  P.m = static_cast<int>(m);
  P.e = e;
  P.trace = trace_buffer();
  return P;
}

// API path: activations given as planes (+ s_a/z_a/rowsum in e); row-tile split.
int run_gemv_imma_planes(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m,
                         const uint64_t* a_planes, unsigned p, const EpiParams& e, cudaStream_t st) {
  if (m == 0 || n == 0) return ABQ_OK;
  ImmaParams P = base_params(frag, q, n, k, m, e);
  P.a_planes = a_planes;
  P.p = static_cast<int>(p);
  P.wpr_a = static_cast<int>(wpr_of(k));
  const int mt = pick_imma_mt(static_cast<int>(m));
  int gx;
  plan_grid(P, mt, false, &gx);
  const int gy = static_cast<int>((m + mt - 1) / mt);
  return launch_mt<true>(P, mt, gx, gy, false, st);
}

// K1 launcher: one CTA per token.  row_ld == 0: B-fragment order for the decode
// GEMV (token blocks of mt); row_ld > 0: the tcgen05 GEMM's tiled operand with
// row_ld = tc_act_groups(m) token groups (k % 16 == 0).  bad_word: zero-initialised, receives atomicMax(~index).
int run_act_quant(const void* x, int x_dtype, size_t m, size_t k, int mt, const QuantParams& qp,
                  uint32_t* out, int row_ld, double* s_a, int32_t* z_a, long long* rowsum,
                  unsigned long long* bad_word, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>(m)), block(kActThreads);
  const int im = static_cast<int>(m), ik = static_cast<int>(k);
#define ABQ_ACTQ(T, ROWL, VR)                                                                                  \
  act_quant_kernel<T, ROWL, VR><<<grid, block, 0, st>>>(static_cast<const T*>(x), im, ik, mt, qp, out, row_ld, s_a, \
                                                       z_a, rowsum, bad_word)
  const bool row = row_ld > 0;
  // vectors per thread of the fp16 fast path: 4 (K <= 8192), 8 (<= 16384), 16 (<= 32768)
  const int vr = k <= static_cast<size_t>(8 * 4 * kActThreads) ? 4 : k <= static_cast<size_t>(8 * 8 * kActThreads) ? 8 : 16;
  switch (x_dtype) {
    case ABQ_F16:
      if (vr == 16) {
        if (row) ABQ_ACTQ(__half, true, 16); else ABQ_ACTQ(__half, false, 16);
      } else if (vr == 8) {
        if (row) ABQ_ACTQ(__half, true, 8); else ABQ_ACTQ(__half, false, 8);
      } else {
        if (row) ABQ_ACTQ(__half, true, 4); else ABQ_ACTQ(__half, false, 4);
      }
      break;
    case ABQ_F32:
      if (row) ABQ_ACTQ(float, true, 4); else ABQ_ACTQ(float, false, 4);
      break;
    default:
      if (row) ABQ_ACTQ(double, true, 4); else ABQ_ACTQ(double, false, 4);
      break;
  }
#undef ABQ_ACTQ
  ABQ_LAUNCHED();
  return ABQ_OK;
}

}  // namespace abq_dev
