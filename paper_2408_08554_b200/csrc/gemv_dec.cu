// gemv_dec.cu -- K2 serving decode GEMV (M <= 8 tokens), sm_100a.
//
// One launch per linear layer: fp16 activations -> per-token ReQuant (FP64
// semantics of quantizer.hpp:146-213) -> exact code product
// acc[i][j] = sum_k a_ik * w_jk over the q-bit weight codes (the value of
// gemm_arbitrary, include/abq/gemm.hpp:150-198) -> zero-point correction +
// dequant (gemm.hpp:235-254, 292-306) -> fp16 / fp32 / fp64 output.
//
// Weights: the fragment-major code-slice layout built once by
// prepack_frag_kernel (gemv_imma.cu): unit (row-tile of 16, k-block of 256) =
// q x 512 contiguous bytes, units ordered row-tile-major.  Same byte count as
// the ABQP planes.
//
// Designed around three measurements (profiles/r01_microbench_burst.txt,
// profiles/r01_trace_gemv.txt):
//  * a memory access issued by an SM while ~200 KB per SM of weight stream is
//    queued waits ~0.8 us even when it hits L2 (64 KB in flight: ~0.33 us), so
//    the kernel keeps a bounded ring (~64-96 KB per CTA) and issues every
//    prologue load (parameters, per-channel epilogue values, activations) in
//    one batch;
//  * back-to-back launches lose ~1.5-2 us each to launch + ramp; with
//    programmatic dependent launch and two co-resident CTAs per SM the next
//    layer's CTA starts streaming its (input-independent) weights during this
//    layer's tail -- it only waits (griddepcontrol.wait) before it reads the
//    activations and before it writes anything;
//  * a single IMMA accumulator chain per warp runs at ~45 cycles per IMMA;
//    four independent chains per warp.
//
// CTA = 8 consumer warps + 1 producer warp.  The producer streams the CTA's
// contiguous unit range [U0, U1) (stream-K split, balanced to one unit)
// through a ring of S slots of 8 units with 1-D TMA bulk copies (full / empty
// mbarriers); consumer warp w multiplies unit w of every slot on the int8
// tensor pipe (legacy IMMA m16n8k32: 16 weight rows x 32 k x 8 tokens).
// Row-tile partial sums meet in shared memory; the (at most two) row-tiles cut
// between CTAs meet in a self-cleaning global accumulator and the last
// contributing CTA runs the epilogue for them.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemv_frag.cuh"
#include "quant_dev.cuh"

namespace abq_dev {

constexpr int kDecWarps = 16;  // consumer warps (4 per SM sub-partition: the loop is latency-bound)
constexpr int kDecUPS = 8;     // units per ring slot = consumer warps sharing one slot
constexpr int kDecThreads = (kDecWarps + 1) * 32;

struct DecParams {
  const uint32_t* frag;
  int q, n, k, rowtiles, kblocks, m;
  int slots;       // ring slots of kDecUPS units
  int U;           // rowtiles * kblocks
  // activations: fp16 rows quantized in the prologue, or codes + stats written
  // by act_quant_kernel (the PDL primary of this launch)
  const __half* x16;
  const uint32_t* act_frag;
  const double* s_a;
  const int32_t* z_a;
  const long long* rowsum;
  QuantParams qp;
  EpiParams e;
  long long* gacc;               // [rowtiles][16][8] int64, zero on entry and exit
  unsigned* gcnt;                // [rowtiles], zero on entry and exit
  unsigned long long* bad_word;  // non-finite input report (see run_gemv_dec)
  unsigned long long* bad_out;
  unsigned long long* trace;     // optional [grid][64] stamps (tools/trace_dec.py)
  int rowsplit;                  // 1: CTAs own whole row-tiles (no cross-CTA sums); 0: stream-K
};

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// named barrier over the consumer warps only (the producer never joins)
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kDecWarps * 32) : "memory");
}

struct DecSmem {  // carve-up of the dynamic shared memory (host and device agree)
  size_t ring, bars, act, accs, csb, czb, ccs, total;
};
__host__ __device__ inline DecSmem dec_smem(int q, int slots, int mt, int kpad, int nlrt_max) {
  DecSmem s;
  s.ring = 0;
  s.bars = s.ring + static_cast<size_t>(slots) * kDecUPS * q * 512;
  s.act = s.bars + static_cast<size_t>(2 * slots) * 8;
  s.accs = (s.act + static_cast<size_t>(mt) * kpad + 15) & ~size_t(15);
  s.csb = (s.accs + static_cast<size_t>(nlrt_max) * 16 * mt * 4 + 15) & ~size_t(15);
  s.czb = s.csb + static_cast<size_t>(nlrt_max) * 16 * 8;
  s.ccs = s.czb + static_cast<size_t>(nlrt_max) * 16 * 8;
  s.total = s.ccs + static_cast<size_t>(nlrt_max) * 16 * 8;
  return s;
}
__host__ __device__ inline int dec_nlrt_max(int U, int grid, int kblocks) {
  return (U + grid - 1) / grid / kblocks + 2;
}

// non-finite inputs of one thread's vectors -> atomicMax(~flat index) (the
// smallest bad index wins); out of line: it only runs when one was seen
static __device__ __noinline__ void report_nonfinite_f16(const uint4* xr, int t, int l, int tpt, int nvec, int k,
                                                         unsigned long long* bad_word) {
  for (int v = l; v < nvec; v += tpt) {
    const uint4 q = xr[v];
    const __half* h = reinterpret_cast<const __half*>(&q);
    for (int e = 0; e < 8; ++e)
      if (!isfinite(__half2float(h[e])))
        atomicMax(bad_word, ~(static_cast<unsigned long long>(t) * k + static_cast<unsigned long long>(v) * 8 + e));
  }
}

template <int QT, int MT, int MINB>
__global__ void __launch_bounds__(kDecThreads, MINB) gemv_dec_kernel(const __grid_constant__ DecParams Pc) {
  constexpr int NW = kDecWarps, UPS = kDecUPS, NG = NW / UPS;
  constexpr int unit_bytes = QT * 512;
  constexpr int slot_bytes = UPS * unit_bytes;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) DecParams P;  // consumers' copy of the parameter block (below)
  __shared__ float r_lo[NW], r_hi[NW];
  __shared__ int r_sum[NW];
  __shared__ double s_sa[MT];
  __shared__ long long s_za[MT], s_ra[MT];
  __shared__ float s_inv[MT];
  __shared__ int s_last;
  __shared__ long long s_wend;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  asm volatile("griddepcontrol.launch_dependents;");

  // this CTA's unit range: whole row-tiles, or an even stream-K share
  // Scalars of the parameter block go through a warp shuffle: left to itself
  // ptxas re-reads them from the constant bank inside the loops (LDC on every
  // iteration), and a constant-cache miss behind the weight stream costs a
  // memory round trip.
  const int G = gridDim.x, U = __shfl_sync(0xffffffffu, Pc.U, 0), kblocks = __shfl_sync(0xffffffffu, Pc.kblocks, 0);
  const int S = __shfl_sync(0xffffffffu, Pc.slots, 0), rowsplit = __shfl_sync(0xffffffffu, Pc.rowsplit, 0);
  const int rowtiles = __shfl_sync(0xffffffffu, Pc.rowtiles, 0);
  const int kpad = kblocks * kKBlock;
  int U0, U1;
  if (rowsplit) {
    U0 = static_cast<int>(static_cast<long long>(blockIdx.x) * rowtiles / G) * kblocks;
    U1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * rowtiles / G) * kblocks;
  } else {
    U0 = static_cast<int>(static_cast<long long>(blockIdx.x) * U / G);
    U1 = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * U / G);
  }
  const int nsl = (U1 - U0 + UPS - 1) / UPS;
  const DecSmem L = dec_smem(QT, S, MT, kpad, dec_nlrt_max(U, G, kblocks));
  unsigned char* ring = smem + L.ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + S;

  // ======================= producer warp: the weight stream ==================
  // Starts at once, from the constant bank; the consumers meet it at named
  // barrier 2 (its arrival publishes the mbarrier initialisation).
  if (warp == NW) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init_n(&full[s], 1);
        mbar_init_n(&empty[s], UPS);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("bar.arrive 2, %0;" ::"n"(kDecThreads) : "memory");
    if (lane == 0) {
      const unsigned char* src = reinterpret_cast<const unsigned char*>(Pc.frag) + static_cast<size_t>(U0) * unit_bytes;
      const uint64_t pol = l2_evict_first_policy();
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nsl; ++i) {
        if (i >= S) mbar_wait_parity(&empty[s], ph ^ 1u);
        const int nu = min(UPS, U1 - U0 - i * UPS);
        const uint32_t bytes = static_cast<uint32_t>(nu * unit_bytes);
        mbar_expect_tx(&full[s], bytes);
        tma_bulk_g2s_hint(ring + static_cast<size_t>(s) * slot_bytes, src + static_cast<size_t>(i) * slot_bytes,
                          bytes, &full[s], pol);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }

  // consumers: the parameter block to shared memory, all threads at once (read
  // lazily from the constant bank, each first touch of a constant-cache line
  // would be a separate memory round trip behind the weight stream)
  for (int i = tid; i < static_cast<int>(sizeof(DecParams) / 4); i += NW * 32)
    reinterpret_cast<uint32_t*>(&P)[i] = reinterpret_cast<const uint32_t*>(&Pc)[i];
  asm volatile("bar.sync 2, %0;" ::"n"(kDecThreads) : "memory");
  unsigned long long* trace = P.trace ? P.trace + 64 * blockIdx.x : nullptr;
  if (trace && tid == 0) {
    trace[0] = clock64();
    trace[8] = gtimer();
    s_wend = 0;
  }
  const int rt_first = U0 / kblocks;
  const int rt_last = U1 > U0 ? (U1 - 1) / kblocks : rt_first - 1;
  const int nlrt = rt_last - rt_first + 1;
  uint32_t* act = reinterpret_cast<uint32_t*>(smem + L.act);
  uint32_t* accs = reinterpret_cast<uint32_t*>(smem + L.accs);
  double* c_sb = reinterpret_cast<double*>(smem + L.csb);
  long long* c_zb = reinterpret_cast<long long*>(smem + L.czb);
  long long* c_cs = reinterpret_cast<long long*>(smem + L.ccs);

  // ======================= consumer warps ===================================
  const bool dequant = P.e.mode != EPI_ACC_I32 && P.e.mode != EPI_ACC_I64;
  const int tok_n = min(MT, P.m);
  // ---- prologue loads, one batch: epilogue parameters of this CTA's channels
  // (weight side: legal before the dependency wait) ...
  constexpr int kCT = NW * 32;
  for (int idx = tid; dequant && idx < nlrt * 16; idx += kCT) {
    const int j = rt_first * kRowTile + idx;
    if (j < P.n) {
      c_sb[idx] = P.e.s_b[static_cast<size_t>(j) * P.e.sb_stride];
      c_zb[idx] = P.e.z_b[static_cast<size_t>(j) * P.e.zb_stride];
      c_cs[idx] = P.e.colsum_b[j];
    }
  }
  for (int idx = tid; idx < nlrt * 16 * MT; idx += kCT) accs[idx] = 0;
  if (P.x16) {  // codes past K (to the k-block multiple) are zero
    const int k4 = P.k >> 2, ntail = (kpad >> 2) - k4;
    for (int idx = tid; idx < ntail * MT; idx += kCT) act[act_frag_index(k4 + idx / MT, idx % MT, MT)] = 0u;
  }
  // ... then the activations, which the previous kernel may still be producing
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trace && tid == 0) trace[4] = clock64();

  if (P.x16) {
    // Fused ReQuant, per token, fp16 rows (K % 8 == 0, K <= 64 * TPT: the
    // host routes longer rows through act_quant_kernel).  GT warps per token;
    // each thread loads its (<= 8) 16-byte vectors of the row in one batch and
    // keeps them in registers for both passes.
    constexpr int GT = NW / MT;  // MT is a power of two <= NW
    constexpr int TPT = GT * 32;
    constexpr int XR = 8;
    const int t = warp / GT;
    const int l = (warp % GT) * 32 + lane;
    const int nvec = P.k >> 3;
    const bool active = t < tok_n;
    const uint4* xr = reinterpret_cast<const uint4*>(P.x16 + static_cast<size_t>(t) * P.k);
    uint4 xv[XR];
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      const int v = l + r * TPT;
      xv[r] = active && v < nvec ? __ldg(xr + v) : make_uint4(0u, 0u, 0u, 0u);
    }
    float lo = CUDART_INF_F, hi = -CUDART_INF_F;
    uint32_t bad = 0;
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      if (!active || l + r * TPT >= nvec) break;
      bad |= f16x8_nonfinite(xv[r]);
      const __half2* h2 = reinterpret_cast<const __half2*>(&xv[r]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h2[e]);
        lo = fminf(lo, fminf(f.x, f.y));
        hi = fmaxf(hi, fmaxf(f.x, f.y));
      }
    }
    const bool report = blockIdx.x == 0 && P.bad_out != nullptr;
    if (report && bad) report_nonfinite_f16(xr, t, l, TPT, nvec, P.k, P.bad_word);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      r_lo[warp] = lo;
      r_hi[warp] = hi;
    }
    consumers_sync();
    if (trace && tid == 0) trace[5] = clock64();
    if (active && warp % GT == 0 && lane == 0) {
      float l2 = r_lo[warp], h2 = r_hi[warp];
      for (int w = 1; w < GT; ++w) {
        l2 = fminf(l2, r_lo[warp + w]);
        h2 = fmaxf(h2, r_hi[warp + w]);
      }
      double step;
      int z;
      group_params(P.qp, l2, h2, &step, &z);
      s_sa[t] = step;
      s_za[t] = z;
      s_inv[t] = f32_reciprocal(step);
    }
    consumers_sync();
    if (trace && tid == 0) trace[6] = clock64();
    int rsum = 0;
    if (active) {
      const double step = s_sa[t];
      const float inv32 = s_inv[t];
      const int zi = static_cast<int>(s_za[t]), topi = static_cast<int>(P.qp.levels - 1);
#pragma unroll
      for (int r = 0; r < XR; ++r) {
        const int v = l + r * TPT;
        if (v >= nvec) break;
        uint32_t w0, w1;
        rsum += quant_codes8_f16(xv[r], step, inv32, zi, topi, &w0, &w1);
        act[act_frag_index(2 * v, t, MT)] = w0;
        act[act_frag_index(2 * v + 1, t, MT)] = w1;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
    if (lane == 0) r_sum[warp] = rsum;
    consumers_sync();
    if (active && warp % GT == 0 && lane == 0) {
      long long rr = 0;
      for (int w = 0; w < GT; ++w) rr += r_sum[warp + w];
      s_ra[t] = rr;
    }
    if (report && tid == 0) {
      const unsigned long long w = atomicExch(P.bad_word, 0ull);
      *P.bad_out = w ? ~w : ~0ull;
    }
  } else {
    // codes + stats from act_quant_kernel
    const uint4* src = reinterpret_cast<const uint4*>(P.act_frag);
    uint4* dst = reinterpret_cast<uint4*>(act);
    const int nv = MT * kpad / 16;  // act_quant_kernel zero-fills codes past K
    for (int idx = tid; idx < nv; idx += kCT) dst[idx] = __ldcg(src + idx);
    if (tid < tok_n) {
      s_sa[tid] = P.s_a[tid];
      s_za[tid] = P.z_a[tid];
      s_ra[tid] = P.rowsum[tid];
    }
    if (blockIdx.x == 0 && tid == 0 && P.bad_out) {
      const unsigned long long w = *P.bad_word;
      *P.bad_out = w ? ~w : ~0ull;
      *P.bad_word = 0ull;
    }
  }
  consumers_sync();
  if (trace && tid == 0) trace[1] = clock64();

  // ---- main loop.  Slot i holds units U0 + i*UPS .. +UPS-1; warp group
  // grp = warp / UPS takes the slots i = grp (mod NG), warp w % UPS its unit.
  // Two register buffers: the next slot's weights are requested before the
  // current unit's IMMAs issue.  No parameter-block reads in here.
  const int g = lane >> 2, tig = lane & 3;
  const int grp = warp / UPS, wi = warp % UPS;
  int acc[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[c][r] = 0;
  auto flush = [&](int r_t) {
    const int lrt = r_t - rt_first;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // the true row-tile sum is < 2^32 (K <= 65536, codes <= 255): exact as unsigned
      const uint32_t v = static_cast<uint32_t>(acc[0][r]) + static_cast<uint32_t>(acc[1][r]) +
                         static_cast<uint32_t>(acc[2][r]) + static_cast<uint32_t>(acc[3][r]);
      acc[0][r] = acc[1][r] = acc[2][r] = acc[3][r] = 0;
      const int row = g + 8 * (r >> 1), tok = 2 * tig + (r & 1);
      if (tok < tok_n) atomicAdd(&accs[(lrt * 16 + row) * MT + tok], v);
    }
  };
  const uint32_t ring_lane = smem_addr(ring) + wi * unit_bytes + lane * 16;
  const uint32_t act_lane = smem_addr(act) + ((g * 4 + tig) * 8);  // B-fragment word pair of (g, tig)
  const bool has_b = g < MT;
  auto wait_full = [&](int sl, uint32_t ph) { mbar_wait_parity(&full[sl], ph); };
  auto lds_unit = [&](int sl, uint4 (&w)[QT]) {
    const uint32_t a = ring_lane + sl * slot_bytes;
#pragma unroll
    for (int t = 0; t < QT; ++t)
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w) : "r"(a + t * 512));
  };
  int cur_rt = -1;
  auto compute = [&](int r_t, int k_b, const uint4 (&w)[QT]) {
    if (r_t != cur_rt) {
      if (cur_rt >= 0) flush(cur_rt);
      cur_rt = r_t;
    }
    uint2 b[8];
    const uint32_t ab = act_lane + k_b * (8 * MT * 4 * 8);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      b[c] = make_uint2(0u, 0u);
      if (has_b) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(b[c].x), "=r"(b[c].y) : "r"(ab + c * MT * 32));
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = widen_slices<QT>(w, 4 * c + r);
      imma_16832(acc[c & 3], a[0], a[1], a[2], a[3], b[c].x, b[c].y);
    }
  };
  {
    constexpr int STEP = NG * UPS;  // units between a warp's consecutive slots
    int i = grp, s = grp;           // NG <= S (host plan)
    uint32_t ph = 0;
    int u = U0 + i * UPS + wi;
    int rt = u / kblocks, kb = u - rt * kblocks;
    auto advance = [&]() {
      i += NG;
      s += NG;
      if (s >= S) {
        s -= S;
        ph ^= 1u;
      }
      u += STEP;
      kb += STEP;
      while (kb >= kblocks) {
        kb -= kblocks;
        ++rt;
      }
    };
    auto release = [&](int sl) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    };
    uint4 wa[QT], wb[QT];
    if (i < nsl) {
      wait_full(s, ph);
      if (u < U1) lds_unit(s, wa);
    }
    while (i < nsl) {
      // iteration A: compute wa, prefetch the next slot into wb
      {
        const int s0 = s, rt0 = rt, kb0 = kb;
        const bool v0 = u < U1;
        advance();
        if (i < nsl) {
          wait_full(s, ph);
          if (u < U1) lds_unit(s, wb);
        }
        if (v0) compute(rt0, kb0, wa);
        release(s0);
      }
      if (i >= nsl) break;
      // iteration B: compute wb, prefetch into wa
      {
        const int s0 = s, rt0 = rt, kb0 = kb;
        const bool v0 = u < U1;
        advance();
        if (i < nsl) {
          wait_full(s, ph);
          if (u < U1) lds_unit(s, wa);
        }
        if (v0) compute(rt0, kb0, wb);
        release(s0);
      }
    }
  }
  if (cur_rt >= 0) flush(cur_rt);
  if (trace && lane == 0) atomicMax(&s_wend, static_cast<long long>(clock64()));
  consumers_sync();
  if (trace && tid == 0) trace[2] = s_wend;

  // ---- epilogue
  const bool stream_k = P.gacc != nullptr;
  auto owned = [&](int r) {
    const int ufirst = r * kblocks;
    return ufirst >= U0 && ufirst + kblocks <= U1;
  };
  const EpiParams& E = P.e;
  auto store = [&](int lrt, int row, int i, long long a) {
    const int j = (rt_first + lrt) * kRowTile + row;
    if (j >= P.n) return;
    if (!dequant) {
      epi_store_v(E, i, j, a, 0.0, 0, 0);
      return;
    }
    const int c = lrt * 16 + row;
    const long long za = s_za[i], zb = c_zb[c];
    const long long corr = a - za * c_cs[c] - zb * s_ra[i] + E.k * za * zb;
    const long long o = static_cast<long long>(i) * E.ldo + j;
    if (E.mode == EPI_CORR_I64) {
      static_cast<int64_t*>(E.out)[o] = corr;
      return;
    }
    const double y = __dmul_rn(__dmul_rn(s_sa[i], c_sb[c]), static_cast<double>(corr));
    if (E.mode == EPI_F64)
      static_cast<double*>(E.out)[o] = y;
    else if (E.mode == EPI_F16)
      static_cast<__half*>(E.out)[o] = __double2half(y);
    else
      static_cast<float*>(E.out)[o] = __double2float_rn(y);
  };
  for (int idx = tid; idx < nlrt * 16 * MT; idx += kCT) {
    const int i = idx & (MT - 1), rc = idx / MT, lrt = rc >> 4;
    if (i < tok_n && (!stream_k || owned(rt_first + lrt))) store(lrt, rc & 15, i, accs[idx]);
  }
  int nsplit = 0;
  for (int lrt = 0; lrt < nlrt; ++lrt) {
    if (!stream_k || owned(rt_first + lrt)) continue;
    ++nsplit;
    long long* gslot = P.gacc + static_cast<size_t>(rt_first + lrt) * 16 * 8;
    for (int idx = tid; idx < 16 * tok_n; idx += kCT)
      atomicAdd(reinterpret_cast<unsigned long long*>(&gslot[(idx / tok_n) * 8 + idx % tok_n]),
                static_cast<unsigned long long>(accs[(lrt * 16 + idx / tok_n) * MT + idx % tok_n]));  // u32 partial
  }
  if (trace && tid == 0) {
    trace[3] = clock64();
    trace[9] = gtimer();
  }
  if (nsplit == 0) return;  // uniform across the consumer warps
  consumers_sync();
  // release: thread 0's gpu-scope fence after the barrier orders every consumer
  // thread's partial-sum atomics before its arrival on the counter
  if (tid == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    int mask = 0;
    for (int e = 0; e < 2; ++e) {  // only the first / last local row-tile can be shared
      const int lrt = e == 0 ? 0 : nlrt - 1;
      if (e == 1 && lrt == 0) break;
      const int r = rt_first + lrt;
      if (owned(r)) continue;
      // contributing CTAs of row-tile r under the split floor(b*U/G)
      const long long uf = static_cast<long long>(r) * kblocks, ul = uf + kblocks - 1;
      const int c = static_cast<int>(((ul + 1) * G - 1) / U) - static_cast<int>(((uf + 1) * G - 1) / U) + 1;
      if (c > 1 && atomicAdd(&P.gcnt[r], 1u) == static_cast<unsigned>(c - 1)) mask |= 1 << e;
    }
    if (mask) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire side for the slot reads below
    s_last = mask;
  }
  consumers_sync();
  const int mask = s_last;
  for (int e = 0; e < 2; ++e) {
    if (!(mask & (1 << e))) continue;
    const int lrt = e == 0 ? 0 : nlrt - 1;
    long long* gslot = P.gacc + static_cast<size_t>(rt_first + lrt) * 16 * 8;
    for (int idx = tid; idx < 16 * tok_n; idx += kCT) {
      const long long a = static_cast<long long>(
          atomicExch(reinterpret_cast<unsigned long long*>(&gslot[(idx / tok_n) * 8 + idx % tok_n]), 0ull));
      store(lrt, idx / tok_n, idx % tok_n, a);
    }
    if (tid == 0) P.gcnt[rt_first + lrt] = 0u;
  }
}

// ============================================================================
// host side
// ============================================================================
unsigned long long*& trace_buffer();

struct DecPlan {
  int grid, slots, minb;
  size_t smem;
};

// Ring of ~80 KB in flight per CTA; two CTAs per SM when the plan fits in
// half the shared memory (so the next launch can stream during this one's tail).
static DecPlan plan_dec(int q, int mt, int kpad, int U, int kblocks, int grid) {
  DecPlan p{};
  p.grid = grid;
  const int nl = dec_nlrt_max(U, p.grid, kblocks);
  const int slot_bytes = kDecUPS * q * 512;
  int target = 96 * 1024;
  if (const char* env = std::getenv("ABQ_DEC_RING_KB")) target = std::atoi(env) * 1024;
  const int min_slots = kDecWarps / kDecUPS;  // every warp group needs its own slot
  int slots = std::max(min_slots, std::min(16, target / slot_bytes));
  p.minb = 1;
  while (slots > min_slots && dec_smem(q, slots, mt, kpad, nl).total > 220 * 1024) --slots;
  p.slots = slots;
  p.smem = dec_smem(q, slots, mt, kpad, nl).total;
  return p;
}

template <int QT, int MT, int MINB>
static int launch_dec3(const DecParams& P, const DecPlan& pl, bool pdl, cudaStream_t st) {
  auto kern = gemv_dec_kernel<QT, MT, MINB>;
  if (pl.smem > 220 * 1024) return fail(ABQ_ERR_VALUE, "gemv_dec: shared memory plan too large (%zu B)", pl.smem);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem));
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_dec: smem attribute: %s", cudaGetErrorString(err));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.grid);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  err = cudaLaunchKernelEx(&cfg, kern, P);
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_dec: launch: %s", cudaGetErrorString(err));
  ABQ_LAUNCHED();
  return ABQ_OK;
}

template <int QT, int MT>
static int launch_dec2(const DecParams& P, const DecPlan& pl, bool pdl, cudaStream_t st) {
  return launch_dec3<QT, MT, 1>(P, pl, pdl, st);
}

template <int MT>
static int launch_dec1(const DecParams& P, const DecPlan& pl, bool pdl, cudaStream_t st) {
  switch (P.q) {
    case 1: return launch_dec2<1, MT>(P, pl, pdl, st);
    case 2: return launch_dec2<2, MT>(P, pl, pdl, st);
    case 3: return launch_dec2<3, MT>(P, pl, pdl, st);
    case 4: return launch_dec2<4, MT>(P, pl, pdl, st);
    case 5: return launch_dec2<5, MT>(P, pl, pdl, st);
    case 6: return launch_dec2<6, MT>(P, pl, pdl, st);
    case 7: return launch_dec2<7, MT>(P, pl, pdl, st);
    default: return launch_dec2<8, MT>(P, pl, pdl, st);
  }
}

int run_act_quant(const void* x, int x_dtype, size_t m, size_t k, int mt, const QuantParams& qp,
                  uint32_t* out, int row_ld, double* s_a, int32_t* z_a, long long* rowsum,
                  unsigned long long* bad_word, cudaStream_t st);

// Serving decode path (m <= 8).  `ws` = imma_ws_bytes(n, k) of zero-filled
// device memory (left zeroed): stream-K accumulators, counters, activation
// codes, stats, the non-finite report word.  fp16 per-token activations with
// K % 8 == 0 are quantized inside the GEMV (one launch); anything else goes
// through act_quant_kernel first, with this kernel as its PDL secondary.
// Every launch is itself PDL-enabled so consecutive layers overlap.
int run_gemv_dec(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const void* x, int x_dtype,
                 const QuantParams& qp, const EpiParams& e, void* ws, unsigned long long* bad_out,
                 cudaStream_t st) {
  if (m == 0 || n == 0) return ABQ_OK;
  if (m > 8) return fail(ABQ_ERR_VALUE, "gemv_dec: m <= 8 only");
  DecParams P{};
  P.frag = frag;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  P.kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  P.m = static_cast<int>(m);
  P.U = P.rowtiles * P.kblocks;
  P.e = e;
  P.qp = qp;
  P.trace = trace_buffer();
  const int mt = m <= 1 ? 1 : m <= 2 ? 2 : m <= 4 ? 4 : 8;
  const int kpad = P.kblocks * kKBlock;
  char* w = static_cast<char*>(ws);
  P.gacc = reinterpret_cast<long long*>(w);
  w += static_cast<size_t>(P.rowtiles) * 16 * 8 * 8;
  P.gcnt = reinterpret_cast<unsigned*>(w);
  w += (static_cast<size_t>(P.rowtiles) * 4 + 255) & ~size_t(255);
  uint32_t* act_frag = reinterpret_cast<uint32_t*>(w);
  w += 8 * static_cast<size_t>(kpad);
  double* s_a = reinterpret_cast<double*>(w);
  int32_t* z_a = reinterpret_cast<int32_t*>(w + 64);
  long long* rowsum = reinterpret_cast<long long*>(w + 128);
  P.bad_word = reinterpret_cast<unsigned long long*>(w + 192);
  P.bad_out = bad_out;
  // fused ReQuant: each of the NW*32/mt threads of a token holds <= 8 vectors of 8
  const bool fused = x_dtype == ABQ_F16 && !qp.per_tensor && k % 8 == 0 &&
                     k <= static_cast<size_t>(64 * kDecWarps * 32 / mt);
  if (fused) {
    P.x16 = static_cast<const __half*>(x);
  } else {
    const int rc = run_act_quant(x, x_dtype, m, k, mt, qp, act_frag, 0, s_a, z_a, rowsum, P.bad_word, st);
    if (rc) return rc;
    P.act_frag = act_frag;
    P.s_a = s_a;
    P.z_a = z_a;
    P.rowsum = rowsum;
  }
  // CTAs own whole row-tiles unless that leaves SMs idle (few row-tiles): the
  // cross-CTA reduction of stream-K costs ~3 dependent global round trips
  P.rowsplit = P.rowtiles >= num_sms() ? 1 : 0;
  if (const char* env = std::getenv("ABQ_DEC_STREAMK")) P.rowsplit = env[0] == '1' ? 0 : 1;
  if (P.rowsplit) {
    P.gacc = nullptr;
    P.gcnt = nullptr;
  }
  const int grid = P.rowsplit ? std::min(num_sms(), P.rowtiles) : std::max(1, std::min(num_sms(), P.U / kDecUPS));
  const DecPlan pl = plan_dec(P.q, mt, kpad, P.U, P.kblocks, grid);
  P.slots = pl.slots;
  bool pdl = true;
  if (const char* env = std::getenv("ABQ_DEC_PDL")) pdl = env[0] == '1';
  switch (mt) {
    case 1: return launch_dec1<1>(P, pl, pdl, st);
    case 2: return launch_dec1<2>(P, pl, pdl, st);
    case 4: return launch_dec1<4>(P, pl, pdl, st);
    default: return launch_dec1<8>(P, pl, pdl, st);
  }
}

}  // namespace abq_dev
