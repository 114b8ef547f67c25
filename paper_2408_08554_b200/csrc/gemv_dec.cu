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
// Shape of the kernel (measurements: profiles/r01_microbench_burst.txt,
// r01_microbench_sync.txt, r01_trace_dec_*.txt):
//  * each CTA owns whole row-tiles (no cross-CTA reduction) and, first thing,
//    asks L2 to prefetch its entire weight range with bulk prefetches
//    (cp.async.bulk.prefetch.L2, evict-first): HBM streams at full rate while
//    the CTA quantizes the activations, with no shared-memory or register
//    cost; the weights are then read with 16-byte loads that hit L2;
//  * 16 warps, one IMMA m16n8k32 (16 weight rows x 32 k x 8 tokens) stream
//    per warp over units U0 + warp + 16 j, D units of loads in flight per warp;
//  * power-of-two code slices (q = 1, 2, 4, 8) are fed to IMMA as raw masked
//    bytes (w & (mask << w*f)): one ALU op per A register, the field's 2^(w f)
//    scale divided out exactly at the row-tile flush; other q widen the slices
//    to byte codes;
//  * launches are programmatic-dependent: parameters and weights are fetched
//    before griddepcontrol.wait, the activations after it.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemv_frag.cuh"
#include "quant_dev.cuh"

namespace abq_dev {

constexpr int kDecWarps = 16;  // 4 per SM sub-partition, <= 128 registers each
constexpr int kDecUPS = 8;     // units per ring slot = warps sharing a slot
constexpr int kDecThreads = kDecWarps * 32;

struct DecParams {
  const uint32_t* frag;
  int q, n, k, rowtiles, kblocks, m;
  int U;  // rowtiles * kblocks
  // activations: fp16 rows quantized in the prologue, or codes + stats written
  // by act_quant_kernel (the PDL primary of this launch)
  const __half* x16;
  const uint32_t* act_frag;
  const double* s_a;
  const int32_t* z_a;
  const long long* rowsum;
  QuantParams qp;
  EpiParams e;
  unsigned long long* bad_word;  // non-finite input report (see run_gemv_dec)
  unsigned long long* bad_out;
  unsigned long long* trace;     // optional [grid][64] stamps (tools/trace_dec.py)
  int prefetch;                  // L2 bulk prefetch of the CTA's weights (default 0)
  int slots;                     // TMA ring slots of kDecUPS units
  int preslots;                  // ring slots issued before the activations are awaited
  const unsigned char* next_frag;  // L2 prefetch hint: the next layer's weights (or null)
  size_t next_bytes;
};

// named barrier over the consumer warps (the producer never joins)
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kDecWarps * 32) : "memory"); }
__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

struct DecSmem {  // carve-up of the dynamic shared memory (host and device agree)
  size_t ring, bars, act, accs, csb, czb, ccs, total;
};
__host__ __device__ inline DecSmem dec_smem(int q, int slots, int mt, int kpad, int nlrt_max) {
  DecSmem s;
  s.ring = 0;
  s.bars = static_cast<size_t>(slots) * kDecUPS * q * 512;
  s.act = s.bars + static_cast<size_t>(2 * slots) * 8;  // full barriers + release counters
  s.accs = (s.act + static_cast<size_t>(mt) * kpad + 15) & ~size_t(15);
  s.csb = (s.accs + static_cast<size_t>(nlrt_max) * 16 * mt * 4 + 15) & ~size_t(15);
  s.czb = s.csb + static_cast<size_t>(nlrt_max) * 16 * 8;
  s.ccs = s.czb + static_cast<size_t>(nlrt_max) * 16 * 8;
  s.total = s.ccs + static_cast<size_t>(nlrt_max) * 16 * 8;
  return s;
}
__host__ __device__ inline int dec_nlrt_max(int rowtiles, int grid) { return (rowtiles + grid - 1) / grid + 1; }

__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
               : "memory");
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

template <int QT, int MT>
__global__ void __launch_bounds__(kDecThreads, 1) gemv_dec_kernel(const __grid_constant__ DecParams Pc) {
  constexpr int NW = kDecWarps, UPS = kDecUPS, NG = NW / UPS;
  constexpr int unit_bytes = QT * 512;
  constexpr int slot_bytes = UPS * unit_bytes;
  constexpr bool RAW = (QT & (QT - 1)) == 0;  // q in {1, 2, 4, 8}: raw masked fields
  constexpr int NF = RAW ? 8 / QT : 1;         // fields (scales) per byte lane
  constexpr int NA = NF >= 2 ? NF : 2;         // accumulator sets (>= 2 independent chains)
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) DecParams P;
  __shared__ float r_lo[NW], r_hi[NW];
  __shared__ int r_sum[NW];
  __shared__ double s_sa[MT];
  __shared__ long long s_za[MT], s_ra[MT];
  __shared__ float s_inv[MT];
  __shared__ long long s_wend;

  const unsigned long long t_entry = gtimer();  // profiling: true CTA start
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  asm volatile("griddepcontrol.launch_dependents;");

  // ---- 0. this CTA's row-tiles [rt_first, rt_end) = units [U0, U1)
  const int G = gridDim.x;
  const int rowtiles = Pc.rowtiles, kblocks = Pc.kblocks, S = Pc.slots;
  // The rowtiles % G CTAs with one row-tile more come FIRST: the next layer's
  // CTAs are launched in blockIdx order onto SMs as this layer's CTAs retire,
  // so its heavy CTAs land on the SMs freed first (by this layer's light ones)
  // and the late starters are light.
  const int rt_base = rowtiles / G, rt_heavy = rowtiles - rt_base * G;
  auto rt_start = [&](int b) { return b < rt_heavy ? b * (rt_base + 1) : rt_heavy + b * rt_base; };
  const int rt_first = rt_start(blockIdx.x);
  const int rt_end = rt_start(blockIdx.x + 1);
  const int U0 = rt_first * kblocks, U1 = rt_end * kblocks;
  const int nlrt = rt_end - rt_first;
  const int nsl = (U1 - U0 + UPS - 1) / UPS;
  const int kpad = kblocks * kKBlock;
  const DecSmem L = dec_smem(QT, S, MT, kpad, dec_nlrt_max(rowtiles, G));
  unsigned char* ring = smem + L.ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  unsigned* relcnt = reinterpret_cast<unsigned*>(full + S);  // warps done with each slot

  // ---- ring set-up by thread 0: full barriers, then (after the CTA barrier
  // below) the L2 bulk prefetch of the CTA's weights and of the next layer's,
  // and the first S slots.  Later slots are refilled by the last warp to
  // release a slot (release() below): no producer warp, so 16 warps x 128
  // registers fit the SM.
  const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(Pc.frag) + static_cast<size_t>(U0) * unit_bytes;
  const uint64_t pol = l2_evict_first_policy();
  auto issue_slot = [&](int i, int sl) {  // thread-level: TMA of slot index i into ring slot sl
    const int nu = min(UPS, U1 - U0 - i * UPS);
    const uint32_t bytes = static_cast<uint32_t>(nu * unit_bytes);
    mbar_expect_tx(&full[sl], bytes);
    tma_bulk_g2s_hint(ring + static_cast<size_t>(sl) * slot_bytes, wsrc + static_cast<size_t>(i) * slot_bytes, bytes,
                      &full[sl], pol);
  };
  // Set-up spread over lanes (one thread doing it serially took ~2 us, all on
  // the launch's critical path): warp 0 lane s initialises barrier s and, once
  // the initialisation is fenced, issues slot s; warp 1's lanes issue the L2
  // bulk prefetches (the CTA's range beyond the ring, then its share of the
  // successor layer), one 32 KB chunk per lane per round.
  if (warp == 0) {
    if (lane < S) {
      mbar_init_n(&full[lane], 1);
      relcnt[lane] = 0;
    }
    __syncwarp();
    if (lane == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    for (int i = lane; i < min(S, Pc.preslots) && i < nsl; i += 32) issue_slot(i, i);
  } else if (warp == 1 && Pc.prefetch) {
    // (the ring slots issued after the activation load are prefetched too, so
    // their copies hit L2)
    const size_t total = static_cast<size_t>(U1 - U0) * unit_bytes;
    for (size_t off = static_cast<size_t>(min(S, Pc.preslots)) * slot_bytes + static_cast<size_t>(lane) * 32768;
         off < total;
         off += 32u * 32768)
      l2_prefetch_bulk(wsrc + off, static_cast<uint32_t>(total - off < 32768 ? total - off : 32768), pol);
    // the next layer's weights (input-independent) stream into L2 behind ours
    if (Pc.next_frag) {
      const size_t nb = Pc.next_bytes, lo = (nb * blockIdx.x / G) & ~size_t(15),
                   hi = (nb * (blockIdx.x + 1) / G) & ~size_t(15);
      for (size_t off = lo + static_cast<size_t>(lane) * 32768; off < hi; off += 32u * 32768)
        l2_prefetch_bulk(Pc.next_frag + off, static_cast<uint32_t>(hi - off < 32768 ? hi - off : 32768), pol);
    }
  }

  // ======================= consumer warps ====================================
  // this thread's epilogue channel parameters (<= 1 channel per thread here;
  // more are loaded below), requested first
  const bool dequant = Pc.e.mode != EPI_ACC_I32 && Pc.e.mode != EPI_ACC_I64;
  const int pj = rt_first * kRowTile + tid;
  const bool has_p = dequant && tid < nlrt * 16 && pj < Pc.n;
  double p_sb = 0.0;
  int p_zb = 0;  // int32 as loaded: a conversion here would wait for the load before the barrier
  long long p_cs = 0;
  if (has_p) {
    p_sb = Pc.e.s_b[static_cast<size_t>(pj) * Pc.e.sb_stride];
    p_zb = Pc.e.z_b[static_cast<size_t>(pj) * Pc.e.zb_stride];
    p_cs = Pc.e.colsum_b[pj];
  }

  // ---- 1. parameter block to shared memory (all threads at once; read lazily
  // from the constant bank, every first touch of a line would be a separate
  // round trip), epilogue parameters of this CTA's channels
  for (int i = tid; i < static_cast<int>(sizeof(DecParams) / 4); i += NW * 32)
    reinterpret_cast<uint32_t*>(&P)[i] = reinterpret_cast<const uint32_t*>(&Pc)[i];
  __syncthreads();  // parameter block and barrier initialisation visible
  unsigned long long* trace = P.trace ? P.trace + 64 * blockIdx.x : nullptr;
  if (trace && tid == 0) {
    trace[0] = clock64();
    trace[8] = gtimer();
    trace[12] = t_entry;
    s_wend = 0;
  }
  uint32_t* act = reinterpret_cast<uint32_t*>(smem + L.act);
  uint32_t* accs = reinterpret_cast<uint32_t*>(smem + L.accs);
  double* c_sb = reinterpret_cast<double*>(smem + L.csb);
  int* c_zb = reinterpret_cast<int*>(smem + L.czb);
  long long* c_cs = reinterpret_cast<long long*>(smem + L.ccs);
  const int tok_n = min(MT, P.m);
  constexpr int kCT = NW * 32;
  if (has_p) {
    c_sb[tid] = p_sb;
    c_zb[tid] = p_zb;
    c_cs[tid] = p_cs;
  }
  for (int idx = tid + kCT; dequant && idx < nlrt * 16; idx += kCT) {
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
  // ---- 2. the activations, which the previous kernel may still be producing
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trace && tid == 0) trace[4] = clock64();

  if (P.x16) {
    // Fused ReQuant, per token, fp16 rows (K % 8 == 0, K <= 32 * TPT: the
    // host routes longer rows through act_quant_kernel).  GT warps per token;
    // each thread loads its (<= XR) 16-byte vectors of the row in one batch.
    // One CTA barrier for the range; every warp then derives step / zero point
    // itself (no second barrier), codes go to shared memory and the code sum to
    // a shared atomic, and the barrier before the main loop publishes both.
    constexpr int GT = NW / MT;  // MT is a power of two <= NW
    constexpr int TPT = GT * 32;
    constexpr int XR = 4;
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
    // the rest of the ring only now: shared-memory-bound TMA traffic into this
    // SM ahead of the activation loads delayed them (~0.2 us on the critical path)
    if (warp == 0)
      for (int i = P.preslots + lane; i < P.slots && i < nsl; i += 32) issue_slot(i, i);
    // min / max in the order-preserving integer image of fp32 (exact for fp16
    // inputs): one REDUX per warp instead of a shuffle tree
    auto ord = [](float f) {
      const int b = __float_as_int(f);
      return b >= 0 ? b : b ^ 0x7FFFFFFF;
    };
    auto unord = [](int o) { return __int_as_float(o >= 0 ? o : o ^ 0x7FFFFFFF); };
    int lo = 0x7FFFFFFF, hi = static_cast<int>(0x80000000u);
    uint32_t bad = 0;
#pragma unroll
    for (int r = 0; r < XR; ++r) {
      if (!active || l + r * TPT >= nvec) break;
      bad |= f16x8_nonfinite(xv[r]);
      const __half2* h2 = reinterpret_cast<const __half2*>(&xv[r]);
      __half2 mn = h2[0], mx = h2[0];
#pragma unroll
      for (int e = 1; e < 4; ++e) {
        mn = __hmin2(mn, h2[e]);
        mx = __hmax2(mx, h2[e]);
      }
      lo = min(lo, min(ord(__low2float(mn)), ord(__high2float(mn))));
      hi = max(hi, max(ord(__low2float(mx)), ord(__high2float(mx))));
    }
    const bool report = blockIdx.x == 0 && P.bad_out != nullptr;
    if (report && bad) report_nonfinite_f16(xr, t, l, TPT, nvec, P.k, P.bad_word);
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      r_lo[warp] = __int_as_float(lo);  // raw bits: decoded below
      r_hi[warp] = __int_as_float(hi);
      if (warp % GT == 0) s_ra[t] = 0;
    }
    cta_sync();
    if (trace && tid == 0) trace[5] = clock64();
    int rsum = 0;
    if (active) {
      const int base = warp - warp % GT;  // first warp of this token
      int l2 = lane < GT ? __float_as_int(r_lo[base + lane]) : 0x7FFFFFFF;
      int h2 = lane < GT ? __float_as_int(r_hi[base + lane]) : static_cast<int>(0x80000000u);
      l2 = __reduce_min_sync(0xffffffffu, l2);
      h2 = __reduce_max_sync(0xffffffffu, h2);
      // step / zero point in FP64 (quantizer.hpp:169-201) by lane 0 of every
      // warp of the token (identical inputs, identical results), broadcast
      double step = 0.0;
      int z = 0;
      float inv32 = 0.0f;
      if (lane < 2) group_params(P.qp, unord(l2), unord(h2), &step, &z);
      if (lane == 1) inv32 = f32_reciprocal(step);  // lane 0 finishes z meanwhile
      step = __shfl_sync(0xffffffffu, step, 0);
      z = __shfl_sync(0xffffffffu, z, 0);
      inv32 = __shfl_sync(0xffffffffu, inv32, 1);
      if (warp == base && lane == 0) {
        s_sa[t] = step;
        s_za[t] = z;
      }
      if (trace && tid == 0) trace[6] = clock64();
      const int topi = static_cast<int>(P.qp.levels - 1);
#pragma unroll
      for (int r = 0; r < XR; ++r) {
        const int v = l + r * TPT;
        if (v >= nvec) break;
        uint32_t w0, w1;
        rsum += quant_codes8_f16(xv[r], step, inv32, z, topi, &w0, &w1);
        act[act_frag_index(2 * v, t, MT)] = w0;
        act[act_frag_index(2 * v + 1, t, MT)] = w1;
      }
      rsum = __reduce_add_sync(0xffffffffu, rsum);  // < 2^31: <= 255 * 65536
      if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ra[t]), static_cast<unsigned long long>(rsum));
    }
    if (report && tid == 0) {
      const unsigned long long w = atomicExch(P.bad_word, 0ull);
      *P.bad_out = w ? ~w : ~0ull;
    }
  } else {
    // codes + stats from act_quant_kernel (the host issues the whole ring up
    // front on this path: preslots == slots)
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
  cta_sync();
  if (trace && tid == 0) trace[1] = clock64();

  // ---- 3. main loop over the TMA ring.
  // Warp group grp = warp / UPS takes the slots i = grp (mod NG), warp % UPS
  // its unit of each.  Per unit: the weights come from shared memory into one
  // of two register buffers (the next unit's are requested before this
  // unit's IMMAs issue), the IMMAs accumulate into one of two accumulator
  // sets, and the other set -- the previous unit's -- is folded into the
  // row-tile sums AFTER these IMMAs are issued, so consecutive units' IMMA
  // chains overlap instead of serialising on the flush.
  const int g = lane >> 2, tig = lane & 3;
  const uint32_t act_lane = smem_addr(act) + ((g * 4 + tig) * 8);  // B-fragment word pair of (g, tig)
  const bool has_b = g < MT;
  uint2 b[8];
  int cur_kb = -1;
  auto load_b = [&](int k_b) {  // B fragments of a k-block (kept while it repeats)
    cur_kb = k_b;
    const uint32_t ab = act_lane + k_b * (8 * MT * 4 * 8);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      b[c] = make_uint2(0u, 0u);
      if (has_b) asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(b[c].x), "=r"(b[c].y) : "r"(ab + c * MT * 32));
    }
  };
  auto mma_unit = [&](int (&acc)[NA][4], const uint4 (&w)[QT]) {
    if constexpr (RAW) {
      // quad Q = w[Q] holds A registers u = 0..3 of the chunks c = f*QT + Q in field f
      constexpr uint32_t M = ((1u << QT) - 1u) * 0x01010101u;
#pragma unroll
      for (int Q = 0; Q < QT; ++Q)
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const uint32_t m = M << (QT * f);
          const int c = f * QT + Q;
          imma_16832(acc[NF >= 2 ? f : (Q & 1)], w[Q].x & m, w[Q].y & m, w[Q].z & m, w[Q].w & m, b[c].x, b[c].y);
        }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = widen_slices<QT>(w, 4 * c + r);
        imma_16832(acc[c & 1], a[0], a[1], a[2], a[3], b[c].x, b[c].y);
      }
    }
  };
  auto flush_set = [&](int (&acc)[NA][4], int r_t) {
    const int lrt = r_t - rt_first;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // field f holds 2^(QT f) * its partial sum, exactly (the true row-tile
      // sum is < 2^32 for K <= 65536, and so is every scaled field sum)
      uint32_t v = 0;
#pragma unroll
      for (int f = 0; f < NA; ++f) {
        const int sh = RAW && NF >= 2 ? QT * f : 0;
        v += static_cast<uint32_t>(acc[f][r]) >> sh;
        acc[f][r] = 0;
      }
      const int row = g + 8 * (r >> 1), tok = 2 * tig + (r & 1);
      if (tok < tok_n) atomicAdd(&accs[(lrt * 16 + row) * MT + tok], v);
    }
  };
  {
    // loop-invariant scalars re-read from the shared copy of the parameter
    // block: left to ptxas they are re-fetched from the constant bank (LDC)
    // inside the loop
    const int S_ = *reinterpret_cast<volatile int*>(&P.slots);
    const int kbl = *reinterpret_cast<volatile int*>(&P.kblocks);
    const int grp = warp / UPS, off = grp * UPS + warp % UPS;
    const int nw = U1 - U0 > off ? (U1 - U0 - off + NW - 1) / NW : 0;  // this warp's units
    const uint32_t ring_lane = smem_addr(ring) + (warp % UPS) * unit_bytes + lane * 16;
    auto lds_unit = [&](int sl, uint4 (&w)[QT]) {
      const uint32_t a = ring_lane + sl * slot_bytes;
#pragma unroll
      for (int t = 0; t < QT; ++t)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w) : "r"(a + t * 512));
    };
    long long t_wait = 0;  // profiling (trace mode only)
    auto wait_full = [&](int sl, uint32_t p) {
      if (trace) {
        const long long t0 = clock64();
        mbar_wait_parity(&full[sl], p);
        t_wait += clock64() - t0;
      } else {
        mbar_wait_parity(&full[sl], p);
      }
    };
    // the last of the UPS warps done with ring slot sl refills it with slot
    // index i + S (its data is in registers: the IMMAs reading it have issued)
    const bool refill = nsl > S_;  // else every slot was loaded once, at kernel start
    auto release = [&](int sl, int i) {
      if (!refill) return;
      __syncwarp();
      if (lane == 0 && i + S_ < nsl && atomicAdd(&relcnt[sl], 1u) == UPS - 1) {
        relcnt[sl] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_slot(i + S_, sl);
      }
    };
    // fetch cursor: slot / parity / row-tile / k-block of the next unit to fetch
    int fs = grp, fi = grp;  // ring slot / slot index of the next fetch (NG <= S)
    uint32_t fph = 0;
    int frt = (U0 + off) / kbl, fkb = U0 + off - frt * kbl;
    auto fetch = [&](uint4 (&w)[QT], int& sl, int& idx, int& r_t, int& k_b) {
      sl = fs;
      idx = fi;
      fi += NG;
      r_t = frt;
      k_b = fkb;
      wait_full(fs, fph);
      lds_unit(fs, w);
      fs += NG;
      if (fs >= S_) {
        fs -= S_;
        fph ^= 1u;
      }
      fkb += NW;
      while (fkb >= kbl) {
        fkb -= kbl;
        ++frt;
      }
    };
    // Fast path, layers with 16 k-blocks (K in (3840, 4096]: LLaMA q/k/v/o/
    // gate/up): warp w owns k-block w of every row-tile of the CTA, so its j-th
    // unit is row-tile rt_first + j.  Each row-tile gets its own accumulator set
    // in registers (fully unrolled, static indices): the IMMA chains of all
    // units are independent and nothing is flushed until the loop is done.
    constexpr int RTMAX = (QT == 4 || QT == 8) ? 6 : (QT == 2 ? 3 : 0);
    bool fast_done = false;
    if constexpr (RTMAX > 0 && NG == 2) {
      if (kbl == NW && nw <= RTMAX) {
        constexpr bool DB = QT <= 4;  // two register buffers where they fit
        if (nw > 0 && cur_kb != warp) load_b(warp);
        int acc[RTMAX][NA][4];
#pragma unroll
        for (int j = 0; j < RTMAX; ++j)
#pragma unroll
          for (int f = 0; f < NA; ++f)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[j][f][r] = 0;
        uint4 wbuf[DB ? 2 : 1][QT];
        int s0 = grp;  // ring slot of the warp's j-th unit (slot index grp + 2 j)
        uint32_t p0 = 0;
        if (DB && nw > 0) {
          wait_full(s0, p0);
          lds_unit(s0, wbuf[0]);
        }
#pragma unroll
        for (int j = 0; j < RTMAX; ++j) {
          if (j < nw) {
            int s1 = s0 + NG;
            uint32_t p1 = p0;
            if (s1 >= S_) {
              s1 -= S_;
              p1 ^= 1u;
            }
            if constexpr (DB) {
              if (j + 1 < nw) {
                wait_full(s1, p1);
                lds_unit(s1, wbuf[(j + 1) & 1]);
              }
            } else {
              wait_full(s0, p0);
              lds_unit(s0, wbuf[0]);
            }
            mma_unit(acc[j], wbuf[DB ? (j & 1) : 0]);
            release(s0, grp + NG * j);
            s0 = s1;
            p0 = p1;
          }
        }
#pragma unroll
        for (int j = 0; j < RTMAX; ++j)
          if (j < nw) flush_set(acc[j], rt_first + j);
        fast_done = true;
      }
    }
    if (trace && lane == 0) trace[24 + warp] = t_wait;
    int accA[NA][4], accB[NA][4];
#pragma unroll
    for (int f = 0; f < NA; ++f)
#pragma unroll
      for (int r = 0; r < 4; ++r) accA[f][r] = accB[f][r] = 0;
    if (fast_done) {
    } else if constexpr (QT <= 6) {
      uint4 wA[QT], wB[QT];
      int sA = 0, iA = 0, rtA = 0, kbA = 0, sB = 0, iB = 0, rtB = 0, kbB = 0;
      if (nw > 0) fetch(wA, sA, iA, rtA, kbA);
      for (int j = 0; j < nw; j += 2) {
        // unit j (buffer A, accumulators A); unit j + 1 prefetched into B
        const int rtB_prev = rtB;  // unit j - 1 (j > 0)
        if (j + 1 < nw) fetch(wB, sB, iB, rtB, kbB);
        if (kbA != cur_kb) load_b(kbA);
        mma_unit(accA, wA);
        if (j > 0) flush_set(accB, rtB_prev);
        release(sA, iA);
        if (j + 1 >= nw) {
          flush_set(accA, rtA);
          break;
        }
        // unit j + 1 (buffer B, accumulators B); unit j + 2 prefetched into A
        const int rtA_done = rtA;
        if (j + 2 < nw) fetch(wA, sA, iA, rtA, kbA);
        if (kbB != cur_kb) load_b(kbB);
        mma_unit(accB, wB);
        flush_set(accA, rtA_done);
        release(sB, iB);
        if (j + 2 >= nw) flush_set(accB, rtB);
      }
    } else {  // one register buffer (two would spill at this register budget)
      uint4 wA[QT];
      int sA = 0, iA = 0, rtA = 0, kbA = 0, rtP = -1;
      for (int j = 0; j < nw; ++j) {
        fetch(wA, sA, iA, rtA, kbA);
        if (kbA != cur_kb) load_b(kbA);
        if (j & 1) {
          mma_unit(accB, wA);
          flush_set(accA, rtP);
        } else {
          mma_unit(accA, wA);
          if (j > 0) flush_set(accB, rtP);
        }
        release(sA, iA);
        rtP = rtA;
      }
      if (nw > 0) {
        if ((nw - 1) & 1) flush_set(accB, rtP);
        else flush_set(accA, rtP);
      }
    }
  }
  if (trace && lane == 0) atomicMax(&s_wend, static_cast<long long>(clock64()));
  cta_sync();
  if (trace && tid == 0) trace[2] = s_wend;

  // ---- 4. epilogue: zero-point correction + dequant of this CTA's channels
  const EpiParams& E = P.e;
  for (int idx = tid; idx < nlrt * 16 * MT; idx += kCT) {
    const int i = idx & (MT - 1), rc = idx / MT, lrt = rc >> 4, row = rc & 15;
    const int j = (rt_first + lrt) * kRowTile + row;
    if (i >= tok_n || j >= P.n) continue;
    const long long a = accs[idx];
    if (!dequant) {
      epi_store_v(E, i, j, a, 0.0, 0, 0);
      continue;
    }
    const long long za = s_za[i], zb = static_cast<long long>(c_zb[rc]);
    const long long corr = a - za * c_cs[rc] - zb * s_ra[i] + E.k * za * zb;
    const long long o = static_cast<long long>(i) * E.ldo + j;
    if (E.mode == EPI_CORR_I64) {
      static_cast<int64_t*>(E.out)[o] = corr;
      continue;
    }
    const double y = __dmul_rn(__dmul_rn(s_sa[i], c_sb[rc]), static_cast<double>(corr));
    if (E.mode == EPI_F64)
      static_cast<double*>(E.out)[o] = y;
    else if (E.mode == EPI_F16)
      static_cast<__half*>(E.out)[o] = __double2half(y);
    else
      static_cast<float*>(E.out)[o] = __double2float_rn(y);
  }
  if (trace && tid == 0) {
    trace[3] = clock64();
    trace[9] = gtimer();
  }
}

// ============================================================================
// host side
// ============================================================================
unsigned long long*& trace_buffer();

template <int QT, int MT>
static int launch_dec2(const DecParams& P, int grid, size_t smem, bool pdl, cudaStream_t st) {
  auto kern = gemv_dec_kernel<QT, MT>;
  if (smem > 220 * 1024) return fail(ABQ_ERR_VALUE, "gemv_dec: shared memory plan too large (%zu B)", smem);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_dec: smem attribute: %s", cudaGetErrorString(err));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = smem;
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

template <int MT>
static int launch_dec1(const DecParams& P, int grid, size_t smem, bool pdl, cudaStream_t st) {
  switch (P.q) {
    case 1: return launch_dec2<1, MT>(P, grid, smem, pdl, st);
    case 2: return launch_dec2<2, MT>(P, grid, smem, pdl, st);
    case 3: return launch_dec2<3, MT>(P, grid, smem, pdl, st);
    case 4: return launch_dec2<4, MT>(P, grid, smem, pdl, st);
    case 5: return launch_dec2<5, MT>(P, grid, smem, pdl, st);
    case 6: return launch_dec2<6, MT>(P, grid, smem, pdl, st);
    case 7: return launch_dec2<7, MT>(P, grid, smem, pdl, st);
    default: return launch_dec2<8, MT>(P, grid, smem, pdl, st);
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
                 cudaStream_t st, const void* next_frag, size_t next_bytes) {
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
  // L2 bulk prefetch of the CTA's range beyond the pre-issued ring slots and of
  // the successor layer: off by default -- measured slower on every decode
  // shape (profiles/r01_dec_prefetch_sweep.txt: W4A4 M=1 7.56 -> 7.32 us, W8A8
  // M=1 10.0 -> 8.4 us, W4A4 M=8 11.3 -> 9.9 us); ABQ_DEC_PREFETCH=1 restores it.
  P.prefetch = 0;
  P.next_frag = static_cast<const unsigned char*>(next_frag);
  P.next_bytes = next_frag ? next_bytes : 0;
  if (const char* env = std::getenv("ABQ_DEC_PREFETCH")) P.prefetch = env[0] == '1';
  const int mt = m <= 1 ? 1 : m <= 2 ? 2 : m <= 4 ? 4 : 8;
  const int kpad = P.kblocks * kKBlock;
  // workspace (imma_ws_bytes layout): [row-tile accumulators][counters][codes][stats][report word]
  char* w = static_cast<char*>(ws);
  w += static_cast<size_t>(P.rowtiles) * 16 * 8 * 8;
  w += (static_cast<size_t>(P.rowtiles) * 4 + 255) & ~size_t(255);
  uint32_t* act_frag = reinterpret_cast<uint32_t*>(w);
  w += 8 * static_cast<size_t>(kpad);
  double* s_a = reinterpret_cast<double*>(w);
  int32_t* z_a = reinterpret_cast<int32_t*>(w + 64);
  long long* rowsum = reinterpret_cast<long long*>(w + 128);
  P.bad_word = reinterpret_cast<unsigned long long*>(w + 192);
  P.bad_out = bad_out;
  // fused ReQuant: each of the 32*kDecWarps/mt consumer threads of a token holds <= 4 vectors of 8
  const bool fused = x_dtype == ABQ_F16 && !qp.per_tensor && k % 8 == 0 &&
                     k <= static_cast<size_t>(32 * kDecWarps * 32 / mt);
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
  const int grid = std::min(num_sms(), P.rowtiles);
  // Ring (one CTA per SM): as deep as the CTA's whole weight share when that
  // fits in shared memory -- then every TMA copy is issued at kernel start and
  // no refill latency is exposed at the tail of the main loop -- else ~208 KB.
  const int nl = dec_nlrt_max(P.rowtiles, grid);
  const size_t slot_bytes = static_cast<size_t>(kDecUPS) * q * 512;
  const int max_units = ((P.rowtiles + grid - 1) / grid) * P.kblocks;
  int slots = (max_units + kDecUPS - 1) / kDecUPS;
  if (const char* env = std::getenv("ABQ_DEC_RING_KB")) slots = static_cast<int>(std::atoi(env) * 1024 / slot_bytes);
  const int min_slots = kDecWarps / kDecUPS;
  slots = std::max(min_slots, std::min(32, slots));
  const size_t budget = 212 * 1024;
  while (slots > min_slots && dec_smem(q, slots, mt, kpad, nl).total > budget) --slots;
  P.slots = slots;
  // slots in flight before the activations are awaited: ~64 KB (the rest is
  // L2-prefetched and copied once the activation loads are issued)
  int pre_kb = 64;
  if (const char* env = std::getenv("ABQ_DEC_PRE_KB")) pre_kb = std::atoi(env);
  P.preslots = fused ? std::max(1, std::min(slots, static_cast<int>(pre_kb * 1024 / slot_bytes))) : slots;
  const size_t smem = dec_smem(q, slots, mt, kpad, nl).total;
  bool pdl = true;
  if (const char* env = std::getenv("ABQ_DEC_PDL")) pdl = env[0] == '1';
  switch (mt) {
    case 1: return launch_dec1<1>(P, grid, smem, pdl, st);
    case 2: return launch_dec1<2>(P, grid, smem, pdl, st);
    case 4: return launch_dec1<4>(P, grid, smem, pdl, st);
    default: return launch_dec1<8>(P, grid, smem, pdl, st);
  }
}

}  // namespace abq_dev
