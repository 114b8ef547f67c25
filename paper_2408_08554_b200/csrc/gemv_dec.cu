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
// Shape of the kernel:
//  * one CTA per SM owning whole row-tiles (no cross-CTA reduction); its
//    packed weights stream into a shared-memory ring by 1-D TMA bulk copies,
//    as deep as the CTA's whole share when that fits (W4 LLaMA-7B up_proj:
//    80 units = 160 KB), issued before the activations are awaited (weights are
//    input-independent) -- the first `preslots` slots at once, the rest right
//    after the activation loads so those do not queue behind the stream;
//  * the epilogue's per-channel values (s_b, z_b, colsum_b) are fetched before
//    the activations are awaited as well;
//  * fused ReQuant prologue: one barrier for the per-token range, step / zero
//    point in FP64 by every warp of the token (same inputs, same results, no
//    broadcast), codes on the fp32 pipe with an exact FP64 tie path
//    (quant_dev.cuh), written to shared memory in IMMA B-fragment order;
//  * main loop: 16 warps, warp w takes units w, w + 16, ... of the CTA's range;
//    per unit one IMMA m16n8k32 stream (16 weight rows x 32 k x 8 tokens):
//    q in {1, 2, 4, 8} fed as raw masked bytes (one LOP3 per A register, the
//    field's 2^(q f) scale divided out exactly when the unit is folded), other
//    q widened to byte codes.  Two accumulator sets alternate between units so
//    that a unit's fold overlaps the next unit's IMMAs; folded sums stay in
//    registers while the row-tile repeats and go to shared memory (one atomic
//    per row and token) when it changes;
//  * launches are programmatic-dependent (PDL): griddepcontrol.launch_dependents
//    first thing, griddepcontrol.wait right before the activations are read.
// Profiling stamps (tools/trace_dec.py) exist only in the ABQ_TRACE build
// (make TRACE=1 -> libabq_cuda_trace.so), not in the product library.
#include <algorithm>

#include "common.cuh"
#include "gemv_frag.cuh"
#include "quant_dev.cuh"

namespace abq_dev {

constexpr int kDecWarps = 16;  // 4 per SM sub-partition, <= 128 registers each
constexpr int kDecUPS = 8;     // units per ring slot = warps sharing a slot
constexpr int kDecThreads = kDecWarps * 32;  // consumer threads
constexpr int kDecBlock = kDecThreads + 32;   // + one TMA producer warp
constexpr int kDecCtasPerSm = 1;
constexpr int kDecXR = 4;      // fused ReQuant: 16-byte activation vectors per thread

struct DecParams {
  const uint32_t* frag;
  int q, n, k, rowtiles, kblocks, m;
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
  int xr;        // fused prologue: 16-byte activation vectors per thread
  int pace_ns;   // producer warp: spacing of the ring slots issued while the activations are awaited
  int slots;     // TMA ring slots of kDecUPS units
  int preslots;  // ring slots issued before the activations are awaited
  // successor layer (abq_weights.next): its decode-layout weights, partition
  // (same row-tile split as its own launch) and the bytes per CTA prefetched
  // into L2 once this CTA's stream has landed
  const unsigned char* nx;
  int nx_rowtiles, nx_kblocks, nx_unit, nx_grid, nx_bytes, nx_at;
  int l2_plain;  // weight TMA without the L2 evict-first hint (sweeps)
  int dbg_nostream;  // TRACE build timing experiment: ring barriers arrive without data
  unsigned long long* trace;  // ABQ_TRACE build only: [grid][64] stamps
};

// named barrier over the consumer warps (the producer warp has exited)
__device__ __forceinline__ void cta_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kDecThreads) : "memory"); }
__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n));
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
__host__ __device__ inline int dec_nlrt_max(int rowtiles, int grid) { return (rowtiles + grid - 1) / grid; }

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

// raw accumulator outputs (gemm_arbitrary modes) out of line: the serving
// epilogue's inline code stays small
static __device__ __noinline__ void epi_store_raw(const EpiParams& E, long long i, long long j, long long acc) {
  epi_store_v(E, i, j, acc, 0.0, 0, 0);
}

#ifdef ABQ_TRACE
#define DEC_STAMP(slot, value)                  \
  do {                                          \
    if (P.trace && tid == 0) trace[slot] = (value); \
  } while (0)
#else
#define DEC_STAMP(slot, value) \
  do {                         \
  } while (0)
#endif

// FUSED: fp16 activations quantized in the prologue (P.x16); else codes +
// stats from a preceding kernel (two instantiations: each launch only fetches
// the code of its own prologue)
// XF > 0: fused, XF 16-byte activation vectors per thread (1, 2 or 4: the
// smallest that covers K, so short rows do not carry the unrolled code of long ones)
template <int QT, int MT, int XF>
__global__ void __launch_bounds__(kDecBlock, kDecCtasPerSm) gemv_dec_kernel(const __grid_constant__ DecParams P) {
  constexpr bool FUSED = XF > 0;
  constexpr int NW = kDecWarps, UPS = kDecUPS, NG = NW / UPS;
  constexpr int unit_bytes = QT * 512;
  constexpr int slot_bytes = UPS * unit_bytes;
  constexpr bool RAW = (QT & (QT - 1)) == 0;  // q in {1, 2, 4, 8}: raw masked fields
  constexpr int NF = RAW ? 8 / QT : 1;         // fields (scales) per byte lane
  constexpr int NA = NF >= 2 ? NF : 2;         // accumulators per set (>= 2 independent chains)
  constexpr int FSH = RAW && NF >= 2 ? QT * (NF - 1) : 0;  // folded row-tile sums hold 2^FSH * the sum
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int r_lo[NW], r_hi[NW];
  __shared__ double s_sa[MT];
  __shared__ int s_za[MT];
  __shared__ long long s_ra[MT];
  __shared__ int r_sum[NW];  // per-warp code sums of the fused ReQuant
  __shared__ float s_inv[MT], s_thr[MT];  // fused ReQuant: RN32(1/step), tie-band threshold
  __shared__ int x_flag;     // consumers -> producer warp: activation loads issued

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool prod = warp == NW;  // the TMA producer warp (no activations, no compute)
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef ABQ_TRACE
  unsigned long long* trace = P.trace ? P.trace + 64 * blockIdx.x : nullptr;
  if (trace && tid == 0) {
    trace[8] = gtimer();
    trace[0] = clock64();
  }
#endif
  // the parameter block is read through the constant cache: touch every line
  // before the weight stream starts (a miss behind it waits for the stream)
  if (warp == NW - 1) warm_param_block(P, lane);

  // ---- 0. this CTA's row-tiles [rt_first, rt_end) = units [U0, U0 + nu)
  const int G = gridDim.x;
  const int rowtiles = P.rowtiles, kbl = P.kblocks, S = P.slots;
  // The rowtiles % G CTAs with one row-tile more come FIRST: the next layer's
  // CTAs are launched in blockIdx order onto SMs as this layer's CTAs retire,
  // so its heavy CTAs land on the SMs freed first.
  const int rt_base = rowtiles / G, rt_heavy = rowtiles - rt_base * G;
  const int rt_first = blockIdx.x < rt_heavy ? blockIdx.x * (rt_base + 1) : rt_heavy + blockIdx.x * rt_base;
  const int nlrt = rt_base + (static_cast<int>(blockIdx.x) < rt_heavy ? 1 : 0);
  const int U0 = rt_first * kbl, nu = nlrt * kbl;
  const int nsl = (nu + UPS - 1) / UPS;
  const int kpad = kbl * kKBlock;
  const DecSmem L = dec_smem(QT, S, MT, kpad, dec_nlrt_max(rowtiles, G));
  unsigned char* ring = smem + L.ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  unsigned* relcnt = reinterpret_cast<unsigned*>(full + S);  // warps done with each slot
  uint32_t* act = reinterpret_cast<uint32_t*>(smem + L.act);
  uint32_t* accs = reinterpret_cast<uint32_t*>(smem + L.accs);
  double* c_sb = reinterpret_cast<double*>(smem + L.csb);
  long long* c_zb = reinterpret_cast<long long*>(smem + L.czb);
  long long* c_cs = reinterpret_cast<long long*>(smem + L.ccs);

  // epilogue values of this CTA's channels (input-independent): requested into
  // registers before the weight stream is started, so they do not queue behind
  // it; stored to shared memory only after the main loop
  const bool dequant = P.e.mode != EPI_ACC_I32 && P.e.mode != EPI_ACC_I64;
  const int pj = rt_first * kRowTile + tid;
  const bool has_p = !prod && dequant && tid < nlrt * 16 && pj < P.n;
  double p_sb = 0.0;
  int p_zb = 0;
  long long p_cs = 0;
  if (has_p) {
    p_sb = P.e.s_b[static_cast<size_t>(pj) * P.e.sb_stride];
    p_zb = P.e.z_b[static_cast<size_t>(pj) * P.e.zb_stride];
    p_cs = P.e.colsum_b[pj];
  }
  const unsigned char* wsrc = reinterpret_cast<const unsigned char*>(P.frag) + static_cast<size_t>(U0) * unit_bytes;
  const uint64_t pol = l2_evict_first_policy();
  auto issue_slot = [&](int i, int sl) {  // thread-level: TMA of slot index i into ring slot sl
    const int n_units = min(UPS, nu - i * UPS);
    const uint32_t bytes = static_cast<uint32_t>(n_units * unit_bytes);
#ifdef ABQ_TRACE
    if (P.dbg_nostream) {  // timing experiment only: no weight bytes (results invalid)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[sl])) : "memory");
      return;
    }
#endif
    mbar_expect_tx(&full[sl], bytes);
    if (P.l2_plain)
      tma_bulk_g2s(ring + static_cast<size_t>(sl) * slot_bytes, wsrc + static_cast<size_t>(i) * slot_bytes, bytes,
                   &full[sl]);
    else
      tma_bulk_g2s_hint(ring + static_cast<size_t>(sl) * slot_bytes, wsrc + static_cast<size_t>(i) * slot_bytes,
                        bytes, &full[sl], pol);
  };
  // ---- 1. ring: the producer warp's lane s initialises barrier s; the
  // slots are issued after the set-up barrier (below)
  if (prod) {
    if (lane < S) {
      mbar_init_n(&full[lane], 1);
      relcnt[lane] = 0;
    }
    if (lane == 0) x_flag = 0;
    __syncwarp();
    if (lane == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // the slots issued up front go out before the set-up barrier
#pragma unroll 1
    for (int i = lane; i < min(S, P.preslots) && i < nsl; i += 32) issue_slot(i, i);
  }
  // zeroed row-tile sums, zero codes past K
  const int tok_n = min(MT, P.m);
  if (!prod) {
    for (int idx = tid; idx < nlrt * 16 * MT; idx += kDecThreads) accs[idx] = 0;
    if constexpr (FUSED) {
      const int k4 = P.k >> 2, ntail = (kpad >> 2) - k4;
      for (int idx = tid; idx < ntail * MT; idx += kDecThreads) act[act_frag_index(k4 + idx / MT, idx % MT, MT)] = 0u;
    }
  }
  // barrier initialisation and the zeroed state visible to the consumers; the
  // producer warp only ARRIVES (it does not wait for the consumers' set-up)
  if (prod) asm volatile("bar.arrive 0, %0;" ::"n"(kDecBlock) : "memory");
  else asm volatile("bar.sync 0, %0;" ::"n"(kDecBlock) : "memory");
  if (prod) {
    // The weights are input-independent.  Fused path: while the consumers
    // await the activations (the previous kernel may still be running), one
    // ring slot per pace_ns -- about the SM's share of HBM bandwidth, so at most
    // ~one slot is queued ahead of the activation loads when the wait returns --
    // then, once the activation loads are issued, the rest at once.  Other
    // paths: everything at once (the preceding kernel's run covers it).
    const int lim = min(S, nsl);
    int i = min(lim, P.preslots);
    if constexpr (FUSED) {
      if (lane == 0) {
        while (i < lim && atomicAdd(&x_flag, 0) == 0) {  // (a timing hint only: an atomic poll)
          if (P.pace_ns > 0) {
            issue_slot(i, i);
            ++i;
          }
          __nanosleep(P.pace_ns > 0 ? P.pace_ns : 64);
        }
      }
      i = __shfl_sync(0xffffffffu, i, 0);
    }
#pragma unroll 1
    for (int j = i + lane; j < lim; j += 32) issue_slot(j, j);  // the rest, one slot per lane
#ifdef ABQ_TRACE
    if (P.trace && lane == 0) {
      P.trace[64 * blockIdx.x + 15] = gtimer();
      if (nsl > 0 && nsl <= S) {  // arrival of the first and the last ring slot
        mbar_wait_parity(&full[0], 0);
        P.trace[64 * blockIdx.x + 41] = gtimer();
        mbar_wait_parity(&full[nsl - 1], 0);
        P.trace[64 * blockIdx.x + 42] = gtimer();
      }
    }
#endif
    // Successor prefetch: once this CTA's whole share has landed (ring not
    // refilled: the last slot's barrier completes exactly once), the SM's HBM
    // stream is done while the grid still finishes, the next launch's CTAs
    // start and their first loads see HBM latency.  The first nx_bytes of the
    // share the next layer's CTA with this index will stream are requested
    // into L2 now (same split as that launch: rt_first / nlrt below).
    if (P.nx && lane == 0 && nsl > 0 && nsl <= S && static_cast<int>(blockIdx.x) < P.nx_grid) {
      mbar_wait_parity(&full[max(0, (nsl * P.nx_at + 99) / 100 - 1)], 0);  // nx_at % of the share landed
      const int gn = P.nx_grid, base = P.nx_rowtiles / gn, hv = P.nx_rowtiles - base * gn;
      const int b = blockIdx.x;
      const int rf = b < hv ? b * (base + 1) : hv + b * base;
      const int nl = base + (b < hv ? 1 : 0);
      const size_t share = static_cast<size_t>(nl) * P.nx_kblocks * P.nx_unit;
      const size_t bytes = min(share, static_cast<size_t>(P.nx_bytes));
      const unsigned char* src = P.nx + static_cast<size_t>(rf) * P.nx_kblocks * P.nx_unit;
#pragma unroll 1
      for (size_t off = 0; off < bytes; off += 16384)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off),
                     "r"(static_cast<uint32_t>(bytes - off < 16384 ? bytes - off : 16384))
                     : "memory");
    }
    return;
  }
  DEC_STAMP(1, clock64());

  // ---- 2. the activations, which the previous kernel may still be producing
  asm volatile("griddepcontrol.wait;" ::: "memory");
  DEC_STAMP(2, clock64());
  DEC_STAMP(12, gtimer());
  if constexpr (FUSED) {
    // Fused ReQuant, per token, fp16 rows (K % 8 == 0, K <= 32 * TPT: the host
    // routes longer rows through act_quant_kernel).  GT warps per token; each
    // thread loads its (<= XR) 16-byte vectors of the row in one batch.
    constexpr int GT = NW / MT;  // MT is a power of two <= NW
    constexpr int TPT = GT * 32;
    constexpr int XR = XF > 0 ? XF : 1;
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
    // activation loads issued: the producer warp issues the rest of the ring
    if (tid == 0) atomicExch(&x_flag, 1);
    // min / max in the order-preserving integer image of fp32 (exact for fp16
    // inputs): one REDUX per warp
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
      r_lo[warp] = lo;
      r_hi[warp] = hi;
    }
    cta_sync();
    DEC_STAMP(3, clock64());
    // step / zero point in FP64 (quantizer.hpp:169-201), the fp32 reciprocal
    // and the per-token tie-band threshold: computed ONCE per token (the first
    // warp of the token) and shared -- all 16 warps redundantly computing them
    // cost more issue slots than the extra barrier
    if (active && warp % GT == 0) {
      int l2 = lane < GT ? r_lo[warp + lane] : 0x7FFFFFFF;
      int h2 = lane < GT ? r_hi[warp + lane] : static_cast<int>(0x80000000u);
      l2 = __reduce_min_sync(0xffffffffu, l2);
      h2 = __reduce_max_sync(0xffffffffu, h2);
      if (lane == 0) {
        // step / zero point (quantizer.hpp:169-201) out of line: this code
        // runs once per launch, and the kernel's code footprint is what it
        // costs (the instruction cache does not hold the whole kernel)
        const float flo = unord(l2), fhi = unord(h2);
        const StepZ sz = group_params_ool(P.qp, flo, fhi);
        const float inv32 = f32_reciprocal_fast(sz.step);
        s_sa[t] = sz.step;
        s_za[t] = sz.z;
        s_inv[t] = inv32;
        s_thr[t] = band_threshold(flo, fhi, inv32);
      }
    }
    cta_sync();
    DEC_STAMP(4, clock64());
    if (active) {
      const double step = s_sa[t];
      const int z = s_za[t];
      const float inv32 = s_inv[t], thr = s_thr[t];
      const int topi = static_cast<int>(P.qp.levels - 1);
      int rsum = 0;
#pragma unroll
      for (int r = 0; r < XR; ++r) {
        const int v = l + r * TPT;
        if (v >= nvec) break;
        uint32_t w0, w1;
        rsum += quant_codes8_f16_band(xv[r], step, inv32, thr, z, topi, &w0, &w1);
        act[act_frag_index(2 * v, t, MT)] = w0;
        act[act_frag_index(2 * v + 1, t, MT)] = w1;
      }
      rsum = __reduce_add_sync(0xffffffffu, rsum);  // < 2^31: <= 255 * 65536
      if (lane == 0) r_sum[warp] = rsum;
    } else if (lane == 0) {
      r_sum[warp] = 0;
    }
    if (report && tid == 0) {
      const unsigned long long w = atomicExch(P.bad_word, 0ull);
      *P.bad_out = w ? ~w : ~0ull;
    }
  } else {
    // codes + stats from act_quant_kernel or a producer-fused ReQuant
    // (producer.cu); the codes past K are zero.  Requested first, then the
    // ring slots not issued yet, then stored.
    constexpr int CR = 4;
    const uint4* src = reinterpret_cast<const uint4*>(P.act_frag);
    uint4* dst = reinterpret_cast<uint4*>(act);
    const int nv = MT * kpad / 16;
    uint4 cv[CR];
#pragma unroll
    for (int r = 0; r < CR; ++r) {
      const int idx = tid + r * kDecThreads;
      if (idx < nv) cv[r] = __ldcg(src + idx);
    }
    double sa = 0.0;
    int za = 0;
    long long ra = 0;
    if (tid < tok_n) {
      sa = P.s_a[tid];
      za = P.z_a[tid];
      ra = P.rowsum[tid];
    }
#pragma unroll
    for (int r = 0; r < CR; ++r) {
      const int idx = tid + r * kDecThreads;
      if (idx < nv) dst[idx] = cv[r];
    }
    for (int idx = tid + CR * kDecThreads; idx < nv; idx += kDecThreads) dst[idx] = __ldcg(src + idx);
    if (tid < tok_n) {
      s_sa[tid] = sa;
      s_za[tid] = za;
      s_ra[tid] = ra;
    }
    if (blockIdx.x == 0 && tid == 0 && P.bad_out) {
      const unsigned long long w = *P.bad_word;
      *P.bad_out = w ? ~w : ~0ull;
      *P.bad_word = 0ull;
    }
  }
  cta_sync();
  DEC_STAMP(5, clock64());
  DEC_STAMP(13, gtimer());

  // ---- 3. main loop.  Local unit l = warp + NW j lives in ring slot index
  // l / UPS = grp + NG j (group grp = warp / UPS takes the slots = grp mod NG),
  // at position warp % UPS within the slot.
  const int g = lane >> 2, tig = lane & 3;
  const bool has_b = g < MT;
  const uint32_t act_lane = smem_addr(act) + ((g * 4 + tig) * 8);  // B-fragment word pair of (g, tig)
  uint2 b[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) b[c] = make_uint2(0u, 0u);
  int cur_kb = -1;
  auto load_b = [&](int k_b) {  // B fragments of a k-block (kept while it repeats)
    cur_kb = k_b;
    if (!has_b) return;
    const uint32_t ab = act_lane + k_b * (8 * MT * 4 * 8);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(b[c].x), "=r"(b[c].y) : "r"(ab + c * MT * 32));
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
  // running sums of the current row-tile (this warp's k-blocks), fields folded
  uint32_t tot[4] = {0u, 0u, 0u, 0u};
  int tot_rt = -1;
  auto flush_tot = [&]() {
    if (tot_rt < 0) return;
    const int lrt = tot_rt - rt_first;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = g + 8 * (r >> 1), tok = 2 * tig + (r & 1);
      if (tok < tok_n) atomicAdd(&accs[(lrt * 16 + row) * MT + tok], tot[r] >> FSH);
      tot[r] = 0u;
    }
  };
  // fold a unit's accumulator set into the row-tile sums.  Field f holds
  // 2^(QT f) * its partial sum S_f exactly; ((acc_0 << QT) + acc_1) << QT ... =
  // 2^FSH * sum_f S_f (one shift-add per field, LEA); the per-warp row-tile sums
  // stay below 2^32 (<= 16 units of <= 2^FSH * 255 * 255 * 256 each for K <=
  // 65536) and 2^FSH is divided out exactly before the shared atomic.
  auto fold = [&](int (&acc)[NA][4], int r_t) {
    if (r_t != tot_rt) {
      flush_tot();
      tot_rt = r_t;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      uint32_t v = static_cast<uint32_t>(acc[0][r]);
      acc[0][r] = 0;
#pragma unroll
      for (int f = 1; f < NA; ++f) {
        v = (FSH ? (v << QT) : v) + static_cast<uint32_t>(acc[f][r]);
        acc[f][r] = 0;
      }
      tot[r] += v;
    }
  };
  {
    const int grp = warp / UPS;
    const int nw = nu > warp ? (nu - warp + NW - 1) / NW : 0;  // this warp's units
    const uint32_t ring_lane = smem_addr(ring) + (warp % UPS) * unit_bytes + lane * 16;
    auto lds_unit = [&](int sl, uint4 (&w)[QT]) {
      const uint32_t a = ring_lane + sl * slot_bytes;
#pragma unroll
      for (int t = 0; t < QT; ++t)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w) : "r"(a + t * 512));
    };
    // the last of the UPS warps done with ring slot sl refills it with slot
    // index i + S (its data is in registers: the loads have returned)
    const bool refill = nsl > S;  // else every slot was loaded once, at kernel start
    auto release = [&](int sl, int i) {
      if (!refill) return;
      __syncwarp();
      if (lane == 0 && i + S < nsl && atomicAdd(&relcnt[sl], 1u) == UPS - 1) {
        relcnt[sl] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_slot(i + S, sl);
      }
    };
    int accA[NA][4], accB[NA][4];
#pragma unroll
    for (int f = 0; f < NA; ++f)
#pragma unroll
      for (int r = 0; r < 4; ++r) accA[f][r] = accB[f][r] = 0;
    // fetch cursor (slot index, ring slot, parity, row-tile, k-block)
    int fi = grp, fs = grp;
    uint32_t fph = 0;
    int frt = (U0 + warp) / kbl, fkb = U0 + warp - frt * kbl;
    auto advance = [&]() {
      fi += NG;
      fs += NG;
      if (fs >= S) {
        fs -= S;
        fph ^= 1u;
      }
      fkb += NW;
      while (fkb >= kbl) {
        fkb -= kbl;
        ++frt;
      }
    };
    uint4 w[QT];
    int rtA = -1, rtB = -1;
    DEC_STAMP(16, clock64());
#ifdef ABQ_TRACE
    unsigned long long last_data = 0;
#define DEC_LAST_DATA() do { if (P.trace && tid == 0) last_data = gtimer(); } while (0)
#else
#define DEC_LAST_DATA() do { } while (0)
#endif
    for (int j = 0; j < nw; j += 2) {
      // unit j -> set A (fold set B = unit j - 1 behind its IMMAs)
      mbar_wait_parity(&full[fs], fph);
      DEC_LAST_DATA();
      if (j == 0) DEC_STAMP(17, clock64());
      if (j == 0) DEC_STAMP(22, gtimer());
      lds_unit(fs, w);
      const int slA = fs, iA = fi, kbA = fkb;
      rtA = frt;
      advance();
      if (kbA != cur_kb) load_b(kbA);
      mma_unit(accA, w);
      release(slA, iA);
      if (j > 0) fold(accB, rtB);
      if (j + 1 >= nw) break;
      // unit j + 1 -> set B (fold set A behind its IMMAs)
      mbar_wait_parity(&full[fs], fph);
      DEC_LAST_DATA();
      lds_unit(fs, w);
      const int slB = fs, iB = fi, kbB = fkb;
      rtB = frt;
      advance();
      if (kbB != cur_kb) load_b(kbB);
      mma_unit(accB, w);
      release(slB, iB);
      fold(accA, rtA);
      if (j == 0) DEC_STAMP(18, clock64());
      rtA = -1;
    }
    DEC_STAMP(19, clock64());
    DEC_STAMP(14, gtimer());
#ifdef ABQ_TRACE
    if (P.trace && tid == 0) trace[21] = last_data;
#endif
    if (rtA >= 0) fold(accA, rtA);
    else if (nw > 0 && (nw & 1) == 0) fold(accB, rtB);
    flush_tot();
    DEC_STAMP(20, clock64());
#ifdef ABQ_TRACE
    if (P.trace && lane == 0) trace[24 + warp] = clock64();
#endif
  }
  // epilogue values to shared memory (requested at kernel start), token code
  // sums of the fused ReQuant from the per-warp partials
  if (has_p) {
    c_sb[tid] = p_sb;
    c_zb[tid] = p_zb;
    c_cs[tid] = p_cs;
  }
  for (int idx = tid + kDecThreads; dequant && idx < nlrt * 16; idx += kDecThreads) {
    const int j = rt_first * kRowTile + idx;
    if (j < P.n) {
      c_sb[idx] = P.e.s_b[static_cast<size_t>(j) * P.e.sb_stride];
      c_zb[idx] = P.e.z_b[static_cast<size_t>(j) * P.e.zb_stride];
      c_cs[idx] = P.e.colsum_b[j];
    }
  }
  if (FUSED && tid < tok_n) {
    constexpr int GT = NW / MT;
    long long s = 0;
#pragma unroll
    for (int w2 = 0; w2 < GT; ++w2) s += r_sum[tid * GT + w2];
    s_ra[tid] = s;
  }
  cta_sync();
  DEC_STAMP(6, clock64());

  // ---- 4. epilogue: zero-point correction + dequant of this CTA's channels
  const EpiParams& E = P.e;
  for (int idx = tid; idx < nlrt * 16 * MT; idx += kDecThreads) {
    const int i = idx & (MT - 1), rc = idx / MT, lrt = rc >> 4, row = rc & 15;
    const int j = (rt_first + lrt) * kRowTile + row;
    if (i >= tok_n || j >= P.n) continue;
    const long long a = accs[idx];
    if (!dequant) {
      epi_store_raw(E, i, j, a);
      continue;
    }
    const long long za = s_za[i], zb = c_zb[rc];
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
#ifdef ABQ_TRACE
  if (trace && tid == 0) {
    trace[7] = clock64();
    trace[9] = gtimer();
  }
#endif
}

// ============================================================================
// host side
// ============================================================================
unsigned long long*& trace_buffer();

DecTuning& dec_tuning() {
  static DecTuning t;
  return t;
}

template <int QT, int MT>
static int launch_dec2(const DecParams& P, int grid, size_t smem, bool pdl, cudaStream_t st) {
  auto kern = !P.x16 ? gemv_dec_kernel<QT, MT, 0>
              : P.xr <= 1 ? gemv_dec_kernel<QT, MT, 1>
              : P.xr <= 2 ? gemv_dec_kernel<QT, MT, 2> : gemv_dec_kernel<QT, MT, 4>;
  if (smem > 220 * 1024) return fail(ABQ_ERR_VALUE, "gemv_dec: shared memory plan too large (%zu B)", smem);
  // the attributes are set once per instantiation and device (and raised when
  // a larger plan needs it): they are host API calls on every launch otherwise
  static size_t set_smem[4][64] = {};  // [kernel variant][device]
  const int var = !P.x16 ? 0 : P.xr <= 1 ? 1 : P.xr <= 2 ? 2 : 3;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t err = cudaSuccess;
  if (dev < 0 || dev >= 64 || smem > set_smem[var][dev]) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (err == cudaSuccess && dev >= 0 && dev < 64) set_smem[var][dev] = smem;
  }
  if (err != cudaSuccess) return fail(ABQ_ERR_CUDA, "gemv_dec: smem attribute: %s", cudaGetErrorString(err));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDecBlock);
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

static int dec_mt(size_t m) { return m <= 1 ? 1 : m <= 2 ? 2 : m <= 4 ? 4 : 8; }
static const size_t kDecSmemBudget = 212 * 1024;

// ring slots for a layer: as deep as the CTA's whole weight share when that
// fits in shared memory (then every TMA copy is issued at kernel start and no
// refill latency is exposed), else as many as fit (>= 2)
static int dec_slots(unsigned q, size_t n, size_t k, int mt, int grid) {
  const int rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  const int kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  const int nl = dec_nlrt_max(rowtiles, grid);
  const int min_slots = 2;
  int slots = std::max(min_slots, std::min(32, (nl * kblocks + kDecUPS - 1) / kDecUPS));
  if (dec_tuning().ring_kb > 0)
    slots = std::max(min_slots, static_cast<int>(dec_tuning().ring_kb * 1024 / (size_t(kDecUPS) * q * 512)));
  while (slots > min_slots && dec_smem(q, slots, mt, kblocks * kKBlock, nl).total > kDecSmemBudget) --slots;
  return slots;
}

// the decode GEMV handles this layer (activation codes of mt tokens plus a
// minimal 2-slot ring and the per-channel epilogue values fit shared memory)
bool dec_supported(unsigned q, size_t n, size_t k, size_t m) {
  if (m < 1 || m > 8 || n == 0 || k == 0 || k > 65536 || q < 1 || q > 8) return false;
  const int mt = dec_mt(m);
  const int rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  const int grid = std::min(num_sms(), rowtiles);
  const int kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  return dec_smem(q, 2, mt, kblocks * kKBlock, dec_nlrt_max(rowtiles, grid)).total <=
         kDecSmemBudget;
}

// Serving decode path (m <= 8).  `ws` = imma_ws_bytes(n, k) of zero-filled
// device memory (left zeroed): activation codes, stats, the non-finite report
// word.  fp16 per-token activations with K % 8 == 0 are quantized inside the
// GEMV (one launch); anything else goes through act_quant_kernel first, with
// this kernel as its PDL secondary.  Every launch is itself PDL-enabled so
// consecutive layers overlap.
static int launch_dec(DecParams& P, size_t m, bool fused, bool qact, cudaStream_t st, const DecNext* nx);

// Consumer of a producer-fused ReQuant (producer.cu): codes already in the
// B-fragment layout of dec_mt(m) tokens, with s_a / z_a / code row sums.
int run_gemv_dec_qact(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const uint32_t* codes,
                      const double* s_a, const int32_t* z_a, const long long* rowsum, const QuantParams& qp,
                      const EpiParams& e, cudaStream_t st, const DecNext* nx) {
  if (m == 0 || n == 0) return ABQ_OK;
  if (!dec_supported(q, n, k, m)) return fail(ABQ_ERR_VALUE, "gemv_dec: layer shape not supported");
  DecParams P{};
  P.frag = frag;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  P.kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  P.m = static_cast<int>(m);
  P.e = e;
  P.qp = qp;
  P.trace = trace_buffer();
  P.act_frag = codes;
  P.s_a = s_a;
  P.z_a = z_a;
  P.rowsum = rowsum;
  return launch_dec(P, m, false, true, st, nx);
}

int run_gemv_dec(const uint32_t* frag, unsigned q, size_t n, size_t k, size_t m, const void* x, int x_dtype,
                 const QuantParams& qp, const EpiParams& e, void* ws, unsigned long long* bad_out,
                 cudaStream_t st, const DecNext* nx) {
  if (m == 0 || n == 0) return ABQ_OK;
  if (!dec_supported(q, n, k, m)) return fail(ABQ_ERR_VALUE, "gemv_dec: layer shape not supported");
  DecParams P{};
  P.frag = frag;
  P.q = static_cast<int>(q);
  P.n = static_cast<int>(n);
  P.k = static_cast<int>(k);
  P.rowtiles = static_cast<int>((n + kRowTile - 1) / kRowTile);
  P.kblocks = static_cast<int>((k + kKBlock - 1) / kKBlock);
  P.m = static_cast<int>(m);
  P.e = e;
  P.qp = qp;
  P.trace = trace_buffer();
  const int mt = dec_mt(m);
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
  // fused ReQuant: each of the 32*kDecWarps/mt threads of a token holds <= kDecXR vectors of 8
  const bool fused = x_dtype == ABQ_F16 && !qp.per_tensor && k % 8 == 0 &&
                     k <= static_cast<size_t>(8 * kDecXR * 32 * kDecWarps / mt);
  if (fused) {
    P.x16 = static_cast<const __half*>(x);
    const size_t tpt = 32 * kDecWarps / mt, nvec = k / 8;
    P.xr = nvec <= tpt ? 1 : nvec <= 2 * tpt ? 2 : 4;
  } else {
    const int rc = run_act_quant(x, x_dtype, m, k, mt, qp, act_frag, 0, s_a, z_a, rowsum, P.bad_word, st);
    if (rc) return rc;
    P.act_frag = act_frag;
    P.s_a = s_a;
    P.z_a = z_a;
    P.rowsum = rowsum;
  }
  return launch_dec(P, m, fused, false, st, nx);
}

// grid: one CTA per SM; with dec_grid_balanced, only as many CTAs as give
// every CTA the same (maximal) number of row-tiles (no light CTAs)
static int dec_grid(int rowtiles) {
  int grid = std::min(num_sms(), rowtiles);
  if (dec_tuning().grid_balanced) {
    const int per = (rowtiles + grid - 1) / grid;
    grid = (rowtiles + per - 1) / per;
  }
  return grid;
}

static int launch_dec(DecParams& P, size_t m, bool fused, bool qact, cudaStream_t st, const DecNext* nx) {
  const unsigned q = static_cast<unsigned>(P.q);
  const size_t n = static_cast<size_t>(P.n), k = static_cast<size_t>(P.k);
  const int mt = dec_mt(m);
  const int kpad = P.kblocks * kKBlock;
  const int grid = dec_grid(P.rowtiles);
  P.l2_plain = dec_tuning().l2_plain;
  P.dbg_nostream = dec_tuning().dbg_nostream;
  // successor prefetch only behind a long stream (measured: +5 % at W4 up_proj,
  // 152 KB per CTA; -1..-5 % for shares <= ~76 KB, profiles/r02_dec_next_sweep.txt)
  const size_t share = static_cast<size_t>(dec_nlrt_max(P.rowtiles, grid)) * P.kblocks * q * 512;
  if (nx && nx->frag && dec_tuning().next_kb > 0 && share >= static_cast<size_t>(dec_tuning().next_min_kb) * 1024) {
    P.nx = reinterpret_cast<const unsigned char*>(nx->frag);
    P.nx_rowtiles = static_cast<int>((nx->n + kRowTile - 1) / kRowTile);
    P.nx_kblocks = static_cast<int>((nx->k + kKBlock - 1) / kKBlock);
    P.nx_unit = static_cast<int>(nx->q) * 512;
    P.nx_grid = dec_grid(P.nx_rowtiles);
    P.nx_bytes = dec_tuning().next_kb * 1024;
    P.nx_at = std::min(100, std::max(1, dec_tuning().next_at));
  }
  const int nl = dec_nlrt_max(P.rowtiles, grid);
  P.slots = dec_slots(q, n, k, mt, grid);
  const size_t slot_bytes = static_cast<size_t>(kDecUPS) * q * 512;
  // slots in flight before the activations are awaited (the rest is issued
  // right behind the activation loads)
  // Measured (profiles/r02_dec_prekb_sweep.txt): when the ring holds the CTA's
  // whole share, issuing it only behind the activation loads is fastest (the
  // activations do not queue behind the stream); when it must be refilled
  // (W8 at LLaMA-7B up_proj: 305 KB per SM), ~64 KB up front is.
  const int whole = (nl * P.kblocks + kDecUPS - 1) / kDecUPS;
  const int pre_kb = dec_tuning().pre_kb >= 0 ? dec_tuning().pre_kb : (P.slots >= whole ? 0 : 64);
  // (the paths whose activations come from a preceding kernel -- the
  // ReQuant kernel or a producer with the ReQuant fused in -- issue the whole
  // ring up front: their wait covers that kernel's run, which the stream then
  // overlaps; measured best in the LLaMA-7B decode chain, profiles/r02_chain_prekb_sweep.txt)
  (void)qact;
  P.preslots = fused ? std::max(0, std::min(P.slots, static_cast<int>(pre_kb * 1024 / slot_bytes))) : P.slots;
  // (measured: ~4x the SM's ~43 B/ns share of HBM bandwidth is best, profiles/r02_dec_pace_sweep.txt)
  // Paced slots only when the ring holds the whole share; a refilled ring
  // keeps its 64 KB up front and waits for the activation loads.
  P.pace_ns = dec_tuning().pace_ns > 0 ? dec_tuning().pace_ns
              : P.slots >= whole         ? static_cast<int>(slot_bytes / 160)
                                         : 0;
  const size_t smem = dec_smem(q, P.slots, mt, kpad, nl).total;
  const bool pdl = dec_tuning().pdl != 0;
  switch (mt) {
    case 1: return launch_dec1<1>(P, grid, smem, pdl, st);
    case 2: return launch_dec1<2>(P, grid, smem, pdl, st);
    case 4: return launch_dec1<4>(P, grid, smem, pdl, st);
    default: return launch_dec1<8>(P, grid, smem, pdl, st);
  }
}

}  // namespace abq_dev
