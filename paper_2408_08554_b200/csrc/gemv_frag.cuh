// gemv_frag.cuh -- pieces shared by the decode GEMV kernels (gemv_imma.cu,
// gemv_dec.cu): the fragment-major weight layout constants, PTX wrappers for
// mbarriers / 1-D TMA bulk copies / PDL / legacy IMMA, the code-slice
// widening and the B-fragment order of the activation codes.
#pragma once

#include "common.cuh"

namespace abq_dev {

constexpr int kRowTile = 16;
constexpr int kKBlock = 256;

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITG_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITG_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// Same copy with an L2 eviction-priority policy (createpolicy): weight streams
// are read once per step, so they are marked evict_first and do not push the
// kernel's code, parameters and activations out of L2 (a 500 MB weight
// rotation otherwise evicts them every launch and each instruction-cache or
// constant miss then waits behind the weight stream in HBM).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                  uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ void imma_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Byte-code register o (= 4c + u: chunk c, A register u) of a lane's unit from
// its 4Q code-slice words (layout in prepack_frag_kernel / common.cuh):
// one shift + one mask-merge per slice, all shifts compile-time constants.
template <int Q>
__device__ __forceinline__ uint32_t widen_slices(const uint4 (&w)[Q], int o) {
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

// CTA that owns unit u under the even split (c*U)/G
__device__ __forceinline__ int cta_of_unit(long long u, long long U, int G) {
  return static_cast<int>(((u + 1) * G - 1) / U);
}

// u32 index of activation codes (k-group v of 4, token i) in B-fragment order:
// [kb][c][token i][tig][h]   (kb = v/64, c = (v%64)/8, h = (v%8)/4, tig = v%4)
__device__ __forceinline__ int act_frag_index(int v, int i, int mt) {
  const int kb = v >> 6, rem = v & 63;
  return ((((kb * 8 + (rem >> 3)) * mt + i) * 4 + (rem & 3)) * 2) + ((rem >> 2) & 1);
}

}  // namespace abq_dev
