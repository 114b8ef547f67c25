// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (the checker, never the product).  Compiled by
// oracle/Makefile against /root/reference/proj/include (never copied into this
// repo) into oracle/_ref/libabqref.so.  Used to (1) pin the C restatement in
// oracle/abq_oracle.c and (2) as the CPU baseline / `bench.py --impl
// reference` arm, which times the reference's own gemm_arbitrary /
// quantized_linear on the GPU box's host cores.
#include <cstdint>
#include <cstring>
#include <optional>
#include <thread>
#include <vector>

#include "abq/bitplane.hpp"
#include "abq/core.hpp"
#include "abq/gemm.hpp"
#include "abq/quantizer.hpp"
#include "abq/tune.hpp"

namespace {

abq::BitPlaneMatrix planes_from(const std::uint64_t* data, unsigned planes, std::size_t rows,
                                std::size_t cols) {
  abq::BitPlaneMatrix m(planes, rows, cols);
  std::memcpy(m.data.data(), data, m.data.size() * sizeof(std::uint64_t));
  return m;
}

int status_of(const abq::Error& e) {
  if (dynamic_cast<const abq::ShapeError*>(&e)) return 1;
  if (dynamic_cast<const abq::ValueError*>(&e)) return 2;
  if (dynamic_cast<const abq::OverflowError*>(&e)) return 3;
  return 4;
}

}  // namespace

extern "C" {

// bitpack  bitplane.hpp:47-64
int ref_bitpack(const std::uint8_t* codes, std::size_t rows, std::size_t cols, unsigned bits,
                std::uint64_t* planes) {
  try {
    abq::CodeMat c(rows, cols);
    std::memcpy(c.data.data(), codes, rows * cols);
    auto m = abq::bitpack(c, bits);
    std::memcpy(planes, m.data.data(), m.data.size() * sizeof(std::uint64_t));
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

// gemm_arbitrary  gemm.hpp:185-198 (default_tile or caller tile)
int ref_gemm_arbitrary(const std::uint64_t* a, unsigned p, std::size_t m, const std::uint64_t* bt,
                       unsigned q, std::size_t n, std::size_t k, std::int32_t* out,
                       unsigned threads) {
  try {
    auto pa = planes_from(a, p, m, k);
    auto pb = planes_from(bt, q, n, k);
    abq::engine_threads() = threads;
    auto r = abq::gemm_arbitrary(pa, pb, abq::default_tile(p, q));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(std::int32_t));
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

// Timing entry: planes already wrapped once (outside the timed region).
void* ref_planes_new(const std::uint64_t* data, unsigned planes, std::size_t rows,
                     std::size_t cols) {
  return new abq::BitPlaneMatrix(planes_from(data, planes, rows, cols));
}
void ref_planes_free(void* h) { delete static_cast<abq::BitPlaneMatrix*>(h); }

// The reference's own bench kernel (abqtool.cpp:129-140): gemm_arbitrary with
// default_tile on pre-packed planes; writes the result so it cannot be elided.
int ref_gemm_arbitrary_h(const void* a, const void* bt, std::int32_t* out, unsigned threads) {
  try {
    const auto& pa = *static_cast<const abq::BitPlaneMatrix*>(a);
    const auto& pb = *static_cast<const abq::BitPlaneMatrix*>(bt);
    abq::engine_threads() = threads;
    auto r = abq::gemm_arbitrary(pa, pb, abq::default_tile(pa.planes, pb.planes));
    if (out) std::memcpy(out, r.data.data(), r.data.size() * sizeof(std::int32_t));
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

int ref_gemm_naive_h(const void* a, const void* bt, std::int32_t* out) {
  const auto& pa = *static_cast<const abq::BitPlaneMatrix*>(a);
  const auto& pb = *static_cast<const abq::BitPlaneMatrix*>(bt);
  auto r = abq::gemm_naive(pa, pb);
  if (out) std::memcpy(out, r.data.data(), r.data.size() * sizeof(std::int32_t));
  return 0;
}

// gemm_arbitrary_wide  gemm.hpp:201-209
int ref_gemm_arbitrary_wide(const std::uint64_t* a, unsigned p, std::size_t m,
                            const std::uint64_t* bt, unsigned q, std::size_t n, std::size_t k,
                            std::int64_t* out) {
  try {
    auto pa = planes_from(a, p, m, k);
    auto pb = planes_from(bt, q, n, k);
    auto r = abq::gemm_arbitrary_wide(pa, pb, abq::default_tile(p, q));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(std::int64_t));
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

// quantize  quantizer.hpp:146-213 (comp_a/comp_b may be null)
int ref_quantize(const double* x, std::size_t rows, std::size_t cols, unsigned bits, int scheme,
                 int granularity, double alpha, double beta, const double* comp_a,
                 const double* comp_b, std::uint8_t* codes, double* scales,
                 std::int32_t* zero_points) {
  try {
    abq::Mat m(rows, cols);
    std::memcpy(m.data.data(), x, rows * cols * sizeof(double));
    abq::QuantSpec spec;
    spec.bits = bits;
    spec.scheme = abq::Scheme(scheme);
    spec.granularity = abq::Granularity(granularity);
    spec.alpha = alpha;
    spec.beta = beta;
    std::optional<abq::CompensationPair> comp;
    if (comp_a && comp_b)
      comp = abq::CompensationPair{std::vector<double>(comp_a, comp_a + rows),
                                   std::vector<double>(comp_b, comp_b + cols)};
    auto q = abq::quantize(m, spec, comp);
    std::memcpy(codes, q.codes.data.data(), rows * cols);
    std::memcpy(scales, q.scales.data(), q.scales.size() * sizeof(double));
    std::memcpy(zero_points, q.zero_points.data(), q.zero_points.size() * sizeof(std::int32_t));
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

// quantized_linear  gemm.hpp:266-307 on pre-quantized tensors
int ref_quantized_linear(const std::uint8_t* act, std::size_t m, unsigned a_bits, int a_scheme,
                         int a_gran, const double* s_a, const std::int32_t* z_a,
                         const std::uint8_t* wt, std::size_t n, unsigned w_bits, int w_scheme,
                         int w_gran, const double* s_b, const std::int32_t* z_b, std::size_t k,
                         double* out, std::uint64_t* stats2) {
  try {
    abq::QuantizedTensor qa, qw;
    qa.codes = abq::CodeMat(m, k);
    std::memcpy(qa.codes.data.data(), act, m * k);
    qa.spec.bits = a_bits;
    qa.spec.scheme = abq::Scheme(a_scheme);
    qa.spec.granularity = abq::Granularity(a_gran);
    std::size_t ga = a_gran == 0 ? 1 : m;
    qa.scales.assign(s_a, s_a + ga);
    qa.zero_points.assign(z_a, z_a + ga);
    qw.codes = abq::CodeMat(n, k);
    std::memcpy(qw.codes.data.data(), wt, n * k);
    qw.spec.bits = w_bits;
    qw.spec.scheme = abq::Scheme(w_scheme);
    qw.spec.granularity = abq::Granularity(w_gran);
    std::size_t gb = w_gran == 0 ? 1 : n;
    qw.scales.assign(s_b, s_b + gb);
    qw.zero_points.assign(z_b, z_b + gb);
    abq::GemmStats st;
    auto r = abq::quantized_linear(qa, qw, &st);
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
    if (stats2) {
      stats2[0] = st.block_tiles;
      stats2[1] = st.plane_pair_products;
    }
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

// ---- reference linear step for the CPU baseline -----------------------------
// quantized_linear's body (gemm.hpp:266-307) with the per-call weight bitpack
// (gemm.hpp:274, 278) hoisted out of the step -- weights are packed once, as the
// engine does -- so the reference is timed on exactly the engine's per-step
// work: quantize(act) -> bitpack(act) -> code_rowsums(act) -> gemm_arbitrary
// (default_tile) -> zero_point_correct -> dequant.  threads > 1 is a
// harness-parallel split of the output channels across std::threads, each
// running the same reference calls on its slice (the reference itself only
// parallelises over 64-row tiles of M, gemm.hpp:150-177).
struct RefLinearSlice {
  std::size_t n0, n1;
  abq::BitPlaneMatrix w;
  std::vector<std::int64_t> colsum;
  std::vector<std::int32_t> z_b;
  std::vector<double> s_b;
};
struct RefLinear {
  std::size_t n, k;
  unsigned w_bits;
  std::vector<RefLinearSlice> slices;
};

void* ref_linear_new(const std::uint8_t* wt_codes, std::size_t n, std::size_t k, unsigned w_bits,
                     const double* s_b, const std::int32_t* z_b, unsigned threads) {
  auto* h = new RefLinear{n, k, w_bits, {}};
  if (threads < 1) threads = 1;
  for (unsigned t = 0; t < threads; ++t) {
    std::size_t n0 = n * t / threads, n1 = n * (t + 1) / threads;
    if (n0 == n1) continue;
    abq::CodeMat c(n1 - n0, k);
    std::memcpy(c.data.data(), wt_codes + n0 * k, (n1 - n0) * k);
    RefLinearSlice s{n0, n1, abq::bitpack(c, w_bits), abq::code_rowsums(c),
                     std::vector<std::int32_t>(z_b + n0, z_b + n1),
                     std::vector<double>(s_b + n0, s_b + n1)};
    h->slices.push_back(std::move(s));
  }
  return h;
}

void ref_linear_free(void* h) { delete static_cast<RefLinear*>(h); }

int ref_linear_run(void* hv, const double* x, std::size_t m, unsigned a_bits, double* out) {
  try {
    auto* h = static_cast<RefLinear*>(hv);
    abq::Mat xm(m, h->k);
    std::memcpy(xm.data.data(), x, m * h->k * sizeof(double));
    abq::QuantSpec spec;
    spec.bits = a_bits;
    spec.granularity = abq::Granularity::PerToken;
    abq::QuantizedTensor qa = abq::quantize(xm, spec);  // ReQuant
    abq::BitPlaneMatrix a = abq::bitpack(qa.codes, spec.planes());
    auto rows_a = abq::code_rowsums(qa.codes);
    abq::engine_threads() = 1;
    auto work = [&](const RefLinearSlice& s) {
      const std::size_t ns = s.n1 - s.n0;
      auto acc = abq::gemm_arbitrary(a, s.w, abq::default_tile(a.planes, s.w.planes));
      auto corrected = abq::zero_point_correct(acc, rows_a, s.colsum, qa.zero_points, s.z_b, h->k);
      for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < ns; ++j)
          out[i * h->n + s.n0 + j] = qa.scales[i] * s.s_b[j] * corrected(i, j);
    };
    if (h->slices.size() == 1) {
      work(h->slices[0]);
    } else {
      std::vector<std::thread> pool;
      for (const auto& s : h->slices) pool.emplace_back(work, std::cref(s));
      for (auto& t : pool) t.join();
    }
    return 0;
  } catch (const abq::Error& e) {
    return status_of(e);
  }
}

double ref_padding_redundancy(std::size_t m, unsigned p, std::size_t mma_m) {
  try {
    return abq::padding_redundancy(m, p, mma_m);
  } catch (const abq::Error&) {
    return -1.0;
  }
}

int ref_fits_int32(unsigned p, unsigned q, std::size_t k) { return abq::fits_int32(p, q, k); }

}  // extern "C"
