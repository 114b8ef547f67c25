// gen_golden.cpp -- emit golden vectors from the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile against
// /root/reference/proj/include into oracle/_ref/gen_golden and run by
// tests/golden/make_golden.py, which converts the stream into the committed
// tests/golden/reference_cases.npz.  Each block below replays one seeded case
// family from the reference's own test suite, with the same abq::Rng seed and
// the same draw order, and records inputs + the reference's outputs:
//   test_bitkernel.cpp:36-180 (seeds 21-29), acceptance.cpp:29-104 (seeds 42,
//   43), test_quantizer.cpp:33-128 (seeds 7, 11, 3 + degenerate case).
//
// Stream format: repeated records
//   u32 name_len, name bytes, u8 dtype (0=u8 1=i32 2=i64 3=u64 4=f64),
//   u32 ndim, u64 dims[ndim], raw little-endian data.
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "abq/bitplane.hpp"
#include "abq/core.hpp"
#include "abq/gemm.hpp"
#include "abq/quantizer.hpp"

namespace {

std::FILE* out_file = nullptr;

template <typename T>
std::uint8_t dtype_code();
template <> std::uint8_t dtype_code<std::uint8_t>() { return 0; }
template <> std::uint8_t dtype_code<std::int32_t>() { return 1; }
template <> std::uint8_t dtype_code<std::int64_t>() { return 2; }
template <> std::uint8_t dtype_code<std::uint64_t>() { return 3; }
template <> std::uint8_t dtype_code<double>() { return 4; }

template <typename T>
void emit(const std::string& name, const T* data, std::vector<std::uint64_t> dims) {
  std::uint32_t nl = std::uint32_t(name.size());
  std::fwrite(&nl, 4, 1, out_file);
  std::fwrite(name.data(), 1, nl, out_file);
  std::uint8_t dt = dtype_code<T>();
  std::fwrite(&dt, 1, 1, out_file);
  std::uint32_t nd = std::uint32_t(dims.size());
  std::fwrite(&nd, 4, 1, out_file);
  std::uint64_t count = 1;
  for (auto d : dims) {
    std::fwrite(&d, 8, 1, out_file);
    count *= d;
  }
  if (count) std::fwrite(data, sizeof(T), count, out_file);
}

template <typename T>
void emit_mat(const std::string& name, const abq::Matrix<T>& m) {
  emit(name, m.data.data(), {m.rows, m.cols});
}

void emit_planes(const std::string& name, const abq::BitPlaneMatrix& m) {
  emit(name, m.data.data(), {m.planes, m.rows, m.words_per_row});
}

template <typename T>
void emit_vec(const std::string& name, const std::vector<T>& v) {
  emit(name, v.data(), {v.size()});
}

void emit_scalar_i64(const std::string& name, std::int64_t v) { emit(name, &v, {1}); }

std::string idx(const std::string& base, int i) { return base + "/" + std::to_string(i); }

void emit_qt(const std::string& base, const abq::QuantizedTensor& q) {
  emit_mat(base + "/codes", q.codes);
  emit_vec(base + "/scales", q.scales);
  emit_vec(base + "/zero_points", q.zero_points);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: gen_golden OUT\n");
    return 2;
  }
  out_file = std::fopen(argv[1], "wb");
  if (!out_file) return 1;

  // test_bitkernel.cpp:36-52 bitpack round trip, seed 21
  {
    abq::Rng rng(21);
    for (unsigned bits = 1; bits <= 8; ++bits) {
      abq::CodeMat c = rng.code_matrix(5, 70, bits);
      emit_mat(idx("bitpack", bits) + "/codes", c);
      emit_planes(idx("bitpack", bits) + "/planes", abq::bitpack(c, bits));
    }
  }
  // test_bitkernel.cpp:54-66 bmma, seed 22
  {
    abq::Rng rng(22);
    abq::CodeMat a = rng.code_matrix(4, 130, 3);
    abq::CodeMat b = rng.code_matrix(5, 130, 2);
    auto pa = abq::bitpack(a, 3), pb = abq::bitpack(b, 2);
    emit_mat("bmma/a", a);
    emit_mat("bmma/b", b);
    for (unsigned s = 0; s < 3; ++s)
      for (unsigned t = 0; t < 2; ++t)
        emit_mat("bmma/out/" + std::to_string(s) + "_" + std::to_string(t), abq::bmma(pa, s, pb, t));
  }
  // test_bitkernel.cpp:68-80 gemm_arbitrary vs oracle, seed 23, 60 trials
  {
    abq::Rng rng(23);
    for (int trial = 0; trial < 60; ++trial) {
      std::size_t m = rng.integer(1, 48), n = rng.integer(1, 48), k = rng.integer(1, 200);
      unsigned p = unsigned(rng.integer(1, 8)), q = unsigned(rng.integer(1, 8));
      abq::CodeMat a = rng.code_matrix(m, k, p);
      abq::CodeMat b = rng.code_matrix(n, k, q);
      auto got = abq::gemm_arbitrary(abq::bitpack(a, p), abq::bitpack(b, q), abq::default_tile(p, q));
      std::int64_t pq[2] = {p, q};
      emit(idx("gemm23", trial) + "/pq", pq, {2});
      emit_mat(idx("gemm23", trial) + "/a", a);
      emit_mat(idx("gemm23", trial) + "/b", b);
      emit_mat(idx("gemm23", trial) + "/out", got);
    }
  }
  // test_bitkernel.cpp:82-88 naive == tiled, seed 24
  {
    abq::Rng rng(24);
    abq::CodeMat a = rng.code_matrix(9, 300, 5);
    abq::CodeMat b = rng.code_matrix(11, 300, 3);
    auto pa = abq::bitpack(a, 5), pb = abq::bitpack(b, 3);
    emit_mat("naive24/a", a);
    emit_mat("naive24/b", b);
    emit_mat("naive24/naive", abq::gemm_naive(pa, pb));
    emit_mat("naive24/tiled", abq::gemm_arbitrary(pa, pb, abq::default_tile(5, 3)));
  }
  // test_bitkernel.cpp:90-102 overflow boundary, seed 25
  {
    abq::Rng rng(25);
    std::size_t k = std::size_t{1} << 15;
    abq::CodeMat a = rng.code_matrix(1, k, 8);
    abq::CodeMat b = rng.code_matrix(1, k, 8);
    auto pa = abq::bitpack(a, 8), pb = abq::bitpack(b, 8);
    int threw = 0;
    try {
      abq::gemm_arbitrary(pa, pb, abq::default_tile(8, 8));
    } catch (const abq::OverflowError&) {
      threw = 1;
    }
    emit_mat("overflow25/a", a);
    emit_mat("overflow25/b", b);
    emit_scalar_i64("overflow25/threw", threw);
    emit_mat("overflow25/wide", abq::gemm_arbitrary_wide(pa, pb, abq::default_tile(8, 8)));
  }
  // test_bitkernel.cpp:104-115 tile transparency, seed 26
  {
    abq::Rng rng(26);
    abq::CodeMat a = rng.code_matrix(33, 500, 3);
    abq::CodeMat b = rng.code_matrix(29, 500, 5);
    auto pa = abq::bitpack(a, 3), pb = abq::bitpack(b, 5);
    emit_mat("tile26/a", a);
    emit_mat("tile26/b", b);
    emit_mat("tile26/out", abq::gemm_arbitrary(pa, pb, abq::default_tile(3, 5)));
  }
  // test_bitkernel.cpp:126-148 zero-point correction, seed 27, 20 trials
  {
    abq::Rng rng(27);
    for (int trial = 0; trial < 20; ++trial) {
      std::size_t m = rng.integer(1, 10), n = rng.integer(1, 10), k = rng.integer(1, 64);
      unsigned p = 4, q = 4;
      abq::CodeMat a = rng.code_matrix(m, k, p);
      abq::CodeMat b = rng.code_matrix(n, k, q);
      std::vector<std::int32_t> za, zb;
      for (std::size_t i = 0; i < m; ++i) za.push_back(std::int32_t(rng.integer(0, 15)));
      for (std::size_t j = 0; j < n; ++j) zb.push_back(std::int32_t(rng.integer(0, 15)));
      auto acc = abq::gemm_arbitrary(abq::bitpack(a, p), abq::bitpack(b, q), abq::default_tile(p, q));
      auto corrected = abq::zero_point_correct(acc, abq::code_rowsums(a), abq::code_rowsums(b), za, zb, k);
      emit_mat(idx("zp27", trial) + "/a", a);
      emit_mat(idx("zp27", trial) + "/b", b);
      emit_vec(idx("zp27", trial) + "/za", za);
      emit_vec(idx("zp27", trial) + "/zb", zb);
      emit_mat(idx("zp27", trial) + "/acc", acc);
      emit_mat(idx("zp27", trial) + "/corrected", corrected);
    }
  }
  // test_bitkernel.cpp:150-168 quantized_linear, seed 28
  {
    abq::Rng rng(28);
    abq::Mat x = rng.gauss_matrix(6, 64);
    abq::Mat w = rng.gauss_matrix(9, 64);
    abq::QuantSpec sa;
    sa.bits = 5;
    sa.granularity = abq::Granularity::PerToken;
    abq::QuantSpec sw;
    sw.bits = 3;
    sw.granularity = abq::Granularity::PerChannel;
    abq::QuantizedTensor qa = abq::quantize(x, sa), qw = abq::quantize(w, sw);
    abq::GemmStats stats;
    abq::Mat got = abq::quantized_linear(qa, qw, &stats);
    emit_mat("qlinear28/x", x);
    emit_mat("qlinear28/w", w);
    emit_qt("qlinear28/qa", qa);
    emit_qt("qlinear28/qw", qw);
    emit_mat("qlinear28/out", got);
    std::int64_t st[2] = {std::int64_t(stats.block_tiles), std::int64_t(stats.plane_pair_products)};
    emit("qlinear28/stats", st, {2});
  }
  // test_bitkernel.cpp:170-180 stats law, seed 29
  {
    abq::Rng rng(29);
    abq::CodeMat a = rng.code_matrix(70, 128, 2);
    abq::CodeMat b = rng.code_matrix(70, 128, 3);
    abq::GemmStats stats;
    abq::TileConfig t{32, 32, 128, 32, 32, 128};
    auto out = abq::gemm_arbitrary(abq::bitpack(a, 2), abq::bitpack(b, 3), t, &stats);
    emit_mat("stats29/a", a);
    emit_mat("stats29/b", b);
    emit_mat("stats29/out", out);
    std::int64_t st[2] = {std::int64_t(stats.block_tiles), std::int64_t(stats.plane_pair_products)};
    emit("stats29/stats", st, {2});
  }
  // acceptance.cpp:29-52 decomposition equivalence, seed 42 (first 120 of 1000 cases)
  {
    abq::Rng rng(42);
    for (int c = 0; c < 120; ++c) {
      std::size_t m = rng.integer(1, 64), n = rng.integer(1, 64), k = rng.integer(1, 64);
      unsigned p = unsigned(rng.integer(1, 8)), q = unsigned(rng.integer(1, 8));
      abq::CodeMat a = rng.code_matrix(m, k, p);
      abq::CodeMat b = rng.code_matrix(n, k, q);
      auto got = abq::gemm_arbitrary(abq::bitpack(a, p), abq::bitpack(b, q), abq::default_tile(p, q));
      std::int64_t pq[2] = {p, q};
      emit(idx("accept42", c) + "/pq", pq, {2});
      emit_mat(idx("accept42", c) + "/a", a);
      emit_mat(idx("accept42", c) + "/b", b);
      emit_mat(idx("accept42", c) + "/out", got);
    }
  }
  // acceptance.cpp:77-104 tiling transparency problem, seed 43 (256^3, A5 W3)
  {
    abq::Rng rng(43);
    abq::CodeMat a = rng.code_matrix(256, 256, 5);
    abq::CodeMat b = rng.code_matrix(256, 256, 3);
    emit_mat("tile43/a", a);
    emit_mat("tile43/b", b);
    emit_mat("tile43/out", abq::gemm_arbitrary(abq::bitpack(a, 5), abq::bitpack(b, 3), abq::default_tile(5, 3)));
  }
  // test_quantizer.cpp:33-74 asymmetric codes with alpha/beta/compensation, seed 7
  {
    abq::Rng rng(7);
    for (int trial = 0; trial < 50; ++trial) {
      std::size_t rows = rng.integer(1, 12), cols = rng.integer(1, 12);
      abq::Mat x = rng.gauss_matrix(rows, cols, 3.0);
      abq::QuantSpec spec;
      spec.bits = unsigned(rng.integer(1, 8));
      spec.scheme = abq::Scheme::Asymmetric;
      spec.granularity = trial % 2 ? abq::Granularity::PerToken : abq::Granularity::PerTensor;
      spec.alpha = rng.uniform(0.5, 1.0);
      spec.beta = rng.uniform(0.5, 1.0);
      abq::CompensationPair comp;
      for (std::size_t i = 0; i < rows; ++i) comp.a.push_back(rng.gauss());
      for (std::size_t j = 0; j < cols; ++j) comp.b.push_back(rng.gauss());
      abq::QuantizedTensor q = abq::quantize(x, spec, comp);
      std::string b = idx("quant7", trial);
      emit_mat(b + "/x", x);
      double ab[2] = {spec.alpha, spec.beta};
      emit(b + "/alpha_beta", ab, {2});
      std::int64_t meta[3] = {spec.bits, int(spec.scheme), int(spec.granularity)};
      emit(b + "/meta", meta, {3});
      emit_vec(b + "/comp_a", comp.a);
      emit_vec(b + "/comp_b", comp.b);
      emit_qt(b + "/q", q);
    }
  }
  // test_quantizer.cpp:76-92 round trip (asym / balanced, per-token), seed 11
  {
    abq::Rng rng(11);
    for (int trial = 0; trial < 30; ++trial) {
      abq::Mat x = rng.gauss_matrix(8, 40, 2.0);
      abq::QuantSpec spec;
      spec.scheme = trial % 2 ? abq::Scheme::Balanced : abq::Scheme::Asymmetric;
      spec.bits = unsigned(rng.integer(2, spec.scheme == abq::Scheme::Balanced ? 7 : 8));
      spec.granularity = abq::Granularity::PerToken;
      abq::QuantizedTensor q = abq::quantize(x, spec);
      std::string b = idx("quant11", trial);
      emit_mat(b + "/x", x);
      std::int64_t meta[3] = {spec.bits, int(spec.scheme), int(spec.granularity)};
      emit(b + "/meta", meta, {3});
      emit_qt(b + "/q", q);
    }
  }
  // test_quantizer.cpp:94-107 balanced 2-bit, seed 3
  {
    abq::Rng rng(3);
    abq::Mat x = rng.gauss_matrix(1, 4096);
    abq::QuantizedTensor q = abq::quantize_balanced(x, 2);
    emit_mat("balanced3/x", x);
    emit_qt("balanced3/q", q);
  }
  // test_quantizer.cpp:119-128 degenerate range
  {
    abq::Mat x(3, 4, 2.5);
    abq::QuantSpec spec;
    spec.bits = 4;
    spec.scheme = abq::Scheme::Asymmetric;
    abq::QuantizedTensor q = abq::quantize(x, spec);
    emit_mat("degenerate/x", x);
    emit_qt("degenerate/q", q);
  }
  std::fclose(out_file);
  return 0;
}
