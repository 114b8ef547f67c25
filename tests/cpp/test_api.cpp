// test_api.cpp -- the reference's hot-path test cases restated against the
// C++ drop-in mirror (include/abq/abq.hpp -> libabq_cuda.so on the GPU).
//
// Each CASE below follows one reference test (paths relative to
// /root/reference/proj), with the same abq::Rng seeds and draw order and the
// same independent in-test oracles (plain int64 loops), so a user switching
// their #include to this engine sees the same contract hold:
//   test_bitkernel.cpp:36-180, acceptance.cpp:29-104, test_quantizer.cpp:94-128,
//   test_tune.cpp:10-70.
// Prints one PASS/FAIL line per case; exit status = number of failures.
#include <cstdio>
#include <set>
#include <string>

#include <cuda_fp16.h>

#include "abq/abq.hpp"

using namespace abq;

static int failures = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("  check failed: %s (line %d)\n", #cond, __LINE__);   \
      ok = false;                                                         \
    }                                                                     \
  } while (0)

static void report(bool ok, const char* name) {
  std::printf("%s - %s\n", ok ? "PASS" : "FAIL", name);
  if (!ok) ++failures;
}

static IntMat naive_codes(const CodeMat& a, const CodeMat& bt) {
  IntMat out(a.rows, bt.rows, 0);
  for (std::size_t i = 0; i < a.rows; ++i)
    for (std::size_t j = 0; j < bt.rows; ++j) {
      std::int64_t acc = 0;
      for (std::size_t k = 0; k < a.cols; ++k) acc += std::int64_t(a(i, k)) * std::int64_t(bt(j, k));
      out(i, j) = acc;
    }
  return out;
}

static void case_bitpack() {
  bool ok = true;
  Rng rng(21);
  for (unsigned bits = 1; bits <= 8; ++bits) {
    CodeMat c = rng.code_matrix(5, 70, bits);
    BitPlaneMatrix m = bitpack(c, bits);
    CHECK(m.planes == bits);
    CHECK(unpack(m) == c);
  }
  CodeMat bad(2, 3, 0);
  bad(1, 2) = 4;
  try {
    bitpack(bad, 2);
    CHECK(false);
  } catch (const ValueError& e) {
    CHECK(std::string(e.what()).find("(1,2)") != std::string::npos);
  }
  report(ok, "bitpack round trips and rejects out-of-range codes (seed 21)");
}

static void case_bmma() {
  bool ok = true;
  Rng rng(22);
  CodeMat a = rng.code_matrix(4, 130, 3), b = rng.code_matrix(5, 130, 2);
  BitPlaneMatrix pa = bitpack(a, 3), pb = bitpack(b, 2);
  for (unsigned s = 0; s < 3; ++s)
    for (unsigned t = 0; t < 2; ++t) {
      auto got = bmma(pa, s, pb, t);
      for (std::size_t i = 0; i < 4; ++i)
        for (std::size_t j = 0; j < 5; ++j) {
          std::int64_t want = 0;
          for (std::size_t k = 0; k < 130; ++k) want += pa.bit(s, i, k) & pb.bit(t, j, k);
          CHECK(got(i, j) == want);
        }
    }
  report(ok, "bmma equals the bit-level triple loop (seed 22)");
}

static void case_gemm_oracle() {
  bool ok = true;
  Rng rng(23);
  for (int trial = 0; trial < 60; ++trial) {
    std::size_t m = rng.integer(1, 48), n = rng.integer(1, 48), k = rng.integer(1, 200);
    unsigned p = unsigned(rng.integer(1, 8)), q = unsigned(rng.integer(1, 8));
    CodeMat a = rng.code_matrix(m, k, p), b = rng.code_matrix(n, k, q);
    auto got = gemm_arbitrary(bitpack(a, p), bitpack(b, q), default_tile(p, q));
    IntMat want = naive_codes(a, b);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < n; ++j) CHECK(std::int64_t(got(i, j)) == want(i, j));
  }
  report(ok, "gemm_arbitrary equals the integer oracle, 60 cases (seed 23)");
}

static void case_naive_overflow_tiles() {
  bool ok = true;
  {
    Rng rng(24);
    CodeMat a = rng.code_matrix(9, 300, 5), b = rng.code_matrix(11, 300, 3);
    auto pa = bitpack(a, 5), pb = bitpack(b, 3);
    CHECK(gemm_naive(pa, pb) == gemm_arbitrary(pa, pb, default_tile(5, 3)));
  }
  {
    CHECK(fits_int32(8, 8, (std::size_t{1} << 15) - 1));
    CHECK(!fits_int32(8, 8, std::size_t{1} << 15));
    Rng rng(25);
    std::size_t k = std::size_t{1} << 15;
    CodeMat a = rng.code_matrix(1, k, 8), b = rng.code_matrix(1, k, 8);
    auto pa = bitpack(a, 8), pb = bitpack(b, 8);
    bool threw = false;
    try {
      gemm_arbitrary(pa, pb, default_tile(8, 8));
    } catch (const OverflowError&) {
      threw = true;
    }
    CHECK(threw);
    CHECK(gemm_arbitrary_wide(pa, pb, default_tile(8, 8))(0, 0) == naive_codes(a, b)(0, 0));
  }
  {
    Rng rng(26);
    CodeMat a = rng.code_matrix(33, 500, 3), b = rng.code_matrix(29, 500, 5);
    auto pa = bitpack(a, 3), pb = bitpack(b, 5);
    auto want = gemm_arbitrary(pa, pb, default_tile(3, 5));
    for (std::size_t bm : {8, 16, 64})
      for (std::size_t bk : {128, 256, 512}) CHECK(gemm_arbitrary(pa, pb, TileConfig{bm, 32, bk, 24, 40, 128}) == want);
  }
  {
    bool t1 = false, t2 = false;
    try {
      TileConfig{8, 8, 100, 8, 8, 128}.require_valid(1, 1);
    } catch (const ValueError&) {
      t1 = true;
    }
    try {
      TileConfig{512, 512, 128, 8, 8, 128}.require_valid(1, 1);
    } catch (const ValueError&) {
      t2 = true;
    }
    CHECK(t1 && t2);
  }
  report(ok, "naive == tiled, overflow boundary + wide, tile transparency (seeds 24-26)");
}

static void case_zero_point() {
  bool ok = true;
  Rng rng(27);
  for (int trial = 0; trial < 20; ++trial) {
    std::size_t m = rng.integer(1, 10), n = rng.integer(1, 10), k = rng.integer(1, 64);
    CodeMat a = rng.code_matrix(m, k, 4), b = rng.code_matrix(n, k, 4);
    std::vector<std::int32_t> za, zb;
    for (std::size_t i = 0; i < m; ++i) za.push_back(std::int32_t(rng.integer(0, 15)));
    for (std::size_t j = 0; j < n; ++j) zb.push_back(std::int32_t(rng.integer(0, 15)));
    auto acc = gemm_arbitrary(bitpack(a, 4), bitpack(b, 4), default_tile(4, 4));
    auto corrected = zero_point_correct(acc, code_rowsums(a), code_rowsums(b), za, zb, k);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < n; ++j) {
        std::int64_t want = 0;
        for (std::size_t kk = 0; kk < k; ++kk)
          want += (std::int64_t(a(i, kk)) - za[i]) * (std::int64_t(b(j, kk)) - zb[j]);
        CHECK(std::int64_t(corrected(i, j)) == want);
      }
  }
  report(ok, "zero-point correction equals the signed oracle (seed 27)");
}

static void case_quantized_linear_and_stats() {
  bool ok = true;
  {
    Rng rng(28);
    Mat x = rng.gauss_matrix(6, 64), w = rng.gauss_matrix(9, 64);
    QuantSpec sa;
    sa.bits = 5;
    sa.granularity = Granularity::PerToken;
    QuantSpec sw;
    sw.bits = 3;
    sw.granularity = Granularity::PerChannel;
    QuantizedTensor qa = quantize(x, sa), qw = quantize(w, sw);
    GemmStats stats;
    Mat got = quantized_linear(qa, qw, &stats);
    // dequantized-code product (test_bitkernel.cpp:164-165), restated in-test
    double worst = 0.0;
    for (std::size_t i = 0; i < 6; ++i)
      for (std::size_t j = 0; j < 9; ++j) {
        double s = 0.0;
        for (std::size_t k = 0; k < 64; ++k)
          s += ((double(qa.codes(i, k)) - qa.zero_points[i]) * qa.scales[i]) *
               ((double(qw.codes(j, k)) - qw.zero_points[j]) * qw.scales[j]);
        double d = got(i, j) - s;
        worst = std::max(worst, d < 0 ? -d : d);
      }
    CHECK(worst < 1e-9);
    CHECK(stats.plane_pair_products > 0 && stats.block_tiles > 0);
  }
  {
    Rng rng(29);
    CodeMat a = rng.code_matrix(70, 128, 2), b = rng.code_matrix(70, 128, 3);
    GemmStats stats;
    gemm_arbitrary(bitpack(a, 2), bitpack(b, 3), TileConfig{32, 32, 128, 32, 32, 128}, &stats);
    CHECK(stats.block_tiles == 9);
    CHECK(stats.plane_pair_products == 9 * 2 * 3);
  }
  report(ok, "quantized_linear vs dequantized product, GemmStats law (seeds 28, 29)");
}

static void case_acceptance_1000() {
  bool ok = true;
  Rng rng(42);
  for (int c = 0; ok && c < 1000; ++c) {
    std::size_t m = rng.integer(1, 64), n = rng.integer(1, 64), k = rng.integer(1, 64);
    unsigned p = unsigned(rng.integer(1, 8)), q = unsigned(rng.integer(1, 8));
    CodeMat a = rng.code_matrix(m, k, p), b = rng.code_matrix(n, k, q);
    auto got = gemm_arbitrary(bitpack(a, p), bitpack(b, q), default_tile(p, q));
    IntMat want = naive_codes(a, b);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = 0; j < n; ++j) CHECK(std::int64_t(got(i, j)) == want(i, j));
  }
  report(ok, "acceptance 1: 1000 random cases vs int64 oracle (seed 42)");
}

static void case_quantizer_and_padding() {
  bool ok = true;
  {
    Rng rng(3);
    Mat x = rng.gauss_matrix(1, 4096);
    QuantizedTensor q = quantize_balanced(x, 2);
    CHECK(q.spec.levels() == 5 && q.spec.planes() == 3);
    std::set<int> seen;
    for (auto c : q.codes.data) seen.insert(int(c) - q.zero_points[0]);
    CHECK((seen == std::set<int>{-2, -1, 0, 1, 2}));
    double amax = 0.0;
    for (double v : x.data) amax = std::max(amax, v < 0 ? -v : v);
    CHECK(q.scales[0] == amax / 2.0);
  }
  {
    Mat x(3, 4, 2.5);
    QuantSpec spec;
    spec.bits = 4;
    QuantizedTensor q = quantize(x, spec);
    CHECK(q.scales[0] == 1.0 && q.zero_points[0] == 0);
    for (auto c : q.codes.data) CHECK(c == 3);
  }
  CHECK(padding_redundancy(1, 1, 8) == 0.875);
  CHECK(padding_redundancy(1, 8, 8) == 0.0);
  report(ok, "balanced 2-bit level set, degenerate range, padding figures");
}

static void case_tune() {
  // test_tune.cpp:25-70 + the reference's own candidate list for (p=4, q=4, M=1)
  // (tests/golden/tune/candidates.json, written by the unmodified
  // enumerate_tile_candidates): 384 candidates, first/last as below
  bool ok = true;
  const auto c = enumerate_tile_candidates(4, 4, 1, 4096, 4096);
  CHECK(c.size() == 384);
  CHECK(c.front().BM == 2 && c.front().BN == 2 && c.front().BK == 128 && c.front().WM == 8 && c.front().WN == 8);
  CHECK(c.back().BM == 64 && c.back().BN == 64 && c.back().BK == 512 && c.back().WM == 64 && c.back().WN == 64);
  std::set<std::string> ids;
  for (const auto& t : c) {
    CHECK(t.valid(4, 4));
    ids.insert(t.describe());
  }
  CHECK(ids.size() == c.size());
  bool threw = false;
  try {
    enumerate_tile_candidates(0, 4, 1, 64, 64);
  } catch (const ValueError&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    autotune({}, BitPlaneMatrix(), BitPlaneMatrix());
  } catch (const ValueError&) {
    threw = true;
  }
  CHECK(threw);
  Rng rng(11);
  const CodeMat a = rng.code_matrix(24, 200, 3), b = rng.code_matrix(30, 200, 5);
  const auto pa = bitpack(a, 3), pb = bitpack(b, 5);
  const auto cands = enumerate_tile_candidates(3, 5, 24, 30, 200);
  const std::vector<TileConfig> tried(cands.begin(), cands.begin() + std::min<std::size_t>(4, cands.size()));
  const AutotuneResult r = autotune(tried, pa, pb, 3);
  CHECK(r.records.size() == tried.size());
  for (const auto& rec : r.records) CHECK(rec.median_us > 0.0 && rec.tops > 0.0 && rec.M == 24 && rec.N == 30);
  const auto got = gemm_arbitrary(pa, pb, r.best);
  const IntMat want = naive_codes(a, b);
  for (std::size_t i = 0; i < 24; ++i)
    for (std::size_t j = 0; j < 30; ++j) CHECK(std::int64_t(got(i, j)) == want(i, j));
  CHECK(BenchRecord::csv_header() == "config_id,BM,BN,BK,WM,WN,p,q,M,N,K,median_us,tops");
  report(ok, "tune: reference candidate list, validity, errors, verified autotune");
}

// SURVEY.md 8f-2 through the C++ drop-in: RMSNorm with the ReQuant fused in,
// consumed by the decode GEMV, equals the one-call linear on the producer's own
// fp16 output (both quantize the same y, quantizer.hpp:146-213), for several
// projections; one resident layout per regime (Layouts::Decode).
static void case_producer_qact() {
  bool ok = true;
  Rng rng(61);
  const std::size_t m = 2, k = 4096, n = 1536;
  std::vector<__half> xh(m * k), gh(k);
  for (auto& v : xh) v = __float2half(static_cast<float>(rng.gauss()));
  for (auto& v : gh) v = __float2half(static_cast<float>(rng.uniform(0.5, 1.5)));
  detail::DeviceBuffer<__half> x(xh), g(gh), y(m * k);
  QuantSpec aspec;
  aspec.bits = 4;
  aspec.granularity = Granularity::PerToken;
  device::QAct qa(m, k, aspec);
  device::rmsnorm_quant(x.get(), g.get(), 1e-6f, m, k, qa, y.get());
  for (int proj = 0; proj < 3; ++proj) {
    QuantSpec wspec;
    wspec.bits = 4;
    wspec.granularity = Granularity::PerChannel;
    const QuantizedTensor wt = quantize(rng.gauss_matrix(n, k, 0.02), wspec);
    const device::Weights wd(wt, proj == 2 ? device::Layouts::Decode : device::Layouts::All);
    const device::Linear lin(wd, aspec, m);
    detail::DeviceBuffer<double> y1(m * n), y2(m * n);
    lin(qa, y1.get(), ABQ_OUT_F64);
    lin(y.get(), ABQ_F16, m, y2.get(), ABQ_OUT_F64);
    std::vector<double> h1(m * n), h2(m * n);
    y1.to_host(h1.data());
    y2.to_host(h2.data());
    CHECK(h1 == h2);
    if (proj == 2) CHECK(wd.resident_bytes() == abq_weights_frag_bytes(4, n, k));
  }
  report(ok, "producer-fused ReQuant (rmsnorm_quant -> QAct -> Linear) == one-call linear on its output");
}

int main() {
  case_bitpack();
  case_bmma();
  case_gemm_oracle();
  case_naive_overflow_tiles();
  case_zero_point();
  case_quantized_linear_and_stats();
  case_acceptance_1000();
  case_quantizer_and_padding();
  case_tune();
  case_producer_qact();
  std::printf("%d failure(s)\n", failures);
  return failures;
}
