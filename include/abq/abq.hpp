// abq/abq.hpp -- C++ drop-in mirror of the reference operator API for the
// bit-plane quantized matmul hot path, backed by the sm_100a engine through
// the C-ABI in abq_cuda.h (libabq_cuda.so).
//
// Same namespace, type names, signatures, value semantics and exception
// classes as the reference headers (paths relative to /root/reference/proj):
//   core.hpp:13-70, 113-145   Error hierarchy, Matrix<T>, Mat/CodeMat/IntMat, Rng
//   quantizer.hpp:14-224      Scheme, Granularity, QuantSpec, CompensationPair,
//                             QuantizedTensor, quantize, quantize_balanced
//   bitplane.hpp:15-96        BitPlaneMatrix, bitpack, unpack, bmma
//   tune.hpp:51-192           enumerate_tile_candidates, BenchRecord, AutotuneResult,
//                             autotune (device engine timed with steady_clock, as the reference)
//   gemm.hpp:19-307           TileConfig, default_tile, GemmStats, fits_int32,
//                             engine_threads, gemm_arbitrary(_wide), gemm_naive,
//                             zero_point_correct, code_rowsums, quantized_linear
//   tune.hpp:17-23            padding_redundancy
// Host containers in, host containers out (the reference's contract): each
// call stages its operands in HBM, runs the kernels, and copies the result
// back.  Nothing numeric is computed on the host.  The device-resident API
// (abq::device::Weights / abq::device::Linear) keeps packed weights in HBM
// across calls for the serving path.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <utility>
#include <chrono>
#include <iterator>
#include <cstdint>
#include <set>
#include <tuple>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "abq_cuda.h"

namespace abq {

// ---- errors (core.hpp:13-36) ------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class ShapeError : public Error {
 public:
  explicit ShapeError(const std::string& m) : Error(m) {}
};
class ValueError : public Error {
 public:
  explicit ValueError(const std::string& m) : Error(m) {}
};
class OverflowError : public Error {
 public:
  explicit OverflowError(const std::string& m) : Error(m) {}
};
class IoError : public Error {
 public:
  explicit IoError(const std::string& m) : Error(m) {}
};

namespace detail {
inline void check(int status) {
  if (status == ABQ_OK) return;
  const std::string msg = abq_last_error();
  switch (status) {
    case ABQ_ERR_SHAPE: throw ShapeError(msg);
    case ABQ_ERR_VALUE: throw ValueError(msg);
    case ABQ_ERR_OVERFLOW: throw OverflowError(msg);
    case ABQ_ERR_IO: throw IoError(msg);
    default: throw Error(msg);
  }
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer used to stage host operands in HBM.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
  }
  DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) {
    if (n) cuda_check(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  explicit DeviceBuffer(const std::vector<T>& v) : DeviceBuffer(v.data(), v.size()) {}
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void to_host(T* host) const {
    if (n_) cuda_check(cudaMemcpy(host, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};
}  // namespace detail

// ---- core containers (core.hpp:39-70) ---------------------------------------
template <typename T>
struct Matrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<T> data;

  Matrix() = default;
  Matrix(std::size_t r, std::size_t c, T fill = T{}) : rows(r), cols(c), data(r * c, fill) {}
  T& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  const T& operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  std::size_t size() const { return rows * cols; }
  bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
  bool operator==(const Matrix& o) const { return same_shape(o) && data == o.data; }
  Matrix<T> transposed() const {  // core.hpp:55-62
    Matrix<T> out(cols, rows);
    for (std::size_t i = 0; i < rows; ++i)
      for (std::size_t j = 0; j < cols; ++j) out.data[j * rows + i] = data[i * cols + j];
    return out;
  }
};

using Mat = Matrix<double>;
using CodeMat = Matrix<std::uint8_t>;
using IntMat = Matrix<std::int64_t>;

// ---- FP64 host helpers of core.hpp:72-111 (test / calibration utilities, not
// the engine: the quantized product itself always runs on the device) --------
inline Mat matmul(const Mat& a, const Mat& b) {
  if (a.cols != b.rows) throw ShapeError("matmul: inner dimensions differ");
  Mat out(a.rows, b.cols, 0.0);
  for (std::size_t i = 0; i < a.rows; ++i)
    for (std::size_t k = 0; k < a.cols; ++k) {
      const double aik = a(i, k);
      double* row = out.data.data() + i * out.cols;
      const double* brow = b.data.data() + k * b.cols;
      for (std::size_t j = 0; j < b.cols; ++j) row[j] += aik * brow[j];
    }
  return out;
}
inline double max_abs_diff(const Mat& a, const Mat& b) {
  if (!a.same_shape(b)) throw ShapeError("max_abs_diff: shape mismatch");
  double m = 0.0;
  for (std::size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::abs(a.data[i] - b.data[i]));
  return m;
}
inline double frobenius(const Mat& a) {
  double s = 0.0;
  for (double v : a.data) s += v * v;
  return std::sqrt(s);
}
inline double rel_diff(const Mat& got, const Mat& want) {
  if (!got.same_shape(want)) throw ShapeError("rel_diff: shape mismatch");
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < got.data.size(); ++i) {
    const double d = got.data[i] - want.data[i];
    num += d * d;
    den += want.data[i] * want.data[i];
  }
  return den == 0.0 ? std::sqrt(num) : std::sqrt(num / den);
}
/// std::round: half away from zero (core.hpp:145)
inline double round_half_away(double v) { return std::round(v); }

/// Seeded generator with the reference's distributions (core.hpp:113-142), so
/// seeded test cases replay the reference's inputs draw for draw.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : gen_(seed) {}
  double gauss(double mean = 0.0, double stddev = 1.0) {
    return std::normal_distribution<double>(mean, stddev)(gen_);
  }
  double uniform(double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(gen_); }
  std::uint64_t integer(std::uint64_t lo, std::uint64_t hi) {
    return std::uniform_int_distribution<std::uint64_t>(lo, hi)(gen_);
  }
  Mat gauss_matrix(std::size_t r, std::size_t c, double stddev = 1.0) {
    Mat m(r, c);
    for (auto& v : m.data) v = gauss(0.0, stddev);
    return m;
  }
  CodeMat code_matrix(std::size_t r, std::size_t c, unsigned bits) {
    CodeMat m(r, c);
    for (auto& v : m.data) v = static_cast<std::uint8_t>(integer(0, (1u << bits) - 1));
    return m;
  }

 private:
  std::mt19937_64 gen_;
};

// ---- quantizer types (quantizer.hpp:14-107) ---------------------------------
enum class Scheme : std::uint8_t { Asymmetric = 0, Symmetric = 1, Balanced = 2 };
enum class Granularity : std::uint8_t { PerTensor = 0, PerChannel = 1, PerToken = 2 };

struct QuantSpec {
  unsigned bits = 8;
  Scheme scheme = Scheme::Asymmetric;
  Granularity granularity = Granularity::PerTensor;
  double alpha = 1.0;
  double beta = 1.0;
  std::vector<double> balance_scale;

  bool passthrough() const { return bits >= 16; }
  abq_quant_spec c_spec() const {
    return abq_quant_spec{bits, int(scheme), int(granularity), alpha, beta};
  }
  unsigned levels() const {
    abq_quant_spec s = c_spec();
    return abq_spec_levels(&s);
  }
  unsigned planes() const {
    abq_quant_spec s = c_spec();
    return abq_spec_planes(&s);
  }
  void validate() const {
    if (bits < 1 || (bits > 8 && !passthrough()))
      throw ValueError("QuantSpec: bits must be in [1,8] (or >=16 for passthrough)");
    if (scheme == Scheme::Balanced && bits > 7 && !passthrough())
      throw ValueError("QuantSpec: balanced codes reach 2^bits and must fit one byte, so bits <= 7");
    if (!(alpha > 0.0 && alpha <= 1.0)) throw ValueError("QuantSpec: alpha must be in (0,1]");
    if (!(beta > 0.0 && beta <= 1.0)) throw ValueError("QuantSpec: beta must be in (0,1]");
    for (double s : balance_scale)
      if (!(s > 0.0)) throw ValueError("QuantSpec: balance_scale entries must be positive");
  }
};

struct CompensationPair {
  std::vector<double> a;
  std::vector<double> b;
};

struct QuantizedTensor {
  CodeMat codes;
  std::vector<double> scales;
  std::vector<std::int32_t> zero_points;
  QuantSpec spec;

  std::size_t rows() const { return codes.rows; }
  std::size_t cols() const { return codes.cols; }
  std::size_t axis_count() const { return scales.size(); }
  std::size_t axis_of(std::size_t i, std::size_t) const {
    return spec.granularity == Granularity::PerTensor ? 0 : i;
  }
  /// quantizer.hpp:95-107: spec valid, every code < levels, one scale / zero
  /// point per axis group
  void validate() const {
    spec.validate();
    const unsigned max_code = spec.levels() - 1;
    for (std::size_t i = 0; i < codes.data.size(); ++i)
      if (codes.data[i] > max_code)
        throw ValueError("QuantizedTensor: code out of range at flat index " + std::to_string(i));
    const std::size_t want = spec.granularity == Granularity::PerTensor ? 1 : codes.rows;
    if (scales.size() != want || zero_points.size() != want)
      throw ValueError("QuantizedTensor: scale/zero_point count does not match granularity");
  }
};

// ---- bit planes (bitplane.hpp:15-44) ---------------------------------------
struct BitPlaneMatrix {
  unsigned planes = 0;
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::size_t words_per_row = 0;
  std::vector<std::uint64_t> data;  // [plane][row][word]

  BitPlaneMatrix() = default;
  BitPlaneMatrix(unsigned p, std::size_t r, std::size_t c)
      : planes(p), rows(r), cols(c), words_per_row((c + 63) / 64),
        data(std::size_t(p) * r * ((c + 63) / 64), 0) {}
  const std::uint64_t* row(unsigned plane, std::size_t r) const {
    return data.data() + (std::size_t(plane) * rows + r) * words_per_row;
  }
  bool bit(unsigned plane, std::size_t r, std::size_t c) const {
    return (row(plane, r)[c / 64] >> (c % 64)) & 1u;
  }
  bool operator==(const BitPlaneMatrix& o) const {
    return planes == o.planes && rows == o.rows && cols == o.cols && data == o.data;
  }
};

// ---- engine types (gemm.hpp:19-84) ------------------------------------------
struct TileConfig {
  std::size_t BM = 64, BN = 64, BK = 512;
  std::size_t WM = 64, WN = 64, WK = 128;
  static constexpr std::size_t mma_m = 8, mma_n = 8, mma_k = 128;

  abq_tile_config c_tile() const { return abq_tile_config{BM, BN, BK, WM, WN, WK}; }
  bool valid(unsigned p, unsigned q) const {
    abq_tile_config t = c_tile();
    return abq_tile_valid(&t, p, q) != 0;
  }
  std::string describe() const {
    std::ostringstream os;
    os << "BM" << BM << "_BN" << BN << "_BK" << BK << "_WM" << WM << "_WN" << WN;
    return os.str();
  }
  void require_valid(unsigned p, unsigned q) const {
    if (!valid(p, q)) {
      std::ostringstream os;
      os << "TileConfig invalid for p=" << p << " q=" << q << ": BM=" << BM << " BN=" << BN
         << " BK=" << BK << " WM=" << WM << " WN=" << WN << " WK=" << WK;
      throw ValueError(os.str());
    }
  }
};

inline TileConfig default_tile(unsigned p, unsigned q) {
  abq_tile_config t = abq_default_tile(p, q);
  return TileConfig{t.BM, t.BN, t.BK, t.WM, t.WN, t.WK};
}

struct GemmStats {
  std::uint64_t block_tiles = 0;
  std::uint64_t plane_pair_products = 0;
};

inline bool fits_int32(unsigned p, unsigned q, std::size_t k) { return abq_fits_int32(p, q, k) != 0; }

/// Process-global knob kept for API parity (gemm.hpp:81-84); the GPU engine's
/// results never depend on it.
inline unsigned& engine_threads() {
  static unsigned n = 0;
  return n;
}

inline double padding_redundancy(std::size_t m, unsigned p, std::size_t mma_m) {
  double out = 0.0;
  detail::check(abq_padding_redundancy(m, p, mma_m, &out));
  return out;
}

// ---- L2 entry points ---------------------------------------------------------
inline BitPlaneMatrix bitpack(const CodeMat& codes, unsigned bits) {
  if (bits < 1 || bits > 8) throw ValueError("bitpack: plane count must be in [1,8]");
  BitPlaneMatrix out(bits, codes.rows, codes.cols);
  detail::DeviceBuffer<std::uint8_t> dc(codes.data);
  detail::DeviceBuffer<std::uint64_t> dp(out.data.size());
  detail::check(abq_bitpack(dc.get(), codes.rows, codes.cols, bits, dp.get(), nullptr));
  dp.to_host(out.data.data());
  return out;
}

inline CodeMat unpack(const BitPlaneMatrix& m) {
  CodeMat codes(m.rows, m.cols);
  detail::DeviceBuffer<std::uint64_t> dp(m.data);
  detail::DeviceBuffer<std::uint8_t> dc(codes.data.size());
  detail::check(abq_unpack(dp.get(), m.planes, m.rows, m.cols, dc.get(), nullptr));
  dc.to_host(codes.data.data());
  return codes;
}

inline Matrix<std::int32_t> bmma(const BitPlaneMatrix& a, unsigned a_plane, const BitPlaneMatrix& bt,
                                 unsigned b_plane) {
  if (a.cols != bt.cols) throw ShapeError("bmma: shared K dimension differs");
  Matrix<std::int32_t> out(a.rows, bt.rows, 0);
  detail::DeviceBuffer<std::uint64_t> da(a.data), db(bt.data);
  detail::DeviceBuffer<std::int32_t> dout(out.data.size());
  detail::check(abq_bmma(da.get(), a.planes, a.rows, a_plane, db.get(), bt.planes, bt.rows, b_plane,
                         a.cols, dout.get(), nullptr));
  dout.to_host(out.data.data());
  return out;
}

// ---- L3 entry points ---------------------------------------------------------
inline Matrix<std::int32_t> gemm_arbitrary(const BitPlaneMatrix& a, const BitPlaneMatrix& bt,
                                           const TileConfig& tile, GemmStats* stats = nullptr) {
  Matrix<std::int32_t> out(a.rows, bt.rows, 0);
  detail::DeviceBuffer<std::uint64_t> da(a.data), db(bt.data);
  detail::DeviceBuffer<std::int32_t> dout(out.data.size());
  abq_tile_config t = tile.c_tile();
  abq_gemm_stats st{stats ? stats->block_tiles : 0, stats ? stats->plane_pair_products : 0};
  detail::check(abq_gemm_arbitrary(da.get(), a.planes, a.rows, a.cols, db.get(), bt.planes, bt.rows,
                                   bt.cols, &t, dout.get(), &st, nullptr));
  dout.to_host(out.data.data());
  if (stats) *stats = GemmStats{st.block_tiles, st.plane_pair_products};
  return out;
}

inline Matrix<std::int64_t> gemm_arbitrary_wide(const BitPlaneMatrix& a, const BitPlaneMatrix& bt,
                                                const TileConfig& tile, GemmStats* stats = nullptr) {
  Matrix<std::int64_t> out(a.rows, bt.rows, 0);
  detail::DeviceBuffer<std::uint64_t> da(a.data), db(bt.data);
  detail::DeviceBuffer<std::int64_t> dout(out.data.size());
  abq_tile_config t = tile.c_tile();
  abq_gemm_stats st{stats ? stats->block_tiles : 0, stats ? stats->plane_pair_products : 0};
  detail::check(abq_gemm_arbitrary_wide(da.get(), a.planes, a.rows, a.cols, db.get(), bt.planes,
                                        bt.rows, bt.cols, &t, dout.get(), &st, nullptr));
  dout.to_host(out.data.data());
  if (stats) *stats = GemmStats{st.block_tiles, st.plane_pair_products};
  return out;
}

inline Matrix<std::int32_t> gemm_naive(const BitPlaneMatrix& a, const BitPlaneMatrix& bt) {
  Matrix<std::int32_t> out(a.rows, bt.rows, 0);
  detail::DeviceBuffer<std::uint64_t> da(a.data), db(bt.data);
  detail::DeviceBuffer<std::int32_t> dout(out.data.size());
  detail::check(abq_gemm_naive(da.get(), a.planes, a.rows, a.cols, db.get(), bt.planes, bt.rows,
                               bt.cols, dout.get(), nullptr));
  dout.to_host(out.data.data());
  return out;
}

// ---- tuning (tune.hpp:51-192) --------------------------------------------------
namespace detail {
/// padded rows summed over the BM-row blocks covering m rows (tune.hpp:35-44)
inline std::size_t total_row_padding(std::size_t m, unsigned p, std::size_t bm, std::size_t mma_m) {
  std::size_t total = 0;
  for (std::size_t start = 0; start < m; start += bm) {
    const std::size_t rows = p * std::min(bm, m - start);
    total += (rows + mma_m - 1) / mma_m * mma_m - rows;
  }
  return total;
}
}  // namespace detail

/// enumerate_tile_candidates  tune.hpp:51-92: warp layouts {1x1,1x2,1x4,2x2,2x4,4x4}
/// x inner tiles {8..64}^2 x BK {128..512}; block tile = ceil(layout x inner / bits);
/// valid + first occurrence only; then the block heights with the least row padding.
inline std::vector<TileConfig> enumerate_tile_candidates(unsigned p, unsigned q, std::size_t m, std::size_t,
                                                         std::size_t) {
  if (p < 1 || p > 8 || q < 1 || q > 8) throw ValueError("enumerate_tile_candidates: p,q must be in [1,8]");
  constexpr unsigned layouts[6][2] = {{1, 1}, {1, 2}, {1, 4}, {2, 2}, {2, 4}, {4, 4}};
  constexpr std::size_t inner[4] = {8, 16, 32, 64}, depth[4] = {128, 256, 384, 512};
  std::set<std::tuple<std::size_t, std::size_t, std::size_t, std::size_t, std::size_t>> seen;
  std::vector<TileConfig> all;
  for (const auto& l : layouts)
    for (std::size_t wm : inner)
      for (std::size_t wn : inner)
        for (std::size_t bk : depth) {
          TileConfig t{(l[0] * wm + p - 1) / p, (l[1] * wn + q - 1) / q, bk, wm, wn, TileConfig::mma_k};
          if (t.valid(p, q) && seen.emplace(t.BM, t.BN, t.BK, t.WM, t.WN).second) all.push_back(t);
        }
  std::size_t least = ~std::size_t(0);
  for (const auto& t : all) least = std::min(least, detail::total_row_padding(m, p, t.BM, TileConfig::mma_m));
  std::vector<TileConfig> out;
  std::copy_if(all.begin(), all.end(), std::back_inserter(out), [&](const TileConfig& t) {
    return detail::total_row_padding(m, p, t.BM, TileConfig::mma_m) == least;
  });
  if (out.empty()) out.push_back(default_tile(p, q));
  return out;
}

/// BenchRecord  tune.hpp:94-105
struct BenchRecord {
  std::string config_id;
  std::size_t BM = 0, BN = 0, BK = 0, WM = 0, WN = 0;
  unsigned p = 0, q = 0;
  std::size_t M = 0, N = 0, K = 0;
  double median_us = 0.0;
  double tops = 0.0;
  static std::string csv_header() { return "config_id,BM,BN,BK,WM,WN,p,q,M,N,K,median_us,tops"; }
};

namespace detail {
/// median  tune.hpp:108-111
inline double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
}
/// tops_of  tune.hpp:129-131
inline double tops_of(std::size_t m, std::size_t n, std::size_t k, double us) {
  return 2.0 * double(m) * double(n) * double(k) / (us * 1e6);
}
/// time_median_us  tune.hpp:114-127 (one discarded warm-up, steady_clock
/// around each synchronous call, median)
template <typename Fn>
inline double time_median_us(Fn&& fn, unsigned trials) {
  fn();
  std::vector<double> us;
  for (unsigned i = 0; i < trials; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    us.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
  return median(std::move(us));
}
}  // namespace detail

struct AutotuneResult {
  TileConfig best;
  std::vector<BenchRecord> records;
};

/// autotune  tune.hpp:141-192: every candidate is timed through the engine's
/// gemm_arbitrary (_wide past the int32 bound) and must reproduce the first
/// candidate's result exactly (else abq::Error); the fastest wins.
inline AutotuneResult autotune(const std::vector<TileConfig>& candidates, const BitPlaneMatrix& a,
                               const BitPlaneMatrix& bt, unsigned trials = 3) {
  if (candidates.empty()) throw ValueError("autotune: no candidates");
  if (trials < 3) throw ValueError("autotune: need at least 3 trials");
  const bool wide = !fits_int32(a.planes, bt.planes, a.cols);
  AutotuneResult res;
  Matrix<std::int64_t> first;
  std::size_t best = 0;
  for (std::size_t i = 0; i < candidates.size(); ++i) {
    const TileConfig& t = candidates[i];
    t.require_valid(a.planes, bt.planes);
    Matrix<std::int64_t> got;
    const double us = detail::time_median_us(
        [&] {
          if (wide) {
            got = gemm_arbitrary_wide(a, bt, t);
          } else {
            const Matrix<std::int32_t> r = gemm_arbitrary(a, bt, t);
            got = Matrix<std::int64_t>(r.rows, r.cols);
            std::copy(r.data.begin(), r.data.end(), got.data.begin());
          }
        },
        trials);
    if (i == 0) first = got;
    else if (!(got == first)) throw Error("autotune: config " + t.describe() + " disagrees with the reference result");
    BenchRecord r;
    r.config_id = t.describe();
    r.BM = t.BM, r.BN = t.BN, r.BK = t.BK, r.WM = t.WM, r.WN = t.WN;
    r.p = a.planes, r.q = bt.planes, r.M = a.rows, r.N = bt.rows, r.K = a.cols;
    r.median_us = us;
    r.tops = detail::tops_of(r.M, r.N, r.K, us);
    if (!res.records.empty() && us < res.records[best].median_us) best = res.records.size();
    res.records.push_back(r);
  }
  res.best = candidates[best];
  return res;
}

template <typename Acc>
inline Matrix<Acc> zero_point_correct(const Matrix<Acc>& acc, const std::vector<std::int64_t>& rowsum_a,
                                      const std::vector<std::int64_t>& colsum_b,
                                      const std::vector<std::int32_t>& z_a,
                                      const std::vector<std::int32_t>& z_b, std::size_t k) {
  static_assert(sizeof(Acc) == 4 || sizeof(Acc) == 8, "int32 or int64 accumulators");
  if (rowsum_a.size() != acc.rows || z_a.size() != acc.rows)
    throw ShapeError("zero_point_correct: row-side vectors do not match");
  if (colsum_b.size() != acc.cols || z_b.size() != acc.cols)
    throw ShapeError("zero_point_correct: col-side vectors do not match");
  Matrix<Acc> out(acc.rows, acc.cols);
  detail::DeviceBuffer<Acc> dacc(acc.data), dout(out.data.size());
  detail::DeviceBuffer<std::int64_t> dra(rowsum_a), dcb(colsum_b);
  detail::DeviceBuffer<std::int32_t> dza(z_a), dzb(z_b);
  if constexpr (sizeof(Acc) == 4)
    detail::check(abq_zero_point_correct_i32(reinterpret_cast<const std::int32_t*>(dacc.get()),
                                             acc.rows, acc.cols, dra.get(), dcb.get(), dza.get(),
                                             dzb.get(), k, reinterpret_cast<std::int32_t*>(dout.get()),
                                             nullptr));
  else
    detail::check(abq_zero_point_correct_i64(reinterpret_cast<const std::int64_t*>(dacc.get()),
                                             acc.rows, acc.cols, dra.get(), dcb.get(), dza.get(),
                                             dzb.get(), k, reinterpret_cast<std::int64_t*>(dout.get()),
                                             nullptr));
  dout.to_host(out.data.data());
  return out;
}

inline std::vector<std::int64_t> code_rowsums(const CodeMat& codes) {
  std::vector<std::int64_t> sums(codes.rows, 0);
  detail::DeviceBuffer<std::uint8_t> dc(codes.data);
  detail::DeviceBuffer<std::int64_t> ds(sums.size());
  detail::check(abq_code_rowsums(dc.get(), codes.rows, codes.cols, ds.get(), nullptr));
  ds.to_host(sums.data());
  return sums;
}

// ---- L1: quantize (quantizer.hpp:146-224) ------------------------------------
inline QuantizedTensor quantize(const Mat& x, const QuantSpec& spec,
                                const std::optional<CompensationPair>& comp = std::nullopt) {
  spec.validate();
  if (spec.passthrough()) throw ValueError("quantize: passthrough spec cannot be materialized");
  QuantizedTensor q;
  q.spec = spec;
  q.codes = CodeMat(x.rows, x.cols);
  const std::size_t groups = spec.granularity == Granularity::PerTensor ? 1 : x.rows;
  q.scales.resize(groups);
  q.zero_points.resize(groups);
  detail::DeviceBuffer<double> dx(x.data);
  detail::DeviceBuffer<double> da, db;
  if (comp) {
    if (comp->a.size() != x.rows || comp->b.size() != x.cols)
      throw ShapeError("quantize: compensation pair does not match matrix shape");
    da = detail::DeviceBuffer<double>(comp->a);
    db = detail::DeviceBuffer<double>(comp->b);
  }
  detail::DeviceBuffer<std::uint8_t> dc(q.codes.data.size());
  detail::DeviceBuffer<double> ds(groups);
  detail::DeviceBuffer<std::int32_t> dz(groups);
  abq_quant_spec cs = spec.c_spec();
  detail::check(abq_quantize(dx.get(), ABQ_F64, x.rows, x.cols, &cs, comp ? da.get() : nullptr,
                             comp ? db.get() : nullptr, dc.get(), ds.get(), dz.get(), nullptr));
  dc.to_host(q.codes.data.data());
  ds.to_host(q.scales.data());
  dz.to_host(q.zero_points.data());
  return q;
}

/// apply_balance  quantizer.hpp:228-241: (W diag(s), diag(s)^-1 X), the
/// offline smoothing rescale (host FP64, like the reference; not the engine)
inline std::pair<Mat, Mat> apply_balance(const Mat& w, const Mat& x, const std::vector<double>& s) {
  if (w.cols != s.size() || x.rows != s.size())
    throw ShapeError("apply_balance: s length must equal the shared inner dimension");
  for (std::size_t k = 0; k < s.size(); ++k)
    if (!(s[k] > 0.0)) throw ValueError("apply_balance: s[" + std::to_string(k) + "] is not positive");
  Mat ws = w, xs = x;
  for (std::size_t i = 0; i < w.rows; ++i)
    for (std::size_t k = 0; k < w.cols; ++k) ws(i, k) *= s[k];
  for (std::size_t k = 0; k < x.rows; ++k)
    for (std::size_t j = 0; j < x.cols; ++j) xs(k, j) /= s[k];
  return {std::move(ws), std::move(xs)};
}

/// dequantize  quantizer.hpp:243-254: (code - z) * step, on the device
inline Mat dequantize(const QuantizedTensor& q) {
  q.validate();
  Mat out(q.rows(), q.cols());
  detail::DeviceBuffer<std::uint8_t> dc(q.codes.data);
  detail::DeviceBuffer<double> ds(q.scales), dout(out.data.size());
  detail::DeviceBuffer<std::int32_t> dz(q.zero_points);
  detail::check(abq_dequantize(dc.get(), q.rows(), q.cols(), ds.get(), dz.get(),
                               q.spec.granularity == Granularity::PerTensor ? 1 : 0, dout.get(), nullptr));
  dout.to_host(out.data.data());
  return out;
}

inline QuantizedTensor quantize_balanced(const Mat& x, unsigned bits,
                                         Granularity granularity = Granularity::PerTensor) {
  QuantSpec spec;
  spec.bits = bits;
  spec.scheme = Scheme::Balanced;
  spec.granularity = granularity;
  return quantize(x, spec);
}

// ---- engine path linear (gemm.hpp:266-307) ------------------------------------
inline Mat quantized_linear(const QuantizedTensor& act, const QuantizedTensor& wt,
                            GemmStats* stats = nullptr) {
  if (act.cols() != wt.cols()) throw ShapeError("quantized_linear: inner dimensions differ");
  const std::size_t k = act.cols();
  const unsigned p = act.spec.planes(), q = wt.spec.planes();
  const std::size_t m = act.rows(), n = wt.rows();
  detail::DeviceBuffer<std::uint8_t> dac(act.codes.data), dwc(wt.codes.data);
  detail::DeviceBuffer<std::uint64_t> dap(std::size_t(p) * m * ((k + 63) / 64));
  detail::DeviceBuffer<std::uint64_t> dwp(std::size_t(q) * n * ((k + 63) / 64));
  detail::check(abq_bitpack(dac.get(), m, k, p, dap.get(), nullptr));
  detail::check(abq_bitpack(dwc.get(), n, k, q, dwp.get(), nullptr));
  detail::DeviceBuffer<std::int64_t> dra(m), dcb(n);
  detail::check(abq_code_rowsums(dac.get(), m, k, dra.get(), nullptr));
  detail::check(abq_plane_rowsums(dwp.get(), q, n, k, dcb.get(), nullptr));
  detail::DeviceBuffer<double> dsa(act.scales), dsb(wt.scales);
  detail::DeviceBuffer<std::int32_t> dza(act.zero_points), dzb(wt.zero_points);
  abq_act a{dap.get(), p, m, k, dsa.get(), dza.get(), dra.get(),
            act.spec.granularity == Granularity::PerTensor};
  // engine re-layout of the planes: fragment-major for the tensor-pipe decode
  // GEMV (m <= 8), tc planes for the tcgen05 prefill GEMM (m >= 9)
  const bool decode = m <= 8;
  detail::DeviceBuffer<std::uint32_t> dlay(decode ? abq_weights_frag_bytes(q, n, k) / 4
                                                  : abq_weights_tc_bytes(q, n, k) / 4);
  if (decode)
    detail::check(abq_weights_prepack(dwp.get(), q, n, k, dlay.get(), nullptr));
  else
    detail::check(abq_weights_prepack_tc(dwp.get(), q, n, k, dlay.get(), nullptr));
  abq_weights w{dwp.get(), q, n, k, dsb.get(), dzb.get(), dcb.get(),
                wt.spec.granularity == Granularity::PerTensor, decode ? dlay.get() : nullptr,
                decode ? nullptr : dlay.get(), nullptr};
  Mat out(m, n);
  detail::DeviceBuffer<double> dy(out.data.size());
  detail::check(abq_linear_planes(&a, &w, dy.get(), ABQ_OUT_F64, nullptr));
  dy.to_host(out.data.data());
  if (stats) {
    const TileConfig t = default_tile(p, q);
    const std::uint64_t tiles = std::uint64_t((m + t.BM - 1) / t.BM) * ((n + t.BN - 1) / t.BN);
    stats->block_tiles += tiles;
    stats->plane_pair_products += tiles * p * q;
  }
  return out;
}

// ---- device-resident serving API (additions, SURVEY.md 8b "Ownership") -------
namespace device {

/// Which packed layouts stay resident in HBM: All = ABQP planes + decode
/// (frag) + prefill (tc) layouts (every entry point, incl. the int64 path);
/// Decode / Prefill / Both keep one layout per serving regime and drop the
/// planes after packing (Decode serves m <= 8, Prefill any m).
enum class Layouts { All, Decode, Prefill, Both };

/// Weights packed once and kept in HBM: engine layouts + per-channel metadata.
class Weights {
 public:
  explicit Weights(const QuantizedTensor& wt, Layouts layouts = Layouts::All)
      : q_(wt.spec.planes()), n_(wt.rows()), k_(wt.cols()),
        per_tensor_(wt.spec.granularity == Granularity::PerTensor),
        planes_(std::size_t(q_) * n_ * ((k_ + 63) / 64)), scales_(wt.scales),
        zps_(wt.zero_points), colsums_(n_),
        frag_(layouts == Layouts::Prefill ? 0 : abq_weights_frag_bytes(q_, n_, k_) / 4),
        tc_(layouts == Layouts::Decode ? 0 : abq_weights_tc_bytes(q_, n_, k_) / 4) {
    detail::DeviceBuffer<std::uint8_t> dc(wt.codes.data);
    detail::check(abq_bitpack(dc.get(), n_, k_, q_, planes_.get(), nullptr));
    detail::check(abq_plane_rowsums(planes_.get(), q_, n_, k_, colsums_.get(), nullptr));
    if (frag_.size()) detail::check(abq_weights_prepack(planes_.get(), q_, n_, k_, frag_.get(), nullptr));
    if (tc_.size()) detail::check(abq_weights_prepack_tc(planes_.get(), q_, n_, k_, tc_.get(), nullptr));
    if (layouts != Layouts::All) {
      detail::cuda_check(cudaDeviceSynchronize(), "Weights: pack");
      planes_ = detail::DeviceBuffer<std::uint64_t>();
    }
  }
  abq_weights view() const {
    return abq_weights{planes_.get(), q_, n_, k_, scales_.get(), zps_.get(), colsums_.get(),
                       per_tensor_ ? 1 : 0, frag_.size() ? frag_.get() : nullptr, tc_.size() ? tc_.get() : nullptr,
                       nullptr};
  }
  std::size_t resident_bytes() const {
    return planes_.size() * 8 + frag_.size() * 4 + tc_.size() * 4;
  }
  std::size_t n() const { return n_; }
  std::size_t k() const { return k_; }

 private:
  unsigned q_;
  std::size_t n_, k_;
  bool per_tensor_;
  detail::DeviceBuffer<std::uint64_t> planes_;
  detail::DeviceBuffer<double> scales_;
  detail::DeviceBuffer<std::int32_t> zps_;
  detail::DeviceBuffer<std::int64_t> colsums_;
  detail::DeviceBuffer<std::uint32_t> frag_;
  detail::DeviceBuffer<std::uint32_t> tc_;
};

/// Per-token quantized decode activations made by a producer op with the
/// ReQuant fused in (rmsnorm_quant / silu_mul_quant below), in
/// the decode GEMV's code layout; one QAct feeds every projection reading it.
class QAct {
 public:
  QAct(std::size_t m, std::size_t k, const QuantSpec& spec)
      : m_(m), k_(k), spec_(spec), codes_(abq_qact_codes_bytes(m, k) / 4), scales_(m), zps_(m), rows_(m) {
    spec.validate();
  }
  abq_qact view() const {
    return abq_qact{codes_.get(), scales_.get(), zps_.get(), rows_.get(), m_, k_, spec_.bits};
  }
  const QuantSpec& spec() const { return spec_; }
  std::size_t m() const { return m_; }
  std::size_t k() const { return k_; }
  /// per-token s_a / z_a / code row sums, copied to the host
  std::vector<double> scales() const {
    std::vector<double> v(m_);
    scales_.to_host(v.data());
    return v;
  }
  std::vector<std::int32_t> zero_points() const {
    std::vector<std::int32_t> v(m_);
    zps_.to_host(v.data());
    return v;
  }

 private:
  std::size_t m_, k_;
  QuantSpec spec_;
  detail::DeviceBuffer<std::uint32_t> codes_;
  detail::DeviceBuffer<double> scales_;
  detail::DeviceBuffer<std::int32_t> zps_;
  detail::DeviceBuffer<std::int64_t> rows_;
};

/// LLaMA RMSNorm y = gain * fp16(x * rsqrt(mean(x^2) + eps)) (device fp16
/// [m][k], gain [k]; y_out may be null) with the per-token ReQuant of y fused
/// in (toyblock.hpp:257 -> quantizer.hpp:146-213).
inline void rmsnorm_quant(const void* x, const void* gain, float eps, std::size_t m, std::size_t k, QAct& out,
                          void* y_out = nullptr, cudaStream_t stream = nullptr) {
  const abq_quant_spec s = out.spec().c_spec();
  const abq_qact v = out.view();
  detail::check(abq_rmsnorm_quant(x, gain, eps, m, k, &s, y_out, &v, nullptr, stream));
}
/// y = fp16(fp16(silu(gate)) * up) with the per-token ReQuant of y fused in.
inline void silu_mul_quant(const void* gate, const void* up, std::size_t m, std::size_t k, QAct& out,
                           void* y_out = nullptr, cudaStream_t stream = nullptr) {
  const abq_quant_spec s = out.spec().c_spec();
  const abq_qact v = out.view();
  detail::check(abq_silu_mul_quant(gate, up, m, k, &s, y_out, &v, nullptr, stream));
}

/// ReQuant + BitPacking + plane GEMV/GEMM + fused epilogue on device pointers.
class Linear {
 public:
  Linear(const Weights& w, const QuantSpec& act_spec, std::size_t max_m)
      : w_(w.view()), spec_(act_spec.c_spec()), max_m_(max_m),
        ws_bytes_(abq_linear_workspace_bytes(max_m, w.n(), w.k(), act_spec.planes())), ws_(ws_bytes_) {
    act_spec.validate();
    // the engine expects a zero-filled workspace and leaves it zeroed
    detail::cuda_check(cudaMemset(ws_.get(), 0, ws_bytes_), "cudaMemset workspace");
  }
  /// x: device [m][k] (x_dtype ABQ_F16/F32/F64); y: device [m][n] of out_kind.
  void operator()(const void* x, int x_dtype, std::size_t m, void* y, int out_kind,
                  cudaStream_t stream = nullptr, std::int64_t* err_index = nullptr) const {
    if (m > max_m_) throw ValueError("device::Linear: m exceeds max_m");
    detail::check(abq_linear(x, x_dtype, m, w_.k, &spec_, &w_, y, out_kind, ws_.get(), ws_bytes_,
                             err_index, stream));
  }
  /// decode linear on producer-quantized activations (one GEMV launch)
  void operator()(const QAct& act, void* y, int out_kind, cudaStream_t stream = nullptr) const {
    if (act.m() > max_m_) throw ValueError("device::Linear: m exceeds max_m");
    const abq_qact v = act.view();
    detail::check(abq_linear_qact(&v, &w_, y, out_kind, stream));
  }
  /// successor-layer hint (abq_weights.next): the linear run next on the same
  /// stream; this layer's decode GEMV prefetches the start of its weights into
  /// L2 in its tail.  `next` must outlive this Linear (nullptr clears).
  void prefetch_next(const Linear* next) { w_.next = next ? &next->w_ : nullptr; }

 private:
  abq_weights w_;
  abq_quant_spec spec_;
  std::size_t max_m_, ws_bytes_;
  detail::DeviceBuffer<std::uint8_t> ws_;
};

}  // namespace device
}  // namespace abq
