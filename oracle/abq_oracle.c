/*
 * abq_oracle.c -- CPU restatement of the ABQ-LLM reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the *checker*: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  The product path (paper_2408_08554_b200/csrc, include/abq)
 * never links, loads or calls it; it fails loudly when the CUDA library is
 * missing instead.
 *
 * Parity status: PINNED.  Every function below is checked against golden
 * vectors produced by the reference headers themselves (oracle/_ref, built
 * from /root/reference/proj/include by oracle/Makefile, fixtures committed
 * under tests/golden/ by tests/golden/make_golden.py) and, when oracle/_ref is
 * present, against the reference on fresh random inputs
 * (tests/test_oracle.py).
 *
 * Conventions follow the reference exactly (cited file:line, paths relative
 * to /root/reference/proj):
 *   - operand a = activation codes (M x K, p planes), bt = weight codes stored
 *     transposed (N x K, q planes)            gemm.hpp:181-185, abqtool.cpp:124-129
 *   - planes [plane][row][word], u64 words, LSB-first, tail bits zero
 *                                             bitplane.hpp:15-44
 *   - FP64 quantizer, round half away from zero, no FMA contraction
 *     (compile with -ffp-contract=off)        quantizer.hpp:146-213, core.hpp:145
 *
 * Status codes mirror the product C-ABI: 0 ok, 1 shape, 2 value, 3 overflow.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE 1
#define ORC_VALUE 2
#define ORC_OVERFLOW 3

/* scheme / granularity enums: quantizer.hpp:14-15 */
#define ORC_ASYM 0
#define ORC_SYM 1
#define ORC_BAL 2
#define ORC_PER_TENSOR 0
#define ORC_PER_CHANNEL 1
#define ORC_PER_TOKEN 2

static size_t wpr_of(size_t cols) { return (cols + 63) / 64; }

/* QuantSpec::levels  quantizer.hpp:49-51 */
unsigned orc_levels(unsigned bits, int scheme) {
  return scheme == ORC_BAL ? (1u << bits) + 1u : (1u << bits);
}

/* QuantSpec::planes  quantizer.hpp:54-59 */
unsigned orc_planes(unsigned bits, int scheme) {
  unsigned L = orc_levels(bits, scheme), p = 0;
  while ((1u << p) < L) ++p;
  return p;
}

/* fits_int32  gemm.hpp:73-77 */
int orc_fits_int32(unsigned p, unsigned q, size_t k) {
  unsigned log_k = 0;
  while (((size_t)1 << log_k) < k + 1) ++log_k;
  return p + q + log_k <= 31;
}

/* TileConfig::valid  gemm.hpp:24-32 */
int orc_tile_valid(size_t BM, size_t BN, size_t BK, size_t WM, size_t WN, size_t WK,
                   unsigned p, unsigned q) {
  if (WK != 128) return 0;
  if (BK != 128 && BK != 256 && BK != 384 && BK != 512) return 0;
  if (BK % WK != 0) return 0;
  if (BM == 0 || BN == 0 || WM == 0 || WN == 0) return 0;
  if (WM % 8 != 0 || WN % 8 != 0) return 0;
  double warps = ((double)BM * p / (double)WM) * ((double)BN * q / (double)WN);
  return warps >= 1.0 && warps <= 32.0;
}

/* padding_redundancy  tune.hpp:17-23 (returns -1 on invalid arguments) */
double orc_padding_redundancy(size_t m, unsigned p, size_t mma_m) {
  if (m == 0 || p == 0 || mma_m == 0) return -1.0;
  size_t expanded = p * m;
  size_t padded = (expanded + mma_m - 1) / mma_m * mma_m;
  return (double)(padded - expanded) / (double)padded;
}

/*
 * quantize  quantizer.hpp:146-213 (+ axis_ranges 116-129, check_finite 131-140).
 * x is rows x cols row-major double; comp_a/comp_b may be NULL (no compensation).
 * scales/zero_points hold 1 entry (per-tensor) or `rows` entries.
 * On a non-finite element returns ORC_VALUE and writes its flat index to *bad.
 */
int orc_quantize(const double* x, size_t rows, size_t cols, unsigned bits, int scheme,
                 int granularity, double alpha, double beta, const double* comp_a,
                 const double* comp_b, uint8_t* codes, double* scales, int32_t* zero_points,
                 int64_t* bad) {
  size_t i, j, gi, groups;
  unsigned L;
  double* v;
  if (bits < 1 || bits > 8) return ORC_VALUE;
  if (scheme == ORC_BAL && bits > 7) return ORC_VALUE;
  if (!(alpha > 0.0 && alpha <= 1.0) || !(beta > 0.0 && beta <= 1.0)) return ORC_VALUE;
  for (i = 0; i < rows * cols; ++i)
    if (!isfinite(x[i])) {
      if (bad) *bad = (int64_t)i;
      return ORC_VALUE;
    }
  v = (double*)malloc(sizeof(double) * (rows * cols != 0 ? rows * cols : 1));
  memcpy(v, x, sizeof(double) * rows * cols);
  if (comp_a && comp_b)
    for (i = 0; i < rows; ++i)
      for (j = 0; j < cols; ++j) v[i * cols + j] += comp_a[i] * comp_b[j];
  L = orc_levels(bits, scheme);
  groups = granularity == ORC_PER_TENSOR ? 1 : rows;
  for (gi = 0; gi < groups; ++gi) {
    double lo = INFINITY, hi = -INFINITY, step;
    int32_t z;
    size_t r0 = granularity == ORC_PER_TENSOR ? 0 : gi;
    size_t r1 = granularity == ORC_PER_TENSOR ? rows : gi + 1;
    for (i = r0; i < r1; ++i)
      for (j = 0; j < cols; ++j) {
        double e = v[i * cols + j];
        lo = e < lo ? e : lo; /* std::min(lo, v) */
        hi = hi < e ? e : hi; /* std::max(hi, v) */
      }
    lo = beta * lo;
    hi = alpha * hi;
    if (scheme == ORC_ASYM) {
      if (hi == lo) {
        step = 1.0;
        z = 0;
      } else {
        double zz;
        step = (hi - lo) / (double)(L - 1);
        zz = round(-lo / step);
        zz = zz < 0.0 ? 0.0 : (zz > (double)(L - 1) ? (double)(L - 1) : zz);
        z = (int32_t)zz;
      }
    } else {
      double amax = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
      int32_t half = (int32_t)(1u << (bits - 1));
      if (amax == 0.0) {
        step = 1.0;
        z = 0;
      } else {
        if (scheme == ORC_BAL)
          step = amax / (double)half;
        else
          step = bits == 1 ? amax : amax / (double)(half - 1);
        z = half;
      }
    }
    scales[gi] = step;
    zero_points[gi] = z;
  }
  for (i = 0; i < rows; ++i) {
    size_t g = granularity == ORC_PER_TENSOR ? 0 : i;
    double step = scales[g], z = (double)zero_points[g];
    for (j = 0; j < cols; ++j) {
      double c = round(v[i * cols + j] / step) + z;
      c = c < 0.0 ? 0.0 : (c > (double)(L - 1) ? (double)(L - 1) : c);
      codes[i * cols + j] = (uint8_t)c;
    }
  }
  free(v);
  return ORC_OK;
}

/* dequantize  quantizer.hpp:243-254 */
void orc_dequantize(const uint8_t* codes, size_t rows, size_t cols, int granularity,
                    const double* scales, const int32_t* zero_points, double* out) {
  size_t i, j;
  for (i = 0; i < rows; ++i) {
    size_t g = granularity == ORC_PER_TENSOR ? 0 : i;
    double step = scales[g], z = (double)zero_points[g];
    for (j = 0; j < cols; ++j) out[i * cols + j] = ((double)codes[i * cols + j] - z) * step;
  }
}

/* bitpack  bitplane.hpp:47-64.  Returns ORC_VALUE with *bad = flat index of the
 * first (row-major) out-of-range code. */
int orc_bitpack(const uint8_t* codes, size_t rows, size_t cols, unsigned bits, uint64_t* planes,
                int64_t* bad) {
  size_t i, j, wpr = wpr_of(cols);
  unsigned s, max_code;
  if (bits < 1 || bits > 8) return ORC_VALUE;
  max_code = bits >= 8 ? 255u : ((1u << bits) - 1u);
  memset(planes, 0, sizeof(uint64_t) * bits * rows * wpr);
  for (i = 0; i < rows; ++i)
    for (j = 0; j < cols; ++j) {
      unsigned c = codes[i * cols + j];
      if (c > max_code) {
        if (bad) *bad = (int64_t)(i * cols + j);
        return ORC_VALUE;
      }
      for (s = 0; s < bits; ++s)
        if ((c >> s) & 1u) planes[((size_t)s * rows + i) * wpr + j / 64] |= (uint64_t)1 << (j % 64);
    }
  return ORC_OK;
}

/* unpack  bitplane.hpp:66-76 */
void orc_unpack(const uint64_t* planes, unsigned bits, size_t rows, size_t cols, uint8_t* codes) {
  size_t i, j, wpr = wpr_of(cols);
  unsigned s;
  for (i = 0; i < rows; ++i)
    for (j = 0; j < cols; ++j) {
      unsigned c = 0;
      for (s = 0; s < bits; ++s)
        if ((planes[((size_t)s * rows + i) * wpr + j / 64] >> (j % 64)) & 1u) c |= 1u << s;
      codes[i * cols + j] = (uint8_t)c;
    }
}

/* bmma  bitplane.hpp:81-96 (single plane pair AND+popcount) */
void orc_bmma(const uint64_t* a, unsigned a_planes, size_t m, unsigned a_plane, const uint64_t* bt,
              unsigned b_planes, size_t n, unsigned b_plane, size_t k, int32_t* out) {
  size_t i, j, w, wpr = wpr_of(k);
  (void)a_planes;
  (void)b_planes;
  for (i = 0; i < m; ++i) {
    const uint64_t* ra = a + ((size_t)a_plane * m + i) * wpr;
    for (j = 0; j < n; ++j) {
      const uint64_t* rb = bt + ((size_t)b_plane * n + j) * wpr;
      int32_t acc = 0;
      for (w = 0; w < wpr; ++w) acc += __builtin_popcountll(ra[w] & rb[w]);
      out[i * n + j] = acc;
    }
  }
}

/*
 * gemm_naive / gemm_arbitrary(_wide)  gemm.hpp:185-231: acc[i][j] =
 * sum_{s<p} sum_{t<q} 2^(s+t) * popc-GEMM(A_s, W_t).  The blocked loop order
 * of gemm_plane_rows (94-146) does not change the exact integer result
 * (README:38-41, test_bitkernel.cpp:104-115), so one plain loop restates all
 * three.  Computed in int64; callers narrow to int32 when fits_int32 holds.
 */
void orc_gemm_planes(const uint64_t* a, unsigned p, size_t m, const uint64_t* bt, unsigned q,
                     size_t n, size_t k, int64_t* out) {
  size_t i, j, w, wpr = wpr_of(k);
  unsigned s, t;
  memset(out, 0, sizeof(int64_t) * m * n);
  for (s = 0; s < p; ++s)
    for (t = 0; t < q; ++t) {
      int64_t weight = (int64_t)1 << (s + t);
      for (i = 0; i < m; ++i) {
        const uint64_t* ra = a + ((size_t)s * m + i) * wpr;
        for (j = 0; j < n; ++j) {
          const uint64_t* rb = bt + ((size_t)t * n + j) * wpr;
          int64_t acc = 0;
          for (w = 0; w < wpr; ++w) acc += __builtin_popcountll(ra[w] & rb[w]);
          out[i * n + j] += weight * acc;
        }
      }
    }
}

/* int32 entry with the reference's validation order: shape, (tile), overflow
 * gemm.hpp:187-194 */
int orc_gemm_arbitrary_i32(const uint64_t* a, unsigned p, size_t m, const uint64_t* bt, unsigned q,
                           size_t n, size_t k, int32_t* out) {
  size_t i;
  int64_t* tmp;
  if (!orc_fits_int32(p, q, k)) return ORC_OVERFLOW;
  tmp = (int64_t*)malloc(sizeof(int64_t) * (m * n != 0 ? m * n : 1));
  orc_gemm_planes(a, p, m, bt, q, n, k, tmp);
  for (i = 0; i < m * n; ++i) out[i] = (int32_t)tmp[i];
  free(tmp);
  return ORC_OK;
}

/* code_rowsums  gemm.hpp:256-261 */
void orc_code_rowsums(const uint8_t* codes, size_t rows, size_t cols, int64_t* out) {
  size_t i, j;
  for (i = 0; i < rows; ++i) {
    int64_t s = 0;
    for (j = 0; j < cols; ++j) s += codes[i * cols + j];
    out[i] = s;
  }
}

/* zero_point_correct  gemm.hpp:235-254 (int64 arithmetic, then the caller's Acc) */
void orc_zero_point_correct(const int64_t* acc, size_t m, size_t n, const int64_t* rowsum_a,
                            const int64_t* colsum_b, const int32_t* z_a, const int32_t* z_b,
                            size_t k, int64_t* out) {
  size_t i, j;
  for (i = 0; i < m; ++i)
    for (j = 0; j < n; ++j)
      out[i * n + j] = acc[i * n + j] - (int64_t)z_a[i] * colsum_b[j] -
                       (int64_t)z_b[j] * rowsum_a[i] + (int64_t)k * z_a[i] * z_b[j];
}

/*
 * quantized_linear  gemm.hpp:266-307: codes in, dequantized doubles out.
 * act: m x k codes with act_planes planes, per-token (or per-tensor) s_a/z_a.
 * wt : n x k codes (stored transposed) with wt_planes planes, per-channel s_b/z_b.
 * a_per_tensor / b_per_tensor select index 0 for every row (axis_of 93-95).
 * The narrowing of `corrected` to int32 (fits_int32 branch, 293-298) is
 * restated by the (int32_t) cast, exactly as static_cast<Acc> does.
 */
int orc_quantized_linear(const uint8_t* act, size_t m, unsigned p, const double* s_a,
                         const int32_t* z_a, int a_per_tensor, const uint8_t* wt, size_t n,
                         unsigned q, const double* s_b, const int32_t* z_b, int b_per_tensor,
                         size_t k, double* out) {
  size_t i, j, wpr = wpr_of(k);
  int64_t bad;
  uint64_t *pa, *pb;
  int64_t *acc, *rows_a, *cols_b, *corr;
  int32_t *za, *zb;
  int wide = !orc_fits_int32(p, q, k);
  pa = (uint64_t*)malloc(sizeof(uint64_t) * (p * m * wpr + 1));
  pb = (uint64_t*)malloc(sizeof(uint64_t) * (q * n * wpr + 1));
  if (orc_bitpack(act, m, k, p, pa, &bad) || orc_bitpack(wt, n, k, q, pb, &bad)) {
    free(pa);
    free(pb);
    return ORC_VALUE;
  }
  acc = (int64_t*)malloc(sizeof(int64_t) * (m * n + 1));
  corr = (int64_t*)malloc(sizeof(int64_t) * (m * n + 1));
  rows_a = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
  cols_b = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  za = (int32_t*)malloc(sizeof(int32_t) * (m + 1));
  zb = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
  orc_gemm_planes(pa, p, m, pb, q, n, k, acc);
  orc_code_rowsums(act, m, k, rows_a);
  orc_code_rowsums(wt, n, k, cols_b);
  for (i = 0; i < m; ++i) za[i] = z_a[a_per_tensor ? 0 : i];
  for (j = 0; j < n; ++j) zb[j] = z_b[b_per_tensor ? 0 : j];
  if (!wide)
    for (i = 0; i < m * n; ++i) acc[i] = (int32_t)acc[i];
  orc_zero_point_correct(acc, m, n, rows_a, cols_b, za, zb, k, corr);
  for (i = 0; i < m; ++i) {
    double sa = s_a[a_per_tensor ? 0 : i];
    for (j = 0; j < n; ++j) {
      double sb = s_b[b_per_tensor ? 0 : j];
      double c = wide ? (double)corr[i * n + j] : (double)(int32_t)corr[i * n + j];
      out[i * n + j] = sa * sb * c;
    }
  }
  free(pa);
  free(pb);
  free(acc);
  free(corr);
  free(rows_a);
  free(cols_b);
  free(za);
  free(zb);
  return ORC_OK;
}

/* GemmStats law  gemm.hpp:61-64, 108-115: block tiles = ceil(M/BM)*ceil(N/BN)
 * (row tiles are split across workers at BM granularity, 155-169, which does
 * not change the count); plane pairs = tiles * p * q. */
void orc_gemm_stats(size_t m, size_t n, size_t BM, size_t BN, unsigned p, unsigned q,
                    uint64_t* block_tiles, uint64_t* plane_pairs) {
  uint64_t tiles = (uint64_t)((m + BM - 1) / BM) * (uint64_t)((n + BN - 1) / BN);
  *block_tiles = tiles;
  *plane_pairs = tiles * p * q;
}
