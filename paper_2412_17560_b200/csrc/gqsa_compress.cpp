// gqsa_compress.cpp -- the method's offline compression front-end (host C++):
// dense layer W -> plain BSR of kept, quantized groups (the storage the
// packer and the GEMV consume).  SURVEY §8(a) row a0, §8(f) NEXT-4.
//
//   Eq. 4      s_{r,c} = W[r,c]^2 / ([H^-1]_cc)^2
//   Fig. 3    group score = mean of s over the G columns of
//                               a group (summed t = 0..G-1 in fp64)
//   group pruning               exactly floor(S * total) lowest-score groups
//                               of the layer pruned; ties -> lower (row, group)
//                               index first (readings R13, R17)
//   Eq. 1-2    per kept group: s = (max-min)/(2^n-1),
//                               z = -round(min/s), q = clamp(round(W/s)+z),
//                               rounding half away from zero (R5); constant
//                               groups by R9; s and z stored as fp16 (RNE, R7)
//
// Every score and parameter is computed in IEEE fp64 in a fixed order, so the
// result is a deterministic function of (W, diag(H^-1), S, n, G).  H^-1's
// diagonal is an INPUT (the Hessian estimate and its inverse are a dense
// library factorisation; paper_2412_17560_b200/frontend.py computes them).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/gqsa.h"

namespace {

// IEEE binary16 bit pattern of v, rounded to nearest even (directly from fp64).
uint16_t f64_to_f16_rne(double v) {
  const uint16_t sign = std::signbit(v) ? 0x8000u : 0u;
  if (std::isnan(v)) return sign | 0x7e00u;
  const double a = std::fabs(v);
  if (a >= 65520.0) return sign | 0x7c00u;  // rounds to infinity
  if (a < 6.103515625e-05) {                 // below 2^-14: subnormal (or zero)
    const double q = std::nearbyint(a * 16777216.0);  // units of 2^-24, exact scaling
    return sign | (uint16_t)q;               // q == 1024 is the smallest normal
  }
  int ex = 0;
  std::frexp(a, &ex);                        // a = m 2^ex, m in [0.5, 1)
  int e = ex - 1;                            // a in [2^e, 2^(e+1))
  double m = std::nearbyint(std::ldexp(a, 10 - e));  // in [1024, 2048]
  if (m >= 2048.0) {
    m = 1024.0;
    ++e;
  }
  if (e + 15 >= 31) return sign | 0x7c00u;
  return sign | (uint16_t)((e + 15) << 10) | (uint16_t)((int)m - 1024);
}

double round_half_away(double v) { return std::copysign(std::floor(std::fabs(v) + 0.5), v); }

int check_args(int32_t rows, int32_t cols, int32_t G, double sparsity) {
  if (rows < 0 || cols <= 0 || G <= 0 || cols % G) return GQSA_ERR_SHAPE;
  if (cols / G > 65536) return GQSA_ERR_UNSUPPORTED;  // group_cols are u16
  if (!(sparsity >= 0.0 && sparsity < 1.0)) return GQSA_ERR_SHAPE;
  return GQSA_OK;
}

}  // namespace

extern "C" int gqsa_compress_nnzg(int32_t rows, int32_t cols, int32_t group_size, double sparsity,
                                  int64_t* nnzg) {
  if (!nnzg) return GQSA_ERR_BUFFER;
  int st = check_args(rows, cols, group_size, sparsity);
  if (st) return st;
  const int64_t total = (int64_t)rows * (cols / group_size);
  *nnzg = total - (int64_t)std::floor(sparsity * (double)total);
  return GQSA_OK;
}

extern "C" int gqsa_compress(const float* W, int32_t rows, int32_t cols, int32_t group_size, int32_t bits,
                             const double* hinv_diag, double sparsity, gqsa_bsr_t* out,
                             double* group_saliency) {
  int st = check_args(rows, cols, group_size, sparsity);
  if (st) return st;
  if (bits != 2 && bits != 4 && bits != 8) return GQSA_ERR_UNSUPPORTED;
  if (!W || !hinv_diag || !out || !out->row_index) return GQSA_ERR_BUFFER;
  const int G = group_size, gpr = cols / G;
  const int64_t total = (int64_t)rows * gpr;
  int64_t nnzg = 0;
  gqsa_compress_nnzg(rows, cols, G, sparsity, &nnzg);
  if (nnzg > 0 && (!out->group_cols || !out->codes || !out->scales_f16 || !out->zeros_f16))
    return GQSA_ERR_BUFFER;
  for (int c = 0; c < cols; ++c)
    if (!std::isfinite(hinv_diag[c]) || !(hinv_diag[c] > 0.0)) return GQSA_ERR_VALIDATION;
  for (int64_t i = 0; i < (int64_t)rows * cols; ++i)
    if (!std::isfinite(W[i])) return GQSA_ERR_VALIDATION;

  // ---- Eq. 4 per weight, averaged per group (fp64, t ascending)
  std::vector<double> score((size_t)total);
  for (int32_t r = 0; r < rows; ++r) {
    const float* wr = W + (int64_t)r * cols;
    for (int g = 0; g < gpr; ++g) {
      double acc = 0.0;
      for (int t = 0; t < G; ++t) {
        const double w = (double)wr[g * G + t];
        const double d = hinv_diag[g * G + t];
        acc = acc + (w * w) / (d * d);
      }
      score[(size_t)r * gpr + g] = acc / G;
    }
  }
  if (group_saliency) std::memcpy(group_saliency, score.data(), sizeof(double) * (size_t)total);

  // ---- prune the floor(S * total) lowest scores; ties by (row, group) index
  const int64_t n_prune = total - nnzg;
  std::vector<uint8_t> keep((size_t)total, 1);
  if (n_prune > 0) {
    std::vector<int64_t> idx((size_t)total);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    auto less = [&](int64_t a, int64_t b) { return score[a] < score[b] || (score[a] == score[b] && a < b); };
    std::nth_element(idx.begin(), idx.begin() + (n_prune - 1), idx.end(), less);
    for (int64_t i = 0; i < n_prune; ++i) keep[(size_t)idx[(size_t)i]] = 0;
  }

  // ---- Eq. 1-2 per kept group, in CSR order
  int32_t* ri = const_cast<int32_t*>(out->row_index);
  uint16_t* gc = const_cast<uint16_t*>(out->group_cols);
  uint8_t* codes = const_cast<uint8_t*>(out->codes);
  uint16_t* s16 = const_cast<uint16_t*>(out->scales_f16);
  uint16_t* z16 = const_cast<uint16_t*>(out->zeros_f16);
  if (nnzg > 0) std::memset(codes, 0, (size_t)((nnzg * G * bits + 7) / 8));
  const int qmax = (1 << bits) - 1;
  int64_t k = 0, e = 0;  // kept-group counter, code element counter
  ri[0] = 0;
  for (int32_t r = 0; r < rows; ++r) {
    const float* wr = W + (int64_t)r * cols;
    for (int g = 0; g < gpr; ++g) {
      if (!keep[(size_t)r * gpr + g]) continue;
      double lo = (double)wr[g * G], hi = lo;
      for (int t = 1; t < G; ++t) {
        const double w = (double)wr[g * G + t];
        lo = std::min(lo, w);
        hi = std::max(hi, w);
      }
      double s, z;
      if (hi == lo) {  // constant group (reading R9): code 0 dequantizes to c exactly
        s = lo == 0.0 ? 1.0 : std::fabs(lo);
        z = lo == 0.0 ? 0.0 : -std::copysign(1.0, lo);
      } else {
        s = (hi - lo) / (double)qmax;
        z = -round_half_away(lo / s);
      }
      const uint16_t sh = f64_to_f16_rne(s), zh = f64_to_f16_rne(z);
      if ((sh & 0x7c00u) == 0x7c00u || (zh & 0x7c00u) == 0x7c00u || (sh & 0x7fffu) == 0 || (sh & 0x8000u))
        return GQSA_ERR_VALIDATION;  // not representable in fp16 (reading R8)
      for (int t = 0; t < G; ++t, ++e) {
        double q = round_half_away((double)wr[g * G + t] / s) + z;
        q = std::min(std::max(q, 0.0), (double)qmax);
        const uint32_t qi = (uint32_t)q;
        const int64_t bit = e * bits;  // low bits first
        codes[bit >> 3] |= (uint8_t)(qi << (bit & 7));
      }
      gc[k] = (uint16_t)g;
      s16[k] = sh;
      z16[k] = zh;
      ++k;
    }
    ri[r + 1] = (int32_t)k;
  }
  out->rows = rows;
  out->cols = cols;
  out->group_size = G;
  out->bits = bits;
  out->nnzg = nnzg;
  return GQSA_OK;
}
