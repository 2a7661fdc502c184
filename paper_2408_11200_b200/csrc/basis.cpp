// basis.cpp — exact basis matrix of the uniform degree-k B-spline (host side).
//
// Restates bspline._segment_polynomials / basis_matrix (bspline.py:24-80): the monomial
// coefficients of B_{j,k}(u) on [0,1) for j = -k..0 from the Cox-de Boor recursion on unit
// knots, in exact rational arithmetic; column j of M is the polynomial of B_{j-k,k}, row i is
// the coefficient of u^i.  Each entry is rounded once to the nearest double
// (float(Fraction) semantics: numerator and denominator are exact in binary64, so one IEEE
// division is correctly rounded).
#include <cstdint>
#include <cstdlib>
#include <map>
#include <vector>

#include "../../include/ukan_b200.h"

namespace {

int64_t gcd64(int64_t a, int64_t b) {
  a = a < 0 ? -a : a;
  b = b < 0 ? -b : b;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

struct Frac {
  int64_t n = 0, d = 1;
  Frac() = default;
  Frac(int64_t n_, int64_t d_ = 1) : n(n_), d(d_) { norm(); }
  void norm() {
    if (d < 0) { n = -n; d = -d; }
    int64_t g = gcd64(n, d);
    if (g > 1) { n /= g; d /= g; }
    if (n == 0) d = 1;
  }
  Frac operator+(const Frac& o) const {
    int64_t g = gcd64(d, o.d);
    return Frac(n * (o.d / g) + o.n * (d / g), (d / g) * o.d);
  }
  Frac operator-(const Frac& o) const { return *this + Frac(-o.n, o.d); }
  Frac operator*(const Frac& o) const {
    int64_t g1 = gcd64(n, o.d), g2 = gcd64(o.n, d);
    if (g1 == 0) g1 = 1;
    if (g2 == 0) g2 = 1;
    return Frac((n / g1) * (o.n / g2), (d / g2) * (o.d / g1));
  }
  double to_double() const { return (double)n / (double)d; }
};

}  // namespace

int ukan_basis_matrix_impl(int k, double* M_out) {
  if (k < 0 || k > UKAN_MAX_DEGREE || M_out == nullptr) return UKAN_E_DEGREE;
  // polys[j] = monomial coefficients (constant first) of B_{j,kk} on [0,1), j in [-kk, 0]
  std::map<int, std::vector<Frac>> polys;
  polys[0] = {Frac(1)};
  for (int kk = 1; kk <= k; ++kk) {
    std::map<int, std::vector<Frac>> nxt;
    for (int j = -kk; j <= 0; ++j) {
      std::vector<Frac> c(kk + 1);
      auto L = polys.find(j), R = polys.find(j + 1);
      if (L != polys.end()) {  // (u - j)/kk * left
        for (size_t i = 0; i < L->second.size(); ++i) {
          c[i + 1] = c[i + 1] + L->second[i] * Frac(1, kk);
          c[i] = c[i] + L->second[i] * Frac(-j, kk);
        }
      }
      if (R != polys.end()) {  // (j + kk + 1 - u)/kk * right
        for (size_t i = 0; i < R->second.size(); ++i) {
          c[i] = c[i] + R->second[i] * Frac(j + kk + 1, kk);
          c[i + 1] = c[i + 1] - R->second[i] * Frac(1, kk);
        }
      }
      nxt[j] = c;
    }
    polys.swap(nxt);
  }
  const int K = k + 1;
  for (int j = 0; j < K; ++j) {
    const std::vector<Frac>& col = polys[j - k];
    for (int i = 0; i < K; ++i) M_out[i * K + j] = col[i].to_double();
  }
  return UKAN_OK;
}
