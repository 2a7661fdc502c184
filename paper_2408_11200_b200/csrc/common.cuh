// common.cuh — shared device helpers for the B200 KAN/UKAN kernels.
//
// Numerics contract: grid indices are computed in fp64 from the
// exactly-upcast fp32 input using the reference's expression order, with every operation
// spelled as an explicitly-rounded intrinsic (__dmul_rn / __dadd_rn / __dsub_rn /
// __ddiv_rn) so nvcc cannot contract them into FMAs.  That makes cells / g_id bit-exact
// against NumPy (layers.py:261-264, 294-300).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/ukan_b200.h"

#define UKAN_CUDA_TRY(expr)                                     \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return (int)_e;                      \
  } while (0)

// Every kernel launch of the library is followed by UKAN_LAUNCH_CHECK(), which also counts it
// (ukan_launch_count(), for the benchmark's gpu_launches figure).
extern "C" void ukan_note_launch(void);
#define UKAN_LAUNCH_CHECK()  \
  do {                       \
    ukan_note_launch();      \
    UKAN_CUDA_TRY(cudaGetLastError()); \
  } while (0)

namespace ukan {

// Stream-ordered scratch for the convenience entry points that take no caller workspace.  The
// device's default pool keeps its memory mapped (release threshold raised once), so repeated
// calls do not remap pages at every synchronisation.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st);

// Epilogue of the FP64 tensor-core GEMMs (cg_dmma.cu): v = D + bias[n]; pre64 = v;
// v = silu(v) if act; c64 = v; c32 = (float)v.  Every pointer is optional; fp64 arithmetic.
struct DgOut {
  float* c32 = nullptr;
  double* c64 = nullptr;
  double* pre64 = nullptr;
  const float* bias = nullptr;
  int act = 0;
};
template <typename TA, typename TB>
int cg_dmma_gemm_t(const TA* A, int64_t sam, int64_t sak, const TB* Bm, int64_t sbk, int64_t sbn, int64_t M,
                   int64_t N, int64_t K, const DgOut& out, double* part, cudaStream_t st);
int64_t cg_dmma_workspace(int64_t M, int64_t N, int64_t K);

constexpr int kMaxK = UKAN_MAX_DEGREE + 1;

// Basis matrix passed by value as a kernel parameter (<= 11*11 doubles).
template <int K>
struct Basis {
  double M[K][K];  // M[m][j]: coefficient of u^m in window slot j (bspline.py:76)
};

// Constants of the bounded KAN grid, computed on the host with the reference's own
// expressions (layers.py:159, 296, 299-300) — never re-derived on the device.
struct KanGrid {
  double g_min;    // layer.g_min
  double hi;       // np.nextafter(g_max, g_min)              layers.py:296
  double dg;       // (g_max - g_min) / G                       layers.py:159
  double inv_dg;   // 1.0 / dg                                  layers.py:300
  double gmin_dg;  // g_min / dg                                layers.py:300
  int G;
};

// Host: build KanGrid exactly as Python would (IEEE binary64, no extended precision).
KanGrid make_kan_grid(double g_min, double g_max, int64_t G);

// KAN locate (layers.py:294-301 + tensor.py:327-338).
//   xc   = clip(x, g_min, hi)
//   mask = (x >= g_min) & (x <= hi)
//   cell = clip(floor((xc - g_min) / dg), 0, G-1)
//   u    = xc * (1/dg) - (cell + g_min/dg)
// Returns false for NaN input (the reference raises IndexError, SURVEY gotcha 10).
__device__ __forceinline__ bool kan_locate(float xf, const KanGrid& g, int& cell, double& u,
                                           bool& mask) {
  const double x = (double)xf;
  mask = (x >= g.g_min) && (x <= g.hi);
  double xc = x;
  if (xc < g.g_min) xc = g.g_min;
  if (xc > g.hi) xc = g.hi;
  const double q = floor(__ddiv_rn(__dsub_rn(xc, g.g_min), g.dg));
  double qc = q < 0.0 ? 0.0 : q;
  const double gm1 = (double)(g.G - 1);
  if (qc > gm1) qc = gm1;
  cell = (int)qc;
  u = __dsub_rn(__dmul_rn(xc, g.inv_dg), __dadd_rn((double)cell, g.gmin_dg));
  return !isnan(x);
}

// Floor division / Euclidean modulo (Python semantics) for int64 (SURVEY gotcha 4).
__device__ __forceinline__ int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

// UKAN locate (layers.py:261-264): s = x * (1/dg); g_id = floor(s); u = s - g_id.
__device__ __forceinline__ void ukan_locate(float xf, double inv_dg, int64_t& g_id, double& u) {
  const double s = __dmul_rn((double)xf, inv_dg);
  const double fl = floor(s);
  g_id = (int64_t)fl;
  u = __dsub_rn(s, fl);
}

// Basis weights w_j(u) = sum_m u^m M[m][j] (layers.py:29-37, d = 0), Horner in fp64.
template <int K>
__device__ __forceinline__ void basis_weights(const Basis<K>& B, double u, double (&w)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double acc = B.M[K - 1][j];
#pragma unroll
    for (int m = K - 2; m >= 0; --m) acc = fma(acc, u, B.M[m][j]);
    w[j] = acc;
  }
}

// First derivative weights w'_j(u) = sum_{m>=1} m u^(m-1) M[m][j] (layers.py:29-37, d = 1).
template <int K>
__device__ __forceinline__ void basis_dweights(const Basis<K>& B, double u, double (&w)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (K == 1) {
      w[j] = 0.0;
    } else {
      double acc = (double)(K - 1) * B.M[K - 1][j];
#pragma unroll
      for (int m = K - 2; m >= 1; --m) acc = fma(acc, u, (double)m * B.M[m][j]);
      w[j] = acc;
    }
  }
}

__device__ __forceinline__ double silu_d(double x) { return x / (1.0 + exp(-x)); }
__device__ __forceinline__ double dsilu_d(double x) {
  const double s = 1.0 / (1.0 + exp(-x));
  return s + x * s * (1.0 - s);
}

}  // namespace ukan

// Host helper: exact basis matrix (basis.cpp).
int ukan_basis_matrix_impl(int k, double* M_out);

// Dispatch helper: call F<K>() for K = k+1 in [1, 11].
#define UKAN_DISPATCH_K(k, ...)                 \
  switch ((k) + 1) {                            \
    case 1: { constexpr int K = 1; __VA_ARGS__ } break;   \
    case 2: { constexpr int K = 2; __VA_ARGS__ } break;   \
    case 3: { constexpr int K = 3; __VA_ARGS__ } break;   \
    case 4: { constexpr int K = 4; __VA_ARGS__ } break;   \
    case 5: { constexpr int K = 5; __VA_ARGS__ } break;   \
    case 6: { constexpr int K = 6; __VA_ARGS__ } break;   \
    case 7: { constexpr int K = 7; __VA_ARGS__ } break;   \
    case 8: { constexpr int K = 8; __VA_ARGS__ } break;   \
    case 9: { constexpr int K = 9; __VA_ARGS__ } break;   \
    case 10: { constexpr int K = 10; __VA_ARGS__ } break; \
    case 11: { constexpr int K = 11; __VA_ARGS__ } break; \
    default: return UKAN_E_DEGREE;              \
  }

// Exact basis matrix for K = k+1, computed once per process and cached.
template <int K>
inline const ukan::Basis<K>& make_basis(int k) {
  static const ukan::Basis<K> cached = [k] {
    ukan::Basis<K> b;
    double M[ukan::kMaxK * ukan::kMaxK];
    ukan_basis_matrix_impl(k, M);
    for (int m = 0; m < K; ++m)
      for (int j = 0; j < K; ++j) b.M[m][j] = M[m * K + j];
    return b;
  }();
  return cached;
}
