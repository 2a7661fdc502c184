// kan_tangent.cu — forward tangent (JVP) of the KAN / UKAN spline layer and its backward
// (the PINN task differentiates df/dt through the layer, tasks.py:153-166).
//
// Reference: the tangent channel of the fused graph ops — basis_features (layers.py:49-53:
// basis.tangent = w'(u) * u.tangent), span_gather (73-74, none: tables carry no tangent here),
// edge_combine (91-104), the clamp tangent (tensor.py:336-337), mul(xc, 1/dg) (layers.py:300,
// UKAN 264) and the silu tangent of the base branch (tensor.py:236-241).  With
//   m_bi = tx[b,i] * mask_bi * (1/dg)                       (u.tangent)
//   v_j  = m_bi * w'_j(u_bi)                                (basis.tangent)
// the tangent output is
//   ty[b,o] = sum_i scale[i,o] sum_j v_j T[row_bi + j, o]  (+ sum_i tx silu'(x) bw[i,o])
// and the reverse pass of sum(ty * gt) through that graph gives
//   dT[row+j, o]  += scale[i,o] * sum_b v_j gt[b,o]
//   dscale[i,o]   += sum_b gt[b,o] sum_j v_j T[row+j, o]
//   dtx[b,i]       = mask/dg * sum_o gt scale sum_j w'_j T  (+ silu'(x) sum_o gt bw)
//   dx[b,i]       += tx mask/dg^2 * sum_o gt scale sum_j w''_j T  (+ tx silu''(x) sum_o gt bw)
//   dbw[i,o]      += sum_b gt[b,o] tx silu'(x)
// (dx here is the tangent path's share; the primal layer's backward adds the rest.)
// The tangent appears in small physics-informed models ([1, 5, 1] at 16-128 collocation
// points), so these kernels are written for clarity and determinism: fp64 evaluation and
// accumulation, fixed summation orders, no atomics; the table gradient is a gather over
// 32-row tiles that scans the batch per tile (O(B * d_in * rows / 32) locates).
#include <algorithm>

#include "common.cuh"
#include "rowmap.cuh"

namespace ukan {

template <int K>
__device__ __forceinline__ void basis_d2weights(const Basis<K>& B, double u, double (&w)[K]) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (K <= 2) {
      w[j] = 0.0;
    } else {
      double acc = (double)((K - 1) * (K - 2)) * B.M[K - 1][j];
#pragma unroll
      for (int m = K - 2; m >= 2; --m) acc = fma(acc, u, (double)(m * (m - 1)) * B.M[m][j]);
      w[j] = acc;
    }
  }
}

__device__ __forceinline__ double silu2_d(double x) {
  const double s = 1.0 / (1.0 + exp(-x));
  return s * (1.0 - s) * (2.0 + x * (1.0 - 2.0 * s));
}

template <bool UKAN>
__device__ __forceinline__ double tan_inv_dg(const RowMap& rm) {
  if constexpr (UKAN) return rm.inv_dg;
  else return rm.grid.inv_dg;
}

// (b, i) -> table row, tangent basis v_j = m * w'_j(u); false for NaN input (no contribution).
template <int K, bool UKAN>
__device__ __forceinline__ bool tan_eval(const RowMap& rm, const Basis<K>& bas, float xv, float tv, int64_t b, int i,
                                         int d_in, int& row, double (&v)[K]) {
  double u;
  bool mask;
  if (!locate_row<UKAN>(rm, xv, b, i, d_in, row, u, mask)) return false;
  const double m = mask ? (double)tv * tan_inv_dg<UKAN>(rm) : 0.0;
  basis_dweights<K>(bas, u, v);
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] *= m;
  return true;
}

constexpr int kTanF = 128;  // features staged per pass

// ty: CTA per sample; threads first evaluate the (row, v) of kTanF features, then sweep outputs.
template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
jvp_forward_kernel(const float* __restrict__ x, const float* __restrict__ tx, const float* __restrict__ T,
                   const float* __restrict__ scale, const float* __restrict__ bw, float* __restrict__ ty, int d_in,
                   int d_out, RowMap rm, Basis<K> bas) {
  __shared__ double sv[kTanF][K];
  __shared__ double sb[kTanF];
  __shared__ int srow[kTanF];
  const int64_t b = blockIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // outputs threadIdx.x + 256 q, q < 4, then a second sweep
  for (int o0 = 0; o0 < d_out; o0 += 1024) {
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = 0.0;
    for (int i0 = 0; i0 < d_in; i0 += kTanF) {
      __syncthreads();
      const int f = threadIdx.x;
      if (f < kTanF && i0 + f < d_in) {
        const int i = i0 + f;
        const float xv = x[b * d_in + i], tv = tx[b * d_in + i];
        double v[K];
        int row;
        const bool ok = tan_eval<K, UKAN>(rm, bas, xv, tv, b, i, d_in, row, v);
        srow[f] = ok ? row : -1;
#pragma unroll
        for (int j = 0; j < K; ++j) sv[f][j] = ok ? v[j] : 0.0;
        sb[f] = bw ? (double)tv * dsilu_d((double)xv) : 0.0;
      }
      __syncthreads();
      const int nf = min(kTanF, d_in - i0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int o = o0 + threadIdx.x + 256 * q;
        if (o >= d_out) continue;
        double a = acc[q];
        for (int f2 = 0; f2 < nf; ++f2) {
          const int i = i0 + f2, row = srow[f2];
          if (row >= 0) {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < K; ++j) t = fma(sv[f2][j], (double)T[(size_t)(row + j) * d_out + o], t);
            a = fma((double)scale[(size_t)i * d_out + o], t, a);
          }
          if (bw) a = fma(sb[f2], (double)bw[(size_t)i * d_out + o], a);
        }
        acc[q] = a;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = o0 + threadIdx.x + 256 * q;
      if (o < d_out) ty[b * d_out + o] = (float)acc[q];
    }
  }
}

// dT: warp per (32-row tile of the table, 32-output slice); for every feature whose row segment
// meets the tile it scans the batch in sample order (lane-parallel evaluation, 32 at a time)
// and accumulates the tile in fp64 shared memory, then writes scale * A for that feature's rows.
template <int K>
__host__ __device__ constexpr int tan_warp_doubles() { return 32 * 32 + 32 * K + 16; }

template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
jvp_dtable_kernel(const float* __restrict__ x, const float* __restrict__ tx, const float* __restrict__ scale,
                  const float* __restrict__ gt, float* __restrict__ dT, int B, int d_in, int d_out, int n_rows,
                  int n_os, RowMap rm, Basis<K> bas) {
  extern __shared__ __align__(16) double tsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double (*A)[32] = reinterpret_cast<double (*)[32]>(tsm + (size_t)warp * tan_warp_doubles<K>());
  double (*sv)[K] = reinterpret_cast<double (*)[K]>(&A[32][0]);
  int* srow = reinterpret_cast<int*>(&sv[32][0]);
  const int64_t unit = (int64_t)blockIdx.x * 8 + warp;
  const int n_rt = (n_rows + 31) / 32;
  if (unit >= (int64_t)n_rt * n_os) return;
  const int t = (int)(unit % n_rt), os = (int)(unit / n_rt);
  const int r0 = t * 32, o = os * 32 + lane;
  const bool live = o < d_out;
  // first feature whose segment contains r0
  int i = 0;
  if constexpr (UKAN) {
    int lo = 0, hi = d_in - 1;
    while (lo < hi) {  // largest i with seg_start[i]*K <= r0
      const int mid = (lo + hi + 1) >> 1;
      if (rm.seg_start[mid] * rm.K <= r0) lo = mid;
      else hi = mid - 1;
    }
    i = lo;
  } else {
    i = r0 / rm.R;
  }
  for (; i < d_in; ++i) {
    int row0, nrows;
    feature_rows<UKAN>(rm, i, row0, nrows);
    if (row0 >= r0 + 32) break;
    if (row0 + nrows <= r0 || nrows == 0) continue;
    for (int r = 0; r < 32; ++r) A[r][lane] = 0.0;
    for (int b0 = 0; b0 < B; b0 += 32) {
      const int b = b0 + lane;
      if (b < B) {
        double v[K];
        int row;
        const bool ok = tan_eval<K, UKAN>(rm, bas, x[(size_t)b * d_in + i], tx[(size_t)b * d_in + i], b, i, d_in,
                                          row, v);
        srow[lane] = (ok && row + K - 1 >= r0 && row < r0 + 32) ? row : INT32_MIN;
#pragma unroll
        for (int j = 0; j < K; ++j) sv[lane][j] = v[j];
      }
      __syncwarp();
      const int nb = min(32, B - b0);
      for (int q = 0; q < nb; ++q) {
        const int row = srow[q];
        if (row == INT32_MIN || !live) continue;
        const double g = (double)gt[(size_t)(b0 + q) * d_out + o];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const int r = row + j - r0;
          if (r >= 0 && r < 32) A[r][lane] = fma(sv[q][j], g, A[r][lane]);
        }
      }
      __syncwarp();
    }
    if (live) {
      const double sc = (double)scale[(size_t)i * d_out + o];
      const int ra = max(r0, row0), rb = min(r0 + 32, row0 + nrows);
      for (int r = ra; r < rb; ++r) dT[(size_t)r * d_out + o] = (float)(sc * A[r - r0][lane]);
    }
    __syncwarp();
  }
}

// dscale (and dbw): CTA per (feature i, 256 outputs); sample order.
template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
jvp_dscale_kernel(const float* __restrict__ x, const float* __restrict__ tx, const float* __restrict__ T,
                  const float* __restrict__ gt, float* __restrict__ dscale, float* __restrict__ dbw, int B, int d_in,
                  int d_out, RowMap rm, Basis<K> bas) {
  __shared__ double sv[256][K];
  __shared__ double sb[256];
  __shared__ int srow[256];
  const int i = blockIdx.x;
  const int o = blockIdx.y * 256 + threadIdx.x;
  double ds = 0.0, db = 0.0;
  for (int b0 = 0; b0 < B; b0 += 256) {
    __syncthreads();
    const int b = b0 + threadIdx.x;
    if (b < B) {
      const float xv = x[(size_t)b * d_in + i], tv = tx[(size_t)b * d_in + i];
      double v[K];
      int row;
      const bool ok = tan_eval<K, UKAN>(rm, bas, xv, tv, b, i, d_in, row, v);
      srow[threadIdx.x] = ok ? row : -1;
#pragma unroll
      for (int j = 0; j < K; ++j) sv[threadIdx.x][j] = ok ? v[j] : 0.0;
      sb[threadIdx.x] = dbw ? (double)tv * dsilu_d((double)xv) : 0.0;
    }
    __syncthreads();
    if (o < d_out) {
      const int nb = min(256, B - b0);
      for (int s = 0; s < nb; ++s) {
        const double g = (double)gt[(size_t)(b0 + s) * d_out + o];
        const int row = srow[s];
        if (row >= 0) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < K; ++j) t = fma(sv[s][j], (double)T[(size_t)(row + j) * d_out + o], t);
          ds = fma(g, t, ds);
        }
        if (dbw) db = fma(g, sb[s], db);
      }
    }
  }
  if (o < d_out) {
    dscale[(size_t)i * d_out + o] = (float)ds;
    if (dbw) dbw[(size_t)i * d_out + o] = (float)db;
  }
}

// dtx / dx: warp per (b, i), lanes over outputs, fixed xor-tree reduction.
template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
jvp_dinput_kernel(const float* __restrict__ x, const float* __restrict__ tx, const float* __restrict__ T,
                  const float* __restrict__ scale, const float* __restrict__ bw, const float* __restrict__ gt,
                  float* __restrict__ dx, float* __restrict__ dtx, int B, int d_in, int d_out, RowMap rm,
                  Basis<K> bas) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (p >= (int64_t)B * d_in) return;
  const int64_t b = p / d_in;
  const int i = (int)(p % d_in);
  const float xv = x[p], tv = tx[p];
  double u;
  bool mask;
  int row;
  const bool ok = locate_row<UKAN>(rm, xv, b, i, d_in, row, u, mask);
  double w1[K], w2[K];
  basis_dweights<K>(bas, u, w1);
  basis_d2weights<K>(bas, u, w2);
  double s1 = 0.0, s2 = 0.0, sbw = 0.0;
  for (int o = lane; o < d_out; o += 32) {
    const double g = (double)gt[(size_t)b * d_out + o];
    if (ok) {
      const double gs = g * (double)scale[(size_t)i * d_out + o];
      double c1 = 0.0, c2 = 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double c = (double)T[(size_t)(row + j) * d_out + o];
        c1 = fma(w1[j], c, c1);
        c2 = fma(w2[j], c, c2);
      }
      s1 = fma(gs, c1, s1);
      s2 = fma(gs, c2, s2);
    }
    if (bw) sbw = fma(g, (double)bw[(size_t)i * d_out + o], sbw);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    sbw += __shfl_xor_sync(0xffffffffu, sbw, off);
  }
  if (lane != 0) return;
  const double inv = mask && ok ? tan_inv_dg<UKAN>(rm) : 0.0;
  const double xd = (double)xv, td = (double)tv;
  if (dtx) {
    double d = inv * s1;
    if (bw) d += dsilu_d(xd) * sbw;
    dtx[p] = (float)d;
  }
  if (dx) {
    double d = td * inv * inv * s2;
    if (bw) d += td * silu2_d(xd) * sbw;
    dx[p] = (float)d;
  }
}

template <int K, bool UKAN>
static int jvp_forward_launch(const float* x, const float* tx, const float* T, const float* scale, const float* bw,
                              float* ty, int64_t B, int d_in, int d_out, const RowMap& rm, cudaStream_t st) {
  jvp_forward_kernel<K, UKAN><<<(unsigned)B, 256, 0, st>>>(x, tx, T, scale, bw, ty, d_in, d_out, rm,
                                                           make_basis<K>(K - 1));
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

template <int K, bool UKAN>
static int jvp_backward_launch(const float* x, const float* tx, const float* T, const float* scale, const float* bw,
                               const float* gt, float* dx, float* dtx, float* dT, float* dscale, float* dbw, int B,
                               int d_in, int d_out, int n_rows, const RowMap& rm, cudaStream_t st) {
  const Basis<K> bas = make_basis<K>(K - 1);
  const int n_os = (d_out + 31) / 32;
  const int64_t units = (int64_t)((n_rows + 31) / 32) * n_os;
  if (units == 0) return UKAN_OK;
  const size_t smem = sizeof(double) * 8 * (size_t)tan_warp_doubles<K>();
  UKAN_CUDA_TRY(cudaFuncSetAttribute(jvp_dtable_kernel<K, UKAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  jvp_dtable_kernel<K, UKAN><<<(unsigned)((units + 7) / 8), 256, smem, st>>>(x, tx, scale, gt, dT, B, d_in, d_out,
                                                                             n_rows, n_os, rm, bas);
  UKAN_LAUNCH_CHECK();
  jvp_dscale_kernel<K, UKAN><<<dim3((unsigned)d_in, (unsigned)((d_out + 255) / 256)), 256, 0, st>>>(
      x, tx, T, gt, dscale, dbw, B, d_in, d_out, rm, bas);
  UKAN_LAUNCH_CHECK();
  if (dx || dtx) {
    const int64_t pairs = (int64_t)B * d_in;
    jvp_dinput_kernel<K, UKAN><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, tx, T, scale, bw, gt, dx, dtx, B,
                                                                            d_in, d_out, rm, bas);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

static int jvp_kan_args(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, double g_min, double g_max) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(g_min < g_max) || G < 1) return UKAN_E_GRID;
  if (B < 0 || d_in < 1 || d_out < 1 || B > INT32_MAX || d_in * (G + k) * d_out >= ((int64_t)1 << 40) ||
      d_in * (G + k) >= ((int64_t)1 << 31))
    return UKAN_E_ARG;
  return UKAN_OK;
}

}  // namespace ukan

using namespace ukan;

extern "C" int ukan_kan_jvp_forward(const float* x, const float* tx, const float* coeffs, const float* scale,
                                    const float* base_weight, float* ty, int64_t B, int64_t d_in, int64_t d_out,
                                    int64_t G, int k, double g_min, double g_max, void* stream) {
  int rc = jvp_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  if (!coeffs || !scale || (B > 0 && (!x || !tx || !ty))) return UKAN_E_ARG;
  if (B == 0) return UKAN_OK;
  RowMap rm{};
  rm.grid = make_kan_grid(g_min, g_max, G);
  rm.R = (int)(G + k);
  cudaStream_t st = (cudaStream_t)stream;
  UKAN_DISPATCH_K(k, return jvp_forward_launch<K, false>(x, tx, coeffs, scale, base_weight, ty, B, (int)d_in, (int)d_out, rm, st););
  return UKAN_OK;
}

extern "C" int ukan_kan_jvp_backward(const float* x, const float* tx, const float* coeffs, const float* scale,
                                     const float* base_weight, const float* gt, float* dx, float* dtx,
                                     float* dcoeffs, float* dscale, float* dbase_weight, int64_t B, int64_t d_in,
                                     int64_t d_out, int64_t G, int k, double g_min, double g_max, void* stream) {
  int rc = jvp_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  if (!coeffs || !scale || !dcoeffs || !dscale || (B > 0 && (!x || !tx || !gt))) return UKAN_E_ARG;
  if ((base_weight == nullptr) != (dbase_weight == nullptr)) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (B == 0) {
    UKAN_CUDA_TRY(cudaMemsetAsync(dcoeffs, 0, sizeof(float) * d_in * (G + k) * d_out, st));
    UKAN_CUDA_TRY(cudaMemsetAsync(dscale, 0, sizeof(float) * d_in * d_out, st));
    if (dbase_weight) UKAN_CUDA_TRY(cudaMemsetAsync(dbase_weight, 0, sizeof(float) * d_in * d_out, st));
    return UKAN_OK;
  }
  RowMap rm{};
  rm.grid = make_kan_grid(g_min, g_max, G);
  rm.R = (int)(G + k);
  const int n_rows = (int)(d_in * (G + k));
  UKAN_DISPATCH_K(k, return jvp_backward_launch<K, false>(x, tx, coeffs, scale, base_weight, gt, dx, dtx, dcoeffs, dscale, dbase_weight, (int)B, (int)d_in, (int)d_out, n_rows, rm, st););
  return UKAN_OK;
}

extern "C" int ukan_ukan_jvp_forward(const float* x, const float* tx, const int32_t* base_row, const float* table,
                                     const float* scale, float* ty, int64_t B, int64_t d_in, int64_t d_out, int k,
                                     double delta_g, void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!table || !scale || B < 0 || d_in < 1 || d_out < 1 || B > INT32_MAX ||
      (B > 0 && (!x || !tx || !ty || !base_row)))
    return UKAN_E_ARG;
  if (B == 0) return UKAN_OK;
  RowMap rm{};
  rm.inv_dg = 1.0 / delta_g;  // layers.py:261
  rm.base_row = base_row;
  rm.K = k + 1;
  cudaStream_t st = (cudaStream_t)stream;
  UKAN_DISPATCH_K(k, return jvp_forward_launch<K, true>(x, tx, table, scale, nullptr, ty, B, (int)d_in, (int)d_out, rm, st););
  return UKAN_OK;
}

extern "C" int ukan_ukan_jvp_backward(const float* x, const float* tx, const int32_t* base_row,
                                      const int32_t* seg_start, const float* table, const float* scale,
                                      const float* gt, float* dx, float* dtx, float* dtable, float* dscale,
                                      int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int k, double delta_g,
                                      void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!table || !scale || !dtable || !dscale || B < 0 || d_in < 1 || d_out < 1 || n_u < 0 || B > INT32_MAX ||
      n_u * (k + 1) >= ((int64_t)1 << 31) || (B > 0 && (!x || !tx || !gt || !base_row || !seg_start)))
    return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (B == 0) {
    UKAN_CUDA_TRY(cudaMemsetAsync(dtable, 0, sizeof(float) * n_u * (k + 1) * d_out, st));
    UKAN_CUDA_TRY(cudaMemsetAsync(dscale, 0, sizeof(float) * d_in * d_out, st));
    return UKAN_OK;
  }
  RowMap rm{};
  rm.inv_dg = 1.0 / delta_g;
  rm.base_row = base_row;
  rm.seg_start = seg_start;
  rm.K = k + 1;
  const int n_rows = (int)(n_u * (k + 1));
  UKAN_DISPATCH_K(k, return jvp_backward_launch<K, true>(x, tx, table, scale, nullptr, gt, dx, dtx, dtable, dscale, nullptr, (int)B, (int)d_in, (int)d_out, n_rows, rm, st););
  return UKAN_OK;
}
