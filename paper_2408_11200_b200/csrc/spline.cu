// spline.cu — matrix-form B-spline layer kernels shared by KAN and UKAN.
//
// Reference path (float64 NumPy, /root/reference/pkg/src/ukan/layers.py):
//   KAN  kan_forward 304-318 = _kan_locate 294-301 -> span_gather 57-75 -> basis_features 40-54
//        -> edge_combine 78-105 (+ base branch 316-317)
//   UKAN ukan_forward 254-291: same span_gather/basis_features/edge_combine over the
//        generator's coefficient table, rows/cols from 284-287.
//   backward = the bwd closures 44-46, 67-70, 84-88 (+ clamp tensor.py:327-338 for KAN).
//
// Both layers evaluate  y[b,o] = sum_i scale[i,o] * sum_j w_j(u_bi) * T[row_bi + j, o]
// over a row-major table T[rows, d_out]:
//   KAN : T = coeffs viewed as [d_in*(G+k), d_out], row_bi = i*(G+k) + cell_bi
//   UKAN: T = CG output viewed as [n_u*K, d_out] (slot-major), row_bi = base_row[b,i]; with
//         feature-major key order the K rows of a window are consecutive (see ukan_b200.h).
// Each feature i owns a contiguous row segment [row0_i, row0_i + R_i) of T.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "rowmap.cuh"

namespace ukan {

KanGrid make_kan_grid(double g_min, double g_max, int64_t G) {
  KanGrid g;
  g.g_min = g_min;
  g.hi = nextafter(g_max, g_min);
  g.dg = (g_max - g_min) / (double)G;
  g.inv_dg = 1.0 / g.dg;
  g.gmin_dg = g_min / g.dg;
  g.G = (int)G;
  return g;
}

// ---------------------------------------------------------------------------------------
// Forward.
// CTA tile = Bt samples x Ot outputs; blockDim = (TO, TS); each thread owns S samples x VEC
// consecutive outputs in registers and sweeps all d_in features.  Per stage of FC features
// the CTA computes (fp64 locate, fp64 basis -> fp32 weights) once for its Bt x FC
// (sample, feature) pairs into shared memory; then every thread gathers its K table rows
// with vector loads through the read-only path (the per-feature slab stays L1-resident while
// the CTA works on it) and accumulates, in edge_combine's order,
//   y[b,o] += scale[i,o] * (sum_j w_j * T[row + j, o])                      (fp32)
// ---------------------------------------------------------------------------------------
constexpr int kFwdFC = 8;
constexpr int kFwdS = 4;

template <int K, int VEC, bool UKAN>
__global__ void __launch_bounds__(256, UKAN ? 4 : 2)  // UKAN: the gathers are latency-bound (4 blocks/SM: 5.6 -> 4.4 ms)
spline_fwd_kernel(const float* __restrict__ x, const float* __restrict__ T,
                  const float* __restrict__ scale, const float* __restrict__ bw,
                  float* __restrict__ y, int B, int d_in, int d_out, RowMap rm, Basis<K> bas,
                  int32_t* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int TO = blockDim.x, TS = blockDim.y;
  const int Bt = TS * kFwdS;
  int* row_s = reinterpret_cast<int*>(smem_raw);                 // [FC][Bt]
  float* w_s = reinterpret_cast<float*>(row_s + kFwdFC * Bt);    // [FC][Bt][K]
  float* sl_s = w_s + kFwdFC * Bt * K;                           // [FC][Bt] silu(x)

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * TO + tx, nthr = TO * TS;
  const int b0 = blockIdx.x * Bt;
  const int o = blockIdx.y * (TO * VEC) + tx * VEC;
  const bool o_ok = o < d_out;
  const bool has_base = bw != nullptr;

  float acc[kFwdS][VEC];
#pragma unroll
  for (int r = 0; r < kFwdS; ++r)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[r][v] = 0.f;

  for (int f0 = 0; f0 < d_in; f0 += kFwdFC) {
    __syncthreads();
    for (int p = tid; p < kFwdFC * Bt; p += nthr) {
      const int s = p / kFwdFC, f = p % kFwdFC;
      const int b = b0 + s, i = f0 + f;
      int row = -1;
      if (b < B && i < d_in) {
        const float xv = x[(size_t)b * d_in + i];
        double u;
        bool mask;
        if (!locate_row<UKAN>(rm, xv, b, i, d_in, row, u, mask)) {
          if (err) atomicExch(err, 1);
          row = UKAN ? row : i * rm.R;
          u = 0.0;
        }
        double w[K];
        basis_weights<K>(bas, u, w);
#pragma unroll
        for (int j = 0; j < K; ++j) w_s[(f * Bt + s) * K + j] = (float)w[j];
        if (has_base) sl_s[f * Bt + s] = (float)silu_d((double)xv);
      }
      row_s[f * Bt + s] = row;
    }
    __syncthreads();
    if (!o_ok) continue;
    const int nf = min(kFwdFC, d_in - f0);
    for (int f = 0; f < nf; ++f) {
      const int i = f0 + f;
      float sc[VEC], bv[VEC];
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        sc[v] = __ldg(scale + (size_t)i * d_out + o + v);
        bv[v] = has_base ? __ldg(bw + (size_t)i * d_out + o + v) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < kFwdS; ++r) {
        const int s = ty + TS * r;
        const int row = row_s[f * Bt + s];
        if (row < 0) continue;
        const float* rp = T + (size_t)row * d_out + o;
        float tmp[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) tmp[v] = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const float wj = w_s[(f * Bt + s) * K + j];
          const float* q = rp + (size_t)j * d_out;
          if constexpr (VEC == 4) {  // packed FFMA2: bitwise equal to four fmaf
            const float4 cv = __ldg(reinterpret_cast<const float4*>(q));
            const float2 w2 = make_float2(wj, wj);
            const float2 t01 = __ffma2_rn(w2, make_float2(cv.x, cv.y), make_float2(tmp[0], tmp[1]));
            const float2 t23 = __ffma2_rn(w2, make_float2(cv.z, cv.w), make_float2(tmp[2], tmp[3]));
            tmp[0] = t01.x;
            tmp[1] = t01.y;
            tmp[2] = t23.x;
            tmp[3] = t23.y;
          } else if constexpr (VEC == 2) {
            const float2 cv = __ldg(reinterpret_cast<const float2*>(q));
            tmp[0] = fmaf(wj, cv.x, tmp[0]);
            tmp[1] = fmaf(wj, cv.y, tmp[1]);
          } else {
            tmp[0] = fmaf(wj, __ldg(q), tmp[0]);
          }
        }
        const float sl = has_base ? sl_s[f * Bt + s] : 0.f;
        if constexpr (VEC == 4) {
          if (!has_base) {
            const float2 a01 = __ffma2_rn(make_float2(sc[0], sc[1]), make_float2(tmp[0], tmp[1]), make_float2(acc[r][0], acc[r][1]));
            const float2 a23 = __ffma2_rn(make_float2(sc[2], sc[3]), make_float2(tmp[2], tmp[3]), make_float2(acc[r][2], acc[r][3]));
            acc[r][0] = a01.x;
            acc[r][1] = a01.y;
            acc[r][2] = a23.x;
            acc[r][3] = a23.y;
            continue;
          }
        }
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          acc[r][v] = fmaf(sc[v], tmp[v], acc[r][v]);
          if (has_base) acc[r][v] = fmaf(sl, bv[v], acc[r][v]);
        }
      }
    }
  }
  if (!o_ok) return;
#pragma unroll
  for (int r = 0; r < kFwdS; ++r) {
    const int b = b0 + ty + TS * r;
    if (b >= B) continue;
    float* yr = y + (size_t)b * d_out + o;
#pragma unroll
    for (int v = 0; v < VEC; ++v) yr[v] = acc[r][v];
  }
}

// ---------------------------------------------------------------------------------------
// Warp-level bitonic sort of 32*P int keys held P per lane (element e = lane*P + q).
// ---------------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void warp_bitonic_sort(int (&a)[P], int lane) {
  constexpr int N = 32 * P;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= P) {
        const int lm = j / P;
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const int e = lane * P + q;
          const int other = __shfl_xor_sync(0xffffffffu, a[q], lm);
          const bool lower = (e & j) == 0;
          const bool asc = (e & k) == 0;
          a[q] = (lower == asc) ? min(a[q], other) : max(a[q], other);
        }
      } else {
#pragma unroll
        for (int q = 0; q < P; ++q) {
          if ((q & j) == 0) {
            const int q2 = q | j;
            const int e = lane * P + q;
            const bool asc = (e & k) == 0;
            const int lo = min(a[q], a[q2]), hi = max(a[q], a[q2]);
            a[q] = asc ? lo : hi;
            a[q2] = asc ? hi : lo;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Backward, table side:  A[row, o] = sum_{(b,j): row_bi + j = row} w_j(b,i) * g[b,o]
//   dT = scale * A,  dscale = sum_rows T * A,  dbw = sum_b silu(x) * g   (KAN base branch).
// One warp per feature i, lanes over OV consecutive outputs; a CTA holds FT features and
// sweeps the whole batch in chunks of BC samples, so each (row, o) is owned by exactly one
// thread: no atomics, fixed summation order -> deterministic.  Per chunk the warp sorts its
// BC samples by (row, sample) with a register bitonic network and streams them in row order
// through a sliding window of K fp64 register accumulators; a row leaving the window is
// added into the fp64 accumulator A (shared memory when the feature's segment fits, a
// global fp64 workspace otherwise).  Products are fp64 basis weights x exactly-upcast fp32
// g, accumulated in fp64.
// ---------------------------------------------------------------------------------------
constexpr int kBwdBC = 128;

template <int K, int OV, bool A_SMEM, bool UKAN>
__global__ void __launch_bounds__(256, 2)
spline_bwd_table_kernel(const float* __restrict__ x, const float* __restrict__ T,
                        const float* __restrict__ scale, const float* __restrict__ gy,
                        float* __restrict__ dT, float* __restrict__ dscale,
                        float* __restrict__ dbw, double* __restrict__ A_glob, int B, int d_in,
                        int d_out, int R_smem, RowMap rm, Basis<K> bas) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int OT = 32 * OV;
  constexpr int P = kBwdBC / 32;
  const int FT = blockDim.x / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i = blockIdx.x * FT + warp;
  const int o0 = blockIdx.y * OT;
  const bool has_base = dbw != nullptr;

  unsigned char* p = smem_raw;
  double* A_s = reinterpret_cast<double*>(p);  // [FT][R_smem][OT]
  if (A_SMEM) p += sizeof(double) * (size_t)FT * R_smem * OT;
  double* w_s = reinterpret_cast<double*>(p);  // [FT][BC][K]
  p += sizeof(double) * FT * kBwdBC * K;
  double* sl_s = reinterpret_cast<double*>(p);  // [FT][BC]
  p += sizeof(double) * FT * kBwdBC;
  float* g_s = reinterpret_cast<float*>(p);  // [BC][OT]
  p += sizeof(float) * kBwdBC * OT;
  int* ent_s = reinterpret_cast<int*>(p);  // [FT][BC]  (local_row << 8 | s)

  const bool active = i < d_in;
  int row0 = 0, nrows = 0;
  if (active) feature_rows<UKAN>(rm, i, row0, nrows);
  double* A = A_SMEM ? A_s + (size_t)warp * R_smem * OT : A_glob + (size_t)row0 * d_out;
  const int a_stride = A_SMEM ? OT : d_out;
  const int a_col = A_SMEM ? lane * OV : o0 + lane * OV;
  bool ovalid[OV];
#pragma unroll
  for (int v = 0; v < OV; ++v) ovalid[v] = (o0 + lane * OV + v) < d_out;

  if (active) {
    for (int r = 0; r < nrows; ++r)
#pragma unroll
      for (int v = 0; v < OV; ++v)
        if (A_SMEM || ovalid[v]) A[(size_t)r * a_stride + a_col + v] = 0.0;
  }
  double bacc[OV];
#pragma unroll
  for (int v = 0; v < OV; ++v) bacc[v] = 0.0;

  int* ent = ent_s + warp * kBwdBC;
  double* wsw = w_s + (size_t)warp * kBwdBC * K;
  double* slw = sl_s + warp * kBwdBC;

  for (int b0 = 0; b0 < B; b0 += kBwdBC) {
    const int nb = min(kBwdBC, B - b0);
    __syncthreads();  // previous chunk fully consumed
    for (int t = threadIdx.x; t < kBwdBC * OT; t += blockDim.x) {
      const int s = t / OT, oc = t % OT;
      float gv = 0.f;
      if (s < nb && o0 + oc < d_out) gv = gy[(size_t)(b0 + s) * d_out + o0 + oc];
      g_s[t] = gv;
    }
    if (active) {
      int keys[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const int s = lane * P + q;
        int key = INT_MAX;
        if (s < nb) {
          const float xv = x[(size_t)(b0 + s) * d_in + i];
          int row;
          double u;
          bool mask;
          locate_row<UKAN>(rm, xv, b0 + s, i, d_in, row, u, mask);
          double w[K];
          basis_weights<K>(bas, u, w);
#pragma unroll
          for (int j = 0; j < K; ++j) wsw[s * K + j] = w[j];
          if (has_base) slw[s] = silu_d((double)xv);
          key = ((row - row0) << 8) | s;
        }
        keys[q] = key;
      }
      warp_bitonic_sort<P>(keys, lane);
#pragma unroll
      for (int q = 0; q < P; ++q) ent[lane * P + q] = keys[q];
    }
    __syncthreads();  // g_s staged, entries sorted
    if (!active) continue;

    double acc[K][OV];
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int v = 0; v < OV; ++v) acc[j][v] = 0.0;
    int cur = -1;
    for (int e = 0; e < nb; ++e) {
      const int pk = ent[e];
      const int c = pk >> 8, s = pk & 255;
      if (c != cur) {
        if (cur >= 0) {
          const int d = c - cur;
#pragma unroll
          for (int t = 0; t < K; ++t) {
            if (t < d) {
              if (cur + t < nrows) {
#pragma unroll
                for (int v = 0; v < OV; ++v)
                  if (A_SMEM || ovalid[v]) A[(size_t)(cur + t) * a_stride + a_col + v] += acc[0][v];
              }
#pragma unroll
              for (int jj = 0; jj < K - 1; ++jj)
#pragma unroll
                for (int v = 0; v < OV; ++v) acc[jj][v] = acc[jj + 1][v];
#pragma unroll
              for (int v = 0; v < OV; ++v) acc[K - 1][v] = 0.0;
            }
          }
        }
        cur = c;
      }
      double gv[OV];
#pragma unroll
      for (int v = 0; v < OV; ++v) gv[v] = (double)g_s[s * OT + lane * OV + v];
      const double* we = wsw + s * K;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const double wj = we[j];
#pragma unroll
        for (int v = 0; v < OV; ++v) acc[j][v] = fma(wj, gv[v], acc[j][v]);
      }
      if (has_base) {
        const double sl = slw[s];
#pragma unroll
        for (int v = 0; v < OV; ++v) bacc[v] = fma(sl, gv[v], bacc[v]);
      }
    }
    if (cur >= 0) {
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (cur + t < nrows)
#pragma unroll
          for (int v = 0; v < OV; ++v)
            if (A_SMEM || ovalid[v]) A[(size_t)(cur + t) * a_stride + a_col + v] += acc[t][v];
    }
  }
  if (!active) return;
  __syncwarp();
#pragma unroll
  for (int v = 0; v < OV; ++v) {
    const int o = o0 + lane * OV + v;
    if (!ovalid[v]) continue;
    const double sc = (double)scale[(size_t)i * d_out + o];
    double ds = 0.0;
    for (int r = 0; r < nrows; ++r) {
      const double a = A[(size_t)r * a_stride + a_col + v];
      const size_t ti = (size_t)(row0 + r) * d_out + o;
      dT[ti] = (float)(sc * a);
      ds = fma((double)T[ti], a, ds);
    }
    dscale[(size_t)i * d_out + o] = (float)ds;
    if (has_base) dbw[(size_t)i * d_out + o] = (float)bacc[v];
  }
}

// ---------------------------------------------------------------------------------------
// Backward, input side:
//   dx[b,i] = mask * inv_dg * sum_j w'_j * sum_o g[b,o]*scale[i,o]*T[row+j,o]
//             (+ dsilu(x) * sum_o g[b,o]*bw[i,o])                               (KAN)
// (UKAN: u = x*inv_dg - g_id, so du/dx = inv_dg and there is no clamp mask.)
// One warp per (b, i), lanes over d_out, fp64 products/accumulators, shuffle reduction.
// ---------------------------------------------------------------------------------------
template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
spline_dx_kernel(const float* __restrict__ x, const float* __restrict__ T,
                 const float* __restrict__ scale, const float* __restrict__ bw,
                 const float* __restrict__ gy, float* __restrict__ dx, int B, int d_in,
                 int d_out, RowMap rm, Basis<K> bas) {
  const int lane = threadIdx.x % 32;
  const int64_t pair = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (pair >= (int64_t)B * d_in) return;
  // feature-major: the warps resident at any time share a few features' table rows, so the
  // gathers hit L2 even when the whole table (UKAN: n_u*K rows) is far larger than L2
  const int i = (int)(pair / B), b = (int)(pair % B);
  const float xv = x[(size_t)b * d_in + i];
  int row;
  double u;
  bool mask;
  locate_row<UKAN>(rm, xv, b, i, d_in, row, u, mask);
  double wp[K];
  basis_dweights<K>(bas, u, wp);
  double S[K];
#pragma unroll
  for (int j = 0; j < K; ++j) S[j] = 0.0;
  double sb = 0.0;
  const float* Ti = T + (size_t)row * d_out;
  const float* gr = gy + (size_t)b * d_out;
  for (int o = lane; o < d_out; o += 32) {
    const double g = (double)gr[o];
    const double gs = g * (double)scale[(size_t)i * d_out + o];
#pragma unroll
    for (int j = 0; j < K; ++j) S[j] = fma(gs, (double)Ti[(size_t)j * d_out + o], S[j]);
    if (bw) sb = fma(g, (double)bw[(size_t)i * d_out + o], sb);
  }
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) t = fma(S[j], wp[j], t);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, off);
    sb += __shfl_xor_sync(0xffffffffu, sb, off);
  }
  if (lane == 0) {
    const double inv = UKAN ? rm.inv_dg : rm.grid.inv_dg;
    double d = mask ? t * inv : 0.0;
    if (bw) d += dsilu_d((double)xv) * sb;
    dx[(size_t)b * d_in + i] = (float)d;
  }
}

// Same dx with g and scale pre-widened to fp64 (one conversion per element per backward instead
// of one per (sample, feature, output)): F2F.F64.F32 issues at 1/4 of the DFMA rate, so the
// per-output conversions of g and scale bound the plain kernel on wide layers.  No base branch.
__global__ void cvt_f64_kernel(const float* __restrict__ in, double* __restrict__ out, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = (double)in[t];
}

template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
spline_dx64_kernel(const float* __restrict__ x, const float* __restrict__ T, const double* __restrict__ s64,
                   const double* __restrict__ g64, float* __restrict__ dx, int B, int d_in, int d_out, RowMap rm,
                   Basis<K> bas) {
  const int lane = threadIdx.x % 32;
  const int64_t pair = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (pair >= (int64_t)B * d_in) return;
  // feature-major inside blocks of 4096 samples: the block's fp64 g rows (32 MB at d_out = 1024)
  // stay in L2 while every feature passes over them, instead of all B rows being re-read from DRAM
  // once per feature (cfg4 at B = 65536: 537 GB of g reads per call)
  constexpr int kBlk = 4096;
  const int64_t blk = (int64_t)kBlk * d_in;
  const int64_t sb = pair / blk, rem = pair % blk;
  const int nb = (int)min((int64_t)kBlk, (int64_t)B - sb * kBlk);
  const int i = (int)(rem / nb), b = (int)(sb * kBlk + rem % nb);
  const float xv = x[(size_t)b * d_in + i];
  int row;
  double u;
  bool mask;
  locate_row<UKAN>(rm, xv, b, i, d_in, row, u, mask);
  double wp[K];
  basis_dweights<K>(bas, u, wp);
  double S[K];
#pragma unroll
  for (int j = 0; j < K; ++j) S[j] = 0.0;
  const float* Ti = T + (size_t)row * d_out;
  const double* gr = g64 + (size_t)b * d_out;
  const double* sr = s64 + (size_t)i * d_out;
  for (int o = lane; o < d_out; o += 32) {
    const double gs = gr[o] * sr[o];  // exact: a product of two fp32 values
#pragma unroll
    for (int j = 0; j < K; ++j) S[j] = fma(gs, (double)Ti[(size_t)j * d_out + o], S[j]);
  }
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) t = fma(S[j], wp[j], t);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  if (lane == 0) {
    const double inv = UKAN ? rm.inv_dg : rm.grid.inv_dg;
    dx[(size_t)b * d_in + i] = (float)(mask ? t * inv : 0.0);
  }
}

__global__ void kan_locate_kernel(const float* __restrict__ x, int32_t* __restrict__ cell,
                                  double* __restrict__ u, int64_t n, KanGrid grid) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int c;
  double uu;
  bool mask;
  kan_locate(x[t], grid, c, uu, mask);
  cell[t] = c;
  u[t] = uu;
}

// ---------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------
struct RegPlan {
  bool ok = false;
  int rmax = 0, ov = 1, fpb = 1, wpf = 1, S = 1, sps = 0;
  size_t smem = 0;
  int64_t ws_bytes = 0;
};
RegPlan kan_bwd_reg_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base, int sms);
template <int K>
int kan_bwd_reg_dispatch(const float* x, const float* C, const float* scale, const float* gy, float* dC,
                         float* dscale, float* dbw, double* ws, int B, int d_in, int d_out, int R,
                         const KanGrid& grid, const RegPlan& p, cudaStream_t st);
template <int K>
int kan_dx_narrow(const float* x, const float* C, const float* scale, const float* bw, const float* gy, float* dx,
                  int B, int d_in, int d_out, int R, const KanGrid& grid, cudaStream_t st);
int kan_num_sms();
struct TcPlan {
  bool ok = false;
  int rb = 0, nt = 4, S = 1, cps = 0, nch = 0, fpb = 4, wpf = 2;
  bool split = false;
  size_t smem = 0;
  int64_t rec_bytes = 0, part_bytes = 0;
};
TcPlan kan_bwd_tc_plan(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base);
int64_t kan_bwd_tc_workspace(const TcPlan& p);
int kan_bwd_tc_run(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                   void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int G, const KanGrid& grid,
                   const TcPlan& p, cudaStream_t st, bool prepared);
int kan_bwd_tc_prep(const float* x, void* workspace, int64_t ws_bytes, int B, int d_in, int G, const KanGrid& grid,
                    const TcPlan& p, cudaStream_t st);
bool kan_dx_tc_applicable(const TcPlan& p, const float* C, const float* gy, int d_out, int G);
int kan_bwd_tc_part(const float* C, const float* scale, const float* gy, float* dx, float* dC, float* dscale,
                    void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int G, const KanGrid& grid,
                    int64_t i_lo, int64_t i_hi, int what, cudaStream_t st);
int kan_dx_tc_run(const float* C, const float* scale, const float* gy, float* dx, void* workspace, int B, int d_in,
                  int d_out, int G, const KanGrid& grid, const TcPlan& p, cudaStream_t st);
bool kan_bwd_dmma_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base, int sms, RegPlan& p);
int kan_bwd_dmma_dispatch(const float* x, const float* C, const float* scale, const float* gy, float* dC,
                          float* dscale, double* ws, int B, int d_in, int d_out, int R, const KanGrid& grid,
                          const RegPlan& p, cudaStream_t st);
struct SwPlan {
  bool ok = false;
  int rm = 0, ov = 1, Z = 1, sps = 0, d_pad = 0;
  size_t smem = 0;
  int64_t g64_bytes = 0, part_bytes = 0;
};
SwPlan kan_bwd_sw_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base);
int64_t kan_bwd_sw_workspace(const SwPlan& p);
template <int K>
int kan_bwd_sw_run(const float* x, const float* gy, const float* C, const float* scale, float* dC, float* dscale,
                   float* dbw, void* ws, int B, int d_in, int d_out, int R, const KanGrid& grid, const SwPlan& p,
                   cudaStream_t st);
struct TmPlan {
  bool ok = false;
  int RP = 0, fpc = 0, S = 1, n_ot = 0, Bp = 0;
  size_t smem = 0;
  int64_t pack_bytes = 0, rec_bytes = 0, part_bytes = 0;
  int depth = 5, db = 1;
};
TmPlan kan_fwd_tm_plan(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base);
// kan_small.cu: small layers (d_in * d_out <= 2^14, k = 3, no base branch)
bool kan_small_ok(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base);
int64_t kan_small_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t G);
// kan_bwd_tc.cu: dense UKAN layers on the KAN tensor-core backward
int64_t ukan_dense_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t max_rows, int k);
int ukan_dense_backward(const float* x, const int32_t* base_row, const int32_t* seg, const float* T,
                        const float* scale, const float* gy, float* dx, float* dT, float* dscale, int B, int d_in,
                        int d_out, int64_t max_rows, double delta_g, void* ws, int64_t ws_bytes, cudaStream_t st,
                        bool table);
int kan_small_forward(const float* x, const float* C, const float* scale, float* y, int B, int d_in, int d_out, int G,
                      const KanGrid& grid, int32_t* err, cudaStream_t st);
int kan_small_records(const float* x, void* ws, int B, int d_in, const KanGrid& grid, cudaStream_t st);
int kan_small_tablegrad(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                        void* ws, int B, int d_in, int d_out, int G, const KanGrid& grid, bool prepared,
                        cudaStream_t st);
int64_t kan_fwd_tm_workspace(const TmPlan& p);
int kan_fwd_tm_run_ukan(const float* x, const float* T, const float* scale, float* y, void* ws, int64_t ws_bytes,
                        int B, int d_in, int d_out, int G, double inv_dg, const int32_t* base_row, const int32_t* seg,
                        const TmPlan& p, cudaStream_t st);
template <int K>
int kan_fwd_tm_run(const float* x, const float* C, const float* scale, float* y, void* ws, int64_t ws_bytes, int B,
                   int d_in, int d_out, int R, const KanGrid& grid, const TmPlan& p, int32_t* err, cudaStream_t st);
template <int K>
int kan_fwd_narrow(const float* x, const float* C, const float* scale, const float* bw, float* y, int B, int d_in,
                   int d_out, int R, const KanGrid& grid, int32_t* err, cudaStream_t st);
template <int K>
int kan_dx_narrow2(const float* x, const float* C, const float* scale, const float* bw, const float* gy, float* dx,
                   int B, int d_in, int d_out, int R, const KanGrid& grid, cudaStream_t st);
struct WidePlan {
  bool ok = false;
  int n_rt = 0, n_os = 0, nch = 0, st_n = 0;
  size_t recb = 0;
  int64_t rec_bytes = 0, part_bytes = 0;
};
WidePlan kan_bwd_wide_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K);
int64_t kan_bwd_wide_workspace(const WidePlan& p);
template <int K>
int kan_bwd_wide_run(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                     float* dbw, void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int R,
                     const KanGrid& grid, const WidePlan& p, cudaStream_t st);
int64_t seg_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t total_rows);
bool seg_uses_sorted(int B, int64_t total_rows, int64_t max_rows_hint);
int seg_dx_sorted(const float* T, const double* s64, const double* g64, float* dx, void* ws, int B, int d_in,
                  int d_out, int64_t total_rows, const RowMap& rm, cudaStream_t st);
bool seg_supported(int64_t B, int64_t d_out);
template <int K, bool UKAN>
int seg_table_grad(const float* x, const float* T, const float* scale, const float* gy, float* dT, float* dscale,
                   void* ws, int64_t ws_bytes, int B, int d_in, int d_out, int64_t total_rows, const RowMap& rm,
                   cudaStream_t st,
                   int64_t max_rows_hint = 0);
template <int K>
int kan_fwd_v2(const float* x, const float* C, const float* scale, const float* bw, float* y, int B, int d_in,
               int d_out, int R, const KanGrid& grid, int32_t* err, cudaStream_t st);

constexpr size_t kSmemCap = 220 * 1024;
constexpr int kBwdOV = 2;

static size_t bwd_smem_bytes(int K, int FT, int OT, int R, bool a_smem) {
  size_t s = 0;
  if (a_smem) s += sizeof(double) * (size_t)FT * R * OT;
  s += sizeof(double) * FT * kBwdBC * K;
  s += sizeof(double) * FT * kBwdBC;
  s += sizeof(float) * kBwdBC * OT;
  s += sizeof(int) * FT * kBwdBC;
  return s;
}

static bool bwd_fits_smem(int K, int R) { return bwd_smem_bytes(K, 1, 32 * kBwdOV, R, true) <= kSmemCap; }

template <int K, bool UKAN>
static int launch_fwd(const float* x, const float* T, const float* scale, const float* bw,
                      float* y, int B, int d_in, int d_out, const RowMap& rm, int32_t* err,
                      cudaStream_t st) {
  if constexpr (!UKAN) {
    // smem-slab variant (kan_fwd.cu): measured slower than this kernel at cfg2 (1.88 vs 1.68 ms,
    // profiles/README.md), kept selectable for experiments via UKAN_FWD_V2=1
    static const bool use_v2 = getenv("UKAN_FWD_V2") != nullptr;
    if (use_v2) {
      const int rc = kan_fwd_v2<K>(x, T, scale, bw, y, B, d_in, d_out, rm.R, rm.grid, err, st);
      if (rc != UKAN_E_ARG) return rc;
    }
  }
  const Basis<K> bas = make_basis<K>(K - 1);
  const int VEC = (d_out % 4 == 0) ? 4 : (d_out % 2 == 0 ? 2 : 1);
  int TO = (d_out + VEC - 1) / VEC;
  if (TO > 32) TO = 32;
  int TS = 256 / TO;
  if (TS > 64) TS = 64;
  {  // narrow layers: shrink the sample tile so the grid still covers ~2 waves
    const int64_t otiles = (d_out + TO * VEC - 1) / (TO * VEC);
    const int64_t want = 2 * (int64_t)kan_num_sms();
    const int64_t ts_fit = ((int64_t)B + kFwdS * (want / otiles) - 1) / std::max<int64_t>(1, kFwdS * (want / otiles));
    if (ts_fit < TS) TS = (int)std::max<int64_t>(1, ts_fit);
  }
  const int Bt = TS * kFwdS;
  dim3 block(TO, TS);
  dim3 gridd((B + Bt - 1) / Bt, (d_out + TO * VEC - 1) / (TO * VEC));
  const size_t smem = (size_t)kFwdFC * Bt * (sizeof(int) + sizeof(float) * (K + 1));
  auto kern = VEC == 4 ? spline_fwd_kernel<K, 4, UKAN>
                       : (VEC == 2 ? spline_fwd_kernel<K, 2, UKAN> : spline_fwd_kernel<K, 1, UKAN>);
  if (smem > 48 * 1024)
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<gridd, block, smem, st>>>(x, T, scale, bw, y, B, d_in, d_out, rm, bas, err);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

template <int K, bool UKAN>
static int launch_bwd(const float* x, const float* T, const float* scale, const float* bw,
                      const float* gy, float* dx, float* dT, float* dscale, float* dbw,
                      double* A_glob, int B, int d_in, int d_out, int R_max, const RowMap& rm,
                      cudaStream_t st) {
  const Basis<K> bas = make_basis<K>(K - 1);
  constexpr int OV = kBwdOV;
  constexpr int OT = 32 * OV;
  int FT = 8;
  bool a_smem = true;
  while (FT > 1 && bwd_smem_bytes(K, FT, OT, R_max, true) > kSmemCap) FT >>= 1;
  if (bwd_smem_bytes(K, FT, OT, R_max, true) > kSmemCap) {
    a_smem = false;
    FT = 8;
    if (A_glob == nullptr) return UKAN_E_WORKSPACE;
  }
  const size_t smem = bwd_smem_bytes(K, FT, OT, R_max, a_smem);
  dim3 gridd((d_in + FT - 1) / FT, (d_out + OT - 1) / OT);
  if (a_smem) {
    auto kern = spline_bwd_table_kernel<K, OV, true, UKAN>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<gridd, FT * 32, smem, st>>>(x, T, scale, gy, dT, dscale, dbw, nullptr, B, d_in, d_out, R_max, rm, bas);
  } else {
    auto kern = spline_bwd_table_kernel<K, OV, false, UKAN>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<gridd, FT * 32, smem, st>>>(x, T, scale, gy, dT, dscale, dbw, A_glob, B, d_in, d_out, 0, rm, bas);
  }
  UKAN_LAUNCH_CHECK();
  if (dx) {
    const int64_t pairs = (int64_t)B * d_in;
    if (pairs > 0) {
      const int wpb = 8;
      spline_dx_kernel<K, UKAN><<<(unsigned)((pairs + wpb - 1) / wpb), wpb * 32, 0, st>>>(
          x, T, scale, bw, gy, dx, B, d_in, d_out, rm, bas);
      UKAN_LAUNCH_CHECK();
    }
  }
  return UKAN_OK;
}

static int check_kan_args(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                          double g_min, double g_max) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(g_min < g_max) || G < 1) return UKAN_E_GRID;
  if (B < 0 || d_in < 1 || d_out < 1) return UKAN_E_ARG;
  if (B > INT32_MAX || d_in * (G + k) >= ((int64_t)1 << 31) || (G + k) >= (1 << 23)) return UKAN_E_ARG;
  return UKAN_OK;
}

}  // namespace ukan

using namespace ukan;

// Forward kernel choice: d_out <= 32 -> lanes-over-samples kernel (kan_narrow.cu); else the
// TMEM-gather kernel (kan_fwd_tm.cu) whenever its plan applies (no base branch, K <= 8,
// G <= 255, (G-1+window)*4 <= 256); the shared-memory gather otherwise.
// UKAN_FWD=smem selects the latter for A/B measurement.
static bool fwd_use_tm() {
  static const char* e = getenv("UKAN_FWD");
  return e == nullptr || e[0] != 's';
}

extern "C" int64_t ukan_kan_forward_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k) {
  if (k < 0 || k > UKAN_MAX_DEGREE || G < 1 || B < 0 || d_in < 1 || d_out < 1) return 0;
  return fwd_use_tm() ? kan_fwd_tm_workspace(kan_fwd_tm_plan(B, d_in, d_out, G, k, false)) : 0;
}

extern "C" int ukan_kan_forward_ws(const float* x, const float* coeffs, const float* scale,
                                   const float* base_weight, float* y, int64_t B, int64_t d_in,
                                   int64_t d_out, int64_t G, int k, double g_min, double g_max,
                                   int32_t* err_flag, void* workspace, int64_t workspace_bytes,
                                   void* stream) {
  int rc = check_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  if (!coeffs || !scale || (B > 0 && (!x || !y))) return UKAN_E_ARG;
  if (B == 0) return UKAN_OK;
  RowMap rm{};
  rm.grid = make_kan_grid(g_min, g_max, G);
  rm.R = (int)(G + k);
  cudaStream_t st = (cudaStream_t)stream;
  if (d_out <= 32 && fwd_use_tm()) {  // narrow layer: lanes over samples (kan_narrow.cu)
    UKAN_DISPATCH_K(k, return kan_fwd_narrow<K>(x, coeffs, scale, base_weight, y, (int)B, (int)d_in, (int)d_out, rm.R, rm.grid, err_flag, st););
  }
  if (fwd_use_tm() && kan_small_ok(B, d_in, d_out, G, k, base_weight != nullptr))  // small layer
    return kan_small_forward(x, coeffs, scale, y, (int)B, (int)d_in, (int)d_out, (int)G, rm.grid, err_flag, st);
  if (base_weight == nullptr && fwd_use_tm()) {
    const TmPlan tp = kan_fwd_tm_plan(B, d_in, d_out, G, k, false);
    if (tp.ok) {
      if (workspace == nullptr || workspace_bytes < kan_fwd_tm_workspace(tp)) return UKAN_E_WORKSPACE;
      UKAN_DISPATCH_K(k, return kan_fwd_tm_run<K>(x, coeffs, scale, y, workspace, workspace_bytes, (int)B, (int)d_in, (int)d_out, rm.R, rm.grid, tp, err_flag, st););
    }
  }
  UKAN_DISPATCH_K(k, return launch_fwd<K, false>(x, coeffs, scale, base_weight, y, (int)B, (int)d_in, (int)d_out, rm, err_flag, st););
  return UKAN_OK;
}

extern "C" int ukan_kan_forward(const float* x, const float* coeffs, const float* scale,
                                const float* base_weight, float* y, int64_t B, int64_t d_in,
                                int64_t d_out, int64_t G, int k, double g_min, double g_max,
                                int32_t* err_flag, void* stream) {
  // Convenience entry without a caller workspace: a stream-ordered allocation (no host sync).
  const int64_t nbytes = base_weight ? 0 : ukan_kan_forward_workspace_size(B, d_in, d_out, G, k);
  void* ws = nullptr;
  if (nbytes > 0) UKAN_CUDA_TRY(scratch_alloc(&ws, (size_t)nbytes, (cudaStream_t)stream));
  const int rc = ukan_kan_forward_ws(x, coeffs, scale, base_weight, y, B, d_in, d_out, G, k, g_min, g_max,
                                     err_flag, ws, nbytes, stream);
  if (ws) cudaFreeAsync(ws, (cudaStream_t)stream);
  return rc;
}

extern "C" int64_t ukan_kan_backward_workspace_size(int64_t B, int64_t d_in, int64_t d_out,
                                                    int64_t G, int k) {
  if (k < 0 || k > UKAN_MAX_DEGREE || G < 1 || B < 0 || d_in < 1 || d_out < 1) return 0;
  const int64_t sm = kan_small_ok(B, d_in, d_out, G, k, false) ? kan_small_workspace(B, d_in, d_out, G) : 0;
  RegPlan dp;
  const bool dm = kan_bwd_dmma_plan(B, d_in, d_out, (int)(G + k), k + 1, false, kan_num_sms(), dp);
  const RegPlan p = kan_bwd_reg_plan(B, d_in, d_out, (int)(G + k), k + 1, true, kan_num_sms());
  const int64_t tc = kan_bwd_tc_workspace(kan_bwd_tc_plan(B, d_in, d_out, G, k, false));
  const int64_t sw = kan_bwd_sw_workspace(kan_bwd_sw_plan(B, d_in, d_out, (int)(G + k), k + 1, true));
  const int64_t wd = kan_bwd_wide_workspace(kan_bwd_wide_plan(B, d_in, d_out, (int)(G + k), k + 1));
  static const bool force_wide = getenv("UKAN_BWD") && getenv("UKAN_BWD")[0] == 'w';
  if ((!p.ok || force_wide) && wd > 0) return std::max<int64_t>(std::max<int64_t>(wd, p.ok ? p.ws_bytes : 0), sm);
  if (p.ok)
    return std::max<int64_t>(std::max<int64_t>(std::max<int64_t>(std::max<int64_t>(p.ws_bytes, dm ? dp.ws_bytes : 0), tc), sw), sm);
  if (bwd_fits_smem(k + 1, (int)(G + k))) return sm;
  return std::max<int64_t>((int64_t)sizeof(double) * d_in * (G + k) * d_out, sm);
}

// A side stream per (host thread, device) to overlap two independent small kernels of one call:
// fork / join through events recorded on the caller's stream, which is also how a stream under
// CUDA-graph capture pulls the side stream into the graph.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream() {
  thread_local SideStream ss[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  SideStream& r = ss[dev];
  if (r.s == nullptr) {
    if (cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming) != cudaSuccess) {
      r.s = nullptr;
      return nullptr;
    }
  }
  return &r;
}

static const char* kan_bwd_selector() {
  static const char* sel_env = getenv("UKAN_BWD");
  return sel_env ? sel_env : "tc";
}

template <int K>
static int kan_backward_impl(const float* x, const float* coeffs, const float* scale, const float* bw,
                             const float* gy, float* dx, float* dC, float* dscale, float* dbw, void* workspace,
                             int64_t workspace_bytes, int B, int d_in, int d_out, const RowMap& rm,
                             cudaStream_t st, bool prepared) {
  // UKAN_BWD selects the table-gradient kernel for A/B measurement ("tc" default: banded DMMA,
  // kan_bwd_tc.cu; "sw": register accumulators, kan_bwd_sw.cu; "dmma", "reg": older variants).
  const char* sel = kan_bwd_selector();
  bool table_done = false;
  if (sel[0] == 's' && B > 0) {
    const SwPlan sp = kan_bwd_sw_plan(B, d_in, d_out, rm.R, K, bw != nullptr);
    if (sp.ok && workspace != nullptr && workspace_bytes >= kan_bwd_sw_workspace(sp)) {
      int rc = kan_bwd_sw_run<K>(x, gy, coeffs, scale, dC, dscale, dbw, workspace, B, d_in, d_out, rm.R, rm.grid,
                                 sp, st);
      if (rc) return rc;
      table_done = true;
    }
  }
  if (table_done) {
    if (dx) {
      if (d_out <= 32) return kan_dx_narrow2<K>(x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm.R, rm.grid, st);
      const Basis<K> bas = make_basis<K>(K - 1);
      const int64_t pairs = (int64_t)B * d_in;
      spline_dx_kernel<K, false><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, coeffs, scale, bw, gy, dx, B, d_in,
                                                                             d_out, rm, bas);
      UKAN_LAUNCH_CHECK();
    }
    return UKAN_OK;
  }
  if (sel[0] == 't' && K == 4 && bw == nullptr && B > 0 && kan_small_ok(B, d_in, d_out, rm.R - K + 1, K - 1, false) &&
      workspace != nullptr && workspace_bytes >= kan_small_workspace(B, d_in, d_out, rm.R - K + 1)) {
    // small layer (kan_small.cu): table gradient over >= 256 CTAs, dx by the per-pair kernel
    int rc = kan_small_tablegrad(x, coeffs, scale, gy, dC, dscale, workspace, B, d_in, d_out, rm.R - K + 1, rm.grid,
                                 prepared, st);
    if (rc) return rc;
    if (dx) {
      const Basis<K> bas = make_basis<K>(K - 1);
      const int64_t pairs = (int64_t)B * d_in;
      spline_dx_kernel<K, false><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, coeffs, scale, bw, gy, dx, B, d_in,
                                                                             d_out, rm, bas);
      UKAN_LAUNCH_CHECK();
    }
    return UKAN_OK;
  }
  if (sel[0] == 't' && K == 4 && bw == nullptr && B > 0) {  // FP64 tensor-core path (kan_bwd_tc.cu)
    const TcPlan tp = kan_bwd_tc_plan(B, d_in, d_out, rm.R - K + 1, K - 1, false);
    if (tp.ok && workspace != nullptr && workspace_bytes >= kan_bwd_tc_workspace(tp)) {
      SideStream* ss = (dx && d_out <= 32) ? side_stream() : nullptr;
      if (ss) {  // narrow layer: dx (independent of the table gradient) on the side stream
        UKAN_CUDA_TRY(cudaEventRecord(ss->fork, st));
        UKAN_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
        int rc = kan_dx_narrow2<K>(x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm.R, rm.grid, ss->s);
        if (rc) return rc;
        UKAN_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
      }
      int rc = kan_bwd_tc_run(x, coeffs, scale, gy, dC, dscale, workspace, workspace_bytes, B, d_in, d_out,
                              rm.R - K + 1, rm.grid, tp, st, prepared);
      if (ss) UKAN_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
      if (rc) return rc;
      if (ss) return UKAN_OK;
      if (dx) {
        if (d_out <= 32) return kan_dx_narrow2<K>(x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm.R, rm.grid, st);
        // wide layers: dx on the FP64 tensor cores from the same sorted records (kan_bwd_tc.cu)
        if (kan_dx_tc_applicable(tp, coeffs, gy, d_out, rm.R - K + 1))
          return kan_dx_tc_run(coeffs, scale, gy, dx, workspace, B, d_in, d_out, rm.R - K + 1, rm.grid, tp, st);
        const Basis<K> bas = make_basis<K>(K - 1);
        const int64_t pairs = (int64_t)B * d_in;
        spline_dx_kernel<K, false><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, coeffs, scale, bw, gy, dx, B, d_in,
                                                                               d_out, rm, bas);
        UKAN_LAUNCH_CHECK();
      }
      return UKAN_OK;
    }
  }
  // Fine grids (R > 72 or K > 6, outside the register sweep) or UKAN_BWD=wide: sorted-chunk
  // sweep whose cost does not grow with G (kan_bwd_wide.cu).
  if (B > 0 && (sel[0] == 'w' || !kan_bwd_reg_plan(B, d_in, d_out, rm.R, K, bw != nullptr, kan_num_sms()).ok)) {
    const WidePlan wp = kan_bwd_wide_plan(B, d_in, d_out, rm.R, K);
    if (wp.ok && workspace != nullptr && workspace_bytes >= kan_bwd_wide_workspace(wp)) {
      int rc = kan_bwd_wide_run<K>(x, coeffs, scale, gy, dC, dscale, dbw, workspace, workspace_bytes, B, d_in, d_out,
                                   rm.R, rm.grid, wp, st);
      if (rc) return rc;
      if (dx) {
        if (d_out <= 32) return kan_dx_narrow2<K>(x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm.R, rm.grid, st);
        const Basis<K> bas = make_basis<K>(K - 1);
        const int64_t pairs = (int64_t)B * d_in;
        spline_dx_kernel<K, false><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, coeffs, scale, bw, gy, dx, B, d_in,
                                                                               d_out, rm, bas);
        UKAN_LAUNCH_CHECK();
      }
      return UKAN_OK;
    }
  }
  RegPlan p;
  const bool dm = sel[0] == 'd' && kan_bwd_dmma_plan(B, d_in, d_out, rm.R, K, bw != nullptr, kan_num_sms(), p);
  if (!dm) p = kan_bwd_reg_plan(B, d_in, d_out, rm.R, K, bw != nullptr, kan_num_sms());
  if (!p.ok)
    return launch_bwd<K, false>(x, coeffs, scale, bw, gy, dx, dC, dscale, dbw, (double*)workspace, B, d_in, d_out,
                                rm.R, rm, st);
  if (p.S > 1 && (workspace == nullptr || workspace_bytes < p.ws_bytes)) {  // no workspace: one split
    p.S = 1;
    p.sps = B > 0 ? B : 1;
  }
  int rc = dm ? kan_bwd_dmma_dispatch(x, coeffs, scale, gy, dC, dscale, (double*)workspace, B, d_in, d_out, rm.R,
                                      rm.grid, p, st)
              : kan_bwd_reg_dispatch<K>(x, coeffs, scale, gy, dC, dscale, dbw, (double*)workspace, B, d_in, d_out,
                                        rm.R, rm.grid, p, st);
  if (rc) return rc;
  if (dx && B > 0) {
    if (d_out <= 32) return kan_dx_narrow2<K>(x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm.R, rm.grid, st);
    const Basis<K> bas = make_basis<K>(K - 1);
    const int64_t pairs = (int64_t)B * d_in;
    const int wpb = 8;
    spline_dx_kernel<K, false><<<(unsigned)((pairs + wpb - 1) / wpb), wpb * 32, 0, st>>>(
        x, coeffs, scale, bw, gy, dx, B, d_in, d_out, rm, bas);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

extern "C" int ukan_kan_backward_ws2(const float* x, const float* coeffs, const float* scale,
                                   const float* base_weight, const float* gy, float* dx,
                                   float* dcoeffs, float* dscale, float* dbase_weight,
                                   int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                                   double g_min, double g_max, void* workspace,
                                   int64_t workspace_bytes, int flags, void* stream) {
  int rc = check_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  if (!coeffs || !scale || !dcoeffs || !dscale || (B > 0 && (!x || !gy))) return UKAN_E_ARG;
  if ((base_weight == nullptr) != (dbase_weight == nullptr)) return UKAN_E_ARG;
  RowMap rm{};
  rm.grid = make_kan_grid(g_min, g_max, G);
  rm.R = (int)(G + k);
  const RegPlan p = kan_bwd_reg_plan(B, d_in, d_out, rm.R, k + 1, base_weight != nullptr, kan_num_sms());
  const WidePlan wp = kan_bwd_wide_plan(B, d_in, d_out, rm.R, k + 1);
  if (!p.ok && wp.ok && B > 0 && (workspace == nullptr || workspace_bytes < kan_bwd_wide_workspace(wp)))
    return UKAN_E_WORKSPACE;
  if (!p.ok && !wp.ok && !bwd_fits_smem(k + 1, rm.R) &&
      (workspace == nullptr || workspace_bytes < (int64_t)sizeof(double) * d_in * rm.R * d_out))
    return UKAN_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  UKAN_DISPATCH_K(k, return kan_backward_impl<K>(x, coeffs, scale, base_weight, gy, dx, dcoeffs, dscale, dbase_weight, workspace, workspace_bytes, (int)B, (int)d_in, (int)d_out, rm, st, (flags & 1) != 0););
  return UKAN_OK;
}

extern "C" int ukan_kan_backward_part_supported(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k) {
  if (check_kan_args(B, d_in, d_out, G, k, -1.0, 1.0) || B < 1) return 0;
  if (kan_bwd_selector()[0] != 't' || kan_small_ok(B, d_in, d_out, G, k, false)) return 0;
  const TcPlan p = kan_bwd_tc_plan(B, d_in, d_out, G, k, false);
  return (p.ok && d_out >= 64 && d_out % 4 == 0) ? 1 : 0;
}

extern "C" int ukan_kan_backward_part(const float* coeffs, const float* scale, const float* gy, float* dx,
                                      float* dcoeffs, float* dscale, int64_t B, int64_t d_in, int64_t d_out,
                                      int64_t G, int k, double g_min, double g_max, void* workspace,
                                      int64_t workspace_bytes, int64_t i_lo, int64_t i_hi, int what, void* stream) {
  int rc = check_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  if (!ukan_kan_backward_part_supported(B, d_in, d_out, G, k)) return UKAN_E_ARG;
  if (!coeffs || !scale || !gy || (what & ~3) || what == 0) return UKAN_E_ARG;
  const KanGrid grid = make_kan_grid(g_min, g_max, G);
  return kan_bwd_tc_part(coeffs, scale, gy, dx, dcoeffs, dscale, workspace, workspace_bytes, (int)B, (int)d_in,
                         (int)d_out, (int)G, grid, i_lo, i_hi, what, (cudaStream_t)stream);
}

extern "C" int ukan_kan_backward_ws(const float* x, const float* coeffs, const float* scale,
                                   const float* base_weight, const float* gy, float* dx,
                                   float* dcoeffs, float* dscale, float* dbase_weight,
                                   int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                                   double g_min, double g_max, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
  return ukan_kan_backward_ws2(x, coeffs, scale, base_weight, gy, dx, dcoeffs, dscale, dbase_weight, B, d_in, d_out,
                               G, k, g_min, g_max, workspace, workspace_bytes, 0, stream);
}

extern "C" int ukan_kan_backward_prep(const float* x, const float* base_weight, int64_t B, int64_t d_in,
                                      int64_t d_out, int64_t G, int k, double g_min, double g_max, void* workspace,
                                      int64_t workspace_bytes, int32_t* prepared, void* stream) {
  if (prepared == nullptr) return UKAN_E_ARG;
  *prepared = 0;
  int rc = check_kan_args(B, d_in, d_out, G, k, g_min, g_max);
  if (rc) return rc;
  const char* sel = kan_bwd_selector();
  if (B < 1 || k != 3 || base_weight != nullptr || sel[0] != 't' || x == nullptr) return UKAN_OK;
  if (kan_small_ok(B, d_in, d_out, G, k, false)) {  // small layer: the records of kan_small.cu
    if (workspace == nullptr || workspace_bytes < kan_small_workspace(B, d_in, d_out, G)) return UKAN_OK;
    rc = kan_small_records(x, workspace, (int)B, (int)d_in, make_kan_grid(g_min, g_max, G), (cudaStream_t)stream);
    if (rc == UKAN_OK) *prepared = 1;
    return rc;
  }
  const TcPlan tp = kan_bwd_tc_plan(B, d_in, d_out, G, k, false);
  if (!tp.ok || workspace == nullptr || workspace_bytes < kan_bwd_tc_workspace(tp)) return UKAN_OK;
  rc = kan_bwd_tc_prep(x, workspace, workspace_bytes, (int)B, (int)d_in, (int)G, make_kan_grid(g_min, g_max, G), tp,
                       (cudaStream_t)stream);
  if (rc == UKAN_OK) *prepared = 1;
  return rc;
}

extern "C" int ukan_kan_backward(const float* x, const float* coeffs, const float* scale,
                                 const float* base_weight, const float* gy, float* dx,
                                 float* dcoeffs, float* dscale, float* dbase_weight, int64_t B,
                                 int64_t d_in, int64_t d_out, int64_t G, int k, double g_min,
                                 double g_max, void* stream) {
  // Convenience entry without a caller workspace: a stream-ordered allocation (no host sync).
  const int64_t nbytes = ukan_kan_backward_workspace_size(B, d_in, d_out, G, k);
  void* ws = nullptr;
  if (nbytes > 0 && B > 0) UKAN_CUDA_TRY(scratch_alloc(&ws, (size_t)nbytes, (cudaStream_t)stream));
  const int rc = ukan_kan_backward_ws(x, coeffs, scale, base_weight, gy, dx, dcoeffs, dscale, dbase_weight, B, d_in,
                                      d_out, G, k, g_min, g_max, ws, ws ? nbytes : 0, stream);
  if (ws) cudaFreeAsync(ws, (cudaStream_t)stream);
  return rc;
}

extern "C" int ukan_kan_locate(const float* x, int32_t* cell, double* u, int64_t B,
                               int64_t d_in, int64_t G, double g_min, double g_max,
                               void* stream) {
  if (!(g_min < g_max) || G < 1) return UKAN_E_GRID;
  if (!x || !cell || !u || B < 0 || d_in < 1) return UKAN_E_ARG;
  const int64_t n = B * d_in;
  if (n == 0) return UKAN_OK;
  const KanGrid grid = make_kan_grid(g_min, g_max, G);
  kan_locate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, cell, u, n, grid);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_ukan_forward(const float* x, const int32_t* base_row, const float* table,
                                 const float* scale, float* y, int64_t B, int64_t d_in,
                                 int64_t d_out, int k, double delta_g, void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!table || !scale || B < 0 || d_in < 1 || d_out < 1 || B > INT32_MAX ||
      (B > 0 && (!x || !base_row || !y)))
    return UKAN_E_ARG;
  if (B == 0) return UKAN_OK;
  RowMap rm{};
  rm.inv_dg = 1.0 / delta_g;  // layers.py:261
  rm.base_row = base_row;
  rm.K = k + 1;
  cudaStream_t st = (cudaStream_t)stream;
  UKAN_DISPATCH_K(k, return launch_fwd<K, true>(x, table, scale, nullptr, y, (int)B, (int)d_in, (int)d_out, rm, nullptr, st););
  return UKAN_OK;
}

// Dense UKAN forward: the TMEM-gather forward over the features' table segments (max_rows from the
// key build <= 67, cubic, d_out >= 128); size 0 when the layer does not qualify.
static TmPlan ukan_dense_fwd_plan(int64_t B, int64_t d_in, int64_t d_out, int64_t max_rows, int k) {
  static const bool off = getenv("UKAN_UKAN_DENSE") && getenv("UKAN_UKAN_DENSE")[0] == '0';  // A/B only
  if (off || k != 3 || B < 1 || max_rows < 4 || max_rows > 67 || !fwd_use_tm()) return TmPlan{};
  return kan_fwd_tm_plan(B, d_in, d_out, max_rows - 3, 3, false);
}

extern "C" int64_t ukan_ukan_forward_dense_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t max_rows,
                                                         int k) {
  if (B > INT32_MAX || d_in < 1 || d_out < 1) return 0;
  return kan_fwd_tm_workspace(ukan_dense_fwd_plan(B, d_in, d_out, max_rows, k));
}

extern "C" int ukan_ukan_forward_dense(const float* x, const int32_t* base_row, const int32_t* seg_start,
                                       const float* table, const float* scale, float* y, int64_t B, int64_t d_in,
                                       int64_t d_out, int64_t max_rows, int k, double delta_g, void* workspace,
                                       int64_t workspace_bytes, void* stream) {
  if (k != 3) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!x || !base_row || !seg_start || !table || !scale || !y || B < 1 || d_in < 1 || d_out < 1 || B > INT32_MAX)
    return UKAN_E_ARG;
  const TmPlan tp = ukan_dense_fwd_plan(B, d_in, d_out, max_rows, k);
  if (!tp.ok) return UKAN_E_ARG;
  return kan_fwd_tm_run_ukan(x, table, scale, y, workspace, workspace_bytes, (int)B, (int)d_in, (int)d_out,
                             (int)max_rows - 3, 1.0 / delta_g, base_row, seg_start, tp, (cudaStream_t)stream);
}

// Sorted-chunk segmented sweep (kan_bwd_wide.cu) when the per-feature local row index fits the
// 23-bit key field (at most 2*B*K rows per feature); the global fp64 accumulator otherwise.
static bool ukan_seg_ok(int64_t B, int64_t d_out, int k) {
  return 2 * B * (k + 1) < ((int64_t)1 << 23) - 64 && seg_supported(B, d_out);
}

static int64_t ukan_dx64_bytes(int64_t B, int64_t d_in, int64_t d_out) {
  return (int64_t)sizeof(double) * (B * d_out + d_in * d_out);
}

extern "C" int64_t ukan_ukan_backward_workspace_size(int64_t B, int64_t d_in, int64_t d_out,
                                                     int64_t n_u, int k) {
  if (ukan_seg_ok(B, d_out, k) && getenv("UKAN_UKAN_BWD") == nullptr)
    return ((seg_workspace(B, d_in, d_out, n_u * (k + 1)) + 255) / 256) * 256 + ukan_dx64_bytes(B, d_in, d_out);
  return (int64_t)sizeof(double) * n_u * (k + 1) * d_out;
}

// Dense UKAN layers: the table gradient on the banded DMMA sweep — block-split when the features'
// segments have >= 24 rows (enough blocks to keep four warps per feature busy), sample-split for
// <= 16 rows — else on the sorted-merge sweep (seg_*); dx always on the DMMA dx.
// A/B: UKAN_DENSE_SWEEP_MIN_ROWS, UKAN_DENSE_SS.
namespace ukan { bool ukan_dense_ss(int64_t max_rows); }
static bool ukan_dense_sweep(int64_t max_rows) {
  static const int64_t min_rows = getenv("UKAN_DENSE_SWEEP_MIN_ROWS") ? atoll(getenv("UKAN_DENSE_SWEEP_MIN_ROWS")) : 24;
  return ukan_dense_ss(max_rows) || max_rows >= min_rows;
}

extern "C" int64_t ukan_ukan_backward_dense_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                                          int64_t max_rows, int k) {
  if (B < 1 || d_in < 1 || d_out < 1 || B > INT32_MAX || n_u < 1 || n_u * (k + 1) >= ((int64_t)1 << 31)) return 0;
  const int64_t tc = ukan_dense_workspace(B, d_in, d_out, max_rows, k);
  if (tc <= 0 || ukan_dense_sweep(max_rows)) return tc;
  if (!ukan_seg_ok(B, d_out, k)) return 0;
  return ((tc + 255) / 256) * 256 + seg_workspace(B, d_in, d_out, n_u * (k + 1));
}

extern "C" int ukan_ukan_backward_dense(const float* x, const int32_t* base_row, const int32_t* seg_start,
                                        const float* table, const float* scale, const float* gy, float* dx,
                                        float* dtable, float* dscale, int64_t B, int64_t d_in, int64_t d_out,
                                        int64_t n_u, int64_t max_rows, int k, double delta_g, void* workspace,
                                        int64_t workspace_bytes, void* stream) {
  if (k != 3) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!x || !base_row || !seg_start || !table || !scale || !gy || !dtable || !dscale || B < 1 || d_in < 1 ||
      d_out < 1 || B > INT32_MAX)
    return UKAN_E_ARG;
  const int64_t need = ukan_ukan_backward_dense_workspace_size(B, d_in, d_out, n_u, max_rows, k);
  if (need <= 0) return UKAN_E_ARG;
  if (workspace == nullptr || workspace_bytes < need) return UKAN_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t tc = ukan_dense_workspace(B, d_in, d_out, max_rows, k);
  const bool sweep = ukan_dense_sweep(max_rows);
  if (!sweep) {  // table gradient on the sorted-merge sweep, in the workspace after the records
    RowMap rm{};
    rm.inv_dg = 1.0 / delta_g;
    rm.base_row = base_row;
    rm.seg_start = seg_start;
    rm.K = k + 1;
    const int64_t off = ((tc + 255) / 256) * 256;
    const int rc = seg_table_grad<4, true>(x, table, scale, gy, dtable, dscale, static_cast<unsigned char*>(workspace) + off,
                                           workspace_bytes - off, (int)B, (int)d_in, (int)d_out, n_u * (k + 1), rm, st);
    if (rc) return rc;
  }
  return ukan_dense_backward(x, base_row, seg_start, table, scale, gy, dx, dtable, dscale, (int)B, (int)d_in,
                             (int)d_out, max_rows, delta_g, workspace, tc, st, sweep);
}

static int ukan_backward_impl(const float* x, const int32_t* base_row, const int32_t* seg_start,
                              const float* table, const float* scale, const float* gy, float* dx, float* dtable,
                              float* dscale, int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int k,
                              double delta_g, void* workspace, int64_t workspace_bytes, void* stream,
                              int64_t max_rows_hint) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!x || !base_row || !seg_start || !table || !scale || !gy || !dtable || !dscale || B < 0 ||
      d_in < 1 || d_out < 1 || B > INT32_MAX || n_u * (k + 1) >= ((int64_t)1 << 31))
    return UKAN_E_ARG;
  const int64_t need = ukan_ukan_backward_workspace_size(B, d_in, d_out, n_u, k);
  if (workspace == nullptr || workspace_bytes < need) return UKAN_E_WORKSPACE;
  RowMap rm{};
  rm.inv_dg = 1.0 / delta_g;
  rm.base_row = base_row;
  rm.seg_start = seg_start;
  rm.K = k + 1;
  cudaStream_t st = (cudaStream_t)stream;
  if (B > 0 && ukan_seg_ok(B, d_out, k) && getenv("UKAN_UKAN_BWD") == nullptr) {
    UKAN_DISPATCH_K(k, {
      int rc = seg_table_grad<K, true>(x, table, scale, gy, dtable, dscale, workspace, workspace_bytes, (int)B,
                                       (int)d_in, (int)d_out, n_u * (k + 1), rm, st, max_rows_hint);
      if (rc) return rc;
      if (dx) {
        const int64_t pairs = B * d_in;
        double* g64 = reinterpret_cast<double*>(static_cast<unsigned char*>(workspace) +
                                                ((seg_workspace(B, d_in, d_out, n_u * (k + 1)) + 255) / 256) * 256);
        double* s64 = g64 + B * d_out;
        cvt_f64_kernel<<<(unsigned)((B * d_out + 255) / 256), 256, 0, st>>>(gy, g64, B * d_out);
        UKAN_LAUNCH_CHECK();
        cvt_f64_kernel<<<(unsigned)((d_in * d_out + 255) / 256), 256, 0, st>>>(scale, s64, d_in * d_out);
        UKAN_LAUNCH_CHECK();
        // A/B only (UKAN_DX_SORTED=1): dx on the sweep's sorted order — measured slower at the cfg4
        // shape (7.4 vs 6.1 ms: latency-bound runs of 4 positions), kept for the record
        static const bool sorted_on = getenv("UKAN_DX_SORTED") && getenv("UKAN_DX_SORTED")[0] == '1';
        if (K == 4 && sorted_on && B <= 8192 && d_out % 4 == 0 &&
            seg_uses_sorted((int)B, n_u * (k + 1), max_rows_hint))
          return seg_dx_sorted(table, s64, g64, dx, workspace, (int)B, (int)d_in, (int)d_out, n_u * (k + 1), rm, st);
        spline_dx64_kernel<K, true><<<(unsigned)((pairs + 7) / 8), 256, 0, st>>>(x, table, s64, g64, dx, (int)B,
                                                                                 (int)d_in, (int)d_out, rm,
                                                                                 make_basis<K>(K - 1));
        UKAN_LAUNCH_CHECK();
      }
      return UKAN_OK;
    });
  }
  // the fp64 accumulator lives in the global workspace (feature segments are data dependent)
  UKAN_DISPATCH_K(k, return launch_bwd<K, true>(x, table, scale, nullptr, gy, dx, dtable, dscale, nullptr, (double*)workspace, (int)B, (int)d_in, (int)d_out, 1 << 30, rm, st););
  return UKAN_OK;
}

extern "C" int ukan_ukan_backward(const float* x, const int32_t* base_row, const int32_t* seg_start,
                                  const float* table, const float* scale, const float* gy, float* dx, float* dtable,
                                  float* dscale, int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int k,
                                  double delta_g, void* workspace, int64_t workspace_bytes, void* stream) {
  return ukan_backward_impl(x, base_row, seg_start, table, scale, gy, dx, dtable, dscale, B, d_in, d_out, n_u, k,
                            delta_g, workspace, workspace_bytes, stream, 0);
}

// With the key build's max_rows: dense layers (<= 67 rows per feature) on the tensor-core path, the
// others on the sorted-merge path with max_rows bounding the per-feature row histogram (cfg4 at
// B = 65536: ~316 rows per feature instead of the 2*B*K bound -> the per-feature sorted sweep).
extern "C" int64_t ukan_ukan_backward2_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                                     int64_t max_rows, int k) {
  const int64_t dense = ukan_ukan_backward_dense_workspace_size(B, d_in, d_out, n_u, max_rows, k);
  return dense > 0 ? dense : ukan_ukan_backward_workspace_size(B, d_in, d_out, n_u, k);
}

extern "C" int ukan_ukan_backward2(const float* x, const int32_t* base_row, const int32_t* seg_start,
                                   const float* table, const float* scale, const float* gy, float* dx, float* dtable,
                                   float* dscale, int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                   int64_t max_rows, int k, double delta_g, void* workspace, int64_t workspace_bytes,
                                   void* stream) {
  if (ukan_ukan_backward_dense_workspace_size(B, d_in, d_out, n_u, max_rows, k) > 0)
    return ukan_ukan_backward_dense(x, base_row, seg_start, table, scale, gy, dx, dtable, dscale, B, d_in, d_out, n_u,
                                    max_rows, k, delta_g, workspace, workspace_bytes, stream);
  return ukan_backward_impl(x, base_row, seg_start, table, scale, gy, dx, dtable, dscale, B, d_in, d_out, n_u, k,
                            delta_g, workspace, workspace_bytes, stream, max_rows);
}
