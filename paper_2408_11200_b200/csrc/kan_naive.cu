// kan_naive.cu — the paper's comparison arm: KAN layer with ALL G+k B-spline bases per input.
//
// Replaces naive_kan_forward (layers.py:321-370): every basis function of the full knot vector is
// evaluated by the Cox-de Boor recursion (_naive_bases, layers.py:324-334) and dotted with the
// whole coefficient table, so the cost grows with G — the baseline the matrix form (spline.cu /
// kan_fwd_tm.cu) is compared against in the grid-size benchmark (bench.py:76-96,
// paper_2408_11200_b200/bench_arms.py).  Backward covers the parameters only (as the reference).
//
// Basis B_{s,k}(x) depends only on knots t[s .. s+k+1], so each thread evaluates its own basis by
// the local triangular recursion (k+1 degree-0 indicators) — no cross-thread levels.  fp64 bases
// (the reference's knots are float64), fp32 coefficients, fp32 sums in the forward as the matrix
// arm, fp64 sums for the parameter gradients.
#include "common.cuh"

namespace ukan {

constexpr int kNvMaxK = UKAN_MAX_DEGREE + 1;

// B_{s,k}(x) over knots t_j = g_min + (j - k) * dg, j = 0 .. G + 2k  (layers.py:349), half-open
// degree-0 intervals, division form of the recursion (layers.py:330-333), NumPy's rounding.
// knot t_j = g_min + (j - k) * dg with the reference's two roundings (np.arange(...) * dg, then
// + g_min: layers.py:349) — no FMA contraction, which moves knots by an ulp (e.g. the last knot
// of G = 14 on [-2, 2] would land above nextafter(2, -2) and drop the last basis)
__device__ __forceinline__ double naive_knot(int j, double g_min, double dg) {
  return __dadd_rn(g_min, __dmul_rn((double)j, dg));
}

__device__ __forceinline__ double naive_basis(double x, int s, int k, double g_min, double dg) {
  double N[kNvMaxK + 1];
  for (int j = 0; j <= k; ++j)
    N[j] = (x >= naive_knot(s + j - k, g_min, dg) && x < naive_knot(s + j + 1 - k, g_min, dg)) ? 1.0 : 0.0;
  for (int d = 1; d <= k; ++d) {
    for (int j = 0; j <= k - d; ++j) {
      const double ts = naive_knot(s + j - k, g_min, dg);          // t[s+j]
      const double tsd = naive_knot(s + j + d - k, g_min, dg);     // t[s+j+d]
      const double ts1 = naive_knot(s + j + 1 - k, g_min, dg);     // t[s+j+1]
      const double tsd1 = naive_knot(s + j + d + 1 - k, g_min, dg);  // t[s+j+d+1]
      N[j] = __dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn(x, ts), __dsub_rn(tsd, ts)), N[j]),
                       __dmul_rn(__ddiv_rn(__dsub_rn(tsd1, x), __dsub_rn(tsd1, ts1)), N[j + 1]));
    }
  }
  return N[0];
}

// y[b,o] = sum_i scale[i,o] * tmp[b,i,o],  tmp[b,i,o] = sum_s B_s(xc_bi) C[i,s,o]; tmp is kept for
// the backward (the reference keeps it too, layers.py:353-356).  CTA = one sample, threads
// first evaluate the R bases of feature i into shared memory, then dot them over outputs.
__global__ void __launch_bounds__(256)
kan_naive_forward_kernel(const float* __restrict__ x, const float* __restrict__ C, const float* __restrict__ scale,
                         float* __restrict__ y, float* __restrict__ tmp, int d_in, int d_out, int R, int k,
                         double g_min, double hi, double dg) {
  extern __shared__ double bas[];  // [R]
  const int b = blockIdx.x;
  for (int o = threadIdx.x; o < d_out; o += blockDim.x) y[(size_t)b * d_out + o] = 0.f;
  for (int i = 0; i < d_in; ++i) {
    double xc = (double)x[(size_t)b * d_in + i];
    xc = xc < g_min ? g_min : (xc > hi ? hi : xc);  // np.clip(x, g_min, nextafter(g_max, g_min))
    __syncthreads();
    for (int s = threadIdx.x; s < R; s += blockDim.x) bas[s] = naive_basis(xc, s, k, g_min, dg);
    __syncthreads();
    for (int o = threadIdx.x; o < d_out; o += blockDim.x) {
      const float* Ci = C + (size_t)i * R * d_out + o;
      float t = 0.f;
      for (int s = 0; s < R; ++s) t = fmaf((float)bas[s], Ci[(size_t)s * d_out], t);
      tmp[((size_t)b * d_in + i) * d_out + o] = t;
      y[(size_t)b * d_out + o] += scale[(size_t)i * d_out + o] * t;
    }
  }
}

// dC[i,s,o] = scale[i,o] * sum_b B_s(xc_bi) g[b,o]  (fp64 sums, sample order).  CTA = (feature i,
// 64 basis rows); thread = (row s, 4 outputs) keeping its sums in registers.
__global__ void __launch_bounds__(256)
kan_naive_dcoeffs_kernel(const float* __restrict__ x, const float* __restrict__ g, const float* __restrict__ scale,
                         float* __restrict__ dC, int B, int d_in, int d_out, int R, int k, double g_min, double hi,
                         double dg) {
  const int i = blockIdx.x;
  const int s = blockIdx.y * 64 + (threadIdx.x & 63);
  const int o0 = (threadIdx.x >> 6) * 4;  // 4 output groups of 4 per pass
  for (int ob = 0; ob < d_out; ob += 16) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (s < R) {
      for (int b = 0; b < B; ++b) {
        double xc = (double)x[(size_t)b * d_in + i];
        xc = xc < g_min ? g_min : (xc > hi ? hi : xc);
        const double beta = naive_basis(xc, s, k, g_min, dg);
        if (beta == 0.0) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int o = ob + o0 + v;
          if (o < d_out) acc[v] = fma(beta, (double)g[(size_t)b * d_out + o], acc[v]);
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int o = ob + o0 + v;
        if (o < d_out) dC[((size_t)i * R + s) * d_out + o] = (float)((double)scale[(size_t)i * d_out + o] * acc[v]);
      }
    }
  }
}

// dscale[i,o] = sum_b g[b,o] tmp[b,i,o]  (fp64, sample order)
__global__ void kan_naive_dscale_kernel(const float* __restrict__ g, const float* __restrict__ tmp,
                                        float* __restrict__ dscale, int B, int d_in, int d_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)d_in * d_out) return;
  const int i = (int)(t / d_out), o = (int)(t % d_out);
  double a = 0.0;
  for (int b = 0; b < B; ++b) a = fma((double)g[(size_t)b * d_out + o], (double)tmp[((size_t)b * d_in + i) * d_out + o], a);
  dscale[t] = (float)a;
}

}  // namespace ukan

using namespace ukan;

extern "C" int ukan_kan_naive_forward(const float* x, const float* coeffs, const float* scale, float* y, float* tmp,
                                      int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, double g_min,
                                      double g_max, void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(g_min < g_max) || G < 1) return UKAN_E_GRID;
  if (B < 0 || d_in < 1 || d_out < 1 || (B > 0 && (!x || !coeffs || !scale || !y || !tmp))) return UKAN_E_ARG;
  if (B == 0) return UKAN_OK;
  const int R = (int)(G + k);
  const double dg = (g_max - g_min) / (double)G, hi = nextafter(g_max, g_min);  // layers.py:159, 346
  const size_t smem = sizeof(double) * R;
  if (smem > 48 * 1024) UKAN_CUDA_TRY(cudaFuncSetAttribute(kan_naive_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kan_naive_forward_kernel<<<(unsigned)B, 256, smem, (cudaStream_t)stream>>>(x, coeffs, scale, y, tmp, (int)d_in,
                                                                              (int)d_out, R, k, g_min, hi, dg);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_kan_naive_backward(const float* x, const float* scale, const float* tmp, const float* gy,
                                       float* dcoeffs, float* dscale, int64_t B, int64_t d_in, int64_t d_out,
                                       int64_t G, int k, double g_min, double g_max, void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(g_min < g_max) || G < 1) return UKAN_E_GRID;
  if (B < 0 || d_in < 1 || d_out < 1 || !dcoeffs || !dscale || (B > 0 && (!x || !scale || !tmp || !gy)))
    return UKAN_E_ARG;
  const int R = (int)(G + k);
  const double dg = (g_max - g_min) / (double)G, hi = nextafter(g_max, g_min);
  cudaStream_t st = (cudaStream_t)stream;
  kan_naive_dcoeffs_kernel<<<dim3((unsigned)d_in, (unsigned)((R + 63) / 64)), 256, 0, st>>>(
      x, gy, scale, dcoeffs, (int)B, (int)d_in, (int)d_out, R, k, g_min, hi, dg);
  UKAN_LAUNCH_CHECK();
  const int64_t n = d_in * d_out;
  kan_naive_dscale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gy, tmp, dscale, (int)B, (int)d_in, (int)d_out);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}
