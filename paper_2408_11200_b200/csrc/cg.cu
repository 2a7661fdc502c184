// cg.cu — UKAN coefficient generator (CG) MLP: grid-group positional encoding + dense GEMMs.
//
// Replaces positional_encoding (layers.py:112-123), _cg_eval (232-243) and the tape
// backward of its matmul / silu / gather_rows / concat_last (tensor.py:189-197, 228-233,
// 257-268, 276-285).
//   inp[r] = [emb[f_r] || PE(g_r)]           PE in fp64 (SURVEY gotcha 3), stored fp32
//   H      = silu(inp @ W1 + b1)             fp32 GEMM (K = d_femb + d_pe)
//   Out    = H @ W2 + b2                     fp32 GEMM (K = d_h) -> table [n_u, K*d_out]
//   backward GEMMs accumulate in fp64 (reductions over n_u / K*d_out).
// Tensor cores for every GEMM: the table GEMM on tcgen05 (cg_tc.cu, tf32 operand splits); the
// gradient GEMMs on the FP64 tensor cores (cg_dmma.cu, IEEE fp64 products and sums) because the
// tcgen05 fp32 accumulator carries ~22 bits per MMA (measured), which misses the UKAN gradient
// parity by 2-3x even with 3-piece operand splits and per-chunk fp64 promotion.  The
// activated GEMM (its pre-activation feeds every gradient) and misaligned shapes use the fp32
// CUDA-core kernel below.
#include "common.cuh"

namespace ukan {

// tensor-core path (cg_tc.cu)
bool cg_tc_applicable(const void* a, const void* b, int64_t M, int64_t N, int64_t K, int64_t ca, int64_t cb);
int cg_tc_gemm(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int64_t M,
               int64_t N, int64_t K, int mode, const float* bias, int act, float* C, float* pre, float* part,
               int S, int64_t kps, cudaStream_t st);
int cg_colsum(const float* X, float* out, int64_t K, int64_t N, cudaStream_t st);
int cg_colsum64(const double* X, float* out, int64_t K, int64_t N, cudaStream_t st);
// fp64 tensor-core gradient GEMMs (cg_dmma.cu)
int64_t cg_dmma_workspace(int64_t M, int64_t N, int64_t K);
int cg_dmma_gemm(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int64_t M,
                 int64_t N, int64_t K, float* C, double* part, cudaStream_t st);
static int dmma_with_ws(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int64_t M,
                        int64_t N, int64_t K, float* C, cudaStream_t st) {
  const int64_t nb = cg_dmma_workspace(M, N, K);
  void* part = nullptr;  // split-K partials: stream-ordered allocation, no host sync
  if (nb > 0) UKAN_CUDA_TRY(scratch_alloc(&part, (size_t)nb, st));
  const int rc = cg_dmma_gemm(A, sam, sak, Bm, sbk, sbn, M, N, K, C, static_cast<double*>(part), st);
  if (part) cudaFreeAsync(part, st);
  return rc;
}

// ---------------------------------------------------------------------------------------
// positional encoding + embedding gather
// ---------------------------------------------------------------------------------------
constexpr int kMaxPeHalf = 128;
struct PeFreqs {
  double f[kMaxPeHalf];
};

__global__ void cg_input_kernel(const int32_t* __restrict__ key_f,
                                const int64_t* __restrict__ key_g, const float* __restrict__ emb,
                                double* __restrict__ inp, int64_t n_u, int d_femb, int d_pe,
                                PeFreqs fr) {
  const int W = d_femb + d_pe;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_u * W) return;
  const int64_t r = t / W;
  const int c = (int)(t % W);
  double v;
  if (c < d_femb) {
    v = (double)emb[(size_t)key_f[r] * d_femb + c];
  } else {  // fp64 PE kept in fp64: rounding it to fp32 alone costs 1.5x the CG-gradient tolerance
    const int m = (c - d_femb) >> 1;
    const double ang = (double)key_g[r] * fr.f[m];  // g[..., None] * freqs  (layers.py:119)
    v = ((c - d_femb) & 1) ? cos(ang) : sin(ang);
  }
  inp[t] = v;
}

// ---------------------------------------------------------------------------------------
// Tiled GEMMs (64x64 CTA tile, 4x4 per thread, BK = 16).
// ---------------------------------------------------------------------------------------
constexpr int TM = 64, TN = 64, TK = 16;

// C = act(A[M,K] @ B[K,N] + bias), fp32 accumulate.  pre_out (optional) = pre-activation.
__global__ void __launch_bounds__(256)
gemm_nn_kernel(const float* __restrict__ A, const float* __restrict__ Bm,
               const float* __restrict__ bias, float* __restrict__ C, float* __restrict__ pre,
               int M, int N, int K, int act) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int t = threadIdx.x; t < TM * TK; t += 256) {
      const int mm = t / TK, kk = t % TK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gm * K + gk] : 0.f;
    }
    for (int t = threadIdx.x; t < TK * TN; t += 256) {
      const int kk = t / TN, nn = t % TN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? Bm[(size_t)gk * N + gn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][ty * 4 + q];
        b[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int gm = m0 + ty * 4 + p;
    if (gm >= M) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gn = n0 + tx * 4 + q;
      if (gn >= N) continue;
      float v = acc[p][q] + (bias ? bias[gn] : 0.f);
      if (pre) pre[(size_t)gm * N + gn] = v;
      if (act == 1) v = (float)silu_d((double)v);
      C[(size_t)gm * N + gn] = v;
    }
  }
}




__global__ void silu_bwd_kernel(const double* __restrict__ pre, const double* __restrict__ dH,
                                double* __restrict__ dpre, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  dpre[t] = dH[t] * dsilu_d(pre[t]);
}

// d_emb[f, c] = sum_{r in seg(f)} dinp[r, c], c < d_femb, fp64, key order.
__global__ void emb_bwd_kernel(const int32_t* __restrict__ seg_start,
                               const double* __restrict__ dinp, float* __restrict__ d_emb,
                               int d_in, int d_femb, int d_cg_in) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)d_in * d_femb) return;
  const int f = (int)(t / d_femb), c = (int)(t % d_femb);
  double s = 0.0;
  for (int r = seg_start[f]; r < seg_start[f + 1]; ++r) s += dinp[(size_t)r * d_cg_in + c];
  d_emb[t] = (float)s;
}

}  // namespace ukan

using namespace ukan;

extern "C" int ukan_ukan_cg_input(const int32_t* key_f, const int64_t* key_g, const float* emb,
                                  double* inp, int64_t n_u, int64_t d_femb, int64_t d_pe,
                                  void* stream) {
  if (d_pe % 2 != 0 || d_pe / 2 > kMaxPeHalf || d_femb < 0 || n_u < 0) return UKAN_E_ARG;
  if (n_u == 0) return UKAN_OK;
  PeFreqs fr;
  for (int m = 0; m < d_pe / 2; ++m)  // freqs = 10000.0 ** (-2.0 * arange(half) / d_pe)
    fr.f[m] = pow(10000.0, (-2.0 * (double)m) / (double)d_pe);
  const int64_t n = n_u * (d_femb + d_pe);
  cg_input_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      key_f, key_g, emb, inp, n_u, (int)d_femb, (int)d_pe, fr);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_gemm_bias_act(const float* A, const float* Bm, const float* bias, float* C,
                                  float* pre_out, int64_t M, int64_t N, int64_t K, int act,
                                  void* stream) {
  if (M < 0 || N < 1 || K < 1 || M > INT32_MAX || !A || !Bm || !C) return UKAN_E_ARG;
  if (M == 0) return UKAN_OK;
  // The table GEMM (act = 0: H @ W2 + b2) feeds only the spline forward and dscale, which keep
  // their parity on the tensor cores; the activated GEMM's pre-activation feeds every CG
  // gradient (silu'), where the tensor core's ~22-bit accumulation measured 2.6x over the bar.
  if (act == 0 && cg_tc_applicable(A, Bm, M, N, K, K, N))  // A [M,K] row-major, B [K,N] row-major
    return cg_tc_gemm(A, K, 1, Bm, N, 1, M, N, K, 0, bias, act, C, pre_out, nullptr, 1, K, (cudaStream_t)stream);
  dim3 g((unsigned)((N + TN - 1) / TN), (unsigned)((M + TM - 1) / TM));
  gemm_nn_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(A, Bm, bias, C, pre_out, (int)M, (int)N, (int)K, act);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_gemm_nt(const float* A, const float* Bm, float* C, int64_t M, int64_t N,
                            int64_t K, void* stream) {
  if (M < 0 || N < 1 || K < 1 || M > INT32_MAX || !A || !Bm || !C) return UKAN_E_ARG;
  if (M == 0) return UKAN_OK;
  return dmma_with_ws(A, K, 1, Bm, 1, K, M, N, K, C, (cudaStream_t)stream);  // A [M,K], B given as [N,K]
}

extern "C" int ukan_gemm_tn(const float* A, const float* Bm, float* C, float* colsum_B,
                            int64_t M, int64_t N, int64_t K, void* stream) {
  if (M < 1 || N < 1 || K < 0 || K > INT32_MAX || !A || !Bm || !C) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (K == 0) {
    UKAN_CUDA_TRY(cudaMemsetAsync(C, 0, sizeof(float) * M * N, st));
    if (colsum_B) UKAN_CUDA_TRY(cudaMemsetAsync(colsum_B, 0, sizeof(float) * N, st));
    return UKAN_OK;
  }
  int rc = dmma_with_ws(A, 1, M, Bm, N, 1, M, N, K, C, st);  // A given as [K,M], B [K,N]
  if (rc) return rc;
  return colsum_B ? cg_colsum(Bm, colsum_B, K, N, st) : UKAN_OK;
}

extern "C" int ukan_silu_backward(const double* pre, const double* dH, double* dpre, int64_t n,
                                  void* stream) {
  if (n < 0 || !pre || !dH || !dpre) return UKAN_E_ARG;
  if (n == 0) return UKAN_OK;
  silu_bwd_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(pre, dH, dpre, n);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_ukan_emb_backward(const int32_t* seg_start, const double* dinp, float* d_emb,
                                      int64_t d_in, int64_t d_femb, int64_t d_cg_in,
                                      void* stream) {
  if (d_in < 1 || d_femb < 0 || d_cg_in < d_femb || !seg_start || !d_emb) return UKAN_E_ARG;
  const int64_t n = d_in * d_femb;
  if (n == 0) return UKAN_OK;
  emb_bwd_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      seg_start, dinp, d_emb, (int)d_in, (int)d_femb, (int)d_cg_in);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

// Mixed-precision GEMM on the FP64 tensor cores (cg_dmma.cu) for the fp64 CG chain.
extern "C" int ukan_gemm_f64(int op, const void* A, int a_dtype, const void* Bm, int b_dtype, const float* bias,
                             int act, double* pre_out, float* C32, double* C64, float* colsum_B, int64_t M, int64_t N,
                             int64_t K, void* stream) {
  if (M < 0 || N < 1 || K < 0 || M > INT32_MAX || K > INT32_MAX || !A || !Bm || (!C32 && !C64 && !pre_out))
    return UKAN_E_ARG;
  if (op < 0 || op > 2 || (a_dtype != UKAN_F32 && a_dtype != UKAN_F64) || (b_dtype != UKAN_F32 && b_dtype != UKAN_F64))
    return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (M == 0) return UKAN_OK;
  DgOut o;
  o.c32 = C32;
  o.c64 = C64;
  o.pre64 = pre_out;
  o.bias = bias;
  o.act = act;
  // strides: NN A [M,K] B [K,N]; NT A [M,K] B [N,K]; TN A [K,M] B [K,N]
  const int64_t sam = op == 2 ? 1 : K, sak = op == 2 ? M : 1;
  const int64_t sbk = op == 1 ? 1 : N, sbn = op == 1 ? K : 1;
  if (K == 0) return UKAN_E_ARG;
  const int64_t nb = cg_dmma_workspace(M, N, K);
  void* part = nullptr;
  if (nb > 0) UKAN_CUDA_TRY(scratch_alloc(&part, (size_t)nb, st));
  double* pd = static_cast<double*>(part);
  int rc;
  if (a_dtype == UKAN_F32 && b_dtype == UKAN_F32)
    rc = cg_dmma_gemm_t<float, float>((const float*)A, sam, sak, (const float*)Bm, sbk, sbn, M, N, K, o, pd, st);
  else if (a_dtype == UKAN_F64 && b_dtype == UKAN_F32)
    rc = cg_dmma_gemm_t<double, float>((const double*)A, sam, sak, (const float*)Bm, sbk, sbn, M, N, K, o, pd, st);
  else if (a_dtype == UKAN_F32)
    rc = cg_dmma_gemm_t<float, double>((const float*)A, sam, sak, (const double*)Bm, sbk, sbn, M, N, K, o, pd, st);
  else
    rc = cg_dmma_gemm_t<double, double>((const double*)A, sam, sak, (const double*)Bm, sbk, sbn, M, N, K, o, pd, st);
  if (part) cudaFreeAsync(part, st);
  if (rc || !colsum_B) return rc;
  if (op != 2) return UKAN_E_ARG;  // column sums of B (the bias gradient) belong to the TN form
  return b_dtype == UKAN_F32 ? cg_colsum((const float*)Bm, colsum_B, K, N, st)
                             : cg_colsum64((const double*)Bm, colsum_B, K, N, st);
}
