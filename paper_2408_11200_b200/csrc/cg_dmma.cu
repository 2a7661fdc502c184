// cg_dmma.cu — the coefficient-generator gradient GEMMs on the FP64 tensor cores (DMMA).
//
// Replaces the tape backward of the CG matmuls (tensor.py:189-197 for _cg_eval, layers.py:241-242):
//   dW2 = H^T dT  (reduction over n_u rows),  dH = dT W2^T (over K*d_out),
//   dW1 = inp^T dpre (over n_u),              dinp = dpre W1^T (over d_h).
// Parity needs more than fp32 accumulation on these reductions and the tcgen05
// tf32 accumulator measured ~22 bits (cg_tc.cu), so they run as IEEE fp64 GEMMs on
// `mma.sync.m8n8k4.f64`: fp32 operands are widened exactly when staged, products and sums are
// fp64 — the same arithmetic as the CUDA-core fp64 kernels they replace, ~10x faster.
//
// CTA = 16 warps, 128 x 128 output tile (warp tile 32 x 32 = 4 x 4 DMMA tiles, fp64 accumulators in
// registers), K staged in chunks of 32 (fp64, padded rows -> conflict-free fragment loads),
// double-buffered with cp.async-free register staging (global fp32 -> registers -> fp64 smem).
// Long reductions are split over blockIdx.z into fp64 partials reduced in fixed order.
#include <algorithm>

#include "common.cuh"

namespace ukan {

constexpr int kDgM = 128, kDgN = 128, kDgK = 32;
constexpr int kDgAS = kDgK + 4;   // As[m][k] row stride (doubles): 288 B rows -> 2 wavefronts per fragment
constexpr int kDgBS = kDgN + 4;   // Bs[k][n] row stride (doubles)
constexpr int kDgThreads = 512;  // 16 warps (4 x 4 warp tiles of 32 x 32): twice the warps per SM of the 8-warp
                                  // 128 x 64 version (latency-bound at 12% warps active), each operand fragment used 4x

__device__ __forceinline__ void dg_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void dg_epilogue(const DgOut& o, int64_t idx, int n, double v) {
  if (o.bias) v += (double)o.bias[n];
  if (o.pre64) o.pre64[idx] = v;
  if (o.act) v = silu_d(v);
  if (o.c64) o.c64[idx] = v;
  if (o.c32) o.c32[idx] = (float)v;
}

// D[m, n] = sum_k A(m,k) B(k,n) with A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn]; TA / TB
// are float (widened exactly when staged) or double.  part == nullptr: epilogue `out`; else
// part[z][m][n] (fp64 partial of K-slice z).
template <typename TA, typename TB>
__global__ void __launch_bounds__(kDgThreads, 1)
cg_dmma_gemm_kernel(const TA* __restrict__ A, int64_t sam, int64_t sak, const TB* __restrict__ Bm, int64_t sbk,
                    int64_t sbn, int M, int N, int K, int kps, DgOut out, double* __restrict__ part) {
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                          // 2 x [kDgM][kDgAS]
  double* Bs = dsm + 2 * kDgM * kDgAS;       // 2 x [kDgK][kDgBS]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  const int m0 = blockIdx.x * kDgM, n0 = blockIdx.y * kDgN;
  const int z = blockIdx.z;
  const int kb = z * kps, ke = min(K, kb + kps);
  const int nch = (ke - kb + kDgK - 1) / kDgK;

  // staging registers: A chunk 128 x 32 = 8 / thread, B chunk 32 x 128 = 8 / thread
  TA ra[8];
  TB rb[8];
  auto fetch = [&](int c) {
    const int k0 = kb + c * kDgK;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = threadIdx.x + q * kDgThreads;  // element of the 128 x 32 chunk
      int m, k;
      if (sak == 1) { m = e >> 5; k = e & 31; } else { k = e >> 7; m = e & 127; }  // walk the contiguous dim
      const int gm = m0 + m, gk = k0 + k;
      ra[q] = (gm < M && gk < ke) ? __ldg(A + (size_t)gm * sam + (size_t)gk * sak) : (TA)0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = threadIdx.x + q * kDgThreads;  // element of the 32 x 128 chunk
      int n, k;
      if (sbk == 1) { n = e >> 5; k = e & 31; } else { k = e >> 7; n = e & 127; }
      const int gn = n0 + n, gk = k0 + k;
      rb[q] = (gn < N && gk < ke) ? __ldg(Bm + (size_t)gk * sbk + (size_t)gn * sbn) : (TB)0;
    }
  };
  auto store = [&](int buf) {  // exact fp32 -> fp64 widening
    double* as = As + buf * kDgM * kDgAS;
    double* bs = Bs + buf * kDgK * kDgBS;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = threadIdx.x + q * kDgThreads;
      int m, k;
      if (sak == 1) { m = e >> 5; k = e & 31; } else { k = e >> 7; m = e & 127; }
      as[m * kDgAS + k] = (double)ra[q];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = threadIdx.x + q * kDgThreads;
      int n, k;
      if (sbk == 1) { n = e >> 5; k = e & 31; } else { k = e >> 7; n = e & 127; }
      bs[k * kDgBS + n] = (double)rb[q];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  if (nch > 0) {
    fetch(0);
    store(0);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) fetch(c + 1);  // global loads in flight during this chunk's DMMAs
    const double* as = As + buf * kDgM * kDgAS;
    const double* bs = Bs + buf * kDgK * kDgBS;
#pragma unroll
    for (int ks = 0; ks < kDgK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(wm + i * 8 + grp) * kDgAS + ks + kq];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(ks + kq) * kDgBS + wn + j * 8 + grp];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dg_dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (c + 1 < nch) store(buf ^ 1);  // the other buffer was last read in chunk c-1 (barrier below)
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int m = m0 + wm + i * 8 + grp, n = n0 + wn + j * 8 + 2 * kq + v;
        if (m < M && n < N) {
          if (part) part[((size_t)z * M + m) * N + n] = acc[i][j][v];
          else dg_epilogue(out, (int64_t)m * N + n, n, acc[i][j][v]);
        }
      }
}

// out[m][n] = epilogue(sum_z part[z][m][n]) (fp64, fixed order).
__global__ void cg_dmma_reduce_kernel(const double* __restrict__ part, DgOut out, int64_t MN, int N, int S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= MN) return;
  double a = 0.0;
  for (int z = 0; z < S; ++z) a += part[(size_t)z * MN + t];
  dg_epilogue(out, t, (int)(t % N), a);
}

int kan_num_sms();

// Split the reduction so the grid covers ~4 waves (one CTA per SM); fp64 partials.
static int dg_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + kDgM - 1) / kDgM) * ((N + kDgN - 1) / kDgN);
  const int64_t want = 4 * (int64_t)kan_num_sms();
  if (tiles >= want) return 1;
  return (int)std::max<int64_t>(1, std::min<int64_t>((want + tiles - 1) / tiles, K / (8 * kDgK)));
}

int64_t cg_dmma_workspace(int64_t M, int64_t N, int64_t K) {
  const int S = dg_splits(M, N, K);
  return S > 1 ? (int64_t)sizeof(double) * S * M * N : 0;
}

template <typename TA, typename TB>
int cg_dmma_gemm_t(const TA* A, int64_t sam, int64_t sak, const TB* Bm, int64_t sbk, int64_t sbn, int64_t M,
                   int64_t N, int64_t K, const DgOut& out, double* part, cudaStream_t st) {
  if (M < 1 || N < 1 || K < 1 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return UKAN_E_ARG;
  const int S = dg_splits(M, N, K);
  if (S > 1 && part == nullptr) return UKAN_E_WORKSPACE;
  const int kps = (int)((K + S - 1) / S + kDgK - 1) / kDgK * kDgK;
  const int Sz = (int)((K + kps - 1) / kps);
  const size_t smem = sizeof(double) * 2 * ((size_t)kDgM * kDgAS + (size_t)kDgK * kDgBS);
  auto kern = cg_dmma_gemm_kernel<TA, TB>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 g((unsigned)((M + kDgM - 1) / kDgM), (unsigned)((N + kDgN - 1) / kDgN), Sz);
  kern<<<g, kDgThreads, smem, st>>>(A, sam, sak, Bm, sbk, sbn, (int)M, (int)N, (int)K, kps, out,
                                    Sz > 1 ? part : nullptr);
  UKAN_LAUNCH_CHECK();
  if (Sz > 1) {
    const int64_t MN = M * N;
    cg_dmma_reduce_kernel<<<(unsigned)((MN + 255) / 256), 256, 0, st>>>(part, out, MN, (int)N, Sz);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}
template int cg_dmma_gemm_t<float, float>(const float*, int64_t, int64_t, const float*, int64_t, int64_t, int64_t,
                                          int64_t, int64_t, const DgOut&, double*, cudaStream_t);
template int cg_dmma_gemm_t<double, float>(const double*, int64_t, int64_t, const float*, int64_t, int64_t, int64_t,
                                           int64_t, int64_t, const DgOut&, double*, cudaStream_t);
template int cg_dmma_gemm_t<float, double>(const float*, int64_t, int64_t, const double*, int64_t, int64_t, int64_t,
                                           int64_t, int64_t, const DgOut&, double*, cudaStream_t);
template int cg_dmma_gemm_t<double, double>(const double*, int64_t, int64_t, const double*, int64_t, int64_t, int64_t,
                                            int64_t, int64_t, const DgOut&, double*, cudaStream_t);

int cg_dmma_gemm(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int64_t M,
                 int64_t N, int64_t K, float* C, double* part, cudaStream_t st) {
  DgOut o;
  o.c32 = C;
  return cg_dmma_gemm_t<float, float>(A, sam, sak, Bm, sbk, sbn, M, N, K, o, part, st);
}

}  // namespace ukan
