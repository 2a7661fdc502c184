// kan_small.cu — KAN forward and table gradient for small layers (BASELINE configs[0]: 64 -> 64,
// G = 10, B = 1024): the tiled kernels keep a handful of CTAs walking every feature with barriers
// between shared-memory stages (65 us each for a 17 MFLOP pass), so a small layer runs latency-
// bound on a few SMs.  Here every launch spreads over >= 256 CTAs instead.
//
// Replaces kan_forward (layers.py:304-318) and the bwd closures of span_gather (67-70) and
// edge_combine (84-88) for k = 3 without the base branch when d_in * d_out <= 2^14:
//   forward   CTA = 2 samples: fp64 locate (reference expression order, layers.py:294-301) and
//             fp64 basis for its 2 x d_in pairs into shared memory, then one thread per (feature
//             quarter, output): p_q = sum_{i in q} scale * (sum_j w_j C[i, cell+j, o]) in feature
//             order for both samples, y = ((p_0 + p_1) + p_2) + p_3 (fp32);
//   records   one thread per (sample, feature) -> cell and fp64 w[4], feature-major (backward);
//   table     cluster of 8 CTAs per (feature, 64 outputs), 32 sample splits of 64 threads: each
//             thread accumulates its R rows A[r] = sum_b w_{r-cell_b} g[b, o] in fp64 over its
//             samples in order (shared memory, 4 samples' loads in flight), the splits are added in
//             order (across the cluster through distributed shared memory), dC = scale * A and
//             dscale = sum_r C * A.  Fixed order everywhere: deterministic.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ukan {

constexpr int kSmThreads = 256;
constexpr int kSmFwdS = 2;     // samples per forward CTA
constexpr int kSmFq = 4;       // feature quarters per forward CTA (x 64 output lanes = 256 threads)
constexpr int kSmSub = 4;      // sample splits per table-gradient CTA (x 64 outputs = 256 threads)
constexpr int kSmCl = 8;       // CTAs per table-gradient cluster (portable maximum)

__global__ void __launch_bounds__(kSmThreads)
kan_small_fwd_kernel(const float* __restrict__ x, const float* __restrict__ C, const float* __restrict__ scale,
                     float* __restrict__ y, int B, int d_in, int d_out, int R, KanGrid grid, Basis<4> bas,
                     int32_t* __restrict__ err) {
  extern __shared__ float4 fw_s[];  // [kSmFwdS * d_in] weights, then the cells, then the partials
  int* cell_s = reinterpret_cast<int*>(fw_s + kSmFwdS * d_in);
  float* part_s = reinterpret_cast<float*>(cell_s + kSmFwdS * d_in);  // [kSmFwdS][kSmFq][d_out]
  const int b0 = blockIdx.x * kSmFwdS;
  for (int p = threadIdx.x; p < kSmFwdS * d_in; p += blockDim.x) {
    const int b = b0 + p / d_in, i = p % d_in;
    int cell = 0;
    double u = 0.0;
    bool mask;
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    if (b < B) {
      if (kan_locate(x[(size_t)b * d_in + i], grid, cell, u, mask)) {
        basis_weights<4>(bas, u, w);
      } else {
        cell = 0;
        if (err) atomicExch(err, 1);  // NaN: the reference raises IndexError (SURVEY gotcha 10)
      }
    }
    fw_s[p] = make_float4((float)w[0], (float)w[1], (float)w[2], (float)w[3]);
    cell_s[p] = cell;
  }
  __syncthreads();
  // thread = (feature quarter fq, output lane): partial sums over its features in order
  const int fq = threadIdx.x >> 6, lane = threadIdx.x & 63;
  const int f_lo = (int)((int64_t)d_in * fq / kSmFq), f_hi = (int)((int64_t)d_in * (fq + 1) / kSmFq);
  for (int o = lane; o < d_out; o += 64) {
    float acc[kSmFwdS];
#pragma unroll
    for (int s = 0; s < kSmFwdS; ++s) acc[s] = 0.f;
#pragma unroll 2
    for (int i = f_lo; i < f_hi; ++i) {
      const float sc = __ldg(scale + (size_t)i * d_out + o);
      const float* Ci = C + (size_t)i * R * d_out + o;
#pragma unroll
      for (int s = 0; s < kSmFwdS; ++s) {
        const float4 w = fw_s[s * d_in + i];
        const float* Cc = Ci + (size_t)cell_s[s * d_in + i] * d_out;
        float t = 0.f;
        t = fmaf(w.x, __ldg(Cc), t);
        t = fmaf(w.y, __ldg(Cc + d_out), t);
        t = fmaf(w.z, __ldg(Cc + 2 * (size_t)d_out), t);
        t = fmaf(w.w, __ldg(Cc + 3 * (size_t)d_out), t);
        acc[s] = fmaf(sc, t, acc[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < kSmFwdS; ++s) part_s[(s * kSmFq + fq) * d_out + o] = acc[s];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kSmFwdS * d_out; q += blockDim.x) {
    const int s = q / d_out, o = q % d_out;
    if (b0 + s >= B) break;
    float a = part_s[(s * kSmFq) * d_out + o];
#pragma unroll
    for (int f = 1; f < kSmFq; ++f) a += part_s[(s * kSmFq + f) * d_out + o];
    y[(size_t)(b0 + s) * d_out + o] = a;
  }
}

__global__ void __launch_bounds__(kSmThreads)
kan_small_records_kernel(const float* __restrict__ x, int* __restrict__ cell_out, double* __restrict__ w_out, int B,
                         int d_in, KanGrid grid, Basis<4> bas) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * d_in) return;
  const int i = (int)(t / B), b = (int)(t % B);
  int cell = 0;
  double u = 0.0;
  bool mask;
  double w[4] = {0.0, 0.0, 0.0, 0.0};
  if (kan_locate(x[(size_t)b * d_in + i], grid, cell, u, mask)) basis_weights<4>(bas, u, w);
  else cell = 0;  // NaN contributes nothing (the forward raised the flag)
  cell_out[t] = cell;
  double2* wd = reinterpret_cast<double2*>(w_out + (size_t)t * 4);
  wd[0] = make_double2(w[0], w[1]);
  wd[1] = make_double2(w[2], w[3]);
}

// Table gradient: a cluster of kSmCl CTAs per (feature i, 64 outputs), each CTA kSmSub sample
// splits of 64 threads; the cluster's split rows are added in order through distributed shared
// memory by CTA rank 0, which writes dC and dscale.
template <int P>
struct SmallRec {
  int c[P];
  double2 w01[P], w23[P];
  float g[P];
};

__global__ void __launch_bounds__(kSmThreads)
kan_small_tablegrad_kernel(const int* __restrict__ cell, const double* __restrict__ w, const float* __restrict__ gy,
                           const float* __restrict__ C, const float* __restrict__ scale, float* __restrict__ dC,
                           float* __restrict__ dscale, int B, int d_in, int d_out, int R) {
  extern __shared__ double A_s[];  // [R][kSmThreads]: each thread's row accumulators
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int i = blockIdx.x;
  const int ol = threadIdx.x & 63, sub = threadIdx.x >> 6;
  const int o = blockIdx.y * 64 + ol;
  double* A = A_s + threadIdx.x;
  for (int r = 0; r < R; ++r) A[r * kSmThreads] = 0.0;
  const int nsplit = kSmSub * kSmCl;
  const int per = (B + nsplit - 1) / nsplit;
  const int lo = min(B, (rank * kSmSub + sub) * per), hi = min(B, lo + per);
  if (o < d_out && lo < hi) {
    const int* cl = cell + (size_t)i * B;
    const double2* wr = reinterpret_cast<const double2*>(w + (size_t)i * B * 4);
    const float* gp = gy + o;
    constexpr int P = 4;  // samples in flight: the loads do not wait for the shared-memory updates
    const int nfull = lo + (hi - lo) / P * P;
    for (int b0 = lo; b0 < nfull; b0 += P) {
      SmallRec<P> q;
#pragma unroll
      for (int j = 0; j < P; ++j) {
        q.c[j] = __ldg(cl + b0 + j);
        q.w01[j] = __ldg(wr + 2 * (size_t)(b0 + j));
        q.w23[j] = __ldg(wr + 2 * (size_t)(b0 + j) + 1);
        q.g[j] = __ldg(gp + (size_t)(b0 + j) * d_out);
      }
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const double g = (double)q.g[j];
        double* Ac = A + (size_t)q.c[j] * kSmThreads;
        Ac[0] = fma(q.w01[j].x, g, Ac[0]);
        Ac[kSmThreads] = fma(q.w01[j].y, g, Ac[kSmThreads]);
        Ac[2 * kSmThreads] = fma(q.w23[j].x, g, Ac[2 * kSmThreads]);
        Ac[3 * kSmThreads] = fma(q.w23[j].y, g, Ac[3 * kSmThreads]);
      }
    }
    for (int b = nfull; b < hi; ++b) {
      const double2 w01 = __ldg(wr + 2 * (size_t)b), w23 = __ldg(wr + 2 * (size_t)b + 1);
      const double g = (double)__ldg(gp + (size_t)b * d_out);
      double* Ac = A + (size_t)__ldg(cl + b) * kSmThreads;
      Ac[0] = fma(w01.x, g, Ac[0]);
      Ac[kSmThreads] = fma(w01.y, g, Ac[kSmThreads]);
      Ac[2 * kSmThreads] = fma(w23.x, g, Ac[2 * kSmThreads]);
      Ac[3 * kSmThreads] = fma(w23.y, g, Ac[3 * kSmThreads]);
    }
  }
  __syncthreads();
  // this CTA's splits, in order, into split 0's slots
  for (int t = threadIdx.x; t < R * 64; t += kSmThreads) {
    const int r = t >> 6, l = t & 63;
    double a = A_s[(size_t)r * kSmThreads + l];
#pragma unroll
    for (int s2 = 1; s2 < kSmSub; ++s2) a += A_s[(size_t)r * kSmThreads + s2 * 64 + l];
    A_s[(size_t)r * kSmThreads + l] = a;
  }
  cluster.sync();
  if (rank == 0) {
    for (int t = threadIdx.x; t < R * 64; t += kSmThreads) {
      const int r = t >> 6, l = t & 63, oo = blockIdx.y * 64 + l;
      double a = A_s[(size_t)r * kSmThreads + l];
#pragma unroll
      for (int q2 = 1; q2 < kSmCl; ++q2) a += cluster.map_shared_rank(A_s, q2)[(size_t)r * kSmThreads + l];
      A_s[(size_t)r * kSmThreads + l] = a;
      if (oo < d_out) dC[((size_t)i * R + r) * d_out + oo] = (float)((double)scale[(size_t)i * d_out + oo] * a);
    }
  }
  cluster.sync();  // the other CTAs' shared memory stays alive until rank 0 has read it
  if (rank == 0 && threadIdx.x < 64 && o < d_out) {
    double ds = 0.0;
    for (int r = 0; r < R; ++r) ds = fma((double)C[((size_t)i * R + r) * d_out + o], A_s[(size_t)r * kSmThreads + ol], ds);
    dscale[(size_t)i * d_out + o] = (float)ds;
  }
}

bool kan_small_ok(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base) {
  static const bool off = getenv("UKAN_SMALL") && getenv("UKAN_SMALL")[0] == '0';  // A/B only
  if (off || k != 3 || has_base || B < 1) return false;
  // measured (profiles/r02/kbench_small.txt): faster than the tiled kernels at cfg1 (1024 x 64 x 64)
  // and 1024 x 32 x 128, slower at 256 x 128 x 128 and from 2048 x 64 x 64 on
  return d_out > 32 && d_in <= 64 && d_in * d_out <= (1 << 14) && B * d_in * d_out <= (int64_t)6 << 20 &&
         (G + 3) * kSmThreads * 8 <= 200 * 1024 && kSmFwdS * (kSmFq * d_out * 4 + d_in * 20) <= 200 * 1024;
}

int64_t kan_small_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t G) { return B * d_in * 36 + 256; }

struct SmallWs {
  double* w;
  int* cell;
};
static const int* cell_cp(const SmallWs& s) { return s.cell; }
static const double* w_cp(const SmallWs& s) { return s.w; }
static SmallWs small_split(void* ws, int64_t B, int64_t d_in) {
  SmallWs s;
  s.w = reinterpret_cast<double*>(ws);
  s.cell = reinterpret_cast<int*>(s.w + (size_t)B * d_in * 4);
  return s;
}

int kan_small_forward(const float* x, const float* C, const float* scale, float* y, int B, int d_in, int d_out, int G,
                      const KanGrid& grid, int32_t* err, cudaStream_t st) {
  const size_t smem = (size_t)kSmFwdS * d_in * (sizeof(float4) + sizeof(int)) + (size_t)kSmFwdS * kSmFq * d_out * 4;
  if (smem > 48 * 1024)
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kan_small_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kan_small_fwd_kernel<<<(unsigned)((B + kSmFwdS - 1) / kSmFwdS), kSmThreads, smem, st>>>(
      x, C, scale, y, B, d_in, d_out, G + 3, grid, make_basis<4>(3), err);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

int kan_small_records(const float* x, void* ws, int B, int d_in, const KanGrid& grid, cudaStream_t st) {
  const SmallWs s = small_split(ws, B, d_in);
  const int64_t n = (int64_t)B * d_in;
  kan_small_records_kernel<<<(unsigned)((n + kSmThreads - 1) / kSmThreads), kSmThreads, 0, st>>>(
      x, s.cell, s.w, B, d_in, grid, make_basis<4>(3));
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

int kan_small_tablegrad(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                        void* ws, int B, int d_in, int d_out, int G, const KanGrid& grid, bool prepared,
                        cudaStream_t st) {
  if (!prepared) {
    const int rc = kan_small_records(x, ws, B, d_in, grid, st);
    if (rc) return rc;
  }
  const SmallWs s = small_split(ws, B, d_in);
  const int R = G + 3;
  const size_t smem = sizeof(double) * (size_t)R * kSmThreads;
  if (smem > 48 * 1024)
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kan_small_tablegrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)d_in, (unsigned)((d_out + 63) / 64), kSmCl);
  cfg.blockDim = dim3(kSmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = kSmCl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  UKAN_CUDA_TRY(cudaLaunchKernelEx(&cfg, kan_small_tablegrad_kernel, cell_cp(s), w_cp(s), gy, C, scale, dC, dscale, B,
                                   d_in, d_out, R));
  return UKAN_OK;
}

}  // namespace ukan
