// kan_narrow.cu — KAN forward and dx for narrow layers (d_out <= 32, e.g. the 256 -> 10 head
// of the MNIST-shaped stack, BASELINE configs[1]).
//
// Replaces kan_forward (layers.py:304-318) and the dx part of its backward (basis_features bwd
// layers.py:44-46 + clamp mask tensor.py:330-333 + base branch) when the output tile is too
// narrow for the TMEM gather (kan_fwd_tm.cu) or the per-feature output tiles of the table
// gradient kernels.  Mapping: lanes = 32 consecutive samples, the 8 warps of a CTA take
// features i = warp, warp+8, ...; every lane keeps its sample's d_out accumulators in
// registers, so the coefficient slab C[i] of the current feature (R x d_out floats) is shared
// by the whole warp through L1 and x is read once.  Forward: the 8 per-warp partial sums are
// combined through shared memory in warp order (deterministic).  dx: each (sample, feature)
// result is produced by one lane; a shared-memory tile turns the per-warp columns into
// coalesced row writes.
#include <algorithm>

#include "common.cuh"

namespace ukan {


template <int K, int DO, int NW>
__global__ void __launch_bounds__(NW * 32)
kan_fwd_narrow_kernel(const float* __restrict__ x, const float* __restrict__ C, const float* __restrict__ scale,
                      const float* __restrict__ bw, float* __restrict__ y, int B, int d_in, int d_out, int R,
                      KanGrid grid, Basis<K> bas, int32_t* __restrict__ err) {
  __shared__ float part[NW][32][DO + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 32 + lane;
  const bool live = b < B;
  float acc[DO];
#pragma unroll
  for (int o = 0; o < DO; ++o) acc[o] = 0.f;
  for (int i = warp; i < d_in; i += NW) {
    const float xv = live ? __ldg(x + (size_t)b * d_in + i) : 0.f;
    int cell;
    double u;
    bool mask;
    if (!kan_locate(xv, grid, cell, u, mask)) {
      if (err && live) atomicExch(err, 1);  // NaN: the reference raises IndexError (SURVEY gotcha 10)
      continue;
    }
    double wd[K];
    basis_weights<K>(bas, u, wd);
    float w[K];
#pragma unroll
    for (int j = 0; j < K; ++j) w[j] = (float)wd[j];
    const float* Ci = C + ((size_t)i * R + cell) * d_out;
    const float* si = scale + (size_t)i * d_out;
    const float sl = bw ? (float)silu_d((double)xv) : 0.f;
#pragma unroll
    for (int o = 0; o < DO; ++o) {
      if (o < d_out) {
        float t = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) t = fmaf(w[j], __ldg(Ci + (size_t)j * d_out + o), t);
        acc[o] = fmaf(__ldg(si + o), t, acc[o]);  // edge_combine order: scale * (sum_j w_j C)
        if (bw) acc[o] = fmaf(sl, __ldg(bw + (size_t)i * d_out + o), acc[o]);
      }
    }
  }
#pragma unroll
  for (int o = 0; o < DO; ++o) part[warp][lane][o] = acc[o];
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * d_out; t += blockDim.x) {
    const int s = t / d_out, o = t % d_out;
    const int bb = blockIdx.x * 32 + s;
    if (bb >= B) continue;
    float a = part[0][s][o];
#pragma unroll
    for (int w = 1; w < NW; ++w) a += part[w][s][o];
    y[(size_t)bb * d_out + o] = a;
  }
}

// dx[b,i] = mask * inv_dg * sum_j w'_j * sum_o g[b,o]*scale[i,o]*C[i,cell+j,o]
//           (+ dsilu(x) * sum_o g[b,o]*bw[i,o])      fp64 products and sums
template <int K, int DO, int NW>
__global__ void __launch_bounds__(NW * 32)
kan_dx_narrow2_kernel(const float* __restrict__ x, const float* __restrict__ C, const float* __restrict__ scale,
                      const float* __restrict__ bw, const float* __restrict__ gy, float* __restrict__ dx, int B,
                      int d_in, int d_out, int R, KanGrid grid, Basis<K> bas) {
  constexpr int FT = 64;  // features per output tile
  __shared__ float tile[32][FT + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 32 + lane;
  const bool live = b < B;
  double g[DO];
#pragma unroll
  for (int o = 0; o < DO; ++o) g[o] = (live && o < d_out) ? (double)__ldg(gy + (size_t)b * d_out + o) : 0.0;
  for (int f0 = 0; f0 < d_in; f0 += FT) {
    for (int fl = warp; fl < FT; fl += NW) {
      const int i = f0 + fl;
      float res = 0.f;
      if (i < d_in && live) {
        const float xv = __ldg(x + (size_t)b * d_in + i);
        int cell;
        double u;
        bool mask;
        if (kan_locate(xv, grid, cell, u, mask)) {
          double wp[K];
          basis_dweights<K>(bas, u, wp);
          const float* Ci = C + ((size_t)i * R + cell) * d_out;
          const float* si = scale + (size_t)i * d_out;
          double S[K];
#pragma unroll
          for (int j = 0; j < K; ++j) S[j] = 0.0;
          double sb = 0.0;
#pragma unroll
          for (int o = 0; o < DO; ++o) {
            if (o < d_out) {
              const double gs = g[o] * (double)__ldg(si + o);
#pragma unroll
              for (int j = 0; j < K; ++j) S[j] = fma(gs, (double)__ldg(Ci + (size_t)j * d_out + o), S[j]);
              if (bw) sb = fma(g[o], (double)__ldg(bw + (size_t)i * d_out + o), sb);
            }
          }
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < K; ++j) t = fma(S[j], wp[j], t);
          double d = mask ? t * grid.inv_dg : 0.0;
          if (bw) d += dsilu_d((double)xv) * sb;
          res = (float)d;
        }
      }
      tile[lane][fl] = res;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 32 * FT; t += blockDim.x) {
      const int s = t / FT, fl = t % FT;
      const int bb = blockIdx.x * 32 + s, i = f0 + fl;
      if (bb < B && i < d_in) dx[(size_t)bb * d_in + i] = tile[s][fl];
    }
    __syncthreads();
  }
}

template <int K>
int kan_fwd_narrow(const float* x, const float* C, const float* scale, const float* bw, float* y, int B, int d_in,
                   int d_out, int R, const KanGrid& grid, int32_t* err, cudaStream_t st) {
  if (B == 0) return UKAN_OK;
  const Basis<K> bas = make_basis<K>(K - 1);
  const dim3 g((B + 31) / 32);
  // 16 warps (more independent feature chains per sample block) where the partial-sum tile fits
  if (d_out <= 8) kan_fwd_narrow_kernel<K, 8, 16><<<g, 16 * 32, 0, st>>>(x, C, scale, bw, y, B, d_in, d_out, R, grid, bas, err);
  else if (d_out <= 16) kan_fwd_narrow_kernel<K, 16, 16><<<g, 16 * 32, 0, st>>>(x, C, scale, bw, y, B, d_in, d_out, R, grid, bas, err);
  else if (d_out <= 32) kan_fwd_narrow_kernel<K, 32, 8><<<g, 8 * 32, 0, st>>>(x, C, scale, bw, y, B, d_in, d_out, R, grid, bas, err);
  else return UKAN_E_ARG;
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

template <int K>
int kan_dx_narrow2(const float* x, const float* C, const float* scale, const float* bw, const float* gy, float* dx,
                   int B, int d_in, int d_out, int R, const KanGrid& grid, cudaStream_t st) {
  if (B == 0) return UKAN_OK;
  const Basis<K> bas = make_basis<K>(K - 1);
  const dim3 g((B + 31) / 32);
  if (d_out <= 8) kan_dx_narrow2_kernel<K, 8, 16><<<g, 16 * 32, 0, st>>>(x, C, scale, bw, gy, dx, B, d_in, d_out, R, grid, bas);
  else if (d_out <= 16) kan_dx_narrow2_kernel<K, 16, 16><<<g, 16 * 32, 0, st>>>(x, C, scale, bw, gy, dx, B, d_in, d_out, R, grid, bas);
  else if (d_out <= 32) kan_dx_narrow2_kernel<K, 32, 8><<<g, 8 * 32, 0, st>>>(x, C, scale, bw, gy, dx, B, d_in, d_out, R, grid, bas);
  else return UKAN_E_ARG;
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

#define UKAN_NARROW_INST(K)                                                                                      \
  template int kan_fwd_narrow<K>(const float*, const float*, const float*, const float*, float*, int, int, int,  \
                                 int, const KanGrid&, int32_t*, cudaStream_t);                                   \
  template int kan_dx_narrow2<K>(const float*, const float*, const float*, const float*, const float*, float*,   \
                                 int, int, int, int, const KanGrid&, cudaStream_t);
UKAN_NARROW_INST(1) UKAN_NARROW_INST(2) UKAN_NARROW_INST(3) UKAN_NARROW_INST(4) UKAN_NARROW_INST(5)
UKAN_NARROW_INST(6) UKAN_NARROW_INST(7) UKAN_NARROW_INST(8) UKAN_NARROW_INST(9) UKAN_NARROW_INST(10)
UKAN_NARROW_INST(11)

}  // namespace ukan
