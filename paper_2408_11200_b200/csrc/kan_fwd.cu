// kan_fwd.cu — KAN forward with shared-memory coefficient slabs (cp.async double buffering).
//
// Replaces kan_forward (layers.py:304-318): _kan_locate (294-301) + span_gather (57-75) +
// basis_features (40-54) + edge_combine (78-105) (+ silu base branch 316-317), fused.
//
// CTA tile = 128 samples x OT outputs (OT = 128 or 64, four consecutive outputs per thread),
// 256 threads, each thread owning S = 128*4*TO/256... = 128/TS samples in registers.  The
// CTA walks d_in two features per pipeline stage: while stage n is consumed, the slab
// coeffs[i, 0:G+k, o0:o0+OT] of the next two features (and their scale / base rows) streams
// into the other shared-memory buffer with cp.async, and the threads evaluate the next
// stage's per-(sample, feature) locate (fp64, reference expression order) and basis weights
// (fp64 -> fp32).  The window rows are then read conflict-free from shared memory with
// 128-bit loads:  y[b,o] += scale[i,o] * sum_j w_j * C[i, cell+j, o]   (fp32, edge_combine
// order).  Each 128-sample tile re-reads a feature's slab once from L2 (instead of once per
// 32 samples in the first version).
#include "common.cuh"

namespace ukan {

constexpr int kF2FC = 2;
constexpr int kF2BT = 128;

__device__ __forceinline__ void f2_cp16(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void f2_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void f2_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

template <int K>
struct F2Layout {
  static constexpr int KP = (K + 3) / 4 * 4;  // weights padded to float4
};

template <int K, int OT>
__global__ void __launch_bounds__(256, 2)
kan_fwd_v2_kernel(const float* __restrict__ x, const float* __restrict__ C,
                  const float* __restrict__ scale, const float* __restrict__ bw,
                  float* __restrict__ y, int B, int d_in, int d_out, int R, KanGrid grid,
                  Basis<K> bas, int32_t* __restrict__ err) {
  constexpr int TO = OT / 4;
  constexpr int TS = 256 / TO;
  constexpr int S = kF2BT / TS;
  constexpr int KP = F2Layout<K>::KP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const bool has_base = bw != nullptr;
  // per buffer: slab [FC][R][OT] | sc [FC][OT] | bwr [FC][OT] | w [FC][BT][KP] | sl [FC][BT] | cell [FC][BT]
  const size_t slab_f = (size_t)kF2FC * R * OT;
  const size_t buf_f = slab_f + 2 * kF2FC * OT + (size_t)kF2FC * kF2BT * (KP + 1) + kF2FC * kF2BT;
  float* buf0 = reinterpret_cast<float*>(smem_raw);

  const int tid = threadIdx.x;
  const int tx = tid % TO, ty = tid / TO;
  const int b0 = blockIdx.x * kF2BT;
  const int o0 = blockIdx.y * OT;
  const int o = o0 + tx * 4;
  const bool o_ok = o < d_out;
  const int nstage = (d_in + kF2FC - 1) / kF2FC;

  auto issue = [&](int n) {
    float* bf = buf0 + (size_t)(n & 1) * buf_f;
    float* slab = bf;
    float* sc = bf + slab_f;
    float* bwr = sc + kF2FC * OT;
    const int q = OT / 4;
    for (int t = tid; t < kF2FC * R * q; t += 256) {
      const int f = t / (R * q), rem = t % (R * q);
      const int r = rem / q, oc = (rem % q) * 4;
      const int i = n * kF2FC + f;
      const int oo = o0 + oc;
      const int bytes = (i < d_in) ? max(0, min(4, d_out - oo)) * 4 : 0;
      const float* src = bytes ? C + ((size_t)i * R + r) * d_out + oo : C;
      f2_cp16(slab + ((size_t)f * R + r) * OT + oc, src, bytes);
    }
    for (int t = tid; t < kF2FC * q * (has_base ? 2 : 1); t += 256) {
      const int which = t / (kF2FC * q), rem = t % (kF2FC * q);
      const int f = rem / q, oc = (rem % q) * 4;
      const int i = n * kF2FC + f;
      const int oo = o0 + oc;
      const int bytes = (i < d_in) ? max(0, min(4, d_out - oo)) * 4 : 0;
      const float* base = which ? bw : scale;
      const float* src = bytes ? base + (size_t)i * d_out + oo : base;
      f2_cp16((which ? bwr : sc) + f * OT + oc, src, bytes);
    }
  };
  auto meta = [&](int n) {
    float* bf = buf0 + (size_t)(n & 1) * buf_f;
    float* wv = bf + slab_f + 2 * kF2FC * OT;
    float* sl = wv + kF2FC * kF2BT * KP;
    int* cell_s = reinterpret_cast<int*>(sl + kF2FC * kF2BT);
    for (int t = tid; t < kF2FC * kF2BT; t += 256) {
      const int s = t / kF2FC, f = t % kF2FC;
      const int b = b0 + s, i = n * kF2FC + f;
      int cell = -1;
      if (b < B && i < d_in) {
        const float xv = x[(size_t)b * d_in + i];
        double u;
        bool mask;
        if (!kan_locate(xv, grid, cell, u, mask)) {
          if (err) atomicExch(err, 1);
          cell = 0;
          u = 0.0;
        }
        double w[K];
        basis_weights<K>(bas, u, w);
#pragma unroll
        for (int j = 0; j < KP; ++j) wv[((size_t)f * kF2BT + s) * KP + j] = j < K ? (float)w[j] : 0.f;
        if (has_base) sl[f * kF2BT + s] = (float)silu_d((double)xv);
      }
      cell_s[f * kF2BT + s] = cell;
    }
  };

  float acc[S][4];
#pragma unroll
  for (int r = 0; r < S; ++r)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[r][v] = 0.f;

  issue(0);
  f2_commit();
  meta(0);
  for (int n = 0; n < nstage; ++n) {
    if (n + 1 < nstage) {
      issue(n + 1);
      meta(n + 1);
    }
    f2_commit();
    f2_wait1();
    __syncthreads();
    const float* bf = buf0 + (size_t)(n & 1) * buf_f;
    const float* slab = bf;
    const float* sc = bf + slab_f;
    const float* bwr = sc + kF2FC * OT;
    const float* wv = bwr + kF2FC * OT;
    const float* sl = wv + kF2FC * kF2BT * KP;
    const int* cell_s = reinterpret_cast<const int*>(sl + kF2FC * kF2BT);
    if (o_ok) {
#pragma unroll
      for (int f = 0; f < kF2FC; ++f) {
        if (n * kF2FC + f >= d_in) break;
        const float4 s4 = *reinterpret_cast<const float4*>(sc + f * OT + tx * 4);
        float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (has_base) b4 = *reinterpret_cast<const float4*>(bwr + f * OT + tx * 4);
        const float* slab_f0 = slab + (size_t)f * R * OT + tx * 4;
#pragma unroll
        for (int r = 0; r < S; ++r) {
          const int s = ty + TS * r;
          const int c = cell_s[f * kF2BT + s];
          if (c < 0) continue;
          const float* wp = wv + ((size_t)f * kF2BT + s) * KP;
          float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const float wj = wp[j];
            const float4 cv = *reinterpret_cast<const float4*>(slab_f0 + (size_t)(c + j) * OT);
            t0 = fmaf(wj, cv.x, t0);
            t1 = fmaf(wj, cv.y, t1);
            t2 = fmaf(wj, cv.z, t2);
            t3 = fmaf(wj, cv.w, t3);
          }
          acc[r][0] = fmaf(s4.x, t0, acc[r][0]);
          acc[r][1] = fmaf(s4.y, t1, acc[r][1]);
          acc[r][2] = fmaf(s4.z, t2, acc[r][2]);
          acc[r][3] = fmaf(s4.w, t3, acc[r][3]);
          if (has_base) {
            const float slv = sl[f * kF2BT + s];
            acc[r][0] = fmaf(slv, b4.x, acc[r][0]);
            acc[r][1] = fmaf(slv, b4.y, acc[r][1]);
            acc[r][2] = fmaf(slv, b4.z, acc[r][2]);
            acc[r][3] = fmaf(slv, b4.w, acc[r][3]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (!o_ok) return;
#pragma unroll
  for (int r = 0; r < S; ++r) {
    const int b = b0 + ty + TS * r;
    if (b >= B) continue;
    float* yr = y + (size_t)b * d_out + o;
    if (o + 4 <= d_out) {
      *reinterpret_cast<float4*>(yr) = make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (o + v < d_out) yr[v] = acc[r][v];
    }
  }
}

template <int K>
static size_t f2_smem(int R, int OT) {
  constexpr int KP = F2Layout<K>::KP;
  const size_t buf_f = (size_t)kF2FC * R * OT + 2 * kF2FC * OT + (size_t)kF2FC * kF2BT * (KP + 1) + kF2FC * kF2BT;
  return 2 * buf_f * sizeof(float);
}

// Returns UKAN_E_ARG when the shape is not served by this kernel (caller falls back).
template <int K>
int kan_fwd_v2(const float* x, const float* C, const float* scale, const float* bw, float* y, int B, int d_in,
               int d_out, int R, const KanGrid& grid, int32_t* err, cudaStream_t st) {
  if (d_out % 4 != 0 || d_out < 32) return UKAN_E_ARG;
  const Basis<K> bas = make_basis<K>(K - 1);
  const int OT = (d_out >= 128 && R <= 40) ? 128 : 64;
  const size_t smem = f2_smem<K>(R, OT);
  if (smem > 110 * 1024) return UKAN_E_ARG;
  dim3 gridd((B + kF2BT - 1) / kF2BT, (d_out + OT - 1) / OT);
  if (OT == 128) {
    auto kern = kan_fwd_v2_kernel<K, 128>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<gridd, 256, smem, st>>>(x, C, scale, bw, y, B, d_in, d_out, R, grid, bas, err);
  } else {
    auto kern = kan_fwd_v2_kernel<K, 64>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<gridd, 256, smem, st>>>(x, C, scale, bw, y, B, d_in, d_out, R, grid, bas, err);
  }
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

#define UKAN_F2_INST(K)                                                                                      \
  template int kan_fwd_v2<K>(const float*, const float*, const float*, const float*, float*, int, int, int, \
                             int, const KanGrid&, int32_t*, cudaStream_t);
UKAN_F2_INST(1) UKAN_F2_INST(2) UKAN_F2_INST(3) UKAN_F2_INST(4) UKAN_F2_INST(5) UKAN_F2_INST(6)
UKAN_F2_INST(7) UKAN_F2_INST(8) UKAN_F2_INST(9) UKAN_F2_INST(10) UKAN_F2_INST(11)

}  // namespace ukan
