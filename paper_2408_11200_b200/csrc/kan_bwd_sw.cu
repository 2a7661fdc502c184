// kan_bwd_sw.cu — KAN table gradient, fp64 accumulators resident in registers.
//
// Replaces the bwd closures of span_gather (layers.py:67-70: np.add.at of the window
// gradient) and edge_combine (layers.py:84-88) for the bounded grid:
//   A[i,r,o] = sum_{(b,j): cell_bi + j = r} w_j(b,i) * g[b,o]        (fp64 products and sums)
//   dC = scale * A,   dscale = sum_r C * A,   dbw = sum_b silu(x) * g  (base branch, 316-317)
//
// Roofline: 2*K FP64 flops per (b, i, o) -> FP64-FMA bound (34 TF/s measured);
// the fp64 accumulation is forced by the parity bar.
//
// Design (B200).  A CTA = 8 warps = 8 consecutive features x one 32*OV-output tile.  Each warp
// keeps the whole accumulator column A[i, 0..R-1, o..o+OV-1] of its feature in REGISTERS and
// streams the batch in sample order.  A sample's cell is warp-uniform, so `switch (cell)`
// compiles to one indirect branch into straight-line code that updates the statically
// indexed registers acc[cell .. cell+K-1] — no sort, no atomics, no shared-memory RMW; each
// (i, r, o) is owned by one thread and summed in sample order (deterministic).
// Per 64-sample chunk the CTA (a) stages g[chunk, o-tile] — already converted to fp64 by a
// one-pass kernel, so no conversion sits in the inner loop — with cp.async into a double
// buffer, and (b) evaluates the fp64 locate + basis once per (sample, feature) into a double-
// buffered shared-memory record; both happen while the warps sweep the previous chunk, with
// one barrier per chunk.  Per warp-sample the inner loop is the broadcast loads of (cell, w),
// one conflict-free load of g, the dispatch on the cell and K*OV DFMAs.
// Measured limits (tools/pipe_bw.cu): a broadcast LDS.128 costs ~2 SM cycles, so the operand
// delivery (w, cell, g: 52 B per lane per sample) bounds this kernel near 45% of FP64 peak.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace ukan {

template <int K, int RM, int OV, int R0>
__device__ __forceinline__ void sw_update(double (&acc)[RM][OV], const double (&w)[K], const double (&g)[OV]) {
  if constexpr (R0 + K <= RM) {
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int v = 0; v < OV; ++v) acc[R0 + j][v] = fma(w[j], g[v], acc[R0 + j][v]);
  }
}

#define UKAN_SW_CASE(r) \
  case r:               \
    sw_update<K, RM, OV, r>(acc, w, g); \
    break;
#define UKAN_SW_CASES8(b) \
  UKAN_SW_CASE(b + 0) UKAN_SW_CASE(b + 1) UKAN_SW_CASE(b + 2) UKAN_SW_CASE(b + 3) \
  UKAN_SW_CASE(b + 4) UKAN_SW_CASE(b + 5) UKAN_SW_CASE(b + 6) UKAN_SW_CASE(b + 7)

// acc[c + j][v] += w[j] * g[v].  NVVM lowers this to a compare-and-branch tree; a PTX jump
// table (brx.idx) was measured ~20x slower per sample on B200 (indexed LDC of the table).
template <int K, int RM, int OV>
__device__ __forceinline__ void sw_dispatch(int c, double (&acc)[RM][OV], const double (&w)[K], const double (&g)[OV]) {
  static_assert(RM <= 72, "extend the case list");
  switch (c) {
    UKAN_SW_CASES8(0)
    UKAN_SW_CASES8(8)
    UKAN_SW_CASES8(16)
    UKAN_SW_CASES8(24)
    UKAN_SW_CASES8(32)
    UKAN_SW_CASES8(40)
    UKAN_SW_CASES8(48)
    UKAN_SW_CASES8(56)
    UKAN_SW_CASES8(64)
    default:
      break;
  }
}

template <int K>
constexpr int sw_rec_bytes() { return (K * 8 + 4 + 15) / 16 * 16; }  // {double w[K]; int cell}

constexpr int kSwChunk = 96;  // samples per staged chunk (a multiple of 3 and 32)
constexpr int kSwFeat = 8;    // features (= warps) per CTA

__global__ void g_to_f64_kernel(const float* __restrict__ gy, double* __restrict__ g64, int64_t B, int d_out,
                                int d_pad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * d_pad) return;
  const int64_t b = t / d_pad;
  const int o = (int)(t % d_pad);
  g64[t] = o < d_out ? (double)gy[b * d_out + o] : 0.0;
}

__device__ __forceinline__ void cp_async4_zfill(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}

template <int K, int RM, int OV>
__global__ void __launch_bounds__(kSwFeat * 32, 1)
kan_bwd_sw_kernel(const float* __restrict__ x, const double* __restrict__ g64, const float* __restrict__ C,
                  const float* __restrict__ scale, float* __restrict__ dC, float* __restrict__ dscale,
                  float* __restrict__ dbw, double* __restrict__ part, double* __restrict__ part_b, int B,
                  int d_in, int d_out, int d_pad, int R, int sps, int has_base, KanGrid grid, Basis<K> bas) {
  constexpr int OT = 32 * OV;
  constexpr int REC = sw_rec_bytes<K>();
  constexpr int NREC = kSwChunk + 3;  // + two read-ahead pads (+1 spare)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* g_s = reinterpret_cast<double*>(smem_raw);                                 // [2][chunk+2][OT]
  unsigned char* rec_s = smem_raw + sizeof(double) * 2 * (kSwChunk + 2) * OT;        // [2][feat][NREC]
  double* sl_s = reinterpret_cast<double*>(rec_s + (size_t)2 * kSwFeat * NREC * REC);  // [2][feat][chunk]
  float* x_s = reinterpret_cast<float*>(sl_s + 2 * kSwFeat * kSwChunk);              // [2][chunk][feat]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * kSwFeat;
  const int i = i0 + warp;
  const int o0 = blockIdx.y * OT;
  const int z = blockIdx.z;
  const int b_lo = z * sps, b_hi = min(B, b_lo + sps);
  const int nch = (b_hi - b_lo + kSwChunk - 1) / kSwChunk;

  // g[chunk, o-tile] (fp64) and x[chunk, feature block] are staged with cp.async one and two
  // chunks ahead, so neither the sweep nor the locate waits on a global load.
  auto stage = [&](int ng, int nx) {
    if (ng < nch) {
      const int b0 = b_lo + ng * kSwChunk;
      constexpr int per_row = OT / 2;  // 16-byte pieces per sample row
      double* dst = g_s + (size_t)(ng & 1) * (kSwChunk + 2) * OT;
      for (int t = threadIdx.x; t < kSwChunk * per_row; t += blockDim.x) {
        const int s = t / per_row, q = t % per_row;
        const bool ok = b0 + s < b_hi;
        const double* src = g64 + (ok ? (size_t)(b0 + s) * d_pad + o0 + 2 * q : 0);
        cp_async16_zfill(dst + s * OT + 2 * q, src, ok ? 16 : 0);
      }
    }
    if (nx < nch) {
      const int b0 = b_lo + nx * kSwChunk;
      float* dst = x_s + (size_t)(nx & 1) * kSwChunk * kSwFeat;
      for (int t = threadIdx.x; t < kSwChunk * kSwFeat; t += blockDim.x) {
        const int s = t / kSwFeat, f = t % kSwFeat;
        const bool ok = b0 + s < b_hi && i0 + f < d_in;
        cp_async4_zfill(dst + t, x + (ok ? (size_t)(b0 + s) * d_in + i0 + f : 0), ok ? 4 : 0);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto prep = [&](int n) {  // fp64 locate + basis once per (sample, feature) of chunk n
    const int buf = n & 1;
    const int b0 = b_lo + n * kSwChunk;
    const float* xs = x_s + (size_t)buf * kSwChunk * kSwFeat;
#pragma unroll
    for (int q = 0; q < kSwFeat * kSwChunk / (kSwFeat * 32); ++q) {
      const int p = q * kSwFeat * 32 + threadIdx.x;
      const int f = p % kSwFeat, s = p / kSwFeat;
      unsigned char* rec = rec_s + ((size_t)(buf * kSwFeat + f) * NREC + s) * REC;
      int cell = 0;  // padding samples: cell 0 with zero weights (the jump table has no default)
      double w[K];
#pragma unroll
      for (int j = 0; j < K; ++j) w[j] = 0.0;
      double sl = 0.0;
      if (b0 + s < b_hi && i0 + f < d_in) {
        const float xv = xs[p];
        double u;
        bool mask;
        kan_locate(xv, grid, cell, u, mask);
        if (isnan(xv)) {  // the forward already raised for NaN input: contribute nothing
          cell = 0;
        } else {
          basis_weights<K>(bas, u, w);
        }
        if (has_base) sl = silu_d((double)xv);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) reinterpret_cast<double*>(rec)[j] = w[j];
      *reinterpret_cast<int*>(rec + 8 * K) = cell;
      sl_s[(buf * kSwFeat + f) * kSwChunk + s] = sl;
    }
  };

  double acc[RM][OV];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int v = 0; v < OV; ++v) acc[r][v] = 0.0;
  double bacc[OV];
#pragma unroll
  for (int v = 0; v < OV; ++v) bacc[v] = 0.0;

  for (int t = threadIdx.x; t < 2 * kSwFeat * 3; t += blockDim.x) {  // read-ahead pads
    unsigned char* rec = rec_s + ((size_t)(t / 3) * NREC + kSwChunk + t % 3) * REC;
    for (int q = 0; q < REC / 4; ++q) reinterpret_cast<int*>(rec)[q] = 0;
  }
  stage(0, 0);
  stage(nch, 1);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  if (nch > 0) prep(0);
  __syncthreads();
  for (int n = 0; n < nch; ++n) {
    const int buf = n & 1;
    stage(n + 1, n + 2);       // g of the next chunk, x of the one after
    if (n + 1 < nch) prep(n + 1);  // x of chunk n+1 landed during the previous iteration
    if (i < d_in) {
      const unsigned char* rec0 = rec_s + (size_t)(buf * kSwFeat + warp) * NREC * REC;
      const double* gp = g_s + (size_t)buf * (kSwChunk + 2) * OT + lane * OV;
      // three rotating operand sets: sample s+2's operands load while sample s's DFMAs issue
      int ca, cb, cc;
      double wa[K], wb[K], wc[K], ga[OV], gb[OV], gc[OV];
      auto load = [&](int s, int& c, double (&w)[K], double (&g)[OV]) {
        const unsigned char* r = rec0 + (size_t)s * REC;
        c = *reinterpret_cast<const int*>(r + 8 * K);
#pragma unroll
        for (int j = 0; j < K; ++j) w[j] = reinterpret_cast<const double*>(r)[j];
#pragma unroll
        for (int v = 0; v < OV; ++v) g[v] = gp[s * OT + v];
      };
      load(0, ca, wa, ga);
      load(1, cb, wb, gb);
#pragma unroll 1
      for (int s = 0; s < kSwChunk; s += 3) {
        load(s + 2, cc, wc, gc);
        sw_dispatch<K, RM, OV>(ca, acc, wa, ga);
        load(s + 3, ca, wa, ga);  // s+3, s+4 may be the sentinel / pad records (read, never used)
        sw_dispatch<K, RM, OV>(cb, acc, wb, gb);
        load(s + 4, cb, wb, gb);
        sw_dispatch<K, RM, OV>(cc, acc, wc, gc);
      }
      if (has_base) {
        const double* slp = sl_s + (buf * kSwFeat + warp) * kSwChunk;
        for (int s = 0; s < kSwChunk; ++s) {
          const double sl = slp[s];
#pragma unroll
          for (int v = 0; v < OV; ++v) bacc[v] = fma(sl, gp[s * OT + v], bacc[v]);
        }
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
  }
  if (i >= d_in) return;
#pragma unroll
  for (int v = 0; v < OV; ++v) {
    const int o = o0 + lane * OV + v;
    if (o >= d_out) continue;
    if (part != nullptr) {
      double* pp = part + ((size_t)z * d_in + i) * R * d_out + o;
#pragma unroll
      for (int r = 0; r < RM; ++r)
        if (r < R) pp[(size_t)r * d_out] = acc[r][v];
      if (has_base) part_b[((size_t)z * d_in + i) * d_out + o] = bacc[v];
    } else {
      const double sc = (double)scale[(size_t)i * d_out + o];
      double ds = 0.0;
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        if (r < R) {
          const size_t ci = ((size_t)i * R + r) * d_out + o;
          dC[ci] = (float)(sc * acc[r][v]);
          ds = fma((double)C[ci], acc[r][v], ds);
        }
      }
      dscale[(size_t)i * d_out + o] = (float)ds;
      if (has_base) dbw[(size_t)i * d_out + o] = (float)bacc[v];
    }
  }
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
__global__ void kan_bwd_reduce_kernel(const double* __restrict__ part, const double* __restrict__ part_b,
                                      const float* __restrict__ C, const float* __restrict__ scale,
                                      float* __restrict__ dC, float* __restrict__ dscale,
                                      float* __restrict__ dbw, int S, int d_in, int d_out, int R);
int kan_num_sms();

struct SwPlan {
  bool ok = false;
  int rm = 0, ov = 1, Z = 1, sps = 0, d_pad = 0;
  size_t smem = 0;
  int64_t g64_bytes = 0, part_bytes = 0;
};

SwPlan kan_bwd_sw_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base) {
  SwPlan p;
  if (K > 6 || B <= 0) return p;
  if (R <= 16) p.rm = 16;
  else if (R <= 36) p.rm = 36;
  else if (R <= 68) p.rm = 68;
  else return p;
  p.ov = p.rm == 16 ? 4 : (p.rm == 36 ? 2 : 1);
  if (d_out <= 32) p.ov = 1;  // narrow layers: one output per lane
  else if (d_out <= 64 && p.ov > 2) p.ov = 2;
  const int OT = 32 * p.ov;
  p.d_pad = (int)((d_out + OT - 1) / OT * OT);
  const int rec = (K * 8 + 4 + 15) / 16 * 16;
  p.smem = sizeof(double) * (size_t)2 * (kSwChunk + 2) * OT + (size_t)2 * kSwFeat * (kSwChunk + 3) * rec +
           sizeof(double) * (size_t)2 * kSwFeat * kSwChunk + sizeof(float) * (size_t)2 * kSwChunk * kSwFeat;
  const int sms = kan_num_sms();
  const int64_t base = ((d_in + kSwFeat - 1) / kSwFeat) * ((d_out + OT - 1) / OT);
  // Split the batch only when the grid is short of two waves (one CTA per SM): pick the split
  // with the best wave efficiency.  Depends on shapes only -> deterministic.
  int64_t Z = 1;
  if (base < 2 * (int64_t)sms) {
    const int64_t max_z = std::max<int64_t>(1, std::min<int64_t>(16, B / (4 * kSwChunk)));
    double best = -1.0;
    for (int64_t c = 1; c <= max_z; ++c) {
      const double waves = (double)(base * c) / sms;
      const double eff = waves / std::ceil(waves) * std::min(1.0, waves / 2.0);
      if (eff > best + 1e-9) { best = eff; Z = c; }
    }
  }
  p.sps = (int)(((B + Z - 1) / Z + kSwChunk - 1) / kSwChunk * kSwChunk);
  p.Z = (int)((B + p.sps - 1) / p.sps);
  p.g64_bytes = (int64_t)sizeof(double) * B * p.d_pad;
  p.part_bytes = p.Z > 1 ? (int64_t)sizeof(double) * p.Z * d_in * d_out * (R + (has_base ? 1 : 0)) : 0;
  p.ok = true;
  return p;
}

int64_t kan_bwd_sw_workspace(const SwPlan& p) { return p.ok ? ((p.g64_bytes + 255) / 256 * 256 + p.part_bytes) : 0; }

template <int K, int RM, int OV>
static int launch_sw(const float* x, const float* gy, const float* C, const float* scale, float* dC, float* dscale,
                     float* dbw, void* ws, int B, int d_in, int d_out, int R, const KanGrid& grid, const SwPlan& p,
                     cudaStream_t st) {
  const Basis<K> bas = make_basis<K>(K - 1);
  double* g64 = static_cast<double*>(ws);
  double* part = p.Z > 1 ? reinterpret_cast<double*>(static_cast<char*>(ws) + (p.g64_bytes + 255) / 256 * 256) : nullptr;
  double* part_b = (p.Z > 1 && dbw) ? part + (size_t)p.Z * d_in * R * d_out : nullptr;
  const int64_t n = (int64_t)B * p.d_pad;
  g_to_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gy, g64, B, d_out, p.d_pad);
  UKAN_LAUNCH_CHECK();
  auto kern = kan_bwd_sw_kernel<K, RM, OV>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 gridd((d_in + kSwFeat - 1) / kSwFeat, (d_out + 32 * OV - 1) / (32 * OV), p.Z);
  kern<<<gridd, kSwFeat * 32, p.smem, st>>>(x, g64, C, scale, dC, dscale, dbw, part, part_b, B, d_in, d_out, p.d_pad,
                                            R, p.sps, dbw != nullptr, grid, bas);
  UKAN_LAUNCH_CHECK();
  if (p.Z > 1) {
    const int64_t m = (int64_t)d_in * d_out;
    kan_bwd_reduce_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(part, part_b, C, scale, dC, dscale, dbw, p.Z,
                                                                       d_in, d_out, R);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

template <int K>
int kan_bwd_sw_run(const float* x, const float* gy, const float* C, const float* scale, float* dC, float* dscale,
                   float* dbw, void* ws, int B, int d_in, int d_out, int R, const KanGrid& grid, const SwPlan& p,
                   cudaStream_t st) {
  if constexpr (K <= 6) {
#define UKAN_SW_LAUNCH(RM_, OV_) \
  if (p.rm == RM_ && p.ov == OV_) return launch_sw<K, RM_, OV_>(x, gy, C, scale, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
    UKAN_SW_LAUNCH(16, 4)
    UKAN_SW_LAUNCH(16, 2)
    UKAN_SW_LAUNCH(16, 1)
    UKAN_SW_LAUNCH(36, 2)
    UKAN_SW_LAUNCH(36, 1)
    UKAN_SW_LAUNCH(68, 1)
#undef UKAN_SW_LAUNCH
  }
  return UKAN_E_ARG;
}

#define UKAN_SW_INST(K)                                                                                          \
  template int kan_bwd_sw_run<K>(const float*, const float*, const float*, const float*, float*, float*, float*, \
                                 void*, int, int, int, int, const KanGrid&, const SwPlan&, cudaStream_t);
UKAN_SW_INST(1) UKAN_SW_INST(2) UKAN_SW_INST(3) UKAN_SW_INST(4) UKAN_SW_INST(5) UKAN_SW_INST(6)
UKAN_SW_INST(7) UKAN_SW_INST(8) UKAN_SW_INST(9) UKAN_SW_INST(10) UKAN_SW_INST(11)

}  // namespace ukan
