// kan_bwd.cu — KAN backward (table side) with register-resident fp64 accumulators.
//
// Replaces the bwd closures of span_gather (layers.py:67-70: np.add.at scatter of the window
// gradient) and edge_combine (84-88) for the bounded grid:
//   A[i,r,o] = sum_{(b,j): cell_bi + j = r} w_j(b,i) * g[b,o]   (fp64 products / sums)
//   dC = scale * A,   dscale = sum_r C * A,   dbw = sum_b silu(x) * g.
//
// B200 design.  A warp owns one feature i and 32*OV consecutive outputs and keeps the whole
// accumulator column A[i, 0..R-1, o] in REGISTERS (R <= RMAX, fp64).  It streams the batch in
// sample order; the sample's cell c is warp-uniform, so a `switch (c)` (a jump table: one
// indirect branch per sample) selects code that updates the statically-indexed registers
// acc[c .. c+K-1] — no sort, no shared-memory read-modify-write, no atomics.  Each (i,r,o)
// is owned by exactly one thread and summed in a fixed order, so the result is deterministic.
// Per 128-sample chunk the CTA stages g[chunk, o-tile] and x[chunk, feature-tile] in shared
// memory and evaluates (fp64 locate, fp64 basis) once per (sample, feature) for all the warps
// that share the feature.  Small layers split the batch over blockIdx.z into fp64 partials
// that a second kernel reduces in fixed order (deterministic), so the grid fills 148 SMs.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace ukan {

constexpr int kRegBC = 128;

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 4 : 0));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage g[b0:b0+nb, o0:o0+OPB] and x[b0:b0+nb, i0:i0+FPB] with cp.async (zero-filled tails).
__device__ __forceinline__ void stage_chunk(float* g_s, float* x_s, const float* __restrict__ gy,
                                           const float* __restrict__ x, int b0, int nb, int o0, int OPB,
                                           int d_out, int i0, int FPB, int d_in) {
  if ((d_out & 3) == 0) {
    const int q = OPB / 4;
    for (int t = threadIdx.x; t < kRegBC * q; t += blockDim.x) {
      const int s = t / q, oc = (t % q) * 4;
      const int o = o0 + oc;
      const int valid = (s < nb) ? max(0, min(4, d_out - o)) * 4 : 0;
      const float* src = gy + (valid ? (size_t)(b0 + s) * d_out + o : 0);
      cp_async16(g_s + (size_t)s * OPB + oc, src, valid);
    }
  } else {
    for (int t = threadIdx.x; t < kRegBC * OPB; t += blockDim.x) {
      const int s = t / OPB, oc = t % OPB;
      const int o = o0 + oc;
      const bool ok = s < nb && o < d_out;
      cp_async4(g_s + t, gy + (ok ? (size_t)(b0 + s) * d_out + o : 0), ok);
    }
  }
  for (int t = threadIdx.x; t < kRegBC * FPB; t += blockDim.x) {
    const int s = t / FPB, f = t % FPB;
    const bool ok = s < nb && i0 + f < d_in;
    cp_async4(x_s + t, x + (ok ? (size_t)(b0 + s) * d_in + i0 + f : 0), ok);
  }
}

template <int K, int RMAX, int OV, int R0>
__device__ __forceinline__ void acc_update(double (&acc)[RMAX][OV], const double (&w)[K],
                                           const double (&g)[OV]) {
  if constexpr (R0 + K <= RMAX) {
#pragma unroll
    for (int j = 0; j < K; ++j)
#pragma unroll
      for (int v = 0; v < OV; ++v) acc[R0 + j][v] = fma(w[j], g[v], acc[R0 + j][v]);
  }
}

#define UKAN_BWD_CASE(r) \
  case r:                \
    acc_update<K, RMAX, OV, r>(acc, w, g); \
    break;

template <int K, int RMAX, int OV>
__global__ void __launch_bounds__(256, (RMAX * OV <= 40 ? 2 : 1))
kan_bwd_reg_kernel(const float* __restrict__ x, const float* __restrict__ C,
                   const float* __restrict__ scale, const float* __restrict__ gy,
                   float* __restrict__ dC, float* __restrict__ dscale, float* __restrict__ dbw,
                   double* __restrict__ part, double* __restrict__ part_b, int B, int d_in,
                   int d_out, int R, int FPB, int WPF, int sps, int has_base, KanGrid grid,
                   Basis<K> bas) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int OPB = WPF * 32 * OV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int fl = warp / WPF, ot = warp % WPF;
  const int i0 = blockIdx.x * FPB;
  const int i = i0 + fl;
  const int o0 = blockIdx.y * OPB;
  const int ol = ot * 32 * OV + lane * OV;  // output offset inside the CTA tile
  const int z = blockIdx.z;
  const int b_lo = z * sps, b_hi = min(B, b_lo + sps);

  // shared layout
  double* w_s = reinterpret_cast<double*>(smem_raw);          // [FPB][BC][K]
  double* g64 = w_s + (size_t)FPB * kRegBC * K;                // [BC][OPB]  fp64 copy of the chunk
  double* sl_s = g64 + (size_t)kRegBC * OPB;                   // [FPB][BC]  (only with the base branch)
  float* g_s0 = reinterpret_cast<float*>(sl_s + (has_base ? (size_t)FPB * kRegBC : 0));  // 2 x [BC][OPB]
  float* x_s0 = g_s0 + (size_t)2 * kRegBC * OPB;               // 2 x [BC][FPB]
  int* c_s = reinterpret_cast<int*>(x_s0 + 2 * kRegBC * FPB);  // [FPB][BC]   cell of sample s

  double acc[RMAX][OV];
#pragma unroll
  for (int r = 0; r < RMAX; ++r)
#pragma unroll
    for (int v = 0; v < OV; ++v) acc[r][v] = 0.0;
  double bacc[OV];
#pragma unroll
  for (int v = 0; v < OV; ++v) bacc[v] = 0.0;

  const int nchunks = (b_hi - b_lo + kRegBC - 1) / kRegBC;
  if (nchunks > 0)
    stage_chunk(g_s0, x_s0, gy, x, b_lo, min(kRegBC, b_hi - b_lo), o0, OPB, d_out, i0, FPB, d_in);
  cp_async_commit();
  for (int n = 0; n < nchunks; ++n) {
    const int b0 = b_lo + n * kRegBC;
    const int nb = min(kRegBC, b_hi - b0);
    const float* g_s = g_s0 + (size_t)(n & 1) * kRegBC * OPB;
    const float* x_s = x_s0 + (size_t)(n & 1) * kRegBC * FPB;
    if (n + 1 < nchunks) {  // prefetch the next chunk into the other buffer
      const int b1 = b0 + kRegBC;
      stage_chunk(g_s0 + (size_t)((n + 1) & 1) * kRegBC * OPB, x_s0 + (size_t)((n + 1) & 1) * kRegBC * FPB, gy,
                  x, b1, min(kRegBC, b_hi - b1), o0, OPB, d_out, i0, FPB, d_in);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    // (1) g chunk -> fp64 once per CTA (shared by the FPB features); (2) per (sample, feature)
    //     fp64 locate + basis, once for all warps of the feature
    for (int t = threadIdx.x; t < kRegBC * OPB; t += blockDim.x) g64[t] = (double)g_s[t];
    for (int t = threadIdx.x; t < kRegBC * FPB; t += blockDim.x) {
      const int f = t / kRegBC, s = t % kRegBC;
      const float xv = x_s[s * FPB + f];
      int cell;
      double u;
      bool mask;
      kan_locate(xv, grid, cell, u, mask);
      double w[K];
      basis_weights<K>(bas, u, w);
#pragma unroll
      for (int j = 0; j < K; ++j) w_s[((size_t)f * kRegBC + s) * K + j] = w[j];
      if (has_base) sl_s[f * kRegBC + s] = silu_d((double)xv);
      c_s[f * kRegBC + s] = cell;
    }
    __syncthreads();
    // (3) sweep in sample order: the cell is warp-uniform, the switch is a jump table into
    //     code that updates the statically indexed registers acc[c .. c+K-1]
    if (i < d_in) {
      const double* wp = w_s + (size_t)fl * kRegBC * K;
      const int* cp = c_s + fl * kRegBC;
      const double* gp = g64 + ol;
#pragma unroll 2
      for (int s = 0; s < nb; ++s) {
        const int c = cp[s];
        double w[K], g[OV];
#pragma unroll
        for (int j = 0; j < K; ++j) w[j] = wp[s * K + j];
#pragma unroll
        for (int v = 0; v < OV; ++v) g[v] = gp[(size_t)s * OPB + v];
        switch (c) {
          UKAN_BWD_CASE(0)
          UKAN_BWD_CASE(1)
          UKAN_BWD_CASE(2)
          UKAN_BWD_CASE(3)
          UKAN_BWD_CASE(4)
          UKAN_BWD_CASE(5)
          UKAN_BWD_CASE(6)
          UKAN_BWD_CASE(7)
          UKAN_BWD_CASE(8)
          UKAN_BWD_CASE(9)
          UKAN_BWD_CASE(10)
          UKAN_BWD_CASE(11)
          UKAN_BWD_CASE(12)
          UKAN_BWD_CASE(13)
          UKAN_BWD_CASE(14)
          UKAN_BWD_CASE(15)
          UKAN_BWD_CASE(16)
          UKAN_BWD_CASE(17)
          UKAN_BWD_CASE(18)
          UKAN_BWD_CASE(19)
          UKAN_BWD_CASE(20)
          UKAN_BWD_CASE(21)
          UKAN_BWD_CASE(22)
          UKAN_BWD_CASE(23)
          UKAN_BWD_CASE(24)
          UKAN_BWD_CASE(25)
          UKAN_BWD_CASE(26)
          UKAN_BWD_CASE(27)
          UKAN_BWD_CASE(28)
          UKAN_BWD_CASE(29)
          UKAN_BWD_CASE(30)
          UKAN_BWD_CASE(31)
          UKAN_BWD_CASE(32)
          UKAN_BWD_CASE(33)
          UKAN_BWD_CASE(34)
          UKAN_BWD_CASE(35)
          UKAN_BWD_CASE(36)
          UKAN_BWD_CASE(37)
          UKAN_BWD_CASE(38)
          UKAN_BWD_CASE(39)
          UKAN_BWD_CASE(40)
          UKAN_BWD_CASE(41)
          UKAN_BWD_CASE(42)
          UKAN_BWD_CASE(43)
          UKAN_BWD_CASE(44)
          UKAN_BWD_CASE(45)
          UKAN_BWD_CASE(46)
          UKAN_BWD_CASE(47)
          UKAN_BWD_CASE(48)
          UKAN_BWD_CASE(49)
          UKAN_BWD_CASE(50)
          UKAN_BWD_CASE(51)
          UKAN_BWD_CASE(52)
          UKAN_BWD_CASE(53)
          UKAN_BWD_CASE(54)
          UKAN_BWD_CASE(55)
          UKAN_BWD_CASE(56)
          UKAN_BWD_CASE(57)
          UKAN_BWD_CASE(58)
          UKAN_BWD_CASE(59)
          UKAN_BWD_CASE(60)
          UKAN_BWD_CASE(61)
          UKAN_BWD_CASE(62)
          UKAN_BWD_CASE(63)
          UKAN_BWD_CASE(64)
          UKAN_BWD_CASE(65)
          UKAN_BWD_CASE(66)
          UKAN_BWD_CASE(67)
          UKAN_BWD_CASE(68)
          UKAN_BWD_CASE(69)
          UKAN_BWD_CASE(70)
          UKAN_BWD_CASE(71)
          default:
            break;
        }
      }
      if (has_base) {
        for (int s = 0; s < nb; ++s) {
          const double sl = sl_s[fl * kRegBC + s];
#pragma unroll
          for (int v = 0; v < OV; ++v) bacc[v] = fma(sl, gp[(size_t)s * OPB + v], bacc[v]);
        }
      }
    }
    __syncthreads();  // buffers of chunk n free for chunk n+2 / next meta
  }
  if (i >= d_in) return;
#pragma unroll
  for (int v = 0; v < OV; ++v) {
    const int o = o0 + ol + v;
    if (o >= d_out) continue;
    if (part != nullptr) {
      double* pp = part + ((size_t)z * d_in + i) * R * d_out + o;
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < R) pp[(size_t)r * d_out] = acc[r][v];
      if (has_base) part_b[((size_t)z * d_in + i) * d_out + o] = bacc[v];
    } else {
      const double sc = (double)scale[(size_t)i * d_out + o];
      double ds = 0.0;
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
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
// FP64 tensor-core variant (cubic splines, K = 4): banded blocks on DMMA.
//
// The table gradient of one feature is a banded product A[r,o] = sum_b W[b,r] g[b,o] with
// W[b, c_b .. c_b+3] = w(u_b).  Rows are covered by 8-row blocks with stride 4 (block bb =
// rows 4bb .. 4bb+7), so every cell's 4-row window lies inside block c>>2.  Samples of a
// 128-sample chunk are counting-sorted by cell per feature; consecutive groups of 4 sorted
// samples form the K=4 operand of one `mma.sync.m8n8k4.f64` per 8-output tile
// (D[8 rows x 8 outputs] += A[8 rows x 4 samples] B[4 samples x 8 outputs]), normally all four
// in the same block.  Accumulators of block bb / tile nt live in registers (statically
// indexed through a uniform unrolled block loop); each row is the sum of the two blocks that
// contain it, reduced in fixed order at the end (deterministic).  IEEE fp64 products and sums.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int RB, int NT>
__global__ void __launch_bounds__(256, 1)
kan_bwd_dmma_kernel(const float* __restrict__ x, const float* __restrict__ C,
                    const float* __restrict__ scale, const float* __restrict__ gy,
                    float* __restrict__ dC, float* __restrict__ dscale, double* __restrict__ part,
                    int B, int d_in, int d_out, int R, int sps, KanGrid grid, Basis<4> bas, int dbg) {
  constexpr int K = 4;
  constexpr int FPB = 8;
  constexpr int OPB = 8 * NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * FPB;
  const int i = i0 + warp;
  const int o0 = blockIdx.y * OPB;
  const int z = blockIdx.z;
  const int b_lo = z * sps, b_hi = min(B, b_lo + sps);
  const int grp = lane >> 2, kq = lane & 3;

  double* g64 = reinterpret_cast<double*>(smem_raw);             // [BC][OPB]
  double* acol = g64 + (size_t)kRegBC * OPB;                      // [FPB][BC][8] A columns (sorted)
  float* g_s0 = reinterpret_cast<float*>(acol + (size_t)FPB * kRegBC * 8);  // 2 x [BC][OPB]
  float* x_s0 = g_s0 + (size_t)2 * kRegBC * OPB;                  // 2 x [BC][FPB]
  int* csort = reinterpret_cast<int*>(x_s0 + 2 * kRegBC * FPB);   // [FPB][BC]
  int* ent = csort + FPB * kRegBC;                                // [FPB][BC]
  int* hist = ent + FPB * kRegBC;                                 // [FPB][2][4*RB + 8]

  double acc[RB][NT][2];
#pragma unroll
  for (int bb = 0; bb < RB; ++bb)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[bb][t][0] = acc[bb][t][1] = 0.0;

  const int nchunks = (b_hi - b_lo + kRegBC - 1) / kRegBC;
  if (nchunks > 0) stage_chunk(g_s0, x_s0, gy, x, b_lo, min(kRegBC, b_hi - b_lo), o0, OPB, d_out, i0, FPB, d_in);
  cp_async_commit();
  for (int n = 0; n < nchunks; ++n) {
    const int b0 = b_lo + n * kRegBC;
    const int nb = min(kRegBC, b_hi - b0);
    const float* g_s = g_s0 + (size_t)(n & 1) * kRegBC * OPB;
    const float* x_s = x_s0 + (size_t)(n & 1) * kRegBC * FPB;
    if (n + 1 < nchunks) {
      const int b1 = b0 + kRegBC;
      stage_chunk(g_s0 + (size_t)((n + 1) & 1) * kRegBC * OPB, x_s0 + (size_t)((n + 1) & 1) * kRegBC * FPB, gy,
                  x, b1, min(kRegBC, b_hi - b1), o0, OPB, d_out, i0, FPB, d_in);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    for (int t = threadIdx.x; t < kRegBC * OPB; t += blockDim.x) g64[t] = (double)g_s[t];
    // per feature (its warp): fp64 locate + basis of the chunk, stable counting sort by cell
    constexpr int NB = 4 * RB + 8;  // histogram bins (cells 0 .. 4RB-1, +1 shift, padding)
    int* st = hist + warp * 2 * NB;  // [NB] run starts, then [NB] scatter cursors
    if (i < d_in && !(dbg & 2)) {
      constexpr int PER = kRegBC / 32;
      int* cur = st + NB;
      for (int c = lane; c < NB; c += 32) cur[c] = 0;
      __syncwarp();
      int cells[PER];
      double w[PER][K];
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int s = q * 32 + lane;
        int cell = -1;
        double u = 0.0;
        bool mask;
        if (s < nb) kan_locate(x_s[s * FPB + warp], grid, cell, u, mask);
        basis_weights<K>(bas, u, w[q]);
        cells[q] = cell;
        const unsigned m = __match_any_sync(0xffffffffu, cell);
        if (cell >= 0 && lane == __ffs(m) - 1) cur[cell + 1] += __popc(m);
        __syncwarp();
      }
      // warp-parallel inclusive scan of the shifted histogram -> start of each cell
      int carry = 0;
      for (int c0 = 0; c0 < NB; c0 += 32) {
        const int c = c0 + lane;
        int v = c < NB ? cur[c] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, v, off);
          if (lane >= off) v += t;
        }
        v += carry;
        if (c < NB) {
          st[c] = v;
          cur[c] = v;
        }
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int cell = cells[q];
        const unsigned m = __match_any_sync(0xffffffffu, cell);
        int base = 0;
        if (cell >= 0) base = cur[cell];
        __syncwarp();
        if (cell >= 0) {
          const int pos = base + __popc(m & ((1u << lane) - 1u));
          ent[warp * kRegBC + pos] = (q * 32 + lane) * OPB;  // g64 row offset of the sample
          csort[warp * kRegBC + pos] = cell;
          // the sample's column of the 8-row block (cell >> 2): weights at rows (cell & 3) + j
          double* ac = acol + ((size_t)warp * kRegBC + pos) * 8;
          const int sh = cell & 3;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int j = r - sh;
            ac[r] = (j == 0) ? w[q][0] : (j == 1) ? w[q][1] : (j == 2) ? w[q][2] : (j == 3) ? w[q][3] : 0.0;
          }
          if (lane == __ffs(m) - 1) cur[cell] = base + __popc(m);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // sweep: block bb (rows 4bb..4bb+7) takes the sorted samples of cells 4bb..4bb+3, four at a
    // time, one DMMA per 8-output tile into the statically indexed accumulators acc[bb][t];
    // the operands of the next group are loaded before the current group's DMMAs issue
    if (i < d_in && !(dbg & 1)) {
      const int* es = ent + warp * kRegBC;
      const double* ac = acol + (size_t)warp * kRegBC * 8 + grp;
      const double* gl = g64 + grp;
#pragma unroll
      for (int bb = 0; bb < RB; ++bb) {
        const int e0 = st[4 * bb], e1 = st[4 * bb + 4];
        if (e0 >= e1) continue;
        int pos = e0 + kq;
        bool vld = pos < e1;
        double a_n = vld ? ac[pos * 8] : 0.0;
        int so = es[pos];
        double b_n[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) b_n[t] = vld ? gl[so + t * 8] : 0.0;
        for (int kc = e0; kc < e1; kc += 4) {
          const double a = a_n;
          double bf[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) bf[t] = b_n[t];
          pos += 4;
          vld = pos < e1;
          a_n = vld ? ac[min(pos, kRegBC - 1) * 8] : 0.0;
          so = es[min(pos, kRegBC - 1)];
#pragma unroll
          for (int t = 0; t < NT; ++t) b_n[t] = vld ? gl[so + t * 8] : 0.0;
#pragma unroll
          for (int t = 0; t < NT; ++t) dmma_884(acc[bb][t][0], acc[bb][t][1], a, bf[t]);
        }
      }
    }
    __syncthreads();
  }
  if (i >= d_in) return;
  // rows 4bb..4bb+3 = lower half of block bb (lanes 0..15) + upper half of block bb-1
  // (lanes 16..31 of block bb-1, moved down by 16 lanes); fixed order -> deterministic
  double ds[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) ds[t][0] = ds[t][1] = 0.0;
#pragma unroll
  for (int bb = 0; bb <= RB; ++bb) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const double lower = bb < RB ? acc[bb][t][v] : 0.0;
        const double upper = bb > 0 ? __shfl_down_sync(0xffffffffu, acc[bb - 1][t][v], 16) : 0.0;
        const double a = lower + upper;
        const int r = 4 * bb + grp;
        const int o = o0 + t * 8 + 2 * kq + v;
        if (lane < 16 && r < R && o < d_out) {
          const size_t ci = ((size_t)i * R + r) * d_out + o;
          if (part != nullptr) {
            part[(size_t)z * d_in * R * d_out + ci] = a;
          } else {
            dC[ci] = (float)((double)scale[(size_t)i * d_out + o] * a);
            ds[t][v] = fma((double)C[ci], a, ds[t][v]);
          }
        }
      }
    }
  }
  if (part == nullptr) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        double d = ds[t][v];
        d += __shfl_xor_sync(0xffffffffu, d, 4);
        d += __shfl_xor_sync(0xffffffffu, d, 8);
        const int o = o0 + t * 8 + 2 * kq + v;
        if (lane < 4 && o < d_out) dscale[(size_t)i * d_out + o] = (float)d;
      }
  }
}

// Fixed-order reduction of the split-batch partials + epilogue.  Thread per (i, o).
__global__ void kan_bwd_reduce_kernel(const double* __restrict__ part, const double* __restrict__ part_b,
                                      const float* __restrict__ C, const float* __restrict__ scale,
                                      float* __restrict__ dC, float* __restrict__ dscale,
                                      float* __restrict__ dbw, int S, int d_in, int d_out, int R) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)d_in * d_out) return;
  const int i = (int)(t / d_out), o = (int)(t % d_out);
  const double sc = (double)scale[t];
  const size_t zstride = (size_t)d_in * R * d_out;
  double ds = 0.0;
  for (int r = 0; r < R; ++r) {
    const size_t ci = ((size_t)i * R + r) * d_out + o;
    double a = 0.0;
    for (int zz = 0; zz < S; ++zz) a += part[zz * zstride + ci];
    dC[ci] = (float)(sc * a);
    ds = fma((double)C[ci], a, ds);
  }
  dscale[t] = (float)ds;
  if (dbw) {
    double b = 0.0;
    for (int zz = 0; zz < S; ++zz) b += part_b[(size_t)zz * d_in * d_out + t];
    dbw[t] = (float)b;
  }
}

// ---------------------------------------------------------------------------------------
// dx for narrow layers (d_out <= 32): one thread per (b, i), sequential fp64 dot over o.
//   dx[b,i] = mask * inv_dg * sum_j w'_j * sum_o g[b,o]*scale[i,o]*C[i,cell+j,o]
//             (+ dsilu(x) * sum_o g[b,o]*bw[i,o])
// ---------------------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(256)
kan_dx_narrow_kernel(const float* __restrict__ x, const float* __restrict__ C,
                     const float* __restrict__ scale, const float* __restrict__ bw,
                     const float* __restrict__ gy, float* __restrict__ dx, int B, int d_in,
                     int d_out, int R, KanGrid grid, Basis<K> bas) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * d_in) return;
  const int b = (int)(t / d_in), i = (int)(t % d_in);
  const float xv = x[t];
  int cell;
  double u;
  bool mask;
  kan_locate(xv, grid, cell, u, mask);
  double wp[K];
  basis_dweights<K>(bas, u, wp);
  const float* Ci = C + ((size_t)i * R + cell) * d_out;
  const float* gr = gy + (size_t)b * d_out;
  const float* sr = scale + (size_t)i * d_out;
  double S[K];
#pragma unroll
  for (int j = 0; j < K; ++j) S[j] = 0.0;
  double sb = 0.0;
  for (int o = 0; o < d_out; ++o) {
    const double g = (double)__ldg(gr + o);
    const double gs = g * (double)__ldg(sr + o);
#pragma unroll
    for (int j = 0; j < K; ++j) S[j] = fma(gs, (double)__ldg(Ci + (size_t)j * d_out + o), S[j]);
    if (bw) sb = fma(g, (double)__ldg(bw + (size_t)i * d_out + o), sb);
  }
  double tt = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) tt = fma(S[j], wp[j], tt);
  double d = mask ? tt * grid.inv_dg : 0.0;
  if (bw) d += dsilu_d((double)xv) * sb;
  dx[t] = (float)d;
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
struct RegPlan {
  bool ok = false;
  int rmax = 0, ov = 1, fpb = 1, wpf = 1, S = 1, sps = 0;
  size_t smem = 0;
  int64_t ws_bytes = 0;
};

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
  }
  return n;
}

RegPlan kan_bwd_reg_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base, int sms) {
  RegPlan p;
  if (K > 6) return p;
  if (R <= 16) p.rmax = 16;
  else if (R <= 40) p.rmax = 40;
  else if (R <= 72) p.rmax = 72;
  else return p;
  p.ov = (p.rmax <= 16 && d_out >= 64) ? 2 : 1;  // acc[RMAX][OV] doubles stay <= ~80 registers
  p.wpf = 1;  // one warp per feature: g[chunk, o-tile] in smem is reused by all 8 features
  p.fpb = 8;
  const int opb = p.wpf * 32 * p.ov;
  p.smem = sizeof(double) * ((size_t)p.fpb * kRegBC * (K + (has_base ? 1 : 0)) + (size_t)kRegBC * opb) +
           sizeof(float) * (size_t)2 * kRegBC * (opb + p.fpb) + sizeof(int) * (size_t)p.fpb * kRegBC;
  const int64_t base = ((d_in + p.fpb - 1) / p.fpb) * ((d_out + opb - 1) / opb);
  // Split the batch only when the grid is short of two waves (one CTA per SM); pick the
  // split with the best wave efficiency.  Depends on shapes only -> deterministic.
  int64_t S = 1;
  if (base < 2 * (int64_t)sms) {
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(16, B / (4 * kRegBC)));
    double best = -1.0;
    for (int64_t c = 1; c <= max_s; ++c) {
      const double waves = (double)(base * c) / sms;
      const double eff = waves / std::ceil(waves) * std::min(1.0, waves / 2.0);
      if (eff > best + 1e-9) { best = eff; S = c; }
    }
  }
  p.S = (int)S;
  p.sps = (int)(((B + S - 1) / S + kRegBC - 1) / kRegBC * kRegBC);
  if (p.sps == 0) p.sps = kRegBC;
  p.S = (int)std::max<int64_t>(1, (B + p.sps - 1) / p.sps);
  if (p.S > 1) p.ws_bytes = (int64_t)sizeof(double) * p.S * d_in * (int64_t)d_out * (R + (has_base ? 1 : 0));
  p.ok = true;
  return p;
}

template <int K, int RMAX, int OV>
static int launch_reg(const float* x, const float* C, const float* scale, const float* gy, float* dC,
                      float* dscale, float* dbw, double* ws, int B, int d_in, int d_out, int R,
                      const KanGrid& grid, const RegPlan& p, cudaStream_t st) {
  const Basis<K> bas = make_basis<K>(K - 1);
  auto kern = kan_bwd_reg_kernel<K, RMAX, OV>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const int opb = p.wpf * 32 * OV;
  dim3 gridd((d_in + p.fpb - 1) / p.fpb, (d_out + opb - 1) / opb, p.S);
  double* part = p.S > 1 ? ws : nullptr;
  double* part_b = (p.S > 1 && dbw) ? ws + (size_t)p.S * d_in * R * d_out : nullptr;
  kern<<<gridd, 32 * p.fpb * p.wpf, p.smem, st>>>(x, C, scale, gy, dC, dscale, dbw, part, part_b, B, d_in,
                                                   d_out, R, p.fpb, p.wpf, p.sps, dbw != nullptr, grid, bas);
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    const int64_t n = (int64_t)d_in * d_out;
    kan_bwd_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, part_b, C, scale, dC, dscale, dbw,
                                                                       p.S, d_in, d_out, R);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

template <int K>
int kan_bwd_reg_dispatch(const float* x, const float* C, const float* scale, const float* gy, float* dC,
                         float* dscale, float* dbw, double* ws, int B, int d_in, int d_out, int R,
                         const KanGrid& grid, const RegPlan& p, cudaStream_t st) {
  if constexpr (K <= 6) {
    if (p.rmax == 16 && p.ov == 2) return launch_reg<K, 16, 2>(x, C, scale, gy, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
    if (p.rmax == 16) return launch_reg<K, 16, 1>(x, C, scale, gy, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
    if (p.rmax == 40 && p.ov == 2) return launch_reg<K, 40, 2>(x, C, scale, gy, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
    if (p.rmax == 40) return launch_reg<K, 40, 1>(x, C, scale, gy, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
    if (p.rmax == 72) return launch_reg<K, 72, 1>(x, C, scale, gy, dC, dscale, dbw, ws, B, d_in, d_out, R, grid, p, st);
  }
  return UKAN_E_ARG;
}

template <int K>
int kan_dx_narrow(const float* x, const float* C, const float* scale, const float* bw, const float* gy, float* dx,
                  int B, int d_in, int d_out, int R, const KanGrid& grid, cudaStream_t st) {
  const Basis<K> bas = make_basis<K>(K - 1);
  const int64_t n = (int64_t)B * d_in;
  if (n == 0) return UKAN_OK;
  kan_dx_narrow_kernel<K><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, C, scale, bw, gy, dx, B, d_in, d_out, R,
                                                                      grid, bas);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

int kan_num_sms() { return num_sms(); }

// DMMA path: cubic splines without the base branch, G <= 64.
bool kan_bwd_dmma_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K, bool has_base, int sms, RegPlan& p) {
  if (K != 4 || has_base) return false;
  const int G = R - K + 1;
  const int rbn = ((G - 1) >> 2) + 1;
  int rb = 0;
  if (rbn <= 4) rb = 4;
  else if (rbn <= 8) rb = 8;
  else if (rbn <= 16) rb = 16;
  else return false;
  const int nt = rb == 16 ? 2 : (d_out <= 8 ? 1 : (d_out <= 16 ? 2 : 4));
  p.rmax = rb;
  p.ov = nt;
  p.fpb = 8;
  p.wpf = 1;
  const int opb = 8 * nt;
  p.smem = sizeof(double) * ((size_t)kRegBC * opb + (size_t)8 * kRegBC * 8) + sizeof(float) * (size_t)2 * kRegBC * (opb + 8) +
           sizeof(int) * ((size_t)2 * 8 * kRegBC + (size_t)8 * 2 * (4 * rb + 8));
  const int64_t base = ((d_in + 7) / 8) * ((d_out + opb - 1) / opb);
  int64_t S = 1;
  if (base < 2 * (int64_t)sms) {
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(16, B / (4 * kRegBC)));
    double best = -1.0;
    for (int64_t c = 1; c <= max_s; ++c) {
      const double waves = (double)(base * c) / sms;
      const double eff = waves / std::ceil(waves) * std::min(1.0, waves / 2.0);
      if (eff > best + 1e-9) { best = eff; S = c; }
    }
  }
  p.sps = (int)(((B + S - 1) / S + kRegBC - 1) / kRegBC * kRegBC);
  if (p.sps == 0) p.sps = kRegBC;
  p.S = (int)std::max<int64_t>(1, (B + p.sps - 1) / p.sps);
  p.ws_bytes = p.S > 1 ? (int64_t)sizeof(double) * p.S * d_in * (int64_t)d_out * R : 0;
  p.ok = true;
  return true;
}

template <int RB, int NT>
static int launch_dmma(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                       double* ws, int B, int d_in, int d_out, int R, const KanGrid& grid, const RegPlan& p,
                       cudaStream_t st) {
  const Basis<4> bas = make_basis<4>(3);
  auto kern = kan_bwd_dmma_kernel<RB, NT>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 gridd((d_in + 7) / 8, (d_out + 8 * NT - 1) / (8 * NT), p.S);
  double* part = p.S > 1 ? ws : nullptr;
  static const int dbg = getenv("UKAN_DBG") ? atoi(getenv("UKAN_DBG")) : 0;  // profiling knobs only
  kern<<<gridd, 256, p.smem, st>>>(x, C, scale, gy, dC, dscale, part, B, d_in, d_out, R, p.sps, grid, bas, dbg);
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    const int64_t n = (int64_t)d_in * d_out;
    kan_bwd_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nullptr, C, scale, dC, dscale, nullptr,
                                                                       p.S, d_in, d_out, R);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

int kan_bwd_dmma_dispatch(const float* x, const float* C, const float* scale, const float* gy, float* dC,
                          float* dscale, double* ws, int B, int d_in, int d_out, int R, const KanGrid& grid,
                          const RegPlan& p, cudaStream_t st) {
  if (p.rmax == 4 && p.ov == 1) return launch_dmma<4, 1>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 4 && p.ov == 2) return launch_dmma<4, 2>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 4) return launch_dmma<4, 4>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 8 && p.ov == 1) return launch_dmma<8, 1>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 8 && p.ov == 2) return launch_dmma<8, 2>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 8) return launch_dmma<8, 4>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  if (p.rmax == 16) return launch_dmma<16, 2>(x, C, scale, gy, dC, dscale, ws, B, d_in, d_out, R, grid, p, st);
  return UKAN_E_ARG;
}

#define UKAN_INST(K)                                                                                            \
  template int kan_bwd_reg_dispatch<K>(const float*, const float*, const float*, const float*, float*, float*,   \
                                       float*, double*, int, int, int, int, const KanGrid&, const RegPlan&,     \
                                       cudaStream_t);                                                           \
  template int kan_dx_narrow<K>(const float*, const float*, const float*, const float*, const float*, float*,    \
                                int, int, int, int, const KanGrid&, cudaStream_t);
UKAN_INST(1) UKAN_INST(2) UKAN_INST(3) UKAN_INST(4) UKAN_INST(5) UKAN_INST(6) UKAN_INST(7) UKAN_INST(8)
UKAN_INST(9) UKAN_INST(10) UKAN_INST(11)

}  // namespace ukan
