// kan_bwd_tc.cu — KAN backward (table side) for cubic splines on the FP64 tensor cores.
//
// Replaces the bwd closures of span_gather (layers.py:67-70, the np.add.at scatter of the window
// gradient) and edge_combine (84-88) for k = 3 without the base branch:
//   A[i,r,o] = sum_{(b,j): cell_bi + j = r} w_j(u_bi) * g[b,o]     (fp64)
//   dC = scale * A,   dscale = sum_r C * A.
//
// Two kernels.
//  * prep: once per (feature, 256-sample chunk) — fp64 locate with the reference's expression
//    order (layers.py:299-300), stable counting sort of the chunk by cell, record
//    {(cell<<8)|sample|clamped<<30, u} in cell order plus the start of every cell.  The records of a layer
//    (~14 B per (sample, feature)) stay L2-resident and are shared by every output tile.
//  * sweep: a CTA owns 8 features x 8*NT outputs; per chunk it stages (cp.async, double
//    buffered) the 8 feature records and g[chunk, o-tile].  Rows are covered by 8-row blocks
//    with stride 4 (block bb = rows 4bb..4bb+7), so a cell's 4-row window lies in block cell>>2.
//    Four consecutive sorted samples of cells 4bb..4bb+3 form the k=4 operand of one
//    `mma.sync.m8n8k4.f64` (DMMA) per 8-output tile:
//        D[8 rows x 8 out] += A[8 rows x 4 samples] * B[4 samples x 8 out],
//    A[r][k] = w_{r - (cell_k & 3)}(u_k) (evaluated in-lane from u, fp64 Horner),
//    B[k][n] = g[sample_k][o_n].  Accumulators acc[bb][t] are statically indexed registers;
//    each row is the sum of the two blocks holding it, reduced in fixed order at the end.
// Deterministic: fixed sample order per chunk, fixed chunk order, fixed reductions.  IEEE fp64
// products and sums throughout.
#include <cuda.h>  // CUtensorMap (the 2-D TMA descriptor of the tc3 sweep)
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace ukan {

constexpr int kTcBC = 256;  // samples per chunk (the sample index is packed in 8 bits)
constexpr int kTcClamped = 1 << 30;  // record flag: x outside [g_min, hi] (clamp mask 0, tensor.py:330)

// prep record layout (bytes, 16-aligned): ent[128] int | u[128] double | st[NBP] int
__host__ __device__ constexpr int tc_nbp(int G) { return ((G + 1 + 3) / 4) * 4; }
__host__ __device__ constexpr size_t tc_rec_bytes(int G) {
  return (size_t)kTcBC * 4 + (size_t)kTcBC * 8 + (size_t)tc_nbp(G) * 4;
}

// Lanes holding the same cell (cell in [-1, 126]): a 7-bit radix multisplit from ballots, which
// measured cheaper than __match_any_sync in this kernel.
__device__ __forceinline__ unsigned tc_same_cell_mask(int cell) {
  const unsigned key = (unsigned)(cell + 1);
  unsigned eq = 0xffffffffu;
#pragma unroll
  for (int bit = 0; bit < 7; ++bit) {
    const unsigned b = __ballot_sync(0xffffffffu, (key >> bit) & 1u);
    eq &= ((key >> bit) & 1u) ? b : ~b;
  }
  return eq;
}

// UK: a dense UKAN layer (every feature's virtual table has <= G + 3 rows): the cell is the
// sample's window start inside its feature's row segment, base_row[b, i] - 4 * seg[i]
// (layers.py:261-287), u = x/dg - floor(x/dg) (layers.py:263), never clamped.
template <bool UK>
__global__ void __launch_bounds__(256)
kan_bwd_tc_prep_kernel(const float* __restrict__ x, unsigned char* __restrict__ recs, int B, int d_in,
                       int nch, int G, KanGrid grid, const int32_t* __restrict__ base_row,
                       const int32_t* __restrict__ seg, double inv_dg) {
  __shared__ float xs[kTcBC][9];
  __shared__ int cnt[8][80];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * 8;
  const int n = blockIdx.y;
  const int b0 = n * kTcBC;
  const int nb = min(kTcBC, B - b0);
  for (int t = threadIdx.x; t < kTcBC * 8; t += blockDim.x) {
    const int s = t / 8, f = t % 8;
    xs[s][f] = (s < nb && i0 + f < d_in) ? x[(size_t)(b0 + s) * d_in + i0 + f] : 0.f;
  }
  __syncthreads();
  const int i = i0 + warp;
  if (i >= d_in) return;
  const size_t rb = tc_rec_bytes(G);
  unsigned char* rec = recs + ((size_t)i * nch + n) * rb;
  int* ent = reinterpret_cast<int*>(rec);
  double* uu = reinterpret_cast<double*>(rec + kTcBC * 4);
  int* st = reinterpret_cast<int*>(rec + kTcBC * 12);
  const int NB = G + 1;
  // shared cursor space: G+1 <= 80 handled here (G <= 64 on this path)
  int* cur = cnt[warp];
  for (int c = lane; c < NB + 1; c += 32) cur[c] = 0;
  __syncwarp();
  constexpr int PER = kTcBC / 32;
  int cells[PER];
  double us[PER];
  unsigned clamped = 0;  // bit q: sample q*32+lane lies outside [g_min, hi] (dx mask = 0)
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int s = q * 32 + lane;
    int cell = -1;
    double u = 0.0;
    bool mask = true;
    if constexpr (UK) {
      if (s < nb) {
        int64_t gid;
        ukan_locate(xs[s][warp], inv_dg, gid, u);
        cell = base_row[(size_t)(b0 + s) * d_in + i] - 4 * seg[i];
        if (cell < 0 || cell > G - 1 || !(u == u)) cell = -1;  // outside the plan (never for valid keys)
      }
    } else {
      if (s < nb) kan_locate(xs[s][warp], grid, cell, u, mask);
    }
    if (!mask) clamped |= 1u << q;
    cells[q] = cell;
    us[q] = u;
    const unsigned m = tc_same_cell_mask(cell);
    if (cell >= 0 && lane == __ffs(m) - 1) cur[cell + 1] += __popc(m);
    __syncwarp();
  }
  // inclusive scan of the shifted histogram -> start of each cell (cur[c]); st[] copy
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
      cur[c] = v;
      st[c] = v;
    }
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
  for (int c = NB + lane; c < tc_nbp(G); c += 32) st[c] = nb;
  __syncwarp();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int cell = cells[q];
    const unsigned m = tc_same_cell_mask(cell);
    int base = 0;
    if (cell >= 0) base = cur[cell];
    __syncwarp();
    if (cell >= 0) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      ent[pos] = (cell << 8) | (q * 32 + lane) | (((clamped >> q) & 1u) ? kTcClamped : 0);
      uu[pos] = us[q];
      if (lane == __ffs(m) - 1) cur[cell] = base + __popc(m);
    }
    __syncwarp();
  }
  // tail positions (partial last chunk): harmless padding
  for (int p = nb + lane; p < kTcBC; p += 32) {
    ent[p] = 0;
    uu[p] = 0.0;
  }
}

__device__ __forceinline__ void tc_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void tc_cp16(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void tc_cp4(void* smem, const void* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(ok ? 4 : 0));
}

template <int RB, int NT>
__global__ void __launch_bounds__(256, (RB <= 8 && NT <= 2) ? 2 : 1)  // narrow outputs: latency-bound, 2 blocks/SM (layer-1 backward 0.207 -> 0.167 ms)
kan_bwd_tc_sweep_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ C,
                        const float* __restrict__ scale, const float* __restrict__ gy,
                        float* __restrict__ dC, float* __restrict__ dscale, double* __restrict__ part,
                        int B, int d_in, int d_out, int G, int nch, int cps, Basis<4> bas) {
  constexpr int OPB = 8 * NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  const int i0 = blockIdx.x * 8;
  const int i = i0 + warp;
  const int o0 = blockIdx.y * OPB;
  const int z = blockIdx.z;
  const int n_lo = z * cps, n_hi = min(nch, n_lo + cps);
  const int R = G + 3;
  const size_t rb = tc_rec_bytes(G);
  __shared__ double Msh[16];  // basis matrix (dynamic column index -> shared, not local memory)
  if (threadIdx.x == 0) {  // constant indices: no local-memory copy of the parameter struct
#pragma unroll
    for (int q = 0; q < 16; ++q) Msh[q] = bas.M[q / 4][q % 4];
  }
  unsigned char* rec_s = smem_raw;                                            // 2 x [8][rb]
  float* g_s = reinterpret_cast<float*>(smem_raw + 2 * 8 * rb);               // 2 x [BC][OPB]

  auto stage = [&](int n, int buf) {
    // feature records (contiguous, 16-byte granules)
    unsigned char* dst = rec_s + (size_t)buf * 8 * rb;
    const int q = (int)(rb / 16);
    for (int t = threadIdx.x; t < 8 * q; t += blockDim.x) {
      const int f = t / q, c = t % q;
      const bool ok = i0 + f < d_in;
      const unsigned char* src = ok ? recs + ((size_t)(i0 + f) * nch + n) * rb + (size_t)c * 16 : recs;
      tc_cp16(dst + (size_t)f * rb + (size_t)c * 16, src, ok ? 16 : 0);
    }
    // g[chunk, o-tile]
    float* gd = g_s + (size_t)buf * kTcBC * OPB;
    const int b0 = n * kTcBC;
    const int nb = min(kTcBC, B - b0);
    if ((d_out & 3) == 0) {
      constexpr int q4 = OPB / 4;
      for (int t = threadIdx.x; t < kTcBC * q4; t += blockDim.x) {
        const int s = t / q4, oc = (t % q4) * 4;
        const int o = o0 + oc;
        const int bytes = (s < nb) ? max(0, min(4, d_out - o)) * 4 : 0;
        tc_cp16(gd + s * OPB + oc, bytes ? gy + (size_t)(b0 + s) * d_out + o : gy, bytes);
      }
    } else {
      for (int t = threadIdx.x; t < kTcBC * OPB; t += blockDim.x) {
        const int s = t / OPB, oc = t % OPB;
        const bool ok = s < nb && o0 + oc < d_out;
        tc_cp4(gd + t, ok ? gy + (size_t)(b0 + s) * d_out + o0 + oc : gy, ok);
      }
    }
  };

  double acc[RB][NT][2];
#pragma unroll
  for (int bb = 0; bb < RB; ++bb)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[bb][t][0] = acc[bb][t][1] = 0.0;

  if (n_lo < n_hi) stage(n_lo, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int n = n_lo; n < n_hi; ++n) {
    const int buf = (n - n_lo) & 1;
    if (n + 1 < n_hi) stage(n + 1, buf ^ 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    if (i < d_in) {
      const unsigned char* rec = rec_s + ((size_t)buf * 8 + warp) * rb;
      const int* ent = reinterpret_cast<const int*>(rec);
      const double* uu = reinterpret_cast<const double*>(rec + kTcBC * 4);
      const int* st = reinterpret_cast<const int*>(rec + kTcBC * 12);
      const float* gl = g_s + (size_t)buf * kTcBC * OPB + grp;
#pragma unroll
      for (int bb = 0; bb < RB; ++bb) {
        const int e0 = st[min(4 * bb, G)], e1 = st[min(4 * bb + 4, G)];
#pragma unroll 2
        for (int kc = e0; kc < e1; kc += 4) {
          const int pos = kc + kq;
          const bool vld = pos < e1;
          const int e = ent[min(pos, kTcBC - 1)];
          const double u = uu[min(pos, kTcBC - 1)];
          const int j = grp - ((e >> 8) & 3);
          double a = 0.0;
          if (vld && j >= 0 && j < 4) {  // w_j(u) = sum_m M[m][j] u^m  (Horner, fp64)
            a = fma(fma(fma(Msh[12 + j], u, Msh[8 + j]), u, Msh[4 + j]), u, Msh[j]);
          }
          const int srow = (e & 255) * OPB;
          double bf[NT];
#pragma unroll
          for (int t = 0; t < NT; ++t) bf[t] = vld ? (double)gl[srow + t * 8] : 0.0;
#pragma unroll
          for (int t = 0; t < NT; ++t) tc_dmma(acc[bb][t][0], acc[bb][t][1], a, bf[t]);
        }
      }
    }
    __syncthreads();
  }
  if (i >= d_in) return;
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

// WPF warps per feature ("tc2"): warp h of feature f owns blocks [h*RB/WPF, (h+1)*RB/WPF), so a
// warp holds a fraction of the block accumulators and can cover more outputs (NT DMMA tiles per
// group share one A operand).  The parts meet in a shared-memory fp64 row buffer in fixed order
// (block order, part 0 first) -> deterministic.
template <int RB, int NT, int FPB, int WPF>
__global__ void __launch_bounds__(FPB * WPF * 32, 1)
kan_bwd_tc2_sweep_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ C,
                         const float* __restrict__ scale, const float* __restrict__ gy,
                         float* __restrict__ dC, float* __restrict__ dscale, double* __restrict__ part,
                         int B, int d_in, int d_out, int G, int nch, int cps, Basis<4> bas) {
  constexpr int OPB = 8 * NT;
  constexpr int GST = OPB + 8;  // g row stride (floats): +32 B puts the 4 sample rows of a DMMA
                                // B operand on disjoint banks (one wavefront instead of four)
  constexpr int BH = RB / WPF;  // blocks per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  const int fl = warp / WPF, h = warp % WPF;
  // Grid walk in panels of kSwFG feature groups x all output tiles, feature group fastest inside a
  // panel: a wave of resident CTAs covers ~148/kSwFG output tiles x kSwFG feature groups, so it
  // shares both the g columns of its output tiles and the records of its feature groups through L2
  // (row-major order re-read all of g once per feature group: 244 GB per call at cfg3, B = 16384).
  constexpr int kSwFG = 16;
  int ot, fg;
  {
    const int n_ot = gridDim.x, n_fg = gridDim.y;
    const int L = blockIdx.y * n_ot + blockIdx.x;
    const int pw = min(kSwFG, n_fg);
    const int sc = L / (pw * n_ot), r = L % (pw * n_ot);
    const int pe = min(pw, n_fg - sc * pw);
    ot = r / pe;
    fg = sc * pw + r % pe;
  }
  const int i0 = fg * FPB;
  const int i = i0 + fl;
  const int o0 = ot * OPB;
  const int z = blockIdx.z;
  const int n_lo = z * cps, n_hi = min(nch, n_lo + cps);
  const int R = G + 3;
  const size_t rb = tc_rec_bytes(G);
  __shared__ double Msh[16];
  if (threadIdx.x == 0) {  // constant indices: no local-memory copy of the parameter struct
#pragma unroll
    for (int q = 0; q < 16; ++q) Msh[q] = bas.M[q / 4][q % 4];
  }
  unsigned char* rec_s = smem_raw;                                              // 2 x [FPB][rb]
  float* g_s = reinterpret_cast<float*>(smem_raw + 2 * FPB * rb);               // 2 x [BC][OPB]
  double* w_s = reinterpret_cast<double*>(g_s + (size_t)2 * kTcBC * GST);       // [FPB][BC][4] basis weights

  auto stage = [&](int n, int buf) {
    unsigned char* dst = rec_s + (size_t)buf * FPB * rb;
    const int q = (int)(rb / 16);
    for (int t = threadIdx.x; t < FPB * q; t += blockDim.x) {
      const int f = t / q, c = t % q;
      const bool ok = i0 + f < d_in;
      const unsigned char* src = ok ? recs + ((size_t)(i0 + f) * nch + n) * rb + (size_t)c * 16 : recs;
      tc_cp16(dst + (size_t)f * rb + (size_t)c * 16, src, ok ? 16 : 0);
    }
    float* gd = g_s + (size_t)buf * kTcBC * GST;
    const int b0 = n * kTcBC;
    const int nb = min(kTcBC, B - b0);
    if ((d_out & 3) == 0) {
      constexpr int q4 = OPB / 4;
      for (int t = threadIdx.x; t < kTcBC * q4; t += blockDim.x) {
        const int s = t / q4, oc = (t % q4) * 4;
        const int o = o0 + oc;
        const int bytes = (s < nb) ? max(0, min(4, d_out - o)) * 4 : 0;
        tc_cp16(gd + s * GST + oc, bytes ? gy + (size_t)(b0 + s) * d_out + o : gy, bytes);
      }
    } else {
      for (int t = threadIdx.x; t < kTcBC * OPB; t += blockDim.x) {
        const int s = t / OPB, oc = t % OPB;
        const bool ok = s < nb && o0 + oc < d_out;
        tc_cp4(gd + s * GST + oc, ok ? gy + (size_t)(b0 + s) * d_out + o0 + oc : gy, ok);
      }
    }
  };

  double acc[BH][NT][2];
#pragma unroll
  for (int bb = 0; bb < BH; ++bb)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[bb][t][0] = acc[bb][t][1] = 0.0;

  if (n_lo < n_hi) stage(n_lo, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  for (int n = n_lo; n < n_hi; ++n) {
    const int buf = (n - n_lo) & 1;
    if (n + 1 < n_hi) stage(n + 1, buf ^ 1);
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncthreads();
    // basis weights of the chunk's sorted samples, once per CTA (fp64 Horner, layers.py:29-37)
    for (int t = threadIdx.x; t < FPB * kTcBC; t += blockDim.x) {
      const int f = t / kTcBC, pos = t % kTcBC;
      const double u = reinterpret_cast<const double*>(rec_s + ((size_t)buf * FPB + f) * rb + kTcBC * 4)[pos];
      double* wd = w_s + (size_t)t * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) wd[j] = fma(fma(fma(Msh[12 + j], u, Msh[8 + j]), u, Msh[4 + j]), u, Msh[j]);
    }
    __syncthreads();
    if (i < d_in) {
      const unsigned char* rec = rec_s + ((size_t)buf * FPB + fl) * rb;
      const double* wf = w_s + (size_t)fl * kTcBC * 4;
      const int* ent = reinterpret_cast<const int*>(rec);
      const int* st = reinterpret_cast<const int*>(rec + kTcBC * 12);
      // B operand: lane (sample kq, column n = grp) of tile t is output o0 + n*NT + t, so a lane's NT
      // values are contiguous (LDS.128); the epilogue maps the columns back
      const float* gl = g_s + (size_t)buf * kTcBC * GST + grp * NT;
      // one group = 4 consecutive sorted samples (the k = 4 operand); invalid positions read a real
      // (zero-filled or other) sample row and are masked by a = 0
      auto load_group = [&](int kc, int e1, double& a, float4 (&gv)[NT / 4]) {
        const int pos = kc + kq;
        const int pc = min(pos, kTcBC - 1);
        const int e = ent[pc];
        const int j = grp - ((e >> 8) & 3);
        const double wj = wf[pc * 4 + (j & 3)];
        a = (pos < e1 && j >= 0 && j < 4) ? wj : 0.0;
        const float* gp = gl + (e & 255) * GST;
#pragma unroll
        for (int q = 0; q < NT / 4; ++q) gv[q] = *reinterpret_cast<const float4*>(gp + 4 * q);
      };
#pragma unroll
      for (int bl = 0; bl < BH; ++bl) {
        const int bb = h * BH + bl;
        const int e0 = st[min(4 * bb, G)], e1 = st[min(4 * bb + 4, G)];
        int kc = e0;
        for (; kc + 4 < e1; kc += 8) {  // two groups in flight
          double a0, a1;
          float4 g0[NT / 4], g1[NT / 4];
          load_group(kc, e1, a0, g0);
          load_group(kc + 4, e1, a1, g1);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v0 = t % 4 == 0 ? g0[t / 4].x : t % 4 == 1 ? g0[t / 4].y : t % 4 == 2 ? g0[t / 4].z : g0[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a0, (double)v0);
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v1 = t % 4 == 0 ? g1[t / 4].x : t % 4 == 1 ? g1[t / 4].y : t % 4 == 2 ? g1[t / 4].z : g1[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a1, (double)v1);
          }
        }
        if (kc < e1) {
          double a0;
          float4 g0[NT / 4];
          load_group(kc, e1, a0, g0);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v0 = t % 4 == 0 ? g0[t / 4].x : t % 4 == 1 ? g0[t / 4].y : t % 4 == 2 ? g0[t / 4].z : g0[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a0, (double)v0);
          }
        }
      }
    }
    __syncthreads();
  }
  // epilogue: rows of both halves meet in S[FPB][R][OPB] (fp64, reuses the staging space)
  double* S = reinterpret_cast<double*>(smem_raw);
  const int RR = 4 * RB + 4;
  for (int t = threadIdx.x; t < FPB * RR * OPB; t += blockDim.x) S[t] = 0.0;
  __syncthreads();
#pragma unroll
  for (int hh = 0; hh < WPF; ++hh) {
    if (h == hh) {
#pragma unroll
      for (int bl = 0; bl < BH; ++bl) {
        const int r = 4 * (h * BH + bl) + grp;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int v = 0; v < 2; ++v) S[((size_t)fl * RR + r) * OPB + (2 * kq + v) * NT + t] += acc[bl][t][v];
        __syncwarp();
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < FPB * OPB; t += blockDim.x) {
    const int f = t / OPB, oc = t % OPB;
    const int ii = i0 + f, o = o0 + oc;
    if (ii >= d_in || o >= d_out) continue;
    const double* Sf = S + (size_t)f * RR * OPB + oc;
    if (part != nullptr) {
      for (int r = 0; r < R; ++r) part[(size_t)z * d_in * R * d_out + ((size_t)ii * R + r) * d_out + o] = Sf[(size_t)r * OPB];
    } else {
      const double sc = (double)scale[(size_t)ii * d_out + o];
      double ds = 0.0;
      for (int r = 0; r < R; ++r) {
        const size_t ci = ((size_t)ii * R + r) * d_out + o;
        const double a = Sf[(size_t)r * OPB];
        dC[ci] = (float)(sc * a);
        ds = fma((double)C[ci], a, ds);
      }
      dscale[(size_t)ii * d_out + o] = (float)ds;
    }
  }
}

// ---------------------------------------------------------------------------------------
// "tc3": the tc2 sweep (NT = 4 or 8, 4 warps per feature) fed by TMA and synchronised by mbarriers
// instead of CTA barriers.
//  * one elected thread streams each chunk into a 2-deep shared ring: the g tile [256 samples x
//    8*NT outputs] with one 2-D tensor-map TMA per 32 outputs (cp.async.bulk.tensor, 128-byte
//    swizzle, zero fill beyond B / d_out) and the FPB feature records with 1-D bulk copies, all completing on the
//    stage's `full` mbarrier — in place of ~2,900 cp.async issued by every thread per chunk;
//  * each warp evaluates the fp64 basis weights of exactly the sorted positions of its own blocks
//    (its samples are a contiguous run of the cell-sorted chunk) into the stage's weight buffer,
//    so no CTA-wide barrier separates the weight phase from the DMMA phase;
//  * a warp releases a stage with one arrive on its `empty` mbarrier; the next-but-one chunk is
//    loaded into a stage once every warp has released it, so warps drift up to one chunk apart
//    (which also keeps the two weight buffers race-free: the block -> position map changes per
//    chunk, so a warp one chunk ahead writes positions another warp may still be reading).
// Same group order and weight formula as tc2: bitwise-identical results.
static __device__ __forceinline__ void tc_mb_init(uint64_t* mb, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)), "r"(count));
}
static __device__ __forceinline__ void tc_mb_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)),
               "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ void tc_mb_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)) : "memory");
}
static __device__ __forceinline__ void tc_mb_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb);
  asm volatile(
      "{\n.reg .pred p;\nTCW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TCW_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ void tc_bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(mb))
               : "memory");
}
static __device__ __forceinline__ void tc_tma_2d(void* smem, const CUtensorMap* map, int c0, int c1, uint64_t* mb) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"((uint32_t)__cvta_generic_to_shared(mb))
      : "memory");
}

constexpr int kTc3Depth = 2;
constexpr uint32_t kTc3BoxBytes = kTcBC * 32 * 4;  // one TMA box: 256 samples x 32 outputs fp32

// SS ("sample split", few-row dense UKAN segments): each of a feature's WPF warps takes a quarter
// of the chunk's sorted positions over ALL RB blocks instead of RB/WPF blocks over all positions,
// so a handful of populated blocks still keeps every warp busy; the warps' partial rows meet in
// the epilogue in warp order (deterministic; the 4-sample grouping differs from SS = false).
template <int RB, int NT, int FPB, int WPF, bool SS = false>
__global__ void __launch_bounds__(FPB * WPF * 32, 1)
kan_bwd_tc3_sweep_kernel(const __grid_constant__ CUtensorMap gmap, const unsigned char* __restrict__ recs,
                         const float* __restrict__ C, const float* __restrict__ scale, float* __restrict__ dC,
                         float* __restrict__ dscale, double* __restrict__ part, int B, int d_in, int d_out, int G,
                         int nch, int cps, Basis<4> bas, const int32_t* __restrict__ seg) {
  constexpr int OPB = 8 * NT, NBOX = OPB / 32;
  constexpr uint32_t kTc3GBytes = NBOX * kTc3BoxBytes;  // one g stage: 256 samples x OPB outputs
  static_assert(NT == 4 || NT == 8, "32-output TMA boxes");
  constexpr int BH = SS ? RB : RB / WPF;  // blocks per warp
  constexpr int NWARP = FPB * WPF;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_s[kTc3Depth], empty_s[kTc3Depth];
  __shared__ double Msh[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  const int fl = warp / WPF, h = warp % WPF;
  constexpr int kSwFG = 16;  // grid walk in panels of feature groups (as tc2)
  int ot, fg;
  {
    const int n_ot = gridDim.x, n_fg = gridDim.y;
    const int L = blockIdx.y * n_ot + blockIdx.x;
    const int pw = min(kSwFG, n_fg);
    const int sc = L / (pw * n_ot), r = L % (pw * n_ot);
    const int pe = min(pw, n_fg - sc * pw);
    ot = r / pe;
    fg = sc * pw + r % pe;
  }
  const int i0 = fg * FPB;
  const int i = i0 + fl;
  const int o0 = ot * OPB;
  const int z = blockIdx.z;
  const int n_lo = z * cps, n_hi = min(nch, n_lo + cps);
  const int R = G + 3;
  const size_t rb = tc_rec_bytes(G);
  const int nf = min(FPB, d_in - i0);  // features of this CTA with records
  // smem: g ring (1024-aligned for the 128-byte swizzle) | record ring | weight ring
  unsigned char* g_ring =  // the 128-byte swizzle needs 1024-byte aligned tiles
      smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u);
  unsigned char* rec_ring = g_ring + kTc3Depth * kTc3GBytes;
  double* w_ring = reinterpret_cast<double*>(rec_ring + (size_t)kTc3Depth * FPB * rb);  // [depth][FPB][BC][4]
  const bool producer = threadIdx.x == 0;
  if (producer) {
    for (int d = 0; d < kTc3Depth; ++d) {
      tc_mb_init(&full_s[d], 1);
      tc_mb_init(&empty_s[d], NWARP * 32);  // every thread releases its own reads (release semantics per thread)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int q = 0; q < 16; ++q) Msh[q] = bas.M[q / 4][q % 4];
  }
  __syncthreads();
  auto issue = [&](int c) {  // chunk n_lo + c -> stage c % depth
    const int n = n_lo + c, d = c % kTc3Depth;
    uint64_t* mb = &full_s[d];
    tc_mb_expect_tx(mb, kTc3GBytes + (uint32_t)(nf * rb));
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      tc_tma_2d(g_ring + (size_t)d * kTc3GBytes + bx * kTc3BoxBytes, &gmap, o0 + 32 * bx, n * kTcBC, mb);
    for (int f = 0; f < nf; ++f)
      tc_bulk_g2s(rec_ring + ((size_t)d * FPB + f) * rb, recs + ((size_t)(i0 + f) * nch + n) * rb, (uint32_t)rb, mb);
  };
  const int nchunk = n_hi - n_lo;
  if (producer)
    for (int c = 0; c < min(kTc3Depth, nchunk); ++c) issue(c);

  double acc[BH][NT][2];
#pragma unroll
  for (int bb = 0; bb < BH; ++bb)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[bb][t][0] = acc[bb][t][1] = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    const int d = c % kTc3Depth;
    double* wf = w_ring + ((size_t)d * FPB + fl) * kTcBC * 4;
    tc_mb_wait(&full_s[d], (uint32_t)((c / kTc3Depth) & 1));
    if (i < d_in) {
      const unsigned char* rec = rec_ring + ((size_t)d * FPB + fl) * rb;
      const int* ent = reinterpret_cast<const int*>(rec);
      const double* uu = reinterpret_cast<const double*>(rec + kTcBC * 4);
      const int* st = reinterpret_cast<const int*>(rec + kTcBC * 12);
      // this warp's sorted positions: the cells of its blocks [h*BH, (h+1)*BH), or (SS) its quarter
      const int p_lo = SS ? min(h * (kTcBC / WPF), st[G]) : st[min(4 * h * BH, G)];
      const int p_hi = SS ? min((h + 1) * (kTcBC / WPF), st[G]) : st[min(4 * (h + 1) * BH, G)];
      for (int p = p_lo + lane; p < p_hi; p += 32) {  // fp64 Horner, layers.py:29-37
        const double u = uu[p];
        double* wd = wf + (size_t)p * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) wd[j] = fma(fma(fma(Msh[12 + j], u, Msh[8 + j]), u, Msh[4 + j]), u, Msh[j]);
      }
      __syncwarp();
      const unsigned char* gt = g_ring + (size_t)d * kTc3GBytes;
      // B operand: lane (sample kq, column grp) of tile t is output o0 + grp*NT + t: 16-byte chunks
      // grp*NT/4 + q of the sample's row, chunk c of a box row stored at c ^ (row & 7) (128-byte swizzle)
      auto load_group = [&](int kc, int e1, double& a, float4 (&gv)[NT / 4]) {
        const int pos = kc + kq;
        const int pc = pos < e1 ? pos : kc;  // masked lanes read an own, finished position
        const int e = ent[pc];
        const int j = grp - ((e >> 8) & 3);
        const double wj = wf[pc * 4 + (j & 3)];
        a = (pos < e1 && j >= 0 && j < 4) ? wj : 0.0;
        const int srow = e & 255;
#pragma unroll
        for (int q = 0; q < NT / 4; ++q) {
          const int cc = grp * (NT / 4) + q;
          gv[q] = *reinterpret_cast<const float4*>(gt + (cc >> 3) * kTc3BoxBytes + srow * 128 + (((cc & 7) ^ (srow & 7)) << 4));
        }
      };
#pragma unroll
      for (int bl = 0; bl < BH; ++bl) {
        const int bb = SS ? bl : h * BH + bl;
        const int e0 = SS ? max(st[min(4 * bb, G)], p_lo) : st[min(4 * bb, G)];
        const int e1 = SS ? min(st[min(4 * bb + 4, G)], p_hi) : st[min(4 * bb + 4, G)];
        int kc = e0;
        for (; kc + 4 < e1; kc += 8) {  // two groups in flight
          double a0, a1;
          float4 g0[NT / 4], g1[NT / 4];
          load_group(kc, e1, a0, g0);
          load_group(kc + 4, e1, a1, g1);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v0 = t % 4 == 0 ? g0[t / 4].x : t % 4 == 1 ? g0[t / 4].y : t % 4 == 2 ? g0[t / 4].z : g0[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a0, (double)v0);
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v1 = t % 4 == 0 ? g1[t / 4].x : t % 4 == 1 ? g1[t / 4].y : t % 4 == 2 ? g1[t / 4].z : g1[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a1, (double)v1);
          }
        }
        if (kc < e1) {
          double a0;
          float4 g0[NT / 4];
          load_group(kc, e1, a0, g0);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float v0 = t % 4 == 0 ? g0[t / 4].x : t % 4 == 1 ? g0[t / 4].y : t % 4 == 2 ? g0[t / 4].z : g0[t / 4].w;
            tc_dmma(acc[bl][t][0], acc[bl][t][1], a0, (double)v0);
          }
        }
      }
    }
    tc_mb_arrive(&empty_s[d]);
    // refill this stage with chunk c+2 once every thread has released chunk c
    if (producer && c + kTc3Depth < nchunk) {
      tc_mb_wait(&empty_s[d], (uint32_t)((c / kTc3Depth) & 1));
      issue(c + kTc3Depth);
    }
  }
  __syncthreads();  // every stage consumed (all issued loads were waited on): the ring is free
  // epilogue (as tc2): rows of both halves meet in S[FPB][R][OPB] (fp64, reuses the ring)
  double* S = reinterpret_cast<double*>(g_ring);
  const int RR = 4 * RB + 4;
  for (int t = threadIdx.x; t < FPB * RR * OPB; t += blockDim.x) S[t] = 0.0;
  __syncthreads();
#pragma unroll
  for (int hh = 0; hh < WPF; ++hh) {
    if (h == hh) {
#pragma unroll
      for (int bl = 0; bl < BH; ++bl) {
        const int r = 4 * (SS ? bl : h * BH + bl) + grp;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int v = 0; v < 2; ++v) S[((size_t)fl * RR + r) * OPB + (2 * kq + v) * NT + t] += acc[bl][t][v];
        __syncwarp();
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < FPB * OPB; t += blockDim.x) {
    const int f = t / OPB, oc = t % OPB;
    const int ii = i0 + f, o = o0 + oc;
    if (ii >= d_in || o >= d_out) continue;
    const double* Sf = S + (size_t)f * RR * OPB + oc;
    int rbase = ii * R, nr = R;  // UKAN: the feature's own row segment of the table
    if (seg != nullptr) {
      rbase = 4 * seg[ii];
      nr = 4 * seg[ii + 1] - rbase;
    }
    if (part != nullptr) {
      for (int r = 0; r < R; ++r) part[(size_t)z * d_in * R * d_out + ((size_t)ii * R + r) * d_out + o] = Sf[(size_t)r * OPB];
    } else {
      const double sc = (double)scale[(size_t)ii * d_out + o];
      double ds = 0.0;
      for (int r = 0; r < nr; ++r) {
        const size_t ci = ((size_t)rbase + r) * d_out + o;
        const double a = Sf[(size_t)r * OPB];
        dC[ci] = (float)(sc * a);
        ds = fma((double)C[ci], a, ds);
      }
      dscale[(size_t)ii * d_out + o] = (float)ds;
    }
  }
}

// Fixed-order reduction of the split-batch partials + epilogue: CTA = (feature i, 32 outputs);
// threads sweep the (row, output) pairs (coalesced over o): dC = scale * sum_z part, and the
// per-row products C * A meet in shared memory for dscale = sum_r C * A (row order).
__global__ void __launch_bounds__(256) kan_bwd_tc_reduce_kernel(const double* __restrict__ part,
                                                                const float* __restrict__ C,
                                                                const float* __restrict__ scale,
                                                                float* __restrict__ dC, float* __restrict__ dscale,
                                                                int S, int d_in, int d_out, int R,
                                                                const int32_t* __restrict__ seg = nullptr) {
  extern __shared__ double prod[];  // [R][32]
  const int i = blockIdx.x, o0 = blockIdx.y * 32;
  const size_t zs = (size_t)d_in * R * d_out;
  // the partials use the padded [d_in][R] row layout; dC / C rows: the feature's segment (UKAN)
  const int rbase = seg ? 4 * seg[i] : i * R, nr = seg ? 4 * (seg[i + 1] - seg[i]) : R;
  for (int p = threadIdx.x; p < R * 32; p += blockDim.x) {
    const int r = p >> 5, ol = p & 31, o = o0 + ol;
    double pr = 0.0;
    if (o < d_out && r < nr) {
      const size_t pi = ((size_t)i * R + r) * d_out + o, ci = ((size_t)rbase + r) * d_out + o;
      double a = 0.0;
      for (int z = 0; z < S; ++z) a += part[z * zs + pi];
      dC[ci] = (float)((double)scale[(size_t)i * d_out + o] * a);
      pr = (double)C[ci] * a;
    }
    prod[p] = pr;
  }
  __syncthreads();
  if (threadIdx.x < 32 && o0 + threadIdx.x < d_out) {
    double ds = 0.0;
    for (int r = 0; r < R; ++r) ds += prod[r * 32 + threadIdx.x];
    dscale[(size_t)i * d_out + o0 + threadIdx.x] = (float)ds;
  }
}

// ---------------------------------------------------------------------------------------
struct TcPlan {
  bool ok = false;
  int rb = 0, nt = 4, S = 1, cps = 0, nch = 0, fpb = 4, wpf = 2;
  bool split = false;
  size_t smem = 0;
  int64_t rec_bytes = 0, part_bytes = 0;
};

static int tc_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
  }
  return n;
}

TcPlan kan_bwd_tc_plan(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base) {
  TcPlan p;
  if (k != 3 || has_base || G < 1 || G > 64 || B < 1) return p;
  const int rbn = (int)((G - 1) >> 2) + 1;
  p.rb = rbn <= 4 ? 4 : (rbn <= 8 ? 8 : 16);
  p.nt = p.rb == 16 ? 2 : (d_out <= 8 ? 1 : (d_out <= 16 ? 2 : 4));
  static const bool no_tc2 = getenv("UKAN_NO_TC2") != nullptr;  // A/B measurement only
  p.split = !no_tc2 && p.rb >= 8 && d_out >= 32;  // two warps per feature (tc2 kernel)
  // Layer 0 of cfg2 (KAN 784->256, B=8192): 4 warps per feature x NT=8 ("16", default) 1.74 ms;
  // 2 warps x NT=4 with 8 features ("4") 1.88 ms; 2 warps x NT=8 ("8") 1.94 ms (A/B via UKAN_TC2_NT)
  static const int tc2_wide = getenv("UKAN_TC2_NT") ? atoi(getenv("UKAN_TC2_NT")) : 16;
  if (p.split) p.nt = (p.rb == 8 && d_out >= 64 && tc2_wide == 8) ? 8 : 4;
  if (p.split && p.rb == 8 && p.nt == 4 && tc2_wide == 4) p.fpb = 8;  // 16 warps, 8 features
  if (p.split && p.rb == 8 && d_out >= 64 && tc2_wide == 16) {  // 16 warps: 4 features x 4 block parts, NT = 8
    p.wpf = 4;
    p.nt = 8;
    p.fpb = 4;
  }
  static const int rb16_wpf = getenv("UKAN_TC2_RB16_WPF") ? atoi(getenv("UKAN_TC2_RB16_WPF")) : 4;
  if (p.split && p.rb == 16 && rb16_wpf == 4) {  // 16 warps: 4 features x 4 block parts, NT = 4
    p.wpf = 4;
    p.nt = 4;
    p.fpb = 4;
  }
  if (p.split && p.rb == 16 && rb16_wpf == 8 && d_out >= 64) {  // 16 warps: 2 features x 8 block parts, NT = 8
    p.wpf = 8;
    p.nt = 8;
    p.fpb = 2;
  }
  if (p.split && p.rb == 16 && rb16_wpf == 84) {  // 32 warps: 4 features x 8 block parts, NT = 4 (64 registers)
    p.wpf = 8;
    p.nt = 4;
    p.fpb = 4;
  }
  const int opb = 8 * p.nt;
  const int fpb = p.split ? p.fpb : 8;
  p.nch = (int)((B + kTcBC - 1) / kTcBC);
  p.smem = 2 * fpb * tc_rec_bytes((int)G) + sizeof(float) * (size_t)2 * kTcBC * (opb + (p.split ? 8 : 0));
  if (p.split) {
    p.smem += sizeof(double) * (size_t)fpb * kTcBC * 4;  // per-sample basis weights
    p.smem = std::max<size_t>(p.smem, sizeof(double) * (size_t)fpb * (4 * p.rb + 4) * opb);
  }
  p.rec_bytes = (int64_t)d_in * p.nch * (int64_t)tc_rec_bytes((int)G);
  const int sms = tc_sms();
  const int64_t base = ((d_in + fpb - 1) / fpb) * ((d_out + opb - 1) / opb);
  int64_t S = 1;
  if (base < 2 * (int64_t)sms) {
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(16, p.nch / 4));
    double best = -1.0;
    for (int64_t c = 1; c <= max_s; ++c) {
      const double waves = (double)(base * c) / sms;
      const double eff = waves / std::ceil(waves) * std::min(1.0, waves / 2.0);
      if (eff > best + 1e-9) { best = eff; S = c; }
    }
  }
  if (getenv("UKAN_TC_S")) S = std::max<int64_t>(1, atoi(getenv("UKAN_TC_S")));  // A/B measurement only
  p.cps = (int)((p.nch + S - 1) / S);
  p.S = (p.nch + p.cps - 1) / p.cps;
  p.part_bytes = p.S > 1 ? (int64_t)sizeof(double) * p.S * d_in * d_out * (G + 3) : 0;
  p.ok = true;
  return p;
}

int64_t kan_bwd_tc_workspace(const TcPlan& p) { return p.ok ? ((p.rec_bytes + 255) / 256) * 256 + p.part_bytes : 0; }

template <int RB, int NT, int FPB, int WPF>
static int tc2_launch(const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                      unsigned char* recs, double* part, int B, int d_in, int d_out, int G, const TcPlan& p,
                      cudaStream_t st) {
  auto kern = kan_bwd_tc2_sweep_kernel<RB, NT, FPB, WPF>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 gridd((d_out + 8 * NT - 1) / (8 * NT), (d_in + FPB - 1) / FPB, p.S);
  kern<<<gridd, FPB * WPF * 32, p.smem, st>>>(recs, C, scale, gy, dC, dscale, p.S > 1 ? part : nullptr, B, d_in, d_out, G,
                                   p.nch, p.cps, make_basis<4>(3));
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    kan_bwd_tc_reduce_kernel<<<dim3(d_in, (d_out + 31) / 32), 256, sizeof(double) * (G + 3) * 32, st>>>(
        part, C, scale, dC, dscale, p.S, d_in, d_out, G + 3);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

// 2-D tensor map of g [B, d_out] fp32: box 32 outputs x 256 samples, 128-byte swizzle, zero fill
static bool tc3_tensor_map(CUtensorMap* map, const float* gy, int B, int d_out) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (encode == nullptr) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)d_out, (cuuint64_t)B};
  const cuuint64_t strides[1] = {(cuuint64_t)d_out * 4};
  const cuuint32_t box[2] = {32, (cuuint32_t)kTcBC};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gy), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t tc3_smem(int G, int fpb, int rb, int nt) {
  const size_t ring = (size_t)kTc3Depth * (nt / 4) * kTc3BoxBytes + (size_t)kTc3Depth * fpb * tc_rec_bytes(G) +
                      sizeof(double) * (size_t)kTc3Depth * fpb * kTcBC * 4;
  return 1024 + std::max(ring, sizeof(double) * (size_t)fpb * (4 * rb + 4) * 8 * nt);  // + alignment slack
}

// tc3 applies to the NT = 4 tc2 shapes (32-output tiles) with 16-byte aligned g rows
static bool tc3_enabled() {
  static const bool off = getenv("UKAN_TC3") && getenv("UKAN_TC3")[0] == '0';  // A/B measurement only
  return !off;
}

template <int RB, int NT, int FPB, int WPF, bool SS = false>
static int tc3_launch(const CUtensorMap& map, const float* C, const float* scale, float* dC, float* dscale,
                      unsigned char* recs, double* part, int B, int d_in, int d_out, int G, const TcPlan& p,
                      cudaStream_t st, const int32_t* seg = nullptr) {
  auto kern = kan_bwd_tc3_sweep_kernel<RB, NT, FPB, WPF, SS>;
  const size_t smem = tc3_smem(G, FPB, RB, NT);
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 gridd((d_out + 8 * NT - 1) / (8 * NT), (d_in + FPB - 1) / FPB, p.S);
  kern<<<gridd, FPB * WPF * 32, smem, st>>>(map, recs, C, scale, dC, dscale, p.S > 1 ? part : nullptr, B, d_in, d_out, G,
                                            p.nch, p.cps, make_basis<4>(3), seg);
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    kan_bwd_tc_reduce_kernel<<<dim3(d_in, (d_out + 31) / 32), 256, sizeof(double) * (G + 3) * 32, st>>>(
        part, C, scale, dC, dscale, p.S, d_in, d_out, G + 3, seg);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

template <int RB, int NT>
static int tc_launch(const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                     unsigned char* recs, double* part, int B, int d_in, int d_out, int G, const TcPlan& p,
                     cudaStream_t st) {
  auto kern = kan_bwd_tc_sweep_kernel<RB, NT>;
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  dim3 gridd((d_in + 7) / 8, (d_out + 8 * NT - 1) / (8 * NT), p.S);
  kern<<<gridd, 256, p.smem, st>>>(recs, C, scale, gy, dC, dscale, p.S > 1 ? part : nullptr, B, d_in, d_out, G,
                                   p.nch, p.cps, make_basis<4>(3));
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    kan_bwd_tc_reduce_kernel<<<dim3(d_in, (d_out + 31) / 32), 256, sizeof(double) * (G + 3) * 32, st>>>(
        part, C, scale, dC, dscale, p.S, d_in, d_out, G + 3);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

// Records only (the first half of kan_bwd_tc_run): lets a caller run the x-only prep early on a
// side stream, overlapping the layers above, and pass prepared = true to kan_bwd_tc_run.
int kan_bwd_tc_prep(const float* x, void* workspace, int64_t ws_bytes, int B, int d_in, int G, const KanGrid& grid,
                    const TcPlan& p, cudaStream_t st) {
  if (!p.ok || workspace == nullptr || ws_bytes < kan_bwd_tc_workspace(p)) return UKAN_E_WORKSPACE;
  dim3 pg((d_in + 7) / 8, p.nch);
  kan_bwd_tc_prep_kernel<false><<<pg, 256, 0, st>>>(x, reinterpret_cast<unsigned char*>(workspace), B, d_in, p.nch, G,
                                                     grid, nullptr, nullptr, 0.0);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

static int tc_sweep_dispatch(const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                             unsigned char* recs, double* part, int B, int d_in, int d_out, int G, const TcPlan& p,
                             cudaStream_t st) {
  CUtensorMap map;  // tc3: the driver's tensor-map encoder is required (else the tc2 sweep runs)
  const bool tc3 = tc3_enabled() && (d_out % 4) == 0 && ((uintptr_t)gy % 16) == 0 && p.split && p.wpf == 4 &&
                   ((p.rb == 16 && p.nt == 4) || (p.rb == 8 && p.nt == 8)) && tc3_tensor_map(&map, gy, B, d_out);
  if (tc3 && p.rb == 16) return tc3_launch<16, 4, 4, 4>(map, C, scale, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (tc3 && p.rb == 8) return tc3_launch<8, 8, 4, 4>(map, C, scale, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 8 && p.wpf == 4) return tc2_launch<8, 8, 4, 4>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 8 && p.nt == 8) return tc2_launch<8, 8, 4, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 8 && p.fpb == 8) return tc2_launch<8, 4, 8, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 8) return tc2_launch<8, 4, 4, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 16 && p.wpf == 4) return tc2_launch<16, 4, 4, 4>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 16 && p.wpf == 8 && p.fpb == 2) return tc2_launch<16, 8, 2, 8>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 16 && p.wpf == 8) return tc2_launch<16, 4, 4, 8>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.split && p.rb == 16) return tc2_launch<16, 4, 4, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 4 && p.nt == 1) return tc_launch<4, 1>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 4 && p.nt == 2) return tc_launch<4, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 4) return tc_launch<4, 4>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 8 && p.nt == 1) return tc_launch<8, 1>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 8 && p.nt == 2) return tc_launch<8, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 8) return tc_launch<8, 4>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  if (p.rb == 16) return tc_launch<16, 2>(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
  return UKAN_E_ARG;
}

int kan_bwd_tc_run(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                   void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int G, const KanGrid& grid,
                   const TcPlan& p, cudaStream_t st, bool prepared) {
  if (!p.ok || workspace == nullptr || ws_bytes < kan_bwd_tc_workspace(p)) return UKAN_E_WORKSPACE;
  unsigned char* recs = reinterpret_cast<unsigned char*>(workspace);
  double* part = reinterpret_cast<double*>(recs + ((p.rec_bytes + 255) / 256) * 256);
  if (!prepared) {
    const int rc = kan_bwd_tc_prep(x, workspace, ws_bytes, B, d_in, G, grid, p, st);
    if (rc) return rc;
  }
  return tc_sweep_dispatch(C, scale, gy, dC, dscale, recs, part, B, d_in, d_out, G, p, st);
}

// ---------------------------------------------------------------------------------------
// dx on the FP64 tensor cores (wide layers, k = 3, no base branch), from the same sorted records
// (replaces the per-(sample, feature) warp dot products of spline_dx_kernel, which are bound by
// the fp32 -> fp64 conversions of every operand):
//   Q[b, r]  = sum_o g[b, o] * C'[i, r, o]          C' = scale * C, exact in fp64
//   dx[b, i] = mask * inv_dg * sum_j w'_j(u_b) * Q[b, cell_b + j]       (layers.py:44-46, 84-88,
//                                                                        tensor.py:330 clamp mask)
// Task = up to 8 consecutive cell-sorted samples of one feature whose cells lie in [c0, c0+4]:
// their windows fit rows c0..c0+7, so one m8n8k4 DMMA per 4 outputs computes
//   D[8 samples x 8 rows] += A[8 samples x 4 outputs] (g) * B[4 outputs x 8 rows] (C'),
// accumulated over ALL outputs in registers (half of D is outside each sample's window: the
// banded product's 50% ceiling).  CTA = 4 features x one 256-sample chunk,
// 16 warps, <= 12 tasks per warp; output tiles of 16: g (fp32, cp.async) and C' (fp64, register
// prefetch, widened and scaled once per CTA) double-buffered in shared memory, one barrier per
// tile.  The grid is walked in bands of `band` chunks x all feature groups so a wave shares the
// band's g rows and a few features' C' through L2.  Deterministic: fixed task order, fixed DMMA
// order over the outputs, fixed 4-lane reduction.
// ---------------------------------------------------------------------------------------
constexpr int kDxF = 4;            // features per CTA (task_at below is written for 4)
constexpr int kDxOT = 16;          // outputs per staged tile
constexpr int kDxGS = kDxOT;       // fp32 g row stride (floats, 64 B): a row's bank half = sample & 1
constexpr int kDxCS = kDxOT + 2;   // fp64 C' row stride (doubles, 144 B): adjacent rows on disjoint banks
// warps per CTA NW and task slots per warp MAXT: tasks per CTA <= 4 * (256/8 + G/5 + 1) <= 184 for G <= 64,
// so 16 warps need 12 slots, 32 warps 6 (fewer registers per thread, twice the warps per scheduler)
constexpr int kDxMaxT = 12;
constexpr int kDxTPF = 48;         // task slots per feature (>= 256/8 + 64/5 + 1)

__host__ __device__ constexpr int dx_rr(int G) { return G + 8; }  // C' tile rows: c0 + 7 <= G + 6

struct DxSmem {  // byte offsets of the dynamic shared-memory regions
  size_t rec, task, g, c, dxs, total;
};
__host__ __device__ inline DxSmem dx_smem_layout(int G) {
  DxSmem L;
  L.rec = 0;
  L.task = L.rec + (size_t)kDxF * tc_rec_bytes(G);
  L.g = L.task + sizeof(int4) * kDxF * kDxTPF + 16;
  L.c = L.g + sizeof(float) * 2 * (kTcBC + 1) * kDxGS;
  L.c = (L.c + 15) / 16 * 16;
  L.dxs = L.c + sizeof(double) * 2 * kDxF * dx_rr(G) * kDxCS;
  L.total = L.dxs + sizeof(float) * kTcBC * kDxF;
  return L;
}

// Position (within a task's sorted run [p0, p1)) whose sample feeds A-row `grp`, or -1 for a
// padding row.  Samples with even and odd g-tile rows are interleaved so the two rows read by one
// quarter-warp of the LDS.128 A load sit in different bank halves whenever the run allows it.
__device__ __forceinline__ int dx_lane_pos(const int* ent, int p0, int p1, int grp) {
  const int n = p1 - p0;
  unsigned em = 0, om = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < n) {
      if (ent[p0 + q] & 1) om |= 1u << q;
      else em |= 1u << q;
    }
  if (grp >= n) return -1;
  const int ne = __popc(em), no = __popc(om), m = min(ne, no);
  unsigned mask;
  int idx;
  if (grp < 2 * m) {
    mask = (grp & 1) ? om : em;
    idx = grp >> 1;
  } else {
    mask = ne > no ? em : om;
    idx = grp - m;
  }
  return (int)__fns(mask, 0, idx + 1);
}

// One staged output tile for NT tasks: per task one LDS.128 of A (4 fp32 g values of this lane's
// sample) and two LDS.128 of B (4 fp64 C' values of row c0 + grp), then 4 DMMAs.  The k slot of
// lane kq in DMMA kk is output 4*kq + kk (any fixed k order is valid: A and B use the same one).
template <int NT, int MAXT>
__device__ __forceinline__ void dx_tile(const float* __restrict__ gb, const double* __restrict__ cb,
                                        const uint32_t (&toff)[MAXT], double (&acc)[MAXT][2]) {
  // tasks in pairs: both tasks' operands are loaded before either DMMA chain starts and the two
  // accumulator chains interleave (the A operand's LDS -> F2F -> DMMA latency overlaps)
#pragma unroll
  for (int t0 = 0; t0 < NT; t0 += 2) {
    constexpr int W = 2;
    float4 a[W];
    double2 b0[W], b1[W];
#pragma unroll
    for (int u = 0; u < W; ++u) {
      if (t0 + u < NT) {
        a[u] = *reinterpret_cast<const float4*>(gb + (toff[t0 + u] & 0xffffu));
        const double* cp = cb + (toff[t0 + u] >> 16);
        b0[u] = *reinterpret_cast<const double2*>(cp);
        b1[u] = *reinterpret_cast<const double2*>(cp + 2);
      }
    }
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (t0 + u < NT) tc_dmma(acc[t0 + u][0], acc[t0 + u][1], (double)a[u].x, b0[u].x);
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (t0 + u < NT) tc_dmma(acc[t0 + u][0], acc[t0 + u][1], (double)a[u].y, b0[u].y);
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (t0 + u < NT) tc_dmma(acc[t0 + u][0], acc[t0 + u][1], (double)a[u].z, b1[u].x);
#pragma unroll
    for (int u = 0; u < W; ++u)
      if (t0 + u < NT) tc_dmma(acc[t0 + u][0], acc[t0 + u][1], (double)a[u].w, b1[u].y);
  }
}

template <int kDxW, int MAXT, bool UK = false>  // UK: dense UKAN, each feature's rows = its table segment (seg)
__global__ void __launch_bounds__(kDxW * 32, 1)
kan_dx_tc_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ C, const float* __restrict__ scale,
                 const float* __restrict__ gy, float* __restrict__ dx, int B, int d_in, int d_out, int G, int nch,
                 int n_fg, int band, int ld, double inv_dg, Basis<4> bas, const int32_t* __restrict__ seg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double Msh[16];
  __shared__ int cnt_s[kDxF];
  __shared__ int rbase_s[kDxF], nr_s[kDxF];  // each feature's row segment (UKAN: its own slice of the table)
  const DxSmem L = dx_smem_layout(G);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  const int R = G + 3, RR = dx_rr(G);
  const size_t rb = tc_rec_bytes(G);
  if (threadIdx.x == 0) {  // constant indices: no local-memory copy of the parameter struct
#pragma unroll
    for (int q = 0; q < 16; ++q) Msh[q] = bas.M[q / 4][q % 4];
  }
  // banded walk: band b covers chunks [b*band, ...) x all feature groups, feature group major
  const int64_t lin = blockIdx.x;
  const int64_t per_band = (int64_t)band * n_fg;
  const int bnd = (int)(lin / per_band);
  const int rem = (int)(lin % per_band);
  const int cb = min(band, nch - bnd * band);
  const int fg = rem / cb, n = bnd * band + rem % cb;
  const int i0 = fg * kDxF;
  const int b0 = n * kTcBC;
  const int nb = min(kTcBC, B - b0);
  if constexpr (UK) {
    if (threadIdx.x < kDxF) {
      const int ii = min(i0 + (int)threadIdx.x, d_in - 1);
      rbase_s[threadIdx.x] = 4 * seg[ii];
      nr_s[threadIdx.x] = 4 * (seg[ii + 1] - seg[ii]);
    }
    __syncthreads();
  }
  unsigned char* rec_s = smem_raw + L.rec;
  int4* task_s = reinterpret_cast<int4*>(smem_raw + L.task);
  float* g_s = reinterpret_cast<float*>(smem_raw + L.g);
  double* c_s = reinterpret_cast<double*>(smem_raw + L.c);
  float* dx_s = reinterpret_cast<float*>(smem_raw + L.dxs);
  const int GSZ = (kTcBC + 1) * kDxGS, CSZ = kDxF * RR * kDxCS;
  
  // records of the 4 features (16-byte granules)
  {
    const int q = (int)(rb / 16);
    for (int t = threadIdx.x; t < kDxF * q; t += blockDim.x) {
      const int f = t / q, c = t % q;
      const bool ok = i0 + f < d_in;
      const unsigned char* src = ok ? recs + ((size_t)(i0 + f) * nch + n) * rb + (size_t)c * 16 : recs;
      tc_cp16(rec_s + (size_t)f * rb + (size_t)c * 16, src, ok ? 16 : 0);
    }
  }
  // zero row 256 of both g buffers (the A operand of padding lanes) and the C' pad rows
  for (int t = threadIdx.x; t < 2 * kDxGS; t += blockDim.x) g_s[(t / kDxGS) * GSZ + kTcBC * kDxGS + t % kDxGS] = 0.f;
  const int nq = kDxOT / 4;
  auto stage_g = [&](int o0, int buf) {
    float* gd = g_s + buf * GSZ;
    for (int t = threadIdx.x; t < kTcBC * nq; t += blockDim.x) {
      const int sm = t / nq, j = (t % nq) * 4;
      const bool ok = sm < nb && o0 + j < d_out;
      tc_cp16(gd + sm * kDxGS + j, ok ? gy + (size_t)(b0 + sm) * d_out + o0 + j : gy, ok ? 16 : 0);
    }
  };
  constexpr int CQ = (kDxF * (64 + 8) * (kDxOT / 4) + kDxW * 32 - 1) / (kDxW * 32);  // float4 per thread (G <= 64)
  float4 cr[CQ];
  auto load_c = [&](int o0) {
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int t = threadIdx.x + q * kDxW * 32;
      const int j = (t % nq) * 4, fr = t / nq, r = fr % RR, f = fr / RR;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (UK) {
        if (f < kDxF && i0 + f < d_in && r < nr_s[f] && o0 + j < d_out)
          v = __ldg(reinterpret_cast<const float4*>(C + ((size_t)rbase_s[f] + r) * d_out + o0 + j));
      } else {
        if (f < kDxF && r < R && i0 + f < d_in && o0 + j < d_out)
          v = __ldg(reinterpret_cast<const float4*>(C + ((size_t)(i0 + f) * R + r) * d_out + o0 + j));
      }
      cr[q] = v;
    }
  };
  auto store_c = [&](int o0, int buf) {
    double* cd = c_s + buf * CSZ;
#pragma unroll
    for (int q = 0; q < CQ; ++q) {
      const int t = threadIdx.x + q * kDxW * 32;
      const int j = (t % nq) * 4, fr = t / nq, r = fr % RR, f = fr / RR;
      if (f >= kDxF) continue;
      float4 sc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + f < d_in && o0 + j < d_out) sc = __ldg(reinterpret_cast<const float4*>(scale + (size_t)(i0 + f) * d_out + o0 + j));
      double* d = cd + ((size_t)f * RR + r) * kDxCS + j;  // C' = scale * C: exact in fp64
      *reinterpret_cast<double2*>(d) = make_double2((double)cr[q].x * (double)sc.x, (double)cr[q].y * (double)sc.y);
      *reinterpret_cast<double2*>(d + 2) = make_double2((double)cr[q].z * (double)sc.z, (double)cr[q].w * (double)sc.w);
    }
  };
  const int n_ot = (d_out + kDxOT - 1) / kDxOT;
  stage_g(0, 0);
  asm volatile("cp.async.commit_group;\n" ::);
  load_c(0);
  store_c(0, 0);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // tasks: greedy runs of <= 8 sorted samples with cells in [c0, c0 + 4] (one thread per feature)
  if (threadIdx.x < kDxF) {
    const int f = threadIdx.x;
    int cnt = 0;
    if (i0 + f < d_in) {
      const int* ent = reinterpret_cast<const int*>(rec_s + (size_t)f * rb);
      int p = 0;
      while (p < nb) {
        const int c0 = (ent[p] >> 8) & 127;
        int q = p + 1;
        while (q < nb && q - p < 8 && ((ent[q] >> 8) & 127) <= c0 + 4) ++q;
        task_s[f * kDxTPF + cnt] = make_int4(f, c0, p, q);
        ++cnt;
        p = q;
      }
    }
    cnt_s[f] = cnt;
  }
  __syncthreads();
  const int T = cnt_s[0] + cnt_s[1] + cnt_s[2] + cnt_s[3];
  const int per = (T + kDxW - 1) / kDxW;
  const int t_lo = min(T, warp * per), nt = min(per, T - t_lo);
  // per task: packed smem offsets (A: g row of this lane's sample, B: C' row c0 + grp)
  auto task_at = [&](int gt) {  // global task index -> its record (feature-major order), no local arrays
    const int c0 = cnt_s[0], c1 = c0 + cnt_s[1], c2 = c1 + cnt_s[2];
    const int f = gt >= c2 ? 3 : (gt >= c1 ? 2 : (gt >= c0 ? 1 : 0));
    const int base = f == 3 ? c2 : (f == 2 ? c1 : (f == 1 ? c0 : 0));
    return task_s[f * kDxTPF + gt - base];
  };
  uint32_t toff[MAXT];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    toff[t] = 0;
    if (t < nt) {
      const int4 ti = task_at(t_lo + t);
      const int f = ti.x;
      const int* ent = reinterpret_cast<const int*>(rec_s + (size_t)f * rb);
      const int q = dx_lane_pos(ent, ti.z, ti.w, grp);
      const int sm = q >= 0 ? (ent[ti.z + q] & 255) : kTcBC;  // padding lanes read the zero row
      toff[t] = (uint32_t)(sm * kDxGS + 4 * kq) | ((uint32_t)((f * RR + ti.y + grp) * kDxCS + 4 * kq) << 16);
    }
  }
  double acc[MAXT][2];
#pragma unroll
  for (int t = 0; t < MAXT; ++t) acc[t][0] = acc[t][1] = 0.0;
  for (int ot = 0; ot < n_ot; ++ot) {
    const int buf = ot & 1;
    const bool more = ot + 1 < n_ot;
    if (more) {
      stage_g((ot + 1) * kDxOT, buf ^ 1);
      asm volatile("cp.async.commit_group;\n" ::);
      load_c((ot + 1) * kDxOT);
    }
    const float* gb = g_s + buf * GSZ;
    const double* cbuf = c_s + buf * CSZ;
    switch (nt) {  // warp-uniform: a fully unrolled, predicate-free body per task count
      case 1: dx_tile<1, MAXT>(gb, cbuf, toff, acc); break;
      case 2: dx_tile<2, MAXT>(gb, cbuf, toff, acc); break;
      case 3: dx_tile<3, MAXT>(gb, cbuf, toff, acc); break;
      case 4: dx_tile<4, MAXT>(gb, cbuf, toff, acc); break;
      case 5: dx_tile<5, MAXT>(gb, cbuf, toff, acc); break;
      case 6: dx_tile<6, MAXT>(gb, cbuf, toff, acc); break;
      default:
        if constexpr (MAXT > 6) {
          switch (nt) {
            case 7: dx_tile<7, MAXT>(gb, cbuf, toff, acc); break;
            case 8: dx_tile<8, MAXT>(gb, cbuf, toff, acc); break;
            case 9: dx_tile<9, MAXT>(gb, cbuf, toff, acc); break;
            case 10: dx_tile<10, MAXT>(gb, cbuf, toff, acc); break;
            case 11: dx_tile<11, MAXT>(gb, cbuf, toff, acc); break;
            case 12: dx_tile<12, MAXT>(gb, cbuf, toff, acc); break;
            default: break;
          }
        }
        break;
    }
    if (more) {
      store_c((ot + 1) * kDxOT, buf ^ 1);
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
  }
  // epilogue: lane (grp, kq) holds Q[sample grp][rows c0 + 2kq, c0 + 2kq + 1]
#pragma unroll
  for (int t = 0; t < MAXT; ++t) {
    if (t < nt) {
      const int4 ti = task_at(t_lo + t);
      const int f = ti.x;
      const int q = dx_lane_pos(reinterpret_cast<const int*>(rec_s + (size_t)f * rb), ti.z, ti.w, grp);
      const int pos = ti.z + max(q, 0);
      const bool vld = q >= 0;
      const unsigned char* rec = rec_s + (size_t)f * rb;
      const int e = vld ? reinterpret_cast<const int*>(rec)[pos] : 0;
      const double u = vld ? reinterpret_cast<const double*>(rec + kTcBC * 4)[pos] : 0.0;
      const int cell = (e >> 8) & 127;
      double part = 0.0;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = ti.y + 2 * kq + v - cell;
        if (vld && j >= 0 && j < 4) {  // w'_j(u) = M1j + 2 u M2j + 3 u^2 M3j (layers.py:29-37, d = 1)
          const double wp = fma(fma(3.0 * Msh[12 + j], u, 2.0 * Msh[8 + j]), u, Msh[4 + j]);
          part = fma(wp, acc[t][v], part);
        }
      }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      if (vld && kq == 0) dx_s[(e & 255) * kDxF + f] = (e & kTcClamped) ? 0.f : (float)(part * inv_dg);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nb * kDxF; t += blockDim.x) {
    const int sm = t / kDxF, f = t % kDxF;
    if (i0 + f < d_in) dx[(size_t)(b0 + sm) * ld + i0 + f] = dx_s[t];
  }
}

bool kan_dx_tc_applicable(const TcPlan& p, const float* C, const float* gy, int d_out, int G) {
  static const bool off = getenv("UKAN_DX") && getenv("UKAN_DX")[0] == 's';  // A/B: the SIMT dx kernel
  return !off && p.ok && G <= 64 && d_out >= 64 && d_out % 4 == 0 && ((uintptr_t)C % 16) == 0 &&
         ((uintptr_t)gy % 16) == 0;
}

// dx from the records kan_bwd_tc_prep left in `recs` (features [0, d_in) of the pointers given;
// dx rows have stride ld).
static int dx_tc_launch(const float* C, const float* scale, const float* gy, float* dx, const unsigned char* recs,
                        int B, int d_in, int d_out, int G, int nch, int ld, const KanGrid& grid, cudaStream_t st,
                        const int32_t* seg = nullptr) {
  const DxSmem L = dx_smem_layout(G);
  const int n_fg = (d_in + kDxF - 1) / kDxF;
  // band 32: at the full cfg3 batch (B = 65536, 256 chunks) wider bands are faster but re-read C'
  // from DRAM more often — dx 1.128 s / 172 GB at band 8, 1.112 s / 201 GB at 16, 1.103 s / 294 GB
  // at 32, 1.094 s / 993 GB at 128 (ncu, profiles/r02/dx_band_sweep.txt); 32 keeps most of the
  // gain at 1.7x the traffic.  16 warps x 12 tasks measured faster than 32 x 6 (64 registers spill)
  static const int band_env = getenv("UKAN_DX_BAND") ? atoi(getenv("UKAN_DX_BAND")) : 32;
  static const int warps_env = getenv("UKAN_DX_WARPS") ? atoi(getenv("UKAN_DX_WARPS")) : 16;
  const int band = std::max(1, std::min(band_env, nch));
  const int64_t nblk = (int64_t)nch * n_fg;
  if (seg != nullptr) {
    auto kern = kan_dx_tc_kernel<16, 12, true>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<(unsigned)nblk, 16 * 32, L.total, st>>>(recs, C, scale, gy, dx, B, d_in, d_out, G, nch, n_fg, band, ld,
                                                   grid.inv_dg, make_basis<4>(3), seg);
  } else if (warps_env == 16) {
    auto kern = kan_dx_tc_kernel<16, 12>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<(unsigned)nblk, 16 * 32, L.total, st>>>(recs, C, scale, gy, dx, B, d_in, d_out, G, nch, n_fg, band, ld,
                                                   grid.inv_dg, make_basis<4>(3), seg);
  } else {
    auto kern = kan_dx_tc_kernel<32, 6>;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<(unsigned)nblk, 32 * 32, L.total, st>>>(recs, C, scale, gy, dx, B, d_in, d_out, G, nch, n_fg, band, ld,
                                                   grid.inv_dg, make_basis<4>(3), seg);
  }
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

int kan_dx_tc_run(const float* C, const float* scale, const float* gy, float* dx, void* workspace, int B, int d_in,
                  int d_out, int G, const KanGrid& grid, const TcPlan& p, cudaStream_t st) {
  return dx_tc_launch(C, scale, gy, dx, reinterpret_cast<const unsigned char*>(workspace), B, d_in, d_out, G, p.nch,
                      d_in, grid, st);
}

// One part of the backward over features [i_lo, i_hi), from records prepared for the WHOLE layer
// (kan_bwd_tc_prep on the same workspace): what & 1 = table gradient (dC, dscale of those
// features), what & 2 = dx of those features.  Lets a data-parallel caller all-reduce finished
// feature slices of dC while later slices are still being computed.
int kan_bwd_tc_part(const float* C, const float* scale, const float* gy, float* dx, float* dC, float* dscale,
                    void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int G, const KanGrid& grid,
                    int64_t i_lo, int64_t i_hi, int what, cudaStream_t st) {
  const TcPlan full = kan_bwd_tc_plan(B, d_in, d_out, G, 3, false);
  if (!full.ok || workspace == nullptr || ws_bytes < kan_bwd_tc_workspace(full)) return UKAN_E_WORKSPACE;
  if (i_lo < 0 || i_hi > d_in || i_lo >= i_hi) return UKAN_E_ARG;
  const int n = (int)(i_hi - i_lo), R = G + 3;
  unsigned char* base = reinterpret_cast<unsigned char*>(workspace);
  const unsigned char* recs = base + (size_t)i_lo * full.nch * tc_rec_bytes(G);
  if (what & 1) {
    if (!dC || !dscale) return UKAN_E_ARG;
    TcPlan p = kan_bwd_tc_plan(B, n, d_out, G, 3, false);
    double* part = reinterpret_cast<double*>(base + ((full.rec_bytes + 255) / 256) * 256);
    if (p.S > 1 && p.part_bytes > full.part_bytes) {  // the slice's split-K partials must fit the workspace
      p.S = 1;
      p.cps = p.nch;
      p.part_bytes = 0;
    }
    const int rc = tc_sweep_dispatch(C + (size_t)i_lo * R * d_out, scale + (size_t)i_lo * d_out, gy,
                                     dC + (size_t)i_lo * R * d_out, dscale + (size_t)i_lo * d_out,
                                     const_cast<unsigned char*>(recs), part, B, n, d_out, G, p, st);
    if (rc) return rc;
  }
  if (what & 2) {
    if (!dx) return UKAN_E_ARG;
    if (!kan_dx_tc_applicable(full, C, gy, d_out, G)) return UKAN_E_ARG;
    return dx_tc_launch(C + (size_t)i_lo * R * d_out, scale + (size_t)i_lo * d_out, gy, dx + i_lo, recs, B, n, d_out,
                        G, full.nch, d_in, grid, st);
  }
  return UKAN_OK;
}

// ---------------------------------------------------------------------------------------
// Dense UKAN layers on the KAN tensor-core backward (round 2).  When every feature's virtual
// table has <= 67 rows (cfg5: <= 32), a 256-sample chunk piles up on a few dozen rows, exactly the
// regime of the banded DMMA sweep and dx above; the UKAN table is then "a KAN table whose feature
// i owns rows [4 seg[i], 4 seg[i+1])".  Records: kan_bwd_tc_prep_kernel<true> (cell = window start
// inside the segment, UKAN u); table gradient: the tc3 sweep writing dT rows of the segment;
// dx: kan_dx_tc_kernel staging C' from the segment.  Replaces the sorted-merge sweep
// (seg_fsweep) and the per-pair dx (spline_dx64) for those layers, layers.py:254-291.
// Segments of <= 16 rows (4 row blocks) take the sample-split sweep (SS), larger ones the
// block-split tc3 sweep over >= 17 cells (two or four 4-block warps per feature).
bool ukan_dense_ss(int64_t max_rows) {
  static const bool off = getenv("UKAN_DENSE_SS") && getenv("UKAN_DENSE_SS")[0] == '0';  // A/B only
  return !off && max_rows <= 16;
}
static int ukan_dense_G(int64_t max_rows) {
  return ukan_dense_ss(max_rows) ? (int)std::max<int64_t>(1, max_rows - 3) : (int)std::max<int64_t>(17, max_rows - 3);
}

int64_t ukan_dense_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t max_rows, int k) {
  static const bool off = getenv("UKAN_UKAN_DENSE") && getenv("UKAN_UKAN_DENSE")[0] == '0';  // A/B only
  if (off || k != 3 || B < 1 || max_rows < 1 || max_rows > 67 || d_out < 64 || d_out % 4 || !tc3_enabled()) return 0;
  const TcPlan p = kan_bwd_tc_plan(B, d_in, d_out, ukan_dense_G(max_rows), 3, false);
  if (!p.ok) return 0;
  if (ukan_dense_ss(max_rows) ? p.rb != 4 : (!p.split || p.wpf != 4)) return 0;
  return kan_bwd_tc_workspace(p);  // records + split-K partials (padded [d_in][G+3] rows)
}

int ukan_dense_backward(const float* x, const int32_t* base_row, const int32_t* seg, const float* T,
                        const float* scale, const float* gy, float* dx, float* dT, float* dscale, int B, int d_in,
                        int d_out, int64_t max_rows, double delta_g, void* ws, int64_t ws_bytes, cudaStream_t st,
                        bool table) {
  const int64_t need = ukan_dense_workspace(B, d_in, d_out, max_rows, 3);
  if (need <= 0 || ws == nullptr || ws_bytes < need) return UKAN_E_WORKSPACE;
  const int G = ukan_dense_G(max_rows);
  const TcPlan p = kan_bwd_tc_plan(B, d_in, d_out, G, 3, false);
  unsigned char* recs = static_cast<unsigned char*>(ws);
  double* part = reinterpret_cast<double*>(recs + ((p.rec_bytes + 255) / 256) * 256);
  KanGrid grid{};
  grid.inv_dg = 1.0 / delta_g;
  grid.G = G;
  if (!table && dx == nullptr) return UKAN_OK;  // the caller computed dT / dscale; no dx wanted
  dim3 pg((d_in + 7) / 8, p.nch);
  kan_bwd_tc_prep_kernel<true><<<pg, 256, 0, st>>>(x, recs, B, d_in, p.nch, G, grid, base_row, seg, grid.inv_dg);
  UKAN_LAUNCH_CHECK();
  if (table) {  // else the caller computed dT / dscale (sorted-merge sweep)
    CUtensorMap map;
    if (!((uintptr_t)gy % 16 == 0 && tc3_tensor_map(&map, gy, B, d_out))) return UKAN_E_ARG;
    int rc = UKAN_E_ARG;
    if (ukan_dense_ss(max_rows)) {
      TcPlan q = p;  // one chunk range per CTA: the SS epilogue writes the rows directly
      q.S = 1;
      q.cps = q.nch;
      rc = tc3_launch<4, 4, 4, 4, true>(map, T, scale, dT, dscale, recs, nullptr, B, d_in, d_out, G, q, st, seg);
    } else if (p.rb == 16 && p.nt == 4)
      rc = tc3_launch<16, 4, 4, 4>(map, T, scale, dT, dscale, recs, part, B, d_in, d_out, G, p, st, seg);
    else if (p.rb == 8 && p.nt == 8)
      rc = tc3_launch<8, 8, 4, 4>(map, T, scale, dT, dscale, recs, part, B, d_in, d_out, G, p, st, seg);
    if (rc) return rc;
  }
  if (dx) {
    if (((uintptr_t)T % 16) != 0) return UKAN_E_ARG;
    return dx_tc_launch(T, scale, gy, dx, recs, B, d_in, d_out, G, p.nch, d_in, grid, st, seg);
  }
  return UKAN_OK;
}

}  // namespace ukan
