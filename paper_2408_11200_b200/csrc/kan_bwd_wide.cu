// kan_bwd_wide.cu — KAN backward (table side) for fine grids: cost independent of G.
//
// Replaces the bwd closures of span_gather (layers.py:67-70, the np.add.at scatter of the window
// gradient), edge_combine (84-88) and the base branch (layers.py:310-316) when the grid is too
// fine for the register / tensor-core sweeps (kan_bwd.cu, kan_bwd_tc.cu: G <= ~64), which is the
// regime of the paper's grid-size benchmark (bench.py:76-96, G up to thousands):
//   A[i,r,o] = sum_{(b,j): cell_bi + j = r} w_j(u_bi) * g[b,o]     (fp64)
//   dC = scale * A,   dscale = sum_r C * A,   dbw = sum_b silu(x) * g.
// Every sample touches K of the R = G + k rows, so the work is O(B * d_in * K * d_out) plus the
// unavoidable R * d_in * d_out writes of dC — flat in G, like the matrix-form forward.
//
//  * prep: one warp per (feature, 256-sample chunk): fp64 locate (layers.py:299-300), a rank sort
//    of the chunk by key (cell << 8 | sample) (keys are unique -> stable, deterministic), and the
//    start of every 32-row tile in the sorted chunk.  Records stay L2-resident.
//  * sweep: one warp per (feature, 32-row tile, 32-output slice), lane = output.  For each chunk
//    it walks only the samples whose window meets its tile (cells [r0-k, r0+31]), evaluates the
//    basis weights lane-parallel (one sample per lane), then runs the samples in sorted order,
//    keeping the window of the current cell in K registers and flushing it into a 32x32 fp64
//    shared-memory tile when the cell changes.  dC and the tile's dscale partial are written
//    once at the end; a second kernel sums the dscale partials over tiles in fixed order.
// Deterministic: fixed chunk order, cell-then-sample order inside a chunk, fixed reductions.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "rowmap.cuh"

namespace ukan {

constexpr int kWdBC = 256;       // samples per chunk (sample index packed in 8 bits)
constexpr int kWdRT = 32;        // rows per tile
constexpr int kWdMaxTiles = 1024;
constexpr int kWdBadCell = (1 << 23) - 1;  // > any valid cell (check_kan_args: G + k < 2^23)

struct WidePlan {
  bool ok = false;
  int n_rt = 0, n_os = 0, nch = 0, st_n = 0;
  size_t recb = 0;
  int64_t rec_bytes = 0, part_bytes = 0;
};

// record layout per (feature, chunk), 16-B aligned: key[256] int | u[256] double | st[st_n] int
__host__ __device__ constexpr int wide_warp_doubles(int K) { return kWdRT * 32 + 32 * K + 32; }

static size_t wide_rec_bytes(int st_n) { return (size_t)kWdBC * 12 + (size_t)st_n * 4; }

__global__ void __launch_bounds__(256)
kan_bwd_wide_prep_kernel(const float* __restrict__ x, unsigned char* __restrict__ recs, int B, int d_in, int nch,
                         int n_rt, int st_n, size_t recb, KanGrid grid) {
  __shared__ float xs[kWdBC][9];
  __shared__ __align__(16) int keys[8][kWdBC];
  __shared__ int sorted[8][kWdBC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * 8, n = blockIdx.y;
  const int b0 = n * kWdBC;
  const int nb = min(kWdBC, B - b0);
  for (int t = threadIdx.x; t < kWdBC * 8; t += blockDim.x) {
    const int s = t / 8, f = t % 8;
    xs[s][f] = (s < nb && i0 + f < d_in) ? x[(size_t)(b0 + s) * d_in + i0 + f] : 0.f;
  }
  __syncthreads();
  const int i = i0 + warp;
  if (i >= d_in) return;
  unsigned char* rec = recs + ((size_t)i * nch + n) * recb;
  int* ent = reinterpret_cast<int*>(rec);
  double* uu = reinterpret_cast<double*>(rec + kWdBC * 4);
  int* st = reinterpret_cast<int*>(rec + kWdBC * 12);
  constexpr int PER = kWdBC / 32;
  int key[PER];
  double us[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int s = q * 32 + lane;
    int cell = kWdBadCell;
    double u = 0.0;
    bool mask;
    if (s < nb && !kan_locate(xs[s][warp], grid, cell, u, mask)) cell = kWdBadCell;  // NaN: no contribution
    key[q] = (cell << 8) | s;
    us[q] = u;
    keys[warp][s] = key[q];
  }
  __syncwarp();
  int rank[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) rank[q] = 0;
  const int4* k4 = reinterpret_cast<const int4*>(keys[warp]);
  for (int m = 0; m < kWdBC / 4; ++m) {
    const int4 v = k4[m];
#pragma unroll
    for (int q = 0; q < PER; ++q)
      rank[q] += (v.x < key[q]) + (v.y < key[q]) + (v.z < key[q]) + (v.w < key[q]);
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    sorted[warp][rank[q]] = key[q];
    ent[rank[q]] = key[q];
    uu[rank[q]] = us[q];
  }
  __syncwarp();
  // st[t] = number of keys with cell < 32 t  (t = 0 .. n_rt), lower bound by binary search
  for (int t = lane; t < st_n; t += 32) {
    const int tt = min(t, n_rt);
    const int kk = (tt * kWdRT) << 8;
    int lo = 0, hi = kWdBC;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sorted[warp][mid] < kk) lo = mid + 1;
      else hi = mid;
    }
    st[t] = lo;
  }
}

template <int K>
__global__ void __launch_bounds__(256)
kan_bwd_wide_sweep_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ C,
                          const float* __restrict__ scale, const float* __restrict__ gy, float* __restrict__ dC,
                          double* __restrict__ part, int d_in, int d_out, int R, int n_rt, int n_os, int nch,
                          size_t recb, Basis<K> bas) {
  extern __shared__ __align__(16) double wsm[];  // per warp: A[32][32] | wb[32][K] | cb[32] bb[32] (int)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double (*A)[32] = reinterpret_cast<double (*)[32]>(wsm + (size_t)warp * wide_warp_doubles(K));
  double (*wb)[K] = reinterpret_cast<double (*)[K]>(&A[kWdRT][0]);
  int* cb = reinterpret_cast<int*>(&wb[32][0]);
  int* bb = cb + 32;
  const int64_t unit = (int64_t)blockIdx.x * 8 + warp;
  if (unit >= (int64_t)d_in * n_rt * n_os) return;
  const int t = (int)(unit % n_rt);
  const int64_t rest = unit / n_rt;
  const int os = (int)(rest % n_os);
  const int i = (int)(rest / n_os);
  const int o = os * 32 + lane;
  const bool live = o < d_out;
  const int r0 = t * kWdRT;
  const int lo_cell = r0 - (K - 1);
#pragma unroll 4
  for (int r = 0; r < kWdRT; ++r) A[r][lane] = 0.0;

  double acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  int cur = INT_MIN;
  auto flush = [&]() {
    if (cur != INT_MIN) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int r = cur + j - r0;
        if (r >= 0 && r < kWdRT) A[r][lane] += acc[j];
        acc[j] = 0.0;
      }
    }
  };

  for (int c = 0; c < nch; ++c) {
    const unsigned char* rec = recs + ((size_t)i * nch + c) * recb;
    const int* ent = reinterpret_cast<const int*>(rec);
    const double* uu = reinterpret_cast<const double*>(rec + kWdBC * 4);
    const int* st = reinterpret_cast<const int*>(rec + kWdBC * 12);
    int lo = __ldg(st + t);
    const int hi = __ldg(st + t + 1);
    // extend backwards over the cells r0-k .. r0-1 whose windows reach into this tile
    while (lo > 0) {
      const int idx = lo - 32 + lane;
      const bool ok = idx >= 0 && (__ldg(ent + idx) >> 8) >= lo_cell;
      const int nk = __popc(__ballot_sync(0xffffffffu, ok));
      lo -= nk;
      if (nk < 32) break;
    }
    for (int p0 = lo; p0 < hi; p0 += 32) {
      const int p = p0 + lane;
      if (p < hi) {
        const int key = __ldg(ent + p);
        double w[K];
        basis_weights<K>(bas, __ldg(uu + p), w);
#pragma unroll
        for (int j = 0; j < K; ++j) wb[lane][j] = w[j];
        cb[lane] = key >> 8;
        bb[lane] = c * kWdBC + (key & 255);
      }
      __syncwarp();
      const int ns = min(32, hi - p0);
      const float* gyo = gy + (live ? o : 0);
      for (int q0 = 0; q0 < ns; q0 += 16) {
        const int nq = min(16, ns - q0);
        unsigned gv[16];  // 16 independent gathers in flight
#pragma unroll
        for (int q = 0; q < 16; ++q)
          gv[q] = (q < nq && live) ? __float_as_uint(__ldg(gyo + (size_t)bb[q0 + q] * d_out)) : 0u;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (q < nq) {
            const int cell = cb[q0 + q];
            if (cell != cur) {
              flush();
              cur = cell;
            }
            const double g = (double)__uint_as_float(gv[q]);
#pragma unroll
            for (int j = 0; j < K; ++j) acc[j] = fma(wb[q0 + q][j], g, acc[j]);
          }
        }
      }
      __syncwarp();
    }
  }
  flush();
  __syncwarp();
  double prod = 0.0;
  if (live) {
    const double sc = (double)__ldg(scale + (size_t)i * d_out + o);
    for (int r = 0; r < kWdRT; ++r) {
      const int row = r0 + r;
      if (row >= R) break;
      const double a = A[r][lane];
      const size_t ci = ((size_t)i * R + row) * d_out + o;
      dC[ci] = (float)(sc * a);
      prod = fma((double)__ldg(C + ci), a, prod);
    }
    part[((size_t)i * n_rt + t) * d_out + o] = prod;
  }
}

// dscale[i,o] = sum_t part[i][t][o]  (fixed tile order)
__global__ void kan_bwd_wide_reduce_kernel(const double* __restrict__ part, float* __restrict__ dscale, int d_in,
                                           int d_out, int n_rt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)d_in * d_out) return;
  const int i = (int)(e / d_out), o = (int)(e % d_out);
  double a = 0.0;
  for (int t = 0; t < n_rt; ++t) a += part[((size_t)i * n_rt + t) * d_out + o];
  dscale[e] = (float)a;
}

// dbw[i,o] = sum_b silu(x[b,i]) g[b,o]  (fp64, sample order).  Warp = feature, lane = output;
// the 8 warps of a CTA share g rows through L1.
__global__ void __launch_bounds__(256)
kan_dbase_kernel(const float* __restrict__ x, const float* __restrict__ gy, float* __restrict__ dbw, int B,
                 int d_in, int d_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + warp, o = blockIdx.y * 32 + lane;
  if (i >= d_in) return;
  double a = 0.0;
  for (int b0 = 0; b0 < B; b0 += 32) {
    const int b = b0 + lane;
    const double s = b < B ? silu_d((double)__ldg(x + (size_t)b * d_in + i)) : 0.0;
    const int nb = min(32, B - b0);
    for (int q = 0; q < nb; ++q) {
      const double sq = __shfl_sync(0xffffffffu, s, q);
      if (o < d_out) a = fma(sq, (double)__ldg(gy + (size_t)(b0 + q) * d_out + o), a);
    }
  }
  if (o < d_out) dbw[(size_t)i * d_out + o] = (float)a;
}

WidePlan kan_bwd_wide_plan(int64_t B, int64_t d_in, int64_t d_out, int R, int K) {
  WidePlan p;
  if (B < 1 || K < 1 || K > kMaxK) return p;
  p.n_rt = (R + kWdRT - 1) / kWdRT;
  if (p.n_rt > kWdMaxTiles) return p;
  p.n_os = (int)((d_out + 31) / 32);
  p.nch = (int)((B + kWdBC - 1) / kWdBC);
  p.st_n = ((p.n_rt + 1 + 3) / 4) * 4;
  p.recb = wide_rec_bytes(p.st_n);
  p.rec_bytes = (int64_t)d_in * p.nch * (int64_t)p.recb;
  p.part_bytes = (int64_t)sizeof(double) * d_in * p.n_rt * d_out;
  p.ok = true;
  return p;
}

int64_t kan_bwd_wide_workspace(const WidePlan& p) {
  return p.ok ? ((p.rec_bytes + 255) / 256) * 256 + p.part_bytes : 0;
}

template <int K>
int kan_bwd_wide_run(const float* x, const float* C, const float* scale, const float* gy, float* dC, float* dscale,
                     float* dbw, void* workspace, int64_t ws_bytes, int B, int d_in, int d_out, int R,
                     const KanGrid& grid, const WidePlan& p, cudaStream_t st) {
  if (!p.ok || workspace == nullptr || ws_bytes < kan_bwd_wide_workspace(p)) return UKAN_E_WORKSPACE;
  unsigned char* recs = reinterpret_cast<unsigned char*>(workspace);
  double* part = reinterpret_cast<double*>(recs + ((p.rec_bytes + 255) / 256) * 256);
  kan_bwd_wide_prep_kernel<<<dim3((d_in + 7) / 8, p.nch), 256, 0, st>>>(x, recs, B, d_in, p.nch, p.n_rt, p.st_n,
                                                                         p.recb, grid);
  UKAN_LAUNCH_CHECK();
  const int64_t units = (int64_t)d_in * p.n_rt * p.n_os;
  const size_t smem = sizeof(double) * 8 * (size_t)wide_warp_doubles(K);
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kan_bwd_wide_sweep_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kan_bwd_wide_sweep_kernel<K><<<(unsigned)((units + 7) / 8), 256, smem, st>>>(
      recs, C, scale, gy, dC, part, d_in, d_out, R, p.n_rt, p.n_os, p.nch, p.recb, make_basis<K>(K - 1));
  UKAN_LAUNCH_CHECK();
  const int64_t n = (int64_t)d_in * d_out;
  kan_bwd_wide_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, dscale, d_in, d_out, p.n_rt);
  UKAN_LAUNCH_CHECK();
  if (dbw) {
    kan_dbase_kernel<<<dim3((d_in + 7) / 8, (d_out + 31) / 32), 256, 0, st>>>(x, gy, dbw, B, d_in, d_out);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

#define UKAN_WIDE_INST(K)                                                                                     \
  template int kan_bwd_wide_run<K>(const float*, const float*, const float*, const float*, float*, float*,   \
                                   float*, void*, int64_t, int, int, int, int, const KanGrid&, const WidePlan&, \
                                   cudaStream_t);
UKAN_WIDE_INST(1) UKAN_WIDE_INST(2) UKAN_WIDE_INST(3) UKAN_WIDE_INST(4) UKAN_WIDE_INST(5) UKAN_WIDE_INST(6)
UKAN_WIDE_INST(7) UKAN_WIDE_INST(8) UKAN_WIDE_INST(9) UKAN_WIDE_INST(10) UKAN_WIDE_INST(11)

// ---------------------------------------------------------------------------------------
// Segmented variant for data-dependent per-feature row segments (UKAN's generated table,
// layers.py:254-291: feature f owns rows [seg_start[f]*K, seg_start[f+1]*K) of the [n_u*K, d_out]
// table, a window is base_row + 0..k).  Same records (256-sample chunks sorted by local row),
// but the tiles are per-feature 32-row tiles enumerated by a prefix over the segment lengths,
// and a CTA of W warps (32*W outputs) shares one tile's sample staging: the chunk bounds are
// found by counting keys (no per-tile index), basis weights evaluated once per CTA.
template <bool UKAN>
__global__ void __launch_bounds__(256)
seg_prep_kernel(const float* __restrict__ x, unsigned char* __restrict__ recs, int B, int d_in, int nch,
                RowMap rm) {
  __shared__ float xs[kWdBC][9];
  __shared__ __align__(16) int keys[8][kWdBC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = blockIdx.x * 8, n = blockIdx.y;
  const int b0 = n * kWdBC;
  const int nb = min(kWdBC, B - b0);
  for (int t = threadIdx.x; t < kWdBC * 8; t += blockDim.x) {
    const int s = t / 8, f = t % 8;
    xs[s][f] = (s < nb && i0 + f < d_in) ? x[(size_t)(b0 + s) * d_in + i0 + f] : 0.f;
  }
  __syncthreads();
  const int i = i0 + warp;
  if (i >= d_in) return;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  unsigned char* rec = recs + ((size_t)i * nch + n) * (kWdBC * 12);
  int* ent = reinterpret_cast<int*>(rec);
  double* uu = reinterpret_cast<double*>(rec + kWdBC * 4);
  constexpr int PER = kWdBC / 32;
  int key[PER];
  double us[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int s = q * 32 + lane;
    int local = kWdBadCell;
    double u = 0.0;
    if (s < nb) {
      int row;
      bool mask;
      if (locate_row<UKAN>(rm, xs[s][warp], (int64_t)(b0 + s), i, d_in, row, u, mask)) local = row - row0;
    }
    key[q] = (local << 8) | s;
    us[q] = u;
    keys[warp][s] = key[q];
  }
  __syncwarp();
  int rank[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) rank[q] = 0;
  const int4* k4 = reinterpret_cast<const int4*>(keys[warp]);
  for (int m = 0; m < kWdBC / 4; ++m) {
    const int4 v = k4[m];
#pragma unroll
    for (int q = 0; q < PER; ++q)
      rank[q] += (v.x < key[q]) + (v.y < key[q]) + (v.z < key[q]) + (v.w < key[q]);
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    ent[rank[q]] = key[q];
    uu[rank[q]] = us[q];
  }
}

// tile_start[f] = sum_{f' < f} ceil(rows(f') / 32)   (one warp, 32 features per step)
template <bool UKAN>
__global__ void seg_tiles_kernel(RowMap rm, int d_in, int* __restrict__ tile_start) {
  const int lane = threadIdx.x;
  int carry = 0;
  for (int f0 = 0; f0 <= d_in; f0 += 32) {
    const int f = f0 + lane;
    int v = 0;
    if (f < d_in) {
      int row0, nrows;
      feature_rows<UKAN>(rm, f, row0, nrows);
      v = (nrows + kWdRT - 1) / kWdRT;
    }
    int inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += t;
    }
    if (f <= d_in) tile_start[f] = carry + inc - v;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
}

constexpr int kSegSB = 256;     // samples staged per batch
constexpr int kSegMaxCh = 512;  // chunks (B <= 131072)
constexpr int kSegGB = 16;      // samples per g stage (cp.async double buffer)

template <int K>
__host__ __device__ constexpr size_t seg_smem_bytes(int W) {
  return sizeof(double) * ((size_t)W * kWdRT * 32 + (size_t)kSegSB * K) + sizeof(float) * 2 * kSegGB * 32 * W +
         sizeof(int) * (2 * kSegSB + 3 * kSegMaxCh + 8);
}

template <int K, bool UKAN>
__global__ void __launch_bounds__(256)
seg_sweep_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ T, const float* __restrict__ scale,
                 const float* __restrict__ gy, float* __restrict__ dT, double* __restrict__ part,
                 const int* __restrict__ tile_start, int d_in, int d_out, int nch, int n_og, RowMap rm,
                 Basis<K> bas) {
  extern __shared__ __align__(16) double ssm[];
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double (*A)[32] = reinterpret_cast<double (*)[32]>(ssm + (size_t)warp * kWdRT * 32);
  double (*wb)[K] = reinterpret_cast<double (*)[K]>(ssm + (size_t)W * kWdRT * 32);
  int* cb = reinterpret_cast<int*>(ssm + (size_t)W * kWdRT * 32 + (size_t)kSegSB * K);
  int* bb = cb + kSegSB;
  int* c_lo = bb + kSegSB;       // [nch] first sorted position of the tile's samples in chunk c
  int* c_off = c_lo + kSegMaxCh;  // [nch + 1] exclusive prefix of the per-chunk counts
  float* gs = reinterpret_cast<float*>(c_off + 2 * kSegMaxCh + 8);  // [2][kSegGB][32*W] g rows of a stage
  const int64_t blk = blockIdx.x;
  const int og = (int)(blk % n_og);
  const int tt = (int)(blk / n_og);
  if (tt >= tile_start[d_in]) return;
  int lo_f = 0, hi_f = d_in - 1;  // feature: largest f with tile_start[f] <= tt
  while (lo_f < hi_f) {
    const int mid = (lo_f + hi_f + 1) >> 1;
    if (tile_start[mid] <= tt) lo_f = mid;
    else hi_f = mid - 1;
  }
  const int i = lo_f;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  const int r0 = (tt - tile_start[i]) * kWdRT;
  const int lo_key = max(0, r0 - (K - 1)) << 8, hi_key = (r0 + kWdRT) << 8;
  const int o = (og * W + warp) * 32 + lane;
  const bool live = o < d_out;
  // 1. the tile's sample range in every sorted chunk (warp per chunk, keys counted lane-parallel)
  for (int c = warp; c < nch; c += W) {
    const int4* e4 = reinterpret_cast<const int4*>(recs + ((size_t)i * nch + c) * (kWdBC * 12)) + lane * 2;
    const int4 ka = __ldg(e4), kb = __ldg(e4 + 1);
    int nlo = (ka.x < lo_key) + (ka.y < lo_key) + (ka.z < lo_key) + (ka.w < lo_key) + (kb.x < lo_key) +
              (kb.y < lo_key) + (kb.z < lo_key) + (kb.w < lo_key);
    int nhi = (ka.x < hi_key) + (ka.y < hi_key) + (ka.z < hi_key) + (ka.w < hi_key) + (kb.x < hi_key) +
              (kb.y < hi_key) + (kb.z < hi_key) + (kb.w < hi_key);
    nlo = __reduce_add_sync(0xffffffffu, nlo);
    nhi = __reduce_add_sync(0xffffffffu, nhi);
    if (lane == 0) {
      c_lo[c] = nlo;
      c_off[c + 1] = nhi - nlo;
    }
  }
#pragma unroll 4
  for (int r = 0; r < kWdRT; ++r) A[r][lane] = 0.0;
  __syncthreads();
  if (warp == 0) {  // inclusive scan of the counts (chunk order = sample order)
    int carry = 0;
    for (int c0 = 0; c0 < nch; c0 += 32) {
      const int c = c0 + lane;
      int v = c < nch ? c_off[c + 1] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += t;
      }
      if (c < nch) c_off[c + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) c_off[0] = 0;
  }
  __syncthreads();
  const int N = c_off[nch];
  double acc[K];
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0.0;
  int cur = INT_MIN;
  auto flush = [&]() {
    if (cur != INT_MIN) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int r = cur + j - r0;
        if (r >= 0 && r < kWdRT) A[r][lane] += acc[j];
        acc[j] = 0.0;
      }
    }
  };
  // 2. stage the tile's samples (chunk order, sorted inside a chunk) in batches, then sweep them
  for (int s0 = 0; s0 < N; s0 += kSegSB) {
    const int nb = min(kSegSB, N - s0);
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int gq = s0 + q;
      int lo = 0, hi = nch - 1;  // chunk: largest c with c_off[c] <= gq
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (c_off[mid] <= gq) lo = mid;
        else hi = mid - 1;
      }
      const int c = lo;
      const int p = c_lo[c] + (gq - c_off[c]);
      const unsigned char* rec = recs + ((size_t)i * nch + c) * (kWdBC * 12);
      const int key = __ldg(reinterpret_cast<const int*>(rec) + p);
      double w[K];
      basis_weights<K>(bas, __ldg(reinterpret_cast<const double*>(rec + kWdBC * 4) + p), w);
#pragma unroll
      for (int j = 0; j < K; ++j) wb[q][j] = w[j];
      cb[q] = key >> 8;
      bb[q] = (c * kWdBC + (key & 255)) * d_out;  // element offset of the sample's g row
    }
    __syncthreads();
    // g rows of the staged samples: coalesced cp.async of [kSegGB samples][32*W outputs], double
    // buffered so the next stage is in flight while this one is swept
    const int OW = 32 * W, o_base = og * OW;
    const int n_st = (nb + kSegGB - 1) / kSegGB;
    auto stage_g = [&](int stg) {
      float* dst = gs + (size_t)(stg & 1) * kSegGB * OW;
      const int q0 = stg * kSegGB;
      const int nq = min(kSegGB, nb - q0);
      if ((d_out & 3) == 0) {
        const int v4 = OW / 4;
        for (int t = threadIdx.x; t < kSegGB * v4; t += blockDim.x) {
          const int q = t / v4, oc = (t % v4) * 4;
          const int oo = o_base + oc;
          const int bytes = q < nq ? max(0, min(4, d_out - oo)) * 4 : 0;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + q * OW + oc);
          const float* src = bytes ? gy + (size_t)(unsigned)bb[q0 + q] + oo : gy;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(bytes));
        }
      } else {
        for (int t = threadIdx.x; t < kSegGB * OW; t += blockDim.x) {
          const int q = t / OW, oc = t % OW;
          const int oo = o_base + oc;
          const bool ok = q < nq && oo < d_out;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + q * OW + oc);
          const float* src = ok ? gy + (size_t)(unsigned)bb[q0 + q] + oo : gy;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 4 : 0));
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };
    stage_g(0);
    for (int stg = 0; stg < n_st; ++stg) {
      if (stg + 1 < n_st) {
        stage_g(stg + 1);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();
      const float* gq = gs + (size_t)(stg & 1) * kSegGB * OW + warp * 32 + lane;
      const int q0 = stg * kSegGB;
      const int nq = min(kSegGB, nb - q0);
      for (int q = 0; q < nq; ++q) {
        const int cell = cb[q0 + q];
        if (cell != cur) {
          if (cell > cur && cell - cur < K && cur != INT_MIN) {
            // sorted run advances: slide the K-row register window, retiring one row per step
            do {
              const int r = cur - r0;
              if (r >= 0 && r < kWdRT) A[r][lane] += acc[0];
#pragma unroll
              for (int j = 0; j + 1 < K; ++j) acc[j] = acc[j + 1];
              acc[K - 1] = 0.0;
            } while (++cur < cell);
          } else {
            flush();
            cur = cell;
          }
        }
        const double g = (double)gq[q * OW];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fma(wb[q0 + q][j], g, acc[j]);
      }
      __syncthreads();  // stage buffer (stg & 1) is refilled by the next iteration's stage_g
    }
  }
  flush();
  __syncwarp();
  if (live) {
    const double sc = (double)__ldg(scale + (size_t)i * d_out + o);
    double prod = 0.0;
    for (int r = 0; r < kWdRT && r0 + r < nrows; ++r) {
      const double a = A[r][lane];
      const size_t ci = (size_t)(row0 + r0 + r) * d_out + o;
      dT[ci] = (float)(sc * a);
      prod = fma((double)__ldg(T + ci), a, prod);
    }
    part[(size_t)tt * d_out + o] = prod;
  }
}

// seg_dmma (cubic splines): the same tiles on the FP64 tensor cores.  A batch of the tile's samples
// is counting-sorted by cell (stable), cells are grouped in 4-cell blocks whose windows span 8 rows
// (stride 4, as kan_bwd_tc.cu), and four samples of a block form the k=4 operand of one
// mma.sync.m8n8k4.f64 per 8 outputs.  A warp owns 64 outputs and keeps only the current block's
// 8x64 accumulators: when it moves to the next block the lower 4 rows are complete (retired into an
// fp64 shared tile) and the upper 4 rows become the next block's lower rows (one shuffle).
constexpr int kSdW = 4;            // warps per CTA
constexpr int kSdNT = 8;           // 8-output DMMA tiles per warp
constexpr int kSdOW = kSdW * 8 * kSdNT;  // outputs per CTA (256)
constexpr int kSdSB = 256;         // samples per batch
constexpr int kSdNC = 36;          // cells v = cell - r0 + 4 in [1, 35]; blocks of 4 -> 9

__host__ __device__ constexpr size_t segd_smem_bytes() {
  return sizeof(double) * ((size_t)kWdRT * kSdOW + (size_t)kSdSB * 4 * 2 + (size_t)kSdSB * 2) +
         sizeof(int) * (4 * kSdSB + 3 * kSegMaxCh + 2 * kSdNC + 16);
}

__device__ __forceinline__ void sd_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool UKAN>
__global__ void __launch_bounds__(32 * kSdW)
seg_dmma_kernel(const unsigned char* __restrict__ recs, const float* __restrict__ T, const float* __restrict__ scale,
                const float* __restrict__ gy, float* __restrict__ dT, double* __restrict__ part,
                const int* __restrict__ tile_start, int d_in, int d_out, int nch, int n_og, RowMap rm, Basis<4> bas) {
  extern __shared__ __align__(16) double sdm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  double* A = sdm;                                   // [32][kSdOW] fp64 tile accumulator
  double* w_st = A + (size_t)kWdRT * kSdOW;          // [SB][4] staging order
  double* w_so = w_st + (size_t)kSdSB * 4;           // [SB][4] cell order
  int* v_st = reinterpret_cast<int*>(w_so + (size_t)kSdSB * 4 + (size_t)kSdSB * 2);
  int* b_st = v_st + kSdSB;                          // g row offsets, staging order
  int* pos = b_st + kSdSB;
  int* b_so = pos + kSdSB;                           // g row offsets, cell order
  int* c_lo = b_so + kSdSB;                          // [nch]
  int* c_off = c_lo + kSegMaxCh;                     // [nch + 1]
  int* cst = c_off + 2 * kSegMaxCh;                  // [kSdNC + 1]
  const int64_t blk = blockIdx.x;
  const int og = (int)(blk % n_og);
  const int tt = (int)(blk / n_og);
  if (tt >= tile_start[d_in]) return;
  int lo_f = 0, hi_f = d_in - 1;
  while (lo_f < hi_f) {
    const int mid = (lo_f + hi_f + 1) >> 1;
    if (tile_start[mid] <= tt) lo_f = mid;
    else hi_f = mid - 1;
  }
  const int i = lo_f;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  const int r0 = (tt - tile_start[i]) * kWdRT;
  const int lo_key = max(0, r0 - 3) << 8, hi_key = (r0 + kWdRT) << 8;
  const int ob = og * kSdOW + warp * (8 * kSdNT);  // this warp's first output
  for (int c = warp; c < nch; c += kSdW) {
    const int4* e4 = reinterpret_cast<const int4*>(recs + ((size_t)i * nch + c) * (kWdBC * 12)) + lane * 2;
    const int4 ka = __ldg(e4), kb = __ldg(e4 + 1);
    int nlo = (ka.x < lo_key) + (ka.y < lo_key) + (ka.z < lo_key) + (ka.w < lo_key) + (kb.x < lo_key) +
              (kb.y < lo_key) + (kb.z < lo_key) + (kb.w < lo_key);
    int nhi = (ka.x < hi_key) + (ka.y < hi_key) + (ka.z < hi_key) + (ka.w < hi_key) + (kb.x < hi_key) +
              (kb.y < hi_key) + (kb.z < hi_key) + (kb.w < hi_key);
    nlo = __reduce_add_sync(0xffffffffu, nlo);
    nhi = __reduce_add_sync(0xffffffffu, nhi);
    if (lane == 0) {
      c_lo[c] = nlo;
      c_off[c + 1] = nhi - nlo;
    }
  }
  for (int t = threadIdx.x; t < kWdRT * kSdOW; t += blockDim.x) A[t] = 0.0;
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    for (int c0 = 0; c0 < nch; c0 += 32) {
      const int c = c0 + lane;
      int v = c < nch ? c_off[c + 1] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += t;
      }
      if (c < nch) c_off[c + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) c_off[0] = 0;
  }
  __syncthreads();
  const int N = c_off[nch];
  for (int s0 = 0; s0 < N; s0 += kSdSB) {
    const int nb = min(kSdSB, N - s0);
    // a. stage in chunk order: cell v, basis weights, g row offset
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int gq = s0 + q;
      int lo = 0, hi = nch - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (c_off[mid] <= gq) lo = mid;
        else hi = mid - 1;
      }
      const int c = lo;
      const int p = c_lo[c] + (gq - c_off[c]);
      const unsigned char* rec = recs + ((size_t)i * nch + c) * (kWdBC * 12);
      const int key = __ldg(reinterpret_cast<const int*>(rec) + p);
      double w[4];
      basis_weights<4>(bas, __ldg(reinterpret_cast<const double*>(rec + kWdBC * 4) + p), w);
#pragma unroll
      for (int j = 0; j < 4; ++j) w_st[q * 4 + j] = w[j];
      v_st[q] = (key >> 8) - r0 + 4;
      b_st[q] = (c * kWdBC + (key & 255)) * d_out;
    }
    __syncthreads();
    // b. stable counting sort by cell (warps split the cells)
    for (int c = warp; c < kSdNC; c += kSdW) {
      int n = 0;
      for (int q0 = 0; q0 < nb; q0 += 32) {
        const int q = q0 + lane;
        n += __popc(__ballot_sync(0xffffffffu, q < nb && v_st[q] == c));
      }
      if (lane == 0) cst[c + 1] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      cst[0] = 0;
      for (int c = 0; c < kSdNC; ++c) cst[c + 1] += cst[c];
    }
    __syncthreads();
    for (int c = warp; c < kSdNC; c += kSdW) {
      int base = cst[c];
      for (int q0 = 0; q0 < nb; q0 += 32) {
        const int q = q0 + lane;
        const bool m = q < nb && v_st[q] == c;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        if (m) pos[q] = base + __popc(bal & ((1u << lane) - 1u));
        base += __popc(bal);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const int ps = pos[q];
#pragma unroll
      for (int j = 0; j < 4; ++j) w_so[ps * 4 + j] = w_st[q * 4 + j];
      b_so[ps] = b_st[q];
    }
    __syncthreads();
    // c. DMMA sweep block by block (cells 4b .. 4b+3 -> rows v = 4b .. 4b+7)
    double acc[kSdNT][2];
#pragma unroll
    for (int t = 0; t < kSdNT; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int bk = 0; bk < kSdNC / 4; ++bk) {
      const int e0 = cst[4 * bk], e1 = cst[4 * bk + 4];
#pragma unroll 2
      for (int kc = e0; kc < e1; kc += 4) {
        const int si = kc + kq;
        const bool vld = si < e1;
        const int sc = vld ? si : e0;
        int vs = 0;
        // the sample's cell: cst is monotone; recover v from the block-local cell boundaries
#pragma unroll
        for (int cc = 1; cc < 4; ++cc) vs += (sc >= cst[4 * bk + cc]) ? 1 : 0;
        const int jj = grp - vs;  // row offset inside the sample's window
        const double a = (vld && jj >= 0 && jj < 4) ? w_so[sc * 4 + (jj & 3)] : 0.0;
        const float* gr = gy + (size_t)(unsigned)b_so[sc] + ob + grp;
        double bf[kSdNT];
#pragma unroll
        for (int t = 0; t < kSdNT; ++t) {
          const int o = ob + t * 8 + grp;
          bf[t] = (vld && o < d_out) ? (double)__ldg(gr + t * 8) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < kSdNT; ++t) sd_dmma(acc[t][0], acc[t][1], a, bf[t]);
      }
      // retire rows v = 4bk .. 4bk+3 (tile rows 4bk-4 .. 4bk-1), slide the upper half down
      const int r = 4 * bk - 4 + grp;
      if (grp < 4 && r >= 0) {
#pragma unroll
        for (int t = 0; t < kSdNT; ++t) {
          double* a2 = A + (size_t)r * kSdOW + warp * (8 * kSdNT) + t * 8 + 2 * kq;
          a2[0] += acc[t][0];
          a2[1] += acc[t][1];
        }
      }
#pragma unroll
      for (int t = 0; t < kSdNT; ++t) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const double up = __shfl_xor_sync(0xffffffffu, acc[t][v], 16);
          acc[t][v] = grp < 4 ? up : 0.0;
        }
      }
    }
    // rows v = 36 .. 39 would be tile rows 32 .. 35: outside the tile, dropped
    __syncthreads();
  }
  // d. epilogue: dT = scale * A, dscale partial = sum_r T * A  (this warp's 64 outputs, 2 per lane)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int oc = warp * (8 * kSdNT) + h * 32 + lane;
    const int o = og * kSdOW + oc;
    if (o >= d_out) continue;
    const double scl = (double)__ldg(scale + (size_t)i * d_out + o);
    double prod = 0.0;
    for (int rr = 0; rr < kWdRT && r0 + rr < nrows; ++rr) {
      const double a = A[(size_t)rr * kSdOW + oc];
      const size_t ci = (size_t)(row0 + r0 + rr) * d_out + o;
      dT[ci] = (float)(scl * a);
      prod = fma((double)__ldg(T + ci), a, prod);
    }
    part[(size_t)tt * d_out + o] = prod;
  }
}

// seg_f*: one sorted pass per feature.  seg_fsort_kernel merges a feature's chunk records into one
// stable order by (row, chunk, sample) with a row histogram in shared memory; seg_fsweep_kernel
// then walks the feature's rows once in 4-cell blocks on the FP64 tensor cores with an 8-row
// register window (as seg_dmma), retiring every row exactly once straight into dT, and reduces
// dscale in registers — no per-tile staging, no fp64 tile in shared memory, no dscale partials.
constexpr int kFsMaxRows = 48 * 1024;  // per-feature rows the shared histogram holds

template <bool UKAN>
__global__ void __launch_bounds__(256)
seg_fsort_kernel(const unsigned char* __restrict__ recs, int nch, int d_in, RowMap rm, int* __restrict__ row_start,
                 int* __restrict__ sorted_b, double* __restrict__ sorted_u, int B) {
  extern __shared__ int cnt[];  // [nrows + 1] histogram -> starts -> cursors
  __shared__ int ks[kWdBC];
  const int i = blockIdx.x;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  int* rs = row_start + row0 + i;  // [nrows + 1]
  int* sb = sorted_b + (size_t)i * B;
  double* su = sorted_u + (size_t)i * B;
  for (int r = threadIdx.x; r <= nrows; r += blockDim.x) cnt[r] = 0;
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int* ent = reinterpret_cast<const int*>(recs + ((size_t)i * nch + c) * (kWdBC * 12));
    for (int p = threadIdx.x; p < kWdBC; p += blockDim.x) {
      const int row = __ldg(ent + p) >> 8;
      if (row < nrows) atomicAdd(&cnt[row], 1);  // padding / NaN keys carry a row beyond the segment
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan (one warp, 32 rows per step)
    const int lane = threadIdx.x;
    int carry = 0;
    for (int r0 = 0; r0 <= nrows; r0 += 32) {
      const int r = r0 + lane;
      const int v = r < nrows ? cnt[r] : 0;
      int inc = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += t;
      }
      if (r <= nrows) {
        cnt[r] = carry + inc - v;
        rs[r] = carry + inc - v;
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {  // chunks in sample order; inside a chunk keys are sorted by (row, sample)
    const unsigned char* rec = recs + ((size_t)i * nch + c) * (kWdBC * 12);
    for (int p = threadIdx.x; p < kWdBC; p += blockDim.x) ks[p] = __ldg(reinterpret_cast<const int*>(rec) + p);
    __syncthreads();
    for (int p = threadIdx.x; p < kWdBC; p += blockDim.x) {
      const int key = ks[p], row = key >> 8;
      if (row >= nrows) continue;
      int lo = 0, hi = p;  // first position of this row in the chunk
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((ks[mid] >> 8) < row) lo = mid + 1;
        else hi = mid;
      }
      const int pos = cnt[row] + (p - lo);
      sb[pos] = c * kWdBC + (key & 255);
      su[pos] = __ldg(reinterpret_cast<const double*>(rec + kWdBC * 4) + p);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < kWdBC; p += blockDim.x) {  // run ends advance the row cursors
      const int row = ks[p] >> 8;
      if (row >= nrows) continue;
      if (p + 1 == kWdBC || (ks[p + 1] >> 8) != row) {
        int lo = 0, hi = p;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((ks[mid] >> 8) < row) lo = mid + 1;
          else hi = mid;
        }
        cnt[row] += p - lo + 1;
      }
    }
    __syncthreads();
  }
}

constexpr int kFsW = 4;   // warps per CTA
constexpr int kFsNT = 8;  // 8-output DMMA tiles per warp (64 outputs)

template <bool UKAN>
__global__ void __launch_bounds__(32 * kFsW, 8)  // occupancy over registers: latency-bound gathers (ncu A/B: 1 -> 8 blocks/SM = 6.8 -> 4.2 ms despite spills)
seg_fsweep_kernel(const int* __restrict__ row_start, const int* __restrict__ sorted_b,
                  const double* __restrict__ sorted_u, const float* __restrict__ T, const float* __restrict__ scale,
                  const float* __restrict__ gy, float* __restrict__ dT, float* __restrict__ dscale, int d_in,
                  int d_out, int B, RowMap rm, Basis<4> bas) {
  __shared__ double Msh[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 2, kq = lane & 3;
  if (threadIdx.x < 16) Msh[threadIdx.x] = bas.M[threadIdx.x / 4][threadIdx.x % 4];
  __syncthreads();
  const int i = blockIdx.y;
  const int ob = (blockIdx.x * kFsW + warp) * (8 * kFsNT);
  if (ob >= d_out) return;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  const int* rs = row_start + row0 + i;
  const int* sb = sorted_b + (size_t)i * B;
  const double* su = sorted_u + (size_t)i * B;
  double acc[kFsNT][2], prod[kFsNT][2];
  float scl[kFsNT][2];
#pragma unroll
  for (int t = 0; t < kFsNT; ++t)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      acc[t][v] = prod[t][v] = 0.0;
      const int o = ob + t * 8 + 2 * kq + v;
      scl[t][v] = o < d_out ? __ldg(scale + (size_t)i * d_out + o) : 0.f;
    }
  const int nblk = (nrows + 3) / 4;
  int c0 = __ldg(rs + 0);
  for (int bb = 0; bb < nblk; ++bb) {
    const int c1 = __ldg(rs + min(4 * bb + 1, nrows)), c2 = __ldg(rs + min(4 * bb + 2, nrows)),
              c3 = __ldg(rs + min(4 * bb + 3, nrows)), c4 = __ldg(rs + min(4 * bb + 4, nrows));
    for (int kc = c0; kc < c4; kc += 4) {
      const int si = kc + kq;
      const bool vld = si < c4;
      const int sc = vld ? si : kc;
      const int vs = (sc >= c1) + (sc >= c2) + (sc >= c3);
      const int jj = grp - vs;
      const double u = __ldg(su + sc);
      const int j3 = jj & 3;
      const double wj = fma(fma(fma(Msh[12 + j3], u, Msh[8 + j3]), u, Msh[4 + j3]), u, Msh[j3]);
      const double a = (vld && jj >= 0 && jj < 4) ? wj : 0.0;
      const float* gr = gy + (size_t)__ldg(sb + sc) * d_out + ob + grp;
      double bf[kFsNT];
#pragma unroll
      for (int t = 0; t < kFsNT; ++t) bf[t] = (vld && ob + t * 8 + grp < d_out) ? (double)__ldg(gr + t * 8) : 0.0;
#pragma unroll
      for (int t = 0; t < kFsNT; ++t) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1])
                     : "d"(a), "d"(bf[t]));
      }
    }
    // rows 4bb .. 4bb+3 are complete: dT, the dscale products, then slide the upper half down
    const int row = 4 * bb + grp;
    if (grp < 4 && row < nrows) {
#pragma unroll
      for (int t = 0; t < kFsNT; ++t)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int o = ob + t * 8 + 2 * kq + v;
          if (o < d_out) {
            const size_t ci = (size_t)(row0 + row) * d_out + o;
            dT[ci] = (float)((double)scl[t][v] * acc[t][v]);
            prod[t][v] = fma((double)__ldg(T + ci), acc[t][v], prod[t][v]);
          }
        }
    }
#pragma unroll
    for (int t = 0; t < kFsNT; ++t)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const double up = __shfl_xor_sync(0xffffffffu, acc[t][v], 16);
        acc[t][v] = grp < 4 ? up : 0.0;
      }
    c0 = c4;
  }
  // dscale: sum the four row residues (grp 0..3) in a fixed order
#pragma unroll
  for (int t = 0; t < kFsNT; ++t)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      double d = prod[t][v];
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      d += __shfl_xor_sync(0xffffffffu, d, 8);
      const int o = ob + t * 8 + 2 * kq + v;
      if (lane < 4 && o < d_out) dscale[(size_t)i * d_out + o] = (float)d;
    }
}

// dx from the per-feature sorted order (UKAN, K = 4; round 2).  seg_fsort left each feature's samples
// sorted by window row; a warp takes a run of kSxRun consecutive positions of one feature, lanes
// own 4 consecutive outputs of each 128-output chunk, and the four window rows of C' (fp64 =
// scale * T) stay in registers while consecutive positions share the row — ~14 samples per row at
// the cfg4 shape, so the per-element fp32 -> fp64 conversions of spline_dx64 (its bound) mostly
// disappear.  Per position: Q_j = sum_o g[b,o] C'[row+j,o] accumulated per lane over the chunks in
// order, a fixed xor-tree over the lanes, dx = inv_dg * sum_j w'_j(u) Q_j (layers.py:44-46, 84-88).
constexpr int kSxRun = 4;
template <bool UKAN>
__global__ void __launch_bounds__(256)
seg_dx_sorted_kernel(const int* __restrict__ row_start, const int* __restrict__ sorted_b,
                     const double* __restrict__ sorted_u, const float* __restrict__ T, const double* __restrict__ s64,
                     const double* __restrict__ g64, float* __restrict__ dx, int d_in, int d_out, int B, RowMap rm,
                     Basis<4> bas) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.y;
  const int p0 = (blockIdx.x * 8 + warp) * kSxRun;
  if (p0 >= B) return;
  int row0, nrows;
  feature_rows<UKAN>(rm, i, row0, nrows);
  const int* rs = row_start + row0 + i;  // [nrows + 1] starts of each row's run of sorted positions
  const int pend = __ldg(rs + nrows);
  int rowp[kSxRun], bp[kSxRun];
  double up[kSxRun];
  {
    int lo = 0, hi = nrows;  // largest r with rs[r] <= p0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(rs + mid) <= p0) lo = mid;
      else hi = mid - 1;
    }
    int r = lo;
#pragma unroll
    for (int q = 0; q < kSxRun; ++q) {
      const int p = p0 + q;
      rowp[q] = -1;
      bp[q] = 0;
      up[q] = 0.0;
      if (p < pend) {
        while (r + 1 <= nrows && __ldg(rs + r + 1) <= p) ++r;
        rowp[q] = r;
        bp[q] = __ldg(sorted_b + (size_t)i * B + p);
        up[q] = __ldg(sorted_u + (size_t)i * B + p);
      }
    }
  }
  double acc[kSxRun][4];
#pragma unroll
  for (int q = 0; q < kSxRun; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[q][j] = 0.0;
  for (int oc = 0; oc < d_out; oc += 128) {
    const int o = oc + 4 * lane;
    if (o < d_out) {  // d_out % 4 == 0
      const double2 sa = __ldg(reinterpret_cast<const double2*>(s64 + (size_t)i * d_out + o));
      const double2 sb2 = __ldg(reinterpret_cast<const double2*>(s64 + (size_t)i * d_out + o) + 1);
      int cur = -1;
      double c[4][4];
#pragma unroll
      for (int q = 0; q < kSxRun; ++q) {
        if (rowp[q] < 0) continue;
        if (rowp[q] != cur) {  // the run moved to another row: its four window rows of C'
          cur = rowp[q];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(T + (size_t)(row0 + cur + j) * d_out + o));
            c[j][0] = sa.x * (double)t.x;
            c[j][1] = sa.y * (double)t.y;
            c[j][2] = sb2.x * (double)t.z;
            c[j][3] = sb2.y * (double)t.w;
          }
        }
        const double2 ga = __ldg(reinterpret_cast<const double2*>(g64 + (size_t)bp[q] * d_out + o));
        const double2 gb = __ldg(reinterpret_cast<const double2*>(g64 + (size_t)bp[q] * d_out + o) + 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double a = acc[q][j];
          a = fma(ga.x, c[j][0], a);
          a = fma(ga.y, c[j][1], a);
          a = fma(gb.x, c[j][2], a);
          a = fma(gb.y, c[j][3], a);
          acc[q][j] = a;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kSxRun; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double a = acc[q][j];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      acc[q][j] = a;
    }
  if (lane < kSxRun) {
    double a[4], wp[4];
    double u = 0.0;
    int row = -1, b = 0;
#pragma unroll
    for (int q = 0; q < kSxRun; ++q)
      if (q == lane) {
        row = rowp[q];
        b = bp[q];
        u = up[q];
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = acc[q][j];
      }
    if (row >= 0) {
      basis_dweights<4>(bas, u, wp);
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) t = fma(a[j], wp[j], t);
      dx[(size_t)b * d_in + i] = (float)(t * rm.inv_dg);
    }
  }
}

bool seg_uses_sorted(int B, int64_t total_rows, int64_t max_rows_hint) {
  static const bool cuda_cores = getenv("UKAN_SEG") != nullptr && getenv("UKAN_SEG")[0] == '1';
  static const bool tiles_only = getenv("UKAN_SEG") != nullptr && getenv("UKAN_SEG")[0] == 't';
  int64_t max_rows = std::min<int64_t>(total_rows, 2 * (int64_t)B * 4);
  if (max_rows_hint > 0) max_rows = std::min<int64_t>(max_rows, max_rows_hint);
  return !cuda_cores && !tiles_only && max_rows + 1 <= kFsMaxRows;
}

// dx on the sorted order seg_table_grad<4, true> just left in `ws` (same ws / shapes); s64 / g64:
// fp64 copies of scale and g.
int seg_dx_sorted(const float* T, const double* s64, const double* g64, float* dx, void* ws, int B, int d_in,
                  int d_out, int64_t total_rows, const RowMap& rm, cudaStream_t st) {
  const int nch = (B + kWdBC - 1) / kWdBC;
  unsigned char* recs = reinterpret_cast<unsigned char*>(ws);
  const int64_t rec = (((int64_t)d_in * nch * kWdBC * 12 + 255) / 256) * 256;
  const int64_t tiles = (total_rows + kWdRT - 1) / kWdRT + d_in;
  unsigned char* base = recs + rec + ((4 * ((int64_t)d_in + 1) + 255) / 256) * 256 +
                        ((int64_t)sizeof(double) * tiles * d_out + 255) / 256 * 256;
  const double* sorted_u = reinterpret_cast<const double*>(base);
  const int* sorted_b = reinterpret_cast<const int*>(base + (int64_t)8 * d_in * B);
  const int* row_start = reinterpret_cast<const int*>(base + ((int64_t)12 * d_in * B + 255) / 256 * 256);
  dim3 grid((unsigned)((B + 8 * kSxRun - 1) / (8 * kSxRun)), (unsigned)d_in);
  seg_dx_sorted_kernel<true><<<grid, 256, 0, st>>>(row_start, sorted_b, sorted_u, T, s64, g64, dx, d_in, d_out, B, rm,
                                                    make_basis<4>(3));
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

// dscale[f,o] = sum over the feature's tiles (fixed order)
__global__ void seg_reduce_kernel(const double* __restrict__ part, const int* __restrict__ tile_start,
                                  float* __restrict__ dscale, int d_in, int d_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)d_in * d_out) return;
  const int i = (int)(e / d_out), o = (int)(e % d_out);
  double a = 0.0;
  for (int t = tile_start[i]; t < tile_start[i + 1]; ++t) a += part[(size_t)t * d_out + o];
  dscale[e] = (float)a;
}

bool seg_supported(int64_t B) { return (B + kWdBC - 1) / kWdBC <= kSegMaxCh; }
bool seg_supported(int64_t B, int64_t d_out) { return seg_supported(B) && B * d_out < ((int64_t)1 << 31); }

int64_t seg_workspace(int64_t B, int64_t d_in, int64_t d_out, int64_t total_rows) {
  const int64_t nch = (B + kWdBC - 1) / kWdBC;
  const int64_t rec = ((d_in * nch * kWdBC * 12 + 255) / 256) * 256;
  const int64_t ts = ((4 * (d_in + 1) + 255) / 256) * 256;
  const int64_t tiles = (total_rows + kWdRT - 1) / kWdRT + d_in;
  const int64_t sorted = ((int64_t)12 * d_in * B + 255) / 256 * 256 + ((4 * (total_rows + d_in + 1)) + 255) / 256 * 256;
  return rec + ts + ((int64_t)sizeof(double) * tiles * d_out + 255) / 256 * 256 + sorted;
}

// max_rows_hint > 0: the largest per-feature row count (the key build reports it); without it the
// bound 2*B*K keeps large batches off the per-feature sorted sweep (its row histogram lives in
// shared memory) although the real segments are a few hundred rows.
template <int K, bool UKAN>
int seg_table_grad(const float* x, const float* T, const float* scale, const float* gy, float* dT, float* dscale,
                   void* ws, int64_t ws_bytes, int B, int d_in, int d_out, int64_t total_rows, const RowMap& rm,
                   cudaStream_t st, int64_t max_rows_hint) {
  if (ws == nullptr || ws_bytes < seg_workspace(B, d_in, d_out, total_rows)) return UKAN_E_WORKSPACE;
  const int nch = (B + kWdBC - 1) / kWdBC;
  unsigned char* recs = reinterpret_cast<unsigned char*>(ws);
  const int64_t rec = (((int64_t)d_in * nch * kWdBC * 12 + 255) / 256) * 256;
  int* tile_start = reinterpret_cast<int*>(recs + rec);
  double* part = reinterpret_cast<double*>(recs + rec + ((4 * ((int64_t)d_in + 1) + 255) / 256) * 256);
  const int64_t tiles = (total_rows + kWdRT - 1) / kWdRT + d_in;
  seg_prep_kernel<UKAN><<<dim3((d_in + 7) / 8, nch), 256, 0, st>>>(x, recs, B, d_in, nch, rm);
  UKAN_LAUNCH_CHECK();
  seg_tiles_kernel<UKAN><<<1, 32, 0, st>>>(rm, d_in, tile_start);
  UKAN_LAUNCH_CHECK();
  static const bool cuda_cores = getenv("UKAN_SEG") != nullptr && getenv("UKAN_SEG")[0] == '1';  // A/B only
  static const bool tiles_only = getenv("UKAN_SEG") != nullptr && getenv("UKAN_SEG")[0] == 't';  // A/B only
  int64_t max_rows = std::min<int64_t>(total_rows, 2 * (int64_t)B * K);
  if (max_rows_hint > 0) max_rows = std::min<int64_t>(max_rows, max_rows_hint);
  if constexpr (K == 4) {
    if (!cuda_cores && !tiles_only && max_rows + 1 <= kFsMaxRows) {
      unsigned char* base = recs + rec + ((4 * ((int64_t)d_in + 1) + 255) / 256) * 256 +
                            ((int64_t)sizeof(double) * tiles * d_out + 255) / 256 * 256;
      double* sorted_u = reinterpret_cast<double*>(base);
      int* sorted_b = reinterpret_cast<int*>(base + (int64_t)8 * d_in * B);
      int* row_start = reinterpret_cast<int*>(base + ((int64_t)12 * d_in * B + 255) / 256 * 256);
      const size_t smem = sizeof(int) * (size_t)(max_rows + 1);
      UKAN_CUDA_TRY(cudaFuncSetAttribute(seg_fsort_kernel<UKAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
      seg_fsort_kernel<UKAN><<<d_in, 256, smem, st>>>(recs, nch, d_in, rm, row_start, sorted_b, sorted_u, B);
      UKAN_LAUNCH_CHECK();
      const int n_og = (d_out + 8 * kFsNT * kFsW - 1) / (8 * kFsNT * kFsW);
      seg_fsweep_kernel<UKAN><<<dim3(n_og, d_in), 32 * kFsW, 0, st>>>(row_start, sorted_b, sorted_u, T, scale, gy, dT,
                                                                      dscale, d_in, d_out, B, rm, make_basis<4>(3));
      UKAN_LAUNCH_CHECK();
      return UKAN_OK;
    }
    if (!cuda_cores) {
      const int n_og = (d_out + kSdOW - 1) / kSdOW;
      const size_t smem = segd_smem_bytes();
      UKAN_CUDA_TRY(cudaFuncSetAttribute(seg_dmma_kernel<UKAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
      seg_dmma_kernel<UKAN><<<(unsigned)(tiles * n_og), 32 * kSdW, smem, st>>>(
          recs, T, scale, gy, dT, part, tile_start, d_in, d_out, nch, n_og, rm, make_basis<4>(3));
      UKAN_LAUNCH_CHECK();
      const int64_t n = (int64_t)d_in * d_out;
      seg_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, tile_start, dscale, d_in, d_out);
      UKAN_LAUNCH_CHECK();
      return UKAN_OK;
    }
  }
  const int n_os = (d_out + 31) / 32;
  const int W = std::min(8, n_os);
  const int n_og = (n_os + W - 1) / W;
  const size_t smem = seg_smem_bytes<K>(W);
  UKAN_CUDA_TRY(cudaFuncSetAttribute(seg_sweep_kernel<K, UKAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  seg_sweep_kernel<K, UKAN><<<(unsigned)(tiles * n_og), 32 * W, smem, st>>>(recs, T, scale, gy, dT, part, tile_start,
                                                                           d_in, d_out, nch, n_og, rm,
                                                                           make_basis<K>(K - 1));
  UKAN_LAUNCH_CHECK();
  const int64_t n = (int64_t)d_in * d_out;
  seg_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, tile_start, dscale, d_in, d_out);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

#define UKAN_SEG_INST(K)                                                                                        \
  template int seg_table_grad<K, true>(const float*, const float*, const float*, const float*, float*, float*, \
                                       void*, int64_t, int, int, int, int64_t, const RowMap&, cudaStream_t, int64_t);
UKAN_SEG_INST(1) UKAN_SEG_INST(2) UKAN_SEG_INST(3) UKAN_SEG_INST(4) UKAN_SEG_INST(5) UKAN_SEG_INST(6)
UKAN_SEG_INST(7) UKAN_SEG_INST(8) UKAN_SEG_INST(9) UKAN_SEG_INST(10) UKAN_SEG_INST(11)

}  // namespace ukan
