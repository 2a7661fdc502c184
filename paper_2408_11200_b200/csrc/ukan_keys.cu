// ukan_keys.cu — UKAN locate + (feature, group) key dedup + window row lookup.
//
// Replaces ukan_forward's index block (layers.py:261-287):
//   g_id = floor(x * (1/dg)) (int64); group = g_id // K; offset = g_id % K (Euclidean);
//   keys (group*d_in + f), ((group+1)*d_in + f); np.unique(..., return_inverse=True);
//   rows = where(offset + j < K, idx_prev, idx_next); cols = (offset + j) % K.
// B200 design: keys are packed feature-major, (f << 44) | (group + 2^43), deduplicated in two
// levels (a per-CTA shared-memory hash set over a tile of many samples x few features, then a
// global open-addressing hash set that only sees each CTA's distinct keys), counted per
// feature, scattered into per-feature segments and sorted per segment.  In feature-major
// order (f, g+1) directly follows (f, g), so a cell's K window rows are the consecutive rows
// base = idx(f, group)*K + offset of the flat [n_u*K, d_out] table.
#include "common.cuh"

namespace ukan {

constexpr uint64_t kEmpty = ~0ull;
constexpr int kGroupBias = 43;  // group + 2^43 must fit in 44 bits
constexpr int64_t kGidLimit = (int64_t)1 << 42;

__device__ __forceinline__ uint64_t pack_key(int f, int64_t grp) {
  return ((uint64_t)f << 44) | (uint64_t)(grp + ((int64_t)1 << kGroupBias));
}
__device__ __forceinline__ int key_feature(uint64_t k) { return (int)(k >> 44); }
__device__ __forceinline__ int64_t key_group(uint64_t k) {
  return (int64_t)(k & ((1ull << 44) - 1)) - ((int64_t)1 << kGroupBias);
}
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}

struct KeyWs {
  uint64_t* slots;  // [H]
  int64_t H;
  int32_t* counts;  // [d_in]
  int32_t* cursor;  // [d_in]
  int32_t* flags;   // [8]: 0 nonfinite, 1 range, 2 table full, 3 n_u, 4 max count
};

__device__ __forceinline__ void global_insert(const KeyWs& ws, uint64_t key) {
  uint64_t h = mix64(key) & (uint64_t)(ws.H - 1);
  for (int64_t probe = 0; probe < ws.H; ++probe) {
    unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(ws.slots + h),
                                       (unsigned long long)kEmpty, (unsigned long long)key);
    if (old == kEmpty) {
      atomicAdd(ws.counts + key_feature(key), 1);
      return;
    }
    if (old == key) return;
    h = (h + 1) & (uint64_t)(ws.H - 1);
  }
  atomicExch(ws.flags + 2, 1);
}

// Tile = kTileRows samples x kTileF features; shared hash set of kLocal slots.
constexpr int kTileRows = 128;
constexpr int kTileF = 32;
constexpr int kLocal = 4096;
constexpr int kLocalProbe = 32;

__global__ void __launch_bounds__(256)
keys_insert_kernel(const float* __restrict__ x, int64_t B, int d_in, int K, double inv_dg,
                   KeyWs ws) {
  __shared__ unsigned long long ls[kLocal];
  for (int t = threadIdx.x; t < kLocal; t += blockDim.x) ls[t] = kEmpty;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * kTileRows;
  const int f0 = blockIdx.y * kTileF;
  const int fl = threadIdx.x % kTileF;
  const int f = f0 + fl;
  bool bad_nf = false, bad_range = false;
  for (int rr = threadIdx.x / kTileF; rr < kTileRows; rr += blockDim.x / kTileF) {
    const int64_t b = b0 + rr;
    if (b >= B || f >= d_in) continue;
    const float xv = x[(size_t)b * d_in + f];
    if (!isfinite(xv)) {
      bad_nf = true;
      continue;
    }
    const double s = __dmul_rn((double)xv, inv_dg);
    if (!(fabs(s) < (double)kGidLimit)) {
      bad_range = true;
      continue;
    }
    const int64_t gid = (int64_t)floor(s);
    const int64_t grp = floor_div(gid, K);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t key = pack_key(f, grp + t);
      uint64_t h = mix64(key) & (kLocal - 1);
      bool done = false;
      for (int probe = 0; probe < kLocalProbe; ++probe) {
        const unsigned long long old = atomicCAS(ls + h, (unsigned long long)kEmpty, (unsigned long long)key);
        if (old == kEmpty || old == key) {
          done = true;
          break;
        }
        h = (h + 1) & (kLocal - 1);
      }
      if (!done) global_insert(ws, key);  // local set saturated: go straight to global
    }
  }
  if (bad_nf) atomicExch(ws.flags + 0, 1);
  if (bad_range) atomicExch(ws.flags + 1, 1);
  __syncthreads();
  for (int t = threadIdx.x; t < kLocal; t += blockDim.x) {
    const uint64_t key = ls[t];
    if (key != kEmpty) global_insert(ws, key);
  }
}

// Exclusive scan of per-feature counts -> seg_start[0..d_in]; n_u and max count to flags.
__global__ void __launch_bounds__(1024) keys_scan_kernel(const int32_t* __restrict__ counts,
                                                         int32_t* __restrict__ seg_start,
                                                         int d_in, int32_t* __restrict__ flags,
                                                         int64_t max_keys) {
  __shared__ int64_t warp_sums[32];
  __shared__ int64_t carry_s;
  __shared__ int maxc_s;
  if (threadIdx.x == 0) {
    carry_s = 0;
    maxc_s = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  int local_max = 0;
  for (int base = 0; base < d_in; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int64_t v = i < d_in ? counts[i] : 0;
    local_max = max(local_max, (int)v);
    int64_t incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t n = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += n;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int64_t ws = lane < (int)(blockDim.x / 32) ? warp_sums[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t n = __shfl_up_sync(0xffffffffu, ws, off);
        if (lane >= off) ws += n;
      }
      warp_sums[lane] = ws;
    }
    __syncthreads();
    const int64_t wprefix = wid > 0 ? warp_sums[wid - 1] : 0;
    const int64_t excl = carry_s + wprefix + incl - v;
    if (i < d_in) seg_start[i] = (int32_t)min(excl, (int64_t)INT32_MAX);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = excl + v;
    __syncthreads();
  }
  atomicMax(&maxc_s, local_max);
  __syncthreads();
  if (threadIdx.x == 0) {
    seg_start[d_in] = (int32_t)min(carry_s, (int64_t)INT32_MAX);
    flags[3] = (int32_t)min(carry_s, (int64_t)INT32_MAX);
    flags[4] = maxc_s;
    if (carry_s > max_keys) flags[5] = 1;
  }
}

__global__ void keys_scatter_kernel(KeyWs ws, const int32_t* __restrict__ seg_start,
                                    int32_t* __restrict__ key_f, int64_t* __restrict__ key_g) {
  if (ws.flags[5]) return;  // capacity exceeded: the host retries with a larger buffer
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ws.H) return;
  const uint64_t key = ws.slots[t];
  if (key == kEmpty) return;
  const int f = key_feature(key);
  const int pos = seg_start[f] + atomicAdd(ws.cursor + f, 1);
  key_f[pos] = f;
  key_g[pos] = key_group(key);
}

// Per-feature ascending sort of key_g[seg]: shared-memory bitonic for segments up to kSegSm,
// in-place global-memory bitonic (same network) for larger ones.
constexpr int kSegSm = 4096;

__device__ void bitonic_block(int64_t* a, int n_pow2) {
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool asc = (i & k) == 0;
          const int64_t ai = a[i], al = a[l];
          if ((ai > al) == asc) {
            a[i] = al;
            a[l] = ai;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(512)
keys_sort_kernel(const int32_t* __restrict__ flags, const int32_t* __restrict__ seg_start,
                 int64_t* __restrict__ key_g, int64_t* __restrict__ scratch) {
  if (flags[5]) return;
  __shared__ int64_t sm[kSegSm];
  const int f = blockIdx.x;
  const int s0 = seg_start[f], n = seg_start[f + 1] - s0;
  if (n <= 1) return;
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  int64_t* a;
  if (np2 <= kSegSm) {
    a = sm;
  } else {
    a = scratch + (int64_t)s0 * 2;  // scratch has 2*n_u capacity -> segment fits (np2 < 2n)
  }
  for (int i = threadIdx.x; i < np2; i += blockDim.x) a[i] = i < n ? key_g[s0 + i] : INT64_MAX;
  __syncthreads();
  bitonic_block(a, np2);
  for (int i = threadIdx.x; i < n; i += blockDim.x) key_g[s0 + i] = a[i];
}

// base_row[b, f] = idx(f, group)*K + offset via binary search in the feature's segment.
__global__ void keys_base_row_kernel(const float* __restrict__ x, int64_t B, int d_in, int K,
                                     double inv_dg, const int32_t* __restrict__ flags,
                                     const int32_t* __restrict__ seg_start,
                                     const int64_t* __restrict__ key_g,
                                     int32_t* __restrict__ base_row) {
  if (flags[0] | flags[1] | flags[2] | flags[5]) return;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * (int64_t)d_in) return;
  const int f = (int)(t % d_in);
  const double s = __dmul_rn((double)x[t], inv_dg);
  const int64_t gid = (int64_t)floor(s);
  const int64_t grp = floor_div(gid, K);
  const int64_t off = gid - grp * K;
  int lo = seg_start[f], hi = seg_start[f + 1];  // find grp in key_g[lo, hi)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key_g[mid] < grp) lo = mid + 1;
    else hi = mid;
  }
  base_row[t] = (int32_t)(lo * (int64_t)K + off);
}

static int64_t next_pow2(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

struct KeysLayout {
  int64_t H, off_slots, off_counts, off_cursor, off_flags, off_scratch, total;
};

static KeysLayout keys_layout(int64_t d_in, int64_t max_keys) {
  KeysLayout L;
  L.H = next_pow2(std::max<int64_t>(2 * max_keys, 1024));
  int64_t o = 0;
  L.off_slots = o;
  o += L.H * 8;
  L.off_counts = o;
  o += ((d_in * 4 + 255) / 256) * 256;
  L.off_cursor = o;
  o += ((d_in * 4 + 255) / 256) * 256;
  L.off_flags = o;
  o += 256;
  L.off_scratch = o;
  o += 2 * max_keys * 8 + 256;
  L.total = o;
  return L;
}

}  // namespace ukan

using namespace ukan;

extern "C" int64_t ukan_ukan_keys_workspace_size(int64_t B, int64_t d_in, int64_t max_keys) {
  (void)B;
  return keys_layout(d_in, max_keys).total;
}

extern "C" int ukan_ukan_build_keys(const float* x, int64_t B, int64_t d_in, int k,
                                    double delta_g, int32_t* key_f, int64_t* key_g,
                                    int32_t* seg_start, int32_t* base_row, int64_t max_keys,
                                    void* workspace, int64_t workspace_bytes,
                                    int64_t* n_unique_host, int64_t* max_rows_host,
                                    int32_t* nonfinite_host, void* stream) {
  if (k < 0 || k > UKAN_MAX_DEGREE) return UKAN_E_DEGREE;
  if (!(delta_g > 0)) return UKAN_E_GRID;
  if (!x || !key_f || !key_g || !seg_start || !base_row || !n_unique_host || !nonfinite_host ||
      B < 0 || d_in < 1 || d_in >= (1 << 19) || max_keys < 1 || max_keys >= ((int64_t)1 << 31))
    return UKAN_E_ARG;
  const KeysLayout L = keys_layout(d_in, max_keys);
  if (!workspace || workspace_bytes < L.total) return UKAN_E_WORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  KeyWs ws;
  ws.slots = (uint64_t*)(w + L.off_slots);
  ws.H = L.H;
  ws.counts = (int32_t*)(w + L.off_counts);
  ws.cursor = (int32_t*)(w + L.off_cursor);
  ws.flags = (int32_t*)(w + L.off_flags);
  int64_t* scratch = (int64_t*)(w + L.off_scratch);
  const int K = k + 1;
  const double inv_dg = 1.0 / delta_g;  // layers.py:261
  UKAN_CUDA_TRY(cudaMemsetAsync(ws.slots, 0xFF, L.H * 8, st));
  UKAN_CUDA_TRY(cudaMemsetAsync(w + L.off_counts, 0, L.off_scratch - L.off_counts, st));
  if (B > 0) {
    dim3 g((unsigned)((B + kTileRows - 1) / kTileRows), (unsigned)((d_in + kTileF - 1) / kTileF));
    keys_insert_kernel<<<g, 256, 0, st>>>(x, B, (int)d_in, K, inv_dg, ws);
    UKAN_LAUNCH_CHECK();
  }
  keys_scan_kernel<<<1, 1024, 0, st>>>(ws.counts, seg_start, (int)d_in, ws.flags, max_keys);
  UKAN_LAUNCH_CHECK();
  keys_scatter_kernel<<<(unsigned)((L.H + 255) / 256), 256, 0, st>>>(ws, seg_start, key_f, key_g);
  UKAN_LAUNCH_CHECK();
  keys_sort_kernel<<<(unsigned)d_in, 512, 0, st>>>(ws.flags, seg_start, key_g, scratch);
  UKAN_LAUNCH_CHECK();
  const int64_t n = B * d_in;
  if (n > 0) {
    keys_base_row_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, B, (int)d_in, K, inv_dg, ws.flags, seg_start, key_g, base_row);
    UKAN_LAUNCH_CHECK();
  }
  int32_t flags[8];
  UKAN_CUDA_TRY(cudaMemcpyAsync(flags, ws.flags, sizeof(flags), cudaMemcpyDeviceToHost, st));
  UKAN_CUDA_TRY(cudaStreamSynchronize(st));
  *nonfinite_host = flags[0] ? 1 : (flags[1] ? 2 : 0);
  *n_unique_host = flags[3];
  if (max_rows_host) *max_rows_host = (int64_t)flags[4] * K;
  if (flags[0] || flags[1]) return UKAN_OK;  // caller raises DomainError
  if (flags[2] || flags[5]) return UKAN_E_CAPACITY;
  if ((int64_t)flags[4] * K >= (1 << 23)) return UKAN_E_CAPACITY;
  return UKAN_OK;
}
