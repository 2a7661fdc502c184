// cg_tc.cu — the coefficient-generator MLP GEMMs on the 5th-generation tensor cores (tcgen05).
//
// Replaces the matmuls of _cg_eval (layers.py:241-243) and their tape backward (tensor.py:189-197):
//   forward  pre = inp @ W1 + b1, H = silu(pre)      table = H @ W2 + b2
//   backward dW2 = H^T dT, dH = dT W2^T, dW1 = inp^T dpre, dinp = dpre W1^T
// which are plain dense GEMMs (the north star's one tensor-core use).  Precision: the reference is
// float64; fp32 products accumulated in fp32 fail the parity bar on the n_u-long weight-gradient
// reductions and plain TF32 fails everywhere.  Measured here: 3xTF32 (two
// pieces, three products) on tcgen05 still misses the UKAN gradient parity by 2-3x, because the
// tensor core's fp32 accumulator truncates and two tf32 pieces carry only ~22 bits.  So this
// kernel is used for the table GEMM only (H @ W2 + b2, whose outputs feed the spline forward):
// operands split into round-to-nearest tf32 pieces (2 pieces / 3 products; a 3-piece / 6-product
// variant is templated), every 32-wide K chunk promoted out of TMEM into fp32 registers.  The
// gradient GEMMs run on the FP64 tensor cores (cg_dmma.cu).
//
// CTA = 8 warps, one 128 x BN output tile (TMEM: 128 lanes x 2 x BN fp32 columns), K in chunks
// of 32.  All threads load a chunk from global (any transpose: the loader reads along the
// contiguous global dimension), splits it into hi/mid/lo tf32 and stores them in the canonical
// K-major no-swizzle shared layout (8-row x 16-byte core matrices, LBO = 128 B, SBO = 1 KB);
// thread 0 issues 4 k-steps x 6 MMAs into the chunk's TMEM buffer and commits to the chunk
// buffer's mbarrier, so the next chunk's loads overlap the tensor-core work (double buffer);
// each chunk's partial is promoted into fp32 registers (see the kernel comment).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace ukan {

constexpr int kTcgM = 128;   // tile rows (TMEM lanes)
constexpr int kTcgK = 32;    // K per chunk
constexpr int kTcgThreads = 256;  // 8 warps: two per TMEM lane quarter (column halves)

// fp32 -> tf32 (10 mantissa bits), round to nearest with ties away from zero, low 13 bits zeroed
// (the same rounding as cvt.rna.tf32.f32, spelled out so the split is exact by construction:
// a - tf32(a) is then exactly representable and carries the remaining 13 bits)
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
}

__device__ __forceinline__ void cg_mb_init(uint64_t* mb, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)), "r"(count));
}
__device__ __forceinline__ void cg_mb_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// sm100 shared-memory matrix descriptor, K-major, no swizzle (layout type 0, version 1).
__device__ __forceinline__ uint64_t cg_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__device__ __forceinline__ void cg_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}

// byte offset of element (row r, k) inside a [rows x 32] K-major canonical tile
__device__ __forceinline__ uint32_t cg_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// a = hi + mid + lo, each a tf32 value (round-to-nearest); the residual after lo is < 2^-33 |a|.
__device__ __forceinline__ void tf32_split3(float a, uint32_t& h, uint32_t& m, uint32_t& l) {
  h = tf32_rna(a);
  const float r1 = a - __uint_as_float(h);  // exact
  m = tf32_rna(r1);
  l = tf32_rna(r1 - __uint_as_float(m));    // exact difference, rounded
}

// Load a [ROWS x 32] chunk of op(X) (element (r, k) at X[r*sr + k*sk]) into hi/mid/lo tiles
// (consecutive, TB bytes apart).
template <int ROWS, int PIECES>
__device__ __forceinline__ void cg_load_tile(const float* __restrict__ X, int64_t sr, int64_t sk, int r0, int k0,
                                             int R, int Kt, unsigned char* t0) {
  constexpr int TB = ROWS * kTcgK * 4;
  if (sk == 1) {  // K contiguous: float4 along k
    for (int t = threadIdx.x; t < ROWS * 8; t += kTcgThreads) {
      const int r = t >> 3, k = (t & 7) * 4;
      float e[4] = {0.f, 0.f, 0.f, 0.f};
      if (r0 + r < R && k0 + k + 3 < Kt) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + (size_t)(r0 + r) * sr + k0 + k));
        e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
      } else if (r0 + r < R) {
#pragma unroll
        for (int q = 0; q < 4; ++q) e[q] = (k0 + k + q < Kt) ? __ldg(X + (size_t)(r0 + r) * sr + k0 + k + q) : 0.f;
      }
      uint32_t h[4], m[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tf32_split3(e[q], h[q], m[q], l[q]);
      const uint32_t o = cg_off(r, k);
      *reinterpret_cast<uint4*>(t0 + o) = make_uint4(h[0], h[1], h[2], h[3]);
      if (PIECES == 2) {  // two pieces: the second carries the whole remainder (rounded)
#pragma unroll
        for (int q = 0; q < 4; ++q) m[q] = tf32_rna(e[q] - __uint_as_float(h[q]));
        *reinterpret_cast<uint4*>(t0 + TB + o) = make_uint4(m[0], m[1], m[2], m[3]);
      } else {
        *reinterpret_cast<uint4*>(t0 + TB + o) = make_uint4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<uint4*>(t0 + 2 * TB + o) = make_uint4(l[0], l[1], l[2], l[3]);
      }
    }
  } else {  // rows contiguous (sr == 1): float4 along r at fixed k
    for (int t = threadIdx.x; t < ROWS / 4 * 32; t += kTcgThreads) {
      const int k = t / (ROWS / 4), r = (t % (ROWS / 4)) * 4;
      float e[4] = {0.f, 0.f, 0.f, 0.f};
      if (k0 + k < Kt) {
        if (r0 + r + 3 < R) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(X + (size_t)(k0 + k) * sk + r0 + r));
          e[0] = v.x; e[1] = v.y; e[2] = v.z; e[3] = v.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) e[q] = (r0 + r + q < R) ? __ldg(X + (size_t)(k0 + k) * sk + r0 + r + q) : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t h, m, l;
        tf32_split3(e[q], h, m, l);
        const uint32_t o = cg_off(r + q, k);
        *reinterpret_cast<uint32_t*>(t0 + o) = h;
        if (PIECES == 2) {
          *reinterpret_cast<uint32_t*>(t0 + TB + o) = tf32_rna(e[q] - __uint_as_float(h));
        } else {
          *reinterpret_cast<uint32_t*>(t0 + TB + o) = m;
          *reinterpret_cast<uint32_t*>(t0 + 2 * TB + o) = l;
        }
      }
    }
  }
}

// D[m, n] = sum_k A(m, k) B(k, n), A(m,k) = A[m*sam + k*sak], B(k,n) = B[k*sbk + n*sbn].
// mode 0: C = act(D + bias[n]) (pre = D + bias when act);   mode 1: C = D * silu'(pre[m, n]);
// mode 2: part[z][m][n] = D over K-chunk z (split-K, fp64-reduced by cg_splitk_reduce_kernel).
//
// Accumulation precision: the tensor core's fp32 accumulator is not IEEE-exact (measured: a
// K=4096 tensor-core sum was 40x less accurate than an fp32 FMA chain), so every 32-wide K chunk
// goes to its own TMEM buffer (two, alternating) and is promoted into fp32 register
// accumulators by the threads while the next chunk's MMAs run.  Thread (warp w, lane l) owns
// row 32*(w%4)+l and columns [(w/4)*BN/2, +BN/2).
template <int BN, typename AccT, int PIECES>
__global__ void __launch_bounds__(kTcgThreads, BN <= 64 ? 2 : 1)
cg_gemm_tc_kernel(const float* __restrict__ A, int64_t sam, int64_t sak, const float* __restrict__ Bm, int64_t sbk,
                  int64_t sbn, int M, int N, int K, int kps, int mode, const float* __restrict__ bias, int act,
                  float* __restrict__ C, float* __restrict__ pre, float* __restrict__ part) {
  constexpr int A_BYTES = kTcgM * kTcgK * 4, B_BYTES = BN * kTcgK * 4;
  constexpr int STAGE = PIECES * (A_BYTES + B_BYTES);  // A pieces | B pieces
  constexpr int HN = BN / 2;                         // columns per thread
  constexpr int TCOLS = 2 * BN < 32 ? 32 : 2 * BN;   // two accumulator buffers
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kTcgM >> 4) << 24);  // f32 accum, tf32 A/B, K-major, M=128
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tbase_s;
  __shared__ __align__(8) uint64_t mma_done[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int m0 = blockIdx.x * kTcgM, n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int kb = z * kps, ke = min(K, kb + kps);
  const int nch = (ke - kb + kTcgK - 1) / kTcgK;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    cg_mb_init(&mma_done[0], 1);
    cg_mb_init(&mma_done[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase_s;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(half * HN);

  AccT acc[HN];  // fp64 for the split-K weight gradients (long reductions), fp32 otherwise
#pragma unroll
  for (int j = 0; j < HN; ++j) acc[j] = (AccT)0;
  auto drain = [&](int c) {  // chunk c's partial (TMEM buffer c&1) -> registers
    const uint32_t ta = trow + (uint32_t)((c & 1) * BN);
#pragma unroll
    for (int cb = 0; cb < HN; cb += 32) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta + (uint32_t)cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (cb + j < HN) acc[cb + j] += (AccT)__uint_as_float(r[j]);
    }
  };

  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c >= 2) {
      cg_mb_wait(&mma_done[buf], (uint32_t)(((c - 2) >> 1) & 1));  // chunk c-2 done: smem + TMEM buffer free
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      drain(c - 2);
    }
    unsigned char* st = smem_raw + (size_t)buf * STAGE;
    const int k0 = kb + c * kTcgK;
    cg_load_tile<kTcgM, PIECES>(A, sam, sak, m0, k0, M, ke, st);
    cg_load_tile<BN, PIECES>(Bm, sbn, sbk, n0, k0, N, ke, st + PIECES * A_BYTES);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic stores -> tensor-core reads
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = sbase + buf * STAGE, b0 = a0 + PIECES * A_BYTES;
      const uint32_t td = tmem + (uint32_t)(buf * BN);
      // products with piece-order sum <= PIECES-1, smallest terms first:
      //   2 pieces: (h,l) (l,h) (h,h);   3 pieces: (l,h) (m,m) (h,l) (m,h) (h,m) (h,h)
      constexpr int NP = PIECES == 2 ? 3 : 6;
      constexpr int PA3[6] = {2, 1, 0, 1, 0, 0}, PB3[6] = {0, 1, 2, 0, 1, 0};
      constexpr int PA2[3] = {0, 1, 0}, PB2[3] = {1, 0, 0};
#pragma unroll
      for (int kk = 0; kk < kTcgK / 8; ++kk) {
        const uint32_t off = kk * 256;  // two 16-byte core-matrix columns per k-step of 8
#pragma unroll
        for (int t = 0; t < NP; ++t)
          cg_mma_tf32(td, cg_desc(a0 + (PIECES == 2 ? PA2[t] : PA3[t]) * A_BYTES + off, 128, 1024),
                      cg_desc(b0 + (PIECES == 2 ? PB2[t] : PB3[t]) * B_BYTES + off, 128, 1024), IDESC,
                      (kk > 0 || t > 0) ? 1 : 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&mma_done[buf]))
                   : "memory");
    }
  }
  for (int c = max(0, nch - 2); c < nch; ++c) {  // the last two chunks, in order
    cg_mb_wait(&mma_done[c & 1], (uint32_t)((c >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    drain(c);
  }

  if (mode == 0) {
    // coalesced epilogue: the thread-per-row accumulators go through shared memory (the pipeline
    // stages are free once every chunk is drained) so each warp stores contiguous row segments
    constexpr int TS = BN + 1;  // odd row stride: the row-per-lane writes hit distinct banks
    float* tile = reinterpret_cast<float*>(smem_raw);
    __syncthreads();
    const int r = 32 * q + lane;
#pragma unroll
    for (int j = 0; j < HN; ++j) {
      const int n = n0 + half * HN + j;
      const float v = (float)acc[j] + ((bias && n < N) ? bias[n] : 0.f);
      tile[r * TS + half * HN + j] = v;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < kTcgM * BN; idx += kTcgThreads) {
      const int rr = idx / BN, cc = idx % BN;
      const int mm = m0 + rr, n = n0 + cc;
      if (mm >= M || n >= N) continue;
      const float v = tile[rr * TS + cc];
      if (act) {
        pre[(size_t)mm * N + n] = v;
        C[(size_t)mm * N + n] = v / (1.f + __expf(-v));
      } else {
        C[(size_t)mm * N + n] = v;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
    return;
  }
  // epilogue: row m, columns n0 + half*HN + j
  const int m = m0 + 32 * q + lane;
  if (m < M) {
#pragma unroll
    for (int j = 0; j < HN; ++j) {  // fully unrolled: acc stays in registers
      const int n = n0 + half * HN + j;
      if (n >= N) continue;
      const float d = (float)acc[j];
      if (mode == 2) {
        part[((size_t)z * M + m) * N + n] = d;
      } else if (mode == 1) {  // dpre = dH * (s + pre*s*(1-s))  (tensor.py:232-233)
        const float p = pre[(size_t)m * N + n];
        const float s = 1.f / (1.f + __expf(-p));
        C[(size_t)m * N + n] = d * (s + p * s * (1.f - s));
      } else {
        const float v = d + (bias ? bias[n] : 0.f);
        if (act) {
          pre[(size_t)m * N + n] = v;
          C[(size_t)m * N + n] = v / (1.f + __expf(-v));
        } else {
          C[(size_t)m * N + n] = v;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
}

// ---------------------------------------------------------------------------------------
// Table GEMM with pre-split operands (round 2): C = A B + bias, A [M, K] row-major, B [K, N]
// row-major, 2 tf32 pieces / 3 products, fp32 promotion per 32-wide K chunk — bitwise the
// cg_gemm_tc_kernel<BN, float, 2> result, but the operand split is done once per call by
// cg_presplit_kernel into the canonical K-major core-matrix layout, tile by tile and chunk by
// chunk, so each (tile, chunk) is one contiguous block: the GEMM then streams them with 1-D bulk
// copies (cp.async.bulk) through a 3-stage mbarrier ring while the tensor core works, instead of
// every thread loading, splitting and storing each chunk (the old kernel waited on those loads:
// long-scoreboard stalls on the split's first instruction, 19% issue).
//   thread 0: waits chunk c's copies + TMEM buffer c&1 drained (chunk c-2), issues the 12 MMAs,
//             commits; refills the stage of chunk c-1 with chunk c-1+NS once its MMAs are done;
//   all:      drain chunk c-1 (TMEM -> fp32 registers), arrive on drained[(c-1)&1].

// Ap[(tile * nch + c) * 2 + piece] = piece of the [ROWS x 32] chunk c of tile `tile` of X, canonical
// layout; rows / k past the ends are zero.  X(r, k) = X[r * sr + k * sk]; one thread per 4 k (sk == 1)
// or 4 rows (sr == 1), vectorised along the contiguous dimension.
template <int ROWS>
__global__ void __launch_bounds__(256) cg_presplit_kernel(const float* __restrict__ X, int64_t sr, int64_t sk, int R,
                                                          int K, int nch, unsigned char* __restrict__ out) {
  constexpr int TB = ROWS * kTcgK * 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_chunk = ROWS * kTcgK / 4;  // 4-element groups per (tile, chunk)
  const int64_t n_tiles = (R + ROWS - 1) / ROWS;
  if (t >= n_tiles * nch * per_chunk) return;
  const int g = (int)(t % per_chunk);
  const int64_t tc = t / per_chunk;
  const int c = (int)(tc % nch), tile = (int)(tc / nch);
  unsigned char* dst = out + (size_t)tc * 2 * TB;
  float e[4];
  int rr[4], kk[4];
  if (sk == 1) {  // 4 consecutive k of one row
    const int r = g / (kTcgK / 4), k = (g % (kTcgK / 4)) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rr[q] = r;
      kk[q] = k + q;
    }
  } else {  // 4 consecutive rows at one k
    const int k = g / (ROWS / 4), r = (g % (ROWS / 4)) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rr[q] = r + q;
      kk[q] = k;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gr = tile * ROWS + rr[q], gk = c * kTcgK + kk[q];
    e[q] = (gr < R && gk < K) ? __ldg(X + (size_t)gr * sr + (size_t)gk * sk) : 0.f;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t h = tf32_rna(e[q]);
    const uint32_t l = tf32_rna(e[q] - __uint_as_float(h));
    const uint32_t o = cg_off(rr[q], kk[q]);
    *reinterpret_cast<uint32_t*>(dst + o) = h;
    *reinterpret_cast<uint32_t*>(dst + TB + o) = l;
  }
}

__device__ __forceinline__ void cg_mb_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cg_mb_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)) : "memory");
}
__device__ __forceinline__ void cg_bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(mb))
               : "memory");
}

template <int BN, int kTpNS>  // kTpNS: smem stages (one K chunk of both operands each)
__global__ void __launch_bounds__(kTcgThreads, BN <= 64 ? 2 : 1)
cg_table_tc_kernel(const unsigned char* __restrict__ Ap, const unsigned char* __restrict__ Bp, int M, int N, int nch,
                   const float* __restrict__ bias, float* __restrict__ C) {
  constexpr int A_BYTES = kTcgM * kTcgK * 4, B_BYTES = BN * kTcgK * 4;
  constexpr int STAGE = 2 * (A_BYTES + B_BYTES);  // A hi | A lo | B hi | B lo
  constexpr int HN = BN / 2;
  constexpr int TCOLS = 2 * BN;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kTcgM >> 4) << 24);  // f32 accum, tf32 A/B, K-major, M=128
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint32_t tbase_s;
  __shared__ __align__(8) uint64_t loaded[kTpNS], mma_done[2], drained[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, half = warp >> 2;
  const int nt = blockIdx.x, mt = blockIdx.y;  // n-tiles fastest: a wave shares A tiles through L2
  const int m0 = mt * kTcgM, n0 = nt * BN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase_s)),
                 "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int d = 0; d < kTpNS; ++d) cg_mb_init(&loaded[d], 1);
    for (int d = 0; d < 2; ++d) {
      cg_mb_init(&mma_done[d], 1);
      cg_mb_init(&drained[d], kTcgThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase_s;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(half * HN);
  auto issue = [&](int c) {  // chunk c of both operands -> stage c % NS
    unsigned char* st = smem_raw + (size_t)(c % kTpNS) * STAGE;
    uint64_t* mb = &loaded[c % kTpNS];
    cg_mb_expect_tx(mb, STAGE);
    cg_bulk_g2s(st, Ap + ((size_t)mt * nch + c) * 2 * A_BYTES, 2 * A_BYTES, mb);
    cg_bulk_g2s(st + 2 * A_BYTES, Bp + ((size_t)nt * nch + c) * 2 * B_BYTES, 2 * B_BYTES, mb);
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < min(kTpNS, nch); ++c) issue(c);

  float acc[HN];
#pragma unroll
  for (int j = 0; j < HN; ++j) acc[j] = 0.f;
  auto drain = [&](int c) {  // chunk c's partial (TMEM buffer c&1) -> registers, then release the buffer
    cg_mb_wait(&mma_done[c & 1], (uint32_t)((c >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t ta = trow + (uint32_t)((c & 1) * BN);
#pragma unroll
    for (int cb = 0; cb < HN; cb += 32) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
          "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta + (uint32_t)cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (cb + j < HN) acc[cb + j] += __uint_as_float(r[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) cg_mb_arrive(&drained[c & 1]);
  };

  for (int c = 0; c < nch; ++c) {
    if (threadIdx.x == 0) {
      cg_mb_wait(&loaded[c % kTpNS], (uint32_t)((c / kTpNS) & 1));
      if (c >= 2) cg_mb_wait(&drained[c & 1], (uint32_t)(((c - 2) >> 1) & 1));  // TMEM buffer free
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = sbase + (uint32_t)((c % kTpNS) * STAGE), b0 = a0 + 2 * A_BYTES;
      const uint32_t td = tmem + (uint32_t)((c & 1) * BN);
      constexpr int PA2[3] = {0, 1, 0}, PB2[3] = {1, 0, 0};  // (h,l) (l,h) (h,h): as cg_gemm_tc_kernel
#pragma unroll
      for (int kk = 0; kk < kTcgK / 8; ++kk) {
        const uint32_t off = kk * 256;
#pragma unroll
        for (int t = 0; t < 3; ++t)
          cg_mma_tf32(td, cg_desc(a0 + PA2[t] * A_BYTES + off, 128, 1024), cg_desc(b0 + PB2[t] * B_BYTES + off, 128, 1024),
                      IDESC, (kk > 0 || t > 0) ? 1 : 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&mma_done[c & 1]))
                   : "memory");
      // the stage of chunk c-1 is free once its MMAs completed: refill it with chunk c-1+NS
      if (c >= 1 && c - 1 + kTpNS < nch) {
        cg_mb_wait(&mma_done[(c - 1) & 1], (uint32_t)(((c - 1) >> 1) & 1));
        issue(c - 1 + kTpNS);
      }
    }
    __syncwarp();
    if (c >= 1) drain(c - 1);
  }
  if (nch > 0) drain(nch - 1);

  // coalesced epilogue through shared memory (every stage consumed): C = acc + bias
  constexpr int TS = BN + 1;
  float* tile = reinterpret_cast<float*>(smem_raw);
  __syncthreads();
  const int r = 32 * q + lane;
#pragma unroll
  for (int j = 0; j < HN; ++j) {
    const int n = n0 + half * HN + j;
    tile[r * TS + half * HN + j] = acc[j] + ((bias && n < N) ? bias[n] : 0.f);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kTcgM * BN; idx += kTcgThreads) {
    const int rr = idx / BN, cc = idx % BN;
    const int mm = m0 + rr, n = n0 + cc;
    if (mm < M && n < N) C[(size_t)mm * N + n] = tile[rr * TS + cc];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
}

// colsum[n] = sum_k X[k][n] (fp64, fixed order): pass 1 sums 32 columns x one row slice per CTA
// (8 warps, rows interleaved, then the 8 warp sums in order) into part[slice][n]; pass 2 adds the
// slices in order.
template <typename T>
__global__ void __launch_bounds__(256) cg_colsum_part_kernel(const T* __restrict__ X, double* __restrict__ part,
                                                             int K, int N, int rows_per_slice) {
  __shared__ double red[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), ty = threadIdx.x >> 5;
  const int k0 = blockIdx.y * rows_per_slice, k1 = min(K, k0 + rows_per_slice);
  double a = 0.0;
  if (c < N)
    for (int k = k0 + ty; k < k1; k += 8) a += (double)X[(size_t)k * N + c];
  red[ty][threadIdx.x & 31] = a;
  __syncthreads();
  if (ty == 0 && c < N) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x & 31];
    part[(size_t)blockIdx.y * N + c] = s;
  }
}
// float4 variant (N % 4 == 0, 16-byte aligned rows): a lane sums 4 adjacent columns, two rows in
// flight per iteration (fixed order: even rows then odd rows of the lane's stride, then the warps)
__global__ void __launch_bounds__(256) cg_colsum_part4_kernel(const float* __restrict__ X, double* __restrict__ part,
                                                              int K, int N, int rows_per_slice) {
  __shared__ double red[8][132];
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + lane * 4;
  const int k0 = blockIdx.y * rows_per_slice, k1 = min(K, k0 + rows_per_slice);
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
  if (c < N) {
    int k = k0 + ty;
    for (; k + 8 < k1; k += 16) {
      const float4 u = __ldg(reinterpret_cast<const float4*>(X + (size_t)k * N + c));
      const float4 v = __ldg(reinterpret_cast<const float4*>(X + (size_t)(k + 8) * N + c));
      a[0] += (double)u.x; a[1] += (double)u.y; a[2] += (double)u.z; a[3] += (double)u.w;
      b[0] += (double)v.x; b[1] += (double)v.y; b[2] += (double)v.z; b[3] += (double)v.w;
    }
    if (k < k1) {
      const float4 u = __ldg(reinterpret_cast<const float4*>(X + (size_t)k * N + c));
      a[0] += (double)u.x; a[1] += (double)u.y; a[2] += (double)u.z; a[3] += (double)u.w;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[ty][lane * 4 + j] = a[j] + b[j];
  __syncthreads();
  if (ty == 0 && c < N) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double s = 0.0;
      for (int q = 0; q < 8; ++q) s += red[q][lane * 4 + j];
      part[(size_t)blockIdx.y * N + c + j] = s;
    }
  }
}

__global__ void cg_colsum_final_kernel(const double* __restrict__ part, float* __restrict__ out, int N, int S) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += part[(size_t)z * N + c];
  out[c] = (float)s;
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
int kan_num_sms();

static size_t cg_smem(int BN, int pieces) { return 2 * (size_t)pieces * (kTcgM * kTcgK * 4 + BN * kTcgK * 4) + 1024; }

template <int BN, typename AccT, int PIECES>
static int cg_launch(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int M,
                     int N, int K, int kps, int S, int mode, const float* bias, int act, float* C, float* pre,
                     float* part, cudaStream_t st) {
  auto kern = cg_gemm_tc_kernel<BN, AccT, PIECES>;
  const size_t smem = cg_smem(BN, PIECES);
  UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 g((M + kTcgM - 1) / kTcgM, (N + BN - 1) / BN, S);
  kern<<<g, kTcgThreads, smem, st>>>(A, sam, sak, Bm, sbk, sbn, M, N, K, kps, mode, bias, act, C, pre, part);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

// Whether the tensor-core path takes this GEMM: contiguous dimensions must allow float4 loads.
static bool cg_tc_ok(int64_t contig_a, int64_t contig_b) { return contig_a % 4 == 0 && contig_b % 4 == 0; }

int cg_tc_gemm(const float* A, int64_t sam, int64_t sak, const float* Bm, int64_t sbk, int64_t sbn, int64_t M,
               int64_t N, int64_t K, int mode, const float* bias, int act, float* C, float* pre, float* part,
               int S, int64_t kps, cudaStream_t st) {
  const int m = (int)M, n = (int)N, k = (int)K, kp = (int)kps;
  static const bool presplit = !(getenv("UKAN_CG_PRESPLIT") && getenv("UKAN_CG_PRESPLIT")[0] == '0');  // A/B only
  if (presplit && mode == 0 && act == 0 && S == 1 && sak == 1 && sbn == 1) {
    // table GEMM: split both operands once into contiguous canonical (tile, chunk) blocks, then
    // stream them with bulk copies (cg_table_tc_kernel, bitwise the same result)
    constexpr int BN = 128, NS = 3;  // measured: 0.83 ms at the cfg4 shape vs 0.89 ms for BN 64 x 2 stages x 2 CTAs/SM
    const int nch = (k + kTcgK - 1) / kTcgK;
    const int64_t mt = (M + kTcgM - 1) / kTcgM, ntl = (N + BN - 1) / BN;
    const size_t a_bytes = (size_t)mt * nch * 2 * kTcgM * kTcgK * 4, b_bytes = (size_t)ntl * nch * 2 * BN * kTcgK * 4;
    void* buf = nullptr;
    UKAN_CUDA_TRY(scratch_alloc(&buf, a_bytes + b_bytes, st));
    unsigned char* ap = static_cast<unsigned char*>(buf);
    unsigned char* bp = ap + a_bytes;
    const int64_t na = mt * nch * (kTcgM * kTcgK / 4), nb = ntl * nch * (BN * kTcgK / 4);
    cg_presplit_kernel<kTcgM><<<(unsigned)((na + 255) / 256), 256, 0, st>>>(A, sam, sak, m, k, nch, ap);
    UKAN_LAUNCH_CHECK();
    cg_presplit_kernel<BN><<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(Bm, sbn, sbk, n, k, nch, bp);
    UKAN_LAUNCH_CHECK();
    auto kern = cg_table_tc_kernel<BN, NS>;
    const size_t smem = std::max<size_t>((size_t)NS * 2 * (kTcgM + BN) * kTcgK * 4, (size_t)kTcgM * (BN + 1) * 4) + 1024;
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<dim3((unsigned)ntl, (unsigned)mt), kTcgThreads, smem, st>>>(ap, bp, m, n, nch, bias, C);
    UKAN_LAUNCH_CHECK();
    cudaFreeAsync(buf, st);
    return UKAN_OK;
  }
  // Only the table GEMM (mode 0, act 0) takes this path: its outputs feed the spline forward, where
  // fp32-level accuracy keeps parity — two tf32 pieces (3 products), fp32 promotion registers.
  static const int bn_env = getenv("UKAN_CG_BN") ? atoi(getenv("UKAN_CG_BN")) : 0;  // A/B measurement only
  if (bn_env == 64) return cg_launch<64, float, 2>(A, sam, sak, Bm, sbk, sbn, m, n, k, kp, S, mode, bias, act, C, pre, part, st);
  if (bn_env == 128) return cg_launch<128, float, 2>(A, sam, sak, Bm, sbk, sbn, m, n, k, kp, S, mode, bias, act, C, pre, part, st);
  if (N >= 256 && (M + kTcgM - 1) / kTcgM * (N / 256) >= kan_num_sms())
    return cg_launch<256, float, 2>(A, sam, sak, Bm, sbk, sbn, m, n, k, kp, S, mode, bias, act, C, pre, part, st);
  if (N > 64) return cg_launch<128, float, 2>(A, sam, sak, Bm, sbk, sbn, m, n, k, kp, S, mode, bias, act, C, pre, part, st);
  return cg_launch<64, float, 2>(A, sam, sak, Bm, sbk, sbn, m, n, k, kp, S, mode, bias, act, C, pre, part, st);
}

bool cg_tc_applicable(const void* a, const void* b, int64_t M, int64_t N, int64_t K, int64_t ca, int64_t cb) {
  static const bool off = getenv("UKAN_CG_CUDA_CORES") != nullptr;  // A/B measurement only
  const bool aligned = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0);  // 16-byte vector loads
  return !off && aligned && M > 0 && N > 0 && K > 0 && cg_tc_ok(ca, cb) && M <= INT32_MAX && N <= INT32_MAX &&
         K <= INT32_MAX;
}

int cg_colsum(const float* X, float* out, int64_t K, int64_t N, cudaStream_t st) {
  const bool v4 = (N % 4 == 0) && ((uintptr_t)X % 16 == 0);
  const int64_t cblk = v4 ? (N + 127) / 128 : (N + 31) / 32;
  const int S = (int)std::max<int64_t>(1, std::min<int64_t>((4 * kan_num_sms() + cblk - 1) / cblk, (K + 255) / 256));
  const int rps = (int)((K + S - 1) / S);
  void* part = nullptr;
  UKAN_CUDA_TRY(scratch_alloc(&part, sizeof(double) * S * N, st));
  if (v4)
    cg_colsum_part4_kernel<<<dim3((unsigned)cblk, S), 256, 0, st>>>(X, static_cast<double*>(part), (int)K, (int)N, rps);
  else
    cg_colsum_part_kernel<float><<<dim3((unsigned)cblk, S), 256, 0, st>>>(X, static_cast<double*>(part), (int)K, (int)N, rps);
  UKAN_LAUNCH_CHECK();
  cg_colsum_final_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(static_cast<double*>(part), out, (int)N, S);
  UKAN_LAUNCH_CHECK();
  cudaFreeAsync(part, st);
  return UKAN_OK;
}

int cg_colsum64(const double* X, float* out, int64_t K, int64_t N, cudaStream_t st) {
  const int64_t cblk = (N + 31) / 32;
  const int S = (int)std::max<int64_t>(1, std::min<int64_t>((4 * kan_num_sms() + cblk - 1) / cblk, (K + 255) / 256));
  const int rps = (int)((K + S - 1) / S);
  void* part = nullptr;
  UKAN_CUDA_TRY(scratch_alloc(&part, sizeof(double) * S * N, st));
  cg_colsum_part_kernel<double><<<dim3((unsigned)cblk, S), 256, 0, st>>>(X, static_cast<double*>(part), (int)K, (int)N, rps);
  UKAN_LAUNCH_CHECK();
  cg_colsum_final_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(static_cast<double*>(part), out, (int)N, S);
  UKAN_LAUNCH_CHECK();
  cudaFreeAsync(part, st);
  return UKAN_OK;
}

}  // namespace ukan

// ---------------------------------------------------------------------------------------
// Diagnostic (not on the product path): the weight-gradient GEMM C = A^T B (A [K,M], B [K,N])
// in the form SURVEY 8c C5 proposed for the CG gradients — tcgen05 kind::tf32 with 3-piece
// round-to-nearest operand splits (6 products), fp64 register promotion of every 32-wide K chunk,
// split-K over 4096-row slices with the fp32 slice results summed in fp64.  The product path runs
// these GEMMs on FP64 DMMA instead (cg_dmma.cu); tests/test_cg_tc.py measures both against an fp64
// reference on a K = 70k reduction to pin why (the tensor core's fp32 accumulator keeps ~22 bits).
// ---------------------------------------------------------------------------------------
namespace ukan {
__global__ void cg_probe_reduce_kernel(const float* __restrict__ part, float* __restrict__ C, int64_t MN, int S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= MN) return;
  double s = 0.0;
  for (int z = 0; z < S; ++z) s += (double)part[(size_t)z * MN + t];
  C[t] = (float)s;
}
}  // namespace ukan

extern "C" int ukan_gemm_tn_tf32x3_probe(const float* A, const float* Bm, float* C, int64_t M, int64_t N, int64_t K,
                                         void* stream) {
  using namespace ukan;
  if (M < 1 || N < 1 || K < 1 || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || !A || !Bm || !C) return UKAN_E_ARG;
  if (M % 4 || N % 4 || ((uintptr_t)A % 16) || ((uintptr_t)Bm % 16)) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t kps = 4096;
  const int S = (int)((K + kps - 1) / kps);
  void* part = nullptr;
  UKAN_CUDA_TRY(scratch_alloc(&part, sizeof(float) * (size_t)S * M * N, st));
  // A(m, k) = A[k*M + m] (sam = 1, sak = M); B(k, n) = B[k*N + n]
  int rc = N > 64 ? cg_launch<128, double, 3>(A, 1, M, Bm, N, 1, (int)M, (int)N, (int)K, (int)kps, S, 2, nullptr, 0,
                                              nullptr, nullptr, static_cast<float*>(part), st)
                  : cg_launch<64, double, 3>(A, 1, M, Bm, N, 1, (int)M, (int)N, (int)K, (int)kps, S, 2, nullptr, 0,
                                             nullptr, nullptr, static_cast<float*>(part), st);
  if (rc == UKAN_OK) {
    cg_probe_reduce_kernel<<<(unsigned)((M * N + 255) / 256), 256, 0, st>>>(static_cast<float*>(part), C, M * N, S);
    UKAN_LAUNCH_CHECK();
  }
  cudaFreeAsync(part, st);
  return rc;
}
