// kan_fwd_tm.cu — KAN forward with the coefficient slab held in Tensor Memory (TMEM).
//
// Replaces kan_forward (layers.py:304-318) = _kan_locate (294-301) + span_gather (57-75) +
// basis_features (40-54) + edge_combine (78-105), fused:
//     y[b,o] = sum_i sum_j w_j(u_bi) * C'[i, cell_bi + j, o],     C' = scale (x) C   (fp32)
// (scale folded into the coefficients once per CTA; SURVEY 8d D2 counts the same K FMAs).
//
// Why TMEM.  The gather is the whole cost: every FMA needs a different coefficient, chosen by
// the sample's cell.  A thread owning outputs o needs C'[i, cell..cell+K-1, o] for each
// (sample, feature); the cell is the same for all lanes of a warp (lanes = outputs), i.e. the
// gather is a *warp-uniform, data-dependent column index* into a per-lane array — exactly what
// `tcgen05.ld.32x32b` does from TMEM: lane L reads its own TMEM lane, columns [col, col+N)
// with `col` in a register.  TMEM feeds ~410 B/clk/SM into the register file (measured,
// tools/pipe_bw.cu) against 128 B/clk for lane-distinct shared-memory loads, which bound the
// previous shared-memory gather (spline_fwd_kernel) at 25% of FP32 peak.
//
// CTA (16 warps, 1 per SM: all 512 TMEM columns): OT = 256 outputs x ST = 128 samples.
//   TMEM lane L holds outputs o0 + (L mod LO)*OV .. +OV-1 (LO = 256/OV lanes per copy; with
//   OV = 4 the 128 lanes hold two copies and the two lane halves serve different samples),
//   column (f*RP + r)*OV + v = C'[i_f, r, o] for the F features of one pipeline stage;
//   two stages (double buffer).  Warp (quarter q, sub-warp ws) owns SW samples x OV outputs
//   per lane as fp32 accumulators in registers (statically indexed).
// Pipeline per stage g (one __syncthreads):
//   cp.async  C[i, :, o0:o0+OT] + scale rows of stage g+2 -> shared slab buffer
//   records   fp64 locate (reference expression order) + fp64 basis -> (column, w fp32) of
//             stage g+1, one thread per (sample, feature); x prefetched a stage ahead
//   fill      slab of stage g+1 (landed last stage) * scale -> TMEM buffer (g+1)&1 (tcgen05.st)
//   compute   stage g: per (sample, feature) one tcgen05.ld of the K*OV window + K*OV FFMA
// Deterministic: each y[b,o] is summed by one thread in feature order; d_in splits (for grid
// fill) are reduced in fixed order.
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace ukan {

constexpr int kTmWarpsQ = 4;                // warps per TMEM lane quarter
constexpr int kTmThreads = 4 * kTmWarpsQ * 32;
constexpr int kTmOT = 256;                  // outputs per CTA
constexpr int kTmST = 128;                  // samples per CTA

// ---- TMEM access (PTX tcgen05, sm_100a) ------------------------------------------------
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t taddr, float (&v)[N]);

template <>
__device__ __forceinline__ void tm_ld<2>(uint32_t a, float (&v)[2]) {
  uint32_t r[2];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(a));
  v[0] = __uint_as_float(r[0]);
  v[1] = __uint_as_float(r[1]);
}
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t a, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t a, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t a, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tm_ld<32>(uint32_t a, float (&v)[32]) {
  tm_ld<16>(a, reinterpret_cast<float(&)[16]>(v[0]));
  tm_ld<16>(a + 16, reinterpret_cast<float(&)[16]>(v[16]));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tm_st4(uint32_t a, float4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

constexpr int tm_pow2ceil(int n) { return n <= 1 ? 1 : 2 * tm_pow2ceil((n + 1) / 2); }

// ---- async-proxy helpers: mbarrier, 1-D TMA bulk copy, tcgen05.cp -----------------------
__device__ __forceinline__ void mb_init(uint64_t* mb, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* mb, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mb)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* mb, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mb);
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(mb))
               : "memory");
}
// Coefficient pack (once per forward): Cp[ot][i][r][256] = scale[i,o] * C[i,r,o], zero for
// r >= R or o >= d_out.  Each (o-tile, feature) slab is then one contiguous RP KB block, so a
// stage is a single 1-D TMA bulk copy, and each lane's 16 bytes of a row are contiguous.
// seg != nullptr (dense UKAN layer): feature i's R rows are rows [4 seg[i], 4 seg[i+1]) of the
// generated table (zero past the segment) instead of C[i].
__global__ void kan_pack_coeffs_kernel(const float* __restrict__ C, const float* __restrict__ scale,
                                       float4* __restrict__ Cp, int d_in, int R, int RP, int d_out, int n_ot,
                                       const int32_t* __restrict__ seg = nullptr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)n_ot * d_in * RP * (kTmOT / 4);
  if (t >= n) return;
  const int q = (int)(t % (kTmOT / 4));
  int64_t rest = t / (kTmOT / 4);
  const int r = (int)(rest % RP);
  rest /= RP;
  const int i = (int)(rest % d_in);
  const int ot = (int)(rest / d_in);
  float v[4];
  const int rbase = seg ? 4 * seg[i] : i * R, nr = seg ? 4 * (seg[i + 1] - seg[i]) : R;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int o = ot * kTmOT + q * 4 + e;
    v[e] = (r < nr && o < d_out) ? C[((size_t)rbase + r) * d_out + o] * scale[(size_t)i * d_out + o] : 0.f;
  }
  Cp[t] = make_float4(v[0], v[1], v[2], v[3]);
}

// Per-(feature, sample) records, feature-major so one stage's records are contiguous:
//   cell[i][b] (u8) and w[i][b][KP] (fp32, from the fp64 basis) — fp64 locate with the
//   reference's expression order (layers.py:299-300).  NaN input sets *err (the reference
//   raises IndexError, SURVEY gotcha 10) and contributes nothing.
// UK (dense UKAN layer): the cell is the window start inside the feature's table segment,
// base_row[b, i] - 4 seg[i], and u = x/dg - floor(x/dg) (layers.py:261-264).
template <int K, bool UK = false>
__global__ void __launch_bounds__(256)
kan_fwd_records_kernel(const float* __restrict__ x, uint8_t* __restrict__ cell_out, float* __restrict__ w_out, int B,
                       int Bp, int d_in, KanGrid grid, Basis<K> bas, int32_t* __restrict__ err,
                       const int32_t* __restrict__ base_row = nullptr, const int32_t* __restrict__ seg = nullptr) {
  constexpr int KP = (K + 3) / 4 * 4;
  __shared__ float xs[32][33];  // 32 samples x 32 features, transposed through shared memory
  const int b0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, i = i0 + tx;
    xs[r][tx] = (b < B && i < d_in) ? x[(size_t)b * d_in + i] : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {  // feature i0 + r, sample b0 + tx
    const int i = i0 + r, b = b0 + tx;
    if (i >= d_in || b >= B) continue;
    int cell = 0;
    float wf[KP];
#pragma unroll
    for (int j = 0; j < KP; ++j) wf[j] = 0.f;
    double u;
    bool mask;
    bool ok;
    if constexpr (UK) {
      int64_t gid;
      ukan_locate(xs[tx][r], grid.inv_dg, gid, u);
      cell = base_row[(size_t)b * d_in + i] - 4 * seg[i];
      ok = cell >= 0 && cell < grid.G && u == u;
    } else {
      ok = kan_locate(xs[tx][r], grid, cell, u, mask);
    }
    if (ok) {
      double w[K];
      basis_weights<K>(bas, u, w);
#pragma unroll
      for (int j = 0; j < K; ++j) wf[j] = (float)w[j];
    } else {
      cell = 0;
      if (err) atomicExch(err, 1);
    }
    const size_t o = (size_t)i * Bp + b;
    cell_out[o] = (uint8_t)cell;
#pragma unroll
    for (int j = 0; j < KP; j += 4) *reinterpret_cast<float4*>(w_out + o * KP + j) = make_float4(wf[j], wf[j + 1], wf[j + 2], wf[j + 3]);
  }
}

constexpr int kTmSDepth = 5;  // shared-memory ring: TMA loads run up to 3 stages ahead

// K basis weights, SW samples per warp, 4 outputs per lane (OV = 4: TMEM lanes L and L+64
// hold the same outputs; the two lane halves serve different samples).  Stage g = feature
// i_lo + g.  Thread 0 streams the packed slab + records of future stages into a 5-deep
// shared ring with 1-D TMA bulk copies (mbarriers full/empty).  Each warp copies its rows of
// the next stage's slab into its own TMEM lane quarter (tcgen05.st; the async tcgen05.cp was
// measured at ~6 B/clk for this shape) and computes the current stage: per sample one
// tcgen05.ld of the K*4-word window + K*4 FFMA.  The only barrier per stage is a 4-warp
// named barrier per lane quarter (TMEM double buffer).
// DEPTH: shared-memory ring depth (5, or 3 when the slabs of finer grids do not fit five times);
// DB: two TMEM slab buffers (the next feature's fill overlaps this feature's gathers) when two
// slabs of RP x 4 columns fit the 512 TMEM columns, else one buffer refilled after a barrier.
// MC: a cluster of two CTAs (adjacent sample tiles of one output tile) shares each coefficient
// slab: each CTA streams half of it with a multicast bulk copy into both CTAs' rings (half the
// L2 -> SM slab traffic); a stage is refilled once the consumers of BOTH CTAs released it (every
// warp arrives on its own and the peer's `empty` barrier).
template <int K, int SW, int DEPTH, bool DB, bool MC = false>
__global__ void __launch_bounds__(kTmThreads, 1)
kan_fwd_tm_kernel(const float* __restrict__ Cp, const uint8_t* __restrict__ rc, const float* __restrict__ rw,
                  float* __restrict__ y, int B, int Bp, int d_in, int d_out, int RP, int fpc) {
  constexpr int OV = 4;
  constexpr int NW = tm_pow2ceil(K * OV);
  constexpr int KP = (K + 3) / 4 * 4;
  constexpr int LO = kTmOT / OV;  // 64 output slots
  constexpr int NWARP = kTmThreads / 32;
  static_assert(2 * kTmWarpsQ * SW == kTmST && SW % 4 == 0, "tile shape");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t full_s[DEPTH], empty_s[DEPTH];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, ws = warp >> 2;
  const int L = 32 * q + lane;
  const int slot = L % LO, cg = L / LO;
  const int ot = blockIdx.y;
  const int b0 = blockIdx.x * kTmST;
  const int i_lo = blockIdx.z * fpc, i_hi = min(d_in, i_lo + fpc);
  const int nstage = i_hi - i_lo;
  const bool producer = threadIdx.x == 0;
  const uint32_t slab_bytes = (uint32_t)RP * kTmOT * 4;
  const uint32_t recw_bytes = (uint32_t)kTmST * KP * 4;
  const uint32_t buf_bytes = slab_bytes + recw_bytes + kTmST;  // slab | w records | cells

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  uint32_t crank = 0;
  if constexpr (MC) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
  if (producer) {
    for (int d = 0; d < DEPTH; ++d) {
      mb_init(&full_s[d], 1);
      mb_init(&empty_s[d], MC ? 2 * NWARP : NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const float* cp_ot = Cp + (size_t)ot * d_in * RP * kTmOT;
  auto buf_ptr = [&](int g) { return smem_raw + (size_t)(g % DEPTH) * buf_bytes; };
  auto issue_loads = [&](int g) {  // slab + records of stage g -> shared buffer g % 5
    unsigned char* d = buf_ptr(g);
    const int i = i_lo + g;
    uint64_t* mb = &full_s[g % DEPTH];
    mb_expect_tx(mb, buf_bytes);
    if constexpr (MC) {  // this CTA's half of the slab, into both CTAs (same offsets, same barrier)
      const uint32_t half = slab_bytes / 2;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;\n" ::"r"(
              (uint32_t)__cvta_generic_to_shared(d + crank * half)),
          "l"(reinterpret_cast<const unsigned char*>(cp_ot + (size_t)i * RP * kTmOT) + crank * half), "r"(half),
          "r"((uint32_t)__cvta_generic_to_shared(mb)), "h"((unsigned short)3)
          : "memory");
    } else {
      bulk_g2s(d, cp_ot + (size_t)i * RP * kTmOT, slab_bytes, mb);
    }
    bulk_g2s(d + slab_bytes, rw + ((size_t)i * Bp + b0) * KP, recw_bytes, mb);
    bulk_g2s(d + slab_bytes + recw_bytes, rc + (size_t)i * Bp + b0, kTmST, mb);
  };
  int next_load = 0;
  auto pump = [&](int upto) {  // loads for stages < upto whose buffer has been released
    for (; next_load < min(upto, nstage); ++next_load) {
      const int g = next_load;
      if (g >= DEPTH) mb_wait(&empty_s[g % DEPTH], (uint32_t)(((g - DEPTH) / DEPTH) & 1));
      issue_loads(g);
    }
  };

  float2 acc2[SW][OV / 2];
#pragma unroll
  for (int s = 0; s < SW; ++s)
#pragma unroll
    for (int v = 0; v < OV / 2; ++v) acc2[s][v] = make_float2(0.f, 0.f);

  tm_fence_before();
  if constexpr (MC) {  // both CTAs' barriers initialised before any multicast / remote arrive
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();  // TMEM address + mbarrier init visible
  }
  tm_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t tl = tbase + ((uint32_t)(32 * q) << 16);
  const int qbar = 1 + q;  // named barrier of this lane quarter (4 warps)
  // this warp's rows of a slab -> TMEM buffer (g & 1), lanes of its quarter
  auto fill = [&](int g) {
    const float4* src = reinterpret_cast<const float4*>(buf_ptr(g)) + slot;
    const uint32_t cbase = tl + (uint32_t)((DB ? (g & 1) : 0) * RP * OV);
    for (int r = ws; r < RP; r += kTmWarpsQ) tm_st4(cbase + (uint32_t)(r * OV), src[(size_t)r * (kTmOT / 4)]);
  };
  if (producer) pump(DEPTH - 1);
  __syncwarp();
  if (nstage > 0) {
    mb_wait(&full_s[0], 0);
    fill(0);
  }
  tm_wait_st();
  tm_fence_before();
  asm volatile("bar.sync %0, %1;\n" ::"r"(qbar), "r"(kTmWarpsQ * 32) : "memory");
  tm_fence_after();

  const int sb = (cg * kTmWarpsQ + ws) * SW;
  for (int g = 0; g < nstage; ++g) {
    const int ds = g % DEPTH;
    if (producer) pump(g + DEPTH - 1);
    __syncwarp();
    if (DB && g + 1 < nstage) {  // stage g+1 -> the other TMEM buffer (freed by the last quarter barrier)
      mb_wait(&full_s[(g + 1) % DEPTH], (uint32_t)(((g + 1) / DEPTH) & 1));
      fill(g + 1);
    }
    const unsigned char* bp = buf_ptr(g);  // stage g landed: waited before its fill
    const float* wr = reinterpret_cast<const float*>(bp + slab_bytes) + (size_t)sb * KP;
    const uint8_t* cr = bp + slab_bytes + recw_bytes + sb;
    const uint32_t tcol = tl + (uint32_t)((DB ? (g & 1) : 0) * RP * OV);
    // two samples per TMEM wait; the cells of four samples come in one 32-bit load
#pragma unroll
    for (int s = 0; s < SW; s += 4) {
      const uint32_t c4 = *reinterpret_cast<const uint32_t*>(cr + s);
#pragma unroll
      for (int h = 0; h < 4; h += 2) {
        float c0[NW], c1[NW];
        tm_ld<NW>(tcol + ((c4 >> (8 * h)) & 0xffu) * OV, c0);
        tm_ld<NW>(tcol + ((c4 >> (8 * h + 8)) & 0xffu) * OV, c1);
        float w0[KP], w1[KP];
#pragma unroll
        for (int j = 0; j < KP; j += 4) {
          const float4 a = *reinterpret_cast<const float4*>(wr + (size_t)(s + h) * KP + j);
          const float4 b = *reinterpret_cast<const float4*>(wr + (size_t)(s + h + 1) * KP + j);
          w0[j] = a.x; w0[j + 1] = a.y; w0[j + 2] = a.z; w0[j + 3] = a.w;
          w1[j] = b.x; w1[j + 1] = b.y; w1[j + 2] = b.z; w1[j + 3] = b.w;
        }
        tm_wait_ld();
        // packed FFMA2 over output pairs: each lane of the pair is an IEEE fma, bitwise equal to
        // two fmaf, at half the issue slots
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const float2 a0 = make_float2(w0[j], w0[j]), a1 = make_float2(w1[j], w1[j]);
#pragma unroll
          for (int v = 0; v < OV; v += 2) {
            acc2[s + h][v / 2] = __ffma2_rn(a0, make_float2(c0[j * OV + v], c0[j * OV + v + 1]), acc2[s + h][v / 2]);
            acc2[s + h + 1][v / 2] = __ffma2_rn(a1, make_float2(c1[j * OV + v], c1[j * OV + v + 1]), acc2[s + h + 1][v / 2]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {  // done with stage g's shared buffer (slab copied into TMEM, records read)
      const uint32_t ea = (uint32_t)__cvta_generic_to_shared(&empty_s[ds]);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(ea) : "memory");
      if constexpr (MC) {  // ... and the peer's: its next multicast into this CTA's buffer waits on it
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(ea), "r"(crank ^ 1u));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra) : "memory");
      }
    }
    tm_wait_st();
    tm_fence_before();
    asm volatile("bar.sync %0, %1;\n" ::"r"(qbar), "r"(kTmWarpsQ * 32) : "memory");
    tm_fence_after();
    if (!DB && g + 1 < nstage) {  // single TMEM buffer: refill after every warp of the quarter is done
      mb_wait(&full_s[(g + 1) % DEPTH], (uint32_t)(((g + 1) / DEPTH) & 1));
      fill(g + 1);
      tm_wait_st();
      tm_fence_before();
      asm volatile("bar.sync %0, %1;\n" ::"r"(qbar), "r"(kTmWarpsQ * 32) : "memory");
      tm_fence_after();
    }
  }

  // epilogue: y (or this split's partial) for SW samples x OV outputs
  const int o = ot * kTmOT + slot * OV;
  float* out = y + (size_t)blockIdx.z * B * d_out;
#pragma unroll
  for (int s = 0; s < SW; ++s) {
    const int b = b0 + sb + s;
    if (b >= B) continue;
    float* yr = out + (size_t)b * d_out + o;
    const float av[OV] = {acc2[s][0].x, acc2[s][0].y, acc2[s][1].x, acc2[s][1].y};
    if (o + OV <= d_out && (d_out % OV) == 0) {
      *reinterpret_cast<float4*>(yr) = make_float4(av[0], av[1], av[2], av[3]);
    } else {
#pragma unroll
      for (int v = 0; v < OV; ++v)
        if (o + v < d_out) yr[v] = av[v];
    }
  }
  tm_fence_before();
  if constexpr (MC) {  // the peer may still arrive on this CTA's barriers until it is done
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
  tm_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

// y = sum over the d_in splits of the partials, fixed order (deterministic).
__global__ void kan_fwd_split_reduce_kernel(const float* __restrict__ part, float* __restrict__ y, int64_t n,
                                            int S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float a = part[t];
  for (int s = 1; s < S; ++s) a += part[(size_t)s * n + t];
  y[t] = a;
}

// ---------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------
int kan_num_sms();

struct TmPlan {
  bool ok = false;
  int RP = 0, fpc = 0, S = 1, n_ot = 0, Bp = 0;
  size_t smem = 0;
  int64_t pack_bytes = 0, rec_bytes = 0, part_bytes = 0;
  int depth = kTmSDepth, db = 1;
};

TmPlan kan_fwd_tm_plan(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k, bool has_base) {
  TmPlan p;
  const int K = k + 1;
  if (has_base || K > 8 || B < 1 || G < 1 || G > 255 || d_out < 128) return p;  // narrow layers: TMEM lanes idle
  int nw = 1;
  while (nw < K * 4) nw *= 2;
  if (nw > 32) return p;
  const int rp = (int)(G - 1) + nw / 4;  // rows reachable by a window load
  if (rp * 4 > 512) return p;     // one stage of one feature must fit TMEM
  const int KP = (K + 3) / 4 * 4;
  p.RP = rp;
  const size_t per = (size_t)rp * kTmOT * 4 + (size_t)kTmST * KP * 4 + kTmST;
  p.depth = (size_t)kTmSDepth * per <= 220 * 1024 ? kTmSDepth : 3;
  // two TMEM stages (the next fill overlaps the gathers) need two slabs in TMEM and the deep ring
  // (with a 3-deep ring the early fill waits on its TMA load: G=48 measured 10.1 ms double- vs
  // 8.9 ms single-buffered at B=16384, 1024->1024, slower than G=64 single-buffered)
  p.db = (2 * rp * 4 <= 512 && p.depth == kTmSDepth) ? 1 : 0;
  p.smem = (size_t)p.depth * per;
  if (p.smem > 220 * 1024) return p;
  p.n_ot = (int)((d_out + kTmOT - 1) / kTmOT);
  static const bool mc = getenv("UKAN_FWD_MC") && getenv("UKAN_FWD_MC")[0] == '1';  // cluster pairs: even tile count
  const int tile = mc ? 2 * kTmST : kTmST;
  p.Bp = (int)((B + tile - 1) / tile * tile);
  const int64_t tiles = (p.Bp / kTmST) * (int64_t)p.n_ot;
  const int sms = kan_num_sms();
  int64_t S = 1;  // split d_in so the grid fills the SMs without a partial second wave
  if (tiles < sms) S = std::min<int64_t>(sms / tiles, std::max<int64_t>(1, d_in / 16));
  p.fpc = (int)((d_in + S - 1) / S);
  p.S = (int)((d_in + p.fpc - 1) / p.fpc);
  p.pack_bytes = (int64_t)sizeof(float) * p.n_ot * d_in * rp * kTmOT;
  p.rec_bytes = (int64_t)d_in * p.Bp * (KP * 4 + 1);
  p.part_bytes = p.S > 1 ? (int64_t)sizeof(float) * p.S * B * d_out : 0;
  p.ok = true;
  return p;
}

static int64_t al256(int64_t n) { return (n + 255) / 256 * 256; }
int64_t kan_fwd_tm_workspace(const TmPlan& p) {
  return p.ok ? al256(p.pack_bytes) + al256(p.rec_bytes) + p.part_bytes : 0;
}

template <int K>
static int launch_tm(const float* x, const float* C, const float* scale, float* y, void* ws, int B, int d_in,
                     int d_out, int R, const KanGrid& grid, const TmPlan& p, int32_t* err, cudaStream_t st,
                     const int32_t* base_row = nullptr, const int32_t* seg = nullptr) {
  constexpr int SW = kTmST / (2 * kTmWarpsQ);
  constexpr int KP = (K + 3) / 4 * 4;
  char* w8 = static_cast<char*>(ws);
  float* Cp = reinterpret_cast<float*>(w8);
  float* recw = reinterpret_cast<float*>(w8 + al256(p.pack_bytes));
  uint8_t* recc = reinterpret_cast<uint8_t*>(recw) + (size_t)d_in * p.Bp * KP * 4;
  float* part = reinterpret_cast<float*>(w8 + al256(p.pack_bytes) + al256(p.rec_bytes));
  const int64_t npack = (int64_t)p.n_ot * d_in * p.RP * (kTmOT / 4);
  kan_pack_coeffs_kernel<<<(unsigned)((npack + 255) / 256), 256, 0, st>>>(C, scale, reinterpret_cast<float4*>(Cp),
                                                                         d_in, R, p.RP, d_out, p.n_ot, seg);
  UKAN_LAUNCH_CHECK();
  if (p.Bp > B) UKAN_CUDA_TRY(cudaMemsetAsync(recw, 0, p.rec_bytes, st));  // padding samples: zero weights
  if (seg != nullptr) {
    if constexpr (K == 4)
      kan_fwd_records_kernel<K, true><<<dim3((B + 31) / 32, (d_in + 31) / 32), 256, 0, st>>>(
          x, recc, recw, B, p.Bp, d_in, grid, make_basis<K>(K - 1), err, base_row, seg);
  } else {
    kan_fwd_records_kernel<K><<<dim3((B + 31) / 32, (d_in + 31) / 32), 256, 0, st>>>(x, recc, recw, B, p.Bp, d_in,
                                                                                     grid, make_basis<K>(K - 1), err);
  }
  UKAN_LAUNCH_CHECK();
  dim3 gridd(p.Bp / kTmST, p.n_ot, p.S);
  float* out = p.S > 1 ? part : y;
  static const bool mc = getenv("UKAN_FWD_MC") && getenv("UKAN_FWD_MC")[0] == '1';  // A/B
  if (mc) {
    auto kern = p.depth == kTmSDepth
                    ? (p.db ? kan_fwd_tm_kernel<K, SW, kTmSDepth, true, true> : kan_fwd_tm_kernel<K, SW, kTmSDepth, false, true>)
                    : (p.db ? kan_fwd_tm_kernel<K, SW, 3, true, true> : kan_fwd_tm_kernel<K, SW, 3, false, true>);
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = gridd;
    cfg.blockDim = dim3(kTmThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    UKAN_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, (const float*)Cp, (const uint8_t*)recc, (const float*)recw, out, B,
                                     p.Bp, d_in, d_out, p.RP, p.fpc));
  } else {
    auto kern = p.depth == kTmSDepth ? (p.db ? kan_fwd_tm_kernel<K, SW, kTmSDepth, true> : kan_fwd_tm_kernel<K, SW, kTmSDepth, false>)
                                      : (p.db ? kan_fwd_tm_kernel<K, SW, 3, true> : kan_fwd_tm_kernel<K, SW, 3, false>);
    UKAN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    kern<<<gridd, kTmThreads, p.smem, st>>>(Cp, recc, recw, out, B, p.Bp, d_in, d_out, p.RP, p.fpc);
  }
  UKAN_LAUNCH_CHECK();
  if (p.S > 1) {
    const int64_t n = (int64_t)B * d_out;
    kan_fwd_split_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, y, n, p.S);
    UKAN_LAUNCH_CHECK();
  }
  return UKAN_OK;
}

template <int K>
int kan_fwd_tm_run(const float* x, const float* C, const float* scale, float* y, void* ws, int64_t ws_bytes, int B,
                   int d_in, int d_out, int R, const KanGrid& grid, const TmPlan& p, int32_t* err, cudaStream_t st) {
  if (!p.ok || ws == nullptr || ws_bytes < kan_fwd_tm_workspace(p)) return UKAN_E_WORKSPACE;
  if constexpr (K <= 8) return launch_tm<K>(x, C, scale, y, ws, B, d_in, d_out, R, grid, p, err, st);
  return UKAN_E_ARG;
}

// Dense UKAN layer (every feature's table segment <= G + 3 rows): the same TMEM forward over the
// segments of the generated table (cubic only).
int kan_fwd_tm_run_ukan(const float* x, const float* T, const float* scale, float* y, void* ws, int64_t ws_bytes,
                        int B, int d_in, int d_out, int G, double inv_dg, const int32_t* base_row, const int32_t* seg,
                        const TmPlan& p, cudaStream_t st) {
  if (!p.ok || ws == nullptr || ws_bytes < kan_fwd_tm_workspace(p)) return UKAN_E_WORKSPACE;
  KanGrid grid{};
  grid.inv_dg = inv_dg;
  grid.G = G;
  return launch_tm<4>(x, T, scale, y, ws, B, d_in, d_out, G + 3, grid, p, nullptr, st, base_row, seg);
}

#define UKAN_TM_INST(K)                                                                                          \
  template int kan_fwd_tm_run<K>(const float*, const float*, const float*, float*, void*, int64_t, int, int, int, \
                                 int, const KanGrid&, const TmPlan&, int32_t*, cudaStream_t);
UKAN_TM_INST(1) UKAN_TM_INST(2) UKAN_TM_INST(3) UKAN_TM_INST(4) UKAN_TM_INST(5) UKAN_TM_INST(6)
UKAN_TM_INST(7) UKAN_TM_INST(8) UKAN_TM_INST(9) UKAN_TM_INST(10) UKAN_TM_INST(11)

}  // namespace ukan
