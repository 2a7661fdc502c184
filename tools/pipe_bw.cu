// Microbenchmarks for the KAN kernel design decisions (run on one B200):
//   TMEM read throughput (tcgen05.ld 32x32b.x64, warp-uniform data-dependent column),
//   shared-memory LDS.128 throughput (per-lane distinct and broadcast),
//   F2F.F64.F32 throughput alone and mixed with DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bw tools/pipe_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tmem_ld64(const int* __restrict__ cols, int iters, unsigned* out, long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int c = cols[(it + warp) & 255];
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 64; i += 8) acc ^= r[i] + r[i + 1] + r[i + 2] + r[i + 3] + r[i + 4] + r[i + 5] + r[i + 6] + r[i + 7];
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

template <bool BCAST>
__global__ void lds128(int iters, float* out, long long* cyc) {
  __shared__ float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 a = make_float4(0, 0, 0, 0);
  int idx = BCAST ? 0 : threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = buf[(idx + u * 32 + (it & 7) * 256) & 2047];
      a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + a.y + a.z + a.w;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>  // 0: F2F only, 1: DFMA only, 2: 1 F2F per 4 DFMA
__global__ void cvt(int iters, double* out, long long* cyc) {
  float f[8];
  double d[8];
  for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 0.1f + i; d[i] = i; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { d[i] += (double)f[i]; f[i] += 1.0f; }
      if (MODE == 1) d[i] = fma(d[i], 1.0000001, 0.5);
      if (MODE == 2) { d[i] = fma(d[i], 1.0000001, (double)f[i & 1]); d[i] = fma(d[i], 1.0000001, 0.5); d[i] = fma(d[i], 1.0000001, 0.25); d[i] = fma(d[i], 1.0000001, 0.125); }
    }
    if (MODE == 2) { f[0] += 1.0f; f[1] += 1.0f; }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int* cols;
  unsigned* ou;
  float* of;
  double* od;
  long long* cyc;
  cudaMalloc(&cols, 256 * 4);
  cudaMalloc(&ou, 148 * 1024 * 4);
  cudaMalloc(&of, 148 * 1024 * 4);
  cudaMalloc(&od, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  int h[256];
  unsigned s = 7;
  for (int i = 0; i < 256; ++i) { s = s * 1103515245u + 12345u; h[i] = (s >> 8) % (512 - 64); }
  cudaMemcpy(cols, h, sizeof h, cudaMemcpyHostToDevice);
  long long c;
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4000;
    tmem_ld64<<<148, warps * 32>>>(cols, iters, ou, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"tmem_ld_x64\", \"warps\": %d, \"B_per_clk_sm\": %.1f, \"err\": \"%s\"}\n", warps,
           (double)warps * iters * 32 * 64 * 4 / c, cudaGetErrorString(cudaGetLastError()));
  }
  for (int warps : {8, 16, 32}) {
    const int iters = 4000;
    lds128<false><<<148, warps * 32>>>(iters, of, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"lds128_lane\", \"warps\": %d, \"B_per_clk_sm\": %.1f}\n", warps, (double)warps * iters * 8 * 32 * 16 / c);
    lds128<true><<<148, warps * 32>>>(iters, of, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"lds128_bcast\", \"warps\": %d, \"warp_loads_per_clk_sm\": %.3f}\n", warps, (double)warps * iters * 8 / c);
  }
  for (int warps : {8, 16, 32}) {
    const int iters = 4000;
    cvt<0><<<148, warps * 32>>>(iters, od, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"f2f_f64_f32\", \"warps\": %d, \"per_clk_sm\": %.2f}\n", warps, (double)warps * iters * 8 * 32 / c);
    cvt<1><<<148, warps * 32>>>(iters, od, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"dfma\", \"warps\": %d, \"per_clk_sm\": %.2f}\n", warps, (double)warps * iters * 8 * 32 / c);
    cvt<2><<<148, warps * 32>>>(iters, od, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"bench\": \"dfma+f2f(1:16)\", \"warps\": %d, \"dfma_per_clk_sm\": %.2f}\n", warps, (double)warps * iters * 32 * 32 / c);
  }
  return 0;
}
