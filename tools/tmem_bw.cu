// TMEM load / store throughput microbenchmark (tcgen05.ld/st 32x32b.xN with a warp-uniform,
// data-dependent column) — decides whether TMEM can serve as the warp-uniform-indexed
// coefficient store of the KAN forward.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t a, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld4(uint32_t a, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st16(uint32_t a, const float (&v)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
               :: "r"(a), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
                 "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}

template <int MODE>
__global__ void bench(const int* __restrict__ cols, int iters, float* out, long long* cyc) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16);
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  // init
  if (warp < 4) for (int c = 0; c < 512; c += 16) st16(base + c, acc);
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int c = cols[(it * 4 + warp) & 1023];  // warp-uniform data-dependent column
    if (MODE == 0) {
      float v[16];
      ld16(base + c, v);
      const float w = 1.0001f;
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(w, v[i], acc[i]);
    } else if (MODE == 1) {
      float v[4];
      ld4(base + c, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = fmaf(1.0001f, v[i], acc[i]);
    } else if (MODE == 2) {
      float v[16];
      ld16(base + c, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = fmaf(1.0001f, acc[i], v[i]);
      st16(base + c, v);
    } else {  // pure FFMA reference: 16 dependent-free FMAs per iter
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(1.0001f, acc[i], (float)c);
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
}

int main() {
  int* cols;
  float* out;
  long long* cyc;
  cudaMalloc(&cols, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  int h[1024];
  unsigned s = 1;
  for (int i = 0; i < 1024; ++i) { s = s * 1103515245u + 12345u; h[i] = (s >> 8) % (512 - 16); }
  cudaMemcpy(cols, h, sizeof h, cudaMemcpyHostToDevice);
  const int iters = 20000;
  const char* names[] = {"ld.x16+16ffma", "ld.x4+4ffma", "ld.x16+16ffma+st.x16", "16ffma only"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      void (*k)(const int*, int, float*, long long*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : bench<3>;
      k<<<148, warps * 32>>>(cols, iters, out, cyc);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<148, warps * 32>>>(cols, iters, out, cyc);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const int words = mode == 1 ? 4 : 16;
      const double bytes_per_cyc = (double)warps * iters * 32 * words * 4 / c * (mode == 3 ? 0 : 1);
      const double fma_per_cyc = (double)warps * iters * 32 * words / c;
      printf("{\"mode\": \"%s\", \"warps\": %d, \"cycles\": %lld, \"ms\": %.3f, \"tmem_read_B_per_clk_sm\": %.1f, \"ffma_per_clk_sm\": %.1f, \"err\": \"%s\"}\n",
             names[mode], warps, c, ms, bytes_per_cyc, fma_per_cyc, cudaGetErrorString(e));
    }
  }
  return 0;
}
