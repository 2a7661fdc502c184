// Micro-benchmarks for the CUDA-core roofs the KAN kernels are bound by:
// FP32 FMA, FP64 FMA, shared-memory gather (LDS.32 distinct banks), LDS.128.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int N>
__global__ void fma32(float* out, int iters, float a, float b) {
  float r[N];
  #pragma unroll
  for (int i = 0; i < N; i++) r[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < N; i++) r[i] = fmaf(r[i], a, b);
  }
  float s = 0; 
  #pragma unroll
  for (int i = 0; i < N; i++) s += r[i];
  if (s == 12345.f) out[0] = s;
}
template<int N>
__global__ void fma64(double* out, int iters, double a, double b) {
  double r[N];
  #pragma unroll
  for (int i = 0; i < N; i++) r[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int i = 0; i < N; i++) r[i] = fma(r[i], a, b);
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < N; i++) s += r[i];
  if (s == 12345.0) out[0] = s;
}
// smem gather: each lane reads a pseudo-random word from a 16K-float table
__global__ void lds_gather(float* out, int iters) {
  __shared__ float t[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) t[i] = i;
  __syncthreads();
  unsigned idx = threadIdx.x * 2654435761u;
  float acc = 0;
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int u = 0; u < 8; u++) {
      unsigned k = (idx + u * 97 + it * 31) & 8191;
      acc += t[k];
    }
  }
  if (acc == 1.5f) out[0] = acc;
}
__global__ void lds128(float* out, int iters) {
  __shared__ float4 t[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 acc = make_float4(0,0,0,0);
  for (int it = 0; it < iters; it++) {
    #pragma unroll
    for (int u = 0; u < 8; u++) {
      float4 v = t[(threadIdx.x + u * 32 + it * 64) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.5f) out[0] = 1;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  float* o; CK(cudaMalloc(&o, 64)); double* od; CK(cudaMalloc(&od, 64));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  // FP32: 1024 threads/block * 4 blocks/SM, 16 independent chains
  { int iters = 20000; dim3 g(sms * 4), bl(512);
    fma32<16><<<g, bl>>>(o, 100, 1.0001f, 0.5f);
    cudaEventRecord(a); fma32<16><<<g, bl>>>(o, iters, 1.0001f, 0.5f); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 16 * iters * (double)g.x * bl.x;
    printf(", \"fp32_tflops\": %.2f", fl / ms / 1e9); }
  { int iters = 10000; dim3 g(sms * 4), bl(512);
    fma64<8><<<g, bl>>>(od, 100, 1.0001, 0.5);
    cudaEventRecord(a); fma64<8><<<g, bl>>>(od, iters, 1.0001, 0.5); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * iters * (double)g.x * bl.x;
    printf(", \"fp64_tflops\": %.2f", fl / ms / 1e9); }
  { int iters = 4000; dim3 g(sms * 2), bl(1024);
    lds_gather<<<g, bl>>>(o, 10);
    cudaEventRecord(a); lds_gather<<<g, bl>>>(o, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double words = 8.0 * iters * (double)g.x * bl.x;
    printf(", \"lds32_random_words_per_clk_per_sm\": %.2f, \"lds32_gwords_s\": %.1f", words / (ms * 1e-3) / sms / (p.clockRate * 1e3), words / ms / 1e6); }
  { int iters = 4000; dim3 g(sms * 2), bl(1024);
    lds128<<<g, bl>>>(o, 10);
    cudaEventRecord(a); lds128<<<g, bl>>>(o, iters); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 16.0 * 8 * iters * (double)g.x * bl.x;
    printf(", \"lds128_TBps\": %.2f", bytes / ms / 1e9); }
  printf(", \"clock_rate_mhz\": %d}\n", p.clockRate / 1000);
  return 0;
}
