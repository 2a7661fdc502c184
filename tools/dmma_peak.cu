// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput microbenchmark, plus a corrected
// LDS.128 bandwidth test (dependent addresses so nothing can be hoisted).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void lds128_dep(float* out, int iters) {
  __shared__ float4 t[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = make_float4(0, 0, 0, 0);
  __syncthreads();
  int idx0 = threadIdx.x & 2047, idx1 = (threadIdx.x + 512) & 2047, idx2 = (threadIdx.x + 1024) & 2047,
      idx3 = (threadIdx.x + 1536) & 2047;
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    float4 v0 = t[idx0], v1 = t[idx1], v2 = t[idx2], v3 = t[idx3];
    // next addresses depend on loaded data (always 0) -> loads cannot be hoisted / merged
    idx0 = (idx0 + 32 + __float_as_int(v0.x)) & 2047;
    idx1 = (idx1 + 32 + __float_as_int(v1.y)) & 2047;
    idx2 = (idx2 + 32 + __float_as_int(v2.z)) & 2047;
    idx3 = (idx3 + 32 + __float_as_int(v3.w)) & 2047;
    acc += v0.w + v1.x + v2.y + v3.z;
  }
  if (acc == 1.5f) out[0] = acc;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* od; cudaMalloc(&od, 64);
  float* of; cudaMalloc(&of, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    int iters = 4000;
    dmma_loop<<<sms * 2, wpb * 32>>>(od, 10);
    cudaEventRecord(a); dmma_loop<<<sms * 2, wpb * 32>>>(od, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 256 * 8 * iters * (double)sms * 2 * wpb;
    printf("{\"dmma_tflops\": %.2f, \"warps_per_cta\": %d}\n", flops / ms / 1e9, wpb);
  }
  for (int thr : {256, 512, 1024}) {
    int iters = 20000;
    lds128_dep<<<sms * 2, thr>>>(of, 10);
    cudaEventRecord(a); lds128_dep<<<sms * 2, thr>>>(of, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 16.0 * 4 * iters * (double)sms * 2 * thr;
    printf("{\"lds128_TBps\": %.2f, \"bytes_per_clk_per_sm\": %.1f, \"threads\": %d}\n", bytes / ms / 1e9,
           bytes / (ms * 1e-3) / sms / (p.clockRate * 1e3), thr);
  }
  return 0;
}
