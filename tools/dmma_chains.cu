// DMMA throughput vs independent accumulator chains per warp (16 warps per SM, one CTA per SM):
// how many chains a warp needs in flight to keep the FP64 tensor pipe busy.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(512, 1) chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

template <int CH>
void run(double* out, int sms) {
  const int iters = 32768 / CH;
  chains<CH><<<sms, 512>>>(out, 16);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  chains<CH><<<sms, 512>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 8 * 8 * 4 * (double)CH * iters * 16 * sms;
  printf("{\"chains_per_warp\": %d, \"warps_per_sm\": 16, \"tflops\": %.2f}\n", CH, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<1>(out, sms);
  run<2>(out, sms);
  run<3>(out, sms);
  run<4>(out, sms);
  run<6>(out, sms);
  run<8>(out, sms);
  return 0;
}
