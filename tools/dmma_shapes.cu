// FP64 tensor-core throughput by mma shape: m8n8k4 vs m16n8k4 / m16n8k8 / m16n8k16 (sm_90+ shapes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_shapes tools/dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void loop(double* out, int iters) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}

template <int SHAPE>
void run(const char* name, double mnk, int sms) {
  double* od;
  cudaMalloc(&od, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int wpb : {4, 8, 16}) {
    const int iters = SHAPE == 0 ? 4000 : 1000;
    loop<SHAPE><<<sms * 2, wpb * 32>>>(od, 10);
    cudaEventRecord(a);
    loop<SHAPE><<<sms * 2, wpb * 32>>>(od, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * mnk * 8 * iters * (double)sms * 2 * wpb;
    printf("{\"shape\": \"%s\", \"tflops\": %.2f, \"warps_per_cta\": %d, \"err\": \"%s\"}\n", name, flops / ms / 1e9, wpb,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  run<0>("m8n8k4", 8 * 8 * 4, p.multiProcessorCount);
  run<1>("m16n8k4", 16 * 8 * 4, p.multiProcessorCount);
  run<2>("m16n8k8", 16 * 8 * 8, p.multiProcessorCount);
  run<3>("m16n8k16", 16 * 8 * 16, p.multiProcessorCount);
  return 0;
}
