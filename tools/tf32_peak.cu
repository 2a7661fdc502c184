// tf32_peak.cu — dense tcgen05 kind::tf32 throughput on this B200 (the tensor-core roof of the CG
// table GEMM).  One CTA per SM, one elected thread issues back-to-back
// tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 256, K = 8; operands resident in shared
// memory, fp32 accumulator in TMEM), commits once per batch and waits on an mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_peak tools/tf32_peak.cu
// Prints one JSON line: {"tf32_tflops": ..., "sms": ..., "mma_per_cta": ...}.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int M = 128, N = 256, KS = 8;        // one MMA: 128 x 256 x 8 (tf32)
constexpr int A_BYTES = M * 32 * 4, B_BYTES = N * 32 * 4;  // one 32-wide K chunk, canonical K-major

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46);
}

__global__ void __launch_bounds__(128, 1) tf32_mma_loop(int iters, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t done;
  for (int t = threadIdx.x; t < (A_BYTES + B_BYTES) / 4; t += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[t] = 0x3f800000u ^ (t & 0xff) << 13;  // tf32-exact values
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sm), b0 = a0 + A_BYTES;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t da = desc(a0 + kk * 256, 128, 1024), db = desc(b0 + kk * 256, 128, 1024);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"((it | kk) != 0 ? 1 : 0)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&done))
                 : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&done))
        : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t r0;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r0) : "r"(tmem + ((threadIdx.x & ~31u) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  if (threadIdx.x == 0) sink[blockIdx.x] = __uint_as_float(r0);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(256));
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* sink;
  cudaMalloc(&sink, sizeof(float) * sms);
  const int smem = A_BYTES + B_BYTES;
  cudaFuncSetAttribute(tf32_mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 20000;  // x4 MMAs per iteration
  tf32_mma_loop<<<sms, 128, smem>>>(100, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    tf32_mma_loop<<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const cudaError_t e = cudaGetLastError();
  const double flops = 2.0 * M * N * KS * 4.0 * iters * sms;
  printf("{\"tf32_tflops\": %.2f, \"sms\": %d, \"mma_per_cta\": %d, \"shape\": \"128x256x8 kind::tf32, cta_group::1\", \"ms\": %.3f, \"err\": \"%s\"}\n",
         flops / (best * 1e-3) / 1e12, sms, 4 * iters, best, cudaGetErrorString(e));
  return 0;
}
