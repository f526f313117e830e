// Throughput of back-to-back tcgen05.mma (kind::f16, M=128, K=16, SS operands from
// SWIZZLE_128B K-major smem) as a function of N, one CTA per SM, no TMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../paper_1812_07816_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"

template <int N, int M = 128>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { us::mbar_init(&bar, 1); us::fence_barrier_init(); }
  if (threadIdx.x / 32 == 0) us::tmem_alloc<256>(&tbase);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  us::tc_fence_before();
  __syncthreads();
  us::tc_fence_after();
  const uint32_t a = us::smem_u32(smem), b = a + 128 * 128;
  constexpr uint32_t idesc = us::idesc_bf16(M, N, 0, 0);
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        us::umma_bf16(tbase, us::smem_desc(a + k * 32, 16, 1024, 2),
                      us::smem_desc(b + k * 32, 16, 1024, 2), idesc, (it | k) != 0);
    }
    us::umma_commit(&bar);
    us::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  us::tc_fence_before();
  __syncthreads();
  if (threadIdx.x / 32 == 0) us::tmem_dealloc<256>(tbase);
}

template <int N, int M = 128>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 20000;
  size_t smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(k_rate<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_rate<N, M><<<sms, 128, smem>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<N, M><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * M * N * 16 * 4 * (double)iters * sms;
  printf("M=%3d N=%3d: ", M, N);
  printf("%.3f ms  %.1f TFLOP/s  %.1f clk per MMA (K16)  err=%s\n", ms, flops / ms / 1e9,
         (double)cyc / (4.0 * iters), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<32>(sms); run<64>(sms); run<128>(sms); run<256>(sms);
  run<64, 64>(sms); run<128, 64>(sms); run<256, 64>(sms);
  return 0;
}
