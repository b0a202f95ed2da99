// Micro-benchmark: tcgen05.mma (kind::f16, bf16 in, fp32 accum, both operands from smem,
// 128B swizzle) issue throughput for M in {64,128} and N in {16..256}, one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/umma_bench.cu -o tools/umma_bench
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int M, int N>
__global__ void __launch_bounds__(128, 1) umma_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t sa = su32(smem), sb = su32(smem + 16384);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(desc_sw128(sa + k * 32)), "l"(desc_sw128(sb + k * 32)), "r"(idesc), "r"(1u));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

template <int M, int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(umma_kernel<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  umma_kernel<M, N><<<148, 128, smem>>>(16, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_kernel<M, N><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double n_mma = 4.0 * iters;
  printf("M=%3d N=%3d K=16: %6.1f cycles/UMMA, %7.1f ns/UMMA (event), %6.0f TFLOP/s chip\n", M, N, cyc / n_mma,
         ms * 1e6 / n_mma, 2.0 * M * N * 16 * n_mma * 148 / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  run<128, 16>(); run<128, 32>(); run<128, 64>(); run<128, 128>(); run<128, 256>();
  run<64, 16>(); run<64, 32>(); run<64, 64>(); run<64, 128>(); run<64, 256>();
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
