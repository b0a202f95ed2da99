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

// MODE bit 0: two accumulators / two A tiles alternating (the paired-tile GEMM pattern);
// MODE bit 1: warps 1-3 write shared memory at full rate meanwhile (TMA fill contention).
__device__ uint8_t g_src[1 << 20];  // L2-resident source of the bulk-copy traffic (MODE bit 2)

// MODE bit 2: warp 1 streams 16 KB bulk copies (global -> shared, the TMA path) into a
// separate 32 KB region meanwhile; the achieved copy rate is reported in out[1].
template <int M, int N, int MODE = 0>
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
  __shared__ volatile int stop;
  __shared__ uint64_t sbar, cmt;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cmt)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&sbar)) : "memory");  // phase 0 completes
  }
  if (threadIdx.x == 0) stop = 0;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  __shared__ uint64_t cbar[2];
  if ((MODE & 4) && threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned long long n = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; !stop; ++i) {
      const int b = i & 1;
      if (i >= 2) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(su32(&cbar[b])), "r"(((i >> 1) - 1) & 1) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cbar[b])), "r"(16384) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(smem + 98304 + b * 16384)), "l"(g_src + (size_t)((i * 16384 + blockIdx.x * 65536) & ((1 << 20) - 1))),
                   "r"(16384), "r"(su32(&cbar[b])) : "memory");
      ++n;
    }
    if (blockIdx.x == 0) out[1] = n * 16384 * 1000 / (clock64() - t0);  // bytes per 1000 cycles
  }
  if ((MODE & 2) && warp > 0) {
    uint4* w = reinterpret_cast<uint4*>(smem + 65536);
    int i = threadIdx.x - 32;
    while (!stop) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) w[(i + j * 96) & 2047] = make_uint4(i, j, 0, 0);
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // MODE bit 3: rotate over 4 distinct A tiles (16 KB) and B tiles (8 KB) like a stage ring
      const int r = (MODE & 8) ? (i & 3) : 0;
      const uint32_t sa = su32(smem + r * 16384), sa2 = su32(smem + ((r + 1) & 3) * 16384),
                     sb = su32(smem + 65536 + r * 8192);
      if ((MODE & 256) && (i & 1) == 0) {  // one try_wait per two stages
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(su32(&sbar)), "r"(0u) : "memory");
      }
      if (MODE & 512) {  // non-blocking test_wait instead of try_wait
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(su32(&sbar)), "r"(0u) : "memory");
      }
      if (MODE & (16 | 64)) {  // per-stage overhead of the GEMM loop: wait on a (completed) barrier
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(su32(&sbar)), "r"(0u) : "memory");
      }
      if (MODE & (16 | 128)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
            "l"(desc_sw128(sa + k * 32)), "l"(desc_sw128(sb + k * 32)), "r"(idesc), "r"(1u));
        if (MODE & 1)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + N),
              "l"(desc_sw128(sa2 + k * 32)), "l"(desc_sw128(sb + k * 32)), "r"(idesc), "r"(1u));
      }
      if (MODE & 32)  // per-stage commit (frees the stage in the GEMM)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&cmt))
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

template <int M, int N, int MODE = 0>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  const int smem = 128 * 1024 + 1024;
  cudaFuncSetAttribute(umma_kernel<M, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  umma_kernel<M, N, MODE><<<148, 128, smem>>>(16, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  umma_kernel<M, N, MODE><<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc, rate[2];
  cudaMemcpy(rate, d, 16, cudaMemcpyDeviceToHost);
  cyc = rate[0];
  const double n_mma = 4.0 * iters * ((MODE & 1) ? 2 : 1);
  printf("mode %d M=%3d N=%3d K=16:", MODE, M, N);
  printf(" %6.1f cycles/UMMA, %7.1f ns/UMMA (event), %6.0f TFLOP/s chip, bulk-copy %.1f B/cycle\n", cyc / n_mma,
         ms * 1e6 / n_mma, 2.0 * M * N * 16 * n_mma * 148 / (ms * 1e-3) / 1e12, rate[1] / 1000.0);
  cudaFree(d);
}

int main() {
  run<128, 16>(); run<128, 32>(); run<128, 64>(); run<128, 128>(); run<128, 256>(); // (B for N=256 overlaps the A ring; fine for timing)
  run<64, 16>(); run<64, 32>(); run<64, 64>(); run<64, 128>(); run<64, 256>();
  run<128, 64, 1>(); run<128, 64, 2>(); run<128, 64, 3>(); run<64, 256, 2>(); run<128, 128, 1>();
  run<128, 64, 4>(); run<128, 64, 5>(); run<64, 128, 4>(); run<128, 128, 4>();
  run<128, 64, 8>(); run<128, 64, 9>(); run<128, 64, 12>(); run<128, 64, 13>(); run<64, 64, 8>(); run<128, 32, 8>();
  run<128, 64, 9 + 16>(); run<128, 64, 9 + 32>(); run<128, 64, 9 + 48>(); run<128, 64, 13 + 48>();
  run<128, 64, 9 + 64>(); run<128, 64, 9 + 128>(); run<128, 64, 9 + 64 + 32>();
  run<128, 64, 9 + 256>(); run<128, 64, 9 + 512>(); run<128, 64, 9 + 512 + 32>();
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
