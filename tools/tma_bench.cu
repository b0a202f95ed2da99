// Micro-benchmark: how fast can 148 CTAs stream a [N x K] bf16 matrix through
// 2-D TMA boxes into shared memory (no compute)?  Varies box height, box count
// per stage and pipeline depth.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int ROWS, int NBOX, int NS>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap map, int nrow_blocks,
                                                        int kblocks, long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[NS];
  constexpr int BOX = ROWS * 128;
  constexpr int STAGE = BOX * NBOX;
  const int units = nrow_blocks * (kblocks / NBOX);
  const int u0 = (long long)units * blockIdx.x / gridDim.x, u1 = (long long)units * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int kb = kblocks / NBOX;
  auto issue = [&](int u, int s) {
    const int b = u / kb, k = (u % kb) * NBOX;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE));
    for (int j = 0; j < NBOX; ++j)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
              "r"(su32(smem + s * STAGE + j * BOX)), "l"((uint64_t)&map), "r"((k + j) * 64), "r"(b * ROWS),
          "r"(su32(&full[s])) : "memory");
  };
  long long acc = 0;
  int i = 0;
  for (int u = u0; u < u1 && i < NS; ++u, ++i) issue(u, i);
  for (int u = u0, j = 0; u < u1; ++u, ++j) {
    const int s = j % NS;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su32(&full[s])), "r"((j / NS) & 1) : "memory");
    acc += smem[s * STAGE + 5];
    if (u + NS < u1) issue(u + NS, s);
  }
  sink[blockIdx.x] = acc;
}

// The same stream from a block-tiled layout [N/8][K/64][8][64] (each 8-row x 64-column atom is
// one contiguous 1 KB run): a 4-D map, box {64, 8, 1, ROWS/8} lands in shared memory exactly as the
// 2-D box of the row-major layout does.
template <int ROWS, int NS>
__global__ void __launch_bounds__(128, 1) stream4d_kernel(const __grid_constant__ CUtensorMap map, int nrow_blocks,
                                                          int kblocks, long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[NS];
  constexpr int STAGE = ROWS * 128;
  const int units = nrow_blocks * kblocks;
  const int u0 = (long long)units * blockIdx.x / gridDim.x, u1 = (long long)units * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int u, int s) {
    const int b = u / kblocks, k = u % kblocks;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(STAGE));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(su32(smem + s * STAGE)), "l"((uint64_t)&map), "r"(0), "r"(0), "r"(k), "r"(b * (ROWS / 8)),
        "r"(su32(&full[s])) : "memory");
  };
  long long acc = 0;
  int i = 0;
  for (int u = u0; u < u1 && i < NS; ++u, ++i) issue(u, i);
  for (int u = u0, j = 0; u < u1; ++u, ++j) {
    const int s = j % NS;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(su32(&full[s])), "r"((j / NS) & 1) : "memory");
    acc += smem[s * STAGE + 5];
    if (u + NS < u1) issue(u + NS, s);
  }
  sink[blockIdx.x] = acc;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void ldg_kernel(const int4* __restrict__ p, size_t n, long long* sink) {
  long long acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v = __ldcs(p + i);
    acc += v.x ^ v.w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

template <int ROWS, int NBOX, int NS>
void run(void* w, int N, int K, long long* sink, void* flush, size_t flush_bytes, CUtensorMapL2promotion promo) {
  static Enc enc = nullptr;
  if (!enc) {
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = (Enc)p;
  }
  CUtensorMap maps[4];
  for (int q = 0; q < 4; ++q) {
  CUtensorMap& m = maps[q];
  void* wq = (char*)w + (size_t)q * N * K * 2;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, ROWS};
  cuuint32_t es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, wq, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int smem = NS * ROWS * 128 * NBOX + 1024;
  cudaFuncSetAttribute(stream_kernel<ROWS, NBOX, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  const int IT = 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    for (int it = 0; it < IT; ++it)
      stream_kernel<ROWS, NBOX, NS><<<148, 128, smem>>>(maps[it % 4], N / ROWS, K / 64, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= IT;
    if (rep > 0 && ms < best) best = ms;
  }
  printf("rows=%3d boxes/stage=%d stages=%2d promo=%d smem=%6d KB: %7.1f us  %6.0f GB/s\n", ROWS, NBOX, NS, (int)promo,
         smem / 1024, best * 1e3, (double)N * K * 2 / (best * 1e-3) / 1e9);
}

template <int ROWS, int NS>
void run4d(void* w, int N, int K, long long* sink) {
  static Enc enc = nullptr;
  if (!enc) {
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = (Enc)p;
  }
  CUtensorMap maps[4];
  for (int q = 0; q < 4; ++q) {
    void* wq = (char*)w + (size_t)q * N * K * 2;
    cuuint64_t dims[4] = {64, 8, (cuuint64_t)K / 64, (cuuint64_t)N / 8};
    cuuint64_t str[3] = {128, 1024, (cuuint64_t)(K / 64) * 1024};
    cuuint32_t box[4] = {64, 8, 1, ROWS / 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&maps[q], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, wq, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode 4d failed %d\n", (int)r); return; }
  }
  const int smem = NS * ROWS * 128 + 1024;
  cudaFuncSetAttribute(stream4d_kernel<ROWS, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  const int IT = 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    for (int it = 0; it < IT; ++it)
      stream4d_kernel<ROWS, NS><<<148, 128, smem>>>(maps[it % 4], N / ROWS, K / 64, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= IT;
    if (rep > 0 && ms < best) best = ms;
  }
  printf("TILED rows=%3d stages=%2d smem=%6d KB: %7.1f us  %6.0f GB/s\n", ROWS, NS, smem / 1024, best * 1e3,
         (double)N * K * 2 / (best * 1e-3) / 1e9);
}

int main() {
  const int N = 10240, K = 5120;
  void* w;
  cudaMalloc(&w, 4 * (size_t)N * K * 2);
  cudaMemset(w, 1, 4 * (size_t)N * K * 2);
  long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  size_t fb = 512ull << 20;
  void* flush;
  cudaMalloc(&flush, fb);
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {148, 296, 592, 1184}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 16; ++it)
          ldg_kernel<<<grid, 512>>>((const int4*)((char*)w + (size_t)(it % 4) * N * K * 2), (size_t)N * K * 2 / 16, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 16;
        if (rep > 0 && ms < best) best = ms;
      }
      printf("LDG.128 grid=%d x 512: %7.1f us  %6.0f GB/s\n", grid, best * 1e3, (double)N * K * 2 / (best * 1e-3) / 1e9);
    }
  }
  run<128, 1, 12>(w, N, K, sink, flush, fb, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run4d<128, 12>(w, N, K, sink);
  run<256, 1, 6>(w, N, K, sink, flush, fb, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run4d<256, 6>(w, N, K, sink);
  run<64, 1, 16>(w, N, K, sink, flush, fb, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  run4d<64, 16>(w, N, K, sink);
  for (auto promo : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
    run<128, 1, 8>(w, N, K, sink, flush, fb, promo);
    run<128, 1, 12>(w, N, K, sink, flush, fb, promo);
    run<128, 2, 6>(w, N, K, sink, flush, fb, promo);
    run<64, 1, 16>(w, N, K, sink, flush, fb, promo);
    run<64, 2, 12>(w, N, K, sink, flush, fb, promo);
    run<256, 1, 6>(w, N, K, sink, flush, fb, promo);
    run<32, 1, 32>(w, N, K, sink, flush, fb, promo);
    run<128, 4, 3>(w, N, K, sink, flush, fb, promo);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
