// Prefill projection GEMM: C[m][n] = sum_k A[m][k] * W[n][k] for the packed prompt rows of a
// prefill (M up to the whole prompt batch), every projection of the prefill: the mixer
// in-projections (R/PAPER.md:1542-1544, 1584-1587, 1614-1622), the out-projections, the FFN
// gate/up (SwiGLU fused into the epilogue) and down-projection, and the LM head.
//
// tcgen05 + TMEM + TMA, one CTA per SM (persistent grid over output tiles).  Tile = 128 rows
// of A x br rows of W (br <= 256: one UMMA M=128, N=br, K=16 per 16 columns), K streamed in
// 64-column atoms through a 4-stage ring of [A 128x64 | W br x64] (128B-swizzled TMA boxes).
// Warp roles as in the decode GEMM (sn_dgemm.cu): 0 = TMA producer, 1 = MMA issuer, 2 = TMEM
// allocator, 4-7 = epilogue; two TMEM accumulators (2 x 256 columns) so one tile's epilogue
// overlaps the next tile's MMAs.  The epilogue is sn_epi.cuh's (STORE / SwiGLU-interleaved).
//
// Rasterisation: tiles are walked in bands of 32 row tiles, the weight block changing slowest
// inside a band, so the ~148 tiles in flight at a time touch 32 A tiles and ~5 weight blocks
// (~55 MB, L2-resident) instead of streaming the whole of A or W per wave.
//
// Measured (tools/bench_pgemm.py, 16K-token prompt, Apriel shapes): 1.40-1.46 PFLOP/s, 88-93 %
// of cuBLAS on the same box (the gate/up figure includes the fused SwiGLU).  The remaining gap
// is L2 -> SM operand traffic (48 KB per 4.2 MFLOP); the 2-CTA (cta_group::2) 256-row tile that
// halves it is the next step.
#include <cuda.h>

#include "sn_common.cuh"
#include "sn_epi.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace pgemm {

using namespace sn::tc;
constexpr int kThreads = 256;
constexpr int BM = 128;
constexpr int kStages = 4;
constexpr int kAccCols = 256;
constexpr int kBand = 32;  // row tiles per rasterisation band (4 / 8 / 16 / 32 measured: 32 best)

struct Args {
  int M, K, kb, br, mtiles, nblocks, band;
  epi::Args e;
};

// tile j -> (row tile, weight block): bands of kBand row tiles, weight block slowest in a band
__device__ __forceinline__ void tile_of(const Args& g, int j, int& mt, int& nb) {
  const int band_tiles = g.band * g.nblocks;
  const int band = j / band_tiles, r = j - band * band_tiles;
  const int rows = min(g.band, g.mtiles - band * g.band);  // the last band may be short
  nb = r / rows;
  mt = band * g.band + (r - nb * rows);
}

__global__ void __launch_bounds__(kThreads, 1)
    pgemm_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x, G = gridDim.x;
  const int tiles = g.mtiles * g.nblocks;
  const int my_tiles = tiles > q ? (tiles - q + G - 1) / G : 0;
  constexpr uint32_t A_BYTES = BM * BK * 2;
  const uint32_t w_bytes = (uint32_t)g.br * BK * 2;
  const uint32_t stage = A_BYTES + w_bytes;
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
    for (int i = 0; i < kStages; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(2 * kAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      // both operands are re-read by other tiles of the band: keep them in L2 (evict-first on
      // either measured 3-15 % slower)
      const uint64_t pw = policy_evict_last(), pa = policy_evict_last();
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my_tiles; ++it) {
        int mt, nb;
        tile_of(g, q + it * G, mt, nb);
        for (int k = 0; k < g.kb; ++k) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          mbar_expect_tx(&full_bar[s], stage);
          uint8_t* st = smem + s * stage;
          tma_load_2d(st, &amap, k * BK, mt * BM, &full_bar[s], pa);
          tma_load_2d(st + A_BYTES, &wmap, k * BK, nb * g.br, &full_bar[s], pw);
          if (++s == kStages) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (warp-converged, one elected lane issues)
    const uint32_t idesc = idesc_bf16(BM, g.br);
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < my_tiles; ++it) {
      const int buf = it & 1;
      if (it >= 2) mbar_wait(&tempty_bar[buf], ((it >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + buf * kAccCols;
      for (int k = 0; k < g.kb; ++k) {
        mbar_wait(&full_bar[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + s * stage), sw = sa + A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_w(acc, desc_sw128(sa + kk * 32), desc_sw128(sw + kk * 32), idesc, (k | kk) ? 1u : 0u);
        commit_w(&empty_bar[s]);
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
      commit_w(&tfull_bar[buf]);
    }
  } else if (warp >= 4) {  // ---------------- epilogue: warp w drains TMEM lanes [32*(w%4), +32)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int sp = warp & 3;
    const uint32_t lane_addr = (uint32_t)(32 * sp) << 16;
    for (int it = 0; it < my_tiles; ++it) {
      const int buf = it & 1;
      int mt, nb;
      tile_of(g, q + it * G, mt, nb);
      const int m = mt * BM + 32 * sp + lane;
      mbar_wait(&tfull_bar[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + lane_addr + buf * kAccCols;
      auto get = [&](int c0, int c1, float* v) {
        tmem_ld16_async(acc + c0, v);
        tmem_ld16_async(acc + c1, v + 16);
        tmem_wait_ld();
        reg_fence16(v);
        reg_fence16(v + 16);
      };
      epi::finalize<__nv_bfloat16>(g.e, m, m < g.M, nb, 0, g.br, get);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[buf]);
    }
  }
  __syncwarp();
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols));
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 0;
    cudaGetLastError();
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace pgemm
}  // namespace sn

using namespace sn;

extern "C" sn_status sn_gemm_prefill(const void* a, int M, int K, int lda, const void* w, int N, int ldw, void* out,
                                     int ldo, int mode, int swiglu_h, void* stream) {
  using namespace sn::pgemm;
  SN_REQUIRE(a && w && out, "sn_gemm_prefill: NULL operand");
  SN_REQUIRE(M >= 1 && N >= 1 && K >= tc::BK && K % tc::BK == 0, "sn_gemm_prefill: M=%d N=%d K=%d (K %% 64)", M, N, K);
  SN_REQUIRE(lda >= K && ldw >= K && ((uintptr_t)a % 16) == 0 && ((uintptr_t)w % 16) == 0 && (lda * 2) % 16 == 0 &&
                 (ldw * 2) % 16 == 0,
             "sn_gemm_prefill: operands must be 16-byte aligned with row pitch >= K");
  SN_REQUIRE(mode == SN_GEMM_STORE || mode == SN_GEMM_SWIGLU_IL, "sn_gemm_prefill: mode %d (STORE or SWIGLU_IL)", mode);
  SN_REQUIRE(ldo >= N && (ldo % 8) == 0, "sn_gemm_prefill: ldo %d", ldo);
  int br = 256, nblocks = (N + 255) / 256;
  uint64_t wrows = (uint64_t)N;
  if (mode == SN_GEMM_SWIGLU_IL) {
    SN_REQUIRE(swiglu_h >= 16 && swiglu_h <= 128 && swiglu_h % 16 == 0, "sn_gemm_prefill: SwiGLU block %d", swiglu_h);
    br = 2 * swiglu_h;
    nblocks = (N + swiglu_h - 1) / swiglu_h;
    wrows = (uint64_t)nblocks * br;
  }
  Args g{};
  g.M = M; g.K = K; g.kb = K / tc::BK; g.br = br; g.mtiles = (M + BM - 1) / BM; g.nblocks = nblocks;
  g.band = kBand;
  g.e.mode = mode; g.e.M = M; g.e.N = N; g.e.out = out; g.e.ldo = ldo; g.e.S = 1;
  CUtensorMap wm, am;
  if (!tc::map_2d(&wm, w, wrows, K, ldw, br) || !tc::map_2d(&am, a, M, K, lda, BM)) {
    set_error("sn_gemm_prefill: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  const int tiles = g.mtiles * g.nblocks;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  const int smem = kStages * (BM + br) * tc::BK * 2 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024);
    attr = true;
  }
  cudaError_t e = launch_pdl(pgemm_kernel, dim3(grid), dim3(kThreads), (size_t)smem, (cudaStream_t)stream, wm, am, g);
  if (e != cudaSuccess) {
    set_error("sn_gemm_prefill launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_gemm_prefill");
}
