// Prefill projection GEMM: C[m][n] = sum_k A[m][k] * W[n][k] for the packed prompt rows of a
// prefill (M up to the whole prompt batch), every projection of the prefill: the mixer
// in-projections (R/PAPER.md:1542-1544, 1584-1587, 1614-1622), the out-projections, the FFN
// gate/up (SwiGLU fused into the epilogue) and down-projection, and the LM head.
//
// tcgen05 + TMEM + TMA, persistent grid of CTA pairs over output tiles (pgemm_kernel): a
// cluster of two CTAs on one TPC computes a 256 x br tile with one cta_group::2 UMMA stream
// (M = 256, N = br <= 256, K = 16 per instruction).  Each CTA stages its own 128 rows of A and
// br / 2 rows of W per 64-column atom through a 7-stage ring, so the pair reads each operand
// byte once per 256 x br tile (half the L2 -> SM bytes per flop of a 128-row tile); the leader
// issues every MMA, both CTAs' TMA loads complete on the leader's barrier, the MMA commits
// multicast to both CTAs' barriers and each CTA drains its own 128 accumulator lanes.  br is
// chosen per shape to minimise the last wave's idle pairs (STORE / fp32 store: 256 or 224;
// SwiGLU: 2h).  mbarrier waits carry a suspend-time hint (sn_tc.cuh).
// Warp roles as in the decode GEMM (sn_dgemm.cu): 0 = TMA producer, 1 = MMA issuer, 2 = TMEM
// allocator, 4-7 = epilogue; two TMEM accumulators (2 x 256 columns) so one tile's epilogue
// overlaps the next tile's MMAs.  The epilogue is sn_epi.cuh's (STORE / SwiGLU-interleaved).
//
// Rasterisation: tiles are walked in bands of 16 (8 for long K) row tiles,
// the weight block changing slowest inside a band, so the tiles in flight at a time share a
// few A row tiles and weight blocks through L2.
//
// Measured (tools/bench_pgemm.py, Apriel shapes, same box): 16K-token prompt 1.55-1.61 PFLOP/s,
// 0.93-1.01 of cuBLAS; 0.9-1.2x at 256-4096 rows; 0.90-1.10x at 64K-128K rows.  A whole 16K
// prefill with these projections matches the cuBLAS-projection prefill (433-446 vs 429-432 ms
// under the sustained power cap).  A 1-CTA 128 x 256 tile kernel (4-stage ring) reached
// 0.87-0.95 at 16K and 0.5-0.9x the 2-CTA kernel at every M; removed.  Clusters of four
// (multicasting A between two pairs) fit only 33 at a time (132 SMs); not used.
#include <cuda.h>
#include <stdlib.h>

#include "sn_common.cuh"
#include "sn_epi.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace pgemm {

using namespace sn::tc;
constexpr int kThreads = 256;
constexpr int kAccCols = 256;

struct Args {
  int M, K, kb, br, mtiles, nblocks, band;
  epi::Args e;
};

// tile j -> (row tile, weight block): bands of g.band row tiles, weight block slowest in a band
__device__ __forceinline__ void tile_of(const Args& g, int j, int& mt, int& nb) {
  const int band_tiles = g.band * g.nblocks;
  const int band = j / band_tiles, r = j - band * band_tiles;
  const int rows = min(g.band, g.mtiles - band * g.band);  // the last band may be short
  nb = r / rows;
  mt = band * g.band + (r - nb * rows);
}

// ---------------------------------------------------------------------------------------
// cta_group::2: the leader CTA (rank 0) issues every MMA, every TMA completes on the leader's
// full barrier (both CTAs' bytes), the MMA commits multicast to both CTAs' empty / TMEM-full
// barriers, and each CTA drains its own 128 accumulator lanes.  SwiGLU (br = 2h): the leader
// holds the gate rows of a block, the peer the up rows; every accumulator row has both halves.
constexpr int kStages2 = 7;
// 256-row tiles per rasterisation band: the band's A rows stay L2-resident while it sweeps the
// weight blocks, so the weights are re-read once per band.  16 for K <= 8192 (K = 5120: a 42 MB
// band; gate/up at 128K rows 0.90 -> 0.92-1.06 of cuBLAS vs 8), 8 for the long-K down-projection
// (K = 14336: 16 would be a 117 MB band).  At 16K rows 8 / 16 / 24 are equal within noise.
constexpr int kBandShortK = 16, kBandLongK = 8;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clear the CTA-rank bit: the leader's copy of a barrier

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerMask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma2_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {  // arrive on this barrier in both CTAs
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {  // arrive on the leader CTA's copy
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    pgemm_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kStages2], empty_bar[kStages2], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  constexpr uint32_t A_BYTES = 128 * BK * 2;
  const int wr = g.br / 2;  // this CTA's weight rows per block
  const uint32_t w_bytes = (uint32_t)wr * BK * 2;
  const uint32_t stage = A_BYTES + w_bytes;
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap)) : "memory");
    for (int i = 0; i < kStages2; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 8); }  // 4 + 4 epilogue warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(2 * kAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrival
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  const int q = blockIdx.x >> 1, G = gridDim.x >> 1;  // pair index / count; g.mtiles counts 256-row tiles
  const int tiles = g.mtiles * g.nblocks;
  const int my_tiles = tiles > q ? (tiles - q + G - 1) / G : 0;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs: own halves, leader's barrier)
      const uint64_t pw = policy_evict_last(), pa = policy_evict_last();
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my_tiles; ++it) {
        int mt, nb;
        tile_of(g, q + it * G, mt, nb);
        for (int k = 0; k < g.kb; ++k) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (leader) mbar_expect_tx(&full_bar[s], 2 * stage);
          uint8_t* st = smem + s * stage;
          tma_load_2d_2sm(st, &amap, k * BK, mt * 256 + (int)rank * 128, &full_bar[s], pa);
          tma_load_2d_2sm(st + A_BYTES, &wmap, k * BK, nb * g.br + (int)rank * wr, &full_bar[s], pw);
          if (++s == kStages2) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {  // ---------------- MMA issuer: the leader drives the pair's UMMA stream
      const uint32_t idesc = idesc_bf16(256, g.br);
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
            umma2_w(acc, desc_sw128(sa + kk * 32), desc_sw128(sw + kk * 32), idesc, (k | kk) ? 1u : 0u);
          commit2_mc(&empty_bar[s]);
          if (++s == kStages2) { s = 0; ph ^= 1; }
        }
        commit2_mc(&tfull_bar[buf]);
      }
    }
  } else if (warp >= 4) {  // ---------------- epilogue (both CTAs): own 128 rows
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int sp = warp & 3;
    const uint32_t lane_addr = (uint32_t)(32 * sp) << 16;
    for (int it = 0; it < my_tiles; ++it) {
      const int buf = it & 1;
      int mt, nb;
      tile_of(g, q + it * G, mt, nb);
      const int m = mt * 256 + (int)rank * 128 + 32 * sp + lane;
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
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty_bar[buf]);
        else mbar_arrive_leader(&tempty_bar[buf]);
      }
    }
  }
  __syncwarp();
  __syncthreads();
  cluster_sync_all();  // the pair's MMAs and epilogues are done before the pair's TMEM is freed
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols));
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
  SN_REQUIRE(mode == SN_GEMM_STORE || mode == SN_GEMM_SWIGLU_IL || mode == SN_GEMM_PARTIAL,
             "sn_gemm_prefill: mode %d (STORE, SWIGLU_IL or PARTIAL = fp32 store)", mode);
  SN_REQUIRE(ldo >= N && (ldo % 8) == 0, "sn_gemm_prefill: ldo %d", ldo);
  const bool swiglu = mode == SN_GEMM_SWIGLU_IL;
  if (swiglu)
    SN_REQUIRE(swiglu_h >= 16 && swiglu_h <= 128 && swiglu_h % 8 == 0, "sn_gemm_prefill: SwiGLU block %d", swiglu_h);
  const int mtiles = (M + 255) / 256;
  const int slots = num_sms() / 2;  // CTA pairs in flight
  int br = 256;
  if (swiglu) {
    br = 2 * swiglu_h;
  } else {  // the block height whose last wave leaves the fewest pairs idle, among 256 / 224
    // (narrower tiles re-read A more per flop: 192 ran at 0.86 and 128-160 at 0.71-0.74 of
    // cuBLAS at 64K-128K rows, where the wave quantisation they save is negligible)
    long best = -1;
    for (int c = 256; c >= 224; c -= 32) {
      const long waves = ((long)((N + c - 1) / c) * mtiles + slots - 1) / slots;
      if (best < 0 || waves * c < best) { best = waves * c; br = c; }
    }
  }
  const int nblocks = swiglu ? (N + swiglu_h - 1) / swiglu_h : (N + br - 1) / br;
  const uint64_t wrows = swiglu ? (uint64_t)nblocks * br : (uint64_t)N;
  Args g{};
  g.M = M; g.K = K; g.kb = K / tc::BK; g.br = br; g.mtiles = mtiles; g.nblocks = nblocks;
  g.band = K <= 8192 ? kBandShortK : kBandLongK;
  g.e.mode = mode; g.e.M = M; g.e.N = N; g.e.out = out; g.e.ldo = ldo; g.e.S = 1;
  CUtensorMap wm, am;
  if (!tc::map_2d(&wm, w, wrows, K, ldw, br / 2) || !tc::map_2d(&am, a, M, K, lda, 128)) {
    set_error("sn_gemm_prefill: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  const int tiles = mtiles * nblocks;
  const int grid = tiles < slots ? tiles : slots;
  const int smem = kStages2 * (128 + br / 2) * tc::BK * 2 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pgemm_kernel, wm, am, g);
  if (e != cudaSuccess) {
    set_error("sn_gemm_prefill launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_gemm_prefill");
}
