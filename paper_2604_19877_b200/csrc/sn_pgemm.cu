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
#include <stdlib.h>

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
  int M, K, kb, br, mtiles, nblocks, band, pol, die;
  epi::Args e;
};

// tile j -> (row tile, weight block): bands of kBand row tiles, weight block slowest in a band
// A CTA's walk: row tiles [mt0, mt0 + mtiles) of the tile space, tiles q, q + G, ...
struct Walk {
  int q, G, mt0, mtiles;
};
__device__ __forceinline__ void tile_of(const Args& g, const Walk& w, int j, int& mt, int& nb) {
  const int band_tiles = g.band * g.nblocks;
  const int band = j / band_tiles, r = j - band * band_tiles;
  const int rows = min(g.band, w.mtiles - band * g.band);  // the last band may be short
  nb = r / rows;
  mt = w.mt0 + band * g.band + (r - nb * rows);
}
__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// EXPERIMENT: die-local walks (one CTA per SM): the two halves of the SMs take the two halves
// of the row tiles.  die = 1: SMs [0, G/2) vs [G/2, G); die = 2: even vs odd SM ids.
__device__ __forceinline__ Walk make_walk(const Args& g, int q, int G, int sm) {
  Walk w{q, G, 0, g.mtiles};
  if (g.die) {
    const int d = g.die == 1 ? (sm >= G / 2) : (sm & 1);
    w.q = g.die == 1 ? sm - d * (G / 2) : sm >> 1;
    w.G = G / 2;
    w.mt0 = d ? g.mtiles / 2 : 0;
    w.mtiles = d ? g.mtiles - g.mtiles / 2 : g.mtiles / 2;
  }
  return w;
}
__device__ __forceinline__ int walk_tiles(const Args& g, const Walk& w) {
  const int tiles = w.mtiles * g.nblocks;
  return tiles > w.q ? (tiles - w.q + w.G - 1) / w.G : 0;
}

__global__ void __launch_bounds__(kThreads, 1)
    pgemm_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Walk wk = make_walk(g, blockIdx.x, gridDim.x, (int)sm_id());
  const int my_tiles = walk_tiles(g, wk);
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
      const uint64_t pw = (g.pol & 1) ? policy_evict_normal() : policy_evict_last();
      const uint64_t pa = (g.pol & 2) ? policy_evict_normal() : (g.pol & 4) ? policy_evict_first() : policy_evict_last();
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my_tiles; ++it) {
        int mt, nb;
        tile_of(g, wk, wk.q + it * wk.G, mt, nb);
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
      tile_of(g, wk, wk.q + it * wk.G, mt, nb);
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

// ---------------------------------------------------------------------------------------
// 2-CTA version (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x br tile with
// one UMMA stream (M = 256, N = br).  Each CTA stages its own 128 rows of A and its own br / 2
// rows of W per 64-column atom (the pair shares both operands: half the L2 -> SM bytes per flop
// of the 1-CTA kernel), the leader CTA (rank 0) issues every MMA, every TMA completes on the
// leader's full barrier, the MMA commits multicast to both CTAs' empty / TMEM-full barriers,
// and each CTA drains its own 128 accumulator lanes.  SwiGLU (br = 2h): the leader holds the
// gate rows of a block, the peer the up rows; every accumulator row has both halves.
constexpr int kStages2 = 7;
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
__device__ __forceinline__ void tma_load_2d_2sm_nh(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerMask)
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
    pgemm2_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kStages2], empty_bar[kStages2], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s, sm_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) sm_s = sm_id();
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
  uint32_t leader_sm;  // the pair's walk follows the leader's SM (TPC) id
  {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(&sm_s)));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(leader_sm) : "r"(remote) : "memory");
  }
  const Walk wk = make_walk(g, blockIdx.x >> 1, gridDim.x >> 1, (int)(leader_sm >> 1));  // 256-row tiles
  const int my_tiles = walk_tiles(g, wk);

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs: own halves, leader's barrier)
      const uint64_t pw = (g.pol & 1) ? policy_evict_normal() : policy_evict_last();
      const uint64_t pa = (g.pol & 2) ? policy_evict_normal() : (g.pol & 4) ? policy_evict_first() : policy_evict_last();
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my_tiles; ++it) {
        int mt, nb;
        tile_of(g, wk, wk.q + it * wk.G, mt, nb);
        for (int k = 0; k < g.kb; ++k) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          if (leader) mbar_expect_tx(&full_bar[s], 2 * stage);
          uint8_t* st = smem + s * stage;
          if (g.pol & 8) {
            tma_load_2d_2sm_nh(st, &amap, k * BK, mt * 256 + (int)rank * 128, &full_bar[s]);
            tma_load_2d_2sm_nh(st + A_BYTES, &wmap, k * BK, nb * g.br + (int)rank * wr, &full_bar[s]);
          } else {
            tma_load_2d_2sm(st, &amap, k * BK, mt * 256 + (int)rank * 128, &full_bar[s], pa);
            tma_load_2d_2sm(st + A_BYTES, &wmap, k * BK, nb * g.br + (int)rank * wr, &full_bar[s], pw);
          }
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
      tile_of(g, wk, wk.q + it * wk.G, mt, nb);
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
  static const int band_env = getenv("SN_PG_BAND") ? atoi(getenv("SN_PG_BAND")) : 0;  // EXPERIMENT
  g.band = band_env > 0 ? band_env : kBand;
  g.pol = getenv("SN_PG_POL") ? atoi(getenv("SN_PG_POL")) : 0;
  g.die = getenv("SN_PG_DIE") ? atoi(getenv("SN_PG_DIE")) : 0;
  if (g.mtiles * nblocks < num_sms()) g.die = 0;
  g.e.mode = mode; g.e.M = M; g.e.N = N; g.e.out = out; g.e.ldo = ldo; g.e.S = 1;
  CUtensorMap wm, am;
  if (!tc::map_2d(&wm, w, wrows, K, ldw, br) || !tc::map_2d(&am, a, M, K, lda, BM)) {
    set_error("sn_gemm_prefill: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  static const bool two = getenv("SN_PG2") && atoi(getenv("SN_PG2"));  // EXPERIMENT A/B
  if (two && br % 32 == 0) {
    CUtensorMap wm2, am2;
    const int pe = getenv("SN_PG_PROMO") ? atoi(getenv("SN_PG_PROMO")) : 256;
    const CUtensorMapL2promotion pr = pe == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : pe == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : pe == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (!tc::map_2d(&wm2, w, wrows, K, ldw, br / 2, pr) || !tc::map_2d(&am2, a, M, K, lda, 128, pr)) {
      set_error("sn_gemm_prefill: cuTensorMapEncodeTiled failed");
      return SN_ECUDA;
    }
    Args g2 = g;
    g2.mtiles = (M + 255) / 256;
    static const int band2_env = getenv("SN_PG_BAND2") ? atoi(getenv("SN_PG_BAND2")) : 0;
    g2.band = band2_env > 0 ? band2_env : 8;
    if (g2.mtiles * g2.nblocks < num_sms() / 2) g2.die = 0;
    const int tiles2 = g2.mtiles * g2.nblocks;
    const bool np = getenv("SN_PG2_NP") && atoi(getenv("SN_PG2_NP"));
    const int pairs = np ? tiles2 : tiles2 < num_sms() / 2 ? tiles2 : num_sms() / 2;
    if (np) g2.die = 0;
    const int smem2 = kStages2 * (128 + br / 2) * tc::BK * 2 + 1024;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(pgemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024);
      attr2 = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem2;
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
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, pgemm2_kernel, wm2, am2, g2);
    if (e2 != cudaSuccess) {
      set_error("sn_gemm_prefill (2-CTA) launch: %s", cudaGetErrorString(e2));
      return SN_ECUDA;
    }
    return check_launch("sn_gemm_prefill");
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
