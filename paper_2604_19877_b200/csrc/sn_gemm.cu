// Weight-streaming decode GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Decode projections/FFN/LM head are  C[m][n] = sum_k X[m][k] * W[n][k]  with a
// tiny batch M (<= 128 sequences) and big weights W [N x K] (58% of the bytes of
// a fastest-preset decode step).  The kernel is therefore an
// HBM stream of W: each CTA owns a 128-row block of W (and optionally a K slice),
// TMA streams [128 x 64] W tiles and the matching [BN x 64] X tiles through an
// mbarrier ring in shared memory (128B swizzle), one elected thread issues
// tcgen05.mma (M=128 weight rows x N=BN batch columns x K=16) into a TMEM
// accumulator, and the 4 warps drain TMEM with tcgen05.ld in the epilogue.
// "Swap-AB": W is the UMMA A operand so the tiny batch sits in the N dimension.
//
// Work split: measured on B200, one SM pulls only ~45-60 GB/s of TMA tiles, so a
// decode GEMM must keep (nearly) every one of the 148 SMs streaming, and split-K
// fix-ups cost more than they save (all partials finish together at the end).
// Instead each CTA owns whole row blocks over the full K: the host picks the
// block height BR (a multiple of 8 <= 128; the UMMA still runs M=128, rows >= BR
// of the smem tile are ignored) that minimises waves x BR, e.g. BR=40 for
// N=5120 (128 CTAs), BR=72 for N=10304 (144 CTAs), BR=128 for the LM head
// (persistent: ~7 blocks per CTA).  No reduction, no workspace, deterministic.
// TMEM holds two accumulators so the epilogue of one block overlaps the MMAs of
// the next; warp roles: 0 = TMA producer, 1 = MMA issuer, 4-7 = epilogue.
// Programmatic dependent launch lets the first stages of W stream in while the
// previous kernel of the decode step is still running.
//
// Epilogues (fused to remove separate elementwise kernels from the step):
//   SN_GEMM_STORE   out[m][n] = acc                         (bf16)
//   SN_GEMM_SWIGLU  W = [gate; up] (2N rows): out[m][n] = silu(g) * u  (bf16)
//   SN_GEMM_RESID   resid[m][n] += acc                      (fp32 residual stream)
#include <cuda.h>
#include <stdlib.h>

#include "sn_common.cuh"

namespace sn {
namespace gemm {

constexpr int BM = 128;     // weight rows per CTA (UMMA M)
constexpr int BK = 64;      // K per stage (one 128-B swizzle row of bf16)
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_noarrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                               uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;              // descriptor version (sm100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::f16, bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct GemmArgs {
  void* out;       // bf16 [M][ldo] | fp32 residual [M][ldo] | fp32 partial slabs [splits][M][ldo]
  int M, N, K, ldo, mode, kblocks;
  int br;          // weight rows per block (multiple of 8, <= BM)
  int nblocks;     // ceil(N / br)
  int splits;      // K splits per block (PARTIAL mode only, else 1)
  int cs;          // CTAs per cluster sharing (multicasting) each activation tile
  unsigned long long* stats;  // optional per-CTA cycle counters (profiling; NULL in production)
  int row_mul;     // weight rows per block: BR (one A tile or SwiGLU pair) or 2*BR (two stacked tiles)
  int a2_base;     // row offset of the second A tile inside a block: N (SwiGLU: up rows) or BR
  int ns;          // pipeline stages (runtime: as many as fit, so small blocks keep W in flight)
  int stage_bytes; // NA * br * 128 + BN * 128 (1024-aligned)
  int dbg;         // experiments (env SN_GEMM_DBG): 1 = no TMA after the prologue (MMA-rate probe)
};

constexpr int kMaxStages = 32;

constexpr int kGemmThreads = 256;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// smem: [stages][ A (NA x 16 KB) | B (BN x 128 B) ].  NA = 2 for SwiGLU.
template <int BN, int NA>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_decode_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                       const GemmArgs g) {
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int ACC = NA * BN;  // TMEM columns per accumulator buffer
  constexpr int TMEM_COLS = (2 * ACC) <= 32 ? 32 : (2 * ACC) <= 64 ? 64 : (2 * ACC) <= 128 ? 128 : (2 * ACC) <= 256 ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BR = g.br, S = g.splits, CS = g.cs;
  const int KB = g.kblocks / S;  // k-blocks per item (the host makes splits divide kblocks)
  // CS CTAs of a cluster take CS adjacent row blocks of the same K split in lockstep and
  // multicast the shared activation tile (each loads BN/CS rows of it for everyone).
  // Work group j = (block group j / S, split j % S); cluster q takes groups q, q+Q, ...
  const int rank = CS > 1 ? (int)cluster_ctarank() : 0;
  const int q = blockIdx.x / CS, Q = gridDim.x / CS;
  const int groups = ((g.nblocks + CS - 1) / CS) * S;
  const int my_blocks = groups > q ? (groups - q + Q - 1) / Q : 0;
  const int my_units = my_blocks * KB;
  const uint16_t cmask = (uint16_t)((1u << CS) - 1);
  const int xrows = BN / CS;
  const uint32_t x_bytes_own = (uint32_t)xrows * BK * 2;
  const uint32_t a_bytes = (uint32_t)BR * BK * 2;  // one A tile: BR rows (the UMMA reads 128; extra rows ignored)
  const int NS = g.ns, STAGE = g.stage_bytes;
  const int A_BYTES = (int)a_bytes;
  pdl_launch_dependents();
  if (g.stats && threadIdx.x == 0) g.stats[blockIdx.x * 8 + 4] = clock64();

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    for (int i = 0; i < NS; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], CS); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers' barriers exist before anyone multicasts into them
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  if (g.stats && threadIdx.x == 32) g.stats[blockIdx.x * 8 + 1] = clock64();  // setup done

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer: one continuous ring over the CTA's blocks
      // PDL: W does not depend on the previous kernel, so the first NS stages of W are
      // requested before griddepcontrol.wait; the stage's single arrival comes with its
      // X half, so a stage can never complete on its W bytes alone.
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      const int npre = min(NS, my_units);
      auto unit = [&](int i, int& blk, int& kc) {
        const int j = q + (i / KB) * Q;
        blk = (j / S) * CS + rank;
        kc = ((j % S) * KB + i % KB) * BK;
      };
      for (int i = 0; i < npre; ++i) {
        int blk, kc;
        unit(i, blk, kc);
        uint8_t* st = smem + i * STAGE;
        mbar_expect_tx_noarrive(&full_bar[i], NA * a_bytes);
        tma_load_2d(st, &wmap, kc, blk * g.row_mul, &full_bar[i], pw);
        if (NA == 2) tma_load_2d(st + A_BYTES, &wmap, kc, blk * g.row_mul + g.a2_base, &full_bar[i], pw);
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      auto load_x = [&](int i, int s) {
        int blk, kc;
        unit(i, blk, kc);
        uint8_t* xs = smem + s * STAGE + NA * A_BYTES;
        if (CS > 1)
          tma_load_2d_mc(xs + rank * x_bytes_own, &xmap, kc, rank * xrows, &full_bar[s], cmask, px);
        else
          tma_load_2d(xs, &xmap, kc, 0, &full_bar[s], px);
      };
      for (int i = 0; i < npre; ++i) {
        mbar_expect_tx(&full_bar[i], B_BYTES);  // the whole tile: own part + the peers' multicasts
        load_x(i, i);
      }
      long long t_wait = 0, t_begin = clock64();
      for (int i = npre; i < my_units; ++i) {
        const int s = i % NS, r = i / NS;
        long long t0 = clock64();
        mbar_wait(&empty_bar[s], (r - 1) & 1);  // consumed by every CTA of the cluster
        t_wait += clock64() - t0;
        uint8_t* st = smem + s * STAGE;
        if (g.dbg & 1) {
          mbar_arrive_local(&full_bar[s]);
          continue;
        }
        mbar_expect_tx(&full_bar[s], NA * a_bytes + B_BYTES);
        int blk, kc;
        unit(i, blk, kc);
        tma_load_2d(st, &wmap, kc, blk * g.row_mul, &full_bar[s], pw);
        if (NA == 2) tma_load_2d(st + A_BYTES, &wmap, kc, blk * g.row_mul + g.a2_base, &full_bar[s], pw);
        load_x(i, s);
      }
      if (g.stats) {
        g.stats[blockIdx.x * 8 + 0] = t_wait;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      long long m_wait = 0, m_begin = clock64();
      for (int blk_i = 0, i = 0; blk_i < my_blocks; ++blk_i) {
        const int buf = blk_i & 1;
        if (blk_i >= 2) mbar_wait(&tempty_bar[buf], ((blk_i >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * ACC;
        for (int kb = 0; kb < KB; ++kb, ++i) {
          const int s = i % NS, r = i / NS;
          long long t0 = clock64();
          mbar_wait(&full_bar[s], r & 1);
          m_wait += clock64() - t0;
          if (g.stats && i == 0) g.stats[blockIdx.x * 8 + 5] = clock64();
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * STAGE);
          const uint32_t sb = sa + NA * A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t bdesc = desc_sw128(sb + k * 32);
            const uint32_t accum = (kb == 0 && k == 0) ? 0u : 1u;
            umma(acc, desc_sw128(sa + k * 32), bdesc, idesc, accum);
            if (NA == 2) umma(acc + BN, desc_sw128(sa + A_BYTES + k * 32), bdesc, idesc, accum);
          }
          if (CS > 1) umma_commit_mc(&empty_bar[s], cmask);  // frees the slot in every CTA of the cluster
          else umma_commit(&empty_bar[s]);
        }
        umma_commit(&tfull_bar[buf]);
      }
      if (g.stats) {
        g.stats[blockIdx.x * 8 + 2] = m_wait;
        g.stats[blockIdx.x * 8 + 3] = clock64() - m_begin;
        g.stats[blockIdx.x * 8 + 6] = clock64();
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue warps: thread t <-> TMEM lane t <-> weight row blk*BR + t
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int t = threadIdx.x - 128;
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int mode = g.mode;
    for (int blk_i = 0; blk_i < my_blocks; ++blk_i) {
      const int buf = blk_i & 1;
      const int j = q + blk_i * Q;
      const int item_split = j % S;
      const int blk = (j / S) * CS + rank;
      const int n = blk * g.row_mul + t;                       // row of accumulator 0
      const int n2 = blk * g.row_mul + g.a2_base + t;          // row of accumulator 1 (paired tiles)
      const bool swiglu = mode == SN_GEMM_SWIGLU;
      mbar_wait(&tfull_bar[buf], (blk_i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + lane_off + buf * ACC;
      // store 16 batch columns [col, col+16) of one output row
      auto emit = [&](int row, int col, const float* v) {
        if (t >= BR || row >= g.N) return;
        if (mode == SN_GEMM_PARTIAL) {
          float* o = reinterpret_cast<float*>(g.out) + (size_t)item_split * g.M * g.ldo + row;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (col + jj < g.M) __stcg(o + (size_t)(col + jj) * g.ldo, v[jj]);
        } else if (mode == SN_GEMM_RESID) {
          float* o = reinterpret_cast<float*>(g.out) + row;
          float old[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) old[jj] = (col + jj < g.M) ? __ldcg(o + (size_t)(col + jj) * g.ldo) : 0.f;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (col + jj < g.M) o[(size_t)(col + jj) * g.ldo] = old[jj] + v[jj];
        } else {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out) + row;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            if (col + jj < g.M) o[(size_t)(col + jj) * g.ldo] = __float2bfloat16_rn(v[jj]);
        }
      };
#pragma unroll 1
      for (int col = 0; col < BN; col += 16) {
        float v[16], w2[16];
        tmem_ld16(acc + col, v);
        if (NA == 2) tmem_ld16(acc + BN + col, w2);
        if (NA == 2 && swiglu) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = silu_f(v[jj]) * w2[jj];
          emit(n, col, v);
        } else {
          emit(n, col, v);
          if (NA == 2) emit(n2, col, w2);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      named_bar(1, 128);
      if (t == 0) mbar_arrive_local(&tempty_bar[buf]);
    }
  }

  __syncwarp();  // warps 0/1 diverged (one elected lane each): reconverge before the CTA barrier
  __syncthreads();
  if (g.stats && threadIdx.x == 0) g.stats[blockIdx.x * 8 + 7] = clock64();
  if (CS > 1) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}
// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static bool map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                   uint32_t box_rows) {
  // (box_rows <= 256; for W it is the block height BR, for X the batch tile BN)
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Work decomposition.  Per-CTA time ~ waves x k-blocks-per-item x (NA*BR + BN) bytes;
// BR >= 48 keeps >= 1.5 KB of W per UMMA (tcgen05.mma issues at ~45 cycles minimum,
// measured), split-K (PARTIAL mode only: the consumer sums the slabs) lets a narrow N
// fill the SMs with tall blocks.  Ties -> fewer splits, then taller blocks.
static unsigned long long* g_stats = nullptr;  // sn_gemm_debug_stats(): profiling only
static int g_cluster = -1;  // CTAs per multicast cluster (env SN_GEMM_CLUSTER, default 2)

static int cluster_size() {
  if (g_cluster < 0) {
    const char* e = getenv("SN_GEMM_CLUSTER");
    g_cluster = e ? atoi(e) : 1;
    if (g_cluster != 1 && g_cluster != 2 && g_cluster != 4) g_cluster = 2;
  }
  return g_cluster;
}

static void pick_tiling(int N, int kblocks, int sms, int na, int bn, int max_splits, int* br_out,
                        int* splits_out) {
  long best_cost = -1;
  const int cs = cluster_size();
  for (int s = 1; s <= max_splits; ++s) {
    if (kblocks % s) continue;
    for (int br = BM; br >= 48; br -= 8) {
      const long items = (long)((N + br * cs - 1) / (br * cs)) * cs * s;
      const long waves = (items + sms - 1) / sms;
      const long cost = waves * (kblocks / s) * (long)(na * br + bn);
      if (best_cost < 0 || cost < best_cost) { best_cost = cost; *br_out = br; *splits_out = s; }
    }
  }
}

static int batch_tile(int M) { return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : 128; }

template <int BN, int NA>
static sn_status launch(const CUtensorMap& wm, const CUtensorMap& xm, GemmArgs g, int grid, cudaStream_t st) {
  constexpr int kSmemMax = 227 * 1024;          // per-CTA opt-in maximum on sm_100
  const int stage = NA * g.br * BK * 2 + BN * BK * 2;
  const int tail = BM * BK * 2;  // the M=128 UMMA of the last stage may read 128 rows past its A tile
  static int budget = getenv("SN_GEMM_SMEM_KB") ? atoi(getenv("SN_GEMM_SMEM_KB")) * 1024 : kSmemMax;
  int ns = ((budget < kSmemMax ? budget : kSmemMax) - 2048 - tail) / stage;  // 1 KB alignment slack + barriers
  if (ns < 2) ns = 2;
  if (ns > kMaxStages) ns = kMaxStages;
  g.ns = ns;
  g.stage_bytes = stage;
  static int dbg = getenv("SN_GEMM_DBG") ? atoi(getenv("SN_GEMM_DBG")) : 0;
  g.dbg = dbg;
  const int smem = ns * stage + tail + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_decode_kernel<BN, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax - 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: overlap with the producer's tail
  attrs[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attrs[1].id = cudaLaunchAttributeClusterDimension;
  attrs[1].val.clusterDim.x = g.cs;
  attrs[1].val.clusterDim.y = 1;
  attrs[1].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_decode_kernel<BN, NA>, wm, xm, g);
  if (e != cudaSuccess) {
    set_error("sn_gemm_decode launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_gemm_decode");
}

struct Plan {
  int bn, br, splits, na, row_mul, nblocks, cs, grid;
  bool swiglu, pair;
};

// Tiling plan: two 128-row A tiles per stage whenever N allows (SwiGLU gate+up, or two
// stacked row blocks) so each activation tile feeds 256 weight rows (smem traffic per W
// byte 2.5 instead of 3), block height / split-K from pick_tiling, multicast cluster size.
static Plan make_plan(int M, int N, int K, int mode) {
  Plan p{};
  static int pair_env = getenv("SN_GEMM_PAIR") ? atoi(getenv("SN_GEMM_PAIR")) : 1;
  const int sms = num_sms();
  p.bn = batch_tile(M);
  p.swiglu = mode == SN_GEMM_SWIGLU;
  p.pair = !p.swiglu && pair_env && N >= 2 * BM;
  p.na = (p.swiglu || p.pair) ? 2 : 1;
  p.br = BM;
  p.splits = 1;
  pick_tiling(p.pair ? (N + 1) / 2 : N, K / BK, sms, p.na, p.bn, mode == SN_GEMM_PARTIAL ? 8 : 1, &p.br, &p.splits);
  if (const char* f = getenv("SN_GEMM_FORCE")) {  // experiments: "br,splits"
    int br = 0, sp = 0;
    if (sscanf(f, "%d,%d", &br, &sp) == 2 && br >= 8 && br <= BM && br % 8 == 0 && sp >= 1 &&
        (K / BK) % sp == 0 && (sp == 1 || mode == SN_GEMM_PARTIAL)) {
      p.br = br;
      p.splits = sp;
    }
  }
  p.row_mul = p.pair ? 2 * p.br : p.br;
  p.nblocks = (N + p.row_mul - 1) / p.row_mul;
  p.cs = cluster_size();
  if (p.nblocks < p.cs || p.bn / p.cs < 8) p.cs = 1;
  const int groups = ((p.nblocks + p.cs - 1) / p.cs) * p.splits;
  const int clusters = groups < sms / p.cs ? groups : sms / p.cs;
  p.grid = clusters * p.cs;
  return p;
}

}  // namespace gemm
}  // namespace sn

namespace sn {
int gemm2_splits(int M, int N, int K, int mode);
int gemm2_swiglu_block(int M, int N, int K);
void gemm2_debug_stats(unsigned long long* s);
sn_status gemm2_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                       int mode, int* splits_out, cudaStream_t st);
}  // namespace sn

using namespace sn;
using namespace sn::gemm;

// Kernel generation: 2 = batch-as-M (sn_gemm2.cu, default), 1 = weights-as-M (this file).
static int gemm_version() {
  static int v = getenv("SN_GEMM_V") ? atoi(getenv("SN_GEMM_V")) : 2;
  return v;
}

extern "C" {

// Profiling aid: later launches write per-CTA counters [producer empty-wait, producer total,
// MMA full-wait, MMA total (clock64); entry, first stage landed, last MMA issued, exit
// (%globaltimer ns)] into dev_stats (8 x #SMs u64); NULL disables.
void sn_gemm_debug_stats(unsigned long long* dev_stats) {
  g_stats = dev_stats;
  gemm2_debug_stats(dev_stats);
}

int sn_gemm_swiglu_block(int M, int N, int K) { return gemm_version() == 2 ? gemm2_swiglu_block(M, N, K) : 0; }

int sn_gemm_decode_splits(int M, int N, int K, int mode) {
  if (gemm_version() == 2) return gemm2_splits(M, N, K, mode);
  if (K % BK || mode != SN_GEMM_PARTIAL) return 1;
  return make_plan(M, N, K, mode).splits;
}

sn_status sn_gemm_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                         int mode, int* splits_out, void* stream) {
  SN_REQUIRE(x && w && out, "sn_gemm_decode: NULL pointer");
  SN_REQUIRE(M >= 1 && M <= 128, "sn_gemm_decode: M=%d must be in [1, 128] (decode batch)", M);
  SN_REQUIRE(K % BK == 0 && K >= BK, "sn_gemm_decode: K=%d must be a multiple of %d", K, BK);
  SN_REQUIRE(N >= 1 && ldw >= K && ldx >= K, "sn_gemm_decode: bad N/ld");
  SN_REQUIRE(mode == SN_GEMM_STORE || mode == SN_GEMM_SWIGLU || mode == SN_GEMM_RESID || mode == SN_GEMM_PARTIAL ||
                 (mode == SN_GEMM_SWIGLU_IL && gemm_version() == 2),
             "sn_gemm_decode: mode %d", mode);
  SN_REQUIRE(((uintptr_t)x % 16) == 0 && ((uintptr_t)w % 16) == 0 && (ldx % 8) == 0 && (ldw % 8) == 0,
             "sn_gemm_decode: operands must be 16-byte aligned");
  if (gemm_version() == 2) return gemm2_decode(x, M, K, ldx, w, N, ldw, out, ldo, mode, splits_out, (cudaStream_t)stream);
  const Plan pl = make_plan(M, N, K, mode);
  CUtensorMap wm, xm;
  const uint64_t wrows = pl.swiglu ? 2ull * N : (uint64_t)N;
  if (!map_2d(&wm, w, wrows, K, ldw, pl.br) || !map_2d(&xm, x, M, K, ldx, pl.bn / pl.cs)) {
    set_error("sn_gemm_decode: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  if (splits_out) *splits_out = pl.splits;
  GemmArgs g{out, M, N, K, ldo, mode, K / BK, pl.br, pl.nblocks, pl.splits, pl.cs, g_stats, pl.row_mul,
             pl.swiglu ? N : pl.br, 0, 0};
  cudaStream_t st = (cudaStream_t)stream;
  if (pl.na == 2) {
    switch (pl.bn) {
      case 16: return launch<16, 2>(wm, xm, g, pl.grid, st);
      case 32: return launch<32, 2>(wm, xm, g, pl.grid, st);
      case 64: return launch<64, 2>(wm, xm, g, pl.grid, st);
      default: return launch<128, 2>(wm, xm, g, pl.grid, st);
    }
  }
  switch (pl.bn) {
    case 16: return launch<16, 1>(wm, xm, g, pl.grid, st);
    case 32: return launch<32, 1>(wm, xm, g, pl.grid, st);
    case 64: return launch<64, 1>(wm, xm, g, pl.grid, st);
    default: return launch<128, 1>(wm, xm, g, pl.grid, st);
  }
}

}  // extern "C"
