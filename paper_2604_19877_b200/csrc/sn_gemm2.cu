// Decode GEMM, batch-as-M formulation (tcgen05 + TMEM + TMA).
//
// C[m][n] = sum_k X[m][k] * W[n][k] with a decode batch M <= 128 and a weight W [N x K]
// streamed from HBM once.  The activation tile X [M x 64] is the UMMA A operand (M = 64 or
// 128 rows, zero-filled past the batch) and a block of up to 256 weight rows is the B
// operand, so one tcgen05.mma (M=64, N=256, K=16) covers a 256-row weight block.
//
// Why not weights-as-M: with W as the M=128 operand every 128 weight rows need their own
// UMMA per k-step and each re-reads the activation tile; measured on B200
// (tools/umma_bench.cu, tools/gemm_force.py) the single issuing thread then spends
// ~120 cycles per M=128 x N=64 UMMA once the stage barrier waits and commits are in the
// loop, which caps a CTA at ~55 GB/s of weights.  An M=64 x N=256 UMMA runs 128 cycles
// of tensor time for 4x the weight bytes, so the issue overhead hides under it and the
// activation tile is read once per k-step.
//
// Work: units (row block, K split) are dealt round-robin to a persistent grid (<= #SMs);
// the host picks the block height and split count that balance 148 SMs (make_plan).
// Warp roles: 0 = TMA producer, 1 = MMA issuer, 2 = TMEM allocator, 4-7 = epilogue
// (TMEM -> registers -> global).  Two TMEM accumulators so a block's epilogue overlaps
// the next block's MMAs.  PDL: the first stages of W are requested before
// griddepcontrol.wait (weights do not depend on the previous kernel).
//
// Epilogues: STORE (bf16), SWIGLU (W = [gate; up], block = half gate rows + half up rows,
// out = silu(g) * u), RESID (fp32 residual += acc), PARTIAL (fp32 split-K slab per split,
// summed by the consumer in a fixed order -> deterministic).
#include <cuda.h>
#include <stdlib.h>

#include "sn_common.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace gemm2 {

using namespace sn::tc;
constexpr int kThreads = 256;
constexpr int kMaxStages = 16;
constexpr int kMaxRows = 256;     // UMMA N limit

struct Args {
  void* out;     // bf16 [M][ldo] | fp32 residual [M][ldo] | fp32 slabs [splits][M][ldo]
  int M, N, K, ldo, mode, kblocks;
  int br;        // weight rows per block = UMMA N (multiple of 16, <= 256); SWIGLU: br/2 gate + br/2 up
  int nblocks;   // row blocks
  int splits;    // K splits per block (PARTIAL only)
  int ns;        // pipeline stages
  int stage_bytes;
  int acc_cols;  // TMEM columns per accumulator buffer
  unsigned long long* stats;
  int dbg;       // experiments (env SN_GEMM_DBG): 2 = no epilogue stores
  int pre;       // W stages requested before griddepcontrol.wait
  int ks;        // 64-column K atoms per pipeline stage (amortises the per-stage barrier cost)
};

// smem stage: [ KS X atoms: UM rows x 128 B | KS W atoms: br rows x 128 B ]
template <int UM>
__global__ void __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = g.splits, KB = g.kblocks / S, BR = g.br, NS = g.ns, STAGE = g.stage_bytes;
  const int KS = g.ks, KU = KB / KS;  // 64-column atoms per stage, stages per item
  const bool swiglu = g.mode == SN_GEMM_SWIGLU || g.mode == SN_GEMM_SWIGLU_IL;
  const bool interleaved = g.mode == SN_GEMM_SWIGLU_IL;
  const int half = BR >> 1;
  const int q = blockIdx.x, Q = gridDim.x;
  const int items = g.nblocks * S;
  const int my_items = items > q ? (items - q + Q - 1) / Q : 0;
  const int my_units = my_items * KU;
  constexpr uint32_t X_BYTES = UM * BK * 2;
  const uint32_t w_bytes = (uint32_t)BR * BK * 2;  // one 64-column atom of the weight block
  const int w_atom = (int)w_bytes;
  const int tmem_cols = 2 * g.acc_cols;
  pdl_launch_dependents();
  if (g.stats && threadIdx.x == 0) g.stats[blockIdx.x * 8 + 4] = clock64();

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xmap)) : "memory");
    for (int i = 0; i < NS; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      // unit = (item, k-step of KS 64-column atoms); walked with incremental counters
      int it = 0, ku = 0, s = 0;
      uint32_t ph = 0;
      auto load = [&](bool w_part, bool x_part) {
        const int j = q + it * Q;
        const int blk = j / S;
        const int kc0 = ((j % S) * KB + ku * KS) * BK;
        uint8_t* st = smem + s * STAGE;
#pragma unroll 1
        for (int a = 0; a < KS; ++a) {
          const int kc = kc0 + a * BK;
          if (w_part) {
            uint8_t* wt = st + KS * X_BYTES + a * w_atom;
            if (swiglu && !interleaved) {
              tma_load_2d(wt, &wmap, kc, blk * half, &full_bar[s], pw);
              tma_load_2d(wt + half * 128, &wmap, kc, g.N + blk * half, &full_bar[s], pw);
            } else {
              tma_load_2d(wt, &wmap, kc, blk * BR, &full_bar[s], pw);
            }
          }
          if (x_part) tma_load_2d(st + a * X_BYTES, &xmap, kc, 0, &full_bar[s], px);
        }
      };
      auto advance = [&]() {
        if (++ku == KU) { ku = 0; ++it; }
        if (++s == NS) { s = 0; ph ^= 1; }
      };
      // Only the first g.pre stages of W are requested before griddepcontrol.wait: the
      // activation tile of stage 0 queues behind them, so a deep W burst delays the first MMA.
      const int npre = min(min(NS, g.pre), my_units);
      for (int u = 0; u < npre; ++u) {
        mbar_expect_tx_noarrive(&full_bar[s], KS * w_bytes);
        load(true, false);
        advance();
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      it = 0; ku = 0; s = 0; ph = 0;
      for (int u = 0; u < npre; ++u) {
        mbar_expect_tx(&full_bar[s], KS * X_BYTES);
        load(false, true);
        advance();
      }
      for (int u = npre; u < my_units; ++u) {
        if (u >= NS) mbar_wait(&empty_bar[s], ph ^ 1);
        mbar_expect_tx(&full_bar[s], KS * (w_bytes + X_BYTES));
        load(true, true);
        advance();
      }
      if (g.stats) g.stats[blockIdx.x * 8 + 1] = clock64();
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (whole warp converged, one elected lane issues)
      const uint32_t idesc = idesc_bf16(UM, BR);
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0; it < my_items; ++it) {
        const int buf = it & 1;
        if (it >= 2) mbar_wait(&tempty_bar[buf], ((it >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * g.acc_cols;
        for (int ku = 0; ku < KU; ++ku) {
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sx = smem_u32(smem + s * STAGE);
          const uint32_t sw = sx + KS * X_BYTES;
#pragma unroll 1
          for (int a = 0; a < KS; ++a) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_w(acc, desc_sw128(sx + a * X_BYTES + k * 32), desc_sw128(sw + a * w_atom + k * 32), idesc,
                   (ku | a | k) ? 1u : 0u);
          }
          commit_w(&empty_bar[s]);
          if (++s == NS) { s = 0; ph ^= 1; }
        }
        commit_w(&tfull_bar[buf]);
      }
      if (g.stats && lane == 0) g.stats[blockIdx.x * 8 + 6] = clock64();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp w drains TMEM lanes [32*(w%4), +32); lane <-> batch row
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int sp = warp & 3;
    // UM=64: the accumulator occupies lanes 0-15 of each 32-lane subpartition (row 16*sp + t)
    const int m = UM == 64 ? 16 * sp + lane : 32 * sp + lane;
    const bool row_ok = (UM == 64 ? lane < 16 : true) && m < g.M;
    const uint32_t lane_addr = (uint32_t)(32 * sp) << 16;
    const int mode = g.mode;
    const bool vec = (g.ldo & 7) == 0;
    // store 16 consecutive output columns [n, n+16) of batch row m
    auto emit = [&](float* v, int n, int split) {
      const bool full = vec && n + 16 <= g.N;
      if (mode == SN_GEMM_PARTIAL || mode == SN_GEMM_RESID) {
        float* o = reinterpret_cast<float*>(g.out) + ((size_t)(mode == SN_GEMM_PARTIAL ? split : 0) * g.M + m) * g.ldo + n;
        if (full) {
          if (mode == SN_GEMM_RESID) {
#pragma unroll
            for (int e = 0; e < 16; e += 4) {
              const float4 old = __ldcg(reinterpret_cast<const float4*>(o + e));
              v[e] += old.x; v[e + 1] += old.y; v[e + 2] += old.z; v[e + 3] += old.w;
            }
          }
#pragma unroll
          for (int e = 0; e < 16; e += 4)
            __stcg(reinterpret_cast<float4*>(o + e), make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (n + e < g.N) o[e] = v[e] + (mode == SN_GEMM_RESID ? o[e] : 0.f);
        }
      } else {  // STORE / SWIGLU: bf16
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(g.out) + (size_t)m * g.ldo + n;
        if (full) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            pk[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
          reinterpret_cast<uint4*>(o)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          reinterpret_cast<uint4*>(o)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (n + e < g.N) o[e] = __float2bfloat16_rn(v[e]);
        }
      }
    };
    for (int it = 0; it < my_items; ++it) {
      const int buf = it & 1;
      const int j = q + it * Q;
      const int blk = j / S, split = j % S;
      mbar_wait(&tfull_bar[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + lane_addr + buf * g.acc_cols;
      const int ncols = swiglu ? half : BR;
      const int n_base = swiglu ? blk * half : blk * BR;
      // 64 columns per round: up to 4 (SwiGLU: 8) TMEM loads in flight, one wait
#pragma unroll 1
      for (int c0 = 0; c0 < ncols; c0 += 64) {
        float v[4][16], u[4][16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          if (c0 + 16 * q4 < ncols) {
            tmem_ld16_async(acc + c0 + 16 * q4, v[q4]);
            if (swiglu) tmem_ld16_async(acc + half + c0 + 16 * q4, u[q4]);
          }
        }
        tmem_wait_ld();
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          reg_fence16(v[q4]);
          if (swiglu) reg_fence16(u[q4]);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int c = c0 + 16 * q4;
          const int n = n_base + c;
          if (c >= ncols || !row_ok || n >= g.N || (g.dbg & 2)) continue;
          float* vv = v[q4];
          if (swiglu) {
#pragma unroll
            for (int e = 0; e < 16; ++e) vv[e] = silu_f(vv[e]) * u[q4][e];
          }
          emit(vv, n, split);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[buf]);  // 4 epilogue warps -> count 4
    }
    if (g.stats && threadIdx.x == 128) g.stats[blockIdx.x * 8 + 7] = clock64();
  }
  __syncwarp();
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// ------------------------------------------------------------------ host
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

struct Plan {
  int um, br, splits, nblocks, grid;
};

// Per-CTA time ~ waves x k-blocks per unit x weight rows (+ a small activation-tile term)
// + the split-K slab traffic the consumer pays.  Ties ->
// fewer splits, then taller blocks.
static Plan make_plan(int M, int N, int K, int mode) {
  Plan p{};
  const int sms = num_sms();
  const int kblocks = K / BK;
  p.um = M <= 64 ? 64 : 128;
  const bool swiglu = mode == SN_GEMM_SWIGLU || mode == SN_GEMM_SWIGLU_IL;
  const int max_splits = mode == SN_GEMM_PARTIAL ? 8 : 1;
  double best = -1;
  for (int s = 1; s <= max_splits; ++s) {
    if (kblocks % s) continue;
    // SwiGLU blocks hold br/2 gate + br/2 up rows; the epilogue drains 16 columns at a time
    for (int br = kMaxRows; br >= 32; br -= swiglu ? 32 : 16) {
      const long blocks = swiglu ? (N + br / 2 - 1) / (br / 2) : (N + br - 1) / br;
      const long items = blocks * s;
      const long waves = (items + sms - 1) / sms;
      // the activation tile is an L2 hit and measured free (SN_GEMM_DBG=4): weigh it lightly
      const double cost = (double)waves * (kblocks / s) * (br + p.um / 8) * 128.0 +
                          (s > 1 ? (double)s * M * N * 8.0 / sms : 0.0);
      if (best < 0 || cost < best * 0.999) { best = cost; p.br = br; p.splits = s; }
    }
  }
  if (const char* f = getenv("SN_GEMM_FORCE")) {  // experiments: "br,splits"
    int br = 0, sp = 0;
    if (sscanf(f, "%d,%d", &br, &sp) == 2 && br >= 16 && br <= kMaxRows && br % (swiglu ? 32 : 16) == 0 && sp >= 1 &&
        kblocks % sp == 0 && (sp == 1 || mode == SN_GEMM_PARTIAL)) {
      p.br = br;
      p.splits = sp;
    }
  }
  p.nblocks = swiglu ? (N + p.br / 2 - 1) / (p.br / 2) : (N + p.br - 1) / p.br;
  const int items = p.nblocks * p.splits;
  p.grid = items < sms ? items : sms;
  return p;
}

static unsigned long long* g_stats2 = nullptr;

template <int UM>
static sn_status launch(const CUtensorMap& wm, const CUtensorMap& xm, Args g, int grid, cudaStream_t st) {
  constexpr int kSmemMax = 227 * 1024;
  // K atoms per stage: >= 32 KB of weights per stage barrier round trip (the issuing
  // thread pays ~500 cycles per stage for the wait/commit/descriptors), >= 3 stages.
  static int ks_env = getenv("SN_GEMM_KS") ? atoi(getenv("SN_GEMM_KS")) : 0;
  const int kb_item = g.kblocks / g.splits;
  int ks = 1;
  if (ks_env > 0) {
    ks = ks_env;
    while (ks > 1 && kb_item % ks) ks >>= 1;
  } else {
    while (ks < 4 && g.br * BK * 2 * ks < 32768 && kb_item % (2 * ks) == 0 &&
           (kSmemMax - 2048) / (2 * ks * (UM + g.br) * BK * 2) >= 3)
      ks *= 2;
  }
  g.ks = ks;
  const int stage = ks * (UM * BK * 2 + g.br * BK * 2);
  int ns = (kSmemMax - 2048) / stage;
  if (ns > kMaxStages) ns = kMaxStages;
  g.ns = ns;
  g.stage_bytes = stage;
  int cols = 32;
  while (cols < g.br) cols <<= 1;
  g.acc_cols = cols;
  const int smem = ns * stage + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm2_kernel<UM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax - 1024);
    attr = true;
  }
  cudaError_t e = launch_pdl(gemm2_kernel<UM>, dim3(grid), dim3(kThreads), (size_t)smem, st, wm, xm, g);
  if (e != cudaSuccess) {
    set_error("sn_gemm_decode launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_gemm_decode");
}

}  // namespace gemm2

// Entry used by sn_gemm_decode (sn_gemm.cu).
int gemm2_swiglu_block(int M, int N, int K) {
  if (K % gemm2::BK) return 0;
  return gemm2::make_plan(M, N, K, SN_GEMM_SWIGLU_IL).br / 2;
}

int gemm2_splits(int M, int N, int K, int mode) {
  if (K % gemm2::BK || mode != SN_GEMM_PARTIAL) return 1;
  return gemm2::make_plan(M, N, K, mode).splits;
}

void gemm2_debug_stats(unsigned long long* s) { gemm2::g_stats2 = s; }

sn_status gemm2_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                       int mode, int* splits_out, cudaStream_t st) {
  using namespace gemm2;
  const Plan pl = make_plan(M, N, K, mode);
  CUtensorMap wm, xm;
  const bool swiglu = mode == SN_GEMM_SWIGLU;
  // SWIGLU_IL: W pre-interleaved in blocks of [h gate rows; h up rows] (h = sn_gemm_swiglu_block)
  const uint64_t wrows = mode == SN_GEMM_SWIGLU_IL ? (uint64_t)pl.nblocks * pl.br : swiglu ? 2ull * N : (uint64_t)N;
  if (!map_2d(&wm, w, wrows, K, ldw, swiglu ? pl.br / 2 : pl.br) || !map_2d(&xm, x, M, K, ldx, pl.um)) {
    set_error("sn_gemm_decode: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  if (splits_out) *splits_out = pl.splits;
  static int dbg = getenv("SN_GEMM_DBG") ? atoi(getenv("SN_GEMM_DBG")) : 0;
  static int pre = getenv("SN_GEMM_PRE") ? atoi(getenv("SN_GEMM_PRE")) : 2;
  Args g{out, M, N, K, ldo, mode, K / BK, pl.br, pl.nblocks, pl.splits, 0, 0, 0, g_stats2, dbg, pre};
  return pl.um == 64 ? launch<64>(wm, xm, g, pl.grid, st) : launch<128>(wm, xm, g, pl.grid, st);
}

}  // namespace sn
