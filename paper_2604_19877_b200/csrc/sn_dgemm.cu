// Decode GEMM: C[m][n] = sum_k X[m][k] * W[n][k] for a decode batch M <= 128 and a weight
// matrix W [N x K] streamed from HBM exactly once, with the consumer's elementwise work fused
// into the epilogue (sn_epi.cuh).  Every projection of the decode step runs here: the mixer
// in-projections (R/PAPER.md:1542-1544, 1584-1587, 1614-1622), the out-projections, the FFN
// gate/up (SwiGLU fused) and down-projection, and the LM head.
//
// bf16: tcgen05 + TMEM + TMA, batch-as-M.  The activation tile X [UM x 64] (UM = 64 or 128,
// zero-filled past the batch) is the UMMA A operand and a block of br weight rows (br = 64,
// 128 or 256) the B operand, so one tcgen05.mma (M=UM, N=br, K=16) covers the whole block and
// the weight bytes are read once.  (Weights-as-M was measured at ~120 issue cycles per
// M=128 x N=64 UMMA, capping an SM at ~55 GB/s, profiles/r01_decode_ablation.md.)
//
// Work split: items = (row block, K split) dealt round-robin to a persistent grid of <= #SM
// CTAs; the host picks the block height and split count that minimise the bytes the busiest
// CTA streams (make_plan).  Measured on B200 (profiles/r02_gemm_plans.md): whole blocks per CTA
// stream at 5.4-6.1 TB/s even when only 80-130 SMs hold one; a stream-K split of blocks across
// CTAs with a last-arriver fix-up was 25-50 % slower — the fix-up (fp32 partial tiles through
// L2 under full HBM load) sits on every kernel's critical path.  K splits are therefore only
// used where the consumer can take them: mode PARTIAL writes one fp32 slab per split and the
// next add + RMSNorm sums the slabs in a fixed order (deterministic).
//
// Warp roles: 0 = TMA producer, 1 = MMA issuer (warp-converged, one elected lane), 2 = TMEM
// allocator, 4-7 = epilogue (TMEM -> registers -> finalize).  Two TMEM accumulators: one
// segment's epilogue overlaps the next segment's MMAs.  Programmatic dependent launch: the
// first weight stages are requested before griddepcontrol.wait.
//
// fp32 (numerics mode, SN_F32 I/O): a CUDA-core tile kernel with the same epilogues.
#include <cuda.h>
#include <stdlib.h>

#include "sn_common.cuh"
#include "sn_dplan.cuh"
#include "sn_epi.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace dgemm {

using namespace sn::tc;
constexpr int kThreads = 256;
constexpr int kMaxStages = 16;
constexpr int kMaxBr = 256;          // UMMA N limit
constexpr int kMaxSplits = 8;

struct Args {
  int K, kb;      // reduction length, 64-column atoms
  int br;         // weight rows per block (UMMA N)
  int nblocks;    // row blocks
  int splits;     // K splits per block (PARTIAL only)
  int ks;         // atoms per unit (pipeline stage)
  int ku;         // units per item
  int ns, stage_bytes, acc_cols;
  epi::Args e;
};

template <int UM>
__global__ void __launch_bounds__(kThreads, 1)
    dgemm_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap, const Args g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int BR = g.br, NS = g.ns, STAGE = g.stage_bytes, KS = g.ks, KU = g.ku, S = g.splits;
  const int q = blockIdx.x, G = gridDim.x;
  const int items = g.nblocks * S;
  const int my_items = items > q ? (items - q + G - 1) / G : 0;
  const int my_units = my_items * KU;
  constexpr uint32_t X_BYTES = UM * BK * 2;
  const uint32_t w_bytes = (uint32_t)BR * BK * 2;  // one 64-column atom of the weight block
  const int tmem_cols = 2 * g.acc_cols;
  pdl_launch_dependents();

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
      int it = 0, ku = 0, s = 0;  // unit = (item, k-step of KS atoms), walked with counters
      uint32_t ph = 0;
      auto load = [&](bool w_part, bool x_part) {
        const int j = q + it * G;
        const int blk = j / S;
        const int kc0 = ((j % S) * KU + ku) * KS * BK;
        uint8_t* st = smem + s * STAGE;
#pragma unroll 1
        for (int a = 0; a < KS; ++a) {
          const int kc = kc0 + a * BK;
          if (w_part) tma_load_2d(st + KS * X_BYTES + a * w_bytes, &wmap, kc, blk * BR, &full_bar[s], pw);
          if (x_part) tma_load_2d(st + a * X_BYTES, &xmap, kc, 0, &full_bar[s], px);
        }
      };
      auto advance = [&]() {
        if (++ku == KU) { ku = 0; ++it; }
        if (++s == NS) { s = 0; ph ^= 1; }
      };
      // the first stages of W do not depend on the previous kernel: requested before the wait
      // (only two: the activation tile of stage 0 queues behind them)
      const int npre = min(min(NS, 2), my_units);
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
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (whole warp converged, one elected lane issues)
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
            umma_w(acc, desc_sw128(sx + a * X_BYTES + k * 32), desc_sw128(sw + a * w_bytes + k * 32), idesc,
                   (ku | a | k) ? 1u : 0u);
        }
        commit_w(&empty_bar[s]);
        if (++s == NS) { s = 0; ph ^= 1; }
      }
      commit_w(&tfull_bar[buf]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: warp w drains TMEM lanes [32*(w%4), +32); lane <-> batch row
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int sp = warp & 3;
    // UM=64: the accumulator occupies lanes 0-15 of each 32-lane subpartition (row 16*sp + t)
    const bool lane_ok = UM == 64 ? lane < 16 : true;
    const int m = UM == 64 ? 16 * sp + (lane & 15) : 32 * sp + lane;
    const bool row_ok = lane_ok && m < g.e.M;
    const uint32_t lane_addr = (uint32_t)(32 * sp) << 16;
    for (int it = 0; it < my_items; ++it) {
      const int buf = it & 1;
      const int j = q + it * G;
      mbar_wait(&tfull_bar[buf], (it >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t acc = tmem + lane_addr + buf * g.acc_cols;
      // two groups of 16 columns, one wait: the loads of both are in flight together
      auto get = [&](int c0, int c1, float* v) {
        tmem_ld16_async(acc + c0, v);
        tmem_ld16_async(acc + c1, v + 16);
        tmem_wait_ld();
        reg_fence16(v);
        reg_fence16(v + 16);
      };
      epi::finalize<__nv_bfloat16>(g.e, m, row_ok, j / S, j % S, BR, get);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[buf]);  // 4 epilogue warps -> count 4
    }
  }
  __syncwarp();
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// ------------------------------------------------------------------ fp32 numerics mode
// CTA = (weight block of br rows, 32-row batch tile): K in 32-column smem chunks, a 32 x br
// fp32 tile, then the same epilogue as the tensor-core kernel (rows by thread).
constexpr int kSimtRows = 32, kSimtK = 32;

__global__ void __launch_bounds__(256) dgemm_f32_kernel(const float* __restrict__ x, int ldx,
                                                        const float* __restrict__ w, int ldw, int K, int br,
                                                        int w_rows, const epi::Args e) {
  extern __shared__ float sm[];
  float* xs = sm;                          // [32][33]
  float* ws = xs + kSimtRows * (kSimtK + 1);  // [br][33]
  float* cs = ws + br * (kSimtK + 1);         // [32][br + 1]
  pdl_launch_dependents();
  pdl_wait();
  const int blk = blockIdx.x, m0 = blockIdx.y * kSimtRows;
  const int tid = threadIdx.x;
  const int n_out = kSimtRows * br;
  float acc[kSimtRows * kMaxBr / 256];
  const int per = n_out / 256;  // br is a multiple of 8 -> n_out a multiple of 256
  for (int i = 0; i < per; ++i) acc[i] = 0.f;
  for (int k0 = 0; k0 < K; k0 += kSimtK) {
    __syncthreads();
    for (int i = tid; i < kSimtRows * kSimtK; i += 256) {
      const int r = i / kSimtK, k = i % kSimtK;
      xs[r * (kSimtK + 1) + k] = (m0 + r < e.M && k0 + k < K) ? x[(size_t)(m0 + r) * ldx + k0 + k] : 0.f;
    }
    for (int i = tid; i < br * kSimtK; i += 256) {
      const int r = i / kSimtK, k = i % kSimtK;
      const int row = blk * br + r;
      ws[r * (kSimtK + 1) + k] = (row < w_rows && k0 + k < K) ? w[(size_t)row * ldw + k0 + k] : 0.f;
    }
    __syncthreads();
    for (int i = 0; i < per; ++i) {
      const int o = tid + i * 256, r = o / br, n = o % br;
      float a = acc[i];
#pragma unroll 8
      for (int k = 0; k < kSimtK; ++k) a += xs[r * (kSimtK + 1) + k] * ws[n * (kSimtK + 1) + k];
      acc[i] = a;
    }
  }
  for (int i = 0; i < per; ++i) {
    const int o = tid + i * 256, r = o / br, n = o % br;
    cs[r * (br + 1) + n] = acc[i];
  }
  __syncthreads();
  if (tid < kSimtRows) {
    const int r = tid, m = m0 + r;
    auto get = [&](int c0, int c1, float* v) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = cs[r * (br + 1) + c0 + j];
        v[16 + j] = cs[r * (br + 1) + c1 + j];
      }
    };
    epi::finalize<float>(e, m, m < e.M, blk, 0, br, get);
  }
}

// ------------------------------------------------------------------ host
int num_sms() {
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

// SwiGLU interleave block h (gate/up rows per block: 2h): the multiple of 16 <= 128 whose
// blocks fill the SMs best (fewest waves x block height; ties -> taller).  FFN 14336 -> 112
// (128 blocks: 86 % of the SMs stream; 128 would leave 36 of 148 idle).
int swiglu_block(int N) {
  const int sms = num_sms();
  int best = 128;
  long best_cost = -1;
  for (int h = 128; h >= 64; h -= 16) {  // (steps of 8: h = 104, 138 blocks on 138 SMs, measured no faster in decode, 0.95 vs 0.97 of cuBLAS in prefill)
    const long blocks = (N + h - 1) / h;
    const long cost = (blocks + sms - 1) / sms * h;
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = h; }
  }
  return best;
}

static int stage_bytes(int um, int br, int ks) { return ks * (um + br) * BK * 2; }

// atoms per stage: >= 32 KB of weights per stage barrier round trip (the issuing thread
// pays a wait / commit per stage), at most 4, dividing the item's k-blocks, >= 3 stages
static int pick_ks(int um, int br, int kb_item) {
  int ks = 1;
  while (ks < 4 && br * BK * 2 * ks < 32768 && kb_item % (2 * ks) == 0 &&
         (kSmemMax - 2048) / stage_bytes(um, br, 2 * ks) >= 3)
    ks *= 2;
  return ks;
}

Plan plan_for(int M, int N, int K, int br, int splits, int sw_half) {
  Plan p{};
  const int sms = num_sms();
  const int kb = K / BK;
  p.um = M <= 64 ? 64 : 128;
  p.br = br;
  p.splits = splits;
  p.ks = pick_ks(p.um, br, kb / splits);
  p.ku = kb / splits / p.ks;
  p.nblocks = sw_half ? (N + sw_half - 1) / sw_half : (N + br - 1) / br;
  const int items = p.nblocks * splits;
  p.grid = items < sms ? items : sms;
  p.stage = stage_bytes(p.um, br, p.ks);
  p.ns = (kSmemMax - 2048) / p.stage;
  if (p.ns > kMaxStages) p.ns = kMaxStages;
  return p;
}

static int g_force_br = 0, g_force_ks = 0, g_force_grid = 0, g_force_splits = 0;  // sn_gemm_decode_tune

// The plan minimising the bytes the busiest CTA streams: waves x (weight rows x k-blocks of an
// item) + the activation tile (an L2 hit, weighed lightly) + the fp32 slabs a K split adds for
// the consumer.  Block heights are multiples of 16 (UMMA N, TMA box <= 256 rows); SwiGLU keeps
// the interleave block of the weight layout (2h rows); the attention in-projection needs
// multiples of 32 (rotary pairs of a 32-column group stay together).  Ties -> fewer splits,
// then taller blocks.
static Plan make_plan_auto(int M, int N, int K, int mode) {
  const int kb = K / BK;
  if (mode == SN_GEMM_SWIGLU_IL) {
    const int h = swiglu_block(N);
    return plan_for(M, N, K, 2 * h, 1, h);
  }
  const int sms = num_sms();
  const int um = M <= 64 ? 64 : 128;
  const int step = mode == SN_GEMM_ATTN_IN ? 32 : 16;
  const int max_splits = mode == SN_GEMM_PARTIAL ? kMaxSplits : 1;
  Plan best{};
  double best_cost = -1.0;
  for (int s = 1; s <= max_splits; ++s) {
    if (kb % s) continue;
    for (int br = kMaxBr; br >= 32; br -= step) {
      const long blocks = (N + br - 1) / br;
      const long waves = (blocks * s + sms - 1) / sms;
      const double cost = (double)waves * (kb / s) * (br + um / 8) * 128.0 +
                          (s > 1 ? (double)s * M * N * 8.0 / sms : 0.0);
      if (best_cost < 0 || cost < best_cost * 0.999) { best_cost = cost; best = plan_for(M, N, K, br, s, 0); }
    }
  }
  return best;
}

Plan make_plan(int M, int N, int K, int mode) {
  Plan p = make_plan_auto(M, N, K, mode);
  if (mode == SN_GEMM_SWIGLU_IL) return p;
  const int kb = K / BK;
  const int br = g_force_br && (mode != SN_GEMM_ATTN_IN || g_force_br % 32 == 0) ? g_force_br : p.br;
  const int sp = g_force_splits && mode == SN_GEMM_PARTIAL && kb % g_force_splits == 0 ? g_force_splits : p.splits;
  if (br != p.br || sp != p.splits) p = plan_for(M, N, K, br, sp, 0);
  if (g_force_ks && (kb / p.splits) % g_force_ks == 0 && (kSmemMax - 2048) / stage_bytes(p.um, p.br, g_force_ks) >= 2) {
    p.ks = g_force_ks;
    p.ku = kb / p.splits / p.ks;
    p.stage = stage_bytes(p.um, p.br, p.ks);
    p.ns = (kSmemMax - 2048) / p.stage;
    if (p.ns > kMaxStages) p.ns = kMaxStages;
  }
  if (g_force_grid > 0 && g_force_grid < p.grid) p.grid = g_force_grid;
  return p;
}

template <int UM>
static sn_status launch(const CUtensorMap& wm, const CUtensorMap& xm, const Plan& p, Args g, cudaStream_t st) {
  g.br = p.br; g.nblocks = p.nblocks; g.splits = p.splits; g.ks = p.ks; g.ku = p.ku;
  g.ns = p.ns; g.stage_bytes = p.stage;
  int cols = 32;
  while (cols < p.br) cols <<= 1;
  g.acc_cols = cols;
  const int smem = p.ns * p.stage + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dgemm_kernel<UM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax - 1024);
    attr = true;
  }
  cudaError_t e = launch_pdl(dgemm_kernel<UM>, dim3(p.grid), dim3(kThreads), (size_t)smem, st, wm, xm, g);
  if (e != cudaSuccess) {
    set_error("sn_gemm_decode launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_gemm_decode");
}

static sn_status run(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, const epi::Args& ea_in,
                     int* splits_out, int dtype, cudaStream_t st) {
  epi::Args ea = ea_in;
  const int mode = ea.mode;
  if (dtype == SN_F32) {  // numerics mode: one tile per (block, 32 rows), never split
    int br = 64;
    if (mode == SN_GEMM_SWIGLU_IL) br = 2 * swiglu_block(N);
    const int sw_half = mode == SN_GEMM_SWIGLU_IL ? br / 2 : 0;
    const int nblocks = sw_half ? (N + sw_half - 1) / sw_half : (N + br - 1) / br;
    const int w_rows = sw_half ? nblocks * br : N;
    ea.S = 1;
    if (splits_out) *splits_out = 1;
    const size_t smem = ((size_t)kSimtRows * (kSimtK + 1) + (size_t)br * (kSimtK + 1) + (size_t)kSimtRows * (br + 1)) * 4;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dgemm_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax - 1024);
      attr = true;
    }
    const dim3 grid(nblocks, (M + kSimtRows - 1) / kSimtRows);
    cudaError_t e = launch_pdl(dgemm_f32_kernel, grid, dim3(256), smem, st, (const float*)x, ldx, (const float*)w, ldw,
                               K, br, w_rows, ea);
    if (e != cudaSuccess) {
      set_error("sn_gemm_decode launch: %s", cudaGetErrorString(e));
      return SN_ECUDA;
    }
    return check_launch("sn_gemm_decode");
  }
  SN_REQUIRE(dtype == SN_BF16, "sn_gemm_decode: dtype %d", dtype);
  SN_REQUIRE(M <= 128, "sn_gemm_decode: M=%d > 128", M);
  const Plan p = make_plan(M, N, K, mode);
  ea.S = p.splits;
  if (splits_out) *splits_out = p.splits;
  CUtensorMap wm, xm;
  const uint64_t wrows = mode == SN_GEMM_SWIGLU_IL ? (uint64_t)p.nblocks * p.br : (uint64_t)N;
  if (!map_2d(&wm, w, wrows, K, ldw, p.br) || !map_2d(&xm, x, M, K, ldx, p.um)) {
    set_error("sn_gemm_decode: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  Args g{};
  g.K = K;
  g.kb = K / BK;
  g.e = ea;
  return p.um == 64 ? launch<64>(wm, xm, p, g, st) : launch<128>(wm, xm, p, g, st);
}

}  // namespace dgemm
}  // namespace sn

using namespace sn;

extern "C" {

void sn_gemm_decode_tune(int br, int ks, int splits, int grid) {
  dgemm::g_force_br = (br >= 16 && br <= 256 && br % 16 == 0) ? br : 0;
  dgemm::g_force_ks = (ks == 1 || ks == 2 || ks == 4 || ks == 8) ? ks : 0;
  dgemm::g_force_splits = (splits >= 1 && splits <= dgemm::kMaxSplits) ? splits : 0;
  dgemm::g_force_grid = grid > 0 ? grid : 0;
}

int sn_gemm_swiglu_block(int N) { return dgemm::swiglu_block(N); }

int sn_gemm_decode_plan(int M, int N, int K, int mode, int* out) {
  if (K % tc::BK || !out) return -1;
  const dgemm::Plan p = dgemm::make_plan(M, N, K, mode);
  out[0] = p.br; out[1] = p.splits; out[2] = p.ks; out[3] = p.nblocks; out[4] = p.grid; out[5] = p.ns;
  return 0;
}

static sn_status check_common(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, int dtype) {
  SN_REQUIRE(x && w, "sn_gemm_decode: NULL operand");
  SN_REQUIRE(M >= 1, "sn_gemm_decode: M=%d", M);
  SN_REQUIRE(K % tc::BK == 0 && K >= tc::BK, "sn_gemm_decode: K=%d must be a multiple of %d", K, tc::BK);
  SN_REQUIRE(N >= 1 && ldw >= K && ldx >= K, "sn_gemm_decode: bad N/ld");
  const int esz = dtype == SN_F32 ? 4 : 2;
  SN_REQUIRE(((uintptr_t)x % 16) == 0 && ((uintptr_t)w % 16) == 0 && (ldx * esz) % 16 == 0 && (ldw * esz) % 16 == 0,
             "sn_gemm_decode: operands must be 16-byte aligned");
  return SN_OK;
}

sn_status sn_gemm_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                         int mode, int* splits_out, int dtype, void* stream) {
  sn_status s = check_common(x, M, K, ldx, w, N, ldw, dtype);
  if (s != SN_OK) return s;
  SN_REQUIRE(out != nullptr && ldo >= N, "sn_gemm_decode: bad output");
  SN_REQUIRE(mode == SN_GEMM_STORE || mode == SN_GEMM_RESID || mode == SN_GEMM_PARTIAL || mode == SN_GEMM_SWIGLU_IL,
             "sn_gemm_decode: mode %d (attention in-projection: sn_gemm_decode_attn_in)", mode);
  epi::Args ea{};
  ea.mode = mode;
  ea.M = M;
  ea.N = N;
  ea.out = out;
  ea.ldo = ldo;
  return dgemm::run(x, M, K, ldx, w, N, ldw, ea, splits_out, dtype, (cudaStream_t)stream);
}

sn_status sn_gemm_decode_attn_in(const void* x, int M, int K, int ldx, const void* w, int ldw,
                                 const int32_t* positions, const float* inv_freq, void* q_out, void* k_cache,
                                 void* v_cache, const int32_t* block_table, int Hq, int Hkv, int D, int page_size,
                                 int max_blocks, int window, int32_t* err_flag, const void* rope_cs, int dtype,
                                 void* stream) {
  const int N = (Hq + 2 * Hkv) * D;
  sn_status s = check_common(x, M, K, ldx, w, N, ldw, dtype);
  if (s != SN_OK) return s;
  SN_REQUIRE(D == 64 || D == 128, "sn_gemm_decode_attn_in: head dim %d", D);
  SN_REQUIRE(positions && inv_freq && q_out && k_cache && v_cache && block_table, "sn_gemm_decode_attn_in: NULL pointer");
  SN_REQUIRE(page_size > 0 && max_blocks > 0 && (window == 0 || window % page_size == 0),
             "sn_gemm_decode_attn_in: bad page geometry");
  epi::Args ea{};
  ea.mode = SN_GEMM_ATTN_IN;
  ea.M = M;
  ea.N = N;
  ea.positions = positions;
  ea.inv_freq = inv_freq;
  ea.q_out = q_out;
  ea.k_cache = k_cache;
  ea.v_cache = v_cache;
  ea.block_table = block_table;
  ea.Hq = Hq;
  ea.Hkv = Hkv;
  ea.D = D;
  ea.page_size = page_size;
  ea.max_blocks = max_blocks;
  ea.window = window;
  ea.err = err_flag;
  ea.rope_cs = reinterpret_cast<const float2*>(rope_cs);
  return dgemm::run(x, M, K, ldx, w, N, ldw, ea, nullptr, dtype, (cudaStream_t)stream);
}

}  // extern "C"
