// Fused decode chain: every projection and norm between two mixer kernels of the decode step
// in one persistent launch (include/sn_abi.h sn_decode_chain).
//
// Why: as separate kernels, each projection of the step (out-proj, FFN gate/up, down, the next
// layer's in-projection) is a persistent 148-CTA grid holding a whole SM's shared memory, so
// the next one cannot become resident until the previous one's CTAs exit: every boundary
// drains HBM (epilogue tail, launch, barrier init, TMEM alloc, first TMA round trip) — about
// 5 us per projection against a 7-45 us weight stream, ~1 ms of the 10.2 ms step
// (profiles/r02_decode_ablation.md).  Here one CTA per SM walks the phases in order; a grid
// barrier separates a phase from the phase it reads, and while a CTA waits at it (or drains its
// epilogue) its producer thread is already streaming the NEXT phase's weights into the
// shared-memory ring — weights never depend on the barrier, only the activation tiles do.
//
// Phases:
//   GEMM: the decode GEMM of sn_dgemm.cu (batch-as-M tcgen05 UMMA, TMA-fed 128B-swizzled
//         stages, two TMEM accumulators, the sn_epi.cuh epilogues, same work plans).
//   NORM: residual += sum of split-K slabs (slab order, deterministic); out = RMSNorm * w.
//         One batch row per CTA (rows are independent), by the 4 epilogue warps.
//
// Grid barrier: a monotonic 64-bit arrival counter per call site.  Barrier b of a launch
// completes when the counter reaches base + (b + 1) * grid, base = the counter at launch
// (a multiple of grid * barriers-per-launch: every earlier launch of the site completed all
// of its barriers).  A CTA arrives at barrier b only after barrier b - 1 completed, so
// arrivals of different barriers never mix.  Writers: generic stores, fence.proxy.async +
// release add; waiters: acquire load, then fence.proxy.async before the TMA reads.
//
// Ring: the stage layout (count x bytes) follows each phase's plan; when it changes the
// producer first drains the ring (waits until the MMA consumed every stage in flight).
#include <cuda.h>

#include "sn_common.cuh"
#include "sn_dplan.cuh"
#include "sn_epi.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace chain {

using namespace sn::tc;
constexpr int kThreads = 256;
constexpr int kMaxStages = 16;
constexpr int kMaxGemm = 6, kMaxNorm = 2, kMaxPhases = 8;
constexpr int kAccCols = 256;  // one TMEM accumulator buffer (UMMA N <= 256)
constexpr int kNormMaxSplit = 8;
constexpr int kNormThreads = 192;  // warps 2-7
constexpr int kNormVec = 7;        // float4 chunks per thread: dim <= 7 * 4 * 192 = 5376

struct alignas(64) GemmP {
  CUtensorMap wmap;
  CUtensorMap xmap;
  int br, nblocks, splits, ks, ku, ns, stage_bytes, pad;
  epi::Args e;
};
struct NormP {
  const float* ss;  // per-block row sums of squares of the residual (RESID GEMM before it), [nss][rows]
  int nss;
  const float* partials;
  float* residual;
  const __nv_bfloat16* weight;
  __nv_bfloat16* out;
  int nsplit, rows, dim;
  float eps;
};
struct Params {
  GemmP g[kMaxGemm];
  NormP n[kMaxNorm];
  unsigned long long* counter;
  int nph, nbar;
  unsigned long long* trace;  // sn_decode_chain_trace: per-CTA globaltimer stamps (tools/chain_trace.py)
  int8_t kind[kMaxPhases], idx[kMaxPhases];
  int8_t wait_bar[kMaxPhases];  // barrier whose completion the phase's inputs need (-1: the previous kernel)
  int8_t arrive[kMaxPhases];    // 1: every CTA arrives at the next barrier after the phase
};

static_assert(sizeof(Params) <= 4096, "chain parameters exceed the classic 4 KB kernel-parameter space");

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(const unsigned long long* counter, unsigned long long base, int b) {
  const unsigned long long target = base + (unsigned long long)(b + 1) * gridDim.x;
  while (ld_acquire_u64(counter) < target) __nanosleep(32);
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slot of CTA q: [0] start, [1] end, then per phase p: [2+4p] producer released (inputs
// ready), [3+4p] epilogue / norm rows done, [4+4p] arrival, [5+4p] norm wait released
#define SN_TRACE(slot) \
  do { if (P.trace) P.trace[(size_t)blockIdx.x * 40 + (slot)] = gtime(); } while (0)

__device__ __forceinline__ int items_of(int items, int q, int G) { return items > q ? (items - q + G - 1) / G : 0; }

template <int UM>
__global__ void __launch_bounds__(kThreads, 1) chain_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ unsigned long long base_s;
  __shared__ float nred[kNormThreads / 32];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x, G = gridDim.x;
  constexpr uint32_t X_BYTES = UM * BK * 2;
  pdl_launch_dependents();
  if (threadIdx.x == 0) SN_TRACE(0);

  if (threadIdx.x == 0) {
    for (int p = 0; p < P.nph; ++p)
      if (P.kind[p] == SN_CHAIN_GEMM) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.g[P.idx[p]].wmap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.g[P.idx[p]].xmap)) : "memory");
      }
    for (int i = 0; i < kMaxStages; ++i) { mbar_init(&full_bar[i], 1); mbar_init(&empty_bar[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull_bar[i], 1); mbar_init(&tempty_bar[i], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // every earlier launch of this call site completed all of its barriers, and this CTA has
    // not arrived yet, so barrier 0 of this launch cannot have completed: the counter lies in
    // [base, base + G)
    if (P.nbar > 0) {
      const unsigned long long c = ld_acquire_u64(P.counter);
      base_s = c - c % ((unsigned long long)G * P.nbar);
    }
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
  const unsigned long long base = base_s;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      uint32_t fpar = 0, ever = 0;  // per slot: parity of its fill count, filled at least once
      int s = 0, cur_ns = 0, cur_sb = 0;
      for (int p = 0; p < P.nph; ++p) {
        if (P.kind[p] != SN_CHAIN_GEMM) continue;
        const GemmP& g = P.g[P.idx[p]];
        const int units = items_of(g.nblocks * g.splits, q, G) * g.ku;
        if (g.ns != cur_ns || g.stage_bytes != cur_sb) {  // new stage layout: drain the ring first
          for (int t = 0; t < cur_ns; ++t)
            if ((ever >> t) & 1) mbar_wait(&empty_bar[t], ((fpar >> t) & 1) ^ 1);
          cur_ns = g.ns;
          cur_sb = g.stage_bytes;
          s = 0;
        }
        const uint32_t wb = (uint32_t)g.br * BK * 2;
        auto issue = [&](int u, bool w_part, bool x_part, int slot) {
          const int it = u / g.ku, ku = u - it * g.ku;
          const int j = q + it * G;
          const int blk = j / g.splits;
          const int kc0 = ((j - blk * g.splits) * g.ku + ku) * g.ks * BK;
          uint8_t* st = smem + slot * g.stage_bytes;
#pragma unroll 1
          for (int a = 0; a < g.ks; ++a) {
            const int kc = kc0 + a * BK;
            if (w_part) tma_load_2d(st + g.ks * X_BYTES + a * wb, &g.wmap, kc, blk * g.br, &full_bar[slot], pw);
            if (x_part) tma_load_2d(st + a * X_BYTES, &g.xmap, kc, 0, &full_bar[slot], px);
          }
        };
        auto acquire = [&](int slot) {
          if ((ever >> slot) & 1) mbar_wait(&empty_bar[slot], ((fpar >> slot) & 1) ^ 1);
          ever |= 1u << slot;
          fpar ^= 1u << slot;
        };
        auto next = [&](int slot) { return slot + 1 == g.ns ? 0 : slot + 1; };
        // the weights of the first stages do not depend on the barrier: requested before it
        const int npre = min(g.ns, units);
        const int s0 = s;
        for (int u = 0; u < npre; ++u) {
          acquire(s);
          mbar_expect_tx_noarrive(&full_bar[s], g.ks * wb);
          issue(u, true, false, s);
          s = next(s);
        }
        if (units > 0) {
          if (P.wait_bar[p] < 0) asm volatile("griddepcontrol.wait;" ::: "memory");
          else bar_wait(P.counter, base, P.wait_bar[p]);
          fence_proxy_async_global();
          SN_TRACE(2 + 4 * p);
        }
        int s1 = s0;
        for (int u = 0; u < npre; ++u) {
          mbar_expect_tx(&full_bar[s1], g.ks * X_BYTES);
          issue(u, false, true, s1);
          s1 = next(s1);
        }
        for (int u = npre; u < units; ++u) {
          acquire(s);
          mbar_expect_tx(&full_bar[s], g.ks * (wb + X_BYTES));
          issue(u, true, true, s);
          s = next(s);
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (whole warp converged, one elected lane issues)
    uint32_t cpar = 0;  // per slot: parity of its consume count
    int s = 0, cur_ns = 0, cur_sb = 0, acc_it = 0;
    for (int p = 0; p < P.nph; ++p) {
      if (P.kind[p] != SN_CHAIN_GEMM) continue;
      const GemmP& g = P.g[P.idx[p]];
      if (g.ns != cur_ns || g.stage_bytes != cur_sb) {
        cur_ns = g.ns;
        cur_sb = g.stage_bytes;
        s = 0;
      }
      const int my_items = items_of(g.nblocks * g.splits, q, G);
      const uint32_t idesc = idesc_bf16(UM, g.br);
      const uint32_t wb = (uint32_t)g.br * BK * 2;
      for (int it = 0; it < my_items; ++it, ++acc_it) {
        const int buf = acc_it & 1;
        if (acc_it >= 2) mbar_wait(&tempty_bar[buf], ((acc_it >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + buf * kAccCols;
        for (int ku = 0; ku < g.ku; ++ku) {
          mbar_wait(&full_bar[s], (cpar >> s) & 1);
          cpar ^= 1u << s;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sx = smem_u32(smem + s * g.stage_bytes);
          const uint32_t sw = sx + g.ks * X_BYTES;
#pragma unroll 1
          for (int a = 0; a < g.ks; ++a) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_w(acc, desc_sw128(sx + a * X_BYTES + k * 32), desc_sw128(sw + a * wb + k * 32), idesc,
                     (ku | a | k) ? 1u : 0u);
          }
          commit_w(&empty_bar[s]);
          s = s + 1 == g.ns ? 0 : s + 1;
        }
        commit_w(&tfull_bar[buf]);
      }
    }
  } else if (warp >= 2) {
    // ---------------- warps 4-7: GEMM epilogues; warps 2-7 (192 threads): NORM rows and the
    // barrier arrivals (warps 2 and 3 have no other work once the TMEM is allocated)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool epi = warp >= 4;
    const int nt = threadIdx.x - 64;  // 0..191
    const int sp = warp & 3;
    const bool lane_ok = UM == 64 ? lane < 16 : true;
    const int m = UM == 64 ? 16 * sp + (lane & 15) : 32 * sp + lane;
    const uint32_t lane_addr = (uint32_t)(32 * sp) << 16;
    int acc_it = 0, arrived = 0;
    for (int p = 0; p < P.nph; ++p) {
      if (P.kind[p] == SN_CHAIN_GEMM) {
        if (epi) {
          const GemmP& g = P.g[P.idx[p]];
          const bool row_ok = lane_ok && m < g.e.M;
          const int my_items = items_of(g.nblocks * g.splits, q, G);
          for (int it = 0; it < my_items; ++it, ++acc_it) {
            const int buf = acc_it & 1;
            const int j = q + it * G;
            mbar_wait(&tfull_bar[buf], (acc_it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t acc = tmem + lane_addr + buf * kAccCols;
            auto get = [&](int c0, int c1, float* v) {
              tmem_ld16_async(acc + c0, v);
              tmem_ld16_async(acc + c1, v + 16);
              tmem_wait_ld();
              reg_fence16(v);
              reg_fence16(v + 16);
            };
            epi::finalize<__nv_bfloat16>(g.e, m, row_ok, j / g.splits, j % g.splits, g.br, get);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[buf]);
          }
        }
      } else {
        const NormP& n = P.n[P.idx[p]];
        if (P.wait_bar[p] >= 0) {
          if (nt == 0) {
            bar_wait(P.counter, base, P.wait_bar[p]);
            SN_TRACE(5 + 4 * p);
          }
          named_bar(2, kNormThreads);
        }
        const int nch = n.dim >> 2;  // float4 chunks of a row
        for (int r = q; r < n.rows; r += G) {
          // the residual and up to 4 slabs are requested together: one L2 round trip per row
          // (the slabs were just written by other CTAs, so they are L2 hits)
          float4 v[kNormVec];
          float* res = n.residual + (size_t)r * n.dim;
#pragma unroll
          for (int c = 0; c < kNormVec; ++c) {
            const int ci = c * kNormThreads + nt;
            if (ci < nch) v[c] = *reinterpret_cast<const float4*>(res + 4 * ci);
          }
#pragma unroll 1
          for (int s0 = 0; s0 < n.nsplit; s0 += 4) {
            float4 t[4][kNormVec];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              if (s0 + s < n.nsplit) {
                const float4* ps = reinterpret_cast<const float4*>(n.partials + ((size_t)(s0 + s) * n.rows + r) * n.dim);
#pragma unroll
                for (int c = 0; c < kNormVec; ++c) {
                  const int ci = c * kNormThreads + nt;
                  if (ci < nch) t[s][c] = __ldcg(ps + ci);
                }
              }
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              if (s0 + s < n.nsplit) {
#pragma unroll
                for (int c = 0; c < kNormVec; ++c) {
                  const int ci = c * kNormThreads + nt;
                  if (ci < nch) { v[c].x += t[s][c].x; v[c].y += t[s][c].y; v[c].z += t[s][c].z; v[c].w += t[s][c].w; }
                }
              }
            }
          }
          float ss = 0.f;
          if (n.nss > 0) {  // the residual GEMM already summed the squares per block: add its blocks
            for (int b = nt; b < n.nss; b += kNormThreads) ss += __ldcg(n.ss + (size_t)b * n.rows + r);
          } else {
#pragma unroll
            for (int c = 0; c < kNormVec; ++c) {
              const int ci = c * kNormThreads + nt;
              if (ci < nch) {
                if (n.nsplit > 0) *reinterpret_cast<float4*>(res + 4 * ci) = v[c];
                ss += v[c].x * v[c].x + v[c].y * v[c].y + v[c].z * v[c].z + v[c].w * v[c].w;
              }
            }
          }
          ss = warp_sum(ss);
          if (lane == 0) nred[warp - 2] = ss;
          named_bar(2, kNormThreads);
          ss = 0.f;
#pragma unroll
          for (int w = 0; w < kNormThreads / 32; ++w) ss += nred[w];
          named_bar(2, kNormThreads);  // nred is reused by the next row
          const float rstd = rsqrtf(ss / (float)n.dim + n.eps);
#pragma unroll
          for (int c = 0; c < kNormVec; ++c) {
            const int ci = c * kNormThreads + nt;
            if (ci < nch) {
              const uint2 wu = *reinterpret_cast<const uint2*>(n.weight + 4 * ci);
              const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wu.x));
              const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wu.y));
              __nv_bfloat162 o01 = __floats2bfloat162_rn(v[c].x * rstd * w01.x, v[c].y * rstd * w01.y);
              __nv_bfloat162 o23 = __floats2bfloat162_rn(v[c].z * rstd * w23.x, v[c].w * rstd * w23.y);
              uint2 ou;
              ou.x = *reinterpret_cast<uint32_t*>(&o01);
              ou.y = *reinterpret_cast<uint32_t*>(&o23);
              *reinterpret_cast<uint2*>(n.out + (size_t)r * n.dim + 4 * ci) = ou;
            }
          }
        }
      }
      if (P.arrive[p]) {  // this CTA's outputs of phase p are written: arrive at the next barrier
        named_bar(2, kNormThreads);  // every writer of the CTA is past its stores
        if (nt == 0) {
          SN_TRACE(3 + 4 * p);
          fence_proxy_async_global();
          __threadfence();  // cumulative: the CTA's writes (ordered by the bar.sync) before the arrival
          if (arrived > 0) bar_wait(P.counter, base, arrived - 1);  // never mix two barriers' arrivals
          red_release_add_u64(P.counter, 1ull);
          SN_TRACE(4 + 4 * p);
        }
        ++arrived;
      }
    }
  }
  __syncwarp();
  __syncthreads();
  if (threadIdx.x == 0) SN_TRACE(1);
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * kAccCols));
}

// ------------------------------------------------------------------ host
template <int UM>
static sn_status launch(const Params& p, int grid, int smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chain_kernel<UM>, cudaFuncAttributeMaxDynamicSharedMemorySize, dgemm::kSmemMax - 1024);
    attr = true;
  }
  cudaError_t e = launch_pdl(chain_kernel<UM>, dim3(grid), dim3(kThreads), (size_t)smem, st, p);
  if (e != cudaSuccess) {
    set_error("sn_decode_chain launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch("sn_decode_chain");
}

}  // namespace chain
}  // namespace sn

using namespace sn;

static unsigned long long* g_chain_trace = nullptr;
extern "C" void sn_decode_chain_trace(unsigned long long* buf) { g_chain_trace = buf; }

extern "C" sn_status sn_decode_chain(sn_chain_phase* ph, int n, int M, unsigned long long* counter, void* stream) {
  using chain::Params;
  SN_REQUIRE(ph && n >= 1 && n <= chain::kMaxPhases, "sn_decode_chain: %d phases (1..%d)", n, chain::kMaxPhases);
  SN_REQUIRE(M >= 1 && M <= 128, "sn_decode_chain: M=%d (1..128)", M);
  static thread_local Params P;  // host staging (the launch copies the parameters)
  memset(&P, 0, sizeof(P));
  P.counter = counter;
  P.nph = n;
  const int sms = dgemm::num_sms();
  const int um = M <= 64 ? 64 : 128;
  int ng = 0, nn = 0, nbar = 0, last_splits = 0, last_ss_blocks = 0, grid = 1, smem_max = 0;
  int latest_bar = -1;
  for (int i = 0; i < n; ++i) {
    sn_chain_phase& c = ph[i];
    if (i > 0 && c.depends) {  // every CTA arrives after phase i-1; phase i waits for that barrier
      P.arrive[i - 1] = 1;
      latest_bar = nbar++;
    }
    P.wait_bar[i] = (int8_t)latest_bar;
    P.kind[i] = (int8_t)c.kind;
    if (c.kind == SN_CHAIN_GEMM) {
      SN_REQUIRE(ng < chain::kMaxGemm, "sn_decode_chain: more than %d GEMM phases", chain::kMaxGemm);
      SN_REQUIRE(c.x && c.w && c.out, "sn_decode_chain: phase %d: NULL operand", i);
      SN_REQUIRE(c.K % tc::BK == 0 && c.K >= tc::BK && c.N >= 1 && c.ldw >= c.K && c.ldx >= c.K,
                 "sn_decode_chain: phase %d: bad K/N/ld", i);
      SN_REQUIRE(((uintptr_t)c.x % 16) == 0 && ((uintptr_t)c.w % 16) == 0 && (c.ldx * 2) % 16 == 0 &&
                     (c.ldw * 2) % 16 == 0,
                 "sn_decode_chain: phase %d: operands must be 16-byte aligned", i);
      SN_REQUIRE(c.mode == SN_GEMM_STORE || c.mode == SN_GEMM_RESID || c.mode == SN_GEMM_PARTIAL ||
                     c.mode == SN_GEMM_SWIGLU_IL || c.mode == SN_GEMM_ATTN_IN,
                 "sn_decode_chain: phase %d: mode %d", i, c.mode);
      if (c.mode == SN_GEMM_ATTN_IN) {
        SN_REQUIRE(c.N == (c.Hq + 2 * c.Hkv) * c.D && (c.D == 64 || c.D == 128) && c.positions && c.inv_freq &&
                       c.q_out && c.k_cache && c.v_cache && c.block_table && c.page_size > 0 && c.max_blocks > 0 &&
                       (c.window == 0 || c.window % c.page_size == 0),
                   "sn_decode_chain: phase %d: bad attention in-projection arguments", i);
      }
      const dgemm::Plan pl = dgemm::make_plan(M, c.N, c.K, c.mode);
      chain::GemmP& g = P.g[ng];
      const uint64_t wrows = c.mode == SN_GEMM_SWIGLU_IL ? (uint64_t)pl.nblocks * pl.br : (uint64_t)c.N;
      if (!tc::map_2d(&g.wmap, c.w, wrows, c.K, c.ldw, pl.br) || !tc::map_2d(&g.xmap, c.x, M, c.K, c.ldx, pl.um)) {
        set_error("sn_decode_chain: cuTensorMapEncodeTiled failed (phase %d)", i);
        return SN_ECUDA;
      }
g.br = pl.br; g.nblocks = pl.nblocks; g.splits = pl.splits; g.ks = pl.ks; g.ku = pl.ku;
      g.ns = pl.ns; g.stage_bytes = pl.stage;
      if (pl.ns * pl.stage > smem_max) smem_max = pl.ns * pl.stage;
      g.e.mode = c.mode; g.e.M = M; g.e.N = c.N; g.e.out = c.out; g.e.ldo = c.ldo; g.e.S = pl.splits;
      g.e.positions = c.positions; g.e.inv_freq = c.inv_freq; g.e.q_out = c.q_out; g.e.k_cache = c.k_cache;
      g.e.v_cache = c.v_cache; g.e.block_table = c.block_table; g.e.Hq = c.Hq; g.e.Hkv = c.Hkv; g.e.D = c.D;
      g.e.page_size = c.page_size; g.e.max_blocks = c.max_blocks; g.e.window = c.window; g.e.err = c.err_flag;
      g.e.rope_cs = reinterpret_cast<const float2*>(c.rope_cs);
      SN_REQUIRE(c.ss_out == nullptr || c.mode == SN_GEMM_RESID, "sn_decode_chain: phase %d: ss_out needs RESID", i);
      g.e.ss_out = c.ss_out;
      if (c.ss_out) last_ss_blocks = pl.nblocks;
      c.splits = pl.splits;
      if (c.mode == SN_GEMM_PARTIAL) last_splits = pl.splits;
      if (pl.grid > grid) grid = pl.grid;
      P.idx[i] = (int8_t)ng++;
    } else if (c.kind == SN_CHAIN_NORM) {
      SN_REQUIRE(nn < chain::kMaxNorm, "sn_decode_chain: more than %d NORM phases", chain::kMaxNorm);
      SN_REQUIRE(c.residual && c.weight && c.norm_out && c.dim > 0 && c.dim % 4 == 0 &&
                     c.dim <= chain::kNormVec * 4 * chain::kNormThreads,
                 "sn_decode_chain: phase %d: bad norm arguments (dim %d)", i, c.dim);
      const int ns = c.nsplit < 0 ? last_splits : c.nsplit;
      SN_REQUIRE(ns >= 0 && ns <= chain::kNormMaxSplit && (ns == 0 || c.partials),
                 "sn_decode_chain: phase %d: bad partials (nsplit %d)", i, ns);
      chain::NormP& nm = P.n[nn];
      nm.partials = c.partials; nm.residual = c.residual;
      nm.weight = reinterpret_cast<const __nv_bfloat16*>(c.weight);
      nm.out = reinterpret_cast<__nv_bfloat16*>(c.norm_out);
      nm.nsplit = ns; nm.rows = M; nm.dim = c.dim; nm.eps = c.eps;
      nm.ss = c.ss_in;
      nm.nss = c.ss_in ? (c.n_ss < 0 ? last_ss_blocks : c.n_ss) : 0;
      SN_REQUIRE(!c.ss_in || (nm.nss > 0 && ns == 0), "sn_decode_chain: phase %d: ss_in needs n_ss > 0 and no slabs", i);
      c.splits = ns;
      if (M > grid) grid = M;
      P.idx[i] = (int8_t)nn++;
    } else {
      SN_REQUIRE(false, "sn_decode_chain: phase %d: kind %d", i, c.kind);
    }
  }
  SN_REQUIRE(nbar == 0 || counter != nullptr, "sn_decode_chain: barriers need a counter");
  if (grid > sms) grid = sms;
  P.nbar = nbar;
  P.trace = g_chain_trace;
  const int smem = smem_max + 1024;
  return um == 64 ? chain::launch<64>(P, grid, smem, (cudaStream_t)stream)
                  : chain::launch<128>(P, grid, smem, (cudaStream_t)stream);
}
