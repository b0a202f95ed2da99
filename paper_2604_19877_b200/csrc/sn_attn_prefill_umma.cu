// Prefill attention on the 5th-generation tensor cores (tcgen05 / TMEM / TMA), D = 128, bf16.
// Same contract as the mma.sync kernel in sn_attn_prefill.cu (packed ragged sequences,
// causal or window mask per (row, key) with each row's own sequence start, GQA).
//
// CTA = 128 query rows x one q head; 4*NS softmax warps + 3 (NS = 2: 11 warps):
//   warps 4NS+1 / 4NS+2 (one lane each): TMA producers — Q once and K blocks of 128 keys / V blocks,
//           each into its own two-stage ring (128B-swizzled 2-D boxes straight from the
//           [rows][H*D] tensors), so the next K block only waits for its S product;
//   warp 4NS (one lane): MMA issuer — S = Q K^T (UMMA M=128, N=128, K=128; both operands
//           K-major) into one of two TMEM score buffers, then O += P V (A = P from shared
//           memory, B = V read MN-major: the [key][d] tile is used as is) into TMEM;
//   warps 0..4NS-1: softmax — warps w, w+4, .. share query rows 32(w%4).. (TMEM lanes), each
//           taking 128/NS of the key columns: tcgen05.ld of its S slice, mask / scale / max /
//           exp2 in registers, the row max combined through a shared-memory atomic max
//           (one 32NS-thread named barrier per lane quadrant), its O slice rescaled in TMEM
//           when the max moved (tcgen05.ld/st), its P slice written (bf16, 128B swizzle) for
//           the PV MMA; finally O / l to global.  More, narrower softmax warps hide the
//           latency of each warp's dependent max / exp chain (the softmax is the limiter).
// The scores of block j+1 are computed while the softmax of block j runs (two TMEM score
// buffers); PV(j) follows as soon as P(j) is in shared memory.
#include "sn_tc.cuh"

namespace sn {
namespace fa5 {

using namespace sn::tc;

constexpr int BM = 128, BN = 128, HD = 128;
constexpr float kLazy = 8.f;  // log2 headroom of the stale running max
constexpr uint32_t ATOM = 128 * 128;  // one [128 rows x 64 bf16] 128B-swizzled atom (16 KB)
constexpr uint32_t TILE = 2 * ATOM;   // [128 x 128] bf16
constexpr int kSmemBytes = 227 * 1024;

// MN-major operand (V as the B operand of P V: N = head dim contiguous, K = keys):
// LBO = stride between 64-element N chunks (the second TMA box), SBO = stride between
// groups of 8 K rows (8 x 128 B).
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(ATOM >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float ex2(float x) {  // 2^x, -inf -> 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (x <= 8): round-to-nearest split x = n + f, f in [-0.5, 0.5],
// cubic in f, n added to the exponent.  Relative error < 7e-4 (P is stored as bf16,
// 3.9e-3).  Part of the exponentials go this way (exp2_fma2, on pairs) so MUFU.EX2 (16 / clock / SM) is not the
// limiter of the softmax (FA4's split).
// Paired fp32 arithmetic (FFMA2 / FADD2 on sm_100a): two lanes of work per instruction.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
// exp2_fma on a pair
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f), nmagic = make_float2(-12582912.f, -12582912.f);
  const float2 t = fadd2(x, magic);
  const float2 r = fadd2(t, nmagic);
  const float2 f = fadd2(x, make_float2(-r.x, -r.y));
  float2 p = ffma2(make_float2(0.05550411f, 0.05550411f), f, make_float2(0.24022651f, 0.24022651f));
  p = ffma2(p, f, make_float2(0.69314718f, 0.69314718f));
  p = ffma2(p, f, make_float2(1.f, 1.f));
  const int nx = __float_as_int(t.x) - 0x4B400000, ny = __float_as_int(t.y) - 0x4B400000;
  return make_float2(__int_as_float(__float_as_int(p.x) + (nx << 23)), __int_as_float(__float_as_int(p.y) + (ny << 23)));
}
__device__ __forceinline__ void smem_max_f32(float* addr, float v) {  // order-preserving int encoding
  if (v >= 0.f) atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
  else atomicMin(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}
__device__ __forceinline__ float max3(float a, float b, float c) {  // FMNMX3 (sm_100)
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }


constexpr int kThreads2 = 16 * 32 + 96;
struct Smem2 {
  uint8_t q[2][TILE];
  uint8_t k[2][TILE];
  uint8_t v[2][TILE];
};
struct Sync2 {
  uint64_t q_full, k_full[2], k_empty[2], v_full[2], v_empty[2], s_full[2], p_full[2], o_done[2];
  uint32_t tmem_base;
  float red[2][3][BM];
  float lsum[2][BM];
};
constexpr int kSync2Bytes = 5120;
static_assert(sizeof(Sync2) <= kSync2Bytes, "sync2 block");
static_assert(sizeof(Smem2) + kSync2Bytes + 1024 <= kSmemBytes, "tiles2");

__global__ void __launch_bounds__(kThreads2, 1)
    attn_prefill_umma2_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                              const __grid_constant__ CUtensorMap vmap, const int32_t* __restrict__ cu,
                              __nv_bfloat16* __restrict__ out, int num_seqs, int rows, int Hq, int Hkv, int window,
                              float scale, const int32_t* __restrict__ cu_k, const int32_t* __restrict__ q_off) {
  constexpr int COLS = 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Sync2& sy = *reinterpret_cast<Sync2*>(smem_raw);
  uint8_t* base = smem_raw + kSync2Bytes;
  base += (1024 - (smem_u32(base) & 1023)) & 1023;
  Smem2& sm = *reinterpret_cast<Smem2*>(base);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctas = (rows + 2 * BM - 1) / (2 * BM);
  const int r0 = (ctas - 1 - (int)blockIdx.x) * 2 * BM;  // heavy (late) tiles first
  const int h = blockIdx.y, hk = h / (Hq / Hkv);
  // the CTA walks the union of both tiles' key blocks
  const int j_lo = min(key_bounds(cu, cu_k, q_off, num_seqs, min(r0, rows - 1), window).lo,
                       key_bounds(cu, cu_k, q_off, num_seqs, min(r0 + BM, rows - 1), window).lo);
  const int j_hi = max(key_bounds(cu, cu_k, q_off, num_seqs, min(r0 + BM - 1, rows - 1), window).hi,
                       key_bounds(cu, cu_k, q_off, num_seqs, min(r0 + 2 * BM - 1, rows - 1), window).hi);
  const int nblk = (j_hi - j_lo) / BN + 1;

  if (threadIdx.x == 0) {
    mbar_init(&sy.q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sy.k_full[i], 1); mbar_init(&sy.k_empty[i], 1);
      mbar_init(&sy.v_full[i], 1); mbar_init(&sy.v_empty[i], 1);
      mbar_init(&sy.s_full[i], 1); mbar_init(&sy.p_full[i], 8 * 32); mbar_init(&sy.o_done[i], 1);
    }
  }
  if (threadIdx.x < 2 * BM) {
    const int q = threadIdx.x / BM, t = threadIdx.x % BM;
    for (int i = 0; i < 3; ++i) sy.red[q][i][t] = -INFINITY;
    sy.lsum[q][t] = 0.f;
  }
  if (threadIdx.x == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sy.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sy.tmem_base;

  if (warp >= 17) {
    if (lane == 0) {  // ---------------- TMA producers
      const bool is_k = warp == 17;
      const CUtensorMap* map = is_k ? &kmap : &vmap;
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
      const uint64_t keep = policy_evict_last();
      if (is_k) {
        mbar_expect_tx(&sy.q_full, 2 * TILE);
        for (int q = 0; q < 2; ++q) {
          tma_load_2d(sm.q[q], &qmap, h * HD, r0 + q * BM, &sy.q_full, policy_evict_first());
          tma_load_2d(sm.q[q] + ATOM, &qmap, h * HD + 64, r0 + q * BM, &sy.q_full, policy_evict_first());
        }
      }
      uint64_t* full = is_k ? sy.k_full : sy.v_full;
      uint64_t* empty = is_k ? sy.k_empty : sy.v_empty;
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        if (j >= 2) mbar_wait(&empty[st], ((j >> 1) - 1) & 1);
        const int jb = j_lo + j * BN;
        uint8_t* dst = is_k ? sm.k[st] : sm.v[st];
        mbar_expect_tx(&full[st], TILE);
        tma_load_2d(dst, map, hk * HD, jb, &full[st], keep);
        tma_load_2d(dst + ATOM, map, hk * HD + 64, jb, &full[st], keep);
      }
    }
  } else if (warp == 16) {
    // ---------------- MMA issuer (whole warp converged, one elected lane issues)
    const uint32_t id_s = idesc_bf16(BM, BN);
    const uint32_t id_o = idesc_bf16(BM, HD) | (1u << 16);  // B (= V) MN-major
    mbar_wait(&sy.q_full, 0);
    auto issue_s = [&](int q, int j) {  // S_q(j) = Q_q K(j)^T into tile q's score columns
      const uint32_t sq = smem_u32(sm.q[q]), sk = smem_u32(sm.k[j & 1]);
#pragma unroll
      for (int k = 0; k < HD / 16; ++k)
        umma_w(tmem + q * 256, desc_sw128(sq + (k >> 2) * ATOM + (k & 3) * 32),
               desc_sw128(sk + (k >> 2) * ATOM + (k & 3) * 32), id_s, k > 0 ? 1u : 0u);
      commit_w(&sy.s_full[q]);
    };
    auto issue_pv = [&](int q, int j) {  // O_q += P_q(j) V(j)
      const uint32_t sv = smem_u32(sm.v[j & 1]);
#pragma unroll
      for (int k = 0; k < BN / 16; ++k)
        umma_ts_w(tmem + q * 256 + 128, tmem + q * 256 + k * 8, desc_mn_sw128(sv + k * 2048), id_o,
                  (j > 0 || k > 0) ? 1u : 0u);
      commit_w(&sy.o_done[q]);
    };
    mbar_wait(&sy.k_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    commit_w(&sy.k_empty[0]);
    for (int j = 0; j < nblk; ++j) {
      mbar_wait(&sy.v_full[j & 1], (j >> 1) & 1);
      mbar_wait(&sy.p_full[0], j & 1);
      tc_fence_after();
      issue_pv(0, j);
      const bool more = j + 1 < nblk;
      if (more) {
        mbar_wait(&sy.k_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
        tc_fence_after();
        issue_s(0, j + 1);  // over P_A(j): PV_A(j) was issued first (in order)
      }
      mbar_wait(&sy.p_full[1], j & 1);
      tc_fence_after();
      issue_pv(1, j);
      commit_w(&sy.v_empty[j & 1]);
      if (more) {
        issue_s(1, j + 1);
        commit_w(&sy.k_empty[(j + 1) & 1]);
      }
    }
  } else {
    // ---------------- softmax: tile q = warp / 8; warps w, w+4 of a tile share TMEM lanes
    // 32(w%4).. (query rows), one half of the 128 key columns (and of O's head dim) each
    const int q = warp >> 3, sub = warp & 3, part = (warp >> 2) & 1;
    const int t = sub * 32 + lane;
    const int r = r0 + q * BM + t;
    const KeyBounds kbr = key_bounds(cu, cu_k, q_off, num_seqs, min(r, rows - 1), window);
    const int lo = kbr.lo, hi = kbr.hi;
    // this tile's first / last rows: blocks inside both bounds need no mask
    const int full_lo = key_bounds(cu, cu_k, q_off, num_seqs, min(r0 + q * BM + BM - 1, rows - 1), window).lo;
    const int full_hi = key_bounds(cu, cu_k, q_off, num_seqs, min(r0 + q * BM, rows - 1), window).hi;
    const float qs = scale * 1.4426950408889634f;
    const uint32_t lane_addr = (uint32_t)(sub * 32) << 16;
    const uint32_t s_addr = tmem + lane_addr + q * 256 + part * COLS;
    const uint32_t o_addr = tmem + lane_addr + q * 256 + 128 + part * COLS;
    const uint32_t p_addr = tmem + lane_addr + q * 256 + part * (COLS / 2);
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int jb = j_lo + j * BN;
      mbar_wait(&sy.s_full[q], j & 1);
      tc_fence_after();
      float s[COLS];
      tmem_ld32(s_addr, s);
      tmem_ld32(s_addr + 32, s + 32);
      tmem_wait_ld();
      const bool full = jb >= full_lo && jb + BN - 1 <= full_hi;
      float mx = -INFINITY;
      if (!full) {
#pragma unroll
        for (int i = 0; i < COLS; ++i) {
          const int jj = jb + part * COLS + i;
          if (jj > hi || jj < lo) s[i] = -INFINITY;
        }
      }
      {
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
        for (int i = 0; i < COLS; i += 8) {
          m0 = max3(m0, s[i], s[i + 1]);
          m1 = max3(m1, s[i + 2], s[i + 3]);
          m2 = max3(m2, s[i + 4], s[i + 5]);
          m3 = max3(m3, s[i + 6], s[i + 7]);
        }
        mx = max3(max3(m0, m1, m2), m3, mx);
      }
      float* red = sy.red[q][j % 3];
      smem_max_f32(red + t, mx);
      tc_fence_before();
      named_bar(1 + q * 4 + sub, 64);
      tc_fence_after();
      mx = red[t] * qs;
      if (part == 0) sy.red[q][(j + 2) % 3][t] = -INFINITY;
      const float mn = mx > m + kLazy ? mx : m;
      const float base_m = mn == -INFINITY ? 0.f : mn;
      const float alpha = ex2(m - base_m);
      float2 rs2 = make_float2(0.f, 0.f);
      const float2 qs2 = make_float2(qs, qs), nb2 = make_float2(-base_m, -base_m);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // P in two 16-column stores (fewer live registers)
        uint32_t p16[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = hf * 32 + c * 8 + 2 * e;
            const float2 x = ffma2(make_float2(s[i], s[i + 1]), qs2, nb2);
            const float2 pv = e == 3 ? exp2_fma2(x) : make_float2(ex2(x.x), ex2(x.y));
            rs2 = fadd2(rs2, pv);
            p16[c * 4 + e] = pack_bf16(pv.x, pv.y);
          }
        }
        tmem_st16u(p_addr + hf * 16, p16);
      }
      l = l * alpha + (rs2.x + rs2.y);
      m = mn;
      // O rescale after the scores are dead (register pressure); PV_q(j) is issued only after
      // p_full, so rescaling here is still before P(j) V(j) is added.  PV_q(j-1) must be done.
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        mbar_wait(&sy.o_done[q], (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < COLS; c += 32) {
          float o[32];
          tmem_ld32(o_addr + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] *= alpha;
          tmem_st32(o_addr + c, o);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&sy.p_full[q]);
    }
    atomicAdd(&sy.lsum[q][t], l);
    named_bar(1 + q * 4 + sub, 64);
    l = sy.lsum[q][t];
    mbar_wait(&sy.o_done[q], (nblk - 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = out + (size_t)min(r, rows - 1) * Hq * HD + h * HD + part * COLS;
#pragma unroll 1
    for (int c = 0; c < COLS; c += 32) {
      float o[32];
      tmem_ld32(o_addr + c, o);
      tmem_wait_ld();
      if (r < rows) {
#pragma unroll
        for (int e = 0; e < 32; e += 8) {
          uint4 pk;
          pk.x = pack_bf16(o[e] * inv, o[e + 1] * inv);
          pk.y = pack_bf16(o[e + 2] * inv, o[e + 3] * inv);
          pk.z = pack_bf16(o[e + 4] * inv, o[e + 5] * inv);
          pk.w = pack_bf16(o[e + 6] * inv, o[e + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c + e) = pk;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace fa5

sn_status attn_prefill_umma_bf16(const void* q, const void* k, const void* v, const int32_t* cu, void* out,
                                 int num_seqs, int rows, int Hq, int Hkv, int window, float scale,
                                 const int32_t* cu_k, const int32_t* q_off, int rows_k, cudaStream_t st) {
  using namespace fa5;
  CUtensorMap qm, km, vm;
  if (!map_2d(&qm, q, rows, (uint64_t)Hq * HD, (uint64_t)Hq * HD, BM) ||
      !map_2d(&km, k, rows_k, (uint64_t)Hkv * HD, (uint64_t)Hkv * HD, BN) ||
      !map_2d(&vm, v, rows_k, (uint64_t)Hkv * HD, (uint64_t)Hkv * HD, BN)) {
    set_error("sn_attn_prefill: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  // The round-1 A/B variants (one query tile per CTA with 3-stage K/V rings, P through shared
  // memory, 16 softmax warps, more exponentials on the FMA pipe) all measured at or below this
  // kernel (profiles/r01_attn_prefill_umma_ncu.txt) and were removed.
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_umma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    attr = true;
  }
  attn_prefill_umma2_kernel<<<dim3((rows + 2 * BM - 1) / (2 * BM), Hq), kThreads2, kSmemBytes, st>>>(
      qm, km, vm, cu, (__nv_bfloat16*)out, num_seqs, rows, Hq, Hkv, window, scale, cu_k, q_off);
  return check_launch("sn_attn_prefill(umma2)");
}

}  // namespace sn
