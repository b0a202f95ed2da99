// Chunked (WY / UT-transform) GDN prefill on tensor cores (R/PAPER.md:1599: "Training
// uses a chunkwise parallel algorithm based on the WY representation"; §6 prefill path,
// R/PAPER.md:845-848).  Oracle: the token-by-token recurrence (oracle/supernet_oracle.py),
// itself pinned to FLA's naive_chunk_gated_delta_rule (3P-FLA/ops/gated_delta_rule/naive.py:67-161).
//
// Per chunk of C = 64 tokens (G = in-chunk cumulative log decay, Gamma_ij = e^{G_i - G_j}):
//   L  = -tril(diag(b) K K^T o Gamma, -1)          T = (I - L)^{-1}   (forward substitution)
//   W  = T (b o e^G o K)      U = T (b o V)         P = tril(Q K^T o Gamma)
//   V' = U - W S              O = (e^G o Q) S + P V'
//   S  = e^{G_C} S + (e^{G_C - G} o K)^T V'
// Every product is a 64 x {64,128} x {64,128} bf16 tensor-core tile (mma.sync m16n8k16,
// fp32 accumulate); the state S stays in registers (fp32) across chunks.  One CTA (4 warps)
// per (sequence, value head, 64-wide value tile); chunks run in order inside it.
#include "sn_mma.cuh"
#include "sn_tc.cuh"

namespace sn {
namespace chunk {

using namespace sn::mma;

constexpr int C = 64;      // chunk length
constexpr int VT = 64;     // value columns per CTA
constexpr int kThreads = 128;


// T = (I - L)^{-1} for a strictly lower-triangular 64x64 L (fp32 rows of stride C + 1).
// Blocked: each warp inverts one 16x16 diagonal block by warp-synchronous substitution
// (lane j < 16 owns column j in registers: T_ii = I + L_ii T_ii), then the three block rows
// below the diagonal, T_ij = T_ii sum_{k=j}^{i-1} L_ik T_kj, one warp per block — 3 block
// barriers instead of one per row.  Same fp32 arithmetic as row-by-row substitution, only
// reassociated.  All 128 threads must call; l must be complete (caller synchronises);
// x is complete on return.  scr: 4 x 16 x 17 floats.
__device__ __forceinline__ void invert_unit_lower(const float (*l)[C + 1], float (*x)[C + 1], float* scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {  // diagonal blocks
    const int b0 = 16 * warp, j = lane;
    if (lane < 16) {
      float xc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float acc = 0.f;
#pragma unroll
        for (int m = 0; m < i; ++m) acc += l[b0 + i][b0 + m] * xc[m];
        xc[i] = i < j ? 0.f : (i == j ? 1.f : acc);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) x[b0 + i][b0 + j] = xc[i];
    }
  }
  for (int idx = tid; idx < 6 * 256; idx += kThreads) {  // blocks above the diagonal are zero
    const int blk = idx >> 8, e = idx & 255;
    const int bi = blk < 3 ? 0 : (blk < 5 ? 1 : 2), bj = blk < 3 ? blk + 1 : (blk < 5 ? blk - 1 : 3);
    x[16 * bi + (e >> 4)][16 * bj + (e & 15)] = 0.f;
  }
  __syncthreads();
  const int r = lane >> 1, c0 = (lane & 1) * 8;
  float* M = scr + warp * 16 * 17;
  for (int bi = 1; bi < 4; ++bi) {
    if (warp < bi) {
      const int bj = warp;
      float acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.f;
      for (int k = bj; k < bi; ++k)
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const float a = l[16 * bi + r][16 * k + m];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] += a * x[16 * k + m][16 * bj + c0 + c];
        }
#pragma unroll
      for (int c = 0; c < 8; ++c) M[r * 17 + c0 + c] = acc[c];
      __syncwarp();
      float res[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) res[c] = 0.f;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float a = x[16 * bi + r][16 * bi + m];
#pragma unroll
        for (int c = 0; c < 8; ++c) res[c] += a * M[m * 17 + c0 + c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) x[16 * bi + r][16 * bj + c0 + c] = res[c];
      __syncwarp();
    }
    __syncthreads();
  }
}


// The same inverse computed in place (T overwrites L: saves the second 64 x 65 fp32 tile).
// Diagonal blocks first (a warp's lanes read their block of L before any lane writes T into
// it); then, per block row bi, every warp first accumulates sum_k L_ik T_kj from blocks of
// row bi that still hold L, a barrier, and only then the T_ij replace them.
__device__ __forceinline__ void invert_unit_lower_inplace(float (*lx)[C + 1], float* scr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {  // diagonal blocks (the blocks above the diagonal already hold zeros: L is strictly lower)
    const int b0 = 16 * warp, j = lane;
    float xc[16];
    if (lane < 16) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float acc = 0.f;
#pragma unroll
        for (int m = 0; m < i; ++m) acc += lx[b0 + i][b0 + m] * xc[m];
        xc[i] = i < j ? 0.f : (i == j ? 1.f : acc);
      }
    }
    __syncwarp();
    if (lane < 16) {
#pragma unroll
      for (int i = 0; i < 16; ++i) lx[b0 + i][b0 + j] = xc[i];
    }
  }
  __syncthreads();
  const int r = lane >> 1, c0 = (lane & 1) * 8;
  float* M = scr + warp * 16 * 17;
  for (int bi = 1; bi < 4; ++bi) {
    if (warp < bi) {
      const int bj = warp;
      float acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.f;
      for (int k = bj; k < bi; ++k)
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const float a = lx[16 * bi + r][16 * k + m];  // L (row bi is replaced only below)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] += a * lx[16 * k + m][16 * bj + c0 + c];
        }
#pragma unroll
      for (int c = 0; c < 8; ++c) M[r * 17 + c0 + c] = acc[c];
    }
    __syncthreads();  // every L block of row bi has been read
    if (warp < bi) {
      const int bj = warp;
      float res[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) res[c] = 0.f;
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const float a = lx[16 * bi + r][16 * bi + m];
#pragma unroll
        for (int c = 0; c < 8; ++c) res[c] += a * M[m * 17 + c0 + c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) lx[16 * bi + r][16 * bj + c0 + c] = res[c];
    }
    __syncthreads();
  }
}

// =====================================================================================
// Two-phase version (the long-prefill path): the chunk-local work (inverse, W, U, P and
// the decayed operands) of all chunks runs in parallel, one CTA per (chunk, value head);
// the sequential state pass then only streams the precomputed tiles through
// double-buffered shared memory and runs the four state-dependent tile products.
// Workspace per (chunk, head), bf16: W, Qg, Kd, U [64][D] and P [64][64]; glast fp32.

template <int D>
__device__ __forceinline__ size_t ws_tile(int n, int h, int Hv) {  // offset of one (chunk, head) record
  return ((size_t)n * Hv + h) * (4 * (size_t)C * D + (size_t)C * C);
}

// ---- GDN chunk-local phase on tcgen05 / TMEM, TMA-fed.  One CTA (4 warps) per (chunk, value
// head).  TMA brings Q, K (bf16, from sn_delta_prep) and V (the conv output) as [64 x D] tiles of
// 128B-swizzled [64 x 64] atoms; the four chunk products run as single-thread UMMAs (M = 64):
//   K K^T, Q K^T           (A, B K-major: the K tile serves both)        -> TMEM cols [0, 128)
//   W = T2 K, U = T1 V     (A = T2 / T1 written swizzled by the CTA, B = K / V MN-major)
//                                                                        -> TMEM cols [0, 2D)
// with T1 = T diag(b), T2 = T diag(b e^G): the beta / decay scaling of the right operands is
// folded into the columns of T, so K and V are consumed straight from their TMA tiles.  The
// inverse T = (I - L)^-1 stays on the CUDA cores (invert_unit_lower, fp32).  Rows past the
// chunk length are whatever the TMA box covers (the next chunk, or zeros past the tensor):
// their beta is 0, so their columns of T1 / T2 are 0, and P / Qg / Kd mask them explicitly.
template <int D>
struct TcIntraSmem {
  static constexpr int AT = 64 * 128;  // one [64 rows x 64 bf16] 128B-swizzled atom
  static constexpr int NA = D / 64;    // atoms per [64 x D] tile
  uint8_t k[NA * AT];
  uint8_t v[NA * AT];
  union {  // Q until its products / outputs are done, then L -> T in place, then T1 / T2
    uint8_t q[NA * AT];
    struct {
      float lx[C][C + 1];
      float scr[4 * 16 * 17];
    } b;
    struct { uint8_t t1[AT]; uint8_t t2[AT]; } t;
  } u;
  float g[C], beta[C], bg[C];  // bg = b e^G (the column scale of T2)
  uint64_t bar_qk, bar_v, bar_m1, bar_m2, bar_m3;
  uint32_t tmem_base;
};

// byte offset of element (r, c) in a [64 x D] tile of 128B-swizzled [64 x 64] atoms
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
  const int atom = c >> 6, cc = c & 63;
  return atom * (64 * 128) + r * 128 + ((((cc >> 3) ^ (r & 7)) & 7) << 4) + ((cc & 7) << 1);
}

// MN-major SW128 operand (B of W = T2 K, U = T1 V: N = head dim contiguous, K = chunk rows):
// LBO = stride between the 64-element N atoms, SBO = 8 K rows x 128 B
__device__ __forceinline__ uint64_t desc_mn_sw128_c(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((64 * 128) >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int D>
__global__ void __launch_bounds__(kThreads)
    gdn_chunk_intra_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                              const __grid_constant__ CUtensorMap vmap, int v_off, const float* __restrict__ glog,
                              const float* __restrict__ beta, const int32_t* __restrict__ chunks,
                              __nv_bfloat16* __restrict__ ws, float* __restrict__ glast, int Hk, int Hv) {
  pdl_launch_dependents();
  using SM = TcIntraSmem<D>;
  constexpr int AT = SM::AT, NA = SM::NA;
  constexpr uint32_t kCols = 128;  // K K^T | Q K^T, then W, then U (3 CTAs per SM)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = blockIdx.x, h = blockIdx.y;
  const int kh = h / (Hv / Hk);
  if (tid == 0) {
    tc::mbar_init(&sm.bar_qk, 1);
    tc::mbar_init(&sm.bar_v, 1);
    tc::mbar_init(&sm.bar_m1, 1);
    tc::mbar_init(&sm.bar_m2, 1);
    tc::mbar_init(&sm.bar_m3, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&sm.tmem_base)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_wait();
  const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
  if (tid < C) {
    sm.g[tid] = tid < len ? glog[(size_t)(c0 + tid) * Hv + h] : 0.f;
    sm.beta[tid] = tid < len ? beta[(size_t)(c0 + tid) * Hv + h] : 0.f;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  if (tid == 0) {  // the three tiles, one TMA box per 64-column atom
    const uint64_t pol = tc::policy_evict_first();
    tc::mbar_expect_tx(&sm.bar_qk, 2 * NA * AT);
    for (int a = 0; a < NA; ++a) {
      tc::tma_load_2d(sm.u.q + a * AT, &qmap, kh * D + 64 * a, c0, &sm.bar_qk, pol);
      tc::tma_load_2d(sm.k + a * AT, &kmap, kh * D + 64 * a, c0, &sm.bar_qk, pol);
    }
    tc::mbar_expect_tx(&sm.bar_v, NA * AT);
    for (int a = 0; a < NA; ++a) tc::tma_load_2d(sm.v + a * AT, &vmap, v_off + h * D + 64 * a, c0, &sm.bar_v, pol);
  }
  if (warp == 0) {  // in-chunk cumulative log decay
    float a0 = sm.g[lane], a1 = sm.g[32 + lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float n0 = __shfl_up_sync(0xffffffffu, a0, o), n1 = __shfl_up_sync(0xffffffffu, a1, o);
      if (lane >= o) { a0 += n0; a1 += n1; }
    }
    a1 += __shfl_sync(0xffffffffu, a0, 31);
    sm.g[lane] = a0;
    sm.g[32 + lane] = a1;
    sm.bg[lane] = sm.beta[lane] * expf(a0);
    sm.bg[32 + lane] = sm.beta[32 + lane] * expf(a1);
  } else if (warp == 1) {  // K K^T -> TMEM [0, 64), Q K^T -> [64, 128)
    tc::mbar_wait(&sm.bar_qk, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t sq = tc::smem_u32(sm.u.q), sk = tc::smem_u32(sm.k), id = tc::idesc_bf16(64, 64);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = (kk >> 2) * AT + (kk & 3) * 32;
      tc::umma_w(tmem, tc::desc_sw128(sk + off), tc::desc_sw128(sk + off), id, kk > 0 ? 1u : 0u);
      tc::umma_w(tmem + 64, tc::desc_sw128(sq + off), tc::desc_sw128(sk + off), id, kk > 0 ? 1u : 0u);
    }
    tc::commit_w(&sm.bar_m1);
  }
  __syncthreads();  // the cumulative decays

  __nv_bfloat16* rec = ws + ws_tile<D>(n, h, Hv);
  __nv_bfloat16* wW = rec;
  __nv_bfloat16* wQg = rec + C * D;
  __nv_bfloat16* wKd = rec + 2 * C * D;
  __nv_bfloat16* wU = rec + 3 * C * D;
  __nv_bfloat16* wP = rec + 4 * C * D;
  // e^G o Q and e^{G_C - G} o K straight from the swizzled tiles (8 columns per step)
  tc::mbar_wait(&sm.bar_qk, 0);
  const float gl = sm.g[C - 1];
  for (int idx = tid; idx < C * D / 8; idx += kThreads) {
    const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
    const uint4 qv = *reinterpret_cast<const uint4*>(sm.u.q + sw_off(r, c8));
    const uint4 kv = *reinterpret_cast<const uint4*>(sm.k + sw_off(r, c8));
    const bool ok = r < len;
    const float eg = ok ? expf(sm.g[r]) : 0.f, ed = ok ? expf(gl - sm.g[r]) : 0.f;
    const uint32_t* qa = reinterpret_cast<const uint32_t*>(&qv);
    const uint32_t* ka = reinterpret_cast<const uint32_t*>(&kv);
    uint4 qo, ko;
    uint32_t* qoa = reinterpret_cast<uint32_t*>(&qo);
    uint32_t* koa = reinterpret_cast<uint32_t*>(&ko);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qa[e]));
      const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
      qoa[e] = pack_bf16(qf.x * eg, qf.y * eg);
      koa[e] = pack_bf16(kf.x * ed, kf.y * ed);
    }
    *reinterpret_cast<uint4*>(wQg + r * D + c8) = qo;
    *reinterpret_cast<uint4*>(wKd + r * D + c8) = ko;
  }
  if (tid == 0) glast[(size_t)n * Hv + h] = gl;
  __syncthreads();  // every read of Q is done: L / X take its place

  // L = -tril(b K K^T o Gamma, -1) -> shared memory, P = tril(Q K^T o Gamma) -> workspace.
  // M = 64 accumulator: row 16w + i sits in TMEM lane 32w + i (i < 16).
  tc::mbar_wait(&sm.bar_m1, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int i = 16 * warp + (lane & 15);
    const bool row = lane < 16;
    const uint32_t la = tmem + ((uint32_t)(32 * warp) << 16);
    const float gi = sm.g[i], bi = sm.beta[i];
#pragma unroll 1
    for (int j0 = 0; j0 < C; j0 += 16) {
      float kk[16], qk[16];
      tc::tmem_ld16_async(la + j0, kk);
      tc::tmem_ld16_async(la + 64 + j0, qk);
      tc::tmem_wait_ld();
      tc::reg_fence16(kk);
      tc::reg_fence16(qk);
      if (row) {
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          float pv[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const int j = j0 + e + d;
            const bool ok = i < len && j < len && i >= j;
            const float gam = ok ? expf(gi - sm.g[j]) : 0.f;
            sm.u.b.lx[i][j] = (ok && i > j) ? -bi * kk[e + d] * gam : 0.f;
            pv[d] = qk[e + d] * gam;
          }
          pk[e >> 1] = pack_bf16(pv[0], pv[1]);
        }
        *reinterpret_cast<uint4*>(wP + i * C + j0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(wP + i * C + j0 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  invert_unit_lower_inplace(sm.u.b.lx, sm.u.b.scr);  // lx = T = (I - L)^-1 (fp32)
  // T1 = T diag(b), T2 = T diag(b e^G) as bf16 K-major A operands (swizzled like a TMA atom),
  // written over T itself: every thread first holds its 4 x 8 entries of T in registers
  constexpr int TI = C * C / 8 / kThreads;
  uint32_t p1[TI][4], p2[TI][4];
#pragma unroll
  for (int u = 0; u < TI; ++u) {
    const int idx = tid + u * kThreads, i = idx >> 3, j8 = (idx & 7) * 8;
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float x0 = sm.u.b.lx[i][j8 + e], x1 = sm.u.b.lx[i][j8 + e + 1];
      p1[u][e >> 1] = pack_bf16(x0 * sm.beta[j8 + e], x1 * sm.beta[j8 + e + 1]);
      p2[u][e >> 1] = pack_bf16(x0 * sm.bg[j8 + e], x1 * sm.bg[j8 + e + 1]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < TI; ++u) {
    const int idx = tid + u * kThreads, i = idx >> 3, j8 = (idx & 7) * 8;
    *reinterpret_cast<uint4*>(sm.u.t.t1 + sw_off(i, j8)) = make_uint4(p1[u][0], p1[u][1], p1[u][2], p1[u][3]);
    *reinterpret_cast<uint4*>(sm.u.t.t2 + sw_off(i, j8)) = make_uint4(p2[u][0], p2[u][1], p2[u][2], p2[u][3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> the MMA's reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  // W = T2 K, then U = T1 V, each through TMEM columns [0, D) (K and V read MN-major from
  // their TMA tiles); the U product is issued once every warp has drained W
  const uint32_t idw = tc::idesc_bf16(64, D) | (1u << 16);  // B MN-major
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t s2 = tc::smem_u32(sm.u.t.t2), sk = tc::smem_u32(sm.k);
#pragma unroll
    for (int kk = 0; kk < C / 16; ++kk)
      tc::umma_w(tmem, tc::desc_sw128(s2 + kk * 32), desc_mn_sw128_c(sk + kk * 2048), idw, kk > 0 ? 1u : 0u);
    tc::commit_w(&sm.bar_m2);
  }
  auto drain = [&](__nv_bfloat16* dst) {  // TMEM [0, D) -> bf16 rows of the workspace
    const int i = 16 * warp + (lane & 15);
    const uint32_t la = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      float va[16], vb[16];
      tc::tmem_ld16_async(la + c, va);
      tc::tmem_ld16_async(la + c + 16, vb);
      tc::tmem_wait_ld();
      tc::reg_fence16(va);
      tc::reg_fence16(vb);
      if (lane < 16) {
        uint32_t pa[8], pb[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          pa[e] = pack_bf16(va[2 * e], va[2 * e + 1]);
          pb[e] = pack_bf16(vb[2 * e], vb[2 * e + 1]);
        }
        *reinterpret_cast<uint4*>(dst + i * D + c) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
        *reinterpret_cast<uint4*>(dst + i * D + c + 8) = make_uint4(pa[4], pa[5], pa[6], pa[7]);
        *reinterpret_cast<uint4*>(dst + i * D + c + 16) = make_uint4(pb[0], pb[1], pb[2], pb[3]);
        *reinterpret_cast<uint4*>(dst + i * D + c + 24) = make_uint4(pb[4], pb[5], pb[6], pb[7]);
      }
    }
  };
  tc::mbar_wait(&sm.bar_m2, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  drain(wW);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();  // W drained: U reuses its columns
  if (warp == 1) {
    tc::mbar_wait(&sm.bar_v, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t s1 = tc::smem_u32(sm.u.t.t1), sv = tc::smem_u32(sm.v);
#pragma unroll
    for (int kk = 0; kk < C / 16; ++kk)
      tc::umma_w(tmem, tc::desc_sw128(s1 + kk * 32), desc_mn_sw128_c(sv + kk * 2048), idw, kk > 0 ? 1u : 0u);
    tc::commit_w(&sm.bar_m3);
  }
  tc::mbar_wait(&sm.bar_m3, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  drain(wU);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// Sequential state pass, warp-specialised (8 warps): warps 0-3 run the recurrence chain of a
// chunk, V' = U - W S and S <- e^{G_C} S + Kd^T V', with S in registers (fp32); warps 4-7
// compute the chunk's output O = Qg S + P V' from the bf16 copies of S and V' the chain warps
// publish, one chunk behind, so the output products (the larger half of the MMAs) leave the
// chain's critical path.  Handoff through double-buffered S / V' tiles and named barriers:
// full[b] (chain -> output: S_n, V'_n in buffer b = n & 1 ready), empty[b] (output -> chain:
// buffer b free again).  Each group streams its own operands of the next chunk (cp.async): the
// chain W, Kd, U and the chunk's decay (a global load of the decay on the chain cost 10 %), the
// output Qg, P.  Measured (tools/bench_prefill.py, 16K tokens, 32 heads): 475 us vs 529 us for
// the single-group kernel with a per-chunk global decay load.
constexpr int kStateThreads = 256;

template <int D, int VTT = VT>
struct StateSmem {
  static constexpr int LDK = D + 8, LDV = VTT + 8, LDC = C + 8;
  // operand buffers per group: the next chunk is in flight while this one is consumed (three
  // buffers measured 2 % slower: 482 vs 475 us for 16K tokens)
  static constexpr int NS = 2;
  struct ChainStage {
    __nv_bfloat16 w[C * LDK];
    __nv_bfloat16 kd[C * LDK];
    __nv_bfloat16 u[C * LDV];
    float gl[D];  // the chunk's last cumulative log decay (GDN: gl[0]; KDA: per key channel)
  } cs[NS];
  struct OutStage {
    __nv_bfloat16 qg[C * LDK];
    __nv_bfloat16 p[C * LDC];
  } os[NS];
  __nv_bfloat16 s[2][D * LDV];
  __nv_bfloat16 vp[2][C * LDV];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
enum : int { kBarChain = 1, kBarOut = 2, kBarFull = 3, kBarEmpty = 5 };  // full / empty: + buffer

// PERCH (KDA): glast holds the chunk's per-key-channel cumulative log decay [D] per (chunk,
// head) and S is decayed row-wise, diag(e^{G_C}) S; otherwise one scalar per (chunk, head).
template <int D, bool PERCH = false, int VTT = VT>
__global__ void __launch_bounds__(kStateThreads, 1)
    gdn_chunk_state_kernel(const __nv_bfloat16* __restrict__ ws, const float* __restrict__ glast,
                           const int32_t* __restrict__ chunks, const int32_t* __restrict__ seq_chunk0,
                           float* __restrict__ o, float* __restrict__ state, const int32_t* __restrict__ slot_idx,
                           int Hv, int init_state) {
  pdl_launch_dependents();
  using SM = StateSmem<D, VTT>;
  constexpr int NTV = VTT / 8;  // n8 tiles of this CTA's value columns
  constexpr int LDK = SM::LDK, LDV = SM::LDV, LDC = SM::LDC;
  constexpr int MT = D / 64;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x & 127, lane = tid & 31, warp = tid >> 5;  // index within the group
  const bool chain = threadIdx.x < 128;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int vt = blockIdx.x, h = blockIdx.y, seq = blockIdx.z;
  const int slot = slot_idx ? slot_idx[seq] : seq;
  const int n0 = seq_chunk0[seq], n1 = seq_chunk0[seq + 1];
  float* Sg = state + ((size_t)slot * Hv + h) * D * D;

  if (chain) {
    float sf[MT][NTV][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kr = (warp * MT + mt) * 16 + g4 + ((e >> 1) << 3);
          const int vc = vt * VTT + nt * 8 + t4 * 2 + (e & 1);
          sf[mt][nt][e] = init_state ? Sg[(size_t)vc * D + kr] : 0.f;
        }
    auto load = [&](int n, int b) {  // W, Kd (rows of D) and this CTA's U columns
      const __nv_bfloat16* rec = ws + ws_tile<D>(n, h, Hv);
      typename SM::ChainStage& S = sm.cs[b];
      for (int idx = tid; idx < C * D / 8; idx += 128) {
        const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
        cp_async16(&S.w[r * LDK + c8], rec + r * D + c8);
        cp_async16(&S.kd[r * LDK + c8], rec + 2 * C * D + r * D + c8);
      }
      for (int idx = tid; idx < C * VTT / 8; idx += 128) {
        const int r = idx / (VTT / 8), c8 = (idx % (VTT / 8)) * 8;
        cp_async16(&S.u[r * LDV + c8], rec + 3 * C * D + r * D + vt * VTT + c8);
      }
      if (PERCH) {
        if (tid < D / 4) cp_async16(&S.gl[4 * tid], glast + ((size_t)n * Hv + h) * D + 4 * tid);
      } else if (tid == 0) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(&S.gl[0])),
                     "l"(glast + (size_t)n * Hv + h)
                     : "memory");
      }
      cp_async_commit();
    };
    constexpr int NS = SM::NS;
    for (int j = 0; j < NS - 1; ++j) {  // chunks n0 .. n0 + NS - 2 in flight
      if (n0 + j < n1) load(n0 + j, j);
      else cp_async_commit();
    }
    for (int n = n0; n < n1; ++n) {
      const int i = n - n0, b = i & 1, sb = i % NS;
      if (n + NS - 1 < n1) load(n + NS - 1, (i + NS - 1) % NS);  // into the buffer of chunk n - 1
      else cp_async_commit();
      cp_async_wait<NS - 1>();  // chunk n's group is complete
      if (i >= 2) named_sync(kBarEmpty + b, 256);  // the output warps are done with buffer b
      __nv_bfloat16* s_b = sm.s[b];
      __nv_bfloat16* vp_b = sm.vp[b];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)  // S -> bf16 operand
#pragma unroll
        for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
          for (int e = 0; e < 4; e += 2) {
            const int kr = (warp * MT + mt) * 16 + g4 + ((e >> 1) << 3);
            *reinterpret_cast<uint32_t*>(&s_b[kr * LDV + nt * 8 + t4 * 2]) = pack_bf16(sf[mt][nt][e], sf[mt][nt][e + 1]);
          }
      named_sync(kBarChain, 128);  // S_n and this chunk's operands visible to the group
      typename SM::ChainStage& St = sm.cs[sb];
      // V' = U - W S
      float vpc[NTV][4];
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = warp * 16 + g4 + ((e >> 1) << 3), cc = nt * 8 + t4 * 2 + (e & 1);
          vpc[nt][e] = __bfloat162float(St.u[r * LDV + cc]);
        }
#pragma unroll
      for (int ks = 0; ks < D; ks += 16) {
        uint32_t a[4];
        lda(St.w, LDK, warp * 16, ks, a);
#pragma unroll
        for (int nt = 0; nt < NTV; nt += 2) {
          uint32_t b0, b1, b2, b3;
          ldb_kn(s_b, LDV, nt * 8, ks, b0, b1, b2, b3);
          float ws0[4] = {0.f, 0.f, 0.f, 0.f}, ws1[4] = {0.f, 0.f, 0.f, 0.f};
          mma_bf16(ws0, a, b0, b1);
          mma_bf16(ws1, a, b2, b3);
#pragma unroll
          for (int e = 0; e < 4; ++e) { vpc[nt][e] -= ws0[e]; vpc[nt + 1][e] -= ws1[e]; }
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const int r = warp * 16 + g4 + ((e >> 1) << 3);
          *reinterpret_cast<uint32_t*>(&vp_b[r * LDV + nt * 8 + t4 * 2]) = pack_bf16(vpc[nt][e], vpc[nt][e + 1]);
        }
      named_sync(kBarChain, 128);  // V'_n complete (the S update reads all of it)
      named_arrive(kBarFull + b, 256);  // -> output warps: S_n, V'_n in buffer b
      // S = e^{G_C} S + Kd^T V'   (KDA: diag(e^{G_C}) S, one factor per key row)
      if (PERCH) {
        const float* gl = St.gl;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const float dec = expf(gl[(warp * MT + mt) * 16 + g4 + (e2 << 3)]);
#pragma unroll
            for (int nt = 0; nt < NTV; ++nt) {
              sf[mt][nt][2 * e2] *= dec;
              sf[mt][nt][2 * e2 + 1] *= dec;
            }
          }
      } else {
        const float dec = expf(St.gl[0]);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) sf[mt][nt][e] *= dec;
      }
#pragma unroll
      for (int ks = 0; ks < C; ks += 16) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a[4];
          lda_t(St.kd, LDK, (warp * MT + mt) * 16, ks, a);
#pragma unroll
          for (int nt = 0; nt < NTV; nt += 2) {
            uint32_t b0, b1, b2, b3;
            ldb_kn(vp_b, LDV, nt * 8, ks, b0, b1, b2, b3);
            mma_bf16(sf[mt][nt], a, b0, b1);
            mma_bf16(sf[mt][nt + 1], a, b2, b3);
          }
        }
      }
      named_sync(kBarChain, 128);  // stage sb is re-filled by a later iteration's load
    }
    // the output warps' last two arrivals on empty[] (every arrival is consumed)
    for (int i = (n1 - n0 >= 2 ? n1 - n0 - 2 : 0); i < n1 - n0; ++i) named_sync(kBarEmpty + (i & 1), 256);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kr = (warp * MT + mt) * 16 + g4 + ((e >> 1) << 3);
          const int vc = vt * VTT + nt * 8 + t4 * 2 + (e & 1);
          Sg[(size_t)vc * D + kr] = sf[mt][nt][e];
        }
  } else {  // ---------------- output warps: O = Qg S + P V'
    auto load = [&](int n, int b) {
      const __nv_bfloat16* rec = ws + ws_tile<D>(n, h, Hv);
      typename SM::OutStage& S = sm.os[b];
      for (int idx = tid; idx < C * D / 8; idx += 128) {
        const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
        cp_async16(&S.qg[r * LDK + c8], rec + C * D + r * D + c8);
      }
      for (int idx = tid; idx < C * C / 8; idx += 128) {
        const int r = idx / (C / 8), c8 = (idx % (C / 8)) * 8;
        cp_async16(&S.p[r * LDC + c8], rec + 4 * C * D + r * C + c8);
      }
      cp_async_commit();
    };
    constexpr int NS = SM::NS;
    for (int j = 0; j < NS - 1; ++j) {
      if (n0 + j < n1) load(n0 + j, j);
      else cp_async_commit();
    }
    for (int n = n0; n < n1; ++n) {
      const int i = n - n0, b = i & 1, sb = i % NS;
      if (n + NS - 1 < n1) load(n + NS - 1, (i + NS - 1) % NS);
      else cp_async_commit();
      cp_async_wait<NS - 1>();
      named_sync(kBarOut, 128);           // this chunk's Qg / P visible to the group
      named_sync(kBarFull + b, 256);      // S_n, V'_n published by the chain warps
      typename SM::OutStage& St = sm.os[sb];
      const __nv_bfloat16* s_b = sm.s[b];
      const __nv_bfloat16* vp_b = sm.vp[b];
      const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
      float oc[NTV][4];
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) oc[nt][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D; ks += 16) {
        uint32_t a[4];
        lda(St.qg, LDK, warp * 16, ks, a);
#pragma unroll
        for (int nt = 0; nt < NTV; nt += 2) {
          uint32_t b0, b1, b2, b3;
          ldb_kn(s_b, LDV, nt * 8, ks, b0, b1, b2, b3);
          mma_bf16(oc[nt], a, b0, b1);
          mma_bf16(oc[nt + 1], a, b2, b3);
        }
      }
#pragma unroll
      for (int ks = 0; ks < C; ks += 16) {
        uint32_t a[4];
        lda(St.p, LDC, warp * 16, ks, a);
#pragma unroll
        for (int nt = 0; nt < NTV; nt += 2) {
          uint32_t b0, b1, b2, b3;
          ldb_kn(vp_b, LDV, nt * 8, ks, b0, b1, b2, b3);
          mma_bf16(oc[nt], a, b0, b1);
          mma_bf16(oc[nt + 1], a, b2, b3);
        }
      }
      named_sync(kBarOut, 128);           // every output warp is done with S_n / V'_n / stage sb
      named_arrive(kBarEmpty + b, 256);   // -> chain: buffer b free
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const int r = warp * 16 + g4 + ((e >> 1) << 3), cc = vt * VTT + nt * 8 + t4 * 2;
          if (r < len)
            *reinterpret_cast<float2*>(o + ((size_t)(c0 + r) * Hv + h) * D + cc) = make_float2(oc[nt][e], oc[nt][e + 1]);
        }
    }
  }
}

// The state pass is sequential over chunks: with few (sequence, head) pairs the value tiles get
// narrower (64 -> 32 columns) so that more CTAs run their chains side by side.  (16 columns
// measured slower: every CTA still streams the full W / Qg / Kd tiles of each chunk.)
template <int D, bool PERCH>
static void launch_state_pass(const __nv_bfloat16* ws, const float* glast, const int32_t* chunks,
                              const int32_t* seq_chunk0, float* o, float* state, const int32_t* slot_idx,
                              int num_seqs, int H, int init_state, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gdn_chunk_state_kernel<D, PERCH, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(StateSmem<D, 64>));
    cudaFuncSetAttribute(gdn_chunk_state_kernel<D, PERCH, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(StateSmem<D, 32>));
    attr = true;
  }
  int vt = 64;
  if (num_seqs * H * (D / 64) < 148) vt = 32;
  if (vt == 64)
    gdn_chunk_state_kernel<D, PERCH, 64><<<dim3(D / 64, H, num_seqs), kStateThreads, sizeof(StateSmem<D, 64>), st>>>(
        ws, glast, chunks, seq_chunk0, o, state, slot_idx, H, init_state);
  else
    gdn_chunk_state_kernel<D, PERCH, 32><<<dim3(D / 32, H, num_seqs), kStateThreads, sizeof(StateSmem<D, 32>), st>>>(
        ws, glast, chunks, seq_chunk0, o, state, slot_idx, H, init_state);
}

template <int D>
static sn_status launch_two_phase(const void* qb, const void* kb, const void* qkv, int v_off, int qkv_stride,
                                  int rows, const float* glog, const float* beta, const int32_t* chunks,
                                  const int32_t* seq_chunk0, int num_chunks, void* ws, float* glast, float* o,
                                  float* state, const int32_t* slot_idx, int num_seqs, int Hk, int Hv,
                                  int init_state, cudaStream_t st) {
  const int smem = (int)sizeof(TcIntraSmem<D>) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gdn_chunk_intra_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  CUtensorMap qm, km, vm;
  if (!tc::map_2d(&qm, qb, rows, (uint64_t)Hk * D, (uint64_t)Hk * D, 64) ||
      !tc::map_2d(&km, kb, rows, (uint64_t)Hk * D, (uint64_t)Hk * D, 64) ||
      !tc::map_2d(&vm, qkv, rows, qkv_stride, qkv_stride, 64)) {
    set_error("sn_gdn_chunk_prefill2: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  cudaError_t e = launch_pdl(gdn_chunk_intra_tc_kernel<D>, dim3(num_chunks, Hv), dim3(kThreads), (size_t)smem, st, qm,
                             km, vm, v_off, glog, beta, chunks, (__nv_bfloat16*)ws, glast, Hk, Hv);
  if (e != cudaSuccess) {
    set_error("sn_gdn_chunk_prefill2(intra) launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  sn_status s = check_launch("sn_gdn_chunk_prefill(intra)");
  if (s != SN_OK) return s;
  launch_state_pass<D, false>((const __nv_bfloat16*)ws, glast, chunks, seq_chunk0, o, state, slot_idx, num_seqs, Hv,
                              init_state, st);
  return check_launch("sn_gdn_chunk_prefill(state)");
}

// =====================================================================================
// KDA (per-key-channel gate) chunk-local phase.  Oracle: the token recurrence
// S_t = (I - b k k^T) diag(e^{g_t}) S_{t-1} + b k v^T (oracle/supernet_oracle.py), pinned to
// FLA's naive_chunk_kda (3P-FLA/ops/kda/naive.py:69-166), whose chunk form this follows with
// G = in-chunk cumulative log decay per channel:
//   A_kk[i][j] = b_i sum_d k_id k_jd e^{G_id - G_jd} (i > j),  A_qk[i][j] = sum_d q_id k_jd e^{G_id - G_jd} (i >= j)
//   T = (I + A_kk)^{-1},  W = T (b o e^G o K),  U = T (b o V),  Qg = e^G o Q,  Kd = e^{G_C - G} o K
// The state pass is the GDN one with a per-channel decay (gdn_chunk_state_kernel<D, true>).
// Per-channel decay factors cannot be pulled out of a plain K K^T product (G spans up to
// hundreds in a 64-token chunk: e^{-G} overflows fp32), so warp w (rows 16w..16w+15, one
// 16-token sub-chunk) factorises the blocks left of its diagonal around its own
// reference row r = 16w:
//   e^{G_i - G_j} = e^{G_i - G_r} . e^{G_r - G_j},   e^{G_i - G_r} <= 1 (i >= r), e^{G_r - G_j} <= 1 (j < r)
// The diagonal 16x16 block (r <= j <= i) is computed exactly in fp32 with e^{G_i - G_j} <= 1
// per term (a factorised form would need e^{G_r - G_j} > 1, which overflows for strong
// gates).
//

// On tcgen05 / TMEM, TMA-fed (one CTA of 4 warps per (chunk, head)): Q, K, V arrive as [64 x D]
// tiles of 128B-swizzled [64 x 64] atoms.  The off-diagonal blocks of all three sub-chunks run
// as two UMMAs (M = 64, N = 96) against one stacked right operand
//   KL[i] = k_i o e^{G_i - G_r(i)},  QL[i] = q_i o e^{G_i - G_r(i)}   (r(i) = 16 floor(i / 16))
//   KR    = [ k_j o e^{G_16 - G_j}, j < 16 ; k_j o e^{G_32 - G_j}, j < 32 ; k_j o e^{G_48 - G_j}, j < 48 ]
// so row i of KL KR^T holds, in the 16 r(i) columns of its own reference block, the factorised
// A_kk[i][j] of every j < r(i) (all exponents <= 0).  The diagonal blocks stay exact fp32 on the
// CUDA cores.  Then W = T1 (e^G o K), U = T1 V with T1 = T diag(b) (the CTA writes T1 and
// e^G o K swizzled; V is the TMA tile).  Rows past the chunk length hold whatever the TMA box
// covers: b = 0 there (zero columns of T1), and P / Qg / Kd mask them.
template <int D>
struct KdaTcSmem {
  static constexpr int AT = 64 * 128;  // [64 rows x 64 bf16] 128B-swizzled atom
  static constexpr int RT = 96 * 128;  // the stacked right operand's atom: 96 rows
  static constexpr int NA = D / 64;
  uint8_t kg[NA * AT];  // e^G o K (B of W, MN-major): lives through both phases
  union {  // phase 1 (operands of the A_kk / A_qk products) / phase 2 (inverse, W / U operands)
    struct {
      uint8_t q[NA * AT];   // Q, then (in place) QL
      uint8_t k[NA * AT];   // K, then (in place) KL
      uint8_t kr[NA * RT];
      float g[C * D];       // G[r][d]: in-chunk cumulative log decay
    } a;
    struct {
      uint8_t t1[AT];
      uint8_t v[NA * AT];   // TMA-loaded once the phase-1 products have consumed the region
      float l[C][C + 1];
      float x[C][C + 1];
      float scr[4 * 16 * 17];
    } b;
  } u;
  float beta[C];
  uint64_t bar_qk, bar_v, bar_m1, bar_m2;
  uint32_t tmem_base;
};

// byte offset of (r, c) in a tile of 128B-swizzled [rows x 64] atoms of `atom` bytes
__device__ __forceinline__ uint32_t sw_off_a(int r, int c, int atom) {
  const int cc = c & 63;
  return (c >> 6) * atom + r * 128 + ((((cc >> 3) ^ (r & 7)) & 7) << 4) + ((cc & 7) << 1);
}

template <int D>
__global__ void __launch_bounds__(kThreads)
    kda_chunk_intra_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                              const __grid_constant__ CUtensorMap vmap, int v_off, const float* __restrict__ glog,
                              const float* __restrict__ beta, const int32_t* __restrict__ chunks,
                              __nv_bfloat16* __restrict__ ws, float* __restrict__ glast, int H) {
  pdl_launch_dependents();
  using SM = KdaTcSmem<D>;
  constexpr int AT = SM::AT, RT = SM::RT, NA = SM::NA;
  constexpr uint32_t kCols = 256;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = blockIdx.x, h = blockIdx.y;
  if (tid == 0) {
    tc::mbar_init(&sm.bar_qk, 1);
    tc::mbar_init(&sm.bar_v, 1);
    tc::mbar_init(&sm.bar_m1, 1);
    tc::mbar_init(&sm.bar_m2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&sm.tmem_base)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_wait();
  const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_base;
  if (tid == 0) {
    const uint64_t pol = tc::policy_evict_first();
    tc::mbar_expect_tx(&sm.bar_qk, 2 * NA * AT);
    for (int a = 0; a < NA; ++a) {
      tc::tma_load_2d(sm.u.a.q + a * AT, &qmap, h * D + 64 * a, c0, &sm.bar_qk, pol);
      tc::tma_load_2d(sm.u.a.k + a * AT, &kmap, h * D + 64 * a, c0, &sm.bar_qk, pol);
    }
  }
  {  // per-channel log decays (rows past the chunk: 0, so G stays flat there)
    constexpr int IT = C * D / 4 / kThreads;
    float4 gv[IT];
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int idx = tid + u * kThreads;
      const int r = idx / (D / 4), c4 = (idx % (D / 4)) * 4;
      gv[u] = r < len ? *reinterpret_cast<const float4*>(glog + ((size_t)(c0 + r) * H + h) * D + c4)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < IT; ++u) {
      const int idx = tid + u * kThreads;
      *reinterpret_cast<float4*>(&sm.u.a.g[(idx / (D / 4)) * D + (idx % (D / 4)) * 4]) = gv[u];
    }
  }
  if (tid < C) sm.beta[tid] = tid < len ? beta[(size_t)(c0 + tid) * H + h] : 0.f;
  __syncthreads();
  for (int d = tid; d < D; d += kThreads) {  // in-chunk cumulative sum per channel
    float acc = 0.f;
#pragma unroll 8
    for (int r = 0; r < C; ++r) {
      acc += sm.u.a.g[r * D + d];
      sm.u.a.g[r * D + d] = acc;
    }
  }
  __syncthreads();
  tc::mbar_wait(&sm.bar_qk, 0);
  // e^G o K (the B operand of W), 8 columns per step
  for (int idx = tid; idx < C * D / 8; idx += kThreads) {
    const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
    const uint32_t o = sw_off_a(r, c8, AT);
    const uint4 kv = *reinterpret_cast<const uint4*>(sm.u.a.k + o);
    const uint32_t* ka = reinterpret_cast<const uint32_t*>(&kv);
    uint4 go;
    uint32_t* goa = reinterpret_cast<uint32_t*>(&go);
    const float* gr = sm.u.a.g + r * D + c8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
      goa[e] = pack_bf16(kf.x * expf(gr[2 * e]), kf.y * expf(gr[2 * e + 1]));
    }
    *reinterpret_cast<uint4*>(sm.kg + o) = go;
  }
  // the stacked right operand: block s (s = 1, 2, 3) = rows j < 16 s scaled to reference 16 s
  for (int idx = tid; idx < 96 * D / 8; idx += kThreads) {
    const int row = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
    const int s = row < 16 ? 1 : row < 48 ? 2 : 3;
    const int j = row - (s == 1 ? 0 : s == 2 ? 16 : 48), rr = 16 * s;
    const uint4 kv = *reinterpret_cast<const uint4*>(sm.u.a.k + sw_off_a(j, c8, AT));
    const uint32_t* ka = reinterpret_cast<const uint32_t*>(&kv);
    uint4 ko;
    uint32_t* koa = reinterpret_cast<uint32_t*>(&ko);
    const float* gj = sm.u.a.g + j * D + c8;
    const float* g0 = sm.u.a.g + rr * D + c8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
      koa[e] = pack_bf16(kf.x * expf(g0[2 * e] - gj[2 * e]), kf.y * expf(g0[2 * e + 1] - gj[2 * e + 1]));
    }
    *reinterpret_cast<uint4*>(sm.u.a.kr + sw_off_a(row, c8, RT)) = ko;
  }
  __nv_bfloat16* rec = ws + ws_tile<D>(n, h, H);
  __nv_bfloat16* wW = rec;
  __nv_bfloat16* wQg = rec + C * D;
  __nv_bfloat16* wKd = rec + 2 * C * D;
  __nv_bfloat16* wU = rec + 3 * C * D;
  __nv_bfloat16* wP = rec + 4 * C * D;
  // diagonal blocks, exact: pairs (i, j) = (r0 + a, r0 + b), 0 <= b <= a < 16, 136 per warp
  const int r0 = 16 * warp;
  constexpr int kPairs = 136, kPerLane = (kPairs + 31) / 32;
  float dkk[kPerLane], dqk[kPerLane];
  int di[kPerLane], dj[kPerLane];
#pragma unroll
  for (int u = 0; u < kPerLane; ++u) {
    const int p = lane + 32 * u;
    dkk[u] = dqk[u] = 0.f;
    di[u] = dj[u] = -1;
    if (p < kPairs) {
      int a = (int)((sqrtf(8.f * p + 1.f) - 1.f) * 0.5f);
      if ((a + 1) * (a + 2) / 2 <= p) ++a;
      if (a * (a + 1) / 2 > p) --a;
      const int b = p - a * (a + 1) / 2;
      const int i = r0 + a, j = r0 + b;
      di[u] = i;
      dj[u] = j;
      const float* gi = sm.u.a.g + i * D;
      const float* gj = sm.u.a.g + j * D;
      float sk = 0.f, sq = 0.f;
#pragma unroll 4
      for (int d = 0; d < D; d += 2) {
        const float2 ki = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sm.u.a.k + sw_off_a(i, d, AT)));
        const float2 qi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sm.u.a.q + sw_off_a(i, d, AT)));
        const float2 kj = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sm.u.a.k + sw_off_a(j, d, AT)));
        const float e0 = expf(gi[d] - gj[d]) * kj.x, e1 = expf(gi[d + 1] - gj[d + 1]) * kj.y;
        sk += ki.x * e0 + ki.y * e1;
        sq += qi.x * e0 + qi.y * e1;
      }
      dkk[u] = sk;
      dqk[u] = sq;
    }
  }
  // e^G o Q and e^{G_C - G} o K -> workspace (state pass operands); the chunk's last decays
  for (int idx = tid; idx < C * D / 8; idx += kThreads) {
    const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
    const uint32_t o = sw_off_a(r, c8, AT);
    const uint4 qv = *reinterpret_cast<const uint4*>(sm.u.a.q + o);
    const uint4 kv = *reinterpret_cast<const uint4*>(sm.u.a.k + o);
    const uint32_t* qa = reinterpret_cast<const uint32_t*>(&qv);
    const uint32_t* ka = reinterpret_cast<const uint32_t*>(&kv);
    const bool ok = r < len;
    const float* gr = sm.u.a.g + r * D + c8;
    const float* gl = sm.u.a.g + (C - 1) * D + c8;
    uint4 qo, ko;
    uint32_t* qoa = reinterpret_cast<uint32_t*>(&qo);
    uint32_t* koa = reinterpret_cast<uint32_t*>(&ko);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qa[e]));
      const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
      qoa[e] = ok ? pack_bf16(qf.x * expf(gr[2 * e]), qf.y * expf(gr[2 * e + 1])) : 0u;
      koa[e] = ok ? pack_bf16(kf.x * expf(gl[2 * e] - gr[2 * e]), kf.y * expf(gl[2 * e + 1] - gr[2 * e + 1])) : 0u;
    }
    *reinterpret_cast<uint4*>(wQg + r * D + c8) = qo;
    *reinterpret_cast<uint4*>(wKd + r * D + c8) = ko;
  }
  for (int d = tid; d < D; d += kThreads) glast[((size_t)n * H + h) * D + d] = sm.u.a.g[(C - 1) * D + d];
  __syncthreads();  // every raw Q / K read is done: the left operands are built in place
  for (int idx = tid; idx < C * D / 8; idx += kThreads) {  // row i scaled to its sub-chunk reference
    const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8, rr = r & ~15;
    const uint32_t o = sw_off_a(r, c8, AT);
    uint4 qv = *reinterpret_cast<const uint4*>(sm.u.a.q + o);
    uint4 kv = *reinterpret_cast<const uint4*>(sm.u.a.k + o);
    uint32_t* qa = reinterpret_cast<uint32_t*>(&qv);
    uint32_t* ka = reinterpret_cast<uint32_t*>(&kv);
    const float* gr = sm.u.a.g + r * D + c8;
    const float* g0 = sm.u.a.g + rr * D + c8;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 qf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&qa[e]));
      const float2 kf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ka[e]));
      const float e0 = expf(gr[2 * e] - g0[2 * e]), e1 = expf(gr[2 * e + 1] - g0[2 * e + 1]);
      qa[e] = pack_bf16(qf.x * e0, qf.y * e1);
      ka[e] = pack_bf16(kf.x * e0, kf.y * e1);
    }
    *reinterpret_cast<uint4*>(sm.u.a.q + o) = qv;
    *reinterpret_cast<uint4*>(sm.u.a.k + o) = kv;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> the MMA's reads
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {  // KL KR^T -> TMEM [0, 96), QL KR^T -> [96, 192)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t sq = tc::smem_u32(sm.u.a.q), sk = tc::smem_u32(sm.u.a.k), sr = tc::smem_u32(sm.u.a.kr);
    const uint32_t id = tc::idesc_bf16(64, 96);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = (kk >> 2) * AT + (kk & 3) * 32, roff = (kk >> 2) * RT + (kk & 3) * 32;
      tc::umma_w(tmem, tc::desc_sw128(sk + off), tc::desc_sw128(sr + roff), id, kk > 0 ? 1u : 0u);
      tc::umma_w(tmem + 96, tc::desc_sw128(sq + off), tc::desc_sw128(sr + roff), id, kk > 0 ? 1u : 0u);
    }
    tc::commit_w(&sm.bar_m1);
  }
  // L = -b_i A_kk (strictly lower) -> shared memory, P = A_qk (lower incl. diagonal) -> workspace.
  // Warp w reads its own sub-chunk's rows: row 16w + i in TMEM lane 32w + i (i < 16); its
  // reference block's columns start at 0 / 16 / 48 (w = 1 / 2 / 3).
  tc::mbar_wait(&sm.bar_m1, 0);  // the phase-1 products have read QL / KL / KR
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {  // V into the phase-2 region (the inverse overlaps its latency)
    tc::mbar_expect_tx(&sm.bar_v, NA * AT);
    for (int a = 0; a < NA; ++a)
      tc::tma_load_2d(sm.u.b.v + a * AT, &vmap, v_off + h * D + 64 * a, c0, &sm.bar_v, tc::policy_evict_first());
  }
  {
    const int i = 16 * warp + (lane & 15);
    const bool row = lane < 16;
    const int cbase = warp == 1 ? 0 : warp == 2 ? 16 : 48;
    const uint32_t la = tmem + ((uint32_t)(32 * warp) << 16);
    const float bi = sm.beta[i];
#pragma unroll 1
    for (int j0 = 0; j0 < C; j0 += 16) {
      float kk[16], qk[16];
      const bool off = j0 < r0;  // warp-uniform: a block left of the diagonal
      if (off) {
        tc::tmem_ld16_async(la + cbase + j0, kk);
        tc::tmem_ld16_async(la + 96 + cbase + j0, qk);
        tc::tmem_wait_ld();
        tc::reg_fence16(kk);
        tc::reg_fence16(qk);
      }
      if (row) {
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          float pv[2];
#pragma unroll
          for (int d = 0; d < 2; ++d) {
            const int j = j0 + e + d;
            const bool ok = off && i < len && j < len;
            sm.u.b.l[i][j] = ok ? -bi * kk[e + d] : 0.f;
            pv[d] = ok ? qk[e + d] : 0.f;
          }
          pk[e >> 1] = pack_bf16(pv[0], pv[1]);
        }
        *reinterpret_cast<uint4*>(wP + i * C + j0) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(wP + i * C + j0 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kPerLane; ++u) {  // the diagonal blocks over the zeros written above
    const int i = di[u], j = dj[u];
    if (i >= 0) {
      const bool ok = i < len && j < len;
      if (i > j) sm.u.b.l[i][j] = ok ? -sm.beta[i] * dkk[u] : 0.f;
      wP[i * C + j] = __float2bfloat16_rn(ok ? dqk[u] : 0.f);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  invert_unit_lower(sm.u.b.l, sm.u.b.x, sm.u.b.scr);  // x = T = (I - L)^-1 (fp32)
  for (int idx = tid; idx < C * C / 8; idx += kThreads) {  // T1 = T diag(b), swizzled K-major
    const int i = idx >> 3, j8 = (idx & 7) * 8;
    uint32_t p1[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2)
      p1[e >> 1] = pack_bf16(sm.u.b.x[i][j8 + e] * sm.beta[j8 + e], sm.u.b.x[i][j8 + e + 1] * sm.beta[j8 + e + 1]);
    *reinterpret_cast<uint4*>(sm.u.b.t1 + sw_off_a(i, j8, AT)) = make_uint4(p1[0], p1[1], p1[2], p1[3]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {  // W = T1 (e^G o K) -> TMEM [0, D), U = T1 V -> [D, 2D)
    tc::mbar_wait(&sm.bar_v, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t id = tc::idesc_bf16(64, D) | (1u << 16);  // B MN-major
    const uint32_t s1 = tc::smem_u32(sm.u.b.t1), sg = tc::smem_u32(sm.kg), sv = tc::smem_u32(sm.u.b.v);
#pragma unroll
    for (int kk = 0; kk < C / 16; ++kk) {
      tc::umma_w(tmem, tc::desc_sw128(s1 + kk * 32), desc_mn_sw128_c(sg + kk * 2048), id, kk > 0 ? 1u : 0u);
      tc::umma_w(tmem + D, tc::desc_sw128(s1 + kk * 32), desc_mn_sw128_c(sv + kk * 2048), id, kk > 0 ? 1u : 0u);
    }
    tc::commit_w(&sm.bar_m2);
  }
  tc::mbar_wait(&sm.bar_m2, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int i = 16 * warp + (lane & 15);
    const uint32_t la = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll 1
    for (int c = 0; c < D; c += 16) {
      float wv[16], uv[16];
      tc::tmem_ld16_async(la + c, wv);
      tc::tmem_ld16_async(la + D + c, uv);
      tc::tmem_wait_ld();
      tc::reg_fence16(wv);
      tc::reg_fence16(uv);
      if (lane < 16) {
        uint32_t pw[8], pu[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          pw[e] = pack_bf16(wv[2 * e], wv[2 * e + 1]);
          pu[e] = pack_bf16(uv[2 * e], uv[2 * e + 1]);
        }
        *reinterpret_cast<uint4*>(wW + i * D + c) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
        *reinterpret_cast<uint4*>(wW + i * D + c + 8) = make_uint4(pw[4], pw[5], pw[6], pw[7]);
        *reinterpret_cast<uint4*>(wU + i * D + c) = make_uint4(pu[0], pu[1], pu[2], pu[3]);
        *reinterpret_cast<uint4*>(wU + i * D + c + 8) = make_uint4(pu[4], pu[5], pu[6], pu[7]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

template <int D>
static sn_status launch_kda_two_phase(const void* qb, const void* kb, const void* qkv, int v_off, int qkv_stride,
                                      int rows, const float* glog, const float* beta, const int32_t* chunks,
                                      const int32_t* seq_chunk0, int num_chunks, void* ws, float* glast, float* o,
                                      float* state, const int32_t* slot_idx, int num_seqs, int H, int init_state,
                                      cudaStream_t st) {
  const int smem = (int)sizeof(KdaTcSmem<D>) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kda_chunk_intra_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  CUtensorMap qm, km, vm;
  if (!tc::map_2d(&qm, qb, rows, (uint64_t)H * D, (uint64_t)H * D, 64) ||
      !tc::map_2d(&km, kb, rows, (uint64_t)H * D, (uint64_t)H * D, 64) ||
      !tc::map_2d(&vm, qkv, rows, (uint64_t)qkv_stride, (uint64_t)qkv_stride, 64)) {
    set_error("sn_kda_chunk_prefill2: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  cudaError_t e = launch_pdl(kda_chunk_intra_tc_kernel<D>, dim3(num_chunks, H), dim3(kThreads), (size_t)smem, st, qm,
                             km, vm, v_off, glog, beta, chunks, (__nv_bfloat16*)ws, glast, H);
  if (e != cudaSuccess) {
    set_error("sn_kda_chunk_prefill2(intra) launch: %s", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  sn_status s = check_launch("sn_kda_chunk_prefill(intra)");
  if (s != SN_OK) return s;
  launch_state_pass<D, true>((const __nv_bfloat16*)ws, glast, chunks, seq_chunk0, o, state, slot_idx, num_seqs, H,
                             init_state, st);
  return check_launch("sn_kda_chunk_prefill(state)");
}

}  // namespace chunk
}  // namespace sn

using namespace sn;

extern "C" {

size_t sn_kda_chunk_workspace_bytes(int num_chunks, int H, int D) {
  return (size_t)num_chunks * H * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2 +
         (size_t)num_chunks * H * D * sizeof(float);
}

sn_status sn_kda_chunk_prefill2(const void* qn, const void* kn, const void* qkv_conv, int v_off, int qkv_stride,
                                int rows, const float* glog, const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace, float* o, float* state,
                                const int32_t* slot_idx, int num_seqs, int H, int D, int init_state, int dtype,
                                void* stream) {
  SN_REQUIRE(qn && kn && qkv_conv && glog && beta && chunks && seq_chunk0 && workspace && o && state,
             "sn_kda_chunk_prefill2: NULL pointer");
  SN_REQUIRE(num_seqs > 0 && num_chunks > 0 && H > 0 && rows > 0, "sn_kda_chunk_prefill2: bad shape");
  SN_REQUIRE(D == 64 || D == 128, "sn_kda_chunk_prefill2: D=%d unsupported", D);
  SN_REQUIRE(dtype == SN_BF16, "sn_kda_chunk_prefill2: bf16 only");
  SN_REQUIRE(((uintptr_t)qn % 16) == 0 && ((uintptr_t)kn % 16) == 0 && ((uintptr_t)qkv_conv % 16) == 0 &&
                 (qkv_stride * 2) % 16 == 0 && (v_off % 64) == 0,
             "sn_kda_chunk_prefill2: TMA operands must be 16-byte aligned (v_off a multiple of 64)");
  cudaStream_t st = (cudaStream_t)stream;
  float* glast = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                          (size_t)num_chunks * H * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2);
  if (D == 128)
    return chunk::launch_kda_two_phase<128>(qn, kn, qkv_conv, v_off, qkv_stride, rows, glog, beta, chunks,
                                                            seq_chunk0, num_chunks, workspace, glast, o, state,
                                                            slot_idx, num_seqs, H, init_state, st);
  return chunk::launch_kda_two_phase<64>(qn, kn, qkv_conv, v_off, qkv_stride, rows, glog, beta, chunks,
                                                         seq_chunk0, num_chunks, workspace, glast, o, state, slot_idx,
                                                         num_seqs, H, init_state, st);
}

size_t sn_gdn_chunk_workspace_bytes(int num_chunks, int Hv, int D) {
  return (size_t)num_chunks * Hv * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2 +
         (size_t)num_chunks * Hv * sizeof(float);
}

sn_status sn_gdn_chunk_prefill2(const void* qn, const void* kn, const void* qkv_conv, int v_off, int qkv_stride,
                                int rows, const float* glog, const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace, float* o, float* state,
                                const int32_t* slot_idx, int num_seqs, int Hk, int Hv, int D, int init_state,
                                int dtype, void* stream) {
  SN_REQUIRE(qn && kn && qkv_conv && glog && beta && chunks && seq_chunk0 && workspace && o && state,
             "sn_gdn_chunk_prefill2: NULL pointer");
  SN_REQUIRE(num_seqs > 0 && num_chunks > 0 && Hk > 0 && Hv % Hk == 0 && rows > 0, "sn_gdn_chunk_prefill2: bad shape");
  SN_REQUIRE(D == 64 || D == 128, "sn_gdn_chunk_prefill2: D=%d unsupported", D);
  SN_REQUIRE(dtype == SN_BF16, "sn_gdn_chunk_prefill2: bf16 only");
  SN_REQUIRE(((uintptr_t)qn % 16) == 0 && ((uintptr_t)kn % 16) == 0 && ((uintptr_t)qkv_conv % 16) == 0 &&
                 (qkv_stride * 2) % 16 == 0 && (v_off % 64) == 0,
             "sn_gdn_chunk_prefill2: TMA operands must be 16-byte aligned (v_off a multiple of 64)");
  cudaStream_t st = (cudaStream_t)stream;
  float* glast = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                          (size_t)num_chunks * Hv * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2);
  if (D == 128)
    return chunk::launch_two_phase<128>(qn, kn, qkv_conv, v_off, qkv_stride, rows, glog, beta, chunks, seq_chunk0,
                                        num_chunks, workspace, glast, o, state, slot_idx, num_seqs, Hk, Hv,
                                        init_state, st);
  return chunk::launch_two_phase<64>(qn, kn, qkv_conv, v_off, qkv_stride, rows, glog, beta, chunks, seq_chunk0,
                                     num_chunks, workspace, glast, o, state, slot_idx, num_seqs, Hk, Hv, init_state,
                                     st);
}

}  // extern "C"
