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


// Chunk-tile loaders with the global loads batched ahead of their conversions (one
// dependent memory round trip per batch instead of one per element: the loops were the
// top long-scoreboard stall of the intra kernels).
// b o V tile [64][D] (bf16, row stride LDK) from the conv output rows c0.. (rows >= len zero).
template <typename T, int D>
__device__ __forceinline__ void load_vb_tile(const T* __restrict__ qkv, int qkv_stride, int v_off, int h, int c0,
                                             int len, const float* beta_s, __nv_bfloat16* dst, int ldk) {
  constexpr int IT = C * D / 8 / kThreads, BATCH = IT < 4 ? IT : 4;
#pragma unroll
  for (int i0 = 0; i0 < IT; i0 += BATCH) {
    float v[BATCH][8];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int idx = threadIdx.x + (i0 + u) * kThreads;
      const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
      if (r < len) load8<T>(qkv + (size_t)(c0 + r) * qkv_stride + v_off + h * D + c8, v[u]);
      else
#pragma unroll
        for (int e = 0; e < 8; ++e) v[u][e] = 0.f;
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int idx = threadIdx.x + (i0 + u) * kThreads;
      const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
      const float b = beta_s[r];
      uint4 pk;
      pk.x = pack_bf16(v[u][0] * b, v[u][1] * b);
      pk.y = pack_bf16(v[u][2] * b, v[u][3] * b);
      pk.z = pack_bf16(v[u][4] * b, v[u][5] * b);
      pk.w = pack_bf16(v[u][6] * b, v[u][7] * b);
      *reinterpret_cast<uint4*>(dst + r * ldk + c8) = pk;
    }
  }
}

// fp32 [rows][heads][D] row slices (head hh, rows c0.. < len, else zero) -> bf16 tile [64][D]
// (row stride ldk); NSRC tensors loaded together.
template <int D, int NSRC>
__device__ __forceinline__ void load_f32_tiles(const float* const* src, int heads, int hh, int c0, int len,
                                               __nv_bfloat16* const* dst, int ldk) {
  constexpr int IT = C * D / 4 / kThreads, BATCH = IT < 4 ? IT : 4;
#pragma unroll
  for (int i0 = 0; i0 < IT; i0 += BATCH) {
    float4 v[NSRC][BATCH];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int idx = threadIdx.x + (i0 + u) * kThreads;
      const int r = idx / (D / 4), c4 = (idx % (D / 4)) * 4;
#pragma unroll
      for (int t = 0; t < NSRC; ++t)
        v[t][u] = r < len ? *reinterpret_cast<const float4*>(src[t] + ((size_t)(c0 + r) * heads + hh) * D + c4)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      const int idx = threadIdx.x + (i0 + u) * kThreads;
      const int r = idx / (D / 4), c4 = (idx % (D / 4)) * 4;
#pragma unroll
      for (int t = 0; t < NSRC; ++t)
        *reinterpret_cast<uint2*>(dst[t] + r * ldk + c4) =
            make_uint2(pack_bf16(v[t][u].x, v[t][u].y), pack_bf16(v[t][u].z, v[t][u].w));
    }
  }
}

// =====================================================================================
// Two-phase version (the long-prefill path): the chunk-local work (inverse, W, U, P and
// the decayed operands) of all chunks runs in parallel, one CTA per (chunk, value head);
// the sequential state pass then only streams the precomputed tiles through
// double-buffered shared memory and runs the four state-dependent tile products.
// Workspace per (chunk, head), bf16: W, Qg, Kd, U [64][D] and P [64][64]; glast fp32.

template <int D>
struct IntraSmem {  // ~74 KB at D = 128: three CTAs per SM
  static constexpr int LDK = D + 8, LDC = C + 8;
  union {
    __nv_bfloat16 q[C * LDK];   // Q until e^G o Q is written out
    float x[C][C + 1];          // then the fp32 inverse
    __nv_bfloat16 vb[C * LDK];  // then b o V
  } qv;
  __nv_bfloat16 k[C * LDK];
  __nv_bfloat16 kb[C * LDK];
  union {
    float l[C][C + 1];            // L until inverted
    __nv_bfloat16 t[C * LDC];     // then T (bf16 operand)
  } lt;
  float scr[4 * 16 * 17];
  float g[C], beta[C];
};

template <int D>
__device__ __forceinline__ size_t ws_tile(int n, int h, int Hv) {  // offset of one (chunk, head) record
  return ((size_t)n * Hv + h) * (4 * (size_t)C * D + (size_t)C * C);
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads)
    gdn_chunk_intra_kernel(const float* __restrict__ qn, const float* __restrict__ kn, const T* __restrict__ qkv,
                           int v_off, int qkv_stride, const float* __restrict__ glog, const float* __restrict__ beta,
                           const int32_t* __restrict__ chunks, __nv_bfloat16* __restrict__ ws,
                           float* __restrict__ glast, int Hk, int Hv) {
  pdl_launch_dependents();
  using SM = IntraSmem<D>;
  constexpr int LDK = SM::LDK, LDC = SM::LDC;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int n = blockIdx.x, h = blockIdx.y;
  const int G = Hv / Hk, kh = h / G;
  const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
  {
    const float* src[2] = {qn, kn};
    __nv_bfloat16* dst[2] = {sm.qv.q, sm.k};
    load_f32_tiles<D, 2>(src, Hk, kh, c0, len, dst, LDK);
  }
  if (tid < C) {
    sm.g[tid] = tid < len ? glog[(size_t)(c0 + tid) * Hv + h] : 0.f;
    sm.beta[tid] = tid < len ? beta[(size_t)(c0 + tid) * Hv + h] : 0.f;
  }
  __syncthreads();
  if (warp == 0) {
    float a0 = sm.g[lane], a1 = sm.g[32 + lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float n0 = __shfl_up_sync(0xffffffffu, a0, o), n1 = __shfl_up_sync(0xffffffffu, a1, o);
      if (lane >= o) { a0 += n0; a1 += n1; }
    }
    a1 += __shfl_sync(0xffffffffu, a0, 31);
    sm.g[lane] = a0;
    sm.g[32 + lane] = a1;
  }
  __syncthreads();
  __nv_bfloat16* rec = ws + ws_tile<D>(n, h, Hv);
  __nv_bfloat16* wW = rec;
  __nv_bfloat16* wQg = rec + C * D;
  __nv_bfloat16* wKd = rec + 2 * C * D;
  __nv_bfloat16* wU = rec + 3 * C * D;
  __nv_bfloat16* wP = rec + 4 * C * D;
  // K K^T -> L, Q K^T -> P (straight to the workspace)
  {
    float kk[8][4], qk[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) kk[nt][e] = qk[nt][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < D; ks += 16) {
      uint32_t ak[4], aq[4];
      lda(sm.k, LDK, warp * 16, ks, ak);
      lda(sm.qv.q, LDK, warp * 16, ks, aq);
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldb_nk(sm.k, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(kk[nt], ak, b0, b1);
        mma_bf16(kk[nt + 1], ak, b2, b3);
        mma_bf16(qk[nt], aq, b0, b1);
        mma_bf16(qk[nt + 1], aq, b2, b3);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        const int i = warp * 16 + g4 + ((e >> 1) << 3), j = nt * 8 + t4 * 2;
        float pv[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
          const float gam = i >= j + d ? expf(sm.g[i] - sm.g[j + d]) : 0.f;
          sm.lt.l[i][j + d] = i > j + d ? -sm.beta[i] * kk[nt][e + d] * gam : 0.f;
          pv[d] = qk[nt][e + d] * gam;
        }
        *reinterpret_cast<uint32_t*>(wP + i * C + j) = pack_bf16(pv[0], pv[1]);
      }
  }
  {
    const float gl = sm.g[C - 1];
    for (int idx = tid; idx < C * D / 2; idx += kThreads) {
      const int r = idx / (D / 2), cc = (idx % (D / 2)) * 2;
      const float eg = expf(sm.g[r]), ed = expf(gl - sm.g[r]);
      const float2 kv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[r * LDK + cc]));
      const float2 qv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.qv.q[r * LDK + cc]));
      *reinterpret_cast<uint32_t*>(&sm.kb[r * LDK + cc]) = pack_bf16(kv.x * sm.beta[r] * eg, kv.y * sm.beta[r] * eg);
      *reinterpret_cast<uint32_t*>(wKd + r * D + cc) = pack_bf16(kv.x * ed, kv.y * ed);
      *reinterpret_cast<uint32_t*>(wQg + r * D + cc) = pack_bf16(qv.x * eg, qv.y * eg);
    }
    if (tid == 0) glast[(size_t)n * Hv + h] = gl;
  }
  __syncthreads();
  // T = (I - L)^{-1}: 16x16 diagonal blocks, then the block rows below them.  Q is dead
  // (e^G o Q went out): its tile holds the fp32 inverse, then b o V (the shared memory fits
  // three CTAs per SM instead of two; the V loads no longer overlap the inverse, the other
  // CTAs on the SM cover that latency)
  invert_unit_lower(sm.lt.l, sm.qv.x, sm.scr);
  for (int idx = tid; idx < C * C; idx += kThreads) {
    const int i = idx / C, j = idx % C;
    sm.lt.t[i * LDC + j] = __float2bfloat16_rn(sm.qv.x[i][j]);
  }
  __syncthreads();
  load_vb_tile<T, D>(qkv, qkv_stride, v_off, h, c0, len, sm.beta, sm.qv.vb, LDK);
  __syncthreads();
  // W = T Kb, U = T Vb  (both [64][D]) -> workspace
  {
    float wacc[D / 8][4], uacc[D / 8][4];
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) wacc[nt][e] = uacc[nt][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < C; ks += 16) {
      uint32_t a[4];
      lda(sm.lt.t, LDC, warp * 16, ks, a);
#pragma unroll
      for (int nt = 0; nt < D / 8; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldb_kn(sm.kb, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(wacc[nt], a, b0, b1);
        mma_bf16(wacc[nt + 1], a, b2, b3);
        ldb_kn(sm.qv.vb, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(uacc[nt], a, b0, b1);
        mma_bf16(uacc[nt + 1], a, b2, b3);
      }
    }
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        const int r = warp * 16 + g4 + ((e >> 1) << 3), cc = nt * 8 + t4 * 2;
        *reinterpret_cast<uint32_t*>(wW + r * D + cc) = pack_bf16(wacc[nt][e], wacc[nt][e + 1]);
        *reinterpret_cast<uint32_t*>(wU + r * D + cc) = pack_bf16(uacc[nt][e], uacc[nt][e + 1]);
      }
  }
}

template <int D, int VTT = VT>
struct StateSmem {
  static constexpr int LDK = D + 8, LDV = VTT + 8, LDC = C + 8;
  struct Stage {
    __nv_bfloat16 w[C * LDK];
    __nv_bfloat16 qg[C * LDK];
    __nv_bfloat16 kd[C * LDK];
    __nv_bfloat16 u[C * LDV];
    __nv_bfloat16 p[C * LDC];
  } st[2];
  __nv_bfloat16 s[D * LDV];
  __nv_bfloat16 vp[C * LDV];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// PERCH (KDA): glast holds the chunk's per-key-channel cumulative log decay [D] per (chunk,
// head) and S is decayed row-wise, diag(e^{G_C}) S; otherwise one scalar per (chunk, head).
template <int D, bool PERCH = false, int VTT = VT>
__global__ void __launch_bounds__(kThreads, 1)
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
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int vt = blockIdx.x, h = blockIdx.y, seq = blockIdx.z;
  const int slot = slot_idx ? slot_idx[seq] : seq;
  const int n0 = seq_chunk0[seq], n1 = seq_chunk0[seq + 1];
  float* Sg = state + ((size_t)slot * Hv + h) * D * D;
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
  auto load_stage = [&](int n, int b) {
    const __nv_bfloat16* rec = ws + ws_tile<D>(n, h, Hv);
    typename SM::Stage& S = sm.st[b];
    for (int idx = tid; idx < C * D / 8; idx += kThreads) {  // W, Qg, Kd rows of D
      const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
      cp_async16(&S.w[r * LDK + c8], rec + r * D + c8);
      cp_async16(&S.qg[r * LDK + c8], rec + C * D + r * D + c8);
      cp_async16(&S.kd[r * LDK + c8], rec + 2 * C * D + r * D + c8);
    }
    for (int idx = tid; idx < C * VTT / 8; idx += kThreads) {  // U tile (this CTA's value columns)
      const int r = idx / (VTT / 8), c8 = (idx % (VTT / 8)) * 8;
      cp_async16(&S.u[r * LDV + c8], rec + 3 * C * D + r * D + vt * VTT + c8);
    }
    for (int idx = tid; idx < C * C / 8; idx += kThreads) {  // P
      const int r = idx / (C / 8), c8 = (idx % (C / 8)) * 8;
      cp_async16(&S.p[r * LDC + c8], rec + 4 * C * D + r * C + c8);
    }
    cp_async_commit();
  };
  if (n0 < n1) load_stage(n0, 0);
  for (int n = n0; n < n1; ++n) {
    const int b = (n - n0) & 1;
    if (n + 1 < n1) {
      load_stage(n + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    // S -> bf16 operand
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const int kr = (warp * MT + mt) * 16 + g4 + ((e >> 1) << 3);
          *reinterpret_cast<uint32_t*>(&sm.s[kr * LDV + nt * 8 + t4 * 2]) = pack_bf16(sf[mt][nt][e], sf[mt][nt][e + 1]);
        }
    __syncthreads();
    typename SM::Stage& St = sm.st[b];
    const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
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
        ldb_kn(sm.s, LDV, nt * 8, ks, b0, b1, b2, b3);
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
        *reinterpret_cast<uint32_t*>(&sm.vp[r * LDV + nt * 8 + t4 * 2]) = pack_bf16(vpc[nt][e], vpc[nt][e + 1]);
      }
    __syncthreads();
    // O = Qg S + P V'
    {
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
          ldb_kn(sm.s, LDV, nt * 8, ks, b0, b1, b2, b3);
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
          ldb_kn(sm.vp, LDV, nt * 8, ks, b0, b1, b2, b3);
          mma_bf16(oc[nt], a, b0, b1);
          mma_bf16(oc[nt + 1], a, b2, b3);
        }
      }
#pragma unroll
      for (int nt = 0; nt < NTV; ++nt)
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const int r = warp * 16 + g4 + ((e >> 1) << 3), cc = vt * VTT + nt * 8 + t4 * 2;
          if (r < len)
            *reinterpret_cast<float2*>(o + ((size_t)(c0 + r) * Hv + h) * D + cc) = make_float2(oc[nt][e], oc[nt][e + 1]);
        }
    }
    // S = e^{G_C} S + Kd^T V'   (KDA: diag(e^{G_C}) S, one factor per key row)
    {
      if (PERCH) {
        const float* gl = glast + ((size_t)n * Hv + h) * D;
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
        const float dec = expf(glast[(size_t)n * Hv + h]);
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
            ldb_kn(sm.vp, LDV, nt * 8, ks, b0, b1, b2, b3);
            mma_bf16(sf[mt][nt], a, b0, b1);
            mma_bf16(sf[mt][nt + 1], a, b2, b3);
          }
        }
      }
    }
    __syncthreads();
  }
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
    gdn_chunk_state_kernel<D, PERCH, 64><<<dim3(D / 64, H, num_seqs), kThreads, sizeof(StateSmem<D, 64>), st>>>(
        ws, glast, chunks, seq_chunk0, o, state, slot_idx, H, init_state);
  else
    gdn_chunk_state_kernel<D, PERCH, 32><<<dim3(D / 32, H, num_seqs), kThreads, sizeof(StateSmem<D, 32>), st>>>(
        ws, glast, chunks, seq_chunk0, o, state, slot_idx, H, init_state);
}

template <typename T, int D>
static sn_status launch_two_phase(const float* qn, const float* kn, const void* qkv, int v_off, int qkv_stride,
                                  const float* glog, const float* beta, const int32_t* chunks,
                                  const int32_t* seq_chunk0, int num_chunks, void* ws, float* glast, float* o,
                                  float* state, const int32_t* slot_idx, int num_seqs, int Hk, int Hv,
                                  int init_state, cudaStream_t st) {
  const int smem_a = (int)sizeof(IntraSmem<D>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gdn_chunk_intra_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a);
    attr = true;
  }
  gdn_chunk_intra_kernel<T, D><<<dim3(num_chunks, Hv), kThreads, smem_a, st>>>(
      qn, kn, (const T*)qkv, v_off, qkv_stride, glog, beta, chunks, (__nv_bfloat16*)ws, glast, Hk, Hv);
  sn_status e = check_launch("sn_gdn_chunk_prefill(intra)");
  if (e != SN_OK) return e;
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
// — the left operand is the warp's own 16 rows, the right operand (the 16w rows j < r of K
// scaled to reference r) a per-warp shared-memory tile, both products on mma.sync.  The
// diagonal 16x16 block (r <= j <= i) is computed exactly in fp32 with e^{G_i - G_j} <= 1
// per term (a factorised form would need e^{G_r - G_j} > 1, which overflows for strong
// gates).

template <int D>
struct KdaIntraSmem {
  static constexpr int LDK = D + 8, LDC = C + 8;
  static constexpr int KR_ROWS = 16 * (0 + 1 + 2 + 3);  // per-warp right operands (rows j < 16w)
  __nv_bfloat16 q[C * LDK];
  __nv_bfloat16 k[C * LDK];
  union {
    struct { __nv_bfloat16 ql[C * LDK]; __nv_bfloat16 kl[C * LDK]; } a;  // A step: left operands
    struct { __nv_bfloat16 kb[C * LDK]; __nv_bfloat16 vb[C * LDK]; } w;  // W/U step
  } u1;
  union {
    __nv_bfloat16 kr[KR_ROWS * LDK];
    struct { float l[C][C + 1]; float x[C][C + 1]; } lx;
  } u2;
  __nv_bfloat16 t[C * LDC];
  float scr[4 * 16 * 17];
  float g[C * D];  // G[r][d]: cumulative log decay
  float beta[C];
};

template <typename T, int D>
__global__ void __launch_bounds__(kThreads)
    kda_chunk_intra_kernel(const float* __restrict__ qn, const float* __restrict__ kn, const T* __restrict__ qkv,
                           int v_off, int qkv_stride, const float* __restrict__ glog, const float* __restrict__ beta,
                           const int32_t* __restrict__ chunks, __nv_bfloat16* __restrict__ ws,
                           float* __restrict__ glast, int H) {
  pdl_launch_dependents();
  using SM = KdaIntraSmem<D>;
  constexpr int LDK = SM::LDK, LDC = SM::LDC;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int n = blockIdx.x, h = blockIdx.y;
  const int c0 = chunks[2 * n], len = chunks[2 * n + 1];
  {
    const float* src[2] = {qn, kn};
    __nv_bfloat16* dst[2] = {sm.q, sm.k};
    load_f32_tiles<D, 2>(src, H, h, c0, len, dst, LDK);
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
      *reinterpret_cast<float4*>(&sm.g[(idx / (D / 4)) * D + (idx % (D / 4)) * 4]) = gv[u];
    }
  }
  if (tid < C) sm.beta[tid] = tid < len ? beta[(size_t)(c0 + tid) * H + h] : 0.f;
  __syncthreads();
  for (int d = tid; d < D; d += kThreads) {  // per-channel prefix sum over the chunk
    float acc = 0.f;
#pragma unroll 8
    for (int r = 0; r < C; ++r) {
      acc += sm.g[r * D + d];
      sm.g[r * D + d] = acc;
    }
  }
  __syncthreads();
  // ---- per-warp operands around reference row r0 = 16 * warp (off-diagonal blocks j < r0)
  const int r0 = 16 * warp, nrows = 16 * warp;
  __nv_bfloat16* kr = sm.u2.kr + 16 * (warp * (warp - 1) / 2) * LDK;
  for (int idx = lane; idx < 16 * D / 2; idx += 32) {
    const int r = r0 + idx / (D / 2), cc = (idx % (D / 2)) * 2;
    const float e0 = expf(sm.g[r * D + cc] - sm.g[r0 * D + cc]), e1 = expf(sm.g[r * D + cc + 1] - sm.g[r0 * D + cc + 1]);
    const float2 qv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.q[r * LDK + cc]));
    const float2 kv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[r * LDK + cc]));
    *reinterpret_cast<uint32_t*>(&sm.u1.a.ql[r * LDK + cc]) = pack_bf16(qv.x * e0, qv.y * e1);
    *reinterpret_cast<uint32_t*>(&sm.u1.a.kl[r * LDK + cc]) = pack_bf16(kv.x * e0, kv.y * e1);
  }
  for (int idx = lane; idx < nrows * D / 2; idx += 32) {
    const int j = idx / (D / 2), cc = (idx % (D / 2)) * 2;
    const float e0 = expf(sm.g[r0 * D + cc] - sm.g[j * D + cc]), e1 = expf(sm.g[r0 * D + cc + 1] - sm.g[j * D + cc + 1]);
    const float2 kv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[j * LDK + cc]));
    *reinterpret_cast<uint32_t*>(&kr[j * LDK + cc]) = pack_bf16(kv.x * e0, kv.y * e1);
  }
  __syncwarp();
  float kk[8][4], qk[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) kk[nt][e] = qk[nt][e] = 0.f;
#pragma unroll
  for (int ks = 0; ks < D; ks += 16) {
    uint32_t ak[4], aq[4];
    lda(sm.u1.a.kl, LDK, r0, ks, ak);
    lda(sm.u1.a.ql, LDK, r0, ks, aq);
#pragma unroll
    for (int nt = 0; nt < 8; nt += 2) {
      if (nt * 8 < nrows) {  // warp-uniform: only the column blocks left of the diagonal block
        uint32_t b0, b1, b2, b3;
        ldb_nk(kr, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(kk[nt], ak, b0, b1);
        mma_bf16(kk[nt + 1], ak, b2, b3);
        mma_bf16(qk[nt], aq, b0, b1);
        mma_bf16(qk[nt + 1], aq, b2, b3);
      }
    }
  }
  // diagonal block, exact: pairs (i, j) = (r0 + a, r0 + b), 0 <= b <= a < 16, 136 per warp
  constexpr int kPairs = 136, kPerLane = (kPairs + 31) / 32;
  float dkk[kPerLane], dqk[kPerLane];
#pragma unroll
  for (int u = 0; u < kPerLane; ++u) {
    const int p = lane + 32 * u;
    dkk[u] = dqk[u] = 0.f;
    if (p < kPairs) {
      int a = (int)((sqrtf(8.f * p + 1.f) - 1.f) * 0.5f);
      if ((a + 1) * (a + 2) / 2 <= p) ++a;
      if (a * (a + 1) / 2 > p) --a;
      const int b = p - a * (a + 1) / 2;
      const int i = r0 + a, j = r0 + b;
      const float* gi = sm.g + i * D;
      const float* gj = sm.g + j * D;
      float sk = 0.f, sq = 0.f;
#pragma unroll 4
      for (int d = 0; d < D; d += 2) {
        const float2 ki = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[i * LDK + d]));
        const float2 qi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.q[i * LDK + d]));
        const float2 kj = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[j * LDK + d]));
        const float e0 = expf(gi[d] - gj[d]) * kj.x, e1 = expf(gi[d + 1] - gj[d + 1]) * kj.y;
        sk += ki.x * e0 + ki.y * e1;
        sq += qi.x * e0 + qi.y * e1;
      }
      dkk[u] = sk;
      dqk[u] = sq;
    }
  }
  __syncthreads();  // every warp is done with kr before l / x (aliased) are written
  __nv_bfloat16* rec = ws + ws_tile<D>(n, h, H);
  __nv_bfloat16* wW = rec;
  __nv_bfloat16* wQg = rec + C * D;
  __nv_bfloat16* wKd = rec + 2 * C * D;
  __nv_bfloat16* wU = rec + 3 * C * D;
  __nv_bfloat16* wP = rec + 4 * C * D;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; e += 2) {
      const int i = r0 + g4 + ((e >> 1) << 3), j = nt * 8 + t4 * 2;
      float pv[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const bool in = j + d < nrows;
        sm.u2.lx.l[i][j + d] = in && i > j + d ? -sm.beta[i] * kk[nt][e + d] : 0.f;
        pv[d] = in && i >= j + d ? qk[nt][e + d] : 0.f;
      }
      *reinterpret_cast<uint32_t*>(wP + i * C + j) = pack_bf16(pv[0], pv[1]);
    }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kPerLane; ++u) {
    const int p = lane + 32 * u;
    if (p < kPairs) {
      int a = (int)((sqrtf(8.f * p + 1.f) - 1.f) * 0.5f);
      if ((a + 1) * (a + 2) / 2 <= p) ++a;
      if (a * (a + 1) / 2 > p) --a;
      const int b = p - a * (a + 1) / 2;
      const int i = r0 + a, j = r0 + b;
      if (a > b) sm.u2.lx.l[i][j] = -sm.beta[i] * dkk[u];
      wP[i * C + j] = __float2bfloat16_rn(dqk[u]);
    }
  }
  // chunk-global operands: b e^G K, b V (W/U step), e^G Q and e^{G_C - G} K (state pass)
  for (int idx = tid; idx < C * D / 2; idx += kThreads) {
    const int r = idx / (D / 2), cc = (idx % (D / 2)) * 2;
    const float g0 = sm.g[r * D + cc], g1 = sm.g[r * D + cc + 1];
    const float gl0 = sm.g[(C - 1) * D + cc], gl1 = sm.g[(C - 1) * D + cc + 1];
    const float2 kv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.k[r * LDK + cc]));
    const float2 qv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sm.q[r * LDK + cc]));
    const float b = sm.beta[r];
    *reinterpret_cast<uint32_t*>(&sm.u1.w.kb[r * LDK + cc]) = pack_bf16(kv.x * b * expf(g0), kv.y * b * expf(g1));
    *reinterpret_cast<uint32_t*>(wKd + r * D + cc) = pack_bf16(kv.x * expf(gl0 - g0), kv.y * expf(gl1 - g1));
    *reinterpret_cast<uint32_t*>(wQg + r * D + cc) = pack_bf16(qv.x * expf(g0), qv.y * expf(g1));
  }
  load_vb_tile<T, D>(qkv, qkv_stride, v_off, h, c0, len, sm.beta, sm.u1.w.vb, LDK);
  for (int d = tid; d < D; d += kThreads) glast[((size_t)n * H + h) * D + d] = sm.g[(C - 1) * D + d];
  __syncthreads();
  // T = (I - L)^{-1}
  invert_unit_lower(sm.u2.lx.l, sm.u2.lx.x, sm.scr);
  for (int idx = tid; idx < C * C; idx += kThreads) {
    const int i = idx / C, j = idx % C;
    sm.t[i * LDC + j] = __float2bfloat16_rn(sm.u2.lx.x[i][j]);
  }
  __syncthreads();
  // W = T Kb, U = T Vb -> workspace
  {
    float wacc[D / 8][4], uacc[D / 8][4];
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) wacc[nt][e] = uacc[nt][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < C; ks += 16) {
      uint32_t a[4];
      lda(sm.t, LDC, warp * 16, ks, a);
#pragma unroll
      for (int nt = 0; nt < D / 8; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldb_kn(sm.u1.w.kb, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(wacc[nt], a, b0, b1);
        mma_bf16(wacc[nt + 1], a, b2, b3);
        ldb_kn(sm.u1.w.vb, LDK, nt * 8, ks, b0, b1, b2, b3);
        mma_bf16(uacc[nt], a, b0, b1);
        mma_bf16(uacc[nt + 1], a, b2, b3);
      }
    }
#pragma unroll
    for (int nt = 0; nt < D / 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        const int r = warp * 16 + g4 + ((e >> 1) << 3), cc = nt * 8 + t4 * 2;
        *reinterpret_cast<uint32_t*>(wW + r * D + cc) = pack_bf16(wacc[nt][e], wacc[nt][e + 1]);
        *reinterpret_cast<uint32_t*>(wU + r * D + cc) = pack_bf16(uacc[nt][e], uacc[nt][e + 1]);
      }
  }
}

template <typename T, int D>
static sn_status launch_kda_two_phase(const float* qn, const float* kn, const void* qkv, int v_off, int qkv_stride,
                                      const float* glog, const float* beta, const int32_t* chunks,
                                      const int32_t* seq_chunk0, int num_chunks, void* ws, float* glast, float* o,
                                      float* state, const int32_t* slot_idx, int num_seqs, int H, int init_state,
                                      cudaStream_t st) {
  const int smem_a = (int)sizeof(KdaIntraSmem<D>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kda_chunk_intra_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_a);
    attr = true;
  }
  kda_chunk_intra_kernel<T, D><<<dim3(num_chunks, H), kThreads, smem_a, st>>>(
      qn, kn, (const T*)qkv, v_off, qkv_stride, glog, beta, chunks, (__nv_bfloat16*)ws, glast, H);
  sn_status e = check_launch("sn_kda_chunk_prefill(intra)");
  if (e != SN_OK) return e;
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

sn_status sn_kda_chunk_prefill2(const float* qn, const float* kn, const void* qkv_conv, int v_off, int qkv_stride,
                                const float* glog, const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace, float* o, float* state,
                                const int32_t* slot_idx, int num_seqs, int H, int D, int init_state, int dtype,
                                void* stream) {
  SN_REQUIRE(qn && kn && qkv_conv && glog && beta && chunks && seq_chunk0 && workspace && o && state,
             "sn_kda_chunk_prefill2: NULL pointer");
  SN_REQUIRE(num_seqs > 0 && num_chunks > 0 && H > 0, "sn_kda_chunk_prefill2: bad shape");
  SN_REQUIRE(D == 64 || D == 128, "sn_kda_chunk_prefill2: D=%d unsupported", D);
  SN_REQUIRE(dtype == SN_BF16, "sn_kda_chunk_prefill2: bf16 only");
  cudaStream_t st = (cudaStream_t)stream;
  float* glast = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                          (size_t)num_chunks * H * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2);
  if (D == 128)
    return chunk::launch_kda_two_phase<__nv_bfloat16, 128>(qn, kn, qkv_conv, v_off, qkv_stride, glog, beta, chunks,
                                                            seq_chunk0, num_chunks, workspace, glast, o, state,
                                                            slot_idx, num_seqs, H, init_state, st);
  return chunk::launch_kda_two_phase<__nv_bfloat16, 64>(qn, kn, qkv_conv, v_off, qkv_stride, glog, beta, chunks,
                                                         seq_chunk0, num_chunks, workspace, glast, o, state, slot_idx,
                                                         num_seqs, H, init_state, st);
}

size_t sn_gdn_chunk_workspace_bytes(int num_chunks, int Hv, int D) {
  return (size_t)num_chunks * Hv * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2 +
         (size_t)num_chunks * Hv * sizeof(float);
}

sn_status sn_gdn_chunk_prefill2(const float* qn, const float* kn, const void* qkv_conv, int v_off, int qkv_stride,
                                const float* glog, const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace, float* o, float* state,
                                const int32_t* slot_idx, int num_seqs, int Hk, int Hv, int D, int init_state,
                                int dtype, void* stream) {
  SN_REQUIRE(qn && kn && qkv_conv && glog && beta && chunks && seq_chunk0 && workspace && o && state,
             "sn_gdn_chunk_prefill2: NULL pointer");
  SN_REQUIRE(num_seqs > 0 && num_chunks > 0 && Hk > 0 && Hv % Hk == 0, "sn_gdn_chunk_prefill2: bad shape");
  SN_REQUIRE(D == 64 || D == 128, "sn_gdn_chunk_prefill2: D=%d unsupported", D);
  SN_REQUIRE(dtype == SN_BF16, "sn_gdn_chunk_prefill2: bf16 only");
  cudaStream_t st = (cudaStream_t)stream;
  float* glast = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                          (size_t)num_chunks * Hv * (4 * (size_t)chunk::C * D + (size_t)chunk::C * chunk::C) * 2);
  if (D == 128)
    return chunk::launch_two_phase<__nv_bfloat16, 128>(qn, kn, qkv_conv, v_off, qkv_stride, glog, beta, chunks,
                                                        seq_chunk0, num_chunks, workspace, glast, o, state, slot_idx,
                                                        num_seqs, Hk, Hv, init_state, st);
  return chunk::launch_two_phase<__nv_bfloat16, 64>(qn, kn, qkv_conv, v_off, qkv_stride, glog, beta, chunks,
                                                     seq_chunk0, num_chunks, workspace, glast, o, state, slot_idx,
                                                     num_seqs, Hk, Hv, init_state, st);
}

}  // extern "C"
