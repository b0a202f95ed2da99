// Prefill attention on tensor cores (FA / SWA layers, R/PAPER.md:1540-1563): causal
// (window == 0) or sliding-window (keys j with i - w < j <= i)
// softmax attention over packed sequences, GQA (q head h reads kv head h / (Hq/Hkv)).
//
// Flash-attention tiling: one CTA = 64 packed query rows x one q head, 4 warps x 16 rows.
// Key/value blocks of 64 rows stream through double-buffered shared memory (cp.async,
// zero-filled past the end); S = Q K^T and O += P V are bf16 mma.sync tiles with fp32
// accumulators; the online softmax runs on the S fragments in registers (row max / sum
// over the 4 lanes of a quad) and P is re-packed in place as the A operand of P V.
// Rows are packed over sequences, so a tile may straddle a sequence boundary: every
// (row, key) pair is masked with the row's own sequence start, which also keeps keys of
// other sequences out.  Oracle: oracle/supernet_oracle.py attention_ref (pinned to
// torch scaled_dot_product_attention); the CUDA-core kernel in sn_attn.cu is kept for
// fp32 I/O (1e-4 parity mode).
#include "sn_mma.cuh"

namespace sn {
namespace fa {

using namespace sn::mma;

constexpr int BM = 64, BN = 64, kThreads = 128;

template <int D>
struct Smem {
  static constexpr int LD = D + 8;
  __nv_bfloat16 q[BM * LD];
  __nv_bfloat16 k[2][BN * LD];
  __nv_bfloat16 v[2][BN * LD];
};

__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


template <int D>
__global__ void __launch_bounds__(kThreads)
    attn_prefill_tc_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                           const __nv_bfloat16* __restrict__ v, const int32_t* __restrict__ cu,
                           __nv_bfloat16* __restrict__ out, int num_seqs, int rows, int Hq, int Hkv, int window,
                           float scale, const int32_t* __restrict__ cu_k, const int32_t* __restrict__ q_off) {
  using SM = Smem<D>;
  constexpr int LD = SM::LD, NT = D / 8, KS = D / 16;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  const int tiles = (rows + BM - 1) / BM;
  const int r0 = (tiles - 1 - (int)blockIdx.x) * BM;  // heavy (late) tiles first
  const int h = blockIdx.y, hk = h / (Hq / Hkv);
  const float qs = scale * 1.4426950408889634f;  // exp2 domain

  // this thread's two rows and their key bounds
  const int ra = r0 + warp * 16 + g4, rb = ra + 8;
  const KeyBounds kba = key_bounds(cu, cu_k, q_off, num_seqs, min(ra, rows - 1), window);
  const KeyBounds kbb = key_bounds(cu, cu_k, q_off, num_seqs, min(rb, rows - 1), window);
  const int lo_a = kba.lo, lo_b = kbb.lo, hi_a = kba.hi, hi_b = kbb.hi;
  // key range of the whole tile
  const int r_last = min(r0 + BM - 1, rows - 1);
  const KeyBounds kb0 = key_bounds(cu, cu_k, q_off, num_seqs, r0, window);
  const KeyBounds kbl = key_bounds(cu, cu_k, q_off, num_seqs, r_last, window);
  const int j_lo = kb0.lo, j_hi = kbl.hi;

  auto load_kv = [&](int jb, int buf) {
#pragma unroll
    for (int it = 0; it < BN * D / 8 / kThreads; ++it) {
      const int idx = tid + it * kThreads;
      const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
      const int j = jb + r;
      const bool ok = j <= j_hi;
      const size_t off = ((size_t)(ok ? j : 0) * Hkv + hk) * D + c8;
      cp16(&sm.k[buf][r * LD + c8], k + off, ok);
      cp16(&sm.v[buf][r * LD + c8], v + off, ok);
    }
    cp_commit();
  };
#pragma unroll
  for (int it = 0; it < BM * D / 8 / kThreads; ++it) {
    const int idx = tid + it * kThreads;
    const int r = idx / (D / 8), c8 = (idx % (D / 8)) * 8;
    const bool ok = r0 + r < rows;
    cp16(&sm.q[r * LD + c8], q + ((size_t)(ok ? r0 + r : 0) * Hq + h) * D + c8, ok);
  }
  load_kv(j_lo, 0);  // (the Q copies join this commit group)

  float o[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[nt][e] = 0.f;
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  uint32_t qa[KS][4];

  int buf = 0;
  bool first = true;
  for (int jb = j_lo; jb <= j_hi; jb += BN, buf ^= 1) {
    if (jb + BN <= j_hi) {
      load_kv(jb + BN, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (first) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) lda(sm.q, LD, warp * 16, ks * 16, qa[ks]);
      first = false;
    }
    // S = Q K^T (16 rows x 64 keys per warp)
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldb_nk(sm.k[buf], LD, nt * 8, ks * 16, b0, b1, b2, b3);
        mma_bf16(s[nt], qa[ks], b0, b1);
        mma_bf16(s[nt + 1], qa[ks], b2, b3);
      }
    // mask: only blocks touching a row's bounds need it
    const bool full = jb >= kbl.lo && jb + BN - 1 <= kb0.hi;
    float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb + nt * 8 + t4 * 2 + (e & 1);
        const bool rowb = e >= 2;
        float x = s[nt][e] * qs;
        if (!full) {
          const int hi = rowb ? hi_b : hi_a, lo = rowb ? lo_b : lo_a;
          if (j > hi || j < lo) x = -INFINITY;
        }
        s[nt][e] = x;
        if (rowb) mx_b = fmaxf(mx_b, x); else mx_a = fmaxf(mx_a, x);
      }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, off));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, off));
    }
    const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
    const float base_a = mn_a == -INFINITY ? 0.f : mn_a, base_b = mn_b == -INFINITY ? 0.f : mn_b;
    const float al_a = exp2f(m_a - base_a), al_b = exp2f(m_b - base_b);
    m_a = mn_a;
    m_b = mn_b;
    l_a *= al_a;
    l_b *= al_b;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      o[nt][0] *= al_a; o[nt][1] *= al_a;
      o[nt][2] *= al_b; o[nt][3] *= al_b;
    }
    uint32_t pa[4][4];  // P as the A operand of P V: 4 k-steps of 16 keys
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - base_a), p1 = exp2f(s[nt][1] - base_a);
      const float p2 = exp2f(s[nt][2] - base_b), p3 = exp2f(s[nt][3] - base_b);
      l_a += p0 + p1;
      l_b += p2 + p3;
      const int kk = nt >> 1, hi = nt & 1;
      pa[kk][hi ? 2 : 0] = pack_bf16(p0, p1);
      pa[kk][hi ? 3 : 1] = pack_bf16(p2, p3);
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int nt = 0; nt < NT; nt += 2) {
        uint32_t b0, b1, b2, b3;
        ldb_kn(sm.v[buf], LD, nt * 8, kk * 16, b0, b1, b2, b3);
        mma_bf16(o[nt], pa[kk], b0, b1);
        mma_bf16(o[nt + 1], pa[kk], b2, b3);
      }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's prefetch
  }
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    l_a += __shfl_xor_sync(0xffffffffu, l_a, off);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, off);
  }
  const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
  const size_t ld_o = (size_t)Hq * D;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = h * D + nt * 8 + t4 * 2;
    if (ra < rows) *reinterpret_cast<uint32_t*>(out + (size_t)ra * ld_o + c) = pack_bf16(o[nt][0] * ia, o[nt][1] * ia);
    if (rb < rows) *reinterpret_cast<uint32_t*>(out + (size_t)rb * ld_o + c) = pack_bf16(o[nt][2] * ib, o[nt][3] * ib);
  }
}

template <int D>
static sn_status launch(const void* q, const void* k, const void* v, const int32_t* cu, void* out, int num_seqs,
                        int rows, int Hq, int Hkv, int window, float scale, const int32_t* cu_k,
                        const int32_t* q_off, cudaStream_t st) {
  const int smem = (int)sizeof(Smem<D>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((rows + BM - 1) / BM, Hq);
  attn_prefill_tc_kernel<D><<<grid, kThreads, smem, st>>>(
      (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, cu, (__nv_bfloat16*)out, num_seqs,
      rows, Hq, Hkv, window, scale, cu_k, q_off);
  return check_launch("sn_attn_prefill(tc)");
}

}  // namespace fa

sn_status attn_prefill_umma_bf16(const void* q, const void* k, const void* v, const int32_t* cu, void* out,
                                 int num_seqs, int rows, int Hq, int Hkv, int window, float scale,
                                 const int32_t* cu_k, const int32_t* q_off, int rows_k,
                                 cudaStream_t st);  // sn_attn_prefill_umma.cu

sn_status attn_prefill_tc_bf16(const void* q, const void* k, const void* v, const int32_t* cu, void* out,
                               int num_seqs, int rows, int Hq, int Hkv, int D, int window, float scale,
                               const int32_t* cu_k, const int32_t* q_off, int rows_k, cudaStream_t st) {
  // head dim 128 (every Apriel attention layer): the tcgen05/TMEM kernel; head dim 64 (the tiny
  // test configuration only): the mma.sync kernel of this file
  if (D == 128)
    return attn_prefill_umma_bf16(q, k, v, cu, out, num_seqs, rows, Hq, Hkv, window, scale, cu_k, q_off, rows_k, st);
  if (D == 64) return fa::launch<64>(q, k, v, cu, out, num_seqs, rows, Hq, Hkv, window, scale, cu_k, q_off, st);
  set_error("sn_attn_prefill: D=%d unsupported", D);
  return SN_EUNSUPPORTED;
}

}  // namespace sn
