// Epilogues of the decode GEMM (sn_dgemm.cu), shared by the tcgen05 kernel (bf16) and the
// CUDA-core kernel of the fp32 numerics mode, so both dtypes run the same output code.
//
// A finished (row m, weight block blk) of the GEMM is handed to finalize() as a getter that
// yields 32 accumulator columns at a time (two 16-column groups at block offsets c0 and c1);
// the getter may be warp-collective (tcgen05.ld), so finalize() keeps every call of it in
// warp-uniform control flow and guards only the global loads / stores by `row_ok`.
//
// Modes (include/sn_abi.h sn_gemm_mode):
//   STORE      out T [M][ldo] = C
//   RESID      out fp32 [M][ldo] += C            (residual stream; one writer per element)
//   PARTIAL    out fp32 [S][M][ldo]: K split s writes slab s (summed by the consumer)
//   SWIGLU_IL  W in blocks of [h gate rows; h up rows]: out T = silu(C_gate) * C_up
//   ATTN_IN    fused attention in-projection epilogue over the [q Hq | k Hkv | v Hkv] heads
//              whose q / k rows are rotary-pair interleaved (row 2i = dim i, row 2i+1 =
//              dim i + D/2, sn_rope_pair_interleave): rotate-half RoPE of q and k at the row's
//              position from the adjacent pair, q -> q_out [M][Hq][D], k / v appended to the
//              page pool / SWA ring (the decode half of sn_rope_kv_append, R/PAPER.md:1540-1563).
#pragma once
#include "sn_common.cuh"

namespace sn {
namespace epi {

struct Args {
  int mode, M, N;
  void* out;
  int ldo;
  int S;  // K splits (PARTIAL)
  // ATTN_IN
  const int32_t* positions;
  const float* inv_freq;
  void* q_out;
  void* k_cache;
  void* v_cache;
  const int32_t* block_table;
  int Hq, Hkv, D, page_size, max_blocks, window;
  int32_t* err;  // set to 1 when a position falls outside the block table (nothing is written)
  const float2* rope_cs;  // ATTN_IN: the step's (cos, sin) per (row, rotary pair) from sn_embed (NULL: sincosf)
  float* ss_out;  // RESID: per-row sum of squares of the updated residual over this block's columns,
                  // [block][M] (the fused chain's next RMSNorm sums the blocks in order)
};

template <typename T>
__device__ __forceinline__ void store32(T* o, const float* v, int n_valid, bool vec) {
  if (vec && n_valid >= 32) {
    if (sizeof(T) == 2) {
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        pk[e] = *reinterpret_cast<uint32_t*>(&b2);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        reinterpret_cast<uint4*>(o)[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
    } else {
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(o) + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (e < n_valid) io<T>::st(o + e, v[e]);
  }
}

// 16 values (two halves of a rotary pair group, or one of the 32-column groups) to T
template <typename T>
__device__ __forceinline__ void store16(T* o, const float* v) {
  if (sizeof(T) == 2) {
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
    for (int e = 0; e < 16; e += 4)
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(o) + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
  }
}

// T = activation / cache element type.  get(c0, c1, v): v[0..15] = columns c0.., v[16..31] =
// columns c1.. of this block (block-relative).  split: the block's K split (PARTIAL).
template <typename T, typename Get>
__device__ __forceinline__ void finalize(const Args& a, int m, bool row_ok, int blk, int split, int br, Get&& get) {
  const int mode = a.mode;
  float v[32];
  if (mode == SN_GEMM_SWIGLU_IL) {
    const int half = br >> 1;
    for (int c = 0; c < half; c += 16) {
      const int n = blk * half + c;
      if (n >= a.N) break;
      get(c, half + c, v);
      if (row_ok) {
        const int nv = min(min(16, half - c), a.N - n);  // h = 8 mod 16: the last group is half full
        float o[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) o[e] = silu_f(v[e]) * v[16 + e];
        T* dst = reinterpret_cast<T*>(a.out) + (size_t)m * a.ldo + n;
        if (nv == 16 && (a.ldo & 7) == 0) {
          store16<T>(dst, o);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < nv) io<T>::st(dst + e, o[e]);
        }
      }
    }
    return;
  }
  if (mode == SN_GEMM_ATTN_IN) {
    // 32-column groups never straddle a head (D and the block height are multiples of 32)
    const int D = a.D, half = D >> 1;
    int pos = 0;
    if (row_ok) pos = a.positions[m];
    for (int c = 0; c < br; c += 32) {
      const int n0 = blk * br + c;
      if (n0 >= a.N) break;
      get(c, c + 16, v);
      if (!row_ok) continue;
      const int head = n0 / D, r0 = n0 - head * D;
      const bool is_q = head < a.Hq, is_k = !is_q && head < a.Hq + a.Hkv;
      T* dst;
      if (is_q) {
        dst = reinterpret_cast<T*>(a.q_out) + ((size_t)m * a.Hq + head) * D;
      } else {
        const int hk = is_k ? head - a.Hq : head - a.Hq - a.Hkv;
        const int slot = a.window > 0 ? pos % a.window : pos;
        const int pi = slot / a.page_size;
        if (pos < 0) continue;             // idle slot (sn_embed): nothing is appended
        if (pi >= a.max_blocks) {          // past the block table: nothing is written
          if (a.err) *a.err = 1;
          continue;
        }
        const int page = a.block_table[(size_t)m * a.max_blocks + pi];
        T* cache = reinterpret_cast<T*>(is_k ? a.k_cache : a.v_cache);
        dst = cache + (((size_t)page * a.Hkv + hk) * a.page_size + slot % a.page_size) * D;
      }
      if (is_q || is_k) {  // 16 rotary pairs: dims p0.. (first halves) and p0 + D/2.. (second)
        const int p0 = r0 >> 1;
        float lo[16], hi[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float sn, cs;
          if (a.rope_cs) {
            const float2 t = a.rope_cs[(size_t)m * half + p0 + e];
            cs = t.x;
            sn = t.y;
          } else {
            sincosf((float)pos * a.inv_freq[p0 + e], &sn, &cs);
          }
          const float x1 = v[2 * e], x2 = v[2 * e + 1];
          lo[e] = x1 * cs - x2 * sn;
          hi[e] = x2 * cs + x1 * sn;
        }
        store16<T>(dst + p0, lo);
        store16<T>(dst + half + p0, hi);
      } else {
        store16<T>(dst + r0, v);
        store16<T>(dst + r0 + 16, v + 16);
      }
    }
    return;
  }
  // STORE / RESID / PARTIAL: 32 contiguous columns per round
  float ss = 0.f;
  for (int c = 0; c < br; c += 32) {
    const int n = blk * br + c;
    if (n >= a.N) break;
    get(c, c + 16, v);
    if (!row_ok) continue;
    const int nv = min(min(32, br - c), a.N - n);  // a block of 16 mod 32 rows ends mid-group
    const bool vec = (a.ldo & 7) == 0;
    if (mode == SN_GEMM_STORE) {
      store32<T>(reinterpret_cast<T*>(a.out) + (size_t)m * a.ldo + n, v, nv, vec);
    } else {
      float* o = reinterpret_cast<float*>(a.out) + ((size_t)split * a.M + m) * a.ldo + n;
      if (mode == SN_GEMM_RESID) {
        if (vec && nv == 32) {
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            const float4 old = __ldcg(reinterpret_cast<const float4*>(o + e));
            v[e] += old.x; v[e + 1] += old.y; v[e + 2] += old.z; v[e + 3] += old.w;
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < nv) v[e] += o[e];
        }
        if (a.ss_out) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e < nv) ss += v[e] * v[e];
        }
      }
      store32<float>(o, v, nv, vec);
    }
  }
  if (mode == SN_GEMM_RESID && a.ss_out && row_ok) a.ss_out[(size_t)blk * a.M + m] = ss;
}

}  // namespace epi
}  // namespace sn
