// FA / SWA mixers (R/PAPER.md:1540-1563): GQA attention with RoPE over a paged
// KV pool (FA) or a per-sequence ring of `window` slots in the same pool (SWA).
//
// Decode cost model (R/PAPER.md:1548-1556): reading K and V is 2*t*Hkv*D*b bytes
// per layer per sequence at intensity ~Hq/(2*Hkv*b) flop/byte, so decode is an
// HBM stream.  This file holds the bookkeeping kernels (RoPE + KV append),
// the CUDA-core split-KV decode (fp32 I/O and cross-check path), and prefill.
// The bf16 tensor-core decode lives in sn_attn_tc.cu.
#include "sn_common.cuh"
#include "sn_attn.cuh"

namespace sn {

// two adjacent elements <-> float2 (one 4-byte access for bf16, 8 for fp32)
template <typename T> __device__ __forceinline__ float2 bf2_or_f2(const T* p);
template <> __device__ __forceinline__ float2 bf2_or_f2<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
template <> __device__ __forceinline__ float2 bf2_or_f2<float>(const float* p) { return *reinterpret_cast<const float2*>(p); }
template <typename T> __device__ __forceinline__ void st2(T* p, float a, float b);
template <> __device__ __forceinline__ void st2<__nv_bfloat16>(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
template <> __device__ __forceinline__ void st2<float>(float* p, float a, float b) { *reinterpret_cast<float2*>(p) = make_float2(a, b); }

// ------------------------------------------------------------------ RoPE + append
// grid (rows, Hq + 2*Hkv): one CTA per (row, head); heads < Hq are query heads
// (rotate, write q_out), the next Hkv are key heads (rotate, append to the cache),
// the last Hkv are value heads (copy to the cache).  Thread i owns rotary pair i.
template <typename T>
__device__ __forceinline__ void rope_kv_one(const T* __restrict__ qkv, const int32_t* __restrict__ row_seq,
                                            const int32_t* __restrict__ row_pos, const int32_t* __restrict__ seq_lens,
                                            const float* __restrict__ inv_freq, T* __restrict__ q_out,
                                            T* __restrict__ k_out, T* __restrict__ v_out, T* __restrict__ k_cache,
                                            T* __restrict__ v_cache, const int32_t* __restrict__ block_table, int Hq,
                                            int Hkv, int D, int page_size, int max_blocks, int window, int r,
                                            int head, int i, int pair_il) {
  const int half = D / 2;
  const int seq = row_seq ? row_seq[r] : r;
  const int pos = row_pos[r];
  const size_t src = (size_t)r * (Hq + 2 * Hkv) * D + (size_t)head * D;
  // cache slot (FA: the position; SWA: ring slot), SWA rows older than the window are not stored
  const int slot = window > 0 ? pos % window : pos;
  // a slot past the block table (position beyond the allocated length) is never written
  const bool write = !(window > 0 && seq_lens != nullptr && pos < seq_lens[seq] - window) && pos >= 0 &&
                     slot / page_size < max_blocks;
  if (head >= Hq + Hkv) {  // value head: plain copy
    const int hk = head - Hq - Hkv;
    const float v1 = io<T>::ld(qkv + src + i), v2 = io<T>::ld(qkv + src + i + half);
    if (v_out) {
      T* dst = v_out + ((size_t)r * Hkv + hk) * D;
      io<T>::st(dst + i, v1);
      io<T>::st(dst + i + half, v2);
    }
    if (write) {
      const int page = block_table[(size_t)seq * max_blocks + slot / page_size];
      T* dst = v_cache + (((size_t)page * Hkv + hk) * page_size + slot % page_size) * D;
      io<T>::st(dst + i, v1);
      io<T>::st(dst + i + half, v2);
    }
    return;
  }
  float sn, cs;
  sincosf((float)pos * inv_freq[i], &sn, &cs);
  // q / k rows rotary-pair interleaved (the decode in-projection's weight order): dims i and
  // i + D/2 sit at columns 2i and 2i + 1 of the head
  const int c1 = pair_il ? 2 * i : i, c2 = pair_il ? 2 * i + 1 : i + half;
  const float x1 = io<T>::ld(qkv + src + c1), x2 = io<T>::ld(qkv + src + c2);
  const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
  if (head < Hq) {
    T* dst = q_out + ((size_t)r * Hq + head) * D;
    io<T>::st(dst + i, y1);
    io<T>::st(dst + i + half, y2);
    return;
  }
  const int hk = head - Hq;
  if (k_out) {
    T* dst = k_out + ((size_t)r * Hkv + hk) * D;
    io<T>::st(dst + i, y1);
    io<T>::st(dst + i + half, y2);
  }
  if (write) {
    const int page = block_table[(size_t)seq * max_blocks + slot / page_size];
    T* dst = k_cache + (((size_t)page * Hkv + hk) * page_size + slot % page_size) * D;
    io<T>::st(dst + i, y1);
    io<T>::st(dst + i + half, y2);
  }
}

// Decode: a CTA per (row, head), a thread per rotation pair.
template <typename T>
__global__ void rope_kv_append_kernel(const T* __restrict__ qkv, const int32_t* __restrict__ row_seq,
                                      const int32_t* __restrict__ row_pos, const int32_t* __restrict__ seq_lens,
                                      const float* __restrict__ inv_freq, T* __restrict__ q_out,
                                      T* __restrict__ k_out, T* __restrict__ v_out, T* __restrict__ k_cache,
                                      T* __restrict__ v_cache, const int32_t* __restrict__ block_table, int Hq,
                                      int Hkv, int D, int page_size, int max_blocks, int window, int pair_il) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  if ((int)threadIdx.x >= D / 2) return;
  rope_kv_one<T>(qkv, row_seq, row_pos, seq_lens, inv_freq, q_out, k_out, v_out, k_cache, v_cache, block_table, Hq,
                 Hkv, D, page_size, max_blocks, window, blockIdx.x, blockIdx.y, threadIdx.x, pair_il);
}

// Prefill (many rows): a 256-thread CTA per row.  The rotation angles depend only on the
// position and the pair index, so the row's D/2 (cos, sin) pairs are computed once into shared
// memory (not once per head: 40 of them at Apriel widths); each thread then rotates two
// adjacent pairs of one head per step with 8-byte loads and 4-byte stores.
template <typename T>
__global__ void __launch_bounds__(256) rope_kv_append_rows_kernel(
    const T* __restrict__ qkv, const int32_t* __restrict__ row_seq, const int32_t* __restrict__ row_pos,
    const int32_t* __restrict__ seq_lens, const float* __restrict__ inv_freq, T* __restrict__ q_out,
    T* __restrict__ k_out, T* __restrict__ v_out, T* __restrict__ k_cache, T* __restrict__ v_cache,
    const int32_t* __restrict__ block_table, int Hq, int Hkv, int D, int page_size, int max_blocks, int window,
    int pair_il) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float s_cs[64], s_sn[64];
  const int half = D / 2, r = blockIdx.x;
  const int seq = row_seq ? row_seq[r] : r;
  const int pos = row_pos[r];
  if ((int)threadIdx.x < half) sincosf((float)pos * inv_freq[threadIdx.x], &s_sn[threadIdx.x], &s_cs[threadIdx.x]);
  __syncthreads();
  const int slot = window > 0 ? pos % window : pos;
  const bool write = !(window > 0 && seq_lens != nullptr && pos < seq_lens[seq] - window) && pos >= 0 &&
                     slot / page_size < max_blocks;
  const int page = write ? block_table[(size_t)seq * max_blocks + slot / page_size] : 0;
  const int npp = half / 2;  // pairs of adjacent rotation pairs per head
  const int n = (Hq + 2 * Hkv) * npp;
  const T* row = qkv + (size_t)r * (Hq + 2 * Hkv) * D;
  for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
    const int head = idx / npp, i = (idx - head * npp) * 2;  // pairs i, i + 1
    const T* src = row + (size_t)head * D;
    float y1[2], y2[2];
    if (head >= Hq + Hkv) {  // value head: plain copy of dims (i, i+1) and (i + D/2, +1)
      const float2 a = bf2_or_f2<T>(src + i), c = bf2_or_f2<T>(src + i + half);
      y1[0] = a.x; y1[1] = a.y; y2[0] = c.x; y2[1] = c.y;
    } else {
      float x1[2], x2[2];
      if (pair_il) {  // columns 2i, 2i+1, 2i+2, 2i+3 = (x1, x2) of pair i, then of pair i+1
        const float2 a = bf2_or_f2<T>(src + 2 * i), c = bf2_or_f2<T>(src + 2 * i + 2);
        x1[0] = a.x; x2[0] = a.y; x1[1] = c.x; x2[1] = c.y;
      } else {
        const float2 a = bf2_or_f2<T>(src + i), c = bf2_or_f2<T>(src + i + half);
        x1[0] = a.x; x1[1] = a.y; x2[0] = c.x; x2[1] = c.y;
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float cs = s_cs[i + e], sn = s_sn[i + e];
        y1[e] = x1[e] * cs - x2[e] * sn;
        y2[e] = x2[e] * cs + x1[e] * sn;
      }
    }
    T* dst;
    if (head < Hq) {
      dst = q_out + ((size_t)r * Hq + head) * D;
    } else {
      const bool is_k = head < Hq + Hkv;
      const int hk = is_k ? head - Hq : head - Hq - Hkv;
      T* extra = is_k ? k_out : v_out;
      if (extra) {
        T* e2 = extra + ((size_t)r * Hkv + hk) * D;
        st2<T>(e2 + i, y1[0], y1[1]);
        st2<T>(e2 + i + half, y2[0], y2[1]);
      }
      if (!write) continue;
      dst = (is_k ? k_cache : v_cache) + (((size_t)page * Hkv + hk) * page_size + slot % page_size) * D;
    }
    st2<T>(dst + i, y1[0], y1[1]);
    st2<T>(dst + i + half, y2[0], y2[1]);
  }
}

// ------------------------------------------------------------------ CUDA-core decode
// CTA = (split, kv head, seq), 4 warps; warp w takes keys w, w+4, ... of the split,
// keeps its own online-softmax state, the 4 states merge in smem.
template <typename T, int D, int GMAX>
__global__ void __launch_bounds__(128) attn_decode_simt_kernel(AttnDecodeArgs a) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  constexpr int EPL = D / 32;
  __shared__ float s_q[GMAX][D];
  __shared__ float s_m[4][GMAX], s_l[4][GMAX];
  __shared__ float s_o[4][GMAX][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int G = a.Hq / a.Hkv;
  const int n_keys = attn_num_keys(a, b);
  const int split_keys = a.split_pages * a.page_size;
  const int num_splits = max(1, (n_keys + split_keys - 1) / split_keys);
  if (split >= num_splits) return;
  const int k0 = split * split_keys, k1 = min(n_keys, k0 + split_keys);
  const T* Q = reinterpret_cast<const T*>(a.q);
  const T* Kc = reinterpret_cast<const T*>(a.k_cache);
  const T* Vc = reinterpret_cast<const T*>(a.v_cache);
  const float qscale = a.scale * 1.4426950408889634f;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int g = idx / D, d = idx - g * D;
    s_q[g][d] = io<T>::ld(Q + ((size_t)b * a.Hq + hk * G + g) * D + d) * qscale;
  }
  __syncthreads();
  float m[GMAX], l[GMAX], o[GMAX][EPL];
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[g][e] = 0.f;
  }
  const int32_t* bt = a.block_table + (size_t)b * a.max_blocks;
  for (int key = k0 + warp; key < k1; key += 4) {
    const int page = bt[key / a.page_size], off = key % a.page_size;
    const size_t base = (((size_t)page * a.Hkv + hk) * a.page_size + off) * D;
    float kv[EPL], vv[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      kv[e] = io<T>::ld(Kc + base + lane + 32 * e);
      vv[e] = io<T>::ld(Vc + base + lane + 32 * e);
    }
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < G) {
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) s += s_q[g][lane + 32 * e] * kv[e];
        s = warp_sum(s);
        const float mn = fmaxf(m[g], s);
        const float alpha = exp2f(m[g] - mn), p = exp2f(s - mn);
        l[g] = l[g] * alpha + p;
#pragma unroll
        for (int e = 0; e < EPL; ++e) o[g][e] = o[g][e] * alpha + p * vv[e];
        m[g] = mn;
      }
    }
  }
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g < G) {
      if (lane == 0) { s_m[warp][g] = m[g]; s_l[warp][g] = l[g]; }
#pragma unroll
      for (int e = 0; e < EPL; ++e) s_o[warp][g][lane + 32 * e] = o[g][e];
    }
  }
  __syncthreads();
  // merge the 4 warps into one partial (m, l, o unnormalised)
  float* ws_o = a.workspace;
  float* ws_ml = a.workspace + (size_t)a.B * a.Hkv * a.max_splits * G * D;
  const size_t part = ((size_t)b * a.Hkv + hk) * a.max_splits + split;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int g = idx / D, d = idx - g * D;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, s_m[w][g]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float f = s_m[w][g] == -INFINITY ? 0.f : exp2f(s_m[w][g] - M);
      L += s_l[w][g] * f;
      O += s_o[w][g][d] * f;
    }
    ws_o[(part * G + g) * D + d] = O;
    if (d == 0) { ws_ml[(part * G + g) * 2] = M; ws_ml[(part * G + g) * 2 + 1] = L; }
  }
  finish_split<T>(a, b, hk, num_splits, G, D);
}

// ------------------------------------------------------------------ prefill (CUDA cores)
// One warp per (query row, q head); keys in blocks of 32: lane j scores key j
// (full-D dot, q broadcast from smem), warp-level online softmax, then lanes
// switch to owning D/32 output dims for the P.V accumulation.
template <typename T, int D>
__global__ void __launch_bounds__(128) attn_prefill_kernel(const T* __restrict__ q, const T* __restrict__ k,
                                                           const T* __restrict__ v, const int32_t* __restrict__ cu,
                                                           T* __restrict__ out, int num_seqs, int rows, int Hq,
                                                           int Hkv, int window, float scale,
                                                           const int32_t* __restrict__ cu_k,
                                                           const int32_t* __restrict__ q_off) {
  constexpr int EPL = D / 32;
  __shared__ float s_q[4][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * 4 + warp;
  const int h = blockIdx.y;
  if (r >= rows) return;
  const KeyBounds kb = key_bounds(cu, cu_k, q_off, num_seqs, r, window);  // keys [lo, hi], packed key indices
  const int i = kb.hi;
  const int G = Hq / Hkv, hk = h / G;
  const float qscale = scale * 1.4426950408889634f;
  for (int d = lane; d < D; d += 32) s_q[warp][d] = io<T>::ld(q + ((size_t)r * Hq + h) * D + d) * qscale;
  __syncwarp();
  const int j_lo = kb.lo;
  float m = -INFINITY, l = 0.f, o[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) o[e] = 0.f;
  for (int jb = j_lo; jb <= i; jb += 32) {
    const int j = jb + lane;
    float sc = -INFINITY;
    if (j <= i) {
      const T* kr = k + ((size_t)j * Hkv + hk) * D;
      float acc = 0.f;
      for (int d = 0; d < D; d += 8) {
        float f[8];
        load8<T>(kr + d, f);
#pragma unroll
        for (int x = 0; x < 8; ++x) acc += f[x] * s_q[warp][d + x];
      }
      sc = acc;
    }
    const float mn = fmaxf(m, warp_max(sc));
    const float p = j <= i ? exp2f(sc - mn) : 0.f;
    const float alpha = exp2f(m - mn);
    l = l * alpha + warp_sum(p);
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[e] *= alpha;
    const int nk = min(32, i - jb + 1);
    for (int x = 0; x < nk; ++x) {
      const float px = __shfl_sync(0xffffffffu, p, x);
      const T* vr = v + ((size_t)(jb + x) * Hkv + hk) * D;
#pragma unroll
      for (int e = 0; e < EPL; ++e) o[e] += px * io<T>::ld(vr + lane + 32 * e);
    }
    m = mn;
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < EPL; ++e) io<T>::st(out + ((size_t)r * Hq + h) * D + lane + 32 * e, o[e] * inv);
}

sn_status attn_decode_tc_bf16(const AttnDecodeArgs& a, int D, cudaStream_t st);  // sn_attn_tc.cu
sn_status attn_prefill_tc_bf16(const void* q, const void* k, const void* v, const int32_t* cu, void* out,
                               int num_seqs, int rows, int Hq, int Hkv, int D, int window, float scale,
                               const int32_t* cu_k, const int32_t* q_off, int rows_k,
                               cudaStream_t st);  // sn_attn_prefill.cu

}  // namespace sn

using namespace sn;

extern "C" {

sn_status sn_rope_kv_append(const void* qkv, const int32_t* row_seq, const int32_t* row_pos,
                            const int32_t* seq_lens, const float* inv_freq, void* q_out, void* k_out,
                            void* v_out, void* k_cache, void* v_cache, const int32_t* block_table, int rows,
                            int Hq, int Hkv, int D, int page_size, int max_blocks, int window, int pair_il,
                            int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0 && D % 4 == 0 && D <= 128, "sn_rope_kv_append: bad shape");
  SN_REQUIRE(page_size > 0 && (window == 0 || window % page_size == 0),
             "sn_rope_kv_append: window %d must be a multiple of page_size %d", window, page_size);
  SN_REQUIRE(qkv && row_pos && inv_freq && q_out && k_cache && v_cache && block_table,
             "sn_rope_kv_append: NULL pointer argument");
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    const T* in = (const T*)qkv;
    if (rows > 1024)
      launch_pdl(rope_kv_append_rows_kernel<T>, dim3(rows), dim3(256), 0, (cudaStream_t)stream, in, row_seq,
                 row_pos, seq_lens, inv_freq, (T*)q_out, (T*)k_out, (T*)v_out, (T*)k_cache, (T*)v_cache,
                 block_table, Hq, Hkv, D, page_size, max_blocks, window, pair_il);
    else
      launch_pdl(rope_kv_append_kernel<T>, dim3(rows, Hq + 2 * Hkv), dim3(((D / 2 + 31) / 32) * 32), 0,
                 (cudaStream_t)stream, in, row_seq, row_pos, seq_lens, inv_freq, (T*)q_out, (T*)k_out, (T*)v_out,
                 (T*)k_cache, (T*)v_cache, block_table, Hq, Hkv, D, page_size, max_blocks, window, pair_il);
    return check_launch("sn_rope_kv_append");
  });
}

size_t sn_attn_decode_workspace_bytes(int B, int Hq, int Hkv, int D, int max_splits) {
  const size_t G = Hkv > 0 ? (size_t)(Hq / Hkv) : 0;
  return (size_t)B * Hkv * max_splits * G * (D + 2) * sizeof(float);
}

sn_status sn_attn_decode(const void* q, const void* k_cache, const void* v_cache, const int32_t* block_table,
                         const int32_t* seq_lens, void* out, float* workspace, int32_t* counters, int B, int Hq,
                         int Hkv, int D, int page_size, int max_blocks, int window, int split_pages,
                         int max_splits, float scale, int dtype, void* stream) {
  SN_REQUIRE(B > 0 && Hkv > 0 && Hq % Hkv == 0 && Hq / Hkv <= 8, "sn_attn_decode: bad heads Hq=%d Hkv=%d", Hq, Hkv);
  SN_REQUIRE(split_pages > 0 && max_splits > 0, "sn_attn_decode: bad split config");
  SN_REQUIRE(window == 0 || window % page_size == 0, "sn_attn_decode: window %% page_size != 0");
  SN_REQUIRE(q && k_cache && v_cache && block_table && seq_lens && out && workspace && counters,
             "sn_attn_decode: NULL pointer argument");
  AttnDecodeArgs a{q, k_cache, v_cache, block_table, seq_lens, out, workspace, counters, B, Hq, Hkv,
                   page_size, max_blocks, window, split_pages, max_splits, scale};
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SN_BF16) {  // tensor-core split-KV decode (sn_attn_tc.cu); fp32 I/O below
    SN_REQUIRE((D == 128 || D == 64) && page_size == 64, "sn_attn_decode: bf16 needs D in {64, 128}, page 64");
    return attn_decode_tc_bf16(a, D, st);
  }
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    dim3 grid(max_splits, Hkv, B);
    if (D == 128) launch_pdl(attn_decode_simt_kernel<T, 128, 8>, grid, dim3(128), 0, st, a);
    else if (D == 64) launch_pdl(attn_decode_simt_kernel<T, 64, 8>, grid, dim3(128), 0, st, a);
    else { set_error("sn_attn_decode: D=%d unsupported", D); return SN_EUNSUPPORTED; }
    return check_launch("sn_attn_decode");
  });
}

sn_status sn_attn_prefill(const void* q, const void* k, const void* v, const int32_t* cu_seqlens,
                          const int32_t* cu_k, const int32_t* q_off, void* out, int num_seqs, int rows,
                          int rows_k, int Hq, int Hkv, int D, int window, float scale, int dtype,
                          void* stream) {
  SN_REQUIRE(num_seqs > 0 && rows > 0 && Hkv > 0 && Hq % Hkv == 0, "sn_attn_prefill: bad shape");
  SN_REQUIRE((cu_k == nullptr) == (q_off == nullptr), "sn_attn_prefill: cu_k and q_off go together");
  if (cu_k == nullptr) rows_k = rows;
  SN_REQUIRE(rows_k > 0, "sn_attn_prefill: no keys");
  if (dtype == SN_BF16)  // tensor-core flash attention (sn_attn_prefill*.cu); fp32 I/O below
    return attn_prefill_tc_bf16(q, k, v, cu_seqlens, out, num_seqs, rows, Hq, Hkv, D, window, scale, cu_k, q_off,
                                rows_k, (cudaStream_t)stream);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    dim3 grid(ceil_div(rows, 4), Hq);
    cudaStream_t st = (cudaStream_t)stream;
    if (D == 128) attn_prefill_kernel<T, 128><<<grid, 128, 0, st>>>((const T*)q, (const T*)k, (const T*)v, cu_seqlens, (T*)out, num_seqs, rows, Hq, Hkv, window, scale, cu_k, q_off);
    else if (D == 64) attn_prefill_kernel<T, 64><<<grid, 128, 0, st>>>((const T*)q, (const T*)k, (const T*)v, cu_seqlens, (T*)out, num_seqs, rows, Hq, Hkv, window, scale, cu_k, q_off);
    else { set_error("sn_attn_prefill: D=%d unsupported", D); return SN_EUNSUPPORTED; }
    return check_launch("sn_attn_prefill");
  });
}

}  // extern "C"
