// Shared pieces of the split-KV decode kernels (CUDA-core and tensor-core).
#pragma once
#include "sn_common.cuh"

namespace sn {

struct AttnDecodeArgs {
  const void* q;
  const void* k_cache;
  const void* v_cache;
  const int32_t* block_table;
  const int32_t* seq_lens;
  void* out;
  float* workspace;
  int32_t* counters;
  int B, Hq, Hkv, page_size, max_blocks, window, split_pages, max_splits;
  float scale;
};

// Number of keys a sequence attends to at decode: all of them (FA) or the
// ring's live slots (SWA: min(len, window), ring slot order is irrelevant
// because keys are stored post-RoPE).  Never more than the block table maps (a length
// past the allocation is a caller error the append reported; nothing is read past it).
__device__ __forceinline__ int attn_num_keys(const AttnDecodeArgs& a, int b) {
  const int len = min(a.seq_lens[b], a.max_blocks * a.page_size);
  return a.window > 0 ? min(len, a.window) : max(len, 0);
}

// Called by every CTA after it wrote its split partial (o unnormalised, m, l in
// log2 domain).  The last CTA of a (seq, kv head) merges all partials and writes
// the normalised output; it also re-arms the counter for the next launch.
template <typename T>
__device__ __forceinline__ void finish_split(const AttnDecodeArgs& a, int b, int hk, int num_splits, int G, int D) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* ctr = a.counters + (size_t)b * a.Hkv + hk;
    const int old = atomicAdd(ctr, 1);
    s_last = (old == num_splits - 1);
    if (s_last) atomicExch(ctr, 0);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* ws_o = a.workspace;
  const float* ws_ml = a.workspace + (size_t)a.B * a.Hkv * a.max_splits * G * D;
  const size_t base = ((size_t)b * a.Hkv + hk) * a.max_splits;
  T* out = reinterpret_cast<T*>(a.out);
  // Unrolled so that 8 splits' partials are in flight at once (one merging CTA per (sequence,
  // kv head) walks every split; a dependent load per split made many-split merges slow).
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int g = idx / D, d = idx - g * D;
    const float* ml = ws_ml + (base * G + g) * 2;
    const float* po = ws_o + base * G * D + (size_t)g * D + d;
    float M = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < num_splits; ++s) M = fmaxf(M, __ldcg(ml + (size_t)s * G * 2));
    float L = 0.f, O = 0.f;
#pragma unroll 8
    for (int s = 0; s < num_splits; ++s) {
      const float ms = __ldcg(ml + (size_t)s * G * 2);
      const float ls = __ldcg(ml + (size_t)s * G * 2 + 1);
      const float os = __ldcg(po + (size_t)s * G * D);
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L += ls * f;
      O += os * f;
    }
    io<T>::st(out + ((size_t)b * a.Hq + hk * G + g) * D + d, L > 0.f ? O / L : 0.f);
  }
}

}  // namespace sn
