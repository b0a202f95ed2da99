// Shared helpers for the sm_100a mixer-step kernels (libsn100.so).
//
// Everything here is device/host plumbing: dtype conversion, warp reductions,
// the thread-local error string behind sn_last_error(), and launch checking.
// No kernel allocates memory; every launch goes on the caller's stream so the
// whole decode step is CUDA-graph capturable (SURVEY.md §8b "Asynchrony").
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/sn_abi.h"

namespace sn {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
sn_status check_launch(const char* what);

#define SN_REQUIRE(cond, ...)                                   \
  do {                                                          \
    if (!(cond)) {                                              \
      ::sn::set_error(__VA_ARGS__);                             \
      return SN_EINVAL;                                         \
    }                                                           \
  } while (0)

// ---------------------------------------------------------------- dtypes
template <typename T> struct io;
template <> struct io<float> {
  static __device__ __forceinline__ float ld(const float* p) { return *p; }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <> struct io<__nv_bfloat16> {
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// 8 consecutive elements <-> 8 floats (16 B for bf16, 32 B for fp32).
template <typename T> __device__ __forceinline__ void load8(const T* p, float* f);
template <> __device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
template <> __device__ __forceinline__ void load8<float>(const float* p, float* f) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// ---------------------------------------------------------------- math
// torch.nn.functional.softplus(beta=1, threshold=20), the form FLA's gate uses
// (3P-FLA/ops/gated_delta_rule/gate.py:20-45, 3P-FLA/ops/kda/gate.py:26-54).
__device__ __forceinline__ float softplus_f(float x) { return x > 20.f ? x : log1pf(expf(x)); }
// Fast-intrinsic logistic (MUFU.EX2 + approximate divide, ~2 ulp): the IEEE expf/div
// sequence measured ~20 us of epilogue time in the fused SwiGLU GEMM.  The exponent is
// clamped so the divisor stays below 2^126, where __fdividef is exact-ish (not 0).
__device__ __forceinline__ float sigmoid_f(float x) { return __fdividef(1.f, 1.f + __expf(fminf(-x, 80.f))); }
__device__ __forceinline__ float silu_f(float x) { return __fdividef(x, 1.f + __expf(fminf(-x, 80.f))); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; `scratch` needs blockDim.x/32 floats. All threads get the result.
__device__ __forceinline__ float block_sum(float v, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += scratch[i];
  return t;
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Programmatic dependent launch: lets the next kernel in the stream (if it was
// launched with the PDL attribute — the decode GEMMs are) start its prologue and
// its weight prefetch while this kernel is still running.  No-op otherwise.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Wait until the previous kernel in the stream has completed and its writes are visible
// (no-op when the kernel was not launched with programmatic stream serialization).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Launch with programmatic dependent launch: the kernel's CTAs may become resident while
// the previous kernel is still running; everything before its pdl_wait() must touch only
// data no earlier kernel of the stream writes (weights, its own state).

// Key bounds [lo, hi] of packed query row r in prefill attention (mask j in (i - w, i],
// SURVEY.md App. A item 3).  Plain prefill: queries and keys share the packed index space
// (cu_k == nullptr).  Continuation: keys are packed per sequence by cu_k and row r of
// sequence s sits at key index cu_k[s] + (r - cu_q[s]) + q_off[s].  Both bounds are
// non-decreasing in r, so a tile's key range is [lo(first row), hi(last row)].
struct KeyBounds {
  int lo, hi;
};
__device__ __forceinline__ KeyBounds key_bounds(const int32_t* __restrict__ cu_q, const int32_t* __restrict__ cu_k,
                                                const int32_t* __restrict__ q_off, int num_seqs, int r, int window) {
  int a = 0, b = num_seqs;  // largest s with cu_q[s] <= r
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (cu_q[mid] <= r) a = mid; else b = mid;
  }
  int ks, hi;
  if (cu_k) {
    ks = cu_k[a];
    hi = ks + (r - cu_q[a]) + q_off[a];
  } else {
    ks = cu_q[a];
    hi = r;
  }
  return {window > 0 ? max(ks, hi - window + 1) : ks, hi};
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace sn

#define SN_DISPATCH_DTYPE(dtype, T, ...)                                  \
  [&]() -> sn_status {                                                    \
    if ((dtype) == SN_BF16) { using T = __nv_bfloat16; return __VA_ARGS__(); } \
    if ((dtype) == SN_F32) { using T = float; return __VA_ARGS__(); }     \
    ::sn::set_error("unsupported dtype code %d", (int)(dtype));           \
    return SN_EUNSUPPORTED;                                               \
  }()
