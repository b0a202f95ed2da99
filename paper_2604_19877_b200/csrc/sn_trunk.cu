// Shared-trunk kernels: embedding (+decode-step prologue), fused residual-add
// RMSNorm, SiLU-gated FFN activation, greedy argmax.  All HBM-bound, one pass
// over their operands, 16-byte vector loads.
//
// Trunk definition: R/PAPER.md:175-182 (Apriel-1.6: d=5120, SiLU-gated FFN
// 14336, vocab 131072), shared across mixers R/PAPER.md:855-856.
#include <stdarg.h>
#include <string.h>

#include "sn_common.cuh"

namespace sn {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

sn_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return SN_OK;
}

// ------------------------------------------------------------------ embed
template <typename T>
__global__ void embed_kernel(const int32_t* __restrict__ tokens, const T* __restrict__ table,
                             float* __restrict__ residual, int32_t* seq_lens, int32_t* positions,
                             int rows, int dim) {
  const int r = blockIdx.x;
  if (seq_lens != nullptr && r == 0) {
    for (int b = threadIdx.x; b < rows; b += blockDim.x) {
      int L = seq_lens[b];
      positions[b] = L;
      seq_lens[b] = L + 1;
    }
  }
  const T* src = table + (size_t)tokens[r] * dim;
  float* dst = residual + (size_t)r * dim;
  for (int i = threadIdx.x * 8; i < dim; i += blockDim.x * 8) {
    float f[8];
    load8<T>(src + i, f);
    *reinterpret_cast<float4*>(dst + i) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(dst + i + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
}

// ------------------------------------------------------------------ add + rmsnorm
// One CTA per row; the row (dim <= 8*256*MAXV floats) stays in registers between
// the sum-of-squares pass and the normalise pass.
template <typename T, int MAXV>
__global__ void __launch_bounds__(256) add_rmsnorm_kernel(const T* __restrict__ delta,
                                                          float* __restrict__ residual,
                                                          const T* __restrict__ weight,
                                                          T* __restrict__ out, int dim, float eps) {
  __shared__ float scratch[32];
  const int r = blockIdx.x;
  float* res = residual + (size_t)r * dim;
  float v[MAXV][8];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < MAXV; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 8;
    if (i < dim) {
      float4 a = *reinterpret_cast<const float4*>(res + i);
      float4 b = *reinterpret_cast<const float4*>(res + i + 4);
      v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
      v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      if (delta != nullptr) {
        float d[8];
        load8<T>(delta + (size_t)r * dim + i, d);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[c][k] += d[k];
        *reinterpret_cast<float4*>(res + i) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
        *reinterpret_cast<float4*>(res + i + 4) = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += v[c][k] * v[c][k];
    }
  }
  ss = block_sum(ss, scratch);
  const float rstd = rsqrtf(ss / (float)dim + eps);
#pragma unroll
  for (int c = 0; c < MAXV; ++c) {
    const int i = (c * blockDim.x + threadIdx.x) * 8;
    if (i < dim) {
      float w[8];
      load8<T>(weight + i, w);
#pragma unroll
      for (int k = 0; k < 8; ++k) io<T>::st(out + (size_t)r * dim + i + k, v[c][k] * rstd * w[k]);
    }
  }
}

// ------------------------------------------------------------------ silu * mul
template <typename T>
__global__ void silu_mul_kernel(const T* __restrict__ gu, T* __restrict__ out, int rows, int ffn) {
  const size_t n8 = (size_t)rows * ffn / 8;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8;
       q += (size_t)gridDim.x * blockDim.x) {
    const size_t e = q * 8;
    const size_t r = e / ffn, i = e % ffn;
    float g[8], u[8];
    load8<T>(gu + r * 2 * ffn + i, g);
    load8<T>(gu + r * 2 * ffn + ffn + i, u);
#pragma unroll
    for (int k = 0; k < 8; ++k) io<T>::st(out + r * ffn + i + k, silu_f(g[k]) * u[k]);
  }
}

// ------------------------------------------------------------------ argmax
template <typename T>
__global__ void __launch_bounds__(1024) argmax_kernel(const T* __restrict__ logits, int vocab,
                                                      int32_t* __restrict__ out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  const T* row = logits + (size_t)blockIdx.x * vocab;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x * 8; i < vocab; i += blockDim.x * 8) {
    float f[8];
    load8<T>(row + i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (f[k] > best) { best = f[k]; bi = i + k; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sv[warp] = best; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    out[blockIdx.x] = bi;
  }
}

}  // namespace sn

using namespace sn;

extern "C" {

const char* sn_last_error(void) { return sn::g_err; }
int sn_abi_version(void) { return SN_ABI_VERSION; }

sn_status sn_embed(const int32_t* tokens, const void* table, float* residual, int32_t* seq_lens,
                   int32_t* positions, int rows, int dim, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && dim > 0 && dim % 8 == 0, "sn_embed: bad shape rows=%d dim=%d", rows, dim);
  SN_REQUIRE((seq_lens == nullptr) == (positions == nullptr), "sn_embed: seq_lens/positions must be both set or both NULL");
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    embed_kernel<T><<<rows, 128, 0, (cudaStream_t)stream>>>(tokens, (const T*)table, residual, seq_lens,
                                                            positions, rows, dim);
    return check_launch("sn_embed");
  });
}

sn_status sn_add_rmsnorm(const void* delta, float* residual, const void* weight, void* out, int rows,
                         int dim, float eps, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && dim > 0 && dim % 8 == 0, "sn_add_rmsnorm: bad shape rows=%d dim=%d", rows, dim);
  SN_REQUIRE(dim <= 8 * 256 * 4, "sn_add_rmsnorm: dim %d > 8192 unsupported", dim);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    const int threads = dim / 8 >= 256 ? 256 : ((dim / 8 + 31) / 32) * 32;
    add_rmsnorm_kernel<T, 4><<<rows, threads, 0, (cudaStream_t)stream>>>(
        (const T*)delta, residual, (const T*)weight, (T*)out, dim, eps);
    return check_launch("sn_add_rmsnorm");
  });
}

sn_status sn_silu_mul(const void* gate_up, void* out, int rows, int ffn, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && ffn > 0 && ffn % 8 == 0, "sn_silu_mul: bad shape rows=%d ffn=%d", rows, ffn);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    const size_t n8 = (size_t)rows * ffn / 8;
    int grid = (int)((n8 + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    silu_mul_kernel<T><<<grid, 256, 0, (cudaStream_t)stream>>>((const T*)gate_up, (T*)out, rows, ffn);
    return check_launch("sn_silu_mul");
  });
}

sn_status sn_argmax(const void* logits, int rows, int vocab, int32_t* out_tokens, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && vocab > 0 && vocab % 8 == 0, "sn_argmax: bad shape rows=%d vocab=%d", rows, vocab);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    argmax_kernel<T><<<rows, 1024, 0, (cudaStream_t)stream>>>((const T*)logits, vocab, out_tokens);
    return check_launch("sn_argmax");
  });
}

}  // extern "C"
