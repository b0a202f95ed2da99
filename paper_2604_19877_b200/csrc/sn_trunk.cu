// Shared-trunk kernels: embedding (+decode-step prologue), fused residual-add
// RMSNorm, SiLU-gated FFN activation, greedy argmax.  All HBM-bound, one pass
// over their operands, 16-byte vector loads.
//
// Trunk definition: R/PAPER.md:175-182 (Apriel-1.6: d=5120, SiLU-gated FFN
// 14336, vocab 131072), shared across mixers R/PAPER.md:855-856.
#include <stdarg.h>
#include <string.h>

#include <cooperative_groups.h>

#include "sn_common.cuh"

namespace cg = cooperative_groups;

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
                             const float* __restrict__ inv_freq, float2* __restrict__ rope_cs, int half, int rows,
                             int dim) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ int s_pos;
  const int r = blockIdx.x;
  const int tok = tokens[r];
  if (seq_lens != nullptr) {  // decode-step prologue: CTA r owns row r's bookkeeping
    if (threadIdx.x == 0) {
      int L = -1;  // idle slot (continuous batching): no position, the length stays
      if (tok >= 0) {
        L = seq_lens[r];
        seq_lens[r] = L + 1;
      }
      positions[r] = L;
      s_pos = L;
    }
    if (rope_cs != nullptr) {  // the step's rotary (cos, sin) per pair, for the fused in-projection epilogue
      __syncthreads();
      const int pos = s_pos;
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        float sn = 0.f, cs = 1.f;
        if (pos >= 0) sincosf((float)pos * inv_freq[t], &sn, &cs);
        rope_cs[(size_t)r * half + t] = make_float2(cs, sn);
      }
    }
  }
  float* dst = residual + (size_t)r * dim;
  if (tok < 0) {  // idle slot: a zero row (its outputs are ignored; nothing is appended)
    for (int i = threadIdx.x * 4; i < dim; i += blockDim.x * 4) *reinterpret_cast<float4*>(dst + i) = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const T* src = table + (size_t)tok * dim;
  for (int i = threadIdx.x * 8; i < dim; i += blockDim.x * 8) {
    float f[8];
    load8<T>(src + i, f);
    *reinterpret_cast<float4*>(dst + i) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(dst + i + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
}

// ------------------------------------------------------------------ add + rmsnorm
// A row is split across a thread-block cluster of CS CTAs (CS = 8 for d = 5120: 4 measured
// 35-40 us per decode step slower), each
// thread owning one 8-element chunk, so a 64-row decode batch runs as 512 CTAs instead
// of 64 long ones.  All of a chunk's inputs (residual, bf16 delta, up to 8 fp32 split-K
// slabs) are loaded in one batch before they are summed in a fixed order, the
// sum of squares is combined through distributed shared memory, and the chunk is
// normalised from registers.
constexpr int kNormMaxSplit = 8;

template <typename T>
__global__ void __launch_bounds__(256) add_rmsnorm_kernel(const T* __restrict__ delta,
                                                          const float* __restrict__ partials, int nsplit,
                                                          float* __restrict__ residual,
                                                          const T* __restrict__ weight,
                                                          T* __restrict__ out, int rows, int dim, float eps) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float scratch[32];
  __shared__ float cta_sum;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int part = (int)cluster.block_rank();
  const int r = blockIdx.x / CS;
  const int per_cta = dim / CS;
  const int i = part * per_cta + threadIdx.x * 8;
  const bool active = threadIdx.x * 8 < per_cta;
  float v[8];
  float ss = 0.f;
  if (active) {
    float* res = residual + (size_t)r * dim + i;
    float4 a = *reinterpret_cast<const float4*>(res);
    float4 b = *reinterpret_cast<const float4*>(res + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    if (delta != nullptr || nsplit > 0) {
      float d[8], p[kNormMaxSplit][8];
      if (delta != nullptr) load8<T>(delta + (size_t)r * dim + i, d);
#pragma unroll
      for (int s = 0; s < kNormMaxSplit; ++s)
        if (s < nsplit) load8<float>(partials + ((size_t)s * rows + r) * dim + i, p[s]);
      if (delta != nullptr) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += d[k];
      }
#pragma unroll
      for (int s = 0; s < kNormMaxSplit; ++s) {
        if (s < nsplit) {
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] += p[s][k];
        }
      }
      *reinterpret_cast<float4*>(res) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(res + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += v[k] * v[k];
  }
  ss = block_sum(ss, scratch);
  if (CS > 1) {
    if (threadIdx.x == 0) cta_sum = ss;
    cluster.sync();
    ss = 0.f;
    for (int q = 0; q < CS; ++q) ss += *cluster.map_shared_rank(&cta_sum, q);
    cluster.sync();  // keep every CTA's cta_sum alive until all ranks have read it
  }
  const float rstd = rsqrtf(ss / (float)dim + eps);
  if (active) {
    float w[8];
    load8<T>(weight + i, w);
#pragma unroll
    for (int k = 0; k < 8; ++k) io<T>::st(out + (size_t)r * dim + i + k, v[k] * rstd * w[k]);
  }
}

// Long-row-count variant (prefill): one CTA of 256 threads per row, each thread owning up to
// 4 chunks of 8 (dim <= 8192), no cluster; delta only (prefill has no split-K slabs).
template <typename T>
__global__ void __launch_bounds__(256) add_rmsnorm_rows_kernel(const T* __restrict__ delta,
                                                               float* __restrict__ residual,
                                                               const T* __restrict__ weight, T* __restrict__ out,
                                                               int dim, float eps) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float scratch[32];
  const int r = blockIdx.x;
  const int nch = dim / 8;
  float v[4][8];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int ch = threadIdx.x + c * 256;
    if (ch < nch) {
      float* res = residual + (size_t)r * dim + ch * 8;
      load8<float>(res, v[c]);
      if (delta != nullptr) {
        float d[8];
        load8<T>(delta + (size_t)r * dim + ch * 8, d);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[c][k] += d[k];
        *reinterpret_cast<float4*>(res) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
        *reinterpret_cast<float4*>(res + 4) = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += v[c][k] * v[c][k];
    }
  }
  ss = block_sum(ss, scratch);
  const float rstd = rsqrtf(ss / (float)dim + eps);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int ch = threadIdx.x + c * 256;
    if (ch < nch) {
      float w[8];
      load8<T>(weight + ch * 8, w);
      uint4 pk;
      uint32_t* pp = reinterpret_cast<uint32_t*>(&pk);
      if (sizeof(T) == 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(v[c][2 * k] * rstd * w[2 * k], v[c][2 * k + 1] * rstd * w[2 * k + 1]);
          pp[k] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(out + (size_t)r * dim + ch * 8) = pk;
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) io<T>::st(out + (size_t)r * dim + ch * 8 + k, v[c][k] * rstd * w[k]);
      }
    }
  }
}

// ------------------------------------------------------------------ silu * mul
// Interleaved gate/up layout (GEMM mode SWIGLU_IL weights, prefill GEMM output): row of
// ceil(ffn/h) blocks of [h gate | h up] columns.
template <typename T>
__global__ void swiglu_il_kernel(const T* __restrict__ gu, T* __restrict__ out, int rows, int ffn, int h, int ld) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  const size_t n8 = (size_t)rows * (ffn / 8);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n8; e += (size_t)gridDim.x * blockDim.x) {
    const size_t r = e / (ffn / 8);
    const int i = (int)(e % (ffn / 8)) * 8;
    const int b = i / h, o = i % h;  // h % 8 == 0: a chunk of 8 stays inside one block
    const T* row = gu + r * ld + (size_t)b * 2 * h + o;
    float g[8], u[8];
    load8<T>(row, g);
    load8<T>(row + h, u);
    if (sizeof(T) == 2) {  // one 16-byte store per 8 outputs
      uint4 pk;
      uint32_t* pp = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 b2 = __floats2bfloat162_rn(silu_f(g[2 * k]) * u[2 * k], silu_f(g[2 * k + 1]) * u[2 * k + 1]);
        pp[k] = *reinterpret_cast<uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(out + r * ffn + i) = pk;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) io<T>::st(out + r * ffn + i + k, silu_f(g[k]) * u[k]);
    }
  }
}

// ------------------------------------------------------------------ argmax
// A row is split across a cluster of CS CTAs (CS = 8 for the 131072-entry vocabulary: 512 CTAs
// for a 64-row batch instead of 64 long ones); each CTA reduces its slice, rank 0 combines the
// CS candidates through distributed shared memory.  Ties resolve to the lowest index at every
// level (deterministic, torch.argmax's first occurrence).
template <typename T>
__global__ void __launch_bounds__(256) argmax_kernel(const T* __restrict__ logits, int vocab, int per_cta,
                                                     int32_t* __restrict__ out, const int32_t* __restrict__ positions) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float sv[8];
  __shared__ int si[8];
  __shared__ float cta_v;
  __shared__ int cta_i;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks(), part = (int)cluster.block_rank();
  const int r = blockIdx.x / CS;
  const T* row = logits + (size_t)r * vocab;
  const int i0 = part * per_cta, i1 = min(vocab, i0 + per_cta);
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = i0 + threadIdx.x * 8; i < i1; i += blockDim.x * 8) {
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
    cta_v = best;
    cta_i = bi;
  }
  cluster.sync();
  if (part == 0 && threadIdx.x == 0) {
    for (int q = 1; q < CS; ++q) {
      const float v = *cluster.map_shared_rank(&cta_v, q);
      const int ix = *cluster.map_shared_rank(&cta_i, q);
      if (v > best || (v == best && ix < bi)) { best = v; bi = ix; }
    }
    // an all-NaN row never beats -inf: return token 0, never an out-of-range id that the
    // graph's token feedback would hand to the embedding gather
    out[r] = (positions && positions[r] < 0) ? -1 : (bi < vocab ? bi : 0);  // idle stays idle
  }
  cluster.sync();  // keep every CTA's candidate alive until rank 0 has read it
}

}  // namespace sn

using namespace sn;

extern "C" {

const char* sn_last_error(void) { return sn::g_err; }
int sn_abi_version(void) { return SN_ABI_VERSION; }

sn_status sn_embed(const int32_t* tokens, const void* table, float* residual, int32_t* seq_lens,
                   int32_t* positions, const float* inv_freq, void* rope_cs, int half, int rows, int dim, int dtype,
                   void* stream) {
  SN_REQUIRE(rows > 0 && dim > 0 && dim % 8 == 0, "sn_embed: bad shape rows=%d dim=%d", rows, dim);
  SN_REQUIRE((seq_lens == nullptr) == (positions == nullptr), "sn_embed: seq_lens/positions must be both set or both NULL");
  SN_REQUIRE(rope_cs == nullptr || (inv_freq != nullptr && half > 0 && seq_lens != nullptr),
             "sn_embed: the rotary table needs inv_freq, half > 0 and the decode prologue");
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    launch_pdl(embed_kernel<T>, dim3(rows), dim3(128), 0, (cudaStream_t)stream, tokens, (const T*)table, residual,
               seq_lens, positions, inv_freq, (float2*)rope_cs, half, rows, dim);
    return check_launch("sn_embed");
  });
}

sn_status sn_add_rmsnorm(const void* delta, const float* partials, int nsplit, float* residual, const void* weight,
                         void* out, int rows, int dim, float eps, int dtype, void* stream) {
  SN_REQUIRE(nsplit >= 0 && nsplit <= kNormMaxSplit && (nsplit == 0 || partials != nullptr),
             "sn_add_rmsnorm: bad partials (nsplit %d)", nsplit);
  SN_REQUIRE(rows > 0 && dim > 0 && dim % 8 == 0, "sn_add_rmsnorm: bad shape rows=%d dim=%d", rows, dim);
  if (rows > 512 && nsplit == 0 && dim <= 8192)  // prefill: a CTA per row, no cluster round trips
    return SN_DISPATCH_DTYPE(dtype, T, [&] {
      launch_pdl(add_rmsnorm_rows_kernel<T>, dim3(rows), dim3(256), 0, (cudaStream_t)stream, (const T*)delta,
                 residual, (const T*)weight, (T*)out, dim, eps);
      return check_launch("sn_add_rmsnorm");
    });
  // cluster size: each CTA owns <= 256 chunks of 8 (and >= 8-way split once rows are long)
  int cs = 1;
  while (cs < 8 && (dim / 8 / cs > 256 || (dim / 8 / cs > 64 && cs < 8)) && dim % (16 * cs) == 0) cs *= 2;
  SN_REQUIRE(dim / 8 / cs <= 256 && dim % (8 * cs) == 0, "sn_add_rmsnorm: dim %d unsupported", dim);
  const int per_cta = dim / cs;
  const int threads = ((per_cta / 8 + 31) / 32) * 32;
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rows * cs);
    cfg.blockDim = dim3(threads);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cs;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, add_rmsnorm_kernel<T>, (const T*)delta, partials, nsplit, residual,
                                       (const T*)weight, (T*)out, rows, dim, eps);
    if (e != cudaSuccess) {
      set_error("sn_add_rmsnorm launch: %s", cudaGetErrorString(e));
      return SN_ECUDA;
    }
    return check_launch("sn_add_rmsnorm");
  });
}

sn_status sn_swiglu_il(const void* gate_up, int ld, void* out, int rows, int ffn, int h, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && ffn > 0 && ffn % 8 == 0 && h > 0 && h % 8 == 0, "sn_swiglu_il: bad shape ffn=%d h=%d",
             ffn, h);
  SN_REQUIRE(ld >= ((ffn + h - 1) / h) * 2 * h && ld % 8 == 0, "sn_swiglu_il: ld %d too small", ld);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    const size_t n8 = (size_t)rows * (ffn / 8);
    int grid = (int)((n8 + 255) / 256);
    if (grid > 148 * 16) grid = 148 * 16;
    launch_pdl(swiglu_il_kernel<T>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const T*)gate_up, (T*)out, rows,
               ffn, h, ld);
    return check_launch("sn_swiglu_il");
  });
}

sn_status sn_argmax(const void* logits, int rows, int vocab, int32_t* out_tokens, const int32_t* positions, int dtype,
                    void* stream) {
  SN_REQUIRE(rows > 0 && vocab > 0 && vocab % 8 == 0, "sn_argmax: bad shape rows=%d vocab=%d", rows, vocab);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    int cs = 1;
    while (cs < 8 && vocab / (cs * 2) >= 8192) cs *= 2;  // >= 8K entries per CTA
    const int per_cta = ((vocab + cs * 8 - 1) / (cs * 8)) * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rows * cs);
    cfg.blockDim = dim3(256);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cs;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, argmax_kernel<T>, (const T*)logits, vocab, per_cta, out_tokens, positions);
    if (e != cudaSuccess) {
      set_error("sn_argmax launch: %s", cudaGetErrorString(e));
      return SN_ECUDA;
    }
    return check_launch("sn_argmax");
  });
}

}  // extern "C"
