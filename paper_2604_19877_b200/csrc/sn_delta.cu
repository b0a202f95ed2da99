// GDN / KDA gated delta-rule mixers (R/PAPER.md:1565-1625).
//
//   GDN: S_t = e^{g_t} (I - b_t k_t k_t^T) S_{t-1} + b_t k_t v_t^T       (scalar gate / value head)
//   KDA: S_t = (I - b_t k_t k_t^T) diag(e^{g_t}) S_{t-1} + b_t k_t v_t^T  (per-key-channel gate)
//   o_t = S_t^T q_t, then gated RMSNorm and the out-projection (a GEMM outside).
//
// Unstated details pinned from FLA 0.5.1: L2-norm
// x/sqrt(sum x^2 + 1e-6) (3P-FLA/modules/l2norm.py:40-43), q scaled by D^-1/2,
// gates g = -exp(A_log) * softplus(raw + dt_bias) (3P-FLA/ops/*/gate.py), beta =
// sigmoid, causal conv width 4 with SiLU (3P-FLA/modules/conv/short_conv.py:201-243),
// output norm RMSNorm(o) * w * act(gate) with act = silu (GDN) / sigmoid (KDA)
// (3P-FLA/modules/fused_norm_gate.py:94-100).
//
// Decode kernel (the hot path): one CTA per (value head, sequence).  The CTA
//   1. runs the conv update for its q/k/v channels against the per-sequence
//      conv ring (slot p % W holds the input of position p, so CTAs that share
//      a key head never race: they read slots != pos % W, one of them writes it),
//   2. L2-normalises q,k, computes the gate(s) and beta (KDA: the second
//      low-rank factors of the gate / output gate are fused here as 128x128
//      matvecs whose weights stay L2-resident across the batch),
//   3. streams the fp32 state once: every warp owns D/8 value columns; a
//      column's D key entries are one coalesced 512 B row (float4 per lane);
//      both dot products (k and q against the decayed state) are taken from the
//      same registers, using  q.S_new = (q*e^g).S + (q.k) u,
//   4. applies the gated RMSNorm over the head and writes bf16/fp32 output.
// The state is read once and written once: 2*D*D*4 bytes per (sequence, head).
#include <type_traits>

#include "sn_common.cuh"

namespace sn {

struct DeltaDecodeArgs {
  const void* proj;   // in-projection row [B][proj_stride] (sn_gemm_decode STORE output)
  int proj_stride;
  void* conv_ring;
  const void* conv_w;
  float* state;
  const int32_t* slot_idx;
  const int32_t* positions;
  const float* A_log;
  const float* dt_bias;
  const void* fg;     // KDA: [2][B][H*D] = (f1 @ f2^T, g1 @ g2^T), the second low-rank factors
  const void* g2_b;
  const void* norm_w;
  void* out;
  int Hk, Hv, rank, conv_channels;
  int B;  // batch (the GDN kernel's persistent item count is Hv * B)
  int q_off, k_off, v_off, z_off, b_off, a_off, f1_off, g1_off;
  float scale, eps_l2, eps_norm;
};

template <int EPL> struct vecf;
template <> struct vecf<4> {  // the recurrent state is streamed: evict-first loads and stores
  static __device__ __forceinline__ void ld(const float* p, float* v) {
    float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  static __device__ __forceinline__ void st(float* p, const float* v) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
};
template <> struct vecf<2> {
  static __device__ __forceinline__ void ld(const float* p, float* v) {
    float2 t = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = t.x; v[1] = t.y;
  }
  static __device__ __forceinline__ void st(float* p, const float* v) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  }
};

template <typename T> __device__ __forceinline__ void load4(const T* p, float* f);
template <> __device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
template <> __device__ __forceinline__ void load4<float>(const float* p, float* f) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}
// n (= 2 or 4) consecutive elements
template <typename T, int N> __device__ __forceinline__ void loadn(const T* p, float* f) {
  if (N == 4) {
    load4<T>(p, f);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) f[i] = io<T>::ld(p + i);
  }
}

// Three block-wide sums in one pass (scratch: 3 * blockDim.x/32 floats).  The caller
// guarantees no thread still reads `scratch` from an earlier use (no leading barrier).
__device__ __forceinline__ void block_sum3(float& x, float& y, float& z, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum(x);
  y = warp_sum(y);
  z = warp_sum(z);
  if (lane == 0) { scratch[warp] = x; scratch[nw + warp] = y; scratch[2 * nw + warp] = z; }
  __syncthreads();
  float tx = 0.f, ty = 0.f, tz = 0.f;
  for (int i = 0; i < nw; ++i) { tx += scratch[i]; ty += scratch[nw + i]; tz += scratch[2 * nw + i]; }
  x = tx;
  y = ty;
  z = tz;
}

constexpr int kDecodeThreads = 256;

__device__ __forceinline__ uint32_t dl_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Width-4 causal conv of one channel at position pos: the ring holds the inputs of
// positions pos-1..pos-3 at slots (pos-d) & 3; x is the new input.
__device__ __forceinline__ float conv4(const float* w, const float* ring, float x, int pos) {
  float acc = w[3] * x;
#pragma unroll
  for (int d = 1; d < 4; ++d)
    if (pos - d >= 0) acc += w[3 - d] * ring[(pos - d) & 3];
  return acc;
}

// N consecutive elements of T kept packed in 32-bit registers (bf16: two per register), loaded
// with 16-byte (or 8-byte) vector loads; element i comes back as float.
template <typename T, int N>
struct Packed {
  static constexpr int R = N * (int)sizeof(T) / 4;
  uint32_t r[R];
  __device__ __forceinline__ void load(const T* p) {
    if (R % 4 == 0) {
#pragma unroll
      for (int i = 0; i < R; i += 4) {
        const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(p) + i);
        r[i] = u.x; r[i + 1] = u.y; r[i + 2] = u.z; r[i + 3] = u.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; i += 2) {
        const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const uint32_t*>(p) + i);
        r[i] = u.x; r[i + 1] = u.y;
      }
    }
  }
  __device__ __forceinline__ float operator[](int i) const {  // i must be a compile-time constant
    if (sizeof(T) == 4) return __uint_as_float(r[i]);
    return __uint_as_float((i & 1) ? (r[i >> 1] & 0xffff0000u) : (r[i >> 1] << 16));
  }
};

// conv4 over channel e of a packed [channels][4] tap block and ring block, p = pos & 3 known
// at compile time (so every ring index is a register, not a local-memory array access).
template <int P, typename TP>
__device__ __forceinline__ float conv4p(const TP& w, const TP& ring, int e, float x, int pos) {
  float acc = w[4 * e + 3] * x;
  acc += pos >= 1 ? w[4 * e + 2] * ring[4 * e + ((P + 3) & 3)] : 0.f;
  acc += pos >= 2 ? w[4 * e + 1] * ring[4 * e + ((P + 2) & 3)] : 0.f;
  acc += pos >= 3 ? w[4 * e + 0] * ring[4 * e + ((P + 1) & 3)] : 0.f;
  return acc;
}

// ---------------------------------------------------------------------------------------
// GDN decode: one CTA per (value head h, sequence b), THREADS/32 warps; lane l of every warp
// owns key entries [l*EPL, +EPL) of the head, warp w owns value columns [w*CPW, +CPW).
//
// Barrier-free prologue: every warp computes, in registers, exactly what it needs —
// the conv + SiLU of its lanes' EPL q and k channels (all D key entries across the warp, so
// |q|^2, |k|^2 and q.k are warp shuffles) and of its own CPW v channels (lane j < CPW holds
// v of column w*CPW + j) — so no block barrier sits between griddepcontrol.wait and the
// state stream.  The conv taps, the ring slots and the first state columns are requested
// before griddepcontrol.wait (none depends on the in-projection); only the projection row
// itself is loaded after it.  The state is then streamed once, software-pipelined (NB columns
// in flight per warp): both dot products come from the same registers using
// q.S_new = (q*e^g).S + (q.k) u, and each new column is stored immediately.  One barrier at
// the end gathers o for the gated RMSNorm over the head.
template <typename T, int D, int THREADS = kDecodeThreads>
__global__ void __launch_bounds__(THREADS, THREADS == kDecodeThreads ? 4 : 1)
    gdn_decode_kernel(const DeltaDecodeArgs a) {
  sn::pdl_launch_dependents();
  constexpr int NW = THREADS / 32;
  constexpr int EPL = D / 32;     // key entries per lane
  constexpr int CPW = D / NW;     // value columns per warp
  constexpr int NB = 4;           // columns in flight per warp
  static_assert(CPW % NB == 0 && CPW <= 32, "columns per warp");
  __shared__ __align__(16) float s_o[D];
  __shared__ float s_red[NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = a.Hv / a.Hk;
  const int items = a.Hv * a.B;
  // items (value head, sequence) = blockIdx.x, + gridDim.x, ...; with a smaller grid the first
  // state columns of the next item are requested before this item's norm epilogue (the launch
  // uses one item per CTA: measured faster, see launch_delta_decode_t)
  int item = blockIdx.x;
  if (item >= items) return;
  int h = item % a.Hv, b = item / a.Hv;
  int slot = a.slot_idx ? a.slot_idx[b] : b;
  float* S = a.state + ((size_t)slot * a.Hv + h) * D * D;
  float s_nx[NB][EPL];
#pragma unroll
  for (int n = 0; n < NB; ++n) vecf<EPL>::ld(S + (size_t)(warp * CPW + n) * D + lane * EPL, s_nx[n]);
  const T* nwp = reinterpret_cast<const T*>(a.norm_w);
  const float nw = tid < D ? io<T>::ld(nwp + tid) : 0.f;
  const T* cw = reinterpret_cast<const T*>(a.conv_w);
  asm volatile("griddepcontrol.wait;" ::: "memory");

#pragma unroll 1
  for (;;) {
    const int kh = h / G;
    const int next = item + gridDim.x;
    // ---- the in-projection row and the ring slots (this layer's previous step): this lane's
    //      q, k, v inputs, the output gate z, a, b; the conv taps (L2-resident weights)
    const int pos = a.positions[b];
    T* ring = reinterpret_cast<T*>(a.conv_ring) + (size_t)slot * a.conv_channels * 4;
    const int qch = a.q_off + kh * D + lane * EPL, kch = a.k_off + kh * D + lane * EPL;
    const int vcol = warp * CPW + (lane < CPW ? lane : 0);
    const int vch = a.v_off + h * D + vcol;
    const T* prow = reinterpret_cast<const T*>(a.proj) + (size_t)b * a.proj_stride;
    if (pos >= 0) {  // (idle slot, sn_embed: state and conv ring untouched)
      Packed<T, 4 * EPL> rgq, rgk, wq, wk;
      Packed<T, 4> rgv, wv;
      rgq.load(ring + (size_t)qch * 4);
      rgk.load(ring + (size_t)kch * 4);
      rgv.load(ring + (size_t)vch * 4);
      float xq[EPL], xk[EPL];
      loadn<T, EPL>(prow + qch, xq);
      loadn<T, EPL>(prow + kch, xk);
      const float xv = io<T>::ld(prow + vch);
      const float zval = tid < D ? io<T>::ld(prow + a.z_off + h * D + tid) : 0.f;
      const float braw = io<T>::ld(prow + a.b_off + h);
      const float graw = io<T>::ld(prow + a.a_off + h) + a.dt_bias[h];
      const float negA = -expf(a.A_log[h]);
      wq.load(cw + (size_t)qch * 4);
      wk.load(cw + (size_t)kch * 4);
      wv.load(cw + (size_t)vch * 4);

      // ---- conv + SiLU in registers; ring slot pos % 4 takes the new input (q/k channels are
      //      shared by the G value heads of a key head: the first of them writes)
      float qv[EPL], kv[EPL], vv = 0.f;
      auto conv_all = [&](auto P) {
        constexpr int p = decltype(P)::value;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          qv[e] = silu_f(conv4p<p>(wq, rgq, e, xq[e], pos));
          kv[e] = silu_f(conv4p<p>(wk, rgk, e, xk[e], pos));
        }
        vv = silu_f(conv4p<p>(wv, rgv, 0, xv, pos));
      };
      switch (pos & 3) {
        case 0: conv_all(std::integral_constant<int, 0>{}); break;
        case 1: conv_all(std::integral_constant<int, 1>{}); break;
        case 2: conv_all(std::integral_constant<int, 2>{}); break;
        default: conv_all(std::integral_constant<int, 3>{}); break;
      }
      if ((h % G) == 0 && warp == 0) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          io<T>::st(ring + (size_t)(qch + e) * 4 + (pos & 3), xq[e]);
          io<T>::st(ring + (size_t)(kch + e) * 4 + (pos & 3), xk[e]);
        }
      }
      if (lane < CPW) io<T>::st(ring + (size_t)vch * 4 + (pos & 3), xv);

      // ---- L2 norms and q.k by warp shuffles (every warp holds all D entries of q and k)
      float qq = 0.f, kk = 0.f, qkr = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        qq += qv[e] * qv[e];
        kk += kv[e] * kv[e];
        qkr += qv[e] * kv[e];
      }
      qq = warp_sum(qq);
      kk = warp_sum(kk);
      qkr = warp_sum(qkr);
      const float rq = rsqrtf(qq + a.eps_l2) * a.scale, rk = rsqrtf(kk + a.eps_l2);
      const float eg = expf(negA * softplus_f(graw));
      const float beta = sigmoid_f(braw);
      const float qk = qkr * rq * rk;
      float kr[EPL], kg[EPL], qg[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        kr[e] = kv[e] * rk;
        kg[e] = kr[e] * eg;
        qg[e] = qv[e] * rq * eg;
      }

      // ---- stream the state; the last batch's registers then take the next item's first columns
#pragma unroll 1
      for (int j0 = 0; j0 < CPW; j0 += NB) {
        const int c0 = warp * CPW + j0;
        float s[NB][EPL];
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
          for (int e = 0; e < EPL; ++e) s[n][e] = s_nx[n][e];
        if (j0 + NB < CPW) {
#pragma unroll
          for (int n = 0; n < NB; ++n) vecf<EPL>::ld(S + (size_t)(c0 + NB + n) * D + lane * EPL, s_nx[n]);
        } else if (next < items) {
          const int hn = next % a.Hv, bn = next / a.Hv;
          const int sn_ = a.slot_idx ? a.slot_idx[bn] : bn;
          const float* Sn = a.state + ((size_t)sn_ * a.Hv + hn) * D * D;
#pragma unroll
          for (int n = 0; n < NB; ++n) vecf<EPL>::ld(Sn + (size_t)(warp * CPW + n) * D + lane * EPL, s_nx[n]);
        }
        float kd[NB], qd[NB];
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          kd[n] = 0.f;
          qd[n] = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) {
            kd[n] += kg[e] * s[n][e];
            qd[n] += qg[e] * s[n][e];
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
          for (int n = 0; n < NB; ++n) {
            kd[n] += __shfl_xor_sync(0xffffffffu, kd[n], o);
            qd[n] += __shfl_xor_sync(0xffffffffu, qd[n], o);
          }
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
          const float vcn = __shfl_sync(0xffffffffu, vv, j0 + n);
          const float u = beta * (vcn - kd[n]);
#pragma unroll
          for (int e = 0; e < EPL; ++e) s[n][e] = eg * s[n][e] + kr[e] * u;
          vecf<EPL>::st(S + (size_t)(c0 + n) * D + lane * EPL, s[n]);
          if (lane == 0) s_o[c0 + n] = qd[n] + qk * u;
        }
      }
      __syncthreads();

      // ---- gated RMSNorm over the head: out = RMSNorm(o) * w * silu(z)
      float oo = 0.f;
      for (int j = tid; j < D; j += THREADS) oo += s_o[j] * s_o[j];
      oo = warp_sum(oo);
      if (lane == 0) s_red[warp] = oo;
      __syncthreads();
      oo = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) oo += s_red[w];
      const float rstd = rsqrtf(oo / (float)D + a.eps_norm);
      if (tid < D) {
        T* out = reinterpret_cast<T*>(a.out) + (size_t)b * a.Hv * D + (size_t)h * D;
        io<T>::st(out + tid, s_o[tid] * rstd * nw * silu_f(zval));
      }
      __syncthreads();  // s_o / s_red are reused by the next item
    } else if (next < items) {  // idle slot: still hand the next item its first columns
      const int hn = next % a.Hv, bn = next / a.Hv;
      const int sn_ = a.slot_idx ? a.slot_idx[bn] : bn;
      const float* Sn = a.state + ((size_t)sn_ * a.Hv + hn) * D * D;
#pragma unroll
      for (int n = 0; n < NB; ++n) vecf<EPL>::ld(Sn + (size_t)(warp * CPW + n) * D + lane * EPL, s_nx[n]);
    }
    if (next >= items) break;
    item = next;
    h = item % a.Hv;
    b = item / a.Hv;
    slot = a.slot_idx ? a.slot_idx[b] : b;
    S = a.state + ((size_t)slot * a.Hv + h) * D * D;
  }
}

// ---------------------------------------------------------------------------------------
// GDN decode, D = 128, state staged through shared memory with cp.async: every warp keeps
// NBUF - 1 batches of NB columns in flight in its own smem ring (lane l copies and later reads
// its own 16-byte slice of each column, so no barrier is needed), the conv / norm / gate prologue
// running under the first batches' latency.  Measured at B=64 (tools/bench_delta.py): 45.0 us
// vs 48.0 for the register pipeline (gdn_decode_kernel, kept for D = 64 and the 512-thread
// small-batch CTAs), and the decode step 10.23 -> 9.77 ms; NBUF = 3 measured 46.0 us.
// One CTA (8 warps) per (value head, sequence).
template <typename T, int NBUF>
__global__ void __launch_bounds__(kDecodeThreads, 4) gdn_decode_cpa_kernel(const DeltaDecodeArgs a) {
  sn::pdl_launch_dependents();
  constexpr int D = 128, THREADS = kDecodeThreads, NW = THREADS / 32;
  constexpr int EPL = D / 32, CPW = D / NW, NB = 4, NBATCH = CPW / NB;
  static_assert(EPL == 4 && NBATCH >= NBUF - 1, "cp.async staging assumes 16-byte lane slices");
  extern __shared__ __align__(16) float ring_all[];  // [NW][NBUF][NB][D]
  __shared__ __align__(16) float s_o[D];
  __shared__ float s_red[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = a.Hv / a.Hk;
  const int h = blockIdx.x % a.Hv, b = blockIdx.x / a.Hv;
  const int slot = a.slot_idx ? a.slot_idx[b] : b;
  float* S = a.state + ((size_t)slot * a.Hv + h) * D * D;
  float* ring = ring_all + (size_t)warp * NBUF * NB * D;
  auto issue = [&](int jb) {  // batch jb of this warp's columns -> ring slot jb % NBUF
    float* dst = ring + (jb % NBUF) * NB * D + lane * EPL;
    const float* src = S + (size_t)(warp * CPW + jb * NB) * D + lane * EPL;
#pragma unroll
    for (int n = 0; n < NB; ++n)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dl_smem_u32(dst + n * D)), "l"(src + (size_t)n * D)
                   : "memory");
  };
#pragma unroll
  for (int jb = 0; jb < NBUF - 1; ++jb) {
    issue(jb);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const T* nwp = reinterpret_cast<const T*>(a.norm_w);
  const float nw = tid < D ? io<T>::ld(nwp + tid) : 0.f;
  const T* cw = reinterpret_cast<const T*>(a.conv_w);
  const int kh = h / G;
  T* ring_c = reinterpret_cast<T*>(a.conv_ring) + (size_t)slot * a.conv_channels * 4;
  const int qch = a.q_off + kh * D + lane * EPL, kch = a.k_off + kh * D + lane * EPL;
  const int vcol = warp * CPW + (lane < CPW ? lane : 0);
  const int vch = a.v_off + h * D + vcol;
  Packed<T, 4 * EPL> rgq, rgk, wq, wk;
  Packed<T, 4> rgv, wv;
  rgq.load(ring_c + (size_t)qch * 4);
  rgk.load(ring_c + (size_t)kch * 4);
  rgv.load(ring_c + (size_t)vch * 4);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int pos = a.positions[b];
  if (pos < 0) {  // idle slot (sn_embed): state and conv ring untouched
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  // the conv taps (L2-resident weights) in the same round trip as the projection row
  wq.load(cw + (size_t)qch * 4);
  wk.load(cw + (size_t)kch * 4);
  wv.load(cw + (size_t)vch * 4);
  const float negA = -expf(a.A_log[h]);
  const float dtb = a.dt_bias[h];
  const T* prow = reinterpret_cast<const T*>(a.proj) + (size_t)b * a.proj_stride;
  float xq[EPL], xk[EPL];
  loadn<T, EPL>(prow + qch, xq);
  loadn<T, EPL>(prow + kch, xk);
  const float xv = io<T>::ld(prow + vch);
  const float zval = tid < D ? io<T>::ld(prow + a.z_off + h * D + tid) : 0.f;
  const float braw = io<T>::ld(prow + a.b_off + h);
  const float graw = io<T>::ld(prow + a.a_off + h) + dtb;
  float qv[EPL], kv[EPL], vv = 0.f;
  auto conv_all = [&](auto P) {
    constexpr int p = decltype(P)::value;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      qv[e] = silu_f(conv4p<p>(wq, rgq, e, xq[e], pos));
      kv[e] = silu_f(conv4p<p>(wk, rgk, e, xk[e], pos));
    }
    vv = silu_f(conv4p<p>(wv, rgv, 0, xv, pos));
  };
  switch (pos & 3) {
    case 0: conv_all(std::integral_constant<int, 0>{}); break;
    case 1: conv_all(std::integral_constant<int, 1>{}); break;
    case 2: conv_all(std::integral_constant<int, 2>{}); break;
    default: conv_all(std::integral_constant<int, 3>{}); break;
  }
  if ((h % G) == 0 && warp == 0) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      io<T>::st(ring_c + (size_t)(qch + e) * 4 + (pos & 3), xq[e]);
      io<T>::st(ring_c + (size_t)(kch + e) * 4 + (pos & 3), xk[e]);
    }
  }
  if (lane < CPW) io<T>::st(ring_c + (size_t)vch * 4 + (pos & 3), xv);
  float qq = 0.f, kk = 0.f, qkr = 0.f;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    qq += qv[e] * qv[e];
    kk += kv[e] * kv[e];
    qkr += qv[e] * kv[e];
  }
  qq = warp_sum(qq);
  kk = warp_sum(kk);
  qkr = warp_sum(qkr);
  const float rq = rsqrtf(qq + a.eps_l2) * a.scale, rk = rsqrtf(kk + a.eps_l2);
  const float eg = expf(negA * softplus_f(graw));
  const float beta = sigmoid_f(braw);
  const float qk = qkr * rq * rk;
  float kr[EPL], kg[EPL], qg[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    kr[e] = kv[e] * rk;
    kg[e] = kr[e] * eg;
    qg[e] = qv[e] * rq * eg;
  }
#pragma unroll 1
  for (int jb = 0; jb < NBATCH; ++jb) {
    if (jb + NBUF - 1 < NBATCH) issue(jb + NBUF - 1);  // its slot was read in iteration jb - 1
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NBUF - 1) : "memory");
    const int c0 = warp * CPW + jb * NB;
    const float* src = ring + (jb % NBUF) * NB * D + lane * EPL;
    float s[NB][EPL];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float4 t = *reinterpret_cast<const float4*>(src + n * D);
      s[n][0] = t.x; s[n][1] = t.y; s[n][2] = t.z; s[n][3] = t.w;
    }
    float kd[NB], qd[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      kd[n] = 0.f;
      qd[n] = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        kd[n] += kg[e] * s[n][e];
        qd[n] += qg[e] * s[n][e];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        kd[n] += __shfl_xor_sync(0xffffffffu, kd[n], o);
        qd[n] += __shfl_xor_sync(0xffffffffu, qd[n], o);
      }
    }
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float vcn = __shfl_sync(0xffffffffu, vv, jb * NB + n);
      const float u = beta * (vcn - kd[n]);
#pragma unroll
      for (int e = 0; e < EPL; ++e) s[n][e] = eg * s[n][e] + kr[e] * u;
      vecf<EPL>::st(S + (size_t)(c0 + n) * D + lane * EPL, s[n]);
      if (lane == 0) s_o[c0 + n] = qd[n] + qk * u;
    }
  }
  __syncthreads();
  float oo = 0.f;
  for (int j = tid; j < D; j += THREADS) oo += s_o[j] * s_o[j];
  oo = warp_sum(oo);
  if (lane == 0) s_red[warp] = oo;
  __syncthreads();
  oo = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) oo += s_red[w];
  const float rstd = rsqrtf(oo / (float)D + a.eps_norm);
  if (tid < D) {
    T* out = reinterpret_cast<T*>(a.out) + (size_t)b * a.Hv * D + (size_t)h * D;
    io<T>::st(out + tid, s_o[tid] * rstd * nw * silu_f(zval));
  }
}

// ---------------------------------------------------------------------------------------
// KDA decode: one CTA per (head, sequence).  The CTA
//   1. runs the conv update of its q/k/v channels against the per-sequence conv ring
//      (KDA heads are not shared: the CTA owns its channels' ring slots),
//   2. L2-normalises q,k, takes the per-channel gate and the output gate from the second
//      low-rank factors (f = f1 @ f2^T, g1 @ g2^T: two decode GEMMs before this kernel,
//      fg = [2][B][H*D]) and beta,
//   3. streams the fp32 state once as in the GDN kernel, with per-key-channel decays,
//   4. applies the gated RMSNorm (sigmoid gate).
template <typename T, int D, int THREADS = kDecodeThreads, bool CPA = false>
__global__ void __launch_bounds__(THREADS, THREADS == kDecodeThreads ? 4 : 1)
    kda_decode_kernel(const DeltaDecodeArgs a) {
  sn::pdl_launch_dependents();
  constexpr int NW = THREADS / 32;
  constexpr int EPL = D / 32;
  constexpr int CPW = D / NW;
  constexpr int NB = 4;
  static_assert(CPW % NB == 0, "columns per warp must be a multiple of NB");

  __shared__ __align__(16) float s_q[D];
  __shared__ __align__(16) float s_k[D];
  __shared__ __align__(16) float s_v[D];
  __shared__ __align__(16) float s_eg[D];
  __shared__ __align__(16) float s_gate[D];
  __shared__ __align__(16) float s_o[D];
  __shared__ float s_red[3 * NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int h = blockIdx.x, b = blockIdx.y;
  const int slot = a.slot_idx ? a.slot_idx[b] : b;
  float* S = a.state + ((size_t)slot * a.Hv + h) * D * D;
  // CPA (D = 128, 256 threads): the state batches are staged through a per-warp shared-memory
  // ring with cp.async (as gdn_decode_cpa_kernel: one batch in flight, no registers held);
  // otherwise the next batch waits in registers
  extern __shared__ __align__(16) float kring_all[];  // CPA: [NW][2][NB][D]
  float* kring = kring_all + (size_t)warp * 2 * NB * D;
  auto issue = [&](int c0, int sl) {
    if constexpr (CPA) {
#pragma unroll
      for (int n = 0; n < NB; ++n)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dl_smem_u32(kring + (sl * NB + n) * D + lane * EPL)),
                     "l"(S + (size_t)(c0 + n) * D + lane * EPL)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  float s_nx[NB][EPL];
  if constexpr (CPA) {
    issue(warp * CPW, 0);
  } else {
#pragma unroll
    for (int n = 0; n < NB; ++n) vecf<EPL>::ld(S + (size_t)(warp * CPW + n) * D + lane * EPL, s_nx[n]);
  }
  T* ring = reinterpret_cast<T*>(a.conv_ring) + (size_t)slot * a.conv_channels * 4;
  const T* cw = reinterpret_cast<const T*>(a.conv_w);
  constexpr int NCH = (3 * D + THREADS - 1) / THREADS;
  float xin[NCH], wt[NCH][4], rg[NCH][4];
  int chn[NCH];
#pragma unroll
  for (int u = 0; u < NCH; ++u) {
    const int c = tid + u * THREADS;
    chn[u] = -1;
    if (c < 3 * D) {
      const int part = c / D, i = c - part * D;
      const int ch = (part == 0 ? a.q_off : part == 1 ? a.k_off : a.v_off) + h * D + i;
      chn[u] = ch;
      load4<T>(cw + (size_t)ch * 4, wt[u]);
      load4<T>(ring + (size_t)ch * 4, rg[u]);
    }
  }
  const float negA = -expf(a.A_log[h]);
  float dtb = 0.f, g2b = 0.f;
  if (tid < D) {
    dtb = a.dt_bias[h * D + tid];
    g2b = io<T>::ld(reinterpret_cast<const T*>(a.g2_b) + h * D + tid);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int pos = a.positions[b];
  if (pos < 0) {  // idle slot (sn_embed): state and conv ring untouched
    if constexpr (CPA) asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  const T* prow = reinterpret_cast<const T*>(a.proj) + (size_t)b * a.proj_stride;

  // ---- 1. prologue loads of the in-projection row and the gate factors, all issued first
#pragma unroll
  for (int u = 0; u < NCH; ++u)
    if (chn[u] >= 0) xin[u] = io<T>::ld(prow + chn[u]);
  float fpre = 0.f, gpre = 0.f;
  if (tid < D) {
    const size_t HD = (size_t)a.Hv * D;
    const T* fgp = reinterpret_cast<const T*>(a.fg) + (size_t)b * 2 * HD + h * D + tid;  // [B][f | g]
    fpre = io<T>::ld(fgp) + dtb;
    gpre = io<T>::ld(fgp + HD) + g2b;
  }
  const float braw = io<T>::ld(prow + a.b_off + h);

  // ---- 2. conv + SiLU
#pragma unroll
  for (int u = 0; u < NCH; ++u) {
    if (chn[u] < 0) continue;
    const int c = tid + u * THREADS;
    const int part = c / D, i = c - part * D;
    const float acc = conv4(wt[u], rg[u], xin[u], pos);
    io<T>::st(ring + (size_t)chn[u] * 4 + (pos & 3), xin[u]);
    (part == 0 ? s_q : part == 1 ? s_k : s_v)[i] = silu_f(acc);
  }
  if (tid < D) {
    s_eg[tid] = expf(negA * softplus_f(fpre));
    s_gate[tid] = gpre;
  }
  __syncthreads();

  // ---- 3. L2 norms and the q.k product of the raw vectors (one three-value reduction), beta
  float qq = 0.f, kk = 0.f, qkr = 0.f;
  for (int i = tid; i < D; i += THREADS) {
    qq += s_q[i] * s_q[i];
    kk += s_k[i] * s_k[i];
    qkr += s_q[i] * s_k[i];
  }
  block_sum3(qq, kk, qkr, s_red);
  const float rq = rsqrtf(qq + a.eps_l2) * a.scale, rk = rsqrtf(kk + a.eps_l2);
  const float beta = sigmoid_f(braw);
  const float qk = qkr * rq * rk;

  // ---- 3. stream the state: warp owns columns [warp*CPW, +CPW), lane owns keys [lane*EPL, +EPL)
  float kr[EPL], eg[EPL], kg[EPL], qg[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int i = lane * EPL + e;
    kr[e] = s_k[i] * rk;
    eg[e] = s_eg[i];
    kg[e] = kr[e] * eg[e];
    qg[e] = s_q[i] * rq * eg[e];
  }
#pragma unroll 1
  for (int c0 = warp * CPW; c0 < (warp + 1) * CPW; c0 += NB) {
    float s[NB][EPL];
    if constexpr (CPA) {
      const int sl = ((c0 - warp * CPW) / NB) & 1;
      if (c0 + NB < (warp + 1) * CPW) issue(c0 + NB, sl ^ 1);  // that slot was read last iteration
      else asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        const float4 t = *reinterpret_cast<const float4*>(kring + (sl * NB + n) * D + lane * EPL);
        s[n][0] = t.x; s[n][1] = t.y; s[n][2] = t.z; s[n][3] = t.w;
      }
    } else {
#pragma unroll
      for (int n = 0; n < NB; ++n)
#pragma unroll
        for (int e = 0; e < EPL; ++e) s[n][e] = s_nx[n][e];
      if (c0 + NB < (warp + 1) * CPW) {
#pragma unroll
        for (int n = 0; n < NB; ++n) vecf<EPL>::ld(S + (size_t)(c0 + NB + n) * D + lane * EPL, s_nx[n]);
      }
    }
    float kd[NB], qd[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      kd[n] = 0.f;
      qd[n] = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        kd[n] += kg[e] * s[n][e];
        qd[n] += qg[e] * s[n][e];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        kd[n] += __shfl_xor_sync(0xffffffffu, kd[n], o);
        qd[n] += __shfl_xor_sync(0xffffffffu, qd[n], o);
      }
    }
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const float u = beta * (s_v[c0 + n] - kd[n]);
#pragma unroll
      for (int e = 0; e < EPL; ++e) s[n][e] = eg[e] * s[n][e] + kr[e] * u;
      vecf<EPL>::st(S + (size_t)(c0 + n) * D + lane * EPL, s[n]);
      if (lane == 0) s_o[c0 + n] = qd[n] + qk * u;
    }
  }
  __syncthreads();

  // ---- 4. gated RMSNorm over the head
  float oo = 0.f;
  for (int j = tid; j < D; j += THREADS) oo += s_o[j] * s_o[j];
  oo = warp_sum(oo);
  if (lane == 0) s_red[warp] = oo;
  __syncthreads();
  oo = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) oo += s_red[w];
  const float rstd = rsqrtf(oo / (float)D + a.eps_norm);
  const T* nwp = reinterpret_cast<const T*>(a.norm_w);
  T* out = reinterpret_cast<T*>(a.out) + (size_t)b * a.Hv * D + (size_t)h * D;
  for (int j = tid; j < D; j += THREADS) io<T>::st(out + j, s_o[j] * rstd * io<T>::ld(nwp + j) * sigmoid_f(s_gate[j]));
}

// =====================================================================
// Prefill building blocks (sequences packed by cu_seqlens).

// Causal conv + SiLU over time.  Thread per (channel, time chunk of 64).
template <typename T>
__global__ void conv_prefill_kernel(const T* __restrict__ x, int x_stride, T* __restrict__ y,
                                    const T* __restrict__ w, T* __restrict__ ring, const T* __restrict__ ring_hist,
                                    const int32_t* __restrict__ cu, const int32_t* __restrict__ slot_idx,
                                    const int32_t* __restrict__ pos0s, int channels, int W) {
  constexpr int CH = 64;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int s = blockIdx.z;
  if (c >= channels) return;
  const int t0 = cu[s], L = cu[s + 1] - t0;
  const int p0 = blockIdx.y * CH;
  if (p0 >= L) return;
  const int p1 = min(p0 + CH, L);
  // continuation: the prompt starts at absolute position pos0; inputs before it come from a
  // copy of the ring taken before this launch (the last chunk rewrites the ring)
  const int pos0 = pos0s ? pos0s[s] : 0;
  auto before = [&](int p) -> float {  // input at chunk-relative position p < 0
    const int P = pos0 + p;
    if (P < 0 || ring_hist == nullptr) return 0.f;
    return io<T>::ld(ring_hist + ((size_t)s * channels + c) * W + (P % W));
  };
  if (W == 4) {  // the pinned width: taps and history in registers, loads batched by 8
    float w4[4];
    load4<T>(w + (size_t)c * 4, w4);
    const T* xc = x + (size_t)t0 * x_stride + c;
    float h1 = p0 >= 1 ? io<T>::ld(xc + (size_t)(p0 - 1) * x_stride) : before(p0 - 1);
    float h2 = p0 >= 2 ? io<T>::ld(xc + (size_t)(p0 - 2) * x_stride) : before(p0 - 2);
    float h3 = p0 >= 3 ? io<T>::ld(xc + (size_t)(p0 - 3) * x_stride) : before(p0 - 3);
    for (int p = p0; p < p1; p += 8) {
      float xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = p + u < p1 ? io<T>::ld(xc + (size_t)(p + u) * x_stride) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (p + u < p1) {
          const float acc = w4[3] * xv[u] + w4[2] * h1 + w4[1] * h2 + w4[0] * h3;
          io<T>::st(y + (size_t)(t0 + p + u) * channels + c, silu_f(acc));
        }
        h3 = h2; h2 = h1; h1 = xv[u];
      }
    }
  } else {
  float wt[8];
  for (int d = 0; d < W; ++d) wt[d] = io<T>::ld(w + (size_t)c * W + d);
  float hist[8];  // hist[d] = x at position p-1-d
  for (int d = 0; d < W - 1; ++d) {
    const int p = p0 - 1 - d;
    hist[d] = p >= 0 ? io<T>::ld(x + (size_t)(t0 + p) * x_stride + c) : before(p);
  }
  for (int p = p0; p < p1; ++p) {
    const float xv = io<T>::ld(x + (size_t)(t0 + p) * x_stride + c);
    float acc = wt[W - 1] * xv;
    for (int d = 1; d < W; ++d) acc += wt[W - 1 - d] * hist[d - 1];
    io<T>::st(y + (size_t)(t0 + p) * channels + c, silu_f(acc));
    for (int d = W - 2; d > 0; --d) hist[d] = hist[d - 1];
    if (W > 1) hist[0] = xv;
  }
  }
  if (p1 == L) {  // the chunk holding the last position leaves the ring for decode
    const int slot = slot_idx ? slot_idx[s] : s;
    T* rrow = ring + ((size_t)slot * channels + c) * W;
    for (int d = 1; d < W; ++d) {
      const int p = L - d;
      const float v = p >= 0 ? io<T>::ld(x + (size_t)(t0 + p) * x_stride + c) : before(p);
      const int P = pos0 + p;
      io<T>::st(rrow + (((P % W) + W) % W), v);
    }
  }
}

// bf16, width 4, even channel count / stride: two adjacent channels per thread (bf16x2 loads
// and stores: a warp moves 128 B per access instead of 64), same math as conv_prefill_kernel.
__global__ void conv4_prefill_bf16x2_kernel(const __nv_bfloat16* __restrict__ x, int x_stride,
                                            __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ w,
                                            __nv_bfloat16* __restrict__ ring,
                                            const __nv_bfloat16* __restrict__ ring_hist,
                                            const int32_t* __restrict__ cu, const int32_t* __restrict__ slot_idx,
                                            const int32_t* __restrict__ pos0s, int channels) {
  constexpr int CH = 64, W = 4;
  const int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int s = blockIdx.z;
  if (c >= channels) return;
  const int t0 = cu[s], L = cu[s + 1] - t0;
  const int p0 = blockIdx.y * CH;
  if (p0 >= L) return;
  const int p1 = min(p0 + CH, L);
  const int pos0 = pos0s ? pos0s[s] : 0;
  auto ld2 = [&](int p) -> float2 {  // inputs of channels c, c+1 at chunk-relative position p
    if (p >= 0) return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(x + (size_t)(t0 + p) * x_stride + c));
    const int P = pos0 + p;
    if (P < 0 || ring_hist == nullptr) return make_float2(0.f, 0.f);
    const __nv_bfloat16* hr = ring_hist + ((size_t)s * channels + c) * W + (P % W);
    return make_float2(__bfloat162float(hr[0]), __bfloat162float(hr[W]));
  };
  float wa[4], wb[4];
  load4<__nv_bfloat16>(w + (size_t)c * 4, wa);
  load4<__nv_bfloat16>(w + (size_t)(c + 1) * 4, wb);
  float2 h1 = ld2(p0 - 1), h2 = ld2(p0 - 2), h3 = ld2(p0 - 3);
  for (int p = p0; p < p1; p += 8) {
    float2 xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = p + u < p1 ? ld2(p + u) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (p + u < p1) {
        const float a0 = wa[3] * xv[u].x + wa[2] * h1.x + wa[1] * h2.x + wa[0] * h3.x;
        const float a1 = wb[3] * xv[u].y + wb[2] * h1.y + wb[1] * h2.y + wb[0] * h3.y;
        *reinterpret_cast<__nv_bfloat162*>(y + (size_t)(t0 + p + u) * channels + c) =
            __floats2bfloat162_rn(silu_f(a0), silu_f(a1));
      }
      h3 = h2; h2 = h1; h1 = xv[u];
    }
  }
  if (p1 == L) {  // the chunk holding the last position leaves the ring for decode
    const int slot = slot_idx ? slot_idx[s] : s;
    __nv_bfloat16* rrow = ring + ((size_t)slot * channels + c) * W;
    for (int d = 1; d < W; ++d) {
      const int p = L - d;
      const float2 v = ld2(p);
      const int P = pos0 + p, k = ((P % W) + W) % W;
      rrow[k] = __float2bfloat16_rn(v.x);
      rrow[W + k] = __float2bfloat16_rn(v.y);
    }
  }
}

// Per (row, key head): l2-normalised q/k (computed once per key head), then exp(gate),
// log gate and beta of the G = Hv/Hk value heads that read it.
template <typename T, int D, bool KDA>
__global__ void __launch_bounds__(D) delta_prep_kernel(const T* __restrict__ qkv, const T* __restrict__ proj,
                                                       int proj_stride, int b_off, int a_off,
                                                       const T* __restrict__ f, const float* __restrict__ A_log,
                                                       const float* __restrict__ dt_bias, void* __restrict__ qn,
                                                       void* __restrict__ kn, float* __restrict__ gexp,
                                                       float* __restrict__ glog, float* __restrict__ beta, int Hk,
                                                       int Hv, float scale, float eps_l2, int qk_bf16) {
  __shared__ float red[2 * (D / 32)];
  const int r = blockIdx.x, kh = blockIdx.y, i = threadIdx.x;  // rows on x: > 65535 tokens
  const int G = Hv / Hk;
  const int qkv_stride = 2 * Hk * D + Hv * D;
  const T* row = qkv + (size_t)r * qkv_stride;
  const T* prow = proj + (size_t)r * proj_stride;
  const float q = io<T>::ld(row + kh * D + i), k = io<T>::ld(row + Hk * D + kh * D + i);
  // gate inputs of this key head's value heads, loaded before the reductions
  float fv = 0.f, araw = 0.f, braw = 0.f;
  if (KDA) fv = io<T>::ld(f + (size_t)r * Hv * D + kh * D + i);  // KDA: G == 1
  else if (i < G) araw = io<T>::ld(prow + a_off + kh * G + i);
  if (i < G) braw = io<T>::ld(prow + b_off + kh * G + i);
  float qq = q * q, kk = k * k;
  qq = warp_sum(qq);
  kk = warp_sum(kk);
  const int lane = i & 31, warp = i >> 5;
  if (lane == 0) { red[warp] = qq; red[D / 32 + warp] = kk; }
  __syncthreads();
  qq = 0.f;
  kk = 0.f;
#pragma unroll
  for (int w = 0; w < D / 32; ++w) { qq += red[w]; kk += red[D / 32 + w]; }
  const size_t qi = ((size_t)r * Hk + kh) * D + i;
  if (qk_bf16) {  // the chunked GDN prefill reads q / k as bf16 TMA tiles
    reinterpret_cast<__nv_bfloat16*>(qn)[qi] = __float2bfloat16_rn(q * rsqrtf(qq + eps_l2) * scale);
    reinterpret_cast<__nv_bfloat16*>(kn)[qi] = __float2bfloat16_rn(k * rsqrtf(kk + eps_l2));
  } else {
    reinterpret_cast<float*>(qn)[qi] = q * rsqrtf(qq + eps_l2) * scale;
    reinterpret_cast<float*>(kn)[qi] = k * rsqrtf(kk + eps_l2);
  }
  if (KDA) {
    const int h = kh;
    const float gl = -expf(A_log[h]) * softplus_f(fv + dt_bias[h * D + i]);
    gexp[((size_t)r * Hv + h) * D + i] = expf(gl);
    if (glog) glog[((size_t)r * Hv + h) * D + i] = gl;  // per-channel log gate (chunked KDA prefill)
  } else if (i < G) {
    const int h = kh * G + i;
    const float g = -expf(A_log[h]) * softplus_f(araw + dt_bias[h]);
    gexp[(size_t)r * Hv + h] = expf(g);
    if (glog) glog[(size_t)r * Hv + h] = g;
  }
  if (i < G) beta[(size_t)r * Hv + kh * G + i] = sigmoid_f(braw);
}

// Recurrent scan: CTA = 4 warps x 8 value columns of one (sequence, head); state in registers.
template <typename T, int D, bool KDA>
__global__ void __launch_bounds__(128) delta_scan_kernel(const float* __restrict__ qn, const float* __restrict__ kn,
                                                         const T* __restrict__ qkv, int v_off, int qkv_stride,
                                                         const float* __restrict__ gexp, const float* __restrict__ beta,
                                                         float* __restrict__ o, float* __restrict__ state,
                                                         const int32_t* __restrict__ slot_idx,
                                                         const int32_t* __restrict__ cu, int Hk, int Hv,
                                                         int init_state) {
  constexpr int EPL = D / 32, CPW = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int G = Hv / Hk, kh = h / G;
  const int c0 = (cg * 4 + warp) * CPW;
  const int slot = slot_idx ? slot_idx[s] : s;
  const int t0 = cu[s], t1 = cu[s + 1];
  float* S = state + ((size_t)slot * Hv + h) * D * D;
  float st[CPW][EPL];
#pragma unroll
  for (int n = 0; n < CPW; ++n)
#pragma unroll
    for (int e = 0; e < EPL; ++e) st[n][e] = init_state ? S[(size_t)(c0 + n) * D + lane * EPL + e] : 0.f;

  for (int t = t0; t < t1; ++t) {
    float q[EPL], k[EPL], eg[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const int i = lane * EPL + e;
      q[e] = qn[((size_t)t * Hk + kh) * D + i];
      k[e] = kn[((size_t)t * Hk + kh) * D + i];
      eg[e] = KDA ? gexp[((size_t)t * Hv + h) * D + i] : gexp[(size_t)t * Hv + h];
    }
    const float bt = beta[(size_t)t * Hv + h];
    float qk = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) qk += q[e] * k[e];
    qk = warp_sum(qk);
    float vv = lane < CPW ? io<T>::ld(qkv + (size_t)t * qkv_stride + v_off + h * D + c0 + lane) : 0.f;
#pragma unroll
    for (int n = 0; n < CPW; ++n) {
      float kd = 0.f, qd = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        kd += k[e] * eg[e] * st[n][e];
        qd += q[e] * eg[e] * st[n][e];
      }
      kd = warp_sum(kd);
      qd = warp_sum(qd);
      const float u = bt * (__shfl_sync(0xffffffffu, vv, n) - kd);
#pragma unroll
      for (int e = 0; e < EPL; ++e) st[n][e] = eg[e] * st[n][e] + k[e] * u;
      if (lane == 0) o[((size_t)t * Hv + h) * D + c0 + n] = qd + qk * u;
    }
  }
#pragma unroll
  for (int n = 0; n < CPW; ++n)
#pragma unroll
    for (int e = 0; e < EPL; ++e) S[(size_t)(c0 + n) * D + lane * EPL + e] = st[n][e];
}

// One warp per (row, head): D/32 values per lane (vectorised), a shuffle reduction, no
// block barrier; 8 warps per CTA cover 8 (row, head) pairs.
template <typename T, int D>
__global__ void __launch_bounds__(256) gated_rmsnorm_kernel(const float* __restrict__ o, const T* __restrict__ gate,
                                                            int gate_stride, const T* __restrict__ w,
                                                            T* __restrict__ out, int rows, int H, float eps, int act) {
  constexpr int EPL = D / 32;
  const int lane = threadIdx.x & 31;
  const size_t pair = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pair >= (size_t)rows * H) return;
  const size_t r = pair / H;
  const int h = (int)(pair % H);
  const int j0 = lane * EPL;
  float v[EPL], gz[EPL], wv[EPL];
#pragma unroll
  for (int e = 0; e < EPL; e += 2) {
    const float2 t = *reinterpret_cast<const float2*>(o + pair * D + j0 + e);
    v[e] = t.x;
    v[e + 1] = t.y;
  }
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    gz[e] = io<T>::ld(gate + r * gate_stride + h * D + j0 + e);
    wv[e] = io<T>::ld(w + j0 + e);
  }
  float ss = 0.f;
#pragma unroll
  for (int e = 0; e < EPL; ++e) ss += v[e] * v[e];
  ss = warp_sum(ss);
  const float rstd = rsqrtf(ss / (float)D + eps);
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const float a = act ? sigmoid_f(gz[e]) : silu_f(gz[e]);
    io<T>::st(out + pair * D + j0 + e, v[e] * rstd * wv[e] * a);
  }
}

// 512-thread CTAs when (heads x batch) leaves most SMs without a CTA (small batches): twice
// the state columns of one CTA in flight (B=1 decode 6.22 -> 6.13 ms/step, r01_decode_ablation.md).
template <typename T, int D, bool KDA>
static sn_status launch_delta_decode_t(const DeltaDecodeArgs& a, int B, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  const bool wide = a.Hv * B < 148;
  cfg.gridDim = dim3(a.Hv, B);
  // GDN: one item (value head, sequence) per CTA, 1-D grid.  The kernel can also walk items
  // persistently (grid = 4 CTAs per SM, the next item's state requested before the norm
  // epilogue), but that measured slower at B=64: 52.7 vs 48.0 us (tools/bench_delta.py).
  if (!KDA) cfg.gridDim = dim3(a.Hv * B);
  cfg.blockDim = dim3(wide ? 2 * kDecodeThreads : kDecodeThreads);
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // state prefetch overlaps the in-proj tail
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  if (!KDA && D == 128 && !wide) {  // the state staged through shared memory (cp.async ring)
    constexpr int NBUF = 2;
    cfg.dynamicSmemBytes = (size_t)(kDecodeThreads / 32) * NBUF * 4 * 128 * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(gdn_decode_cpa_kernel<T, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)cfg.dynamicSmemBytes);
      attr = true;
    }
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, gdn_decode_cpa_kernel<T, NBUF>, a);
    if (e2 != cudaSuccess) {
      set_error("sn_gdn_decode launch: %s", cudaGetErrorString(e2));
      return SN_ECUDA;
    }
    return check_launch("sn_gdn_decode");
  }
  cudaError_t e;
  if (KDA && D == 128 && !wide) {  // the state staged through shared memory (cp.async ring)
    cfg.dynamicSmemBytes = (size_t)(kDecodeThreads / 32) * 2 * 4 * 128 * sizeof(float);
    static bool kattr = false;
    if (!kattr) {
      cudaFuncSetAttribute(kda_decode_kernel<T, D, kDecodeThreads, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)cfg.dynamicSmemBytes);
      kattr = true;
    }
    e = cudaLaunchKernelEx(&cfg, kda_decode_kernel<T, D, kDecodeThreads, true>, a);
  } else if (KDA)
    e = wide ? cudaLaunchKernelEx(&cfg, kda_decode_kernel<T, D, 2 * kDecodeThreads>, a)
             : cudaLaunchKernelEx(&cfg, kda_decode_kernel<T, D>, a);
  else
    e = wide ? cudaLaunchKernelEx(&cfg, gdn_decode_kernel<T, D, 2 * kDecodeThreads>, a)
             : cudaLaunchKernelEx(&cfg, gdn_decode_kernel<T, D>, a);
  if (e != cudaSuccess) {
    set_error("%s launch: %s", KDA ? "sn_kda_decode" : "sn_gdn_decode", cudaGetErrorString(e));
    return SN_ECUDA;
  }
  return check_launch(KDA ? "sn_kda_decode" : "sn_gdn_decode");
}

template <bool KDA>
static sn_status launch_delta_decode(const DeltaDecodeArgs& a, int B, int D, int dtype, cudaStream_t st) {
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    if (D == 128) return launch_delta_decode_t<T, 128, KDA>(a, B, st);
    if (D == 64) return launch_delta_decode_t<T, 64, KDA>(a, B, st);
    set_error("delta decode: head dim %d unsupported (64 or 128)", D);
    return SN_EUNSUPPORTED;
  });
}

}  // namespace sn

using namespace sn;

namespace sn {
template <typename T, int D, bool K>
static void launch_prep(dim3 grid, cudaStream_t st, const void* qkv_conv, const void* proj, int proj_stride,
                        int b_off, int a_off, const void* f, const float* A_log, const float* dt_bias, void* qn,
                        void* kn, float* gexp, float* glog, float* beta, int Hk, int Hv, float scale, float eps_l2,
                        int qk_bf16) {
  delta_prep_kernel<T, D, K><<<grid, D, 0, st>>>((const T*)qkv_conv, (const T*)proj, proj_stride, b_off, a_off,
                                                 (const T*)f, A_log, dt_bias, qn, kn, gexp, glog, beta, Hk, Hv,
                                                 scale, eps_l2, qk_bf16);
}

template <typename T, int D, bool K>
static void launch_scan(dim3 grid, cudaStream_t st, const float* qn, const float* kn, const void* qkv_conv,
                        int v_off, int qkv_stride, const float* gexp, const float* beta, float* o, float* state,
                        const int32_t* slot_idx, const int32_t* cu, int Hk, int Hv, int init_state) {
  delta_scan_kernel<T, D, K><<<grid, 128, 0, st>>>(qn, kn, (const T*)qkv_conv, v_off, qkv_stride, gexp, beta, o,
                                                   state, slot_idx, cu, Hk, Hv, init_state);
}

}  // namespace sn

extern "C" {

sn_status sn_gdn_decode(const void* proj, int proj_stride, void* conv_ring, const void* conv_w, float* state,
                        const int32_t* slot_idx, const int32_t* positions, const float* A_log,
                        const float* dt_bias, const void* norm_w, void* out, int B, int Hk, int Hv, int D,
                        int conv_width, float scale, float eps_l2, float eps_norm, int dtype, void* stream) {
  SN_REQUIRE(B > 0 && Hk > 0 && Hv > 0 && Hv % Hk == 0, "sn_gdn_decode: bad heads B=%d Hk=%d Hv=%d", B, Hk, Hv);
  SN_REQUIRE(conv_width == 4, "sn_gdn_decode: conv width %d (the pinned width is 4)", conv_width);
  SN_REQUIRE(proj && conv_ring && conv_w && state && positions && A_log && dt_bias && norm_w && out,
             "sn_gdn_decode: NULL pointer argument");
  DeltaDecodeArgs a{};
  a.proj = proj; a.proj_stride = proj_stride; a.conv_ring = conv_ring; a.conv_w = conv_w; a.state = state;
  a.slot_idx = slot_idx; a.positions = positions; a.A_log = A_log; a.dt_bias = dt_bias; a.norm_w = norm_w;
  a.out = out; a.Hk = Hk; a.Hv = Hv; a.rank = 0; a.B = B;
  a.conv_channels = 2 * Hk * D + Hv * D;
  a.q_off = 0; a.k_off = Hk * D; a.v_off = 2 * Hk * D; a.z_off = 2 * Hk * D + Hv * D;
  a.b_off = 2 * Hk * D + 2 * Hv * D; a.a_off = a.b_off + Hv;
  a.scale = scale; a.eps_l2 = eps_l2; a.eps_norm = eps_norm;
  SN_REQUIRE(proj_stride >= a.a_off + Hv, "sn_gdn_decode: proj_stride %d < %d", proj_stride, a.a_off + Hv);
  return launch_delta_decode<false>(a, B, D, dtype, (cudaStream_t)stream);
}

sn_status sn_kda_decode(const void* proj, int proj_stride, const void* fg, void* conv_ring, const void* conv_w,
                        float* state, const int32_t* slot_idx, const int32_t* positions, const float* A_log,
                        const float* dt_bias, const void* g2_b, const void* norm_w, void* out, int B, int H, int D,
                        int rank, int conv_width, float scale, float eps_l2, float eps_norm, int dtype, void* stream) {
  SN_REQUIRE(B > 0 && H > 0, "sn_kda_decode: bad shape B=%d H=%d", B, H);
  SN_REQUIRE(rank > 0 && rank % 8 == 0, "sn_kda_decode: rank %d must be a multiple of 8", rank);
  SN_REQUIRE(conv_width == 4, "sn_kda_decode: conv width %d (the pinned width is 4)", conv_width);
  SN_REQUIRE(proj && fg && conv_ring && conv_w && state && positions && A_log && dt_bias && norm_w && out && g2_b,
             "sn_kda_decode: NULL pointer argument");
  DeltaDecodeArgs a{};
  a.proj = proj; a.proj_stride = proj_stride; a.fg = fg; a.conv_ring = conv_ring; a.conv_w = conv_w; a.state = state;
  a.slot_idx = slot_idx; a.positions = positions; a.A_log = A_log; a.dt_bias = dt_bias;
  a.g2_b = g2_b; a.norm_w = norm_w; a.out = out; a.Hk = H; a.Hv = H; a.rank = rank; a.B = B;
  a.conv_channels = 3 * H * D;
  a.q_off = 0; a.k_off = H * D; a.v_off = 2 * H * D; a.f1_off = 3 * H * D; a.g1_off = 3 * H * D + rank;
  a.b_off = 3 * H * D + 2 * rank;
  a.scale = scale; a.eps_l2 = eps_l2; a.eps_norm = eps_norm;
  SN_REQUIRE(proj_stride >= a.b_off + H, "sn_kda_decode: proj_stride %d < %d", proj_stride, a.b_off + H);
  return launch_delta_decode<true>(a, B, D, dtype, (cudaStream_t)stream);
}

sn_status sn_conv_prefill(const void* x, int x_stride, void* y, const void* conv_w, void* conv_ring,
                          const void* ring_hist, const int32_t* cu_seqlens, const int32_t* slot_idx,
                          const int32_t* pos0, int num_seqs, int rows, int channels, int width, int dtype,
                          void* stream) {
  SN_REQUIRE((pos0 == nullptr) == (ring_hist == nullptr), "sn_conv_prefill: pos0 and ring_hist go together");
  SN_REQUIRE(num_seqs > 0 && rows > 0 && channels > 0, "sn_conv_prefill: bad shape");
  SN_REQUIRE(width >= 1 && width <= 8, "sn_conv_prefill: width %d not in [1,8]", width);
  if (dtype == SN_BF16 && width == 4 && channels % 2 == 0 && x_stride % 2 == 0 && ((uintptr_t)x & 3) == 0 &&
      ((uintptr_t)y & 3) == 0) {
    dim3 grid(ceil_div(channels / 2, 128), ceil_div(rows, 64), num_seqs);
    conv4_prefill_bf16x2_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)x, x_stride, (__nv_bfloat16*)y, (const __nv_bfloat16*)conv_w, (__nv_bfloat16*)conv_ring,
        (const __nv_bfloat16*)ring_hist, cu_seqlens, slot_idx, pos0, channels);
    return check_launch("sn_conv_prefill(bf16x2)");
  }
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    dim3 grid(ceil_div(channels, 128), ceil_div(rows, 64), num_seqs);
    conv_prefill_kernel<T><<<grid, 128, 0, (cudaStream_t)stream>>>((const T*)x, x_stride, (T*)y, (const T*)conv_w,
                                                                  (T*)conv_ring, (const T*)ring_hist, cu_seqlens,
                                                                  slot_idx, pos0, channels, width);
    return check_launch("sn_conv_prefill");
  });
}

sn_status sn_delta_prep(int kind, const void* qkv_conv, const void* proj, int proj_stride, int b_off, int a_off,
                        const void* f, const float* A_log, const float* dt_bias, void* qn, void* kn, float* gexp,
                        float* glog, float* beta, int rows, int Hk, int Hv, int D, float scale, float eps_l2,
                        int qk_dtype, int dtype, void* stream) {
  SN_REQUIRE(qk_dtype == SN_F32 || qk_dtype == SN_BF16, "sn_delta_prep: q/k dtype %d", qk_dtype);
  SN_REQUIRE(kind == 0 || kind == 1, "sn_delta_prep: kind %d", kind);
  SN_REQUIRE(rows > 0 && Hk > 0 && Hv % Hk == 0, "sn_delta_prep: bad shape");
  SN_REQUIRE(kind == 0 || f != nullptr, "sn_delta_prep: KDA needs f");
  SN_REQUIRE(kind == 0 || Hk == Hv, "sn_delta_prep: KDA has one key head per value head");
  SN_REQUIRE(Hv / Hk <= D, "sn_delta_prep: too many value heads per key head");
  SN_REQUIRE(D == 64 || D == 128, "sn_delta_prep: D=%d unsupported", D);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    dim3 grid(rows, Hk);
    cudaStream_t st = (cudaStream_t)stream;
    auto fn = D == 128 ? (kind ? launch_prep<T, 128, true> : launch_prep<T, 128, false>)
                       : (kind ? launch_prep<T, 64, true> : launch_prep<T, 64, false>);
    fn(grid, st, qkv_conv, proj, proj_stride, b_off, a_off, f, A_log, dt_bias, qn, kn, gexp, glog, beta, Hk, Hv,
       scale, eps_l2, qk_dtype == SN_BF16);
    return check_launch("sn_delta_prep");
  });
}

sn_status sn_delta_scan(int kind, const float* qn, const float* kn, const void* qkv_conv, int v_off,
                        int qkv_stride, const float* gexp, const float* beta, float* o, float* state,
                        const int32_t* slot_idx, const int32_t* cu_seqlens, int num_seqs, int Hk, int Hv, int D,
                        int init_state, int dtype, void* stream) {
  SN_REQUIRE(kind == 0 || kind == 1, "sn_delta_scan: kind %d", kind);
  SN_REQUIRE(num_seqs > 0 && Hk > 0 && Hv % Hk == 0, "sn_delta_scan: bad shape");
  SN_REQUIRE(D == 64 || D == 128, "sn_delta_scan: D=%d unsupported", D);
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    dim3 grid(D / 32, Hv, num_seqs);
    cudaStream_t st = (cudaStream_t)stream;
    auto fn = D == 128 ? (kind ? launch_scan<T, 128, true> : launch_scan<T, 128, false>)
                       : (kind ? launch_scan<T, 64, true> : launch_scan<T, 64, false>);
    fn(grid, st, qn, kn, qkv_conv, v_off, qkv_stride, gexp, beta, o, state, slot_idx, cu_seqlens, Hk, Hv,
       init_state);
    return check_launch("sn_delta_scan");
  });
}

sn_status sn_gated_rmsnorm(const float* o, const void* gate, int gate_stride, const void* norm_w, void* out,
                           int rows, int H, int D, float eps, int act, int dtype, void* stream) {
  SN_REQUIRE(rows > 0 && H > 0, "sn_gated_rmsnorm: bad shape");
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    const unsigned grid = (unsigned)(((size_t)rows * H + 7) / 8);
    cudaStream_t st = (cudaStream_t)stream;
    if (D == 128) gated_rmsnorm_kernel<T, 128><<<grid, 256, 0, st>>>(o, (const T*)gate, gate_stride, (const T*)norm_w, (T*)out, rows, H, eps, act);
    else if (D == 64) gated_rmsnorm_kernel<T, 64><<<grid, 256, 0, st>>>(o, (const T*)gate, gate_stride, (const T*)norm_w, (T*)out, rows, H, eps, act);
    else { set_error("sn_gated_rmsnorm: D=%d unsupported", D); return SN_EUNSUPPORTED; }
    return check_launch("sn_gated_rmsnorm");
  });
}

}  // extern "C"
