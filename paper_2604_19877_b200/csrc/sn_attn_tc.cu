// bf16 split-KV flash-decode for FA/SWA (R/PAPER.md:1540-1563), the decode
// hot path for attention layers.
//
// Shape of the work: per (sequence, kv head) the GQA group of G = Hq/Hkv query
// heads reads every K/V byte once.  With G=4 the arithmetic intensity is ~4
// flop/byte, too close to the CUDA-core FMA budget at the power-capped clock
// (~1.3 GHz) to stay on the HBM roofline, so both products run on tensor cores:
//
//   S[16 x 32]  = Q[16 x D] . K_tile^T     (rows 0..G-1 real, the rest zero)
//   O[16 x D]  += P[16 x 32] . V_tile       (P re-used from S's accumulators)
//
// Data movement: the page pool is laid out [page][Hkv][page_size][D] so one
// head's 32-key half page is a contiguous 32 x D tile.  Each warp owns NST
// shared-memory stages and streams its tiles with 2-D TMA loads
// (cp.async.bulk.tensor, 128B swizzle) completing on per-stage mbarriers; the
// swizzle makes every ldmatrix conflict-free.  Warps are independent (own
// tiles, own online-softmax state) and merge once at the end; splits merge in
// the last CTA of a (sequence, kv head) through finish_split().
#include <cuda.h>

#include "sn_attn.cuh"
#include "sn_tc.cuh"

namespace sn {

namespace tc {

constexpr int KT = 32;   // keys per tile (half of a 64-key page)
constexpr int NW = 4;    // warps per CTA
constexpr int NST = 3;   // stages per warp

// mbarrier / TMA helpers: sn_tc.cuh.  KV pages are read exactly once per decode step and
// are loaded evict-first so they do not displace the L2-resident activations / block tables.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Byte offset of element (row, dim) inside a KT x D tile stored as D/64 boxes of
// KT rows x 128 B with the TMA 128B swizzle (16-B chunk index ^= row % 8).
__device__ __forceinline__ uint32_t swz(int row, int dim) {
  const int box = dim >> 6, chunk = (dim & 63) >> 3;
  return box * (KT * 128) + row * 128 + ((chunk ^ (row & 7)) << 4) + ((dim & 7) << 1);
}

template <int D>
__global__ void __launch_bounds__(NW * 32, 1)
    attn_decode_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                          const AttnDecodeArgs a) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  constexpr int TILE_BYTES = KT * D * 2;        // one of K or V
  constexpr int STAGE_BYTES = 2 * TILE_BYTES;   // K then V
  constexpr int NKS = D / 16;                   // k-steps of Q.K^T
  constexpr int NDT = D / 8;                    // dim tiles of O
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t bars[NW * NST];
  // 128B-swizzled TMA destinations need 1024-B aligned shared addresses.
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ float s_m[NW][16], s_l[NW][16];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int G = a.Hq / a.Hkv;
  const int n_keys = attn_num_keys(a, b);
  const int split_keys = a.split_pages * a.page_size;
  const int num_splits = max(1, (n_keys + split_keys - 1) / split_keys);
  if (split >= num_splits) return;
  const int k0 = split * split_keys, k1 = min(n_keys, k0 + split_keys);
  const int n_tiles = (k1 - k0 + KT - 1) / KT;
  const int my_n = warp < n_tiles ? (n_tiles - warp + NW - 1) / NW : 0;
  const int32_t* bt = a.block_table + (size_t)b * a.max_blocks;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NW * NST; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  uint64_t evict_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(evict_first));
  uint8_t* my_stages = smem + (size_t)warp * NST * STAGE_BYTES;
  uint64_t* my_bars = bars + warp * NST;
  auto issue = [&](int j) {
    const int tile = warp + j * NW;
    const int key0 = k0 + tile * KT;
    const int page = bt[key0 / a.page_size];
    const int row = (page * a.Hkv + hk) * a.page_size + (key0 % a.page_size);
    uint8_t* st = my_stages + (j % NST) * STAGE_BYTES;
    uint64_t* bar = my_bars + (j % NST);
    mbar_expect_tx(bar, STAGE_BYTES);
#pragma unroll
    for (int box = 0; box < D / 64; ++box) {
      tma_load_2d(st + box * KT * 128, &kmap, box * 64, row, bar, evict_first);
      tma_load_2d(st + TILE_BYTES + box * KT * 128, &vmap, box * 64, row, bar, evict_first);
    }
  };
  if (lane == 0)
    for (int j = 0; j < min(NST, my_n); ++j) issue(j);

  // Q fragments (A operand, row-major 16 x D; rows >= G are zero).
  const __nv_bfloat16* Q = reinterpret_cast<const __nv_bfloat16*>(a.q) + ((size_t)b * a.Hq + hk * G) * D;
  const int r0 = lane >> 2, cq = (lane & 3) * 2;
  uint32_t qa[NKS][4];
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks) {
    const int c = ks * 16 + cq;
    qa[ks][0] = r0 < G ? *reinterpret_cast<const uint32_t*>(Q + r0 * D + c) : 0u;
    qa[ks][1] = r0 + 8 < G ? *reinterpret_cast<const uint32_t*>(Q + (r0 + 8) * D + c) : 0u;
    qa[ks][2] = r0 < G ? *reinterpret_cast<const uint32_t*>(Q + r0 * D + c + 8) : 0u;
    qa[ks][3] = r0 + 8 < G ? *reinterpret_cast<const uint32_t*>(Q + (r0 + 8) * D + c + 8) : 0u;
  }
  const float qscale = a.scale * 1.4426950408889634f;

  float o[NDT][4];
#pragma unroll
  for (int i = 0; i < NDT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  const int mi = lane >> 3, ri = lane & 7;
  for (int j = 0; j < my_n; ++j) {
    const int tile = warp + j * NW;
    const int key0 = k0 + tile * KT;
    uint8_t* st = my_stages + (j % NST) * STAGE_BYTES;
    mbar_wait(my_bars + (j % NST), (j / NST) & 1);
    const uint32_t kbase = smem_u32(st), vbase = kbase + TILE_BYTES;

    // ---- S = Q K^T : 4 key n-tiles of 8
    float s[KT / 8][4];
#pragma unroll
    for (int nt = 0; nt < KT / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < NKS; ks += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kbase + swz(nt * 8 + ri, ks * 16 + mi * 8), b0, b1, b2, b3);
        mma_bf16(s[nt], qa[ks], b0, b1);
        mma_bf16(s[nt], qa[ks + 1], b2, b3);
      }
    }
    // ---- online softmax (rows lo = lane/4, hi = lane/4 + 8), log2 domain
    float tmax_lo = -INFINITY, tmax_hi = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < KT / 8; ++nt) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool valid = key0 + nt * 8 + cq + c < k1;
        s[nt][c] = valid ? s[nt][c] * qscale : -INFINITY;
        s[nt][2 + c] = valid ? s[nt][2 + c] * qscale : -INFINITY;
        tmax_lo = fmaxf(tmax_lo, s[nt][c]);
        tmax_hi = fmaxf(tmax_hi, s[nt][2 + c]);
      }
    }
    tmax_lo = fmaxf(tmax_lo, __shfl_xor_sync(0xffffffffu, tmax_lo, 1));
    tmax_lo = fmaxf(tmax_lo, __shfl_xor_sync(0xffffffffu, tmax_lo, 2));
    tmax_hi = fmaxf(tmax_hi, __shfl_xor_sync(0xffffffffu, tmax_hi, 1));
    tmax_hi = fmaxf(tmax_hi, __shfl_xor_sync(0xffffffffu, tmax_hi, 2));
    const float mn_lo = fmaxf(m_lo, tmax_lo), mn_hi = fmaxf(m_hi, tmax_hi);
    const float al_lo = exp2f(m_lo - mn_lo), al_hi = exp2f(m_hi - mn_hi);
    m_lo = mn_lo;
    m_hi = mn_hi;
    l_lo *= al_lo;
    l_hi *= al_hi;
#pragma unroll
    for (int i = 0; i < NDT; ++i) {
      o[i][0] *= al_lo; o[i][1] *= al_lo;
      o[i][2] *= al_hi; o[i][3] *= al_hi;
    }
    uint32_t pa[KT / 16][4];
#pragma unroll
    for (int nt = 0; nt < KT / 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mn_lo), p1 = exp2f(s[nt][1] - mn_lo);
      const float p2 = exp2f(s[nt][2] - mn_hi), p3 = exp2f(s[nt][3] - mn_hi);
      l_lo += p0 + p1;
      l_hi += p2 + p3;
      pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(p0, p1);
      pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(p2, p3);
    }
    // ---- O += P V : k-steps of 16 keys, dim n-tiles in pairs
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk) {
      const uint32_t a_frag[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
      for (int nd = 0; nd < NDT; nd += 2) {
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vbase + swz(kk * 16 + (mi & 1) * 8 + ri, nd * 8 + (mi >> 1) * 8), b0, b1, b2, b3);
        mma_bf16(o[nd], a_frag, b0, b1);
        mma_bf16(o[nd + 1], a_frag, b2, b3);
      }
    }
    __syncwarp();
    if (lane == 0 && j + NST < my_n) issue(j + NST);
  }

  // ---- merge the NW warps (reuse the stage memory once everyone is done)
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  __syncthreads();
  float* s_o = reinterpret_cast<float*>(smem);  // [NW][16][D]
  if ((lane & 3) == 0) {
    s_m[warp][r0] = m_lo; s_l[warp][r0] = l_lo;
    s_m[warp][r0 + 8] = m_hi; s_l[warp][r0 + 8] = l_hi;
  }
#pragma unroll
  for (int i = 0; i < NDT; ++i) {
    const int d = i * 8 + cq;
    s_o[(warp * 16 + r0) * D + d] = o[i][0];
    s_o[(warp * 16 + r0) * D + d + 1] = o[i][1];
    s_o[(warp * 16 + r0 + 8) * D + d] = o[i][2];
    s_o[(warp * 16 + r0 + 8) * D + d + 1] = o[i][3];
  }
  __syncthreads();
  float* ws_o = a.workspace;
  float* ws_ml = a.workspace + (size_t)a.B * a.Hkv * a.max_splits * G * D;
  const size_t part = ((size_t)b * a.Hkv + hk) * a.max_splits + split;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int g = idx / D, d = idx - g * D;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w][g]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < NW; ++w) {
      const float f = s_m[w][g] == -INFINITY ? 0.f : exp2f(s_m[w][g] - M);
      L += s_l[w][g] * f;
      O += s_o[(w * 16 + g) * D + d] * f;
    }
    ws_o[(part * G + g) * D + d] = O;
    if (d == 0) { ws_ml[(part * G + g) * 2] = M; ws_ml[(part * G + g) * 2 + 1] = L; }
  }
  finish_split<__nv_bfloat16>(a, b, hk, num_splits, G, D);
}

// --------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D view of a page pool: rows = (page, head, slot), cols = D; box = KT rows x 64 cols.
static bool make_map(CUtensorMap* map, const void* base, int D) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)1 << 30};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)KT};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tc

sn_status attn_decode_tc_bf16(const AttnDecodeArgs& a, int D, cudaStream_t st) {
  using namespace tc;
  SN_REQUIRE(a.page_size % KT == 0, "attn_decode_tc: page_size %d must be a multiple of %d", a.page_size, KT);
  SN_REQUIRE(a.Hq / a.Hkv <= 16, "attn_decode_tc: GQA group %d > 16", a.Hq / a.Hkv);
  SN_REQUIRE(((uintptr_t)a.k_cache % 16) == 0 && ((uintptr_t)a.v_cache % 16) == 0,
             "attn_decode_tc: cache pointers must be 16-byte aligned");
  CUtensorMap kmap, vmap;
  if (!make_map(&kmap, a.k_cache, D) || !make_map(&vmap, a.v_cache, D)) {
    set_error("attn_decode_tc: cuTensorMapEncodeTiled failed");
    return SN_ECUDA;
  }
  dim3 grid(a.max_splits, a.Hkv, a.B);
  const int smem = NW * NST * 2 * KT * D * 2;
  const int smem_merge = NW * 16 * D * 4;
  const int dyn = (smem > smem_merge ? smem : smem_merge) + 1024;
  if (D == 128) {
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(attn_decode_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn); attr = true; }
    launch_pdl(attn_decode_tc_kernel<128>, grid, dim3(NW * 32), dyn, st, kmap, vmap, a);
  } else if (D == 64) {
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(attn_decode_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn); attr = true; }
    launch_pdl(attn_decode_tc_kernel<64>, grid, dim3(NW * 32), dyn, st, kmap, vmap, a);
  } else {
    set_error("attn_decode_tc: D=%d unsupported", D);
    return SN_EUNSUPPORTED;
  }
  return check_launch("sn_attn_decode(tc)");
}

}  // namespace sn
