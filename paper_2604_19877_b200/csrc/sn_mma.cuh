// Warp-level bf16 tensor-core helpers (mma.sync m16n8k16 + ldmatrix) shared by the
// attention decode and the chunked delta-rule prefill.
#pragma once
#include "sn_common.cuh"

namespace sn {
namespace mma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
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
// D[16x8] += A[16x16] (row) . B[16x8] (col), bf16 in, fp32 accumulate.
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

// Fragment loaders for bf16 tiles in shared memory with row stride `ld` elements
// (padded so the 8 rows an ldmatrix touches fall in different banks).
//
// A fragment (16x16, row-major storage A[row][col]) at (r0, c0).
__device__ __forceinline__ void lda(const __nv_bfloat16* base, int ld, int r0, int c0, uint32_t* a) {
  const int lane = threadIdx.x & 31;
  const int row = r0 + (lane & 15), col = c0 + ((lane >> 4) << 3);
  ldsm_x4(smem_u32(base + row * ld + col), a[0], a[1], a[2], a[3]);
}
// A fragment of A = X^T where X is stored row-major X[k][m] (i.e. A column-major): the
// 16x16 block A[r0.., c0..] = X[c0.., r0..]^T.
__device__ __forceinline__ void lda_t(const __nv_bfloat16* x, int ld, int r0, int c0, uint32_t* a) {
  const int lane = threadIdx.x & 31;
  // matrices: (rows r0..+7, cols c0..+7), (rows r0+8.., c0..), (r0.., c0+8..), (r0+8.., c0+8..)
  const int mi = lane >> 3, ri = lane & 7;
  const int m = r0 + ((mi & 1) << 3), k = c0 + ((mi >> 1) << 3) + ri;
  ldsm_x4_t(smem_u32(x + k * ld + m), a[0], a[1], a[2], a[3]);
}
// B fragments for two adjacent n8 tiles from B^T stored row-major Bt[n][k] ("col" B):
// returns (b0,b1) for n-tile n0 and (b2,b3) for n0+8, k-step k0..k0+15.
__device__ __forceinline__ void ldb_nk(const __nv_bfloat16* bt, int ld, int n0, int k0, uint32_t& b0, uint32_t& b1,
                                       uint32_t& b2, uint32_t& b3) {
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  const int n = n0 + ((mi >> 1) << 3) + ri, k = k0 + ((mi & 1) << 3);
  ldsm_x4(smem_u32(bt + n * ld + k), b0, b1, b2, b3);
}
// Same from B stored row-major B[k][n] (uses the transposing ldmatrix).
__device__ __forceinline__ void ldb_kn(const __nv_bfloat16* b, int ld, int n0, int k0, uint32_t& b0, uint32_t& b1,
                                       uint32_t& b2, uint32_t& b3) {
  const int lane = threadIdx.x & 31;
  const int mi = lane >> 3, ri = lane & 7;
  const int k = k0 + ((mi & 1) << 3) + ri, n = n0 + ((mi >> 1) << 3);
  ldsm_x4_t(smem_u32(b + k * ld + n), b0, b1, b2, b3);
}

}  // namespace mma
}  // namespace sn
