// C-ABI entry points of the decode GEMM (include/sn_abi.h).  The kernel is the
// batch-as-M tcgen05 / TMEM / TMA weight stream in sn_gemm2.cu (the design notes there
// record why the earlier weights-as-M formulation was retired: ~120 issue cycles per
// M=128 x N=64 UMMA capped an SM at ~55 GB/s of weights).
#include <stdint.h>

#include "sn_common.cuh"

namespace sn {
int gemm2_splits(int M, int N, int K, int mode);
int gemm2_swiglu_block(int M, int N, int K);
void gemm2_debug_stats(unsigned long long* s);
sn_status gemm2_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                       int mode, int* splits_out, cudaStream_t st);
}  // namespace sn

using namespace sn;

extern "C" {

// Profiling aid: later launches write per-CTA clock64 counters into dev_stats (8 x #SMs u64:
// [1] producer done, [4] entry, [6] last MMA issued, [7] epilogue done); NULL disables.
void sn_gemm_debug_stats(unsigned long long* dev_stats) { gemm2_debug_stats(dev_stats); }

int sn_gemm_swiglu_block(int M, int N, int K) { return gemm2_swiglu_block(M, N, K); }

int sn_gemm_decode_splits(int M, int N, int K, int mode) { return gemm2_splits(M, N, K, mode); }

sn_status sn_gemm_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw, void* out, int ldo,
                         int mode, int* splits_out, void* stream) {
  constexpr int BK = 64;
  SN_REQUIRE(x && w && out, "sn_gemm_decode: NULL pointer");
  SN_REQUIRE(M >= 1 && M <= 128, "sn_gemm_decode: M=%d must be in [1, 128] (decode batch)", M);
  SN_REQUIRE(K % BK == 0 && K >= BK, "sn_gemm_decode: K=%d must be a multiple of %d", K, BK);
  SN_REQUIRE(N >= 1 && ldw >= K && ldx >= K, "sn_gemm_decode: bad N/ld");
  SN_REQUIRE(mode == SN_GEMM_STORE || mode == SN_GEMM_SWIGLU || mode == SN_GEMM_RESID || mode == SN_GEMM_PARTIAL ||
                 mode == SN_GEMM_SWIGLU_IL,
             "sn_gemm_decode: mode %d", mode);
  SN_REQUIRE(((uintptr_t)x % 16) == 0 && ((uintptr_t)w % 16) == 0 && (ldx % 8) == 0 && (ldw % 8) == 0,
             "sn_gemm_decode: operands must be 16-byte aligned");
  return gemm2_decode(x, M, K, ldx, w, N, ldw, out, ldo, mode, splits_out, (cudaStream_t)stream);
}

}  // extern "C"
