// Decode-GEMM work plans (sn_dgemm.cu), shared with the fused decode chain (sn_chain.cu).
#pragma once

namespace sn {
namespace dgemm {

constexpr int kSmemMax = 227 * 1024;

// um: batch tile (UMMA M); br: weight rows per block (UMMA N); splits: K splits (PARTIAL);
// ks: 64-column atoms per pipeline stage; nblocks: row blocks; ku: stages per item;
// grid: CTAs; ns: pipeline stages; stage: bytes per stage
struct Plan {
  int um, br, splits, ks, nblocks, ku, grid, ns, stage;
};

int num_sms();
int swiglu_block(int N);
Plan plan_for(int M, int N, int K, int br, int splits, int sw_half);
Plan make_plan(int M, int N, int K, int mode);

}  // namespace dgemm
}  // namespace sn
