// Head-parallel decode: the row-parallel projection's all-reduce fused into the next
// residual-add + RMSNorm, over peer memory ("head-parallel + fused
// out-proj/all-reduce"; §8e).
//
// Every rank owns one symmetric buffer (mapped into every peer through CUDA IPC by the host,
// dist.SymmetricSlabs): word 0 is an arrival counter, then two parity regions of fp32 split-K
// slabs [8][rows][dim].  Per row-parallel projection each rank
//   1. writes its partial product straight into its parity region (the decode GEMM's
//      PARTIAL epilogue, no copy),
//   2. sn_tp_arrive: bumps its own counter (one thread, after the GEMM in stream order),
//   3. sn_tp_allreduce_add_rmsnorm: waits until every peer's counter has reached its own,
//      then every CTA reads all ranks' slabs over NVLink (P2P loads), sums them in rank order
//      then slab order — the same order on every rank, so the residual streams stay
//      bit-identical across ranks — adds the residual and applies the RMSNorm.
// Counters only grow, so the same captured CUDA graph serves every step.  Buffer reuse is
// safe with two parities: a rank writes parity p again only two arrivals later, after
// passing the wait of the arrival in between, which every peer reaches only after it has
// finished reading parity p.  The out-projection uses parity 0 and the FFN down-projection
// parity 1 (two arrivals per layer).
#include <cooperative_groups.h>

#include "sn_common.cuh"

namespace cg = cooperative_groups;

namespace sn {

__global__ void tp_arrive_kernel(unsigned int* counter) {
  __threadfence_system();
  atomicAdd(counter, 1u);
}

// One row per cluster of CS CTAs (each CTA dim / CS columns, one float4 per thread), the
// sum of squares combined through distributed shared memory: at B=64 that is 512 CTAs pulling
// world x S partials in parallel instead of 64 (15.5 -> see profiles/r02_tp_allreduce.md).
template <typename T>
__global__ void __launch_bounds__(256)
    tp_allreduce_add_rmsnorm_kernel(const unsigned long long* __restrict__ peer_slabs,
                                    const unsigned long long* __restrict__ peer_counters, int world, int rank,
                                    int nsplit, float* __restrict__ residual, const T* __restrict__ weight,
                                    T* __restrict__ out, int rows, int dim, float eps) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float scratch[32];
  __shared__ float cta_ss;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks(), part = (int)cluster.block_rank();
  if (threadIdx.x < 32) {  // lane r watches peer r: the world counters are polled in parallel
    const unsigned mine = *reinterpret_cast<volatile unsigned*>(peer_counters[rank]);
    for (int r = threadIdx.x; r < world; r += 32) {
      if (r == rank) continue;
      const volatile unsigned* c = reinterpret_cast<const volatile unsigned*>(peer_counters[r]);
      while ((int)(*c - mine) < 0) __nanosleep(64);
    }
    __syncwarp();
    if (threadIdx.x == 0) __threadfence_system();
  }
  __syncthreads();
  const int row = blockIdx.x / CS;
  const int per = dim / CS;
  const int i = part * per + threadIdx.x * 4;
  const bool active = threadIdx.x * 4 < per;
  const size_t slab = (size_t)rows * dim;
  const int parts = world * nsplit;  // summed in (rank, slab) order on every rank: identical residuals
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  float ss = 0.f;
  if (active) {
    v = *reinterpret_cast<const float4*>(residual + (size_t)row * dim + i);
    // 8 partials requested before any is added: one NVLink round trip per 8, not per partial
    for (int p0 = 0; p0 < parts; p0 += 8) {
      float4 pv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = p0 + u;
        if (p < parts) {
          const float* base = reinterpret_cast<const float*>(peer_slabs[p / nsplit]) + (size_t)row * dim + i;
          pv[u] = __ldcv(reinterpret_cast<const float4*>(base + (p % nsplit) * slab));  // peers' memory: no stale lines
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (p0 + u < parts) { v.x += pv[u].x; v.y += pv[u].y; v.z += pv[u].z; v.w += pv[u].w; }
      }
    }
    *reinterpret_cast<float4*>(residual + (size_t)row * dim + i) = v;
    ss = v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum(ss, scratch);
  if (threadIdx.x == 0) cta_ss = ss;
  cluster.sync();
  ss = 0.f;
  for (int r = 0; r < CS; ++r) ss += *cluster.map_shared_rank(&cta_ss, r);
  cluster.sync();  // every CTA's cta_ss stays alive until all ranks have read it
  const float rstd = rsqrtf(ss / (float)dim + eps);
  if (active) {
    T* o = out + (size_t)row * dim + i;
    io<T>::st(o, v.x * rstd * io<T>::ld(weight + i));
    io<T>::st(o + 1, v.y * rstd * io<T>::ld(weight + i + 1));
    io<T>::st(o + 2, v.z * rstd * io<T>::ld(weight + i + 2));
    io<T>::st(o + 3, v.w * rstd * io<T>::ld(weight + i + 3));
  }
}

}  // namespace sn

using namespace sn;

extern "C" {

sn_status sn_tp_arrive(unsigned int* counter, void* stream) {
  SN_REQUIRE(counter, "sn_tp_arrive: NULL counter");
  tp_arrive_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(counter);
  return check_launch("sn_tp_arrive");
}

sn_status sn_tp_allreduce_add_rmsnorm(const unsigned long long* peer_slabs, const unsigned long long* peer_counters,
                                      int world, int rank, int nsplit, float* residual, const void* weight, void* out,
                                      int rows, int dim, float eps, int dtype, void* stream) {
  SN_REQUIRE(peer_slabs && peer_counters && residual && weight && out, "sn_tp_allreduce_add_rmsnorm: NULL pointer");
  SN_REQUIRE(world >= 1 && rank >= 0 && rank < world, "sn_tp_allreduce_add_rmsnorm: rank %d of %d", rank, world);
  SN_REQUIRE(nsplit >= 1 && nsplit <= 8, "sn_tp_allreduce_add_rmsnorm: nsplit %d", nsplit);
  SN_REQUIRE(rows > 0 && dim > 0 && dim % 4 == 0, "sn_tp_allreduce_add_rmsnorm: bad shape");
  int cs = 8;  // CTAs per row: each owns dim / cs columns, one float4 per thread
  while (cs > 1 && (dim % (4 * cs) || dim / cs / 4 < 32)) cs >>= 1;
  SN_REQUIRE(dim / cs / 4 <= 256, "sn_tp_allreduce_add_rmsnorm: dim %d too large", dim);
  const int threads = ((dim / cs / 4 + 31) / 32) * 32;
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, tp_allreduce_add_rmsnorm_kernel<T>, peer_slabs, peer_counters, world,
                                       rank, nsplit, residual, (const T*)weight, (T*)out, rows, dim, eps);
    if (e != cudaSuccess) {
      set_error("sn_tp_allreduce_add_rmsnorm launch: %s", cudaGetErrorString(e));
      return SN_ECUDA;
    }
    return check_launch("sn_tp_allreduce_add_rmsnorm");
  });
}

}  // extern "C"
