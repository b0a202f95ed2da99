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
#include "sn_common.cuh"

namespace sn {

__global__ void tp_arrive_kernel(unsigned int* counter) {
  __threadfence_system();
  atomicAdd(counter, 1u);
}

template <typename T>
__global__ void __launch_bounds__(256)
    tp_allreduce_add_rmsnorm_kernel(const unsigned long long* __restrict__ peer_slabs,
                                    const unsigned long long* __restrict__ peer_counters, int world, int rank,
                                    int nsplit, float* __restrict__ residual, const T* __restrict__ weight,
                                    T* __restrict__ out, int rows, int dim, float eps) {
  sn::pdl_launch_dependents();
  sn::pdl_wait();
  __shared__ float scratch[32];
  if (threadIdx.x == 0) {
    const unsigned mine = *reinterpret_cast<volatile unsigned*>(peer_counters[rank]);
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      const volatile unsigned* c = reinterpret_cast<const volatile unsigned*>(peer_counters[r]);
      while ((int)(*c - mine) < 0) __nanosleep(64);
    }
    __threadfence_system();
  }
  __syncthreads();
  const int row = blockIdx.x;
  const size_t slab = (size_t)rows * dim;
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < dim; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(residual + (size_t)row * dim + i);
    for (int r = 0; r < world; ++r) {
      const float* base = reinterpret_cast<const float*>(peer_slabs[r]) + (size_t)row * dim + i;
      for (int s = 0; s < nsplit; ++s) {
        const float4 p = __ldcv(reinterpret_cast<const float4*>(base + s * slab));  // peers' memory: no stale lines
        v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
      }
    }
    *reinterpret_cast<float4*>(residual + (size_t)row * dim + i) = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum(ss, scratch);
  const float rstd = rsqrtf(ss / (float)dim + eps);
  for (int i = threadIdx.x * 4; i < dim; i += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(residual + (size_t)row * dim + i);
    io<T>::st(out + (size_t)row * dim + i, v.x * rstd * io<T>::ld(weight + i));
    io<T>::st(out + (size_t)row * dim + i + 1, v.y * rstd * io<T>::ld(weight + i + 1));
    io<T>::st(out + (size_t)row * dim + i + 2, v.z * rstd * io<T>::ld(weight + i + 2));
    io<T>::st(out + (size_t)row * dim + i + 3, v.w * rstd * io<T>::ld(weight + i + 3));
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
  return SN_DISPATCH_DTYPE(dtype, T, [&] {
    launch_pdl(tp_allreduce_add_rmsnorm_kernel<T>, dim3(rows), dim3(256), 0, (cudaStream_t)stream, peer_slabs,
               peer_counters, world, rank, nsplit, residual, (const T*)weight, (T*)out, rows, dim, eps);
    return check_launch("sn_tp_allreduce_add_rmsnorm");
  });
}

}  // extern "C"
