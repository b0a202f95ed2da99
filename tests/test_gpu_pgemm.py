"""Prefill projection GEMM (2-CTA tcgen05, csrc/sn_pgemm.cu) against a plain PyTorch fp32
reference of the same op: STORE and the fused SwiGLU epilogue, ragged M / N, K from one atom to
the FFN width, both block heights the wave-filling rule picks (224, 256), more tiles than CTA
pairs (the persistent walk), M not a multiple of the 256-row pair tile.  Tolerance: max-abs
error / max |ref| <= 1e-2 (bf16 output rounding, fp32 accumulate)."""
import pytest
import torch

TOL = 1e-2


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (127, 1000, 256), (300, 6144, 5120), (2100, 10304, 5120),
                                   (257, 5120, 14336), (4096, 256, 128),
                                   # Apriel widths at prompt sizes where the rule picks 224 or 256
                                   (16384, 5120, 256), (9000, 10304, 128), (5000, 6144, 192),
                                   (12345, 4000, 64)])
def test_store_matches_fp32_reference(M, N, K):
    from paper_2604_19877_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    out = ops.gemm_prefill(a, w)
    ref = a.float() @ w.float().t()
    assert out.shape == (M, N)
    assert rel(out, ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("M,F,K", [(5, 768, 256), (700, 14336, 5120), (4100, 14336, 256)])
def test_swiglu_epilogue_matches_reference(M, F, K):
    from paper_2604_19877_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(M + F)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    gu = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    h = ops.gemm_swiglu_block(F)
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    ops.gemm_prefill(a, ops.interleave_swiglu(gu, h), out, swiglu_h=h)
    x = a.float() @ gu.float().t()
    ref = torch.nn.functional.silu(x[:, :F]) * x[:, F:]
    assert rel(out, ref) <= TOL


@pytest.mark.gpu
def test_block_height_rule():
    """The block height fills the last wave of CTA pairs (host-side choice between 256 and 224,
    checked through the results: N = 5120 picks 224 at 16384 rows, 256 at 131072)."""
    from paper_2604_19877_b200 import ops
    for M in (16384, 131072):
        a = torch.randn(M, 128, device="cuda").to(torch.bfloat16)
        w = (torch.randn(5120, 128, device="cuda") * 0.05).to(torch.bfloat16)
        assert rel(ops.gemm_prefill(a, w), a.float() @ w.float().t()) <= TOL


@pytest.mark.gpu
def test_strided_operands():
    """A row-strided activation view (the in-projection columns of a wider buffer)."""
    from paper_2604_19877_b200 import ops
    a_full = torch.randn(200, 384, device="cuda").to(torch.bfloat16)
    a = a_full[:, 128:256]
    w = (torch.randn(512, 128, device="cuda") * 0.05).to(torch.bfloat16)
    out = ops.gemm_prefill(a, w)
    assert rel(out, a.float() @ w.float().t()) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(70, 256, 128), (3000, 5120, 512)])
def test_fp32_out_for_row_parallel_partials(M, N, K):
    """fp32 out (SN_GEMM_PARTIAL): the tensor-parallel prefill sums these partials in fp32."""
    from paper_2604_19877_b200 import ops
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.05).to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    ops.gemm_prefill(a, w, out)
    ref = a.float() @ w.float().t()
    assert ((out - ref).abs().max() / ref.abs().max()).item() <= 1e-4
