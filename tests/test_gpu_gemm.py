"""tcgen05 decode GEMM vs an fp32 torch reference on the same bf16 operands
(all three fused epilogues, split-K clusters, ragged N, small batches)."""
import pytest
import torch

from paper_2604_19877_b200 import ops


def _ref(x, w):
    return x.float() @ w.float().t()


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.mark.gpu
@pytest.mark.parametrize("M", [1, 7, 16, 33, 64, 100, 128])
@pytest.mark.parametrize("N,K", [(300, 256), (5120, 4096), (1000, 1024), (131072, 512), (10304, 5120)])
def test_gemm_store(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm_decode(x, w, out, "store")
    torch.cuda.synchronize()
    assert rel(out, _ref(x, w)) < 8e-3


@pytest.mark.gpu
@pytest.mark.parametrize("M", [1, 64, 128])
@pytest.mark.parametrize("F,K", [(768, 512), (14336, 5120), (1000, 256)])
@pytest.mark.parametrize("mode", ["swiglu", "swiglu_il"])
def test_gemm_swiglu(M, F, K, mode):
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    out = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    wk = w if mode == "swiglu" else ops.interleave_swiglu(w, ops.gemm_swiglu_block(M, F, K))
    ops.gemm_decode(x, wk, out, mode)
    torch.cuda.synchronize()
    gu = _ref(x, w)
    ref = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    assert rel(out, ref) < 8e-3


@pytest.mark.gpu
@pytest.mark.parametrize("M", [3, 64])
@pytest.mark.parametrize("N,K", [(640, 4096), (5120, 14336), (300, 64)])
def test_gemm_resid_deterministic(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    r0 = torch.randn(M, N, device="cuda", generator=g)
    outs = []
    for _ in range(2):
        r = r0.clone()
        ops.gemm_decode(x, w, r, "resid")
        outs.append(r)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]), "GEMM must be deterministic"
    ref = r0 + _ref(x, w)
    assert ((outs[0] - ref).abs().max() / ref.abs().max()).item() < 5e-5


@pytest.mark.gpu
@pytest.mark.parametrize("M", [1, 64])
@pytest.mark.parametrize("N,K", [(5120, 4096), (5120, 14336), (256, 768)])
def test_gemm_partial_slabs_and_norm(M, N, K):
    """Split-K partial slabs summed by sn_add_rmsnorm reproduce residual + x @ w.T (deterministic)."""
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    slabs = torch.empty(8, M, N, device="cuda")
    S = ops.gemm_decode(x, w, slabs, "partial")
    assert 1 <= S <= 8 and S == ops.gemm_decode_splits(M, N, K)
    torch.cuda.synchronize()
    assert rel(slabs[:S].sum(0), _ref(x, w)) < 1e-5
    resid = torch.randn(M, N, device="cuda", generator=g)
    ref_resid = resid.clone() + slabs[:S].sum(0)
    nw = torch.rand(N, device="cuda", generator=g).to(torch.bfloat16) + 0.5
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.add_rmsnorm(None, resid, nw, out, 1e-5, partials=slabs, nsplit=S)
    torch.cuda.synchronize()
    assert (resid - ref_resid).abs().max().item() < 1e-5
    ref_out = ref_resid * torch.rsqrt(ref_resid.pow(2).mean(-1, keepdim=True) + 1e-5) * nw.float()
    assert rel(out, ref_out) < 1e-2
