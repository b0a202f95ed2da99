"""Causal depthwise conv (width 4) + SiLU over packed ragged sequences (sn_conv_prefill) vs a
plain fp32 reference: the bf16 two-channel kernel (even channel count and stride) and the
generic kernel (odd channels, fp32), fresh prompts and continuations from a ring snapshot,
and the conv ring left for decode (slot P % W holds the input of absolute position P)."""
import pytest
import torch

W = 4


def reference(x, w, lens, pos0, hist):
    """x [rows, C] fp32, w [C, W], hist [S, C, W] ring snapshot or None -> y [rows, C], last inputs."""
    out, tails, t0 = [], [], 0
    for s, L in enumerate(lens):
        p0 = pos0[s]
        prev = torch.zeros(W - 1, x.shape[1])
        for d in range(1, W):  # absolute position p0 - d
            P = p0 - d
            if P >= 0 and hist is not None:
                prev[W - 1 - d] = hist[s, :, P % W]
        seq = torch.cat([prev, x[t0:t0 + L]])
        y = sum(w[:, k] * seq[k:k + L] for k in range(W))
        out.append(torch.nn.functional.silu(y))
        tails.append(seq[-(W - 1):])  # inputs of absolute positions p0+L-3 .. p0+L-1
        t0 += L
    return torch.cat(out), tails


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,channels,stride", [(torch.bfloat16, 64, 70), (torch.bfloat16, 37, 41),
                                                   (torch.float32, 64, 70)])
@pytest.mark.parametrize("continuation", [False, True])
def test_conv_prefill(dtype, channels, stride, continuation):
    from paper_2604_19877_b200 import ops
    g = torch.Generator().manual_seed(channels + stride + int(continuation))
    lens = [1, 70, 3, 130]
    S, rows = len(lens), sum(lens)
    pos0 = [0, 5, 2, 200] if continuation else [0] * S
    xs = torch.randn(rows, stride, generator=g).to(dtype)
    w = torch.randn(channels, W, generator=g).to(dtype)
    hist = torch.randn(S, channels, W, generator=g).to(dtype) if continuation else None
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
    slots = torch.tensor([2, 0, 3, 1], dtype=torch.int32, device="cuda")
    ring = torch.zeros(4, channels, W, dtype=dtype, device="cuda")
    y = torch.empty(rows, channels, dtype=dtype, device="cuda")
    ops.conv_prefill(xs.cuda(), stride, y, w.cuda(), ring, cu, slots, channels, W,
                     ring_hist=hist.cuda() if continuation else None,
                     pos0=torch.tensor(pos0, dtype=torch.int32, device="cuda") if continuation else None)
    torch.cuda.synchronize()
    ref, tails = reference(xs[:, :channels].float(), w.float(), lens, pos0,
                           hist.float() if continuation else None)
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    err = ((y.float().cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < tol, err
    ring = ring.float().cpu()
    for s, L in enumerate(lens):
        for d in range(1, W):
            P = pos0[s] + L - d
            if P < 0:
                continue
            assert torch.equal(ring[int(slots[s]), :, P % W], tails[s][W - 1 - d].to(dtype).float()), (s, d)
