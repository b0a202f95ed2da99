"""The A/B variants of the tcgen05 attention prefill (selected once per process by environment
switches, so each runs in a subprocess): one query tile per CTA with P in TMEM, P through
shared memory, 16 softmax warps, half of the exponentials on the FMA pipe — all against the
same fp32 reference as the default kernel."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import math, sys, torch
sys.path.insert(0, %r)
sys.path.insert(0, %r)
from test_gpu_attn_prefill import reference
from paper_2604_19877_b200 import ops
Hq, Hkv, D = 8, 2, 128
worst = 0.0
for lens, window in (([37, 200, 5, 64, 91], 0), ([700], 100), ([1100], 0)):
    g = torch.Generator().manual_seed(sum(lens) + window)
    T = sum(lens)
    q = torch.randn(T, Hq, D, generator=g).to(torch.bfloat16)
    k = (torch.randn(T, Hkv, D, generator=g) * torch.linspace(0.1, 6.0, T)[:, None, None]).to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32)
    out = torch.empty(T, Hq * D, dtype=torch.bfloat16, device="cuda")
    ops.attn_prefill(q.cuda(), k.cuda(), v.cuda(), cu.cuda(), out, Hq, Hkv, D, window, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    ref = reference(q, k, v, lens, window, 1 / math.sqrt(D)).reshape(T, Hq * D)
    worst = max(worst, ((out.float().cpu() - ref).abs().max() / ref.abs().max()).item())
print(worst)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"SN_FA5_TWO": "0"}, {"SN_FA5_TWO": "0", "SN_FA5_PTMEM": "0"},
                                 {"SN_FA5_TWO": "0", "SN_FA5_SLICES": "4"},
                                 {"SN_FA5_TWO": "0", "SN_FA5_SLICES": "4", "SN_FA5_PTMEM": "0"},
                                 {"SN_FA5_TWO": "0", "SN_FA5_POLY": "2"}])
def test_attn_prefill_variant(env):
    code = SCRIPT % (ROOT, os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) < 2e-2, r.stdout
