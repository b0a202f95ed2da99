"""Freeze FLA 0.5.1's own module kernels for the oracle pinning tests -> tests/golden/fla_modules.pt.

FLA realises the mixer details the paper leaves open: the GDN / KDA gate
functions, the L2 norm of q / k, the short causal convolution (prefill and its one-token
`ShortConvolution.step`) and the gated RMSNorm.  Its gate functions have torch references, but
the conv, L2 norm and gated norm exist only as Triton kernels, so this script runs on a GPU box:

    gpurun -- python tools/make_golden_fla_gpu.py     # writes gpurun_out/fla_modules.pt
    cp gpurun_out/fla_modules.pt tests/golden/

Inputs are small and seeded; the outputs of FLA's own code are what tests/test_oracle_pinning.py
compares oracle/supernet_oracle.py's restatements with (on the CPU, from the frozen file).
"""
from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(out_path):
    import fla
    from fla.modules.conv.short_conv import ShortConvolution
    from fla.modules.fused_norm_gate import FusedRMSNormGated
    from fla.modules.l2norm import l2norm
    from fla.ops.gated_delta_rule.gate import fused_gdn_gate, naive_gdn_gate
    from fla.ops.kda.gate import fused_kda_gate, naive_kda_gate

    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(17)
    out = {"fla_version": fla.__version__, "device": torch.cuda.get_device_name()}
    cpu = lambda t: t.detach().float().cpu()

    # gates (3P-FLA/ops/gated_delta_rule/gate.py:20-45, 3P-FLA/ops/kda/gate.py:26-54)
    B, T, Hv, H, K = 2, 5, 6, 3, 16
    a = torch.randn(B, T, Hv, generator=g) * 3
    A_log = torch.log(torch.rand(Hv, generator=g) * 16 + 1e-3)
    dt_bias = torch.randn(Hv, generator=g)
    out["gdn_gate"] = dict(a=a, A_log=A_log, dt_bias=dt_bias, naive=naive_gdn_gate(a, A_log, dt_bias),
                           fused=cpu(fused_gdn_gate(a.to(dev), A_log.to(dev), dt_bias.to(dev))))
    f = torch.randn(B, T, H, K, generator=g) * 3
    A_log_k = torch.log(torch.rand(H, generator=g) * 15 + 1)
    dt_bias_k = torch.randn(H * K, generator=g)
    out["kda_gate"] = dict(f=f, A_log=A_log_k, dt_bias=dt_bias_k, naive=naive_kda_gate(f, A_log_k, dt_bias_k),
                           fused=cpu(fused_kda_gate(f.to(dev), A_log_k.to(dev), dt_bias_k.to(dev))))

    # L2 norm (3P-FLA/modules/l2norm.py)
    x = torch.randn(40, 128, generator=g) * 2
    x[3] *= 1e-4  # small-norm row: the eps matters
    out["l2norm"] = dict(x=x, eps=1e-6, y=cpu(l2norm(x.to(dev), eps=1e-6)))

    # short causal conv + SiLU (3P-FLA/modules/conv/short_conv.py): prefill over T tokens with
    # the final cache, then three one-token steps from that cache
    C, W, T = 96, 4, 11
    conv = ShortConvolution(C, W, bias=False, activation="silu").to(dev)
    with torch.no_grad():
        conv.weight.copy_((torch.rand(C, 1, W, generator=g) * 2 - 1) * 0.5)
    xs = torch.randn(B, T, C, generator=g)
    steps = torch.randn(3, B, 1, C, generator=g)
    with torch.no_grad():
        y, cache = conv(xs.to(dev), output_final_state=True)
        cache_prefill = cpu(cache)
        ys = []
        for t in range(3):
            yt, cache = conv.step(steps[t].to(dev), None, cache, output_final_state=True)
            ys.append(cpu(yt))
    out["short_conv"] = dict(weight=cpu(conv.weight[:, 0]), x=xs, y=cpu(y), cache_prefill=cache_prefill,
                             steps=steps, y_steps=torch.stack(ys), cache_steps=cpu(cache))

    # gated RMSNorm (3P-FLA/modules/fused_norm_gate.py, FusedRMSNormGated): swish for GDN,
    # sigmoid for KDA, eps 1e-5, per head of 128
    D = 128
    o = torch.randn(30, 4, D, generator=g)
    gate = torch.randn(30, 4, D, generator=g) * 2
    wn = 1 + 0.1 * torch.randn(D, generator=g)
    res = {}
    for act in ("swish", "sigmoid"):
        m = FusedRMSNormGated(D, eps=1e-5, activation=act).to(dev)
        with torch.no_grad():
            m.weight.copy_(wn)
            res[act] = cpu(m(o.to(dev), gate.to(dev)))
    out["gated_norm"] = dict(o=o, gate=gate, weight=wn, eps=1e-5, **res)
    torch.save(out, out_path)
    print("wrote", out_path)


if __name__ == "__main__":
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "fla_modules.pt")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    main(path)
