"""Small workload that reaches every libsn100 kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) — tools/sanitize.sh runs it under each tool.

  * tiny supernet "ASKG", bf16 and fp32: embed, add+RMSNorm, decode GEMM (every epilogue:
    STORE / PARTIAL / SwiGLU / ATTN_IN), attention decode (FA + SWA ring), GDN / KDA decode,
    KDA gate factors, argmax; prefill: conv, delta prep, chunked GDN / KDA (bf16) and the token
    scan (fp32), mma.sync attention prefill (D=64), gated RMSNorm, SwiGLU;
  * the same decode through the fused decode chains (grid barriers, csrc/sn_chain.cu);
  * the tcgen05 attention prefill and the chunked prefill at head dim 128;
  * an idle slot (token -1) in one decode step.
"""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19877_b200 import TINY, ops  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402


def supernet_pass(dtype, chain):
    m = Supernet(TINY, "ASKG", batch=2, max_len=80, dtype=dtype, fused_chain=chain)
    toks = torch.randint(0, TINY.vocab, (2, 70), generator=torch.Generator().manual_seed(0))
    m.prefill(toks[:, :66])
    g = DecodeGraph(m, preserve_state=True)
    for t in range(66, 69):
        m.step_tokens.copy_(toks[:, t].to(torch.int32))
        g.replay()
    m.step_tokens.copy_(torch.tensor([int(toks[0, 69]), -1], dtype=torch.int32))  # slot 1 idle
    g.replay()
    torch.cuda.synchronize()


def attn_prefill_d128():
    T, Hq, Hkv, D = 300, 4, 1, 128
    q = torch.randn(T, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, Hkv, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0, 170, T], dtype=torch.int32, device="cuda")
    o = torch.empty(T, Hq * D, device="cuda", dtype=torch.bfloat16)
    for window in (0, 64):
        ops.attn_prefill(q, k, v, cu, o, Hq, Hkv, D, window, 1 / math.sqrt(D))
    torch.cuda.synchronize()


def chunk_prefill_d128():
    lens, Hk, Hv, D = [130, 40], 1, 2, 128
    T = sum(lens)
    g = torch.Generator().manual_seed(2)
    qn = torch.nn.functional.normalize(torch.randn(T, Hk, D, generator=g), dim=-1).cuda() / math.sqrt(D)
    kn = torch.nn.functional.normalize(torch.randn(T, Hk, D, generator=g), dim=-1).cuda()
    qkv = torch.randn(T, (2 * Hk + Hv) * D, generator=g).to(torch.bfloat16).cuda()
    glog = (-torch.rand(T, Hv, generator=g) * 0.3).cuda()
    beta = torch.rand(T, Hv, generator=g).cuda()
    cu = [0, lens[0], T]
    chunks, c0 = ops.chunk_plan(cu)
    S = torch.zeros(len(lens), Hv, D, D, device="cuda")
    o = torch.zeros(T, Hv, D, device="cuda")
    ops.gdn_chunk_prefill2(qn, kn, qkv, 2 * Hk * D, glog, beta, chunks, c0, o, S, None, Hk, Hv, D, init_state=False)
    glog_k = (-torch.rand(T, Hv, D, generator=g) * 0.3).cuda()
    qkv_k = torch.randn(T, 3 * Hv * D, generator=g).to(torch.bfloat16).cuda()
    qn_k = torch.nn.functional.normalize(torch.randn(T, Hv, D, generator=g), dim=-1).cuda() / math.sqrt(D)
    kn_k = torch.nn.functional.normalize(torch.randn(T, Hv, D, generator=g), dim=-1).cuda()
    ops.kda_chunk_prefill2(qn_k, kn_k, qkv_k, 2 * Hv * D, glog_k, beta, chunks, c0, o, S, None, Hv, D,
                           init_state=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    supernet_pass(torch.bfloat16, chain=False)
    supernet_pass(torch.float32, chain=False)
    supernet_pass(torch.bfloat16, chain=True)
    attn_prefill_d128()
    chunk_prefill_d128()
    print("sanitize workload done")
