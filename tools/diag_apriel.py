"""Diagnose Apriel-shaped parity: per placement / length group, the max rel error of the prefill
positions and of each decode step against the fp32 oracle (run on the GPU, TF32 off).

  python tools/diag_apriel.py AGKS 64 300,273,129,64 [eager]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.supernet_oracle import OracleSupernet  # noqa: E402  (checker)
from paper_2604_19877_b200 import APRIEL  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402
from paper_2604_19877_b200.placement import GDN, KDA, layer_kinds  # noqa: E402
from paper_2604_19877_b200.weights import cast_weights, init_weights  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


def poison(gb=60):
    """Fill the caching allocator's free blocks with NaN so reads of never-written memory show."""
    big = torch.full((int(gb * 2**30) // 4,), float("nan"), device="cuda")
    small = [torch.full((1 << 16,), float("nan"), device="cuda") for _ in range(2000)]
    del big, small


def main():
    if os.environ.get("POISON"):
        poison()
    for placement in sys.argv[1].split(","):
        run(placement)


def run(placement):
    B = int(sys.argv[2])
    LENS = [int(x) for x in sys.argv[3].split(",")]
    eager = len(sys.argv) > 4 and sys.argv[4] == "eager"
    window = int(os.environ.get("WINDOW", "256"))
    STEPS = 8
    cfg = APRIEL.scaled(num_layers=len(placement), window=window)
    dev = torch.device("cuda")
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(cfg, kinds, seed=0, device=dev), dev, torch.bfloat16)
    lens = [LENS[b % len(LENS)] for b in range(B)]
    g = torch.Generator().manual_seed(7)
    seqs = [torch.randint(0, cfg.vocab, (L + STEPS,), generator=g) for L in lens]
    model = Supernet(cfg, placement, batch=B, max_len=max(lens) + STEPS, dtype=torch.bfloat16, weights=w)
    pre = model.prefill([s[:L] for s, L in zip(seqs, lens)], return_all=True)
    graph = None if eager else DecodeGraph(model, preserve_state=True)
    dec = []
    for t in range(STEPS):
        tok = torch.tensor([int(s[L + t]) for s, L in zip(seqs, lens)], dtype=torch.int32)
        if eager:
            model.decode(tok)
        else:
            model.step_tokens.copy_(tok)
            graph.replay()
        dec.append(model.logits.clone())
    torch.cuda.synchronize()
    print(f"placement {placement} B={B} lens {LENS} {'eager' if eager else 'graph'} err_flag {int(model.err_flag.item())}")
    for L in sorted(set(lens)):
        members = [b for b in range(B) if lens[b] == L]
        toks = torch.stack([seqs[b] for b in members])
        oracle = OracleSupernet(cfg, kinds, w, batch=len(members), max_len=L + STEPS, device=dev)
        ref = oracle.run(toks)
        worst_pre = max(rel(pre[b], ref[i, :L]) for i, b in enumerate(members))
        worst_dec = [max(rel(dec[t][b], ref[i, L + t]) for i, b in enumerate(members)) for t in range(STEPS)]
        bad = [b for i, b in enumerate(members) if rel(dec[0][b], ref[i, L]) > 2e-2]
        st = {}
        for l, kind in enumerate(kinds):
            if kind in (GDN, KDA):
                st[l] = round(rel(model.recurrent_state(l)[members], oracle.recurrent_state(l)), 5)
        print(f"  len {L:4d} n={len(members):3d}: prefill {worst_pre:.2e}  decode " +
              " ".join(f"{e:.1e}" for e in worst_dec) + f"  states {st}  bad-slots {bad[:8]}")


if __name__ == "__main__":
    main()
