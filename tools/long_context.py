"""BASELINE.json config 5: one long sequence — chunked prefill of T tokens, then graphed decode.

  python tools/long_context.py --tokens 131072 [--preset 'Reg|Lklhd-10'] [--decode 64]
  python tools/long_context.py --gpus N ...   # head-parallel TP over N GPUs (self-launches torchrun)
                                                           # (one all-reduce per row-parallel projection)
Prints one JSON line: prefill tokens/s and decode tokens/s (B = 1), timed with CUDA events
(max over ranks under torchrun).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import barrier, dist_setup, max_over_ranks  # noqa: E402
from paper_2604_19877_b200 import APRIEL, PRESETS  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--tokens", type=int, default=131072)
ap.add_argument("--decode", type=int, default=64)
ap.add_argument("--gpus", type=int, default=1, help="head-parallel ranks (self-launches torchrun, one per GPU)")
a = ap.parse_args()
if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
    from bench import self_launch
    sys.exit(self_launch(a.gpus))  # fails loudly when the box has fewer GPUs
if int(os.environ.get("WORLD_SIZE", "1")) != a.gpus:
    sys.exit(f"long_context.py: --gpus {a.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
ws, rank, _ = dist_setup()
tp_group = None
if ws > 1:
    import torch.distributed as dist
    tp_group = dist.group.WORLD
layers = PRESETS[a.preset].layer_string
m = Supernet(APRIEL, layers, batch=1, max_len=a.tokens + a.decode + 8, dtype=torch.bfloat16, tp_group=tp_group)
toks = torch.randint(0, APRIEL.vocab, (1, a.tokens), generator=torch.Generator().manual_seed(1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
barrier(ws)
torch.cuda.synchronize()
e0.record()
m.prefill(toks)
e1.record()
torch.cuda.synchronize()
prefill_ms = max_over_ranks(e0.elapsed_time(e1), ws)
g = DecodeGraph(m, feedback=True, preserve_state=True)  # decode continues the prefilled context
for _ in range(3):
    g.replay()
barrier(ws)
torch.cuda.synchronize()
e0.record()
for _ in range(a.decode):
    g.replay()
e1.record()
torch.cuda.synchronize()
dec_ms = max_over_ranks(e0.elapsed_time(e1), ws) / a.decode
if rank == 0:
    print(json.dumps({"workload": "long-context (config 5)", "preset": a.preset, "placement": layers,
                      "tokens": a.tokens, "n_gpus": ws, "parallelism": f"head-parallel tp{ws}" if ws > 1 else "tp1",
                      "prefill_ms": prefill_ms, "prefill_tok_s": a.tokens / prefill_ms * 1e3,
                      "decode_ms_per_token": dec_ms, "decode_tok_s": 1e3 / dec_ms,
                      "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
