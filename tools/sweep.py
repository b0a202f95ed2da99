"""Preset sweep (BASELINE.json config 4).

Decode tokens/s of every paper preset (all-FA ... Reg|Lklhd-10) at 8K / 32K / 128K context,
per-GPU batch = min(64, HBM capacity), plus a few random mixed placements (every count 0 or
>= 3, R/PAPER.md:1802) at 32K.  Under torchrun each rank decodes its own batch (batch
sharding, no collective) and the reported tokens/s is the sum over ranks, timed as the max
over ranks.  Writes:
  --records  ThroughputRecord JSONL (R/SPEC.md:192) at one context, the input of the
             reference's `placeopt fit-cost --records ... --out cost.json`;
  --out      one JSON object per measurement (preset, context, batch, tok/s, step GB/s,
             fraction of the measured HBM peak).

  python tools/sweep.py --contexts 8192,32768,131072 --records gpurun_out/b200_records.jsonl \
      --out gpurun_out/sweep.jsonl
"""
import argparse
import json
import os
import random
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import barrier, dist_setup, fill_synthetic, load_peaks, max_over_ranks  # noqa: E402
from paper_2604_19877_b200 import APRIEL, PRESETS, roofline  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402
from paper_2604_19877_b200.placement import DEFAULT_CATALOG, layer_kinds, spread_layer_string  # noqa: E402
from paper_2604_19877_b200.records import throughput_record  # noqa: E402


def capacity_batch(cfg, kinds, max_len, reserve_gb=6.0, cap=64):
    free, _ = torch.cuda.mem_get_info()
    page = cfg.page_size
    padded = -(-max_len // page) * page
    per_seq = sum(roofline.mixer_state_bytes(cfg, k, padded) for k in kinds)
    weights = roofline.weight_bytes(cfg, kinds) + cfg.vocab * cfg.hidden * 2
    avail = free - weights - reserve_gb * 1e9
    return max(1, min(cap, int(avail // max(per_seq, 1))))


def random_allocations(n, L, seed=7):
    """Allocations with every count 0 or >= 3 (the paper's class-size rule)."""
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        cuts = sorted(rng.sample(range(1, L), 3))
        c = [cuts[0], cuts[1] - cuts[0], cuts[2] - cuts[1], L - cuts[2]]
        c = [x if x >= 3 else 0 for x in c]
        c[3] += L - sum(c)
        if all(x == 0 or x >= 3 for x in c) and tuple(c) not in out:
            out.append(tuple(c))
    return out


def measure(cfg, layer_string, B, ctx, steps, warmup, ws):
    m = Supernet(cfg, layer_string, batch=B, max_len=ctx + warmup + steps + 8, dtype=torch.bfloat16, seed=0)
    g = DecodeGraph(m, feedback=True, preserve_state=False)  # warm-up + capture on the empty engine (it resets)
    fill_synthetic(m, ctx)  # then the KV pools / states at the context length
    for _ in range(warmup):
        g.replay()
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(e0.elapsed_time(e1), ws) / steps
    nbytes = roofline.step_bytes(cfg, layer_kinds(layer_string), B, ctx)
    del g, m
    torch.cuda.empty_cache()
    return ms, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--contexts", default="8192,32768,131072")
    ap.add_argument("--presets", default=",".join(p for p in PRESETS if p != "Idealized|All-6"))
    ap.add_argument("--random", type=int, default=6, help="random mixed placements at the records context")
    ap.add_argument("--records-context", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--records", default="")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ws, rank, _ = dist_setup()
    cfg = APRIEL
    peak, _src = load_peaks()
    jobs = [(name, PRESETS[name].layer_string, int(c)) for c in a.contexts.split(",") for name in a.presets.split(",")]
    for counts in random_allocations(a.random, cfg.num_layers):
        jobs.append(("random" + "".join(f"{DEFAULT_CATALOG.short_codes[i]}{n}" for i, n in enumerate(counts)),
                     spread_layer_string(counts), a.records_context))
    rows, records = [], []
    for name, ls, ctx in jobs:
        kinds = layer_kinds(ls)
        B = capacity_batch(cfg, kinds, ctx + a.warmup + a.steps + 8, cap=a.batch)
        ms, nbytes = measure(cfg, ls, B, ctx, a.steps, a.warmup, ws)
        tok_s = ws * B / (ms / 1e3)
        row = {"preset": name, "placement": ls, "context": ctx, "batch_per_gpu": B, "n_gpus": ws, "tok_s": tok_s,
               "ms_per_step": ms, "step_gbs": nbytes / (ms * 1e6), "frac_of_peak": nbytes / (ms * 1e6) / peak,
               "frac_of_8tbs": nbytes / (ms * 1e6) / 8000}
        rows.append(row)
        if ctx == a.records_context:
            records.append(throughput_record(ls, tok_s))
        if rank == 0:
            print(json.dumps(row), flush=True)
    if rank == 0:
        if a.out:
            with open(a.out, "w") as f:
                for r in rows:
                    f.write(json.dumps(r) + "\n")
        if a.records:
            with open(a.records, "w") as f:
                for r in records:
                    f.write(json.dumps(r, sort_keys=True) + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
