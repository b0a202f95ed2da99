#!/usr/bin/env python
"""bench.py — decode tokens/s of the Super Apriel supernet per placement preset,
with the HBM roofline fraction (BASELINE.json metric).

Workload (BASELINE.json config 3): Apriel-1.6-shaped 48-layer random-init
supernet, fastest hybrid preset Reg|Lklhd-10 (0 FA / 10 SWA / 5 KDA / 33 GDN),
batch 64 per GPU, fixed 32K-token context, bf16 weights/activations, fp32
recurrent state.  KV pools and recurrent states are filled synthetically to
the target length (decode cost is content-independent).  One "step" = one
decode token for every sequence: one replay of the placement's CUDA graph.
The per-step working set (~50 GB) is far larger than the 126 MB L2, so no L2
flush is needed between steps.  The all-FA preset is measured beside it at
its HBM-capacity-capped batch for the paper's ~10x long-context speedup.

  python bench.py [--gpus N --steps K --warmup W]           # our CUDA path
  python bench.py --impl reference [...]                     # CPU oracle arm
Under torchrun each rank decodes its own batch (weak scaling, no data-path
collective), rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2604_19877_b200 import APRIEL, PRESETS  # noqa: E402
from paper_2604_19877_b200.placement import FA, GDN, KDA, SWA, layer_kinds  # noqa: E402
from paper_2604_19877_b200 import roofline  # noqa: E402

METRIC = "decode tokens/s (Apriel-48L supernet, preset Reg|Lklhd-10, batch 64 x 32K context)"
UNIT = "tokens/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def self_launch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with one rank
    per GPU (NCCL, 127.0.0.1 rendezvous).  Fails loudly when the box has fewer than N GPUs
    instead of measuring one GPU and calling it N."""
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} requested but this box has {have} visible GPU(s)", file=sys.stderr)
        return 2
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the driver can see the communicator's rank count
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(sys.argv[0])] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ synthetic state
def fill_synthetic(model, ctx: int, seed: int = 1234):
    g = torch.Generator(device=model.device)
    g.manual_seed(seed)
    model.seq_lens.fill_(ctx)
    for st, kind in zip(model.state, model.kinds):
        if kind in (FA, SWA):
            st["k"].normal_(0.0, 1.0, generator=g)
            st["v"].normal_(0.0, 1.0, generator=g)
        else:
            st["S"].normal_(0.0, 0.05, generator=g)
            st["conv"].normal_(0.0, 0.5, generator=g)
    torch.cuda.synchronize()


def fa_capacity_batch(cfg, kinds, max_len, reserve_gb=8.0):
    free, _ = torch.cuda.mem_get_info()
    per_seq = sum(2 * math.ceil(max_len / cfg.page_size) * cfg.page_size * roofline.kv_token_bytes(cfg) // 2
                  for k in kinds if k == FA)
    weights = roofline.weight_bytes(cfg, kinds) + cfg.vocab * cfg.hidden * 2  # + embedding table
    avail = free - weights - reserve_gb * 1e9
    return max(1, min(64, int(avail // max(per_seq, 1))))


# ------------------------------------------------------------------ our path
def measure_preset(cfg, preset, B, ctx, steps, warmup, ws, rank, local, probe_steps=10, e2e=True):
    from paper_2604_19877_b200.graphs import DecodeGraph
    from paper_2604_19877_b200.model import KernelProbe, Supernet

    kinds = layer_kinds(PRESETS[preset].layer_string)
    extra = warmup + 2 * steps + probe_steps + 16
    model = Supernet(cfg, PRESETS[preset].layer_string, batch=B, max_len=ctx + extra, dtype=torch.bfloat16,
                     seed=0)
    graph = DecodeGraph(model, feedback=True)  # warm-up + capture on the empty engine (then reset)
    fill_synthetic(model, ctx)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        graph.replay()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local, ws)

    res = {"preset": preset, "B": B, "ctx": ctx, "kinds": kinds, "ms_per_step": ms / steps,
           "tok_s": ws * B * steps / (ms / 1e3), "clocks": clk,
           "launches_per_step": model.kernels_per_step()}

    if e2e:  # public API, host tokens in / host tokens out every step
        toks = torch.randint(0, cfg.vocab, (B,), dtype=torch.int32)
        graph.step_host(toks)
        barrier(ws)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            toks = graph.step_host(toks)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        ms_e2e = max_over_ranks(e0.elapsed_time(e1), ws)
        res["e2e"] = {"value": ws * B * steps / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * 4,
                      "d2h_bytes_per_step": B * 4, "ms_per_step": ms_e2e / steps}

    # per-kernel device time inside the step: a second capture with timing events around
    # every mixer kernel (graph event-record nodes on the launching stream)
    model.probe = KernelProbe(fine=True)
    pgraph = DecodeGraph(model, feedback=True, preserve_state=False, warmup=0)
    model.probe_pairs = model.probe
    model.probe = None
    per = {}
    for _ in range(probe_steps):
        pgraph.replay()
        torch.cuda.synchronize()
        for n, v in model.probe_pairs.collect().items():
            per.setdefault(n, []).extend(v)
    kernels = {}
    for n, v in per.items():
        launches = len(v) // probe_steps
        mean_ms = sum(v) / len(v)
        step_b = roofline.role_step_bytes(cfg, kinds, n, B, ctx)
        nbytes = step_b // launches if step_b is not None else None
        kernels[n] = {"launches_per_step": launches, "ms_per_launch": mean_ms,
                      "share_of_step": launches * mean_ms / res["ms_per_step"],
                      "bytes_per_launch": nbytes, "gbs": nbytes / (mean_ms * 1e6) if nbytes else None}
    res["kernels"] = kernels
    res["step_bytes"] = roofline.step_bytes(cfg, kinds, B, ctx)
    del graph, pgraph, model
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ prefill (side measurement)
def measure_prefill(cfg, preset, tokens, reps=2):
    """One prompt of `tokens` tokens through the chunked / tensor-core prefill (B=1): tokens/s
    with CUDA events, plus the attention-prefill kernel alone (TFLOP/s of the masked
    attention, causal, same length, Apriel heads)."""
    from paper_2604_19877_b200 import ops
    from paper_2604_19877_b200.model import Supernet
    model = Supernet(cfg, PRESETS[preset].layer_string, batch=1, max_len=tokens, dtype=torch.bfloat16, seed=0)
    toks = torch.randint(0, cfg.vocab, (1, tokens), generator=torch.Generator().manual_seed(1))
    model.prefill(toks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        model.prefill(toks)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del model
    torch.cuda.empty_cache()
    Hq, Hkv, D = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
    q = torch.randn(tokens, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(tokens, Hkv, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(tokens, Hkv, D, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0, tokens], dtype=torch.int32, device="cuda")
    o = torch.empty(tokens, Hq * D, device="cuda", dtype=torch.bfloat16)
    ops.attn_prefill(q, k, v, cu, o, Hq, Hkv, D, 0, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        ops.attn_prefill(q, k, v, cu, o, Hq, Hkv, D, 0, 1 / math.sqrt(D))
    e1.record()
    torch.cuda.synchronize()
    attn_ms = e0.elapsed_time(e1) / 3
    flops = 4.0 * (tokens * (tokens + 1) / 2) * Hq * D
    return {"preset": preset, "tokens": tokens, "batch": 1, "ms": best, "tok_s": tokens / best * 1e3,
            "attention_kernel": {"mask": "causal", "ms": attn_ms, "tflops": flops / attn_ms / 1e9,
                                 "kernel": "tcgen05/TMEM flash attention (sn_attn_prefill_umma.cu)"}}


# ------------------------------------------------------------------ CPU reference (oracle) arm
class CPUComposedStep:
    """One decode step of a preset on the CPU fp32 oracle, composed from one measured layer per
    mixer type (+ one FFN layer, + LM head) weighted by the allocation — the reference's own
    additive cost model (R/pkg/src/placeopt/cost.py:73-80).  Weights/KV are built once."""

    def __init__(self, cfg, counts, B, ctx, threads):
        from oracle.supernet_oracle import attention_ref, gdn_core, kda_core, rmsnorm, rope
        from paper_2604_19877_b200.weights import init_mixer

        torch.set_num_threads(threads)
        self.cfg, self.counts, self.B = cfg, counts, B
        g = torch.Generator().manual_seed(0)
        d, F = cfg.hidden, cfg.ffn
        x = torch.randn(B, d, generator=g)
        nw = torch.ones(d)
        gu = torch.randn(2 * F, d, generator=g) * 0.02
        dn = torch.randn(d, F, generator=g) * 0.02
        lm = torch.randn(cfg.vocab, d, generator=g) * 0.02
        self.fns = {}

        def ffn():
            h = rmsnorm(x, nw, cfg.norm_eps) @ gu.T
            return (torch.nn.functional.silu(h[:, :F]) * h[:, F:]) @ dn.T
        self.fns["ffn_layer"] = ffn
        self.fns["lm_head"] = lambda: (rmsnorm(x, nw, cfg.norm_eps) @ lm.T).argmax(-1)
        for kind, n in zip((FA, SWA, KDA, GDN), counts):
            if n == 0:
                continue
            w = init_mixer(cfg, 0, kind, seed=0)
            name = ("FA", "SWA", "KDA", "GDN")[kind]
            if kind in (FA, SWA):
                S = ctx if kind == FA else min(ctx, cfg.window)
                keys = torch.randn(B, S, cfg.n_kv_heads, cfg.head_dim, generator=g)
                vals = torch.randn(B, S, cfg.n_kv_heads, cfg.head_dim, generator=g)
                inv = cfg.inv_freq().float()
                Hq, Hkv, D = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim

                def attn(w=w, keys=keys, vals=vals):
                    p = rmsnorm(x, nw, cfg.norm_eps) @ w["qkv"].T
                    pos = torch.full((B,), ctx, dtype=torch.long)
                    q = rope(p[:, :Hq * D].view(B, Hq, D), pos, inv)
                    keys[:, -1] = rope(p[:, Hq * D:(Hq + Hkv) * D].view(B, Hkv, D), pos, inv)
                    vals[:, -1] = p[:, (Hq + Hkv) * D:].view(B, Hkv, D)
                    return attention_ref(q, keys, vals, D ** -0.5).reshape(B, -1) @ w["o"].T
                self.fns[name] = attn
            else:
                if kind == GDN:
                    Hv, Dd, C, core = cfg.gdn_v_heads, cfg.gdn_head_dim, cfg.gdn_conv_channels, gdn_core
                else:
                    Hv, Dd, C, core = cfg.kda_heads, cfg.kda_head_dim, cfg.kda_conv_channels, kda_core
                Sst = torch.randn(B, Hv, Dd, Dd, generator=g) * 0.05
                hist = torch.randn(B, C, cfg.conv_width - 1, generator=g)

                def delta(w=w, Sst=Sst, hist=hist, core=core):
                    p = rmsnorm(x, nw, cfg.norm_eps) @ w["w_in"].T
                    o, _, _ = core(cfg, p, hist, Sst, w)
                    return o @ w["o"].T
                self.fns[name] = delta

    @torch.no_grad()
    def run(self):
        times = {}
        for name, fn in self.fns.items():
            t = time.perf_counter()
            fn()
            times[name] = time.perf_counter() - t
        step = times["lm_head"] + self.cfg.num_layers * times["ffn_layer"]
        for name, n in zip(("FA", "SWA", "KDA", "GDN"), self.counts):
            if n:
                step += n * times[name]
        return step, times


def cpu_baseline(cfg, preset, B_cpu, ctx):
    threads = os.cpu_count() or 1
    runner = CPUComposedStep(cfg, PRESETS[preset].counts, B_cpu, ctx, threads)
    runner.run()
    samples = [runner.run() for _ in range(3)]
    step, times = min(samples, key=lambda s: s[0])
    return {"value": B_cpu / step, "unit": UNIT, "cores": threads, "kind": "port", "composed": True,
            "batch": B_cpu,
            "sample": (f"CPU fp32 oracle (oracle/supernet_oracle.py), batch {B_cpu} x {ctx} context: one decode "
                       f"step of one layer per mixer type + one FFN layer + LM head, composed over the "
                       f"{preset} allocation {PRESETS[preset].counts} (additive cost model, "
                       f"R/pkg/src/placeopt/cost.py:73-80); per-layer seconds {json.dumps({k: round(v, 4) for k, v in times.items()})}")}


def run_reference(args):
    """The reference arm: the CPU fp32 oracle (the reference ships no implementation of this
    path) on the same preset, batch and context as our arm, on all host threads.
    A step is COMPOSED (marked "composed": true): one decode step of one layer per mixer type,
    one FFN layer and the LM head are executed and timed, then weighted by the preset's
    allocation — the reference's own additive cost model (R/pkg/src/placeopt/cost.py:73-80) —
    because an executed 48-layer fp32 step at B=64 does not fit the host's RAM or a
    minutes-long run.  The seconds actually executed are reported beside the composed ones."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = APRIEL
    B_cpu = args.cpu_batch
    threads = os.cpu_count() or 1
    runner = CPUComposedStep(cfg, PRESETS[args.preset].counts, B_cpu, args.context, threads)
    for _ in range(args.warmup):
        runner.run()
    t, executed, per = 0.0, 0.0, {}
    w0 = time.perf_counter()
    for _ in range(args.steps):
        s, detail = runner.run()
        t += s
        for k, v in detail.items():
            per[k] = per.get(k, 0.0) + v / args.steps
    executed = time.perf_counter() - w0
    value = B_cpu * args.steps / t
    counts = PRESETS[args.preset].counts
    mult = {"lm_head": 1, "ffn_layer": cfg.num_layers}
    mult.update({n: c for n, c in zip(("FA", "SWA", "KDA", "GDN"), counts) if c})
    sample = (f"CPU fp32 oracle, batch {B_cpu} x {args.context} context; each step = one decode step of one "
              f"layer per mixer type + one FFN layer + LM head, executed, then composed over the {args.preset} "
              f"allocation {counts} (R/pkg/src/placeopt/cost.py:73-80)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, random KV/state)",
            "config": {"workload": "apriel48-decode", "preset": args.preset,
                       "placement": PRESETS[args.preset].layer_string, "batch_per_gpu": B_cpu,
                       "global_batch": B_cpu, "context": args.context},
            "composed": True,
            "composition": {"per_layer_seconds": {k: round(v, 5) for k, v in per.items()},
                            "multiplicity": mult, "executed_seconds_timed_region": round(executed, 3),
                            "composed_seconds_timed_region": round(t, 3)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "composed": True},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--preset", default="Reg|Lklhd-10")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--context", type=int, default=32768)
    ap.add_argument("--cpu-batch", type=int, default=None,
                    help="batch of the CPU oracle legs (default: --batch, i.e. the same config)")
    ap.add_argument("--no-fa-compare", action="store_true")
    ap.add_argument("--prefill-tokens", type=int, default=16384, help="side measurement; 0 = skip")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    env_ws = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and env_ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws} (launch one rank per GPU)", file=sys.stderr)
        return 2
    if args.cpu_batch is None:
        args.cpu_batch = args.batch
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)

    ws, rank, local = dist_setup()
    cfg = APRIEL
    peak, peak_src = load_peaks()
    main_res = measure_preset(cfg, args.preset, args.batch, args.context, args.steps, args.warmup, ws, rank, local)

    fa_res = None
    if not args.no_fa_compare:
        kinds_fa = layer_kinds(PRESETS["all-FA"].layer_string)
        extra = args.warmup + 2 * args.steps + 26
        B_fa = fa_capacity_batch(cfg, kinds_fa, args.context + extra)
        fa_res = measure_preset(cfg, "all-FA", B_fa, args.context, max(10, args.steps // 4), args.warmup, ws, rank,
                                local, probe_steps=3, e2e=False)

    if rank != 0:
        return 0
    kernels = main_res["kernels"]
    # dominant kernel: the largest share of the step among the bandwidth-bound roles (the
    # probe brackets every launch with graph event nodes, which breaks PDL overlap, so the
    # per-launch times here are slightly above the in-step ones)
    dom = max((n for n in kernels if kernels[n]["bytes_per_launch"]),
              key=lambda n: kernels[n]["launches_per_step"] * kernels[n]["ms_per_launch"])
    kd = kernels[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    step_gbs = main_res["step_bytes"] / (main_res["ms_per_step"] * 1e6)
    per_step_launches = main_res["launches_per_step"]
    out = {
        "metric": METRIC, "value": main_res["tok_s"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights; KV pools / recurrent states filled to the context length)",
        "config": {"workload": "apriel48-decode", "preset": args.preset,
                   "placement": PRESETS[args.preset].layer_string, "batch_per_gpu": args.batch,
                   "global_batch": args.batch * ws, "context": args.context,
                   "l2": "no flush: per-step working set %.1f GB >> 126 MB L2" % (main_res["step_bytes"] / 1e9),
                   "parallelism": f"batch-sharded x{ws} (no collective)"},
        "e2e": main_res.get("e2e"),
        "gpu_launches": per_step_launches["sn"] * args.steps,
        "clocks": {k: main_res["clocks"][k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kd["gbs"], "peak": peak, "unit": "GB/s",
                     "frac": kd["gbs"] / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": kd["bytes_per_launch"], "ms_per_launch": kd["ms_per_launch"]},
        "step_roofline": {"achieved": step_gbs, "peak": peak, "frac": step_gbs / peak, "frac_of_8tbs": step_gbs / 8000,
                          "bytes_per_step": main_res["step_bytes"]},
        "kernels": kernels,
        "launches_per_step": per_step_launches,
    }
    if fa_res is not None:
        fa_gbs = fa_res["step_bytes"] / (fa_res["ms_per_step"] * 1e6)
        out["all_fa"] = {"batch_per_gpu": fa_res["B"], "tok_s": fa_res["tok_s"], "ms_per_step": fa_res["ms_per_step"],
                         "step_gbs": fa_gbs, "step_frac": fa_gbs / peak,
                         "speedup_of_preset": main_res["tok_s"] / fa_res["tok_s"],
                         "note": "all-FA batch capped by HBM capacity at this context",
                         "kernels": fa_res["kernels"]}
    if ws == 1 and args.prefill_tokens > 0:
        out["prefill"] = measure_prefill(cfg, args.preset, args.prefill_tokens)
    if ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, args.preset, args.cpu_batch, args.context)
    print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
