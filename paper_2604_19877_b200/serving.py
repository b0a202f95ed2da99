"""Multi-placement serving on one resident supernet.

The paper serves several placements from one set of supernet weights: "CUDA graphs are
pre-captured for allowed placements, and at runtime the model runner selects the correct
graph" by `placement_id`, with no global mutable state (R/PAPER.md:860-865, 875-880; Table 8
R/PAPER.md:1872-1896).  Here:

* `SupernetStore` keeps the shared trunk (embedding, norms, FFN, LM head) resident once and
  materialises each (layer, mixer) weight set on first use — every layer can hold all four
  mixers (R/PAPER.md:239-241).  The tensors are the ones `weights.init_weights` draws for
  the same seed, so a placement built from the store equals a standalone `Supernet`.  The
  decode layout of the FFN gate/up weights (SwiGLU-interleaved) is built once per layer and
  shared by every engine.
* `PlacementRouter` holds one engine (state pools + decode CUDA graph) per
  (placement, batch) and routes requests by placement: same-placement requests are batched
  together (ragged prompt lengths in one packed prefill), then decoded greedily through
  their placement's graph.
"""
from __future__ import annotations

from collections import OrderedDict

import torch

from . import ops
from .config import SupernetConfig
from .placement import DEFAULT_CATALOG, coerce_placement, layer_kinds
from .weights import init_mixer, init_trunk


def _to(obj, device):
    if isinstance(obj, dict):
        return {k: _to(v, device) for k, v in obj.items()}
    if isinstance(obj, list):
        return [_to(v, device) for v in obj]
    return obj.to(device) if torch.is_tensor(obj) else obj


def placement_code(placement) -> str:
    return coerce_placement(placement).to_codes(DEFAULT_CATALOG)


class SupernetStore:
    """Resident supernet weights: the trunk once, each (layer, mixer kind) on first use."""

    def __init__(self, cfg: SupernetConfig, seed: int = 0, device="cuda", dtype=torch.bfloat16, init_device=None):
        """init_device: where the seeded draws happen (default: device).  The CPU and CUDA
        generators give different numbers for one seed; init_device="cpu" reproduces the
        weights the CPU oracle / tests draw (slow for Apriel-size supernets)."""
        self.cfg, self.seed, self.device, self.dtype = cfg, seed, torch.device(device), dtype
        self.init_device = torch.device(init_device) if init_device is not None else self.device
        self.trunk = _to(init_trunk(cfg, seed, self.init_device, dtype), self.device)
        self._mixers: dict[tuple[int, int], dict] = {}
        self._gu_il: dict[tuple[int, int], torch.Tensor] = {}

    def mixer(self, layer: int, kind: int) -> dict:
        key = (layer, kind)
        if key not in self._mixers:
            m = init_mixer(self.cfg, layer, kind, self.seed, self.init_device, self.dtype)
            self._mixers[key] = {k: (v if k in ("A_log", "dt_bias") else v.to(self.dtype)).to(self.device)
                                 for k, v in m.items()}
        return self._mixers[key]

    def swiglu_interleaved(self, layer: int, block: int) -> torch.Tensor:
        key = (layer, block)
        if key not in self._gu_il:
            self._gu_il[key] = ops.interleave_swiglu(self.trunk["layers"][layer]["ffn_gu"], block)
        return self._gu_il[key]

    def weights(self, placement, swiglu_block: int | None = None) -> dict:
        """Weight structure of one placement (tensors shared with the store, nothing copied).
        swiglu_block: also hand out the shared SwiGLU-interleaved FFN layout for that block."""
        kinds = layer_kinds(placement)
        if len(kinds) != self.cfg.num_layers:
            raise ValueError(f"placement has {len(kinds)} layers, config {self.cfg.name} has {self.cfg.num_layers}")
        layers = []
        for l, k in enumerate(kinds):
            lw = dict(self.trunk["layers"][l])
            lw["mixer"] = self.mixer(l, k)
            if swiglu_block:
                lw["ffn_gu_il"] = self.swiglu_interleaved(l, swiglu_block)
                lw["ffn_gu_hb"] = swiglu_block
                del lw["ffn_gu"]
            layers.append(lw)
        return {"embed": self.trunk["embed"], "final_norm": self.trunk["final_norm"],
                "lm_head": self.trunk["lm_head"], "layers": layers}

    def resident_bytes(self) -> int:
        def walk(o):
            if isinstance(o, dict):
                return sum(walk(v) for v in o.values())
            if isinstance(o, list):
                return sum(walk(v) for v in o)
            return o.numel() * o.element_size() if torch.is_tensor(o) else 0
        return walk(self.trunk) + walk(self._mixers) + sum(t.numel() * t.element_size() for t in self._gu_il.values())


class PlacementRouter:
    """Per-request placement routing over one SupernetStore (graph per (placement, batch))."""

    def __init__(self, store: SupernetStore, max_len: int, max_engines: int = 8):
        self.store, self.max_len, self.max_engines = store, max_len, max_engines
        self._engines: OrderedDict = OrderedDict()

    def engine(self, placement, batch: int):
        """(Supernet, DecodeGraph) of a placement at a batch size; least-recently-used engines
        beyond max_engines are dropped (their state pools and graphs freed)."""
        from .graphs import DecodeGraph
        from .model import Supernet
        key = (placement_code(placement), batch)
        if key in self._engines:
            self._engines.move_to_end(key)
            return self._engines[key]
        cfg = self.store.cfg
        block = ops.gemm_swiglu_block(cfg.ffn)
        model = Supernet(cfg, key[0], batch=batch, max_len=self.max_len, dtype=self.store.dtype,
                         device=self.store.device, weights=self.store.weights(key[0], swiglu_block=block))
        graph = DecodeGraph(model, feedback=True)  # built on the empty engine (construction resets it)
        self._engines[key] = (model, graph)
        while len(self._engines) > self.max_engines:
            self._engines.popitem(last=False)
        return model, graph

    def generate(self, requests, max_new_tokens: int):
        """requests: list of (placement, prompt tokens [T]).  Greedy decoding; returns a list of
        int32 CPU tensors [max_new_tokens] in request order.  Requests are grouped by placement
        (same-placement batching, R/PAPER.md:860-865); each group is one ragged prefill (prompts
        of any lengths) and then decodes through its placement's graph."""
        groups: OrderedDict = OrderedDict()
        for i, (placement, prompt) in enumerate(requests):
            prompt = torch.as_tensor(prompt, dtype=torch.int32).reshape(-1)
            groups.setdefault(placement_code(placement), []).append((i, prompt))
        out = [None] * len(requests)
        for code, items in groups.items():
            T = max(p.numel() for _, p in items)
            if T + max_new_tokens > self.max_len:
                raise ValueError(f"prompt {T} + {max_new_tokens} new tokens > max_len {self.max_len}")
            model, graph = self.engine(code, len(items))
            logits = model.prefill([p for _, p in items])
            first = torch.argmax(logits.float(), dim=-1).to(torch.int32)
            model.step_tokens.copy_(first)
            toks = [first]
            for _ in range(max_new_tokens - 1):
                graph.replay()  # feedback graph: next_tokens -> step_tokens on device
                toks.append(model.next_tokens.clone())
            gen = torch.stack(toks, 1).cpu()
            for row, (i, _) in enumerate(items):
                out[i] = gen[row]
        return out
