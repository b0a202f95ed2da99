"""Probe: device facts + cuBLAS skinny-GEMM bandwidth at Apriel decode shapes (M = batch)."""
import torch, json, subprocess, os
p = torch.cuda.get_device_properties(0)
print(json.dumps({"name": p.name, "sms": p.multi_processor_count, "mem_gb": p.total_memory/1e9,
                  "l2": getattr(p, "L2_cache_size", None)}))
print(subprocess.run(["nproc"], capture_output=True, text=True).stdout.strip(),
      subprocess.run("lscpu | grep 'Model name'", shell=True, capture_output=True, text=True).stdout.strip())
shapes = {"ffn_gu": (28672, 5120), "ffn_down": (5120, 14336), "gdn_in": (10304, 5120), "gdn_out": (5120, 4096),
          "attn_qkv": (6144, 5120), "attn_o": (5120, 4096), "kda_in": (12576, 5120), "lm_head": (131072, 5120)}
for M in (1, 8, 32, 64, 128):
    for name, (N, K) in shapes.items():
        nbuf = max(2, int(2e9 // (N * K * 2)))
        nbuf = min(nbuf, 8)
        Ws = [torch.randn(N, K, device="cuda", dtype=torch.bfloat16) for _ in range(nbuf)]
        x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        for i in range(5):
            y = x @ Ws[i % nbuf].t()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        it = 40
        e0.record()
        for i in range(it):
            y = x @ Ws[i % nbuf].t()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        gbs = (N * K * 2 + M * K * 2 + M * N * 2) / ms / 1e6
        print(f"M={M:4d} {name:9s} N={N:6d} K={K:5d} {ms*1e3:8.1f} us  {gbs:7.0f} GB/s")
        del Ws
