"""One block per captured kernel from the ncu --page raw CSVs tools/ncu_capture.sh writes
(gpurun_out/ncu_<tag>_raw.csv): duration, DRAM bytes, throughputs, tensor pipe, occupancy."""
import csv
import glob
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
M = [("duration", "gpu__time_duration.sum"), ("dram read", "dram__bytes_read.sum"),
     ("dram write", "dram__bytes_write.sum"),
     ("dram throughput %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
     ("sm throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
     ("tensor pipe active %", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
     ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
     ("regs/thread", "launch__registers_per_thread"), ("grid", "launch__grid_size"),
     ("block", "launch__block_size"), ("cluster", "launch__cluster_dim_x")]
print("ncu --set full --clock-control none, one launch each (tools/ncu_capture.sh, round 2, B200).")
print("Decode: Reg|Lklhd-10, B=64, 32K context (tools/profile_step.py; the fused chain with --chain);")
print("prefill: tools/bench_pgemm.py 16384 (2-CTA pgemm), tools/bench_prefill.py T=16384 (chunk kernels).")
print("Cold-cache serialised replays: compare shares and DRAM bytes, not absolute in-step times.\n")
for f in sorted(glob.glob(os.path.join(d, "ncu_*_raw.csv"))):
    tag = os.path.basename(f)[4:-8]
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) < len(h) or not r[0].strip().isdigit():
            continue
        print(f"[{tag}] {r[h.index('Kernel Name')][:110]}")
        for label, key in M:
            if key in h:
                i = h.index(key)
                print(f"    {label}: {r[i]} {units[i]}".rstrip())
        print()
