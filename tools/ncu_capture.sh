# Round-2 ncu evidence (single GPU): the launch list of one decode step and one --set full
# capture per hot kernel.  Outputs under gpurun_out/ (summaries are copied to profiles/).
#   gpurun --timeout 2400 -- bash tools/ncu_capture.sh
set -x
mkdir -p gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
PROF="python tools/profile_step.py"
# launch list of one Reg|Lklhd-10 decode step (B=64, 32K): per-kernel time and DRAM bytes
ncu --profile-from-start off --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file gpurun_out/r02_launches.csv $PROF > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches_summary.txt 2>&1
# one launch of each decode kernel class (-s skips into the step: the 3rd layer's GEMMs)
$NCU --profile-from-start off -k regex:gdn_decode -c 1 -o gpurun_out/ncu_gdn_decode $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:kda_decode -c 1 -o gpurun_out/ncu_kda_decode $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:attn_decode_tc -c 1 -o gpurun_out/ncu_swa_decode $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:dgemm_kernel -s 8 -c 4 -o gpurun_out/ncu_dgemm $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:chain_kernel -s 3 -c 1 -o gpurun_out/ncu_chain $PROF --chain > /dev/null 2>&1
# prefill at 16K tokens: the 2-CTA projection GEMM (gdn_in, attn_qkv: first timed launches),
# the chunked GDN and KDA phases (the T=16384 launches of tools/bench_prefill.py)
$NCU -k regex:pgemm_kernel -s 1 -c 1 -o gpurun_out/ncu_pgemm python tools/bench_pgemm.py 16384 > /dev/null 2>&1
$NCU -k regex:"gdn_chunk_(intra|state)" -s 16 -c 2 -o gpurun_out/ncu_gdn_chunk python tools/bench_prefill.py > /dev/null 2>&1
$NCU -k regex:kda_chunk_intra -s 8 -c 1 -o gpurun_out/ncu_kda_chunk python tools/bench_prefill.py > /dev/null 2>&1
for f in gdn_decode kda_decode swa_decode dgemm chain pgemm gdn_chunk kda_chunk; do
  ncu -i gpurun_out/ncu_$f.ncu-rep --page raw --csv > gpurun_out/ncu_${f}_raw.csv 2>/dev/null
done
python tools/ncu_report.py gpurun_out > gpurun_out/r02_ncu_kernels.txt 2>&1
ls -la gpurun_out/*.ncu-rep
