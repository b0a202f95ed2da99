# One ncu --set full capture per decode / prefill kernel class (single GPU, one launch each):
#   bash tools/ncu_capture.sh   -> gpurun_out/ncu_<name>.ncu-rep
set -x
NCU="ncu --set full --import-source on --clock-control none"
PROF="python tools/profile_step.py"
$NCU --profile-from-start off -k regex:delta_decode_kernel -c 1 -o gpurun_out/ncu_gdn_decode $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:attn_decode_tc -c 1 -o gpurun_out/ncu_swa_decode $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:gemm2_kernel -c 3 -o gpurun_out/ncu_gemm2 $PROF > /dev/null 2>&1
$NCU --profile-from-start off -k regex:add_rmsnorm -c 1 -o gpurun_out/ncu_norm $PROF > /dev/null 2>&1
$NCU -k regex:"chunk_(intra|state)" -s 3 -c 2 -o gpurun_out/ncu_gdn_chunk python tools/bench_prefill.py > /dev/null 2>&1
