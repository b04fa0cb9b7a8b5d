mkdir -p gpurun_out
CMD="python tools/bench_configs.py c5t:4096x16384:tf32 --reps 1"
$CMD > gpurun_out/tc_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 4 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1
tail -3 gpurun_out/ncu_tc.log
