mkdir -p gpurun_out
CMD="python tools/bench_configs.py c2 --reps 1"
$CMD > gpurun_out/fl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cheb_flow -s 1 -c 1 -o gpurun_out/prof_flow $CMD > gpurun_out/ncu_fl.log 2>&1
tail -2 gpurun_out/ncu_fl.log
