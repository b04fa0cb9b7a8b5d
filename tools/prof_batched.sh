mkdir -p gpurun_out
python -m pytest tests/test_batched_gpu.py -q -x 2>&1 | tail -1
CMD="python tools/bench_configs.py c3:16384 --reps 1"
$CMD > gpurun_out/b_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_batched -s 1 -c 1 -o gpurun_out/prof_batched $CMD > gpurun_out/ncu_b.log 2>&1
tail -1 gpurun_out/ncu_b.log
