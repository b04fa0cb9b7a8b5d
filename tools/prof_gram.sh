mkdir -p gpurun_out
python -m pytest tests/test_dense_gpu.py -q -x 2>&1 | tail -1
CMD="python tools/bench_configs.py c2 --reps 1"
$CMD > gpurun_out/gr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dmma_gemm -s 1 -c 1 -o gpurun_out/prof_gram $CMD > gpurun_out/ncu_gr.log 2>&1
tail -1 gpurun_out/ncu_gr.log
