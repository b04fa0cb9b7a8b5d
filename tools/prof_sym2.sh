mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/pytest_q.log 2>&1; tail -1 gpurun_out/pytest_q.log
for sp in 1 2 3 4; do echo "split=$sp"; CPA_SVT_FLOW_SPLIT=$sp python tools/bench_configs.py c2 --reps 5 | tail -1; done > gpurun_out/sweep_sym.log 2>&1
cat gpurun_out/sweep_sym.log | cut -c1-600
CMD="python tools/bench_configs.py c2 --reps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cheb_sym -s 1 -c 1 -o gpurun_out/prof_sym3 $CMD > gpurun_out/ncu_sym.log 2>&1
tail -2 gpurun_out/ncu_sym.log
