mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/pytest_q.log 2>&1; tail -1 gpurun_out/pytest_q.log
for sp in 0 5 6 7; do echo "split=$sp"; CPA_SVT_FLOW_SPLIT=$sp python tools/bench_configs.py c2 --reps 5 | tail -1; done > gpurun_out/sweep_sym.log 2>&1
cat gpurun_out/sweep_sym.log | cut -c1-600
CMD="python tools/bench_configs.py c2 --reps 1"
timeout 600 true
tail -2 gpurun_out/ncu_sym.log
