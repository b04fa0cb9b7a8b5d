python -m pytest tests/test_dense_gpu.py -q -x 2>&1 | tail -1
for sp in 1 2 4 8; do echo "split=$sp"; CPA_SVT_FLOW_SPLIT=$sp python tools/bench_configs.py c2 --reps 5 | tail -1; done
