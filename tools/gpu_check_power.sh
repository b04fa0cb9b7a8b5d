mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_transform_gpu.py tests/test_admm_gpu.py -q -x > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout 120 python tools/bench_configs.py c1 c2 --reps 10 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
