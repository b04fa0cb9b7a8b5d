timeout 600 python -m pytest tests/test_dense_gpu.py -q -x -k "tma_kernels" 2>&1 | tail -1
timeout 300 python __graft_entry__.py 2>&1 | tail -2
timeout 600 python tools/bench_configs.py c5t:16384x65536:3xtf32 c5t:16384x65536:tf32 --reps 3 | python -c "import sys,json; [print(json.loads(l)['config'], json.loads(l)['math'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
