timeout 300 python tools/tma_race.py 4096x16384 2>&1 | tail -1
timeout 300 python tools/tma_race.py 1000x1024 2>&1 | tail -1
for t in "" 1; do
  echo "notma=$t"; CPA_SVT_SYM_NOTMA=$t timeout 300 python tools/bench_configs.py c1 c2 c5:8192x32768 --reps 10 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_transform_gpu.py tests/test_admm_gpu.py -q -x 2>&1 | tail -1
