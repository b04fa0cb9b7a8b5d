timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_transform_gpu.py tests/test_admm_gpu.py -q -x 2>&1 | tail -1
for v in "" "CPA_SVT_GRAM_SPLIT=2" "CPA_SVT_GRAM_SPLIT=4" "CPA_SVT_GRAM_SPLIT=6" "CPA_SVT_GRAM_SPLIT=8"; do
  echo "[$v]"; env $v timeout 120 python tools/bench_configs.py c2 --reps 10 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
