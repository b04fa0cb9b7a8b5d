timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for t in "" 1; do
  echo "gemm_notma=$t"; CPA_SVT_GEMM_NOTMA=$t timeout 300 python tools/bench_configs.py c1 c2 c5:8192x32768 --reps 10 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
