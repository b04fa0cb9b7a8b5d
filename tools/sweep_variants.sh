for v in "" bk32s3 bk32s2 bk8s6 bk16s3m3; do
  if [ -z "$v" ]; then L=""; else L="paper_1705_07112_b200/libcpasvt_$v.so"; fi
  echo "variant=${v:-default}"; CPA_SVT_LIB=$L python tools/bench_configs.py c2 c5:8192x32768 --reps 3 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
