for v in "" bk32s2 bk16s5 bk8s8; do
  if [ -z "$v" ]; then L=""; else L="paper_1705_07112_b200/libcpasvt_$v.so"; fi
  echo "variant=${v:-default}"; CPA_SVT_LIB=$L python tools/bench_configs.py c2 c5:4096x16384 --reps 3 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), json.loads(l)['phases_ms']) for l in sys.stdin]"
done
