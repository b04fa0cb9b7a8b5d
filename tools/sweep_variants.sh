for v in "" nowait; do
  if [ -z "$v" ]; then L=""; else L="paper_1705_07112_b200/libcpasvt_$v.so"; fi
  for sp in 0 1 3 6; do
  echo "variant=${v:-default} split=$sp"; CPA_SVT_FLOW_SPLIT=$sp CPA_SVT_LIB=$L python tools/bench_configs.py c2 --reps 5 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), json.loads(l)['phases_ms']['step']) for l in sys.stdin]"
  done
done
