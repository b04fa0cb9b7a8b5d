# usage: bash tools/sweep_variants.sh "configs" variant...   ("" = default library)
CFG=$1; shift
for v in "$@"; do
  if [ "$v" = "default" ]; then L=""; else L="paper_1705_07112_b200/libcpasvt_$v.so"; fi
  echo "variant=$v"; CPA_SVT_LIB=$L timeout 600 python tools/bench_configs.py $CFG --reps 5 | python -c "import sys,json; [print(json.loads(l)['config'], round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
