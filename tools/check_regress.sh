for v in old default; do
  if [ $v = default ]; then L=""; else L=paper_1705_07112_b200/libcpasvt_$v.so; fi
  CPA_SVT_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/l_$v.csv python tools/bench_configs.py c2 --reps 2 > /dev/null 2>&1
  echo "== $v"; python tools/ncu_summary.py gpurun_out/l_$v.csv
done
