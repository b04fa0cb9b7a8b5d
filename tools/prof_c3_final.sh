mkdir -p gpurun_out
C="tools/bench_configs.py c3 --reps 1"
python $C > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_batched_tc -s 1 -c 1 -o gpurun_out/prof_btc_final python $C > gpurun_out/ncu_btc.log 2>&1; echo "btc rc=$?"
ncu -i gpurun_out/prof_btc_final.ncu-rep --page raw --csv > gpurun_out/prof_btc_final_raw.csv 2>/dev/null; echo raw rc=$?
rm -f gpurun_out/prof_btc_final.ncu-rep
