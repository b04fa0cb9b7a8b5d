# round-end evidence: bench line, launch list of the bench command, ncu captures of the top kernels
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cheb_sym -s 3 -c 1 -o gpurun_out/prof_sym_final $CMD > /dev/null 2>&1; echo "sym rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batched_tc -c 1 -o gpurun_out/prof_btc_final python tools/bench_configs.py c3:16384 --reps 1 > /dev/null 2>&1; echo "btc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 6 -c 1 -o gpurun_out/prof_tc_final python tools/bench_configs.py c5t:4096x16384:tf32 --reps 1 > /dev/null 2>&1; echo "tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_power_warp -c 1 -o gpurun_out/prof_power_final $CMD > /dev/null 2>&1; echo "power rc=$?"
ls -la gpurun_out/*.ncu-rep
