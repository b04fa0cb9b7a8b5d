# round-end evidence: bench line, launch list of the bench command, ncu captures of the top kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $CMD > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cheb_sym -s 3 -c 1 -o gpurun_out/prof_sym_final $CMD > /dev/null 2>&1; echo "sym rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dmma_gemm_tma -s 12 -c 1 -o gpurun_out/prof_gemm_final $CMD > /dev/null 2>&1; echo "gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_power_warp -c 1 -o gpurun_out/prof_power_final $CMD > /dev/null 2>&1; echo "power rc=$?"
ls -la gpurun_out/*final*
