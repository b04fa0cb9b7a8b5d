# round-2 bench-kernel evidence: launch list of the bench command and one full capture of k_cheb_sym_tma (c2)
mkdir -p gpurun_out
CMD="bench.py --steps 2 --warmup 3 --no-cpu-baseline"
python $CMD > gpurun_out/plain_c2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches_c2.csv python $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
python $CMD > gpurun_out/plain_c2b.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_cheb_sym_tma -s 3 -c 1 -o gpurun_out/prof_sym_c2 python $CMD > gpurun_out/ncu_sym.log 2>&1; echo "sym rc=$?"
