# measure: bench line, per-config numbers ($@ configs), ncu launch list + full capture of k_cheb_sym
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json | cut -c1-3000; tail -2 gpurun_out/bench.err
timeout 1800 python tools/bench_configs.py "$@" > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"; tail -3 gpurun_out/configs.err
cut -c1-700 gpurun_out/configs.jsonl
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cheb_sym -s 3 -c 1 -o gpurun_out/prof_sym $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
