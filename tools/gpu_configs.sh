mkdir -p gpurun_out
timeout 2400 python tools/bench_configs.py c1 c2 c3 c4 c5 c5t:16384x65536:tf32 c5t:16384x65536:3xtf32 --oracle > gpurun_out/configs_all.jsonl 2> gpurun_out/configs_all.err; echo rc=$?
tail -2 gpurun_out/configs_all.err; cut -c1-400 gpurun_out/configs_all.jsonl
