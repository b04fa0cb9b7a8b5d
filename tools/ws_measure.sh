# warp-specialized recurrence: bitwise tests, then c2 / c5-shape timing against the default kernel
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q tests/test_dense_gpu.py -k "warp_specialized" > gpurun_out/t_ws.txt 2>&1; tail -3 gpurun_out/t_ws.txt
for ws in 0 1; do
CPA_SVT_SYM_WS=$ws timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench_ws$ws.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_ws$ws.json')); print('ws=$ws', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), {k: round(v,4) for k,v in d['roofline']['phase_ms_per_step'].items()})"
done
for ws in 0 1; do CPA_SVT_SYM_WS=$ws timeout 600 python tools/bench_configs.py c5:8192x32768 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 half ws=$ws', d['ms_per_svt'], d['phases_ms'].get('step'), d.get('recurrence_frac_of_dmma_peak'))"; done
