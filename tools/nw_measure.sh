# 8-warp recurrence tiles: bitwise tests, then c2 / c5-shape timing against the 4-warp kernel
mkdir -p gpurun_out
timeout 900 python -m pytest -m gpu -q tests/test_dense_gpu.py -k "eight_warp" > gpurun_out/t_nw.txt 2>&1; tail -3 gpurun_out/t_nw.txt
for nw in 4 8 4 8; do CPA_SVT_DEBUG_OCC=1 CPA_SVT_SYM_NW=$nw python tools/ab_c2.py . 40 2>&1 | tail -2; done
for nw in 4 8; do CPA_SVT_SYM_NW=$nw timeout 600 python tools/bench_configs.py c5:8192x32768 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 half nw=$nw', d['ms_per_svt'], d['phases_ms'].get('step'), d.get('recurrence_frac_of_dmma_peak'))"; done
