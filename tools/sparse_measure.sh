mkdir -p gpurun_out
for np in 1 2 4; do CPA_SVT_SP_PASSES=$np timeout 900 python tools/bench_configs.py c4 --reps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('passes $np', round(d['ms_per_svt'],1), 'pair/step', round(d['spmm_pair_ms_per_step'],2), {k: round(v,1) for k,v in d['phases_ms'].items()}, 'l2 frac', round(d['l2_frac'],3))"; done
timeout 600 python -m pytest -m gpu -q tests/test_sparse_gpu.py 2>&1 | tail -2
