timeout 600 python -m pytest tests/test_dense_gpu.py -q -x -k "apply_host" 2>&1 | tail -3
for v in "" 1; do echo "nopipe=$v"; CPA_SVT_HOST_NOPIPE=$v timeout 300 python bench.py --no-cpu-baseline | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])"; done
