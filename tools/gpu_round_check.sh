# full GPU suite, smoke, bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches'])"
