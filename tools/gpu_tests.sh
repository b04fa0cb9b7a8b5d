# GPU suite (continue past failures), smoke, c2 bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gputests.txt 2>&1; tail -5 gpurun_out/gputests.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
python -c "import json,sys; d=json.load(open('gpurun_out/bench_c2.json')); print(d['config']['workload'], d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches'], d.get('nccl'))"
