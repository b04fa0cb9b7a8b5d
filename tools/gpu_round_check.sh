# full GPU suite, smoke, bench lines (c2 default; c5 column-sharded through the one-rank NCCL path)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gputests.txt; tail -3 gpurun_out/gputests.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt; grep -c "NCCL INFO" gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
for f in gpurun_out/bench_c2.json gpurun_out/bench_c5.json; do
python -c "import json,sys; d=json.load(open('$f')); print(d['config']['workload'], d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches'], d.get('nccl'))"; done
