# full GPU suite, smoke, bench lines c2 (default) and c5 (column-sharded, one-rank communicator)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/gputests.txt 2>&1; tail -4 gpurun_out/gputests.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config c5 --math 3xtf32 --steps 3 --no-cpu-baseline > gpurun_out/bench_c5_3x.json 2> gpurun_out/bench_c5_3x.err; echo "bench c5 3x rc=$?"
for f in gpurun_out/bench_c2.json gpurun_out/bench_c5.json gpurun_out/bench_c5_3x.json; do
python -c "import json,sys; d=json.load(open('$f')); print(d['config']['workload'][:40], round(d['ms_per_step'],3), round(d['value']), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), d['clocks'], d['gpu_launches'], d.get('nccl'))"; done
