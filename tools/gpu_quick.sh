# quick GPU iteration: selected tests ($1 = pytest -k expr or file) + bench (no cpu baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest ${1:-tests} -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -5 gpurun_out/pytest_q.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?" >> gpurun_out/bench_q.err
cat gpurun_out/bench_q.json; tail -3 gpurun_out/bench_q.err
