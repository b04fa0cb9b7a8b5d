python tools/bench_configs.py c2 --reps 5 | tail -1 | cut -c1-400
python -m pytest tests -m gpu -q -x -k "power or config or dense" 2>&1 | tail -2
