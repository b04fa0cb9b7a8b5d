for v in "" 1; do echo "nosmall=$v"; CPA_SVT_NO_SMALL=$v timeout 120 python tools/bench_configs.py c1 --reps 20 | python -c "import sys,json; [print(json.loads(l)['config'], json.loads(l)['form'], round(json.loads(l)['ms_per_svt'],4), {k: round(v,4) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"; done
timeout 300 python bench.py --config c1 --no-cpu-baseline | cut -c1-600
timeout 300 python __graft_entry__.py | tail -1
