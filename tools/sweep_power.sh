# power-iteration variants at c2: squarings (SQ), warp-per-row kernel (WARP=1 plain, 2 cluster gather), polling lanes
for v in "SQ=2" "SQ=3" "SQ=2 WARP=1" "SQ=3 WARP=1" "SQ=2 WARP=2" "SQ=3 WARP=2" "SQ=2 WARP=1 POLL=128"; do
  echo "$v"; env $(for kv in $v; do echo CPA_SVT_POWER_$kv; done) timeout 120 python tools/bench_configs.py c2 --reps 10 | python -c "import sys,json; [print(round(json.loads(l)['ms_per_svt'],3), {k: round(v,3) for k,v in json.loads(l)['phases_ms'].items()}) for l in sys.stdin]"
done
for w in 1 2; do CPA_SVT_POWER_WARP=$w timeout 300 python -m pytest tests/test_dense_gpu.py -q -x 2>&1 | tail -1; done
