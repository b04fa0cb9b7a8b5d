# c2: the Gram / power-squaring product (k_dmma_gemm_tma, EPI_GRAM) at forced k-splits; gap_trace
# gives each kernel's duration.  Usage (GPU box): bash tools/gram_split_sweep.sh
for S in 0 1 2 3 4 5 6 8; do
  if [ "$S" = 0 ]; then unset CPA_SVT_GRAM_SPLIT; else export CPA_SVT_GRAM_SPLIT=$S; fi
  python tools/gap_trace.py c2 3 > /tmp/g.json 2>/dev/null
  python - "$S" <<'PY'
import json, sys
d = json.load(open('/tmp/g.json'))
ops = [o for s in d['svts'] for o in s['ops']]
g = [o[1] for o in ops if 'k_dmma_gemm_tma<false, false, 0>' in o[0]]
print(f"split={sys.argv[1]} ms/SVT={d['event_ms_per_svt']:.4f} gram-kernel mean={sum(g)/len(g):.1f} us (n={len(g)})")
PY
done
