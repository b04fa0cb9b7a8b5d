# A/B of run-time knobs on the c2 SVT (tools/ab_c2.py)
for r in 1 2; do
  echo "tma (PP=0)"; CPA_SVT_SYM_PP=0 python tools/ab_c2.py . 20
  for st in 4 5; do for m in 2 3; do for q in 2 3; do
    echo "pp stages=$st m=$m S=$q"; CPA_SVT_PP_STAGES=$st CPA_SVT_SYM_CHAIN=$m CPA_SVT_CHAIN_SPLIT=$q python tools/ab_c2.py . 20
  done; done; done
done
