for r in 1 2; do
  echo "line 12 folded"; python tools/ab_c2.py . 30
  echo "separate line 12"; CPA_SVT_NO_L12_FOLD=1 python tools/ab_c2.py . 30
done
