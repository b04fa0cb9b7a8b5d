# A/B of run-time experiment knobs on the c2 SVT (tools/ab_c2.py), two passes
for r in 1 2; do
for b in 0 10 20 35 50; do
  echo "RED_BIAS=$b"; CPA_SVT_RED_BIAS=$b python tools/ab_c2.py . 30
done; done
