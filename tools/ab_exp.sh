# A/B of run-time experiment knobs on the c2 SVT (tools/ab_c2.py), two passes
for r in 1 2; do
  echo "psi2 from the squaring"; python tools/ab_c2.py . 30
  echo "NO_PSI2_SQ"; CPA_SVT_NO_PSI2_SQ=1 python tools/ab_c2.py . 30
done
