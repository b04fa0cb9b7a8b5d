# A/B: the committed library (.ab/old) against the working tree, one-chain and two-chain, alternating
for r in 1 2; do
  python tools/ab_c2.py .ab/old 30
  CPA_SVT_SYM_CHAIN=0 python tools/ab_c2.py . 30
  CPA_SVT_SYM_CHAIN=1 python tools/ab_c2.py . 30
done
for d in .ab/old .; do PKG_DIR=$d SWEEP_ONECHAIN=1 python tools/chain_sweep.py 5 4096,8192 2>&1 | grep "chain=0" | sed "s#^#$d #"; done
