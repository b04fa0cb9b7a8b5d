for r in 1 2; do
  echo "default"; python tools/ab_c2.py . 30
  echo "last arrival"; CPA_SVT_CHAIN_LAST=1 python tools/ab_c2.py . 30
  echo "last arrival S=2"; CPA_SVT_CHAIN_LAST=1 CPA_SVT_CHAIN_SPLIT=2 python tools/ab_c2.py . 30
  echo "last arrival S=4"; CPA_SVT_CHAIN_LAST=1 CPA_SVT_CHAIN_SPLIT=4 python tools/ab_c2.py . 30
done
