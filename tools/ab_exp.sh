for r in 1 2; do
for sp in 0 2 3 4; do
  if [ $sp = 0 ]; then echo "gram split default"; python tools/ab_c2.py . 30; else echo "gram split $sp"; CPA_SVT_GRAM_SPLIT=$sp python tools/ab_c2.py . 30; fi
done; done
