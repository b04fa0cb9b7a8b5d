for v in pw1 pw2 pw4 pw8; do
  echo "variant=$v"; CPA_SVT_LIB=paper_1705_07112_b200/libcpasvt_$v.so python tools/power_trace.py 2>&1 | tail -4
done
