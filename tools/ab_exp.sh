# sparse c4 SpMM pair (tools/sparse_step.py)
echo "nohint"; CPA_SVT_SP_NOHINT=1 python tools/sparse_step.py 5 1
echo "hint"; python tools/sparse_step.py 5 1
echo "hint U4"; CPA_SVT_SP_UNROLL=4 python tools/sparse_step.py 5 1
