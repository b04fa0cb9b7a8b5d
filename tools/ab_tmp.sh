for r in 1 2; do
echo "psi2 from squaring"; python tools/bench_configs.py c3 --reps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_svt_batch'],3), round(d['tensor_frac_of_m64_ceiling'],3))"
echo "product path"; CPA_SVT_NO_PSI2_SQ=1 python tools/bench_configs.py c3 --reps 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_svt_batch'],3), round(d['tensor_frac_of_m64_ceiling'],3))"
done
