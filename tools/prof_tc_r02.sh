# ncu captures of the tcgen05 kernels (round 2): a c5 TF32 recurrence step, a c5 3xTF32 step, the c3 batched kernel
mkdir -p gpurun_out
A="tools/bench_configs.py c5t:16384x65536:tf32 --reps 1"
B="tools/bench_configs.py c5t:16384x65536:3xtf32 --reps 1"
C="tools/bench_configs.py c3 --reps 1"
python $A > gpurun_out/plain_tf32.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 3 -c 1 -o gpurun_out/prof_tc_tf32 python $A > gpurun_out/ncu_tc_tf32.log 2>&1; echo "tf32 rc=$?"
python $B > gpurun_out/plain_3x.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -s 3 -c 1 -o gpurun_out/prof_tc_3x python $B > gpurun_out/ncu_tc_3x.log 2>&1; echo "3x rc=$?"
python $C > gpurun_out/plain_c3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_batched_tc -s 1 -c 1 -o gpurun_out/prof_btc python $C > gpurun_out/ncu_btc.log 2>&1; echo "btc rc=$?"
tail -2 gpurun_out/plain_tf32.log gpurun_out/plain_3x.log gpurun_out/plain_c3.log
