mkdir -p gpurun_out
CMD="python tools/bench_configs.py c4 --reps 1"
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_bytes.sum --clock-control none -k regex:k_spmm -s 4 -c 2 --csv $CMD > gpurun_out/ncu_sparse.csv 2> gpurun_out/ncu_sparse.err
tail -3 gpurun_out/ncu_sparse.err
