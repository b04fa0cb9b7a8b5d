# c4 evidence (round 2): L2 counters of the sparse SpMM pair next to the L2 gather probe that sets
# its ceiling (the same metrics on both, so the probe's lts__throughput is the attainable one)
mkdir -p gpurun_out
M="gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"
ncu --metrics $M --clock-control none -k regex:k_gather -s 36 -c 3 --csv tools/probes/l2_gather > gpurun_out/ncu_probe.csv 2> gpurun_out/ncu_probe.err; echo "probe rc=$?"
# ncu --metrics $M --clock-control none -k regex:"k_spmm" -s 2 -c 4 --csv python tools/sparse_step.py 3 1 > gpurun_out/ncu_spmm.csv 2> gpurun_out/ncu_spmm.err; echo "spmm rc=$?"
