# c4 evidence (round 2, 64-row blocks): L2 / DRAM counters of the sparse SpMM pair next to the
# 512-byte L2 gather probe that sets its ceiling (the same metrics on both).
mkdir -p gpurun_out
M="gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/l2_gather512 tools/probes/l2_gather512.cu
tools/probes/l2_gather512 > gpurun_out/probe512.txt 2>&1
# the 51.2 MB footprint (one column pass of c4), 512-byte segments, 8 CTAs per SM, U = 2: launches 205-206
ncu --metrics $M --clock-control none -k regex:k_g -s 204 -c 2 --csv tools/probes/l2_gather512 > gpurun_out/ncu_probe512.csv 2> gpurun_out/ncu_probe512.err; echo "probe rc=$?"
# sparse_step.py 5 1: one warm-up call, then one timed call (K = 5: steps k = 1..4); skip the warm-up's launches
ncu --metrics $M --clock-control none -k regex:"k_spmm" -s 12 -c 12 --csv python tools/sparse_step.py 5 1 > gpurun_out/ncu_spmm.csv 2> gpurun_out/ncu_spmm.err; echo "spmm rc=$?"
