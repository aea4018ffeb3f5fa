#!/bin/bash
# r02ac: k_first_win, two windows per CTA step (long slice of one with the short slice of the other)
OUT=gpurun_out; T=r02ac; mkdir -p $OUT
for w in 256 32 256; do QVB_F1_WINDOW=$w timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_w$w.txt 2>&1; echo "window $w"; cat $OUT/${T}_ap_w$w.txt; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k k_first_win -c 1 python experiments/ap_bench.py C4 > $OUT/${T}_ncu.txt 2>&1; grep -E "k_first|\.sum|\.pct" $OUT/${T}_ncu.txt | head -12
timeout 2400 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py tests/test_fap_gpu.py tests/test_dropin_graph_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
