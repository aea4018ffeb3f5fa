#!/bin/bash
# r02aa: k_first DRAM traffic and L1 load at f1 window 32 (node order) vs 256 (degree-sorted windows)
OUT=gpurun_out; T=r02aa; mkdir -p $OUT
for w in 32 256; do
  QVB_F1_WINDOW=$w timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
    --clock-control none -k k_first -c 1 python experiments/ap_bench.py C4 > $OUT/${T}_w$w.txt 2>&1
  echo "window $w"; grep -E "k_first|\.sum|\.pct" $OUT/${T}_w$w.txt | head -16
done
