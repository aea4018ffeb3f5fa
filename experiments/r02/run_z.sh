#!/bin/bash
# r02z: k_products_tma with 2-warp CTAs (more resident warps under the shared-memory limit)
OUT=gpurun_out; T=r02z; mkdir -p $OUT
timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap.txt 2>&1; cat $OUT/${T}_ap.txt
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__grid_size \
  --clock-control none -k regex:k_products_tma -c 1 python experiments/ap_bench.py C4 2>&1 | grep -E "k_products|duration|warps_active|issue_active|occupancy|grid_size" | head -12
timeout 1200 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
