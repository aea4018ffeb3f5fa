#!/bin/bash
# r02al: ncu of one k_pass_fused launch (pass 0) and one k_codes launch at C4
OUT=gpurun_out; T=${T:-r02al}; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_fused -c 2 -o $OUT/${T}_fused \
  python experiments/ap_bench.py C4 "QVB_PRODUCTS=fused" > $OUT/${T}_ncu.log 2>&1; tail -3 $OUT/${T}_ncu.log
ncu -i $OUT/${T}_fused.ncu-rep --page details --csv > $OUT/${T}_fused_details.csv 2>&1
ncu -i $OUT/${T}_fused.ncu-rep --page raw --csv > $OUT/${T}_fused_raw.csv 2>&1
ls -la $OUT
