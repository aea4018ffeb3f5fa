#!/bin/bash
# r01c: re-verify HEAD on the B200 (tests, bench) and profile the C4 node-major sweep.
OUT=gpurun_out; TAG=r01c
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/${TAG}_tests.log 2>&1; tail -3 $OUT/${TAG}_tests.log
timeout 600 python experiments/ap_bench.py C4 "" "QVB_NM_KERNEL=tma" "QVB_PF_BLOCKS=0" > $OUT/${TAG}_ap_c4.log 2>&1
timeout 300 python experiments/ap_bench.py C2 "" > $OUT/${TAG}_ap_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_nm -s 0 -c 3 -o $OUT/${TAG}_c4_nm -f python experiments/ap_bench.py C4 > $OUT/${TAG}_ncu.log 2>&1
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo done
