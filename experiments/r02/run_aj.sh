#!/bin/bash
# r02aj: fused segment passes (k_pass_fused) — parity tests, then C4 / C2 sweep times against the decoupled sweep
OUT=gpurun_out; T=${T:-r02aj}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_passes_gpu.py -q -x > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
timeout 600 python experiments/ap_bench.py C4 "" "QVB_PRODUCTS=fused" "" "QVB_PRODUCTS=fused" > $OUT/${T}_ap_c4.txt 2>&1; cat $OUT/${T}_ap_c4.txt
timeout 300 python experiments/ap_bench.py C2 "QVB_SEG_MB=4" "QVB_SEG_MB=4 QVB_PRODUCTS=fused" > $OUT/${T}_ap_c2.txt 2>&1; cat $OUT/${T}_ap_c2.txt
