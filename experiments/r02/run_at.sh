#!/bin/bash
# r02at: packed-quad first-sweep class stream — parity suites touching K1, then C4 / C2 sweep times
OUT=gpurun_out; T=${T:-r02at}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py tests/test_fused_passes_gpu.py tests/test_cpp_dropin_gpu.py -q -x > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
timeout 600 python experiments/ap_bench.py C4 "" "" > $OUT/${T}_ap_c4.txt 2>&1; cat $OUT/${T}_ap_c4.txt
timeout 300 python experiments/ap_bench.py C2 "" > $OUT/${T}_ap_c2.txt 2>&1; cat $OUT/${T}_ap_c2.txt
