#!/bin/bash
# r02u: products staging buffers sized for one more CTA per SM (QVB_PT_FIT)
OUT=gpurun_out; T=r02u; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
for f in 1 0; do QVB_PT_FIT=$f timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_f$f.txt 2>&1; echo "fit $f"; cat $OUT/${T}_ap_f$f.txt; done
