#!/bin/bash
# r02w: narrow k_first (4-byte class table, exception bitmap word loaded with the slice bounds)
OUT=gpurun_out; T=r02w; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py -x -q -m gpu -k "narrow or c2 or sharded or first" > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
for nw in 1 0 1 0; do QVB_F1_NARROW=$nw timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_n$nw.txt 2>&1; echo "narrow $nw"; cat $OUT/${T}_ap_n$nw.txt; done
timeout 1500 python experiments/r02/host_knobs.py > $OUT/${T}_host_knobs.txt 2>&1; cat $OUT/${T}_host_knobs.txt
