#!/bin/bash
# r02y: host-tier policy (order tiers >= 1 GB, flat kernel up to 128K ids with a host tier, bucket bits by batch)
OUT=gpurun_out; T=r02y; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gather_gpu.py tests/test_dist_gpu.py tests/test_calibrate_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
timeout 1500 python experiments/r02/host_knobs.py > $OUT/${T}_host_knobs.txt 2>&1; cat $OUT/${T}_host_knobs.txt
timeout 1500 python experiments/gather_sweep.py C4 > $OUT/${T}_gather_sweep_C4.jsonl 2> $OUT/${T}_gather_sweep_C4.err
timeout 1500 python experiments/gather_sweep.py C2 > $OUT/${T}_gather_sweep_C2.jsonl 2> $OUT/${T}_gather_sweep_C2.err
echo done
