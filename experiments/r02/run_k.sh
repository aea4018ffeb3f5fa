#!/bin/bash
# r02k: sharded P tests, the rest of the GPU suite pieces touched since r02f
OUT=gpurun_out; T=r02k; mkdir -p $OUT
timeout 1500 python -m pytest -q tests/test_sharded_p_gpu.py tests/test_dist_gpu.py tests/test_cpp_dropin_gpu.py tests/test_access_prob_gpu.py tests/test_gather_gpu.py tests/test_multi_device_gpu.py -k "not c4_full" > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
grep -E "FAILED|Error" $OUT/${T}_tests.log | head -20
