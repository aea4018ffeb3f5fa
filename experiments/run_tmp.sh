OUT=gpurun_out
timeout 1500 python -m pytest tests/test_access_prob_gpu.py -q -x -k "in_rows or c4_sampled" > $OUT/t2.log 2>&1; tail -3 $OUT/t2.log
