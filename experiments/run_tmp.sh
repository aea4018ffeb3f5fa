OUT=gpurun_out
timeout 900 python -m pytest tests/test_access_prob_gpu.py tests/test_cpp_dropin_gpu.py -q -x > $OUT/t1.log 2>&1; tail -3 $OUT/t1.log
