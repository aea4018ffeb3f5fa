OUT=gpurun_out
timeout 900 python -m pytest tests/test_sampler_gpu.py tests/test_cpp_dropin_gpu.py -q -x > $OUT/t4.log 2>&1; tail -3 $OUT/t4.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline > $OUT/bs.json 2> $OUT/bs.err
