OUT=gpurun_out
timeout 900 python -m pytest tests/test_access_prob_gpu.py -q -x > $OUT/t1.log 2>&1; tail -3 $OUT/t1.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --sample-seeds 0 > $OUT/b2.json 2> $OUT/b2.err
timeout 900 python bench.py --config C4 --steps 10 --no-cpu-baseline --no-e2e --sample-seeds 0 > $OUT/b4.json 2> $OUT/b4.err
