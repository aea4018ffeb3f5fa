OUT=gpurun_out
timeout 900 python -m pytest tests/test_gather_gpu.py -q -x > $OUT/t5.log 2>&1; tail -3 $OUT/t5.log
for k in 0 1; do for c in C2 C4; do QVB_LUT_KEEP=$k timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e --sample-seeds 0 > $OUT/bg_${c}_$k.json 2> $OUT/bg_$c.err; done; done
