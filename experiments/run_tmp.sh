OUT=gpurun_out
timeout 900 python -m pytest tests/test_access_prob_gpu.py -q -x > $OUT/t1.log 2>&1; tail -3 $OUT/t1.log
for c in C1 C2 C3 C4; do timeout 300 python experiments/ap_bench.py $c "" >> $OUT/ap2.log 2>&1; done
