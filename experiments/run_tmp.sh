OUT=gpurun_out
timeout 900 python -m pytest tests/test_gather_gpu.py tests/test_dist_gpu.py -q -x > $OUT/t5.log 2>&1; tail -3 $OUT/t5.log
for c in C2 C4 C3; do timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline --no-e2e --sample-seeds 0 $( [ $c = C3 ] && echo "--batch 262144" ) > $OUT/bg_$c.json 2> $OUT/bg_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_gather -c 3 --log-file $OUT/kg.csv python bench.py --steps 3 --warmup 1 --clock-window 0 --no-cpu-baseline --no-e2e --sample-seeds 0 > /dev/null 2>&1
