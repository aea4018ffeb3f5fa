OUT=gpurun_out
QVB_CODES_KERNEL=tma timeout 900 python -m pytest tests/test_access_prob_gpu.py -q -x > $OUT/t1.log 2>&1; tail -3 $OUT/t1.log
timeout 300 python experiments/ap_bench.py C4 "" "QVB_CODES_KERNEL=tma" >> $OUT/ap4.log 2>&1
QVB_CODES_KERNEL=tma timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_codes" --log-file $OUT/kct.csv python experiments/ap_bench.py C4 > /dev/null 2>&1
