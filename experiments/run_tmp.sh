OUT=gpurun_out
timeout 900 python -m pytest tests/test_access_prob_gpu.py tests/test_cpp_dropin_gpu.py -q -x > $OUT/t1.log 2>&1; tail -3 $OUT/t1.log
for c in C2 C4; do timeout 300 python experiments/ap_bench.py $c >> $OUT/ap4.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"k_first|k_codes|k_products" --log-file $OUT/c4_gp.csv python experiments/ap_bench.py C4 > /dev/null 2>&1
