OUT=gpurun_out
cp experiments/libs/libqvb_c32.so paper_2305_10863_b200/libqvb.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_codes" --log-file $OUT/kc_32.csv python experiments/ap_bench.py C4 > /dev/null 2>&1
cp experiments/libs/libqvb_c16.so paper_2305_10863_b200/libqvb.so
for mb in 56 64 72 80; do echo "SEG_MB=$mb" >> $OUT/ap5.log; QVB_SEG_MB=$mb timeout 300 python experiments/ap_bench.py C4 >> $OUT/ap5.log 2>&1; done
