OUT=gpurun_out
timeout 600 python experiments/ap_bench.py C4 "QVB_OVERLAP=0" "QVB_OV_F=1 QVB_OV_G=4" "QVB_OV_F=2 QVB_OV_G=2" "QVB_OV_F=4 QVB_OV_G=3" "QVB_OV_F=8 QVB_OV_G=3" "QVB_OV_F=2 QVB_OV_G=3" >> $OUT/ap4.log 2>&1
QVB_OV_F=2 QVB_OV_G=3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_first|k_codes|k_products" --log-file $OUT/c4_ov.csv python experiments/ap_bench.py C4 > /dev/null 2>&1
