OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_codes" -s 7 -c 2 -o $OUT/c4_g2 -f python experiments/ap_bench.py C4 > /dev/null 2>&1
