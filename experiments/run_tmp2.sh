OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_first" -c 1 -o $OUT/c4_f -f python experiments/ap_bench.py C4 > /dev/null 2>&1
