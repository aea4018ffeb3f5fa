OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_first -c 1 -o $OUT/c4_first4 -f python experiments/ap_bench.py C4 > /dev/null 2>&1
