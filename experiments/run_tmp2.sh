OUT=gpurun_out
QVB_SEG_MB=64 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_products" -c 1 -o $OUT/c4_p -f python experiments/ap_bench.py C4 > /dev/null 2>&1
