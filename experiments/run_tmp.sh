OUT=gpurun_out
for f in small tma; do QVB_F1_KERNEL=$f QVB_SEG_MB=64 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:"k_first" --log-file $OUT/f1_$f.csv python experiments/ap_bench.py C4 > /dev/null 2>&1; done
