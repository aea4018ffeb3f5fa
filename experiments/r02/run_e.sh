#!/bin/bash
# r02e: ncu evidence of the default (C4) bench: launch list with DRAM bytes,
# full captures of the dominant kernels (k_gather_rows, k_codes x7, k_products_tma,
# k_first) and a host-tier capture of the class gather with PCIe counters
OUT=gpurun_out; T=r02e; mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e --sample-seeds 0"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/${T}_launches.csv $B > $OUT/${T}_launches.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_rows -s 3 -c 1 -o $OUT/${T}_gather -f $B > $OUT/${T}_gather.log 2>&1; echo gather=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_codes -s 7 -c 7 -o $OUT/${T}_codes -f $B > $OUT/${T}_codes.log 2>&1; echo codes=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_products -s 1 -c 1 -o $OUT/${T}_products -f $B > $OUT/${T}_products.log 2>&1; echo products=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_first -s 1 -c 1 -o $OUT/${T}_first -f $B > $OUT/${T}_first.log 2>&1; echo first=$?
ncu --query-metrics > $OUT/${T}_ncu_metrics_all.txt 2>&1
PM=$(grep -oE "\bpcie__[a-z0-9_]*bytes[a-z0-9_]*" $OUT/${T}_ncu_metrics_all.txt | sort -u | head -6 | sed 's/$/.sum/' | tr '\n' ',' | sed 's/,$//')
echo "pcie metrics: $PM"
timeout 900 ncu --set full ${PM:+--metrics $PM,lts__t_sectors_aperture_sysmem.sum} --clock-control none --import-source on -k regex:k_gather_classes -s 3 -c 1 -o $OUT/${T}_host25 -f $B --host-frac 0.25 > $OUT/${T}_host25.log 2>&1; echo host25=$?
ls -la $OUT/ | grep $T
