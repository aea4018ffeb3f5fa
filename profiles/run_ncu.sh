#!/bin/bash
# The ncu launch list of the default bench workload (C4) and one full capture
# per dominant kernel, plus a host-tier capture with the PCIe byte counters
# (run under gpurun on ONE GPU; never multi-rank; numbers printed under ncu
# are not bench values).
#   bash profiles/run_ncu.sh [tag] [extra bench args]
set -u
TAG=${1:-r02}; shift || true
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e --sample-seeds 0 $*"
F="ncu --set full --clock-control none --import-source on"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv $B > $OUT/${TAG}_launches.log 2>&1
$F -k regex:k_gather_rows -s 3 -c 1 -o $OUT/${TAG}_gather -f $B > $OUT/${TAG}_gather.log 2>&1
$F -k regex:k_codes -s 7 -c 7 -o $OUT/${TAG}_codes -f $B > $OUT/${TAG}_codes.log 2>&1
$F -k regex:k_products -s 1 -c 1 -o $OUT/${TAG}_products -f $B > $OUT/${TAG}_products.log 2>&1
$F -k regex:k_first -s 1 -c 1 -o $OUT/${TAG}_first -f $B > $OUT/${TAG}_first.log 2>&1
$F --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,lts__t_sectors_aperture_sysmem.sum -k regex:k_gather_classes \
   -s 3 -c 1 -o $OUT/${TAG}_host25 -f $B --host-frac 0.25 > $OUT/${TAG}_host25.log 2>&1
echo done
