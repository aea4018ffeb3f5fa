#!/bin/bash
# Capture the launch list and one full ncu report per dominant kernel of the
# default bench workload (run under gpurun on ONE GPU; never multi-rank).
#   bash profiles/run_ncu.sh [tag] [extra bench args]
set -u
TAG=${1:-r01}; shift || true
OUT=gpurun_out
mkdir -p $OUT
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e $*"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > $OUT/${TAG}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o $OUT/${TAG}_sweep -f $B > $OUT/${TAG}_sweep.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o $OUT/${TAG}_gather -f $B > $OUT/${TAG}_gather.log 2>&1
echo done
