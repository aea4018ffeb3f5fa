#!/bin/bash
OUT=gpurun_out; TAG=r01e
mkdir -p $OUT
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 5 > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 10 --batch 262144 > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_codes|k_products|k_first" -s 4 -c 3 -o $OUT/${TAG}_c4_ap -f python experiments/ap_bench.py C4 > /dev/null 2>&1
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > /dev/null 2>&1
echo done
