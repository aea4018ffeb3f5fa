#!/bin/bash
# r01zq: end-of-session evidence — full GPU tests, smoke, bench lines (C2 default, reference, C4, C3,
# host tier), the C2 launch list and a full ncu capture of the C2 gather and the C4 k_products
OUT=gpurun_out; TAG=r01zq
mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu > $OUT/${TAG}_tests.log 2>&1; tail -2 $OUT/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/${TAG}_smoke.log 2>&1; tail -1 $OUT/${TAG}_smoke.log
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
timeout 900 python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 10 > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 10 --batch 262144 > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
timeout 600 python bench.py --host-frac 0.25 --no-cpu-baseline --no-e2e --steps 10 > $OUT/${TAG}_bench_host25.json 2> $OUT/${TAG}_bench_host25.err
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o $OUT/${TAG}_gather -f $B > /dev/null 2>&1
echo done
