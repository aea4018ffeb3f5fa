#!/bin/bash
# One GPU call's worth of round evidence (run under gpurun, 1 GPU):
#   tests, the default bench line, the reference arm, the ncu launch list and
#   one --set full capture each of k_gather_rows and k_sweep (C2), plus a C4
#   sweep pass capture.
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -q -m gpu > $OUT/${TAG}_tests.log 2>&1; tail -3 $OUT/${TAG}_tests.log
python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather -s 3 -c 1 -o $OUT/${TAG}_gather -f $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o $OUT/${TAG}_sweep -f $B > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_sweep -s 16 -c 2 -o $OUT/${TAG}_c4_sweep -f $B --config C4 > /dev/null 2>&1
python bench.py --config C4 --no-cpu-baseline --no-e2e --steps 5 > $OUT/${TAG}_bench_c4.json 2> $OUT/${TAG}_bench_c4.err
python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 10 --batch 262144 > $OUT/${TAG}_bench_c3.json 2> $OUT/${TAG}_bench_c3.err
python bench.py --host-frac 0.25 --no-cpu-baseline --no-e2e --steps 10 > $OUT/${TAG}_bench_host25.json 2> $OUT/${TAG}_bench_host25.err
echo done
