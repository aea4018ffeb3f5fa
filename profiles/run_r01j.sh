#!/bin/bash
# r01j: C5-style gather sweep (batch x host fraction x request stream) on C2 and C4,
# refreshed default bench lines and the C4 launch list with the identity-slice first sweep
OUT=gpurun_out; TAG=r01j
mkdir -p $OUT
timeout 900 python experiments/gather_sweep.py C2 > $OUT/${TAG}_gather_sweep_c2.jsonl 2> $OUT/${TAG}_gather_sweep_c2.err
timeout 1500 python experiments/gather_sweep.py C4 > $OUT/${TAG}_gather_sweep_c4.jsonl 2> $OUT/${TAG}_gather_sweep_c4.err
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
B="python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_c4.csv $B --config C4 --sample-seeds 0 > /dev/null 2>&1
echo done
