#!/bin/bash
# r02av: full round evidence on the final code: GPU suite, smoke, default C4 bench + reference arm,
# ncu launch list + full captures (profiles/run_round.sh), host-tier bench lines
OUT=gpurun_out; T=r02av; mkdir -p $OUT
bash profiles/run_round.sh $T
B="python bench.py --no-cpu-baseline --steps 20 --warmup 5"
timeout 900 $B --host-frac 0.25 > $OUT/${T}_bench_host25.json 2> $OUT/${T}_bench_host25.err
timeout 900 $B --host-frac 0.1 > $OUT/${T}_bench_host10.json 2> $OUT/${T}_bench_host10.err
timeout 900 $B --host-frac 0.05 > $OUT/${T}_bench_host05.json 2> $OUT/${T}_bench_host05.err
echo all-done
