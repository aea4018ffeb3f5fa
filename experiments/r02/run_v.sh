#!/bin/bash
# r02v: round evidence on the current code (GPU suite, smoke, default C4 bench + reference arm,
# ncu launch list + captures), plus host-tier bench lines, C2/C3 lines and the C4 gather sweep
OUT=gpurun_out; T=r02v; mkdir -p $OUT
bash profiles/run_round.sh $T
B="python bench.py --no-cpu-baseline --steps 20 --warmup 5"
timeout 900 $B --host-frac 0.25 > $OUT/${T}_bench_host25.json 2> $OUT/${T}_bench_host25.err
timeout 900 $B --host-frac 0.1 > $OUT/${T}_bench_host10.json 2> $OUT/${T}_bench_host10.err
timeout 900 $B --config C2 > $OUT/${T}_bench_c2.json 2> $OUT/${T}_bench_c2.err
timeout 900 $B --config C3 > $OUT/${T}_bench_c3.json 2> $OUT/${T}_bench_c3.err
timeout 1500 python experiments/gather_sweep.py C4 > $OUT/${T}_gather_sweep_C4.jsonl 2> $OUT/${T}_gather_sweep_C4.err
echo all-done
