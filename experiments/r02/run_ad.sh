#!/bin/bash
# r02ad: round evidence on the final code: GPU suite, smoke, default C4 bench + reference arm, ncu;
# host-tier / C2 / C3 bench lines; sanitizers over every kernel family; the C4 gather sweep
OUT=gpurun_out; T=r02ad; mkdir -p $OUT
bash profiles/run_round.sh $T
B="python bench.py --no-cpu-baseline --steps 20 --warmup 5"
timeout 900 $B --host-frac 0.25 > $OUT/${T}_bench_host25.json 2> $OUT/${T}_bench_host25.err
timeout 900 $B --host-frac 0.1 > $OUT/${T}_bench_host10.json 2> $OUT/${T}_bench_host10.err
timeout 900 $B --host-frac 0.05 > $OUT/${T}_bench_host05.json 2> $OUT/${T}_bench_host05.err
timeout 900 $B --config C2 > $OUT/${T}_bench_c2.json 2> $OUT/${T}_bench_c2.err
timeout 900 $B --config C3 > $OUT/${T}_bench_c3.json 2> $OUT/${T}_bench_c3.err
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python experiments/r02/sanitize.py > $OUT/${T}_sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -2 $OUT/${T}_sanitize_$tool.log
done
timeout 1500 python experiments/gather_sweep.py C4 > $OUT/${T}_gather_sweep_C4.jsonl 2> $OUT/${T}_gather_sweep_C4.err
echo all-done
