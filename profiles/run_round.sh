#!/bin/bash
# One GPU call's worth of round evidence (run under gpurun, 1 GPU):
#   the GPU suite and smoke, the default bench line (C4) and the reference arm,
#   then the ncu launch list and full captures (profiles/run_ncu.sh).
#   bash profiles/run_round.sh r02x
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu > $OUT/${TAG}_tests.log 2>&1; tail -3 $OUT/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; tail -1 $OUT/${TAG}_smoke.log
timeout 1700 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/${TAG}_bench_ref.json 2> $OUT/${TAG}_bench_ref.err
bash profiles/run_ncu.sh $TAG
echo done
