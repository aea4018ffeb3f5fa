#!/bin/bash
# r02f: full GPU suite (timed, slowest tests), smoke, row-gather ceiling microbenchmark,
# default bench without the CPU baseline (new drop-in P leg)
OUT=gpurun_out; T=r02f; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o experiments/r02/rowgather experiments/r02/rowgather.cu
./experiments/r02/rowgather > $OUT/${T}_rowgather.txt 2>&1; cat $OUT/${T}_rowgather.txt
( time timeout 2400 python -m pytest tests -q -m gpu --durations=20 ) > $OUT/${T}_tests.log 2>&1; tail -32 $OUT/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${T}_smoke.log 2>&1; tail -1 $OUT/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
python -c "
import json; d=json.load(open('$OUT/${T}_bench.json')); a=d['access_prob']
print('gather', d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['roofline']['kernel'])
print('P', a['ms_per_call'], a['survey_model']['frac'], a['roofline'].get('traffic'))
print('e2e', d['e2e']['value'], a['e2e']['wall_s'], a.get('e2e_dropin'))
print('planner', d['planner'])"
