#!/bin/bash
# r02b: default bench (C4) with CPU baseline + reference arm at C4; new placement/gather tests
OUT=gpurun_out; T=r02b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_placement_gpu.py tests/test_gather_gpu.py tests/test_reads_resident_gpu.py -q -x > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
( time timeout 1700 python bench.py --steps 20 --warmup 5 ) > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err
tail -4 $OUT/${T}_bench.err
( time timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/${T}_bench_ref.json 2> $OUT/${T}_bench_ref.err
tail -4 $OUT/${T}_bench_ref.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02b_bench.json')); a=d['access_prob']
print('gather',d['value'],d['roofline']['frac'],'e2e',d['e2e']['value'])
print('P',a['ms_per_call'],a['survey_model']['frac'],{k:round(v['ms_per_call'],3) for k,v in a['kernels'].items()})
print('cpu',d['cpu_baseline']); print('apcpu',a.get('cpu_baseline'))
r=json.load(open('gpurun_out/r02b_bench_ref.json')); print('ref',r['value'],r['access_prob'],r['planner'])
print('same_config', r['config']==d['config'])
PY
