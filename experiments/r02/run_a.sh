#!/bin/bash
# r02a: state at the start of round 2 — box resources, GPU suite, C4 bench (no CPU baseline)
OUT=gpurun_out; T=r02a; mkdir -p $OUT
{ free -g; nproc; lscpu | grep -i "model name\|socket\|numa node(s)"; nvidia-smi --query-gpu=name,memory.total --format=csv; } > $OUT/${T}_box.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
( time timeout 1200 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline ) > $OUT/${T}_bench_c4.json 2> $OUT/${T}_bench_c4.err
tail -4 $OUT/${T}_bench_c4.err
python -c "
import json;d=json.load(open('$OUT/${T}_bench_c4.json'));a=d['access_prob']
print('gather',d['value'],d['roofline']['frac']); print('P',a['ms_per_call'],a['survey_model']['frac'],{k:round(v['ms_per_call'],3) for k,v in a['kernels'].items()}); print('e2e',d['e2e'],a.get('e2e'))"
