#!/bin/bash
# r02ah: 1-row host groups on the ordered host list: gather tests, uniform host knobs, C4 host bench lines
OUT=gpurun_out; T=r02ah; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gather_gpu.py tests/test_calibrate_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
timeout 1500 python experiments/r02/host_knobs.py > $OUT/${T}_host_knobs.txt 2>&1; cat $OUT/${T}_host_knobs.txt
B="python bench.py --no-cpu-baseline --sample-seeds 0 --steps 20 --warmup 5"
for h in 0.25 0.1 0.05; do
  timeout 900 $B --host-frac $h > $OUT/${T}_bench_h$h.json 2> $OUT/${T}_bench_h$h.err
  python -c "
import json; d=json.load(open('$OUT/${T}_bench_h$h.json')); r=d['roofline']
print('h=$h', 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']), 'e2e %.1f' % d['e2e']['value'])"
done
timeout 1500 python experiments/gather_sweep.py C4 > $OUT/${T}_gather_sweep_C4.jsonl 2> $OUT/${T}_gather_sweep_C4.err
