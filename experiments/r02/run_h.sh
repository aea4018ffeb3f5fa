#!/bin/bash
# r02h: 512-byte row gather A/B with deeper lookup prefetch; class gather (host tier) with the 512-byte path
OUT=gpurun_out; T=r02h; mkdir -p $OUT
timeout 900 python -m pytest -q -x tests/test_gather_gpu.py > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'])" $1 $2; }
for v in 0 5 6 7 4 0; do
  QVB_GATHER_U=$v timeout 600 $B > $OUT/${T}_C4_u$v.json 2> $OUT/${T}_C4_u$v.err; summ $OUT/${T}_C4_u$v.json C4_u$v
done
for h in 0.1 0.25; do
  timeout 600 $B --host-frac $h > $OUT/${T}_C4_h$h.json 2> $OUT/${T}_C4_h$h.err; summ $OUT/${T}_C4_h$h.json C4_h$h
done
