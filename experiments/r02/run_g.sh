#!/bin/bash
# r02g: row-gather kernel A/B at C4 (D=128) and C2 (D=100: k_gather_rows either way), tests of the new kernel
OUT=gpurun_out; T=r02g; mkdir -p $OUT
timeout 900 python -m pytest -q -x tests/test_gather_gpu.py > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']), d['clocks'])" $1 $2; }
for v in 0 5 7 4; do
  QVB_GATHER_U=$v timeout 600 $B > $OUT/${T}_C4_u$v.json 2> $OUT/${T}_C4_u$v.err; summ $OUT/${T}_C4_u$v.json C4_u$v
done
for v in 0 4; do
  QVB_GATHER_U=$v timeout 600 $B --config C2 > $OUT/${T}_C2_u$v.json 2> $OUT/${T}_C2_u$v.err; summ $OUT/${T}_C2_u$v.json C2_u$v
done
ncu --set full --clock-control none --import-source on -k regex:k_gather_rows512 -s 3 -c 1 -o $OUT/${T}_gather512 -f $B --steps 3 > /dev/null 2>&1; echo ncu=$?
