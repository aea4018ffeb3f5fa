#!/bin/bash
# r02p: k_first with the whole slice in flight (C4 P call, f1 window 32 vs 256),
# host-tier class gather with small host groups (QVB_HOST_GROUP A/B)
OUT=gpurun_out; T=r02p; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gather_gpu.py tests/test_access_prob_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
for w in 32 256; do QVB_F1_WINDOW=$w timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_w$w.txt 2>&1; echo "f1 window $w"; cat $OUT/${T}_ap_w$w.txt; done
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']), 'P', d['access_prob']['ms_per_call'], d['access_prob']['kernels']['k_first']['ms_per_call'])" $1 $2; }
for hg in "0.25 4" "0.25 1" "0.25 2" "0.25 32" "0.1 4" "0.1 32"; do set -- $hg; h=$1; g=$2
  QVB_HOST_GROUP=$g timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_g$g.json 2> $OUT/${T}_h${h}_g$g.err
  summ $OUT/${T}_h${h}_g$g.json h${h}_group$g
done
