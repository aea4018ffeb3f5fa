#!/bin/bash
# r02q: k_first with the 4-byte class table (narrow) vs the 8-byte one; host groups at h=0.1
OUT=gpurun_out; T=r02q; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
for nw in 1 0; do QVB_F1_NARROW=$nw timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_n$nw.txt 2>&1; echo "narrow $nw"; cat $OUT/${T}_ap_n$nw.txt; done
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']), 'P', d['access_prob']['ms_per_call'], d['access_prob']['kernels']['k_first']['ms_per_call'])" $1 $2; }
for hg in "0.1 2" "0.1 1"; do set -- $hg; h=$1; g=$2
  QVB_HOST_GROUP=$g timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_g$g.json 2> $OUT/${T}_h${h}_g$g.err
  summ $OUT/${T}_h${h}_g$g.json h${h}_group$g
done
