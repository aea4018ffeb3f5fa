#!/bin/bash
# r02d: host-tier ordering A/B (C4/C2 at h=0.1/0.25: split+bucketed, split unordered, mixed), sanitizers, gather tests
OUT=gpurun_out; T=r02d; mkdir -p $OUT
timeout 900 python -m pytest -q -x tests/test_gather_gpu.py -k "split or host" > $OUT/${T}_tests.log 2>&1; tail -2 $OUT/${T}_tests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python experiments/r02/sanitize.py > $OUT/${T}_sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -2 $OUT/${T}_sanitize_$tool.log
done
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 10 --warmup 3 --clock-window 0.3"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f (%s) ms %.3f' % (d['value'], r['frac'], r['bound'], r['per_launch_ms']))" $1 $2; }
for cfg in C4 C2; do for h in 0.1 0.25; do for mode in "1 1" "1 0" "0 1"; do set -- $mode
  QVB_GATHER_SPLIT=$1 QVB_HOST_SORT=$2 timeout 600 $B --config $cfg --host-frac $h > $OUT/${T}_${cfg}_h${h}_s$1$2.json 2> $OUT/${T}_${cfg}_h${h}_s$1$2.err
  summ $OUT/${T}_${cfg}_h${h}_s$1$2.json ${cfg}_h${h}_split$1_sort$2
done; done; done
timeout 600 $B --config C4 --host-frac 0.25 --planned > $OUT/${T}_C4_h0.25_planned.json 2>/dev/null; summ $OUT/${T}_C4_h0.25_planned.json C4_h0.25_planned
ncu --query-metrics 2>/dev/null | grep -iE "^(pcie|nvl|lts__t_sectors_srcunit|dram__bytes)" | head -40 > $OUT/${T}_ncu_metric_names.txt
wc -l $OUT/${T}_ncu_metric_names.txt
