#!/bin/bash
# r02c: new GPU tests (drop-in graph/view, resident read plans, tier-split gather,
# the reference's own unit tests on the drop-in) + split-gather and segment-size A/B
OUT=gpurun_out; T=r02c; mkdir -p $OUT
timeout 1500 python -m pytest -q -x tests/test_reference_tests_gpu.py tests/test_dropin_graph_gpu.py \
  tests/test_reads_resident_gpu.py tests/test_gather_gpu.py tests/test_cpp_dropin_gpu.py \
  tests/test_placement_gpu.py > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python experiments/r02/sanitize.py > $OUT/${T}_sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -2 $OUT/${T}_sanitize_$tool.log
done
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 10 --warmup 3 --clock-window 0.3"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); a=d['access_prob']; r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f (%s) ms %.3f' % (d['value'], r['frac'], r['bound'], r['per_launch_ms']), 'P %.3f ms %.3f' % (a['ms_per_call'], a['survey_model']['frac']), {k: round(v['ms_per_call'],3) for k,v in a['kernels'].items()})" $1 $2; }
for cfg in C4 C2; do for h in 0.1 0.25; do for sp in 1 0; do
  QVB_GATHER_SPLIT=$sp timeout 600 $B --config $cfg --host-frac $h > $OUT/${T}_${cfg}_h${h}_s${sp}.json 2> $OUT/${T}_${cfg}_h${h}_s${sp}.err
  summ $OUT/${T}_${cfg}_h${h}_s${sp}.json ${cfg}_h${h}_split${sp}
done; done; done
for mb in 40 48 56 64; do
  QVB_SEG_MB=$mb timeout 600 $B --config C4 > $OUT/${T}_seg${mb}.json 2> $OUT/${T}_seg${mb}.err
  summ $OUT/${T}_seg${mb}.json seg${mb}
done
