#!/bin/bash
# r02j: sharded P tests (thread ranks, two gloo processes), host bucket bits A/B with the device scan
OUT=gpurun_out; T=r02j; mkdir -p $OUT
timeout 1200 python -m pytest -q -x tests/test_sharded_p_gpu.py tests/test_dist_gpu.py tests/test_gather_gpu.py tests/test_access_prob_gpu.py -k "not c4_full" > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']))" $1 $2; }
for h in 0.25 0.1; do for bits in 16 17 18 14; do
  QVB_HOST_BUCKET_BITS=$bits timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_b$bits.json 2> $OUT/${T}_h${h}_b$bits.err
  summ $OUT/${T}_h${h}_b$bits.json h${h}_bits$bits
done; done
