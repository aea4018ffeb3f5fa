#!/bin/bash
# r02af: qvb_gather_host pipeline depth (QVB_HOST_CHUNKS) against the 57.3 GB/s pinned D2H ceiling
OUT=gpurun_out; T=r02af; mkdir -p $OUT
B="python bench.py --no-cpu-baseline --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.3"
for c in 8 16 32 4; do
  QVB_HOST_CHUNKS=$c timeout 900 $B > $OUT/${T}_c$c.json 2> $OUT/${T}_c$c.err
  python -c "
import json,sys; d=json.load(open('$OUT/${T}_c$c.json')); print('chunks $c', 'e2e %.2f GB/s' % d['e2e']['value'], 'gather %.1f' % d['value'])"
done
