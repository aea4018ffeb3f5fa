#!/bin/bash
# r02i: host-tier A/B (bucket bits 16 vs 18, class 512-byte path on/off), row gather through a lookup table (microbench)
OUT=gpurun_out; T=r02i; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o experiments/r02/rowgather experiments/r02/rowgather.cu
./experiments/r02/rowgather > $OUT/${T}_rowgather.txt 2>&1; tail -4 $OUT/${T}_rowgather.txt
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']))" $1 $2; }
for h in 0.25 0.1; do for cfg in "18 1" "16 1" "18 0" "16 0"; do set -- $cfg
  QVB_HOST_BUCKET_BITS=$1 QVB_CLASS_R512=$2 timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_b$1_r$2.json 2> $OUT/${T}_h${h}_b$1_r$2.err
  summ $OUT/${T}_h${h}_b$1_r$2.json h${h}_bits$1_r512$2
done; done
