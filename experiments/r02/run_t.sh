#!/bin/bash
# r02t: k_split_classes with block-aggregated list atomics; products loop in whole 4-step rounds
OUT=gpurun_out; T=r02t; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gather_gpu.py tests/test_access_prob_gpu.py tests/test_sharded_p_gpu.py -x -q -m gpu > $OUT/${T}_tests.log 2>&1; tail -3 $OUT/${T}_tests.log
timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap.txt 2>&1; cat $OUT/${T}_ap.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${T}_launches_h0.1.csv \
   python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e --sample-seeds 0 --host-frac 0.1 > /dev/null 2>&1
python - $OUT/${T}_launches_h0.1.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
seq = [(r[ki].split("(")[0][-40:], float(r[vi].replace(",", "")), r[ui]) for r in rows[1:]]
for name, v, u in seq[-12:]:
    print(f"{name:42s} {v:12.1f} {u}")
PY
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']))" $1 $2; }
for he in "0.1 8" "0.1 2" "0.25 8" "0.25 2"; do set -- $he; h=$1; e=$2
  QVB_HOST_EVERY=$e timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_e$e.json 2> $OUT/${T}_h${h}_e$e.err
  summ $OUT/${T}_h${h}_e$e.json h${h}_every$e
done
