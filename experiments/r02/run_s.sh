#!/bin/bash
# r02s: host-tier gather breakdown (ncu launch list at h=0.1) and QVB_HOST_EVERY A/B
OUT=gpurun_out; T=r02s; mkdir -p $OUT
B="python bench.py --no-cpu-baseline --no-e2e --sample-seeds 0 --steps 20 --warmup 5 --clock-window 0.5"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${T}_launches_h0.1.csv \
   python bench.py --steps 3 --warmup 3 --clock-window 0 --no-cpu-baseline --no-e2e --sample-seeds 0 --host-frac 0.1 > /dev/null 2>&1
python - $OUT/${T}_launches_h0.1.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
seq = [(r[ki].split("(")[0][-40:], float(r[vi].replace(",", "")), r[ui]) for r in rows[1:]]
for name, v, u in seq[-40:]:
    print(f"{name:42s} {v:12.1f} {u}")
PY
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1])); r=d['roofline']
print(sys.argv[2], 'gather %.1f GB/s frac %.3f ms %.4f' % (d['value'], r['frac'], r['per_launch_ms']))" $1 $2; }
for he in "0.1 2" "0.1 4" "0.1 16" "0.25 4"; do set -- $he; h=$1; e=$2
  QVB_HOST_EVERY=$e timeout 600 $B --host-frac $h > $OUT/${T}_h${h}_e$e.json 2> $OUT/${T}_h${h}_e$e.err
  summ $OUT/${T}_h${h}_e$e.json h${h}_every$e
done
