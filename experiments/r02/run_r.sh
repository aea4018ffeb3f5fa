#!/bin/bash
# r02r: k_codes gathers with L2 evict_last (QVB_CODES_KEEP=1) vs plain ldg: time and DRAM bytes
OUT=gpurun_out; T=r02r; mkdir -p $OUT
for kp in 0 1; do QVB_CODES_KEEP=$kp timeout 900 python experiments/ap_bench.py C4 > $OUT/${T}_ap_k$kp.txt 2>&1; echo "keep $kp"; cat $OUT/${T}_ap_k$kp.txt; done
for kp in 0 1; do
  QVB_CODES_KEEP=$kp timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
     --clock-control none --csv -k regex:k_codes -c 14 --log-file $OUT/${T}_codes_k$kp.csv python experiments/ap_bench.py C4 > /dev/null 2>&1
  python - $OUT/${T}_codes_k$kp.csv $kp <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit"); ii = h.index("ID")
d = collections.defaultdict(dict)
for r in rows[1:]:
    d[r[ii]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
ids = sorted(d, key=int)[-7:]  # one P call's 7 segment launches
def tot(m):
    s = 0.0
    for i in ids:
        v, u = d[i][m]
        s += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
    return s
print("keep", sys.argv[2], "k_codes x7: time %.3f ms, DRAM read %.2f GB write %.2f GB" % (tot("gpu__time_duration.sum") * 1e3, tot("dram__bytes_read.sum") / 1e9, tot("dram__bytes_write.sum") / 1e9),
      "L2 hit %s" % [round(d[i]["lts__t_sector_hit_rate.pct"][0], 1) for i in ids])
PY
done
