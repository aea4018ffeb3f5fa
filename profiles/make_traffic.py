"""Writes profiles/traffic.json from ncu --set full captures: per-launch
dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernels, which
bench.py reports as roofline.traffic.

    python profiles/make_traffic.py KEY KERNEL profiles/rXX_gather.ncu-rep

KEY names the exact bench line the capture belongs to,
"<config>|b<batch>|r<replicate>|h<host_frac>|n<gpus>" (bench.traffic_key), e.g.
"C4|b1048576|r0|h0|n1"; bench.py reports a traffic number only for a line
with exactly that key (otherwise null).
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def dram_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for v in rows[2:]:
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(v[i].replace(",", "")) * scale[u[i]]
        out.append(tot)
    return out


if __name__ == "__main__":
    cfg, kernel, rep = sys.argv[1:4]
    path = os.path.join(HERE, "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    b = dram_bytes(rep)
    ent = {"bytes_per_launch": sum(b) / len(b), "launches": len(b), "source": os.path.basename(rep)}
    data.setdefault(cfg, {})[kernel] = ent
    json.dump(data, open(path, "w"), indent=1, sort_keys=True)
    print(cfg, kernel, ent)
