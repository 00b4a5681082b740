"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of one kernel from an
`ncu --set full` capture -> profiles/traffic.json, read by bench.py for roofline.traffic.

    python tools/traffic_from_ncu.py <rep.ncu-rep> <kernel-substring> <committed-copy-of-summary>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, kname, src = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
vals = []
for r in rows[2:]:
    if kname not in r[hdr.index("Kernel Name")]:
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        b += float(r[i]) * scale[units[i]]
    vals.append(b)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
res = {"kernel": kname, "launches": len(vals), "per_launch_bytes": sum(vals) / len(vals),
       "each": vals, "source": src}
json.dump(res, open(os.path.join(root, "profiles", "traffic.json"), "w"), indent=1)
print(res)
