"""profiles/traffic.json from an ncu report: DRAM bytes (read + write) per
launch of the bench's dominant kernels (bench.py fills roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    key = "tttp" if "tttp_kernel" in name else ("mttkrp0" if "mttkrp_kernel" in name else None)
    if key is None or key in res:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(r[hdr.index(m)])
        u = units[hdr.index(m)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        tot += v * scale
    res[key] = tot
res["source"] = rep
json.dump(res, open(out, "w"), indent=1)
print(res)
