"""DRAM bytes per launch of the step kernels from an ncu --set full capture
(for bench.py's roofline.traffic): python tools/ncu_traffic.py rep.ncu-rep out.json"""
import csv
import json
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = rows[0]
out = {"source": sys.argv[1]}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    b = sum(float(r[hdr.index(k)].replace(",", "")) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    unit = rows[1][hdr.index("dram__bytes_read.sum")]
    b *= scale.get(unit, 1)
    key = "postmult" if "k_post" in name else "grammian" if "k_gram" in name else "inner" if "k_inner" in name else None
    if key:
        out["%s_dram_bytes_per_launch" % key] = b
        out["%s_kernel" % key] = name.split("(")[0]
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(out)
