"""Write profiles/ncu_traffic.json: per-kernel DRAM bytes per launch from an ncu --set full report."""
import csv
import io
import json
import subprocess
import sys

rep, out, nodes = sys.argv[1], sys.argv[2], int(sys.argv[3])
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("<")[0].replace("void ", "").strip()
    rd = float(r[hdr.index("dram__bytes_read.sum")]) * scale[units[hdr.index("dram__bytes_read.sum")]]
    wr = float(r[hdr.index("dram__bytes_write.sum")]) * scale[units[hdr.index("dram__bytes_write.sum")]]
    res[name] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                 "per_node": (rd + wr) / nodes}
json.dump({"source": rep, "nodes": nodes, "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
