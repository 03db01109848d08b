"""Write profiles/traffic.json: DRAM bytes per launch of each pass's kernels, from ncu
--set full reports (one report per kernel, as captured by tools/gpu_prof.sh).
    python tools/ncu_traffic.py CONFIG pass=report.ncu-rep [pass=report.ncu-rep ...]
CONFIG = the BASELINE config index the captures were taken on (bench.py only uses the file
for that config)."""
import csv
import io
import json
import subprocess
import sys

out = {"how": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full --clock-control none",
       "config": int(sys.argv[1]), "passes": {}, "kernels": {}}
for arg in sys.argv[2:]:
    pas, rep = arg.split("=", 1)
    raw = (open(rep).read() if rep.endswith(".csv") else
           subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(v[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
    wr = float(v[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else rep
    out["kernels"][name[:80]] = {"pass": pas, "dram_bytes": rd + wr, "report": rep}
    out["passes"][pas] = out["passes"].get(pas, 0.0) + rd + wr
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
