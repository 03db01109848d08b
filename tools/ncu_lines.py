"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "":
        continue
    try:
        samp = float(r[4])
        ex = float(r[7] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, r[1][:100]])
    a[0] += samp
    a[1] += ex
tot = sum(v[0] for v in agg.values()) or 1
by = 1 if (len(sys.argv) > 3 and sys.argv[3] == "inst") else 0
for (f, ln), (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][by])[:top]:
    print(f"{100 * s / tot:5.1f}%  inst {e:10.3g}  {f}:{ln}  {src}")
