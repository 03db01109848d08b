"""Per-pass timings of repeated calls (median of K) on one config: python tools/dev_timing.py CFG K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen
import paper_1911_10616_b200 as pkg

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
serial = "--serial" in sys.argv
warm = int(sys.argv[sys.argv.index("--warm") + 1]) if "--warm" in sys.argv else 2
g = graphgen.config(cfg)
dev = torch.device("cuda:0")
edges = torch.from_numpy(g.edges).to(dev)
out = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
rows = []
walls = []
for i in range(k + warm):
    _, st = pkg.evoke_orbits_edges(g.n, edges, out=out, return_stats=True, serial=serial)
    torch.cuda.synchronize()
    if i >= warm:
        rows.append(st["ms_pass"])
        walls.append(st["ms_total"])
if not rows:
    sys.exit(0)
keys = list(rows[0].keys())
med = {kk: float(np.median([r[kk] for r in rows])) for kk in keys}
mn = {kk: float(np.min([r[kk] for r in rows])) for kk in keys}
print(f"config {cfg}: wall median {float(np.median(walls)):.3f} ms (min {min(walls):.3f}); "
      f"sum of pass times {sum(med.values()):.3f} ms (concurrent passes overlap)")
for kk in keys:
    print(f"  {kk:14s} median {med[kk]:8.3f}  min {mn[kk]:8.3f}  all {[round(r[kk], 2) for r in rows]}")
