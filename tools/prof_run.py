"""Minimal profiling target: W warm-up calls + 1 call on config CFG (device pointers, serial
passes so each kernel runs alone).   python tools/prof_run.py CFG [W] [--concurrent]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen
import paper_1911_10616_b200 as pkg

cfg = int(sys.argv[1])
w = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
serial = "--concurrent" not in sys.argv
g = graphgen.config(cfg)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
out = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
for _ in range(w + 1):
    pkg.evoke_orbits_edges(g.n, e, out=out, serial=serial)
torch.cuda.synchronize()
print("ok")
