"""Work-model units of one config (one untimed call): python tools/dev_units.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import graphgen
import paper_1911_10616_b200 as pkg

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = graphgen.config(cfg)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
_, wm = pkg.evoke_orbits_edges(g.n, e, workmodel=True)
torch.cuda.synchronize()
print(f"config {cfg} units {wm['units']}")
print(f"config {cfg} alg_bytes {wm['alg_bytes']}")
