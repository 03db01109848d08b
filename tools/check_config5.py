"""Developer check: config 5 (R-MAT 23, ~66M edges) end to end on one GPU with the
whole-matrix invariants of the GPU test suite (orbit 0 = degree, per-pattern consistency)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch

import graphgen
import paper_1911_10616_b200 as pkg
from test_gpu_parity import _invariants

g = graphgen.config(5)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
t0 = time.perf_counter()
out, st = pkg.evoke_orbits_edges(g.n, e, return_stats=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"config 5: n {g.n} m {st['m']} wall {t1 - t0:.1f} s, lib {st['ms_total'] / 1e3:.1f} s")
print({k: round(v / 1e3, 2) for k, v in st["ms_pass"].items() if v > 100})
if "--no-check" not in sys.argv:
    x = out.cpu().numpy().view("uint64")
    _invariants(g, x, check_cliques=False)
    print("invariants ok")
