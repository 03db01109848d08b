"""Developer probe: where the end-to-end (host buffers) call spends its time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen
import paper_1911_10616_b200 as pkg

g = graphgen.config(2)
h_edges = torch.from_numpy(g.edges).pin_memory()
h_out = torch.empty((g.n, 73), dtype=torch.int64).pin_memory()
he = h_edges.numpy()
ho = h_out.numpy().view(np.uint64)
for i in range(6):
    t0 = time.perf_counter()
    _, st = pkg.evoke_orbits_edges(g.n, he, out=ho, return_stats=True)
    t1 = time.perf_counter()
    print(f"host {1e3 * (t1 - t0):.2f} ms  lib total {st['ms_total']:.2f}  h2d {st['ms_pass']['h2d']:.3f} "
          f"d2h {st['ms_pass']['d2h']:.3f} canon {st['ms_pass']['canonicalise']:.3f}")
ho2 = np.empty((g.n, 73), dtype=np.uint64)  # pageable
t0 = time.perf_counter()
_, st = pkg.evoke_orbits_edges(g.n, he, out=ho2, return_stats=True)
print(f"pageable out: host {1e3 * (time.perf_counter() - t0):.2f} ms  d2h {st['ms_pass']['d2h']:.3f}")
