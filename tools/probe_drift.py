"""Developer probe: per-call time over many calls (drift?), device pointers, torch stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen
import paper_1911_10616_b200 as pkg

g = graphgen.config(2)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
out = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev)
ts = []
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 60):
    if "--flush" in sys.argv:
        flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    pkg.evoke_orbits_edges(g.n, e, out=out, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = np.array(ts)
for a in range(0, len(ts), 10):
    print(f"calls {a:3d}-{a + 9:3d}: mean {ts[a:a + 10].mean():.3f} min {ts[a:a + 10].min():.3f} max {ts[a:a + 10].max():.3f}")
