"""Developer probe: per-call time by the stream the caller passes (own / torch default / side)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen
import paper_1911_10616_b200 as pkg

g = graphgen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)
out = torch.empty((g.n, 73), dtype=torch.int64, device=dev)
side = torch.cuda.Stream(dev)
for name, st in [("own", None), ("torch-default", torch.cuda.current_stream(dev)), ("side", side)]:
    for stats in (False, True):
        ts, libs = [], []
        for i in range(12):
            s = st if st is not None else torch.cuda.current_stream(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            r = pkg.evoke_orbits_edges(g.n, e, out=out, stream=None if st is None else st.cuda_stream,
                                       return_stats=stats)
            e1.record(s)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
                if stats:
                    libs.append(r[1]["ms_total"])
        print(f"{name:14s} stats={stats}: event median {np.median(ts):.3f} mean {np.mean(ts):.3f}"
              + (f"  lib ms_total median {np.median(libs):.3f}" if libs else ""))
