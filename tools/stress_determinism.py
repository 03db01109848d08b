"""Developer stress test: repeated calls must give bit-identical matrices.
    python tools/stress_determinism.py CFG REPS [--shards N] [--serial]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen
import paper_1911_10616_b200 as pkg

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
shards = int(sys.argv[sys.argv.index("--shards") + 1]) if "--shards" in sys.argv else 1
serial = "--serial" in sys.argv
induced = "--raw" not in sys.argv  # --raw: non-induced DM columns (which raw count differs)
g = graphgen.config(cfg)
dev = torch.device("cuda:0")
e = torch.from_numpy(g.edges).to(dev)


def run():
    tot = None
    for si in range(shards):
        out = pkg.evoke_orbits_edges(g.n, e, shard_index=si, num_shards=shards, serial=serial, induced=induced)
        torch.cuda.synchronize()
        x = out.cpu().numpy().view(np.uint64).copy()
        tot = x if tot is None else tot + x
    return tot


ref = run()
bad = 0
for r in range(reps):
    x = run()
    d = np.argwhere(x != ref)
    if d.size:
        bad += 1
        rows = np.unique(d[:, 0])
        print(f"rep {r}: {len(d)} differing entries in {len(rows)} rows, e.g. {d[:6].tolist()}")
        for v in rows[:3]:
            cols = np.nonzero(x[v] != ref[v])[0]
            print(f"   vertex {v}: columns {cols.tolist()} diff {[(int(x[v][c]) - int(ref[v][c])) for c in cols[:6]]}")
print(f"config {cfg} shards {shards} serial {serial}: {bad}/{reps} runs differ from the first")
