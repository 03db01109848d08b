"""Developer: smallest hubby random graph on which two library builds differ (non-induced).
    python tools/find_small_diff.py OTHER_SO"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
other = sys.argv[1]


def gen(seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(50, 4000))
    extra = int(rng.integers(0, 300))
    n = 1 + k + extra
    hubs = int(rng.integers(1, 4))
    E = []
    for h in range(hubs):
        kk = int(rng.integers(k // 2, k + 1))
        nb = rng.choice(np.arange(hubs, n), size=min(kk, n - hubs), replace=False)
        E += [(h, int(x)) for x in nb]
    mm = int(rng.integers(n, 6 * n))
    a = rng.integers(0, n, mm)
    b = rng.integers(0, n, mm)
    E += [(int(x), int(y)) for x, y in zip(a, b) if x != y]
    perm = rng.permutation(n)
    return n, np.array([(perm[x], perm[y]) for x, y in E], dtype=np.int32)


graphs = [gen(s) for s in range(150)]
np.save("/tmp/graphs.npy", np.array(graphs, dtype=object), allow_pickle=True)
code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1911_10616_b200 as p; "
        "G = np.load('/tmp/graphs.npy', allow_pickle=True); "
        "np.save(sys.argv[1], np.array([p.evoke_orbits_edges(n, e, induced=False) for n, e in G], dtype=object), "
        "allow_pickle=True)") % ROOT
subprocess.check_call([sys.executable, "-c", code, "/tmp/A.npy"])
env = dict(os.environ, EVOKE_LIB_PATH=other)
subprocess.check_call([sys.executable, "-c", code, "/tmp/B.npy"], env=env)
A = np.load("/tmp/A.npy", allow_pickle=True)
B = np.load("/tmp/B.npy", allow_pickle=True)
bad = [(graphs[i][0], len(graphs[i][1]), i) for i in range(len(graphs)) if not np.array_equal(A[i], B[i])]
print("differing graphs:", len(bad), "of", len(graphs))
bad.sort()
for n, m, i in bad[:3]:
    a, b = A[i], B[i]
    cols = np.flatnonzero((a != b).any(axis=0)).tolist()
    rows = np.flatnonzero((a != b).any(axis=1)).tolist()
    print(f"graph {i}: n={n} m={m} cols {cols} rows {rows}")
    print(" new", [a[r, 51] for r in rows][:10], "\n ref", [b[r, 51] for r in rows][:10])
    print(" edges", json.dumps(graphs[i][1].tolist()))
