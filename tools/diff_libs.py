"""Developer A/B: run the in-tree library and another build (EVOKE_LIB_PATH of a child) on one
config and report which orbit columns differ, for how many vertices, and those vertices'
degrees.   python tools/diff_libs.py CFG OTHER_SO [ENV=VAL ...]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(cfg, lib, env_kv, out):
    env = dict(os.environ)
    if lib:
        env["EVOKE_LIB_PATH"] = lib
    for kv in env_kv:
        k, v = kv.split("=", 1)
        env[k] = v
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import numpy as np, graphgen, paper_1911_10616_b200 as p; "
            f"g = graphgen.config({cfg}); np.save({out!r}, p.evoke_orbits_edges(g.n, g.edges, induced=False, serial=bool(int(__import__('os').environ.get('DIFF_SERIAL', '0')))))")
    subprocess.check_call([sys.executable, "-c", code], env=env)


if __name__ == "__main__":
    cfg, other = int(sys.argv[1]), sys.argv[2]
    kv = sys.argv[3:]
    run(cfg, None, kv, "/tmp/a.npy")
    run(cfg, other, kv, "/tmp/b.npy")
    a, b = np.load("/tmp/a.npy"), np.load("/tmp/b.npy")
    sys.path.insert(0, ROOT)
    import graphgen
    g = graphgen.config(cfg)
    e = np.unique(np.sort(g.edges.astype(np.int64), axis=1), axis=0)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=g.n)
    diff = a != b
    print(f"config {cfg} {kv}: {int(diff.any(axis=1).sum())} rows differ")
    for c in np.flatnonzero(diff.any(axis=0)):
        rows = np.flatnonzero(diff[:, c])
        print(f"  orbit {c}: {rows.size} rows; degrees {np.sort(deg[rows])[-8:].tolist()} (max), first rows {rows[:5].tolist()}")
        d = (a[rows, c].astype(np.uint64) - b[rows, c].astype(np.uint64)).astype(np.int64)
        print(f"    new - other: {d[:12].tolist()}; degrees {deg[rows][:12].tolist()}")
