"""Seeded synthetic graph generators shared by the oracle tests and the CUDA path.

This module holds NO orbit-counting arithmetic: it only produces raw undirected edge
lists (int32 pairs, possibly with duplicates / reverse duplicates / self-loops, exactly
like a raw input file -- cleaning is the counted method's job).

The five BASELINE.json configs:
  1  Erdos-Renyi G(n=120, p=0.05), seed 1
  2  Chung-Lu, n=100,000, expected degrees Pareto tail exponent gamma=2.5, mean 10, seed 2
  3  R-MAT scale 18, edge factor 16, (a,b,c,d)=(.57,.19,.19,.05), seed 3
  4  Holme-Kim n=2,000,000, m=8, triad probability 0.5, seed 4
  5  R-MAT scale 23, edge factor 8, (.57,.19,.19,.05), seed 5
plus closed-form families (K_n, C_n, K_{1,s}, K_{a,b}, Petersen) and tiled disjoint
unions used for parity at scale.  These synthetic graphs stand in for the paper's
public datasets (Table 1), which are not available offline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lock = threading.Lock()
_hk = None


@dataclass
class Graph:
    name: str
    n: int
    edges: np.ndarray  # int32 [k, 2], raw (may contain duplicates / self-loops)

    @property
    def m_raw(self) -> int:
        return int(self.edges.shape[0])


def _hk_lib():
    global _hk
    with _lock:
        if _hk is None:
            src = os.path.join(_HERE, "holme_kim.c")
            so = os.path.join(_HERE, "_build", "libholmekim.so")
            os.makedirs(os.path.dirname(so), exist_ok=True)
            if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
                tmp = so + f".tmp{os.getpid()}"
                subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, src])
                os.replace(tmp, so)
            lib = ctypes.CDLL(so)
            lib.holme_kim.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                      ctypes.POINTER(ctypes.c_int32)]
            lib.holme_kim.restype = ctypes.c_int64
            _hk = lib
    return _hk


def erdos_renyi(n: int, p: float, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    r = rng.random((n, n))
    iu = np.triu_indices(n, 1)
    keep = r[iu] < p
    e = np.stack([iu[0][keep], iu[1][keep]], axis=1).astype(np.int32)
    return Graph(f"er_n{n}_p{p}_s{seed}", n, e)


def chung_lu(n: int, gamma: float, mean_degree: float, seed: int) -> Graph:
    """Fast Chung-Lu: weights with P(W > x) ~ x^-(gamma-1), rescaled to the mean degree;
    n*mean/2 edges with both endpoints drawn proportional to weight (then the method
    dedupes and drops self-loops)."""
    rng = np.random.default_rng(seed)
    w = 1.0 + rng.pareto(gamma - 1.0, size=n)
    w *= mean_degree / w.mean()
    m = int(round(n * mean_degree / 2))
    p = w / w.sum()
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    u = np.searchsorted(cdf, rng.random(m), side="right")
    v = np.searchsorted(cdf, rng.random(m), side="right")
    e = np.stack([np.minimum(u, n - 1), np.minimum(v, n - 1)], axis=1).astype(np.int32)
    return Graph(f"chunglu_n{n}_g{gamma}_d{mean_degree}_s{seed}", n, e)


def rmat(scale: int, edge_factor: int, a: float, b: float, c: float, d: float, seed: int,
         chunk: int = 1 << 24) -> Graph:
    """R-MAT (Chakrabarti et al.): each edge picks one quadrant per level; no noise,
    no id permutation.  Symmetrisation/dedupe/self-loop removal is the method's job."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    out = np.empty((m, 2), dtype=np.int32)
    ab, abc = a + b, a + b + c
    for s in range(0, m, chunk):
        k = min(chunk, m - s)
        src = np.zeros(k, dtype=np.int64)
        dst = np.zeros(k, dtype=np.int64)
        for level in range(scale):
            r = rng.random(k)
            bit = np.int64(1) << (scale - 1 - level)
            down = r >= ab                      # quadrants c, d: source bit set
            right = ((r >= a) & (r < ab)) | (r >= abc)  # quadrants b, d: target bit set
            src += down * bit
            dst += right * bit
        out[s:s + k, 0] = src
        out[s:s + k, 1] = dst
    return Graph(f"rmat_s{scale}_ef{edge_factor}_s{seed}", n, out)


def holme_kim(n: int, m: int, p: float, seed: int) -> Graph:
    lib = _hk_lib()
    buf = np.empty((n * m, 2), dtype=np.int32)
    k = lib.holme_kim(n, m, p, seed, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return Graph(f"holmekim_n{n}_m{m}_p{p}_s{seed}", n, np.ascontiguousarray(buf[:k]))


def config(i: int) -> Graph:
    """BASELINE.json configs[i-1] (1-based)."""
    if i == 1:
        return erdos_renyi(120, 0.05, 1)
    if i == 2:
        return chung_lu(100_000, 2.5, 10.0, 2)
    if i == 3:
        return rmat(18, 16, 0.57, 0.19, 0.19, 0.05, 3)
    if i == 4:
        return holme_kim(2_000_000, 8, 0.5, 4)
    if i == 5:
        return rmat(23, 8, 0.57, 0.19, 0.19, 0.05, 5)
    raise ValueError(i)


CONFIG_NAMES = {
    1: "ER G(120,0.05) seed 1",
    2: "Chung-Lu n=1e5 gamma=2.5 mean deg 10 seed 2",
    3: "R-MAT scale 18 ef 16 (.57,.19,.19,.05) seed 3",
    4: "Holme-Kim n=2e6 m=8 p=0.5 seed 4",
    5: "R-MAT scale 23 ef 8 (.57,.19,.19,.05) seed 5",
}


# ---- closed-form families and tiled graphs ---------------------------------

def complete(n: int) -> Graph:
    iu = np.triu_indices(n, 1)
    return Graph(f"K{n}", n, np.stack(iu, axis=1).astype(np.int32))


def cycle(n: int) -> Graph:
    a = np.arange(n)
    return Graph(f"C{n}", n, np.stack([a, (a + 1) % n], axis=1).astype(np.int32))


def path(n: int) -> Graph:
    a = np.arange(n - 1)
    return Graph(f"P{n}", n, np.stack([a, a + 1], axis=1).astype(np.int32))


def star(s: int) -> Graph:
    leaves = np.arange(1, s + 1)
    return Graph(f"K1,{s}", s + 1, np.stack([np.zeros(s, dtype=np.int64), leaves], axis=1).astype(np.int32))


def complete_bipartite(a: int, b: int) -> Graph:
    x, y = np.meshgrid(np.arange(a), np.arange(a, a + b), indexing="ij")
    return Graph(f"K{a},{b}", a + b, np.stack([x.ravel(), y.ravel()], axis=1).astype(np.int32))


def petersen() -> Graph:
    outer = [(i, (i + 1) % 5) for i in range(5)]
    spokes = [(i, i + 5) for i in range(5)]
    inner = [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    return Graph("petersen", 10, np.array(outer + spokes + inner, dtype=np.int32))


def disjoint_union(parts: list[Graph], name: str = "union") -> tuple[Graph, np.ndarray]:
    """Concatenate graphs with shifted ids. Returns (graph, offsets[len(parts)+1])."""
    offs = np.zeros(len(parts) + 1, dtype=np.int64)
    for i, g in enumerate(parts):
        offs[i + 1] = offs[i] + g.n
    e = np.concatenate([g.edges.astype(np.int64) + offs[i] for i, g in enumerate(parts)], axis=0)
    return Graph(name, int(offs[-1]), e.astype(np.int32)), offs


def tiled(num_tiles: int, tile_n: int, tile_p: float, seed: int, distinct: int = 64) -> tuple[Graph, list[int]]:
    """Disjoint union of ``num_tiles`` copies drawn from ``distinct`` seeded G(tile_n, tile_p)
    tiles. Returns (graph, tile_index_per_copy) so an oracle need only solve the distinct
    tiles."""
    tiles = [erdos_renyi(tile_n, tile_p, seed * 1000 + i) for i in range(distinct)]
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, distinct, size=num_tiles)
    g, _ = disjoint_union([tiles[i] for i in pick], f"tiled_{num_tiles}x{tile_n}_p{tile_p}_s{seed}")
    return g, [int(i) for i in pick]


def random_small(n: int, p: float, seed: int) -> Graph:
    return erdos_renyi(n, p, seed)


def add_noise(g: Graph, seed: int, frac: float = 0.1) -> Graph:
    """Append reverse duplicates, exact duplicates and self-loops (input-cleaning tests)."""
    rng = np.random.default_rng(seed)
    k = max(1, int(frac * g.m_raw)) if g.m_raw else 0
    extra = []
    if k:
        idx = rng.integers(0, g.m_raw, size=k)
        extra.append(g.edges[idx][:, ::-1])
        extra.append(g.edges[idx])
    if g.n:
        loops = rng.integers(0, g.n, size=max(1, k // 2))
        extra.append(np.stack([loops, loops], axis=1).astype(np.int32))
    e = np.concatenate([g.edges] + extra, axis=0).astype(np.int32) if extra else g.edges
    perm = rng.permutation(e.shape[0])
    return Graph(g.name + "+noise", g.n, np.ascontiguousarray(e[perm]))
