"""Degree-only closed forms of the non-induced counts DM(v, theta) (Def. "unlabeled-match",
P:419-422) for the star-like orbits, exact modulo 2^64 at any size (R20):

  theta0  = d(v)                         theta2  = C(d(v), 2)      (P3 centre)
  theta1  = sum_{u in N(v)} (d(u) - 1)   theta6  = sum_{u in N(v)} C(d(u) - 1, 2)  (3-star leaf)
  theta7  = C(d(v), 3)    (3-star centre)  theta22 = sum_{u in N(v)} C(d(u) - 1, 3) (4-star leaf)
  theta23 = C(d(v), 4)    (4-star centre)

(Lemma 4vertexorbit P:704-713 for theta1/theta2/theta6/theta7, P:1154/P:1158 for theta22 /
theta23.)  Pinned against the non-induced brute force in tests/test_oracle_pins.py; used on
every vertex of the large configs, hub rows included, by tests/test_gpu_parity.py.
"""
from math import comb

import numpy as np

M64 = 1 << 64
COLUMNS = (0, 1, 2, 6, 7, 22, 23)


def _binom_mod(x: np.ndarray, k: int) -> np.ndarray:
    u, inv = np.unique(x, return_inverse=True)
    tab = np.array([comb(int(v), k) % M64 if v >= k else 0 for v in u], dtype=np.uint64)
    return tab[inv.reshape(-1)]


def degree_forms(n: int, edges) -> dict:
    """{orbit: uint64[n]} for the columns in COLUMNS."""
    e = np.sort(np.asarray(edges, dtype=np.int64).reshape(-1, 2), axis=1)
    e = e[e[:, 0] != e[:, 1]]
    key = np.sort(e[:, 0] * max(n, 1) + e[:, 1])
    key = key[np.concatenate([[True], key[1:] != key[:-1]])] if key.size else key  # each edge once
    lo, hi = key // max(n, 1), key % max(n, 1)
    a = np.concatenate([lo, hi])
    b = np.concatenate([hi, lo])
    deg = np.bincount(a, minlength=n).astype(np.int64)

    def nbr_sum(f: np.ndarray) -> np.ndarray:  # sum_{u in N(v)} f(u), wrapping uint64
        # in three 22-bit limbs: each limb's sum over a neighbourhood stays below 2^53, so the
        # float64 bincount is exact; the limbs are recombined modulo 2^64
        out = np.zeros(n, dtype=np.uint64)
        vals = f[b].astype(np.uint64)
        for sh in (0, 22, 44):
            limb = ((vals >> np.uint64(sh)) & np.uint64((1 << 22) - 1)).astype(np.float64)
            s = np.bincount(a, weights=limb, minlength=n).astype(np.uint64)
            out += s << np.uint64(sh)
        return out

    dm1 = np.maximum(deg - 1, 0)
    return {0: deg.astype(np.uint64),
            1: nbr_sum(dm1.astype(np.uint64)),
            2: _binom_mod(deg, 2),
            6: nbr_sum(_binom_mod(dm1, 2)),
            7: _binom_mod(deg, 3),
            22: nbr_sum(_binom_mod(dm1, 3)),
            23: _binom_mod(deg, 4)}
