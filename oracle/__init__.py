"""CPU oracle for EVOKE's n x 73 induced vertex-orbit matrix -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1911_10616_b200``) never imports it and shares no code with it.

The arithmetic lives in ``evoke_oracle.c`` (plain C: ESU enumeration + adjacency-mask
lookup).  This module only
compiles it with gcc and marshals arguments through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

NUM_ORBITS = 73
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "evoke_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc -O2 -fopenmp). Returns its path."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            i64, i32p, u64p = ctypes.c_int64, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint64)
            ip = ctypes.POINTER(ctypes.c_int)
            lib.oracle_orbits_esu.argtypes = [i64, i64, i32p, u64p, ctypes.c_int]
            lib.oracle_orbit_row.argtypes = [i64, i64, i32p, i64, u64p, ctypes.c_uint64]
            lib.oracle_orbit_rows.argtypes = [i64, i64, i32p, i64, ctypes.POINTER(ctypes.c_int64), u64p,
                                              ip, ctypes.c_uint64, ctypes.c_int]
            lib.oracle_orbits_bruteforce.argtypes = [i64, i64, i32p, u64p]
            lib.oracle_noninduced_bruteforce.argtypes = [i64, i64, i32p, u64p]
            lib.oracle_clique_totals.argtypes = [i64, i64, i32p, u64p, ctypes.c_int, ctypes.c_int]
            lib.oracle_clique_totals_bits.argtypes = [i64, i64, i32p, u64p, ctypes.c_int, ctypes.c_int]
            lib.oracle_clique_counts_vertex.argtypes = [i64, i64, i32p, u64p, ctypes.c_int, ctypes.c_int]
            lib.oracle_dm4_vertex.argtypes = [i64, i64, i32p, u64p, ctypes.c_int, ctypes.c_int]
            lib.oracle_c5_rows.argtypes = [i64, i64, i32p, i64, ctypes.POINTER(ctypes.c_int64), u64p, ip,
                                           ctypes.c_uint64, ctypes.c_int]
            lib.oracle_pattern.argtypes = [ctypes.c_int, ip, ip, ip, ip]
            lib.oracle_automorphism_classes.argtypes = [ctypes.c_int, ip, ip]
            lib.oracle_classify.argtypes = [ctypes.c_int, ctypes.c_int, ip]
            _lib = lib
    return _lib


def _edges(edges) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    return e


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def orbits(n: int, edges, threads: int = 0) -> np.ndarray:
    """Induced orbit counts DIM(v, theta) for every vertex: uint64[n, 73] (ESU)."""
    lib = _load()
    e = _edges(edges)
    out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
    rc = lib.oracle_orbits_esu(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(out, ctypes.c_uint64), threads)
    if rc != 0:
        raise RuntimeError(f"oracle_orbits_esu failed: {rc}")
    return out


def orbit_rows(n: int, edges, roots, cap: int = 0, threads: int = 0):
    """Exact rows DIM(r, .) for the given roots by rooted ESU.

    ``cap`` bounds the work per root (connected sets visited + extension-set elements
    built).  Returns (rows uint64[len(roots), 73], status int[len(roots)]); status 0 =
    exact, 1 = work cap hit (row incomplete, must not be compared), <0 = error."""
    lib = _load()
    e = _edges(edges)
    r = np.ascontiguousarray(np.asarray(roots, dtype=np.int64))
    rows = np.zeros((r.shape[0], NUM_ORBITS), dtype=np.uint64)
    st = np.zeros(r.shape[0], dtype=np.intc)
    rc = lib.oracle_orbit_rows(n, e.shape[0], _ptr(e, ctypes.c_int32), r.shape[0], _ptr(r, ctypes.c_int64),
                               _ptr(rows, ctypes.c_uint64), _ptr(st, ctypes.c_int), cap, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_orbit_rows failed: {rc}")
    return rows, st


def orbits_bruteforce(n: int, edges) -> np.ndarray:
    """Induced counts by enumerating every k-subset (n <= 64; for pinning ESU)."""
    lib = _load()
    e = _edges(edges)
    out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
    if lib.oracle_orbits_bruteforce(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(out, ctypes.c_uint64)):
        raise RuntimeError("oracle_orbits_bruteforce failed")
    return out


def noninduced_bruteforce(n: int, edges) -> np.ndarray:
    """Non-induced DM(v, theta) by enumerating vertex subsets x edge subsets (tiny n)."""
    lib = _load()
    e = _edges(edges)
    out = np.zeros((n, NUM_ORBITS), dtype=np.uint64)
    if lib.oracle_noninduced_bruteforce(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(out, ctypes.c_uint64)):
        raise RuntimeError("oracle_noninduced_bruteforce failed")
    return out


def clique_totals(n: int, edges, threads: int = 0, kmax: int = 5):
    """(#triangles, #4-cliques, #5-cliques) by plain nested enumeration; cliques larger than
    ``kmax`` (3..5) are not counted and come back as None."""
    lib = _load()
    e = _edges(edges)
    c = np.zeros(3, dtype=np.uint64)
    if lib.oracle_clique_totals(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(c, ctypes.c_uint64), threads,
                                int(kmax)):
        raise RuntimeError("oracle_clique_totals failed")
    return int(c[0]), (int(c[1]) if kmax >= 4 else None), (int(c[2]) if kmax >= 5 else None)


def clique_totals_bits(n: int, edges, threads: int = 0, kmax: int = 5):
    """The same totals as ``clique_totals`` (same definition, same counting vertex), with
    the membership tests on a local adjacency bitmap of N>(a): fast enough for config 3's
    5-cliques and config 5's 4- and 5-cliques."""
    lib = _load()
    e = _edges(edges)
    c = np.zeros(3, dtype=np.uint64)
    if lib.oracle_clique_totals_bits(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(c, ctypes.c_uint64), threads,
                                     int(kmax)):
        raise RuntimeError("oracle_clique_totals_bits failed")
    return int(c[0]), (int(c[1]) if kmax >= 4 else None), (int(c[2]) if kmax >= 5 else None)



def clique_counts_vertex(n: int, edges, threads: int = 0, kmax: int = 5) -> np.ndarray:
    """uint64[n, 3]: the triangles / 4-cliques / 5-cliques containing each vertex (= columns
    3 / 14 / 72 of the orbit matrix, induced or not); columns beyond ``kmax`` stay 0."""
    lib = _load()
    e = _edges(edges)
    out = np.zeros((n, 3), dtype=np.uint64)
    if lib.oracle_clique_counts_vertex(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(out, ctypes.c_uint64),
                                       threads, int(kmax)):
        raise RuntimeError("oracle_clique_counts_vertex failed")
    return out



def dm4_vertex(n: int, edges, threads: int = 0, with_c4: bool = True, with_k4: bool = True) -> np.ndarray:
    """uint64[n, 15]: the NON-induced counts DM(v, theta_0..14) of the orbits with at most 4
    vertices on every vertex, by Lemma 4vertexorbit from plain definitions of its
    inputs; theta_14 = K4(v) from ``clique_counts_vertex``.  Columns skipped by the flags
    (theta_8 / theta_14) stay 0."""
    lib = _load()
    e = _edges(edges)
    out = np.zeros((n, 15), dtype=np.uint64)
    if lib.oracle_dm4_vertex(n, e.shape[0], _ptr(e, ctypes.c_int32), _ptr(out, ctypes.c_uint64), threads,
                             int(bool(with_c4))):
        raise RuntimeError("oracle_dm4_vertex failed")
    if with_k4:
        out[:, 14] = clique_counts_vertex(n, e, threads=threads, kmax=4)[:, 1]
    return out



def c5_rows(n: int, edges, roots, cap: int = 0, threads: int = 0):
    """(counts uint64[len(roots)], status int32[len(roots)]): the number of (non-induced)
    5-cycles through each root = DM(root, theta_34), from the definition; status 1 = abandoned
    after ``cap`` innermost steps."""
    lib = _load()
    e = _edges(edges)
    r = np.ascontiguousarray(np.asarray(roots, dtype=np.int64).reshape(-1))
    out = np.zeros(r.size, dtype=np.uint64)
    st = np.zeros(r.size, dtype=np.int32)
    if lib.oracle_c5_rows(n, e.shape[0], _ptr(e, ctypes.c_int32), r.size, _ptr(r, ctypes.c_int64),
                          _ptr(out, ctypes.c_uint64), _ptr(st, ctypes.c_int), int(cap), threads):
        raise RuntimeError("oracle_c5_rows failed")
    return out, st


def catalog():
    """List of 30 patterns: dicts with k, edges, orbit-per-vertex."""
    lib = _load()
    pats = []
    for p in range(30):
        k, ne = ctypes.c_int(), ctypes.c_int()
        edges = (ctypes.c_int * 20)()
        orb = (ctypes.c_int * 5)()
        lib.oracle_pattern(p, ctypes.byref(k), ctypes.byref(ne), edges, orb)
        pats.append({"k": k.value, "edges": [(edges[2 * i], edges[2 * i + 1]) for i in range(ne.value)],
                     "orb": [orb[i] for i in range(k.value)]})
    return pats


def automorphism_classes(p: int):
    lib = _load()
    cls = (ctypes.c_int * 5)()
    na = ctypes.c_int()
    lib.oracle_automorphism_classes(p, cls, ctypes.byref(na))
    k = catalog()[p]["k"]
    return [cls[i] for i in range(k)], na.value


def classify(k: int, mask: int):
    """Orbit per position for a connected mask over k positions, else None."""
    lib = _load()
    orb = (ctypes.c_int * 5)()
    if lib.oracle_classify(k, mask, orb) != 0:
        return None
    return [orb[i] for i in range(k)]
