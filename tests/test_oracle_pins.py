"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

* catalog vs the exhaustive enumeration of connected graphs on 2..5 vertices and the
  automorphism definition; textual anchors of Fig. 2 (P:129-146, P:377-379,
  P:613-664);
* ESU vs all-subsets brute force (>= 200 random graphs);
* the catalog vs the paper's printed equations (Lemma 4vertexorbit, Thm B.1
  P:1121-1350) through the non-induced brute force, plus each erratum's printed form
  failing (readings R6-R13);
* Fig. 11 (golden) vs the brute-force transform, with the R18 erratum at A[5][13];
* closed forms (K_n, C_n, K_{1,s}, K_{a,b}) and named fixtures (Petersen, K5, K6).
"""
import itertools
import os
import random
from math import comb

import numpy as np
import pytest

import graphgen
import oracle
from paper_equations import G, noninduced_equations, theta18_alt, theta27_alt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def C(x, k):
    return comb(x, k) if x >= k else 0


def load_matrix(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append([int(t) for t in line.split()])
    return np.array(rows, dtype=np.int64)


def rand_graph(rng, nmin, nmax, pmin=0.1, pmax=0.9):
    n = rng.randint(nmin, nmax)
    p = rng.uniform(pmin, pmax)
    e = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    return n, e


# ---------------------------------------------------------------- catalog ---
def test_catalog_orbits_are_automorphism_classes():
    cat = oracle.catalog()
    assert len(cat) == 30
    seen = []
    for p, P in enumerate(cat):
        cls, _ = oracle.automorphism_classes(p)
        k = P["k"]
        for a in range(k):
            for b in range(k):
                assert (cls[a] == cls[b]) == (P["orb"][a] == P["orb"][b]), (p, a, b)
        seen += sorted(set(P["orb"]))
    assert seen == list(range(73))  # 73 orbits, numbered in pattern order


def test_catalog_covers_every_connected_graph_exactly():
    """Exhaustive: connected labelled graphs on k=2..5 vertices fall into exactly
    1/2/6/21 isomorphism classes, one catalog pattern each."""
    cat = oracle.catalog()
    for k, expect in [(2, 1), (3, 2), (4, 6), (5, 21)]:
        npairs = k * (k - 1) // 2
        found = set()
        for mask in range(1 << npairs):
            # connectivity by BFS over the mask (independent of the oracle's test)
            adj = {i: set() for i in range(k)}
            bit = 0
            for j in range(1, k):
                for i in range(j):
                    if mask >> bit & 1:
                        adj[i].add(j)
                        adj[j].add(i)
                    bit += 1
            seen, stack = {0}, [0]
            while stack:
                x = stack.pop()
                for y in adj[x]:
                    if y not in seen:
                        seen.add(y)
                        stack.append(y)
            orb = oracle.classify(k, mask)
            assert (orb is not None) == (len(seen) == k), (k, mask)
            if orb is not None:
                found.add(min(orb))  # the smallest orbit id identifies the pattern
                # degrees per position must match the pattern's degree per orbit
        pats = [P for P in cat if P["k"] == k]
        assert len(found) == expect == len(pats)


def test_catalog_textual_anchors():
    cat = oracle.catalog()
    byid = {i: P for i, P in enumerate(cat)}
    # H15 = 5-cycle, H29 = 5-clique (one orbit each); H10 has four orbits
    assert len(byid[15]["edges"]) == 5 and set(byid[15]["orb"]) == {34}
    assert len(byid[29]["edges"]) == 10 and set(byid[29]["orb"]) == {72}
    assert len(set(byid[10]["orb"])) == 4
    # P:143-146 / P:1062 / P:1074: orbit 15 = end of the 4-path, 17 = its centre
    P9 = byid[9]
    deg = [sum(a in e for e in P9["edges"]) for a in range(5)]
    assert sorted(deg) == [1, 1, 2, 2, 2] and len(P9["edges"]) == 4
    assert {P9["orb"][a] for a in range(5) if deg[a] == 1} == {15}
    # H28 = K5 minus an edge, orbit 70 = the two degree-3 vertices
    P28 = byid[28]
    deg = [sum(a in e for e in P28["edges"]) for a in range(5)]
    assert {P28["orb"][a] for a in range(5) if deg[a] == 3} == {70}
    # P:613-664 (Fig. 4): H12 = triangle {1,2,3} + pendants 4~2, 5~3; orbit 26 = {2,3};
    # H' = diamond with chord 2-3, orbit 13 = {2,3}
    fig4 = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 4)]
    mask = 0
    for a, b in fig4:
        a, b = min(a, b), max(a, b)
        mask |= 1 << (b * (b - 1) // 2 + a)
    orb = oracle.classify(5, mask)
    assert orb[1] == orb[2] == 26
    hp = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)]
    mask = 0
    for a, b in hp:
        mask |= 1 << (b * (b - 1) // 2 + a)
    orb = oracle.classify(4, mask)
    assert orb[1] == orb[2] == 13


# ------------------------------------------------------------ enumeration ---
def test_esu_equals_all_subsets_bruteforce():
    rng = random.Random(2024)
    for _ in range(220):
        n, e = rand_graph(rng, 1, 12)
        a = oracle.orbits(n, e)
        b = oracle.orbits_bruteforce(n, e)
        assert np.array_equal(a, b), (n, e)


def test_rooted_rows_equal_full_rows():
    rng = random.Random(7)
    for _ in range(40):
        n, e = rand_graph(rng, 2, 14, 0.1, 0.6)
        full = oracle.orbits(n, e)
        rows, st = oracle.orbit_rows(n, e, list(range(n)))
        assert (st == 0).all()
        assert np.array_equal(rows, full)


def test_input_cleaning_and_isolated_ids():
    g = graphgen.add_noise(graphgen.erdos_renyi(30, 0.2, 3), seed=1)
    clean = graphgen.erdos_renyi(30, 0.2, 3)
    assert np.array_equal(oracle.orbits(g.n, g.edges), oracle.orbits(clean.n, clean.edges))
    # ids never mentioned get zero rows (reading R21: ids are kept)
    out = oracle.orbits(10, [(0, 1), (1, 2)])
    assert out[3:].sum() == 0 and out[0, 0] == 1


# ---------------------------------------------- paper's equations (Thm B.1) ---
def _small_graphs(seed, count):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        n, e = rand_graph(rng, 5, 9, 0.3, 0.85)
        out.append((n, e, oracle.noninduced_bruteforce(n, e)))
    return out


def test_paper_equations_match_noninduced_bruteforce():
    """Every printed equation (with the DESIGN.md readings) reproduces the brute-force
    DM on every vertex: pins the orbit numbering of all 73 orbits except 34 and 72,
    for which the paper prints no equation (those are pinned by closed forms)."""
    for n, e, B in _small_graphs(11, 45):
        DM = noninduced_equations(G(n, e))
        for u in range(n):
            for th in range(72):
                if DM[u][th] is not None:
                    assert DM[u][th] == int(B[u][th]), (th, u, n, e)
            assert theta18_alt(G(n, e), DM, u) == DM[u][18]
            assert theta27_alt(G(n, e), DM, u, 2) == DM[u][27]  # R8


@pytest.mark.parametrize("variant,orbits", [
    ("theta19", [19]), ("theta20_21", [20, 21]), ("theta40", [40]), ("D", [64, 68]),
    ("theta66", [66]), ("theta69", [69])])
def test_printed_errata_fail(variant, orbits):
    bad = {th: 0 for th in orbits}
    for n, e, B in _small_graphs(12, 25):
        DM = noninduced_equations(G(n, e), {variant: 1})
        for th in orbits:
            bad[th] += sum(DM[u][th] != int(B[u][th]) for u in range(n))
    assert all(v > 0 for v in bad.values()), bad


def test_theta27_printed_alternative_fails():
    bad = 0
    for n, e, B in _small_graphs(13, 15):
        g = G(n, e)
        DM = noninduced_equations(g)
        bad += sum(theta27_alt(g, DM, u, 1) != DM[u][27] for u in range(n))
    assert bad > 0


# ------------------------------------------------------- Fig. 11 / Fig. 12 ---
def _A_block(lo, hi):
    """A[i][j] = DM_{H(j)}(w_j, theta_i) from the non-induced brute force
    on each pattern graph H(j) at a vertex w_j of orbit j."""
    cat = oracle.catalog()
    size = hi - lo + 1
    A = np.zeros((size, size), dtype=np.int64)
    for P in cat:
        for j in sorted(set(P["orb"])):
            if not lo <= j <= hi:
                continue
            w = P["orb"].index(j)
            dm = oracle.noninduced_bruteforce(P["k"], P["edges"])
            A[:, j - lo] = dm[w, lo:hi + 1].astype(np.int64)
    return A


def test_fig11_transform_matrix():
    A = _A_block(4, 14)
    printed = load_matrix("fig11_A.txt")
    diff = np.argwhere(A != printed)
    # the only disagreement is row theta5, column theta13 (R18: printed 2, true 4)
    assert [tuple(x) for x in diff] == [(5 - 4, 13 - 4)]
    assert A[1, 9] == 4 and printed[1, 9] == 2


def test_fig12_is_inverse_of_printed_fig11():
    A = load_matrix("fig11_A.txt")
    Ai = load_matrix("fig12_Ainv.txt")
    assert np.array_equal(A @ Ai, np.eye(11, dtype=np.int64))
    # and the true inverse differs from the printed one only in row theta5 (R18)
    At = _A_block(4, 14)
    Ati = np.rint(np.linalg.inv(At)).astype(np.int64)
    assert np.array_equal(At @ Ati, np.eye(11, dtype=np.int64))
    rows = sorted(set(int(r) for r, _ in np.argwhere(Ati != Ai)))
    assert rows == [1]


def test_induced_equals_inverse_transform_of_noninduced():
    """DIM = A^-1 DM per vertex for the full 73 orbits, A built blockwise."""
    blocks = [(0, 0), (1, 3), (4, 14), (15, 72)]
    mats = [(lo, hi, _A_block(lo, hi)) for lo, hi in blocks]
    rng = random.Random(5)
    for _ in range(12):
        n, e = rand_graph(rng, 5, 9, 0.3, 0.8)
        dm = oracle.noninduced_bruteforce(n, e).astype(object)
        dim = oracle.orbits(n, e).astype(object)
        for lo, hi, A in mats:
            lhs = A.astype(object).dot(dim[:, lo:hi + 1].T).T
            assert (lhs == dm[:, lo:hi + 1]).all()


# ------------------------------------------------------------ closed forms ---
def _row(**kw):
    r = np.zeros(73, dtype=object)
    for k, v in kw.items():
        r[int(k[1:])] = v
    return r


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 8, 9])
def test_closed_form_complete_graph(n):
    g = graphgen.complete(n)
    out = oracle.orbits(g.n, g.edges)
    exp = _row(t0=n - 1, t3=C(n - 1, 2), t14=C(n - 1, 3), t72=C(n - 1, 4))
    for v in range(n):
        assert list(out[v].astype(object)) == list(exp)


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 11])
def test_closed_form_cycle(n):
    g = graphgen.cycle(n)
    out = oracle.orbits(g.n, g.edges)
    if n == 3:
        exp = _row(t0=2, t3=1)
    elif n == 4:
        exp = _row(t0=2, t1=2, t2=1, t8=1)
    elif n == 5:
        exp = _row(t0=2, t1=2, t2=1, t4=2, t5=2, t34=1)
    else:
        exp = _row(t0=2, t1=2, t2=1, t4=2, t5=2, t15=2, t16=2, t17=1)
    for v in range(n):
        assert list(out[v].astype(object)) == list(exp), v


@pytest.mark.parametrize("s", [1, 2, 3, 4, 7, 12])
def test_closed_form_star(s):
    g = graphgen.star(s)
    out = oracle.orbits(g.n, g.edges)
    assert list(out[0].astype(object)) == list(_row(t0=s, t2=C(s, 2), t7=C(s, 3), t23=C(s, 4)))
    for v in range(1, s + 1):
        assert list(out[v].astype(object)) == list(_row(t0=1, t1=s - 1, t6=C(s - 1, 2), t22=C(s - 1, 3)))


@pytest.mark.parametrize("a,b", [(1, 1), (2, 2), (2, 3), (3, 4), (4, 6), (5, 5)])
def test_closed_form_complete_bipartite(a, b):
    g = graphgen.complete_bipartite(a, b)
    out = oracle.orbits(g.n, g.edges)

    def side(a, b):  # a vertex on the a-side (degree b)
        return _row(t0=b, t1=(a - 1) * b, t2=C(b, 2), t6=b * C(a - 1, 2), t7=C(b, 3),
                    t8=(a - 1) * C(b, 2), t22=b * C(a - 1, 3), t23=C(b, 4),
                    t49=C(a - 1, 2) * C(b, 2), t50=(a - 1) * C(b, 3))
    for v in range(a):
        assert list(out[v].astype(object)) == list(side(a, b))
    for v in range(a, a + b):
        assert list(out[v].astype(object)) == list(side(b, a))


def test_named_fixtures():
    p = graphgen.petersen()
    out = oracle.orbits(p.n, p.edges)
    assert (out[:, 34] == 6).all()  # 12 five-cycles x 5 / 10 vertices, all induced
    dm = oracle.noninduced_bruteforce(p.n, p.edges)
    assert (dm[:, 34] == 6).all()
    k5 = graphgen.complete(5)
    dm = oracle.noninduced_bruteforce(5, k5.edges)
    assert (dm[:, 34] == 12).all()   # Hamiltonian cycles of K5 through a vertex: 4!/2
    assert (oracle.orbits(5, k5.edges)[:, 34] == 0).all()
    k6 = graphgen.complete(6)
    assert (oracle.orbits(6, k6.edges)[:, 72] == 5).all()


def test_whole_matrix_invariants():
    g = graphgen.config(1)
    out = oracle.orbits(g.n, g.edges).astype(object)
    e = np.unique(np.sort(g.edges, axis=1), axis=0)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=g.n)
    assert list(out[:, 0]) == list(deg)
    t3, t4, t5 = oracle.clique_totals(g.n, g.edges)
    assert out[:, 3].sum() == 3 * t3 and out[:, 14].sum() == 4 * t4 and out[:, 72].sum() == 5 * t5
    # per-pattern consistency: sz(b) * sum DIM(a) == sz(a) * sum DIM(b) for orbits of one pattern
    cat = oracle.catalog()
    for P in cat:
        orbs = sorted(set(P["orb"]))
        sz = {o: P["orb"].count(o) for o in orbs}
        for a_, b_ in itertools.combinations(orbs, 2):
            assert sz[b_] * out[:, a_].sum() == sz[a_] * out[:, b_].sum()


# ------------------------------------------------------------ clique totals ---
# oracle.clique_totals feeds the whole-matrix invariants Sigma DIM3 = 3 #K3, Sigma DIM14 =
# 4 #K4, Sigma DIM72 = 5 #K5 (cliques: P:702) on configs the ESU cannot reach.
def _cliques_by_subsets(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in edges:
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    out = []
    for k in (3, 4, 5):
        out.append(sum(1 for S in itertools.combinations(range(n), k)
                       if all(y in adj[x] for x, y in itertools.combinations(S, 2))))
    return tuple(out)


def test_clique_totals_vs_all_subsets():
    rng = random.Random(71)
    for _ in range(60):
        n, e = rand_graph(rng, 3, 14, 0.2, 0.95)
        assert oracle.clique_totals(n, e) == _cliques_by_subsets(n, e), (n, e)


def test_clique_totals_vs_esu_on_dense_graphs():
    """the ESU's column sums (pinned to all-subsets brute force above) divided by the orbit
    multiplicity: Sigma DIM3 / 3, Sigma DIM14 / 4, Sigma DIM72 / 5"""
    rng = random.Random(72)
    for t in range(24):
        n, e = rand_graph(rng, 15, 32, 0.45, 0.92)
        dim = oracle.orbits(n, e).astype(object)
        s3, s14, s72 = dim[:, 3].sum(), dim[:, 14].sum(), dim[:, 72].sum()
        assert s3 % 3 == 0 and s14 % 4 == 0 and s72 % 5 == 0
        assert oracle.clique_totals(n, e) == (s3 // 3, s14 // 4, s72 // 5), (t, n, len(e))


@pytest.mark.parametrize("n", [3, 4, 5, 6, 9, 17, 40])
def test_clique_totals_complete_graph(n):
    assert oracle.clique_totals(n, graphgen.complete(n).edges) == (C(n, 3), C(n, 4), C(n, 5))


def test_clique_totals_complete_multipartite():
    """K_{p1,...,pr}: #K_k = e_k(p1..pr) (elementary symmetric polynomial: one vertex from each of
    k distinct parts); equal degrees inside a part exercise the order's id tie-break"""
    for parts in [(2, 3, 4), (1, 1, 5, 2), (3, 3, 3, 3, 3), (4, 1, 2, 6, 3)]:
        offs = np.cumsum((0,) + parts)
        e = [(a, b) for i in range(len(parts)) for j in range(i + 1, len(parts))
             for a in range(offs[i], offs[i + 1]) for b in range(offs[j], offs[j + 1])]
        ek = [sum(int(np.prod(c)) for c in itertools.combinations(parts, k)) for k in (3, 4, 5)]
        assert oracle.clique_totals(int(offs[-1]), e) == tuple(ek), parts


def test_clique_totals_kmax():
    rng = random.Random(73)
    for _ in range(10):
        n, e = rand_graph(rng, 8, 14, 0.5, 0.95)
        t3, t4, t5 = _cliques_by_subsets(n, e)
        assert oracle.clique_totals(n, e, kmax=3) == (t3, None, None)
        assert oracle.clique_totals(n, e, kmax=4) == (t3, t4, None)


# oracle.clique_totals_bits: the same totals with the membership tests on a bitmap of N>(a)
# (what the golden totals of configs 3 and 5 need); pinned by the same brute force and
# closed forms, with lists longer than one 64-bit word
def test_clique_totals_bits_vs_all_subsets_and_plain():
    rng = random.Random(75)
    for _ in range(60):
        n, e = rand_graph(rng, 3, 14, 0.2, 0.95)
        assert oracle.clique_totals_bits(n, e) == _cliques_by_subsets(n, e), (n, e)
    for t in range(6):  # rows of 2-4 words: N>(a) up to ~200 vertices
        g = graphgen.erdos_renyi(int(rng.randint(90, 220)), rng.uniform(0.3, 0.6), 700 + t)
        assert oracle.clique_totals_bits(g.n, g.edges) == oracle.clique_totals(g.n, g.edges), g.name


@pytest.mark.parametrize("n", [3, 5, 17, 64, 65, 66, 130])
def test_clique_totals_bits_complete_graph(n):
    assert oracle.clique_totals_bits(n, graphgen.complete(n).edges) == (C(n, 3), C(n, 4), C(n, 5))


def test_clique_totals_bits_complete_multipartite_and_kmax():
    for parts in [(2, 3, 4), (1, 1, 5, 2), (3, 3, 3, 3, 3), (4, 1, 2, 6, 3), (20, 30, 25, 1, 9)]:
        offs = np.cumsum((0,) + parts)
        e = [(a, b) for i in range(len(parts)) for j in range(i + 1, len(parts))
             for a in range(offs[i], offs[i + 1]) for b in range(offs[j], offs[j + 1])]
        ek = [sum(int(np.prod(c)) for c in itertools.combinations(parts, k)) for k in (3, 4, 5)]
        assert oracle.clique_totals_bits(int(offs[-1]), e) == tuple(ek), parts
        assert oracle.clique_totals_bits(int(offs[-1]), e, kmax=3) == (ek[0], None, None)
        assert oracle.clique_totals_bits(int(offs[-1]), e, kmax=4) == (ek[0], ek[1], None)


# oracle.clique_counts_vertex: T(v), K4(v), K5(v) on every vertex = columns 3 / 14 / 72 of the
# orbit matrix (a clique is an induced copy of itself), the
# per-vertex check the GPU tests apply to the hub rows of the full configs
def _cliques_per_vertex_by_subsets(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in edges:
        if a != b:
            adj[a].add(b)
            adj[b].add(a)
    out = np.zeros((n, 3), dtype=np.uint64)
    for c, k in enumerate((3, 4, 5)):
        for S in itertools.combinations(range(n), k):
            if all(y in adj[x] for x, y in itertools.combinations(S, 2)):
                for v in S:
                    out[v, c] += np.uint64(1)
    return out


def test_clique_counts_vertex_vs_all_subsets():
    rng = random.Random(76)
    for _ in range(60):
        n, e = rand_graph(rng, 3, 14, 0.2, 0.95)
        assert (oracle.clique_counts_vertex(n, e) == _cliques_per_vertex_by_subsets(n, e)).all(), (n, e)


def test_clique_counts_vertex_vs_esu_columns():
    """columns 3 / 14 / 72 of the ESU matrix (pinned to brute force above) on dense graphs and
    on graphs whose N>(a) bitmaps have rows of several words; sums = k * totals"""
    rng = random.Random(77)
    graphs = [rand_graph(rng, 15, 32, 0.45, 0.92) for _ in range(20)]
    graphs += [(g.n, g.edges) for g in (graphgen.erdos_renyi(100, 0.45, 801), graphgen.erdos_renyi(70, 0.8, 802),
                                        graphgen.config(1))]
    for n, e in graphs:
        dim = oracle.orbits(n, e)
        got = oracle.clique_counts_vertex(n, e)
        assert (got[:, 0] == dim[:, 3]).all() and (got[:, 1] == dim[:, 14]).all() and (got[:, 2] == dim[:, 72]).all()
        t3, t4, t5 = oracle.clique_totals(n, e)
        assert [int(x) for x in got.astype(object).sum(axis=0)] == [3 * t3, 4 * t4, 5 * t5]


@pytest.mark.parametrize("n", [3, 5, 17, 64, 65, 66, 130])
def test_clique_counts_vertex_complete_graph_and_kmax(n):
    e = graphgen.complete(n).edges
    exp = np.array([C(n - 1, 2), C(n - 1, 3), C(n - 1, 4)], dtype=np.uint64)  # P: every vertex of K_n
    assert (oracle.clique_counts_vertex(n, e) == exp).all()
    got = oracle.clique_counts_vertex(n, e, kmax=4)
    assert (got[:, :2] == exp[:2]).all() and (got[:, 2] == 0).all()
    got = oracle.clique_counts_vertex(n, e, kmax=3)
    assert (got[:, 0] == exp[0]).all() and (got[:, 1:] == 0).all()


def test_clique_counts_vertex_star_of_cliques():
    """a hub joined to every vertex of several disjoint cliques K_s: the hub is in sum C(s,k-1)
    k-cliques, a clique vertex in C(s-1,k-1) + C(s-1,k-2) (asymmetric roles, so a credit given
    to the wrong member shows)"""
    sizes = (3, 4, 6, 9)
    e, off = [], 1
    for s in sizes:
        e += [(off + i, off + j) for i in range(s) for j in range(i + 1, s)] + [(0, off + i) for i in range(s)]
        off += s
    got = oracle.clique_counts_vertex(off, e)
    assert got[0].tolist() == [sum(C(s, k - 1) for s in sizes) for k in (3, 4, 5)]
    off = 1
    for s in sizes:
        for i in range(s):
            assert got[off + i].tolist() == [C(s - 1, k - 1) + C(s - 1, k - 2) for k in (3, 4, 5)], (s, i)
        off += s


# oracle.dm4_vertex: Lemma 4vertexorbit on every vertex from plain definitions of
# d, T(u,v), T(u), C4(u) -- the non-induced columns 0..14 the GPU tests check on the hub rows
def test_dm4_vertex_vs_noninduced_bruteforce():
    rng = random.Random(78)
    for _ in range(80):
        n, e = rand_graph(rng, 2, 10, 0.15, 0.95)
        assert (oracle.dm4_vertex(n, e) == oracle.noninduced_bruteforce(n, e)[:, :15]).all(), (n, e)


def test_dm4_vertex_is_transform_of_esu_on_larger_graphs():
    """DM = A . DIM restricted to the 4-vertex orbits, A = the brute-force
    transform pinned to Fig. 11: on graphs past brute-force size the lemma's columns must equal
    the ESU's induced counts pushed through A"""
    mats = [(lo, hi, _A_block(lo, hi).astype(object)) for lo, hi in [(0, 0), (1, 3), (4, 14)]]
    for g in (graphgen.erdos_renyi(60, 0.3, 811), graphgen.erdos_renyi(200, 0.06, 812), graphgen.config(1)):
        dim = oracle.orbits(g.n, g.edges).astype(object)
        got = oracle.dm4_vertex(g.n, g.edges).astype(object)
        for lo, hi, A in mats:
            assert (A.dot(dim[:, lo:hi + 1].T).T == got[:, lo:hi + 1]).all(), (g.name, lo)


@pytest.mark.parametrize("n", [4, 5, 9, 40])
def test_dm4_vertex_complete_graph(n):
    d = n - 1
    exp = [d, d * (d - 1), C(d, 2), C(d, 2), d * (d - 1) * (d - 2), d * (d - 1) * (d - 2), d * C(d - 1, 2), C(d, 3),
           3 * C(d, 3), d * (d - 1) * (d - 2) // 2, d * (d - 1) * (d - 2), C(d, 2) * (d - 2), C(d, 2) * (n - 3),
           d * C(n - 2, 2), C(d, 3)]
    got = oracle.dm4_vertex(n, graphgen.complete(n).edges)
    assert (got == np.array(exp, dtype=np.uint64)).all(), (got[0].tolist(), exp)


def test_dm4_vertex_complete_bipartite_and_flags():
    a, b = 9, 700
    e = [(i, a + j) for i in range(a) for j in range(b)]
    got = oracle.dm4_vertex(a + b, e)
    # no triangles; a 4-cycle through v = another vertex of its side and two of the other side
    assert (got[:, [3, 9, 10, 11, 12, 13, 14]] == 0).all()
    assert (got[:a, 8] == (a - 1) * C(b, 2)).all() and (got[a:, 8] == (b - 1) * C(a, 2)).all()
    assert (got[:a, 0] == b).all() and (got[:a, 1] == b * (a - 1)).all() and (got[:a, 7] == C(b, 3)).all()
    assert (got[:a, 4] == b * (a - 1) * (b - 1)).all() and (got[:a, 5] == b * (a - 1) * (b - 1)).all()
    off = oracle.dm4_vertex(a + b, e, with_c4=False, with_k4=False)
    assert (off[:, 8] == 0).all() and (np.delete(off, 8, axis=1) == np.delete(got, 8, axis=1)).all()


# oracle.c5_rows: the 5-cycles through chosen vertices (non-induced theta34) from the
# definition -- what the GPU tests compare the hub rows of configs 2 and 4 with
def test_c5_rows_vs_noninduced_bruteforce_and_closed_forms():
    rng = random.Random(79)
    for _ in range(60):
        n, e = rand_graph(rng, 3, 10, 0.2, 0.95)
        got, st = oracle.c5_rows(n, e, range(n))
        assert (st == 0).all() and (got == oracle.noninduced_bruteforce(n, e)[:, 34]).all(), (n, e)
    for n in (5, 6, 9, 30):  # K_n: choose the 4 others, 4!/2 cyclic orders
        got, _ = oracle.c5_rows(n, graphgen.complete(n).edges, range(n))
        assert (got == C(n - 1, 4) * 12).all()
    got, _ = oracle.c5_rows(10, graphgen.petersen().edges, range(10))
    assert (got == 6).all()  # P: each vertex of the Petersen graph is in 6 five-cycles (theta34 = 6)
    got, _ = oracle.c5_rows(12, graphgen.cycle(12).edges, range(12))
    assert (got == 0).all()
    got, _ = oracle.c5_rows(5, graphgen.cycle(5).edges, range(5))
    assert (got == 1).all()


def test_c5_rows_cap_and_larger_graph():
    """past brute-force size: non-induced theta34 = (A . DIM)[34] of the ESU matrix, A's row
    from the brute-force transform on the 5-vertex patterns; a tiny cap abandons the root"""
    A = _A_block(15, 72).astype(object)
    for g in (graphgen.erdos_renyi(45, 0.3, 821), graphgen.config(1)):
        dim = oracle.orbits(g.n, g.edges)[:, 15:].astype(object)
        exp = dim.dot(A[34 - 15])
        got, st = oracle.c5_rows(g.n, g.edges, range(g.n))
        assert (st == 0).all() and (got.astype(object) == exp).all(), g.name
    g = graphgen.complete(30)
    got, st = oracle.c5_rows(g.n, g.edges, [0, 1], cap=10)
    assert (st == 1).all() and (got == 0).all()


def test_degree_forms_vs_noninduced_bruteforce():
    """the degree-only closed forms the GPU tests apply to every vertex of configs 2-4
    (tests/degree_forms.py) equal the non-induced brute force on random graphs"""
    from degree_forms import COLUMNS, degree_forms
    rng = random.Random(74)
    for _ in range(40):
        n, e = rand_graph(rng, 2, 10, 0.15, 0.95)
        dm = oracle.noninduced_bruteforce(n, e)
        f = degree_forms(n, e)
        for c in COLUMNS:
            assert (dm[:, c] == f[c]).all(), (c, n, e)
    # wrap-around: C(s, 4) >= 2^64 for the centre of K_{1,s}, s = 145,100 (R20)
    s = 145_100
    f = degree_forms(s + 1, graphgen.star(s).edges)
    assert comb(s, 4) >= 1 << 64 and int(f[23][0]) == comb(s, 4) % (1 << 64)
    assert int(f[22][1]) == comb(s - 1, 3) and int(f[6][1]) == comb(s - 1, 2) and int(f[1][1]) == s - 1
