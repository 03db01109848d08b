"""Parity of the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Bar: bit-exact equality of the uint64 n x 73 matrix (integer work).
Sizes span many tiles / CTAs and ragged tails; the full BASELINE configs are covered by
sampled rows (rooted oracle) + whole-matrix invariants, the tiled graph and the closed
forms give full-matrix parity at millions of edges and at wrap-around (>= 2^64) counts.
"""
import hashlib
import json
import os
from math import comb

import numpy as np
import pytest

import graphgen
import oracle
from degree_forms import COLUMNS as DEGREE_FORM_COLUMNS, degree_forms

GOLDEN_CLIQUES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "clique_totals.json")))

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_10616_b200 as p
    p.lib()
    return p


def _rand(rng, nmin, nmax, pmin, pmax, seed):
    n = int(rng.integers(nmin, nmax + 1))
    p = float(rng.uniform(pmin, pmax))
    return graphgen.erdos_renyi(n, p, seed)


def _unique_edges(n, edges):
    """the distinct unordered pairs of an edge list as sorted (lo, hi) rows (what
    np.unique(np.sort(edges, axis=1), axis=0) returns, by one key sort: np.unique with
    axis=0 takes minutes on config 5's 67M pairs)"""
    e = np.sort(np.asarray(edges, dtype=np.int64).reshape(-1, 2), axis=1)
    key = np.sort(e[:, 0] * max(n, 1) + e[:, 1])
    if key.size:
        key = key[np.concatenate([[True], key[1:] != key[:-1]])]
    return np.stack([key // max(n, 1), key % max(n, 1)], axis=1)


def _assert_equal(got, exp, what=""):
    got = np.asarray(got)
    if got.dtype != np.uint64:
        got = got.view(np.uint64)
    bad = np.argwhere(got != exp)
    assert bad.size == 0, f"{what}: {len(bad)} mismatches, first (vertex, orbit) {bad[:8].tolist()}"


# ----------------------------------------------------------------- small graphs ---
def test_small_random_graphs_induced(pkg):
    rng = np.random.default_rng(11)
    for t in range(240):
        g = _rand(rng, 1, 13, 0.05, 0.95, 5000 + t)
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name)


def test_small_random_graphs_noninduced(pkg):
    rng = np.random.default_rng(12)
    for t in range(80):
        g = _rand(rng, 2, 9, 0.2, 0.95, 7000 + t)
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges, induced=False),
                      oracle.noninduced_bruteforce(g.n, g.edges), g.name)


def test_sparse_medium_graphs(pkg):
    """ragged sizes spanning several CTAs/warps (n up to 3000, sparse)"""
    rng = np.random.default_rng(13)
    for t in range(6):
        n = int(rng.integers(200, 3000))
        g = graphgen.erdos_renyi(n, 6.0 / n, 9000 + t)
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name)


def test_dense_medium_graphs(pkg):
    """dense graphs: large out-degree bins of the clique kernel, many 5-cliques"""
    for n, p, s in [(40, 0.5, 1), (60, 0.35, 2), (34, 0.9, 3)]:
        g = graphgen.erdos_renyi(n, p, s)
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name)


def test_config1_full_matrix(pkg):
    g = graphgen.config(1)
    _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), "config 1")


# --------------------------------------------------------------- degenerate cases ---
def test_degenerate_inputs(pkg):
    assert pkg.evoke_orbits_edges(0, np.zeros((0, 2), np.int32)).shape == (0, 73)
    out = pkg.evoke_orbits_edges(7, np.zeros((0, 2), np.int32))
    assert (out == 0).all()
    out = pkg.evoke_orbits_edges(5, np.array([[1, 1], [3, 3]], np.int32))  # only self-loops
    assert (out == 0).all()
    out = pkg.evoke_orbits_edges(6, np.array([[4, 2]], np.int32))          # one edge, isolated ids
    exp = np.zeros((6, 73), np.uint64)
    exp[4, 0] = exp[2, 0] = 1
    _assert_equal(out, exp, "single edge")
    for g in [graphgen.complete(2), graphgen.complete(3), graphgen.complete(5), graphgen.complete(6),
              graphgen.path(5), graphgen.cycle(5), graphgen.star(4), graphgen.petersen()]:
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name)


def test_input_cleaning(pkg):
    g = graphgen.erdos_renyi(300, 0.03, 21)
    noisy = graphgen.add_noise(g, 5, frac=0.5)
    _assert_equal(pkg.evoke_orbits_edges(noisy.n, noisy.edges), oracle.orbits(g.n, g.edges), "noisy")


def test_invalid_vertex_id(pkg):
    with pytest.raises(pkg.EvokeError) as ei:
        pkg.evoke_orbits_edges(3, np.array([[0, 1], [1, 3]], np.int32))
    assert ei.value.code == pkg.EVOKE_EINVAL


# ---------------------------------------------------------------- API variants ---
def test_csr_and_device_pointer_paths(pkg):
    import torch
    g = graphgen.erdos_renyi(500, 0.02, 31)
    ref = oracle.orbits(g.n, g.edges)
    # CSR (directed, unsorted rows) on the host
    e = g.edges.astype(np.int64)
    order = np.argsort(e[:, 0], kind="stable")
    rowptr = np.zeros(g.n + 1, np.int64)
    np.add.at(rowptr, e[:, 0] + 1, 1)
    rowptr = np.cumsum(rowptr)
    col = e[order, 1].astype(np.int32)
    _assert_equal(pkg.evoke_orbits_csr(g.n, rowptr, col), ref, "csr host")
    dev = torch.device("cuda:0")
    out = pkg.evoke_orbits_edges(g.n, torch.from_numpy(g.edges).to(dev))
    torch.cuda.synchronize()
    _assert_equal(out.cpu().numpy(), ref, "edges device")
    out = pkg.evoke_orbits_csr(g.n, torch.from_numpy(rowptr).to(dev), torch.from_numpy(col).to(dev))
    torch.cuda.synchronize()
    _assert_equal(out.cpu().numpy(), ref, "csr device")


def test_multi_device_call(pkg):
    """evoke_orbits_edges_multi (the C ABI's several-GPUs-in-one-process call): the shards on
    a device list -- here the one GPU named 2, 3 and 4 times, so the decomposition, the
    per-device workers, the sum modulo 2^64 and the staged result all run; the peer-memory
    read of another GPU's partial needs a second GPU -- equal the oracle / the one-call
    matrix bit for bit; shard arguments compose; a failing shard leaves out untouched"""
    import torch
    rng = np.random.default_rng(11)
    for t in range(20):
        g = graphgen.erdos_renyi(int(rng.integers(5, 14)), float(rng.uniform(0.2, 0.8)), 4000 + t)
        ref = oracle.orbits(g.n, g.edges)
        _assert_equal(pkg.evoke_orbits_edges_multi(g.n, g.edges, [0, 0]), ref, g.name + " multi2")
        _assert_equal(pkg.evoke_orbits_edges_multi(g.n, g.edges, [0, 0, 0]), ref, g.name + " multi3")
    g = graphgen.config(2)
    full = pkg.evoke_orbits_edges(g.n, g.edges)
    _assert_equal(pkg.evoke_orbits_edges_multi(g.n, g.edges, [0, 0, 0, 0]), full, "config2 multi4")
    ed = torch.from_numpy(g.edges).to("cuda:0")
    parts = [pkg.evoke_orbits_edges_multi(g.n, ed, [0, 0], shard_index=r, num_shards=2) for r in range(2)]
    tot = (parts[0] + parts[1]).cpu().numpy()  # int64 addition wraps like uint64
    _assert_equal(tot, full, "config2 2 x 2 shards")
    out = np.full((4, 73), 7, np.uint64)
    with pytest.raises(pkg.EvokeError) as ei:
        pkg.evoke_orbits_edges_multi(4, np.array([[0, 1], [1, 7]], np.int32), [0, 0], out=out)
    assert ei.value.code == pkg.EVOKE_EINVAL and (out == 7).all()
    with pytest.raises(pkg.EvokeError):
        pkg.evoke_orbits_edges_multi(4, np.array([[0, 1]], np.int32), [0, 99])


def test_sharded_partials_sum_to_full(pkg):
    """multi-GPU decomposition on one device: partials of every shard sum (mod 2^64) to
    the full matrix bit for bit"""
    for g in [graphgen.erdos_renyi(200, 0.08, 41), graphgen.config(2)]:
        full = pkg.evoke_orbits_edges(g.n, g.edges)
        for ns in (2, 3):
            acc = np.zeros_like(full)
            for si in range(ns):
                acc += pkg.evoke_orbits_edges(g.n, g.edges, shard_index=si, num_shards=ns)
            _assert_equal(acc, full, f"{g.name} shards={ns}")


def test_deterministic(pkg):
    """Repeated calls are bit-identical (exact integer sums; any schedule).  Several repeats:
    a work-list or counter race shows up as an occasional difference, not on every call."""
    g = graphgen.config(2)
    a = pkg.evoke_orbits_edges(g.n, g.edges)
    for r in range(8):
        b = pkg.evoke_orbits_edges(g.n, g.edges, serial=(r % 4 == 3))
        _assert_equal(b, a, f"repeat {r}")


# ---------------------------------------------------------- closed forms at scale ---
def _row(**kw):
    r = np.zeros(73, dtype=object)
    for k, v in kw.items():
        r[int(k[1:])] = v % (1 << 64)
    return r


def _rows_equal(got_row, exp_row):
    return [int(x) for x in got_row] == [int(x) for x in exp_row]


def test_closed_form_star_wraps_modulo_2_64(pkg):
    """K_{1,s} with s >= 145,057: C(s,4) >= 2^64, the hub row must be exact mod 2^64 (R20)"""
    s = 145_100
    assert comb(s, 4) >= 1 << 64
    g = graphgen.star(s)
    out = pkg.evoke_orbits_edges(g.n, g.edges)
    assert _rows_equal(out[0], _row(t0=s, t2=comb(s, 2), t7=comb(s, 3), t23=comb(s, 4)))
    leaf = _row(t0=1, t1=s - 1, t6=comb(s - 1, 2), t22=comb(s - 1, 3))
    for v in (1, 2, s // 2, s):
        assert _rows_equal(out[v], leaf)


def test_closed_form_complete_and_cycle_and_bipartite(pkg):
    n = 48
    out = pkg.evoke_orbits_edges(n, graphgen.complete(n).edges)
    exp = _row(t0=n - 1, t3=comb(n - 1, 2), t14=comb(n - 1, 3), t72=comb(n - 1, 4))
    assert all(_rows_equal(out[v], exp) for v in range(n))
    n = 100_003
    out = pkg.evoke_orbits_edges(n, graphgen.cycle(n).edges)
    exp = _row(t0=2, t1=2, t2=1, t4=2, t5=2, t15=2, t16=2, t17=1)
    assert (out == np.array([int(x) for x in exp], dtype=np.uint64)).all()
    a, b = 9, 700
    out = pkg.evoke_orbits_edges(a + b, graphgen.complete_bipartite(a, b).edges)

    def side(a, b):
        return _row(t0=b, t1=(a - 1) * b, t2=comb(b, 2), t6=b * comb(a - 1, 2), t7=comb(b, 3),
                    t8=(a - 1) * comb(b, 2), t22=b * comb(a - 1, 3), t23=comb(b, 4),
                    t49=comb(a - 1, 2) * comb(b, 2), t50=(a - 1) * comb(b, 3))
    assert all(_rows_equal(out[v], side(a, b)) for v in range(a))
    assert all(_rows_equal(out[v], side(b, a)) for v in range(a, a + b))


# ------------------------------------------------------ full-matrix parity at scale ---
def test_tiled_graph_full_matrix(pkg):
    """~1.2M-edge disjoint union of seeded G(40, 0.15) tiles: the oracle solves only the
    64 distinct tiles; the CUDA result must equal the tiled oracle matrix everywhere"""
    tiles = [graphgen.erdos_renyi(40, 0.15, 77 * 1000 + i) for i in range(64)]
    refs = [oracle.orbits(t.n, t.edges) for t in tiles]
    rng = np.random.default_rng(77)
    pick = rng.integers(0, 64, size=10_000)
    g, offs = graphgen.disjoint_union([tiles[i] for i in pick], "tiled")
    exp = np.concatenate([refs[i] for i in pick], axis=0)
    assert g.edges.shape[0] > 1_000_000
    _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), exp, "tiled")


# ----------------------------------------------- BASELINE configs: rows + invariants ---
def _golden_cliques(cfg, g):
    """(#K3, #K4 or None, #K5 or None) of config `cfg` from tests/golden/clique_totals.json
    (written by tools/make_golden_cliques.py with the oracle), after checking that the
    generated edge list is the one the file was written for"""
    ent = GOLDEN_CLIQUES[str(cfg)]
    assert hashlib.sha256(g.edges.tobytes()).hexdigest() == ent["edges_sha256"], "generator changed"
    return ent["triangles"], ent["k4"], ent["k5"]


def _invariants(g, out, check_cliques=True, cliques=None):
    e = _unique_edges(g.n, g.edges)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=g.n).astype(np.uint64)
    assert (out[:, 0] == deg).all(), "orbit 0 = degree"
    cat = oracle.catalog()
    colsum = [int(x) for x in out.sum(axis=0, dtype=np.uint64)]  # mod 2^64
    for P in cat:
        orbs = sorted(set(P["orb"]))
        sz = {o: P["orb"].count(o) for o in orbs}
        for a in orbs:
            for b in orbs:
                assert (sz[b] * colsum[a] - sz[a] * colsum[b]) % (1 << 64) == 0, (a, b)
    if check_cliques:
        t3, t4, t5 = cliques if cliques is not None else oracle.clique_totals(g.n, g.edges, threads=0)
        assert colsum[3] == (3 * t3) % (1 << 64)
        if t4 is not None:
            assert colsum[14] == (4 * t4) % (1 << 64)
        if t5 is not None:
            assert colsum[72] == (5 * t5) % (1 << 64)


def _cheap_roots(g, k, seed, pool=4000):
    """roots whose rooted enumeration is small: lowest 3-hop path count sum_w s2(w),
    s2(w) = sum_{x in N(w)} d(x), plus a few uniformly random roots"""
    e = _unique_edges(g.n, g.edges)
    e = e[e[:, 0] != e[:, 1]]
    a = np.concatenate([e[:, 0], e[:, 1]])
    b = np.concatenate([e[:, 1], e[:, 0]])
    deg = np.bincount(a, minlength=g.n).astype(np.float64)
    s2 = np.bincount(a, weights=deg[b], minlength=g.n)
    s3 = np.bincount(a, weights=s2[b], minlength=g.n)
    cand = np.flatnonzero(deg > 0)
    cand = cand[np.argsort(s3[cand], kind="stable")][:pool]
    rng = np.random.default_rng(seed)
    pick = rng.choice(cand, size=min(k, cand.size), replace=False)
    extra = rng.choice(g.n, size=max(1, k // 10), replace=False)
    return np.unique(np.concatenate([pick, extra]))


def _sampled_rows(g, out, k, seed, cap):
    roots = _cheap_roots(g, k, seed)
    rows, st = oracle.orbit_rows(g.n, g.edges, roots, cap=cap)
    done = 0
    for r, row, s in zip(roots, rows, st):
        if s == 0:
            assert (out[r] == row).all(), f"row {r}: got {out[r].tolist()} exp {row.tolist()}"
            done += 1
    return done


def test_config2_bench_size_rows_and_invariants(pkg):
    g = graphgen.config(2)
    out = pkg.evoke_orbits_edges(g.n, g.edges)
    _invariants(g, out, cliques=_golden_cliques(2, g))
    done = _sampled_rows(g, out, 300, 2, cap=20_000_000)
    assert done >= 20, done


def test_config2_low_degree_core_full_matrix(pkg):
    """the config-2 subgraph induced by its vertices of degree <= 12: same generator and
    degree tail cut, small enough for the full ESU oracle at n = 1e5"""
    g = graphgen.config(2)
    e = _unique_edges(g.n, g.edges)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=g.n)
    keep = deg <= 12
    e = e[keep[e[:, 0]] & keep[e[:, 1]]].astype(np.int32)
    ref = oracle.orbits(g.n, e)
    _assert_equal(pkg.evoke_orbits_edges(g.n, e), ref, "config2 core")
    # EVOKE-4 and the serial schedule against the oracle at this size too
    got4 = pkg.evoke_orbits_edges(g.n, e, four_only=True)
    _assert_equal(got4[:, :15], ref[:, :15], "config2 core four")
    assert (got4[:, 15:] == 0).all()
    _assert_equal(pkg.evoke_orbits_edges(g.n, e, serial=True), ref, "config2 core serial")


def test_config3_rows_and_invariants(pkg):
    """R-MAT 18 (BASELINE configs[2]): invariants incl. Sigma DIM3 = 3 #K3, Sigma DIM14 =
    4 #K4 and Sigma DIM72 = 5 #K5 (golden totals from the oracle), sampled rooted rows (cheapest roots plus a few
    drawn uniformly, each kept when the rooted oracle finishes within its cap); the hub rows
    are covered by test_noninduced_degree_forms_every_vertex and the invariants"""
    g = graphgen.config(3)
    out = pkg.evoke_orbits_edges(g.n, g.edges)
    _invariants(g, out, cliques=_golden_cliques(3, g))
    done = _sampled_rows(g, out, 100, 3, cap=20_000_000)
    assert done >= 3, done


def test_config4_invariants_and_low_degree_core(pkg):
    """Holme-Kim n = 2e6, ~16M edges (BASELINE configs[3]): whole-matrix invariants (orbit 0
    = degree, per-pattern consistency mod 2^64, clique totals from the independent CPU
    counter) on the full graph, and the full matrix bit-exact against the ESU oracle on the
    subgraph induced by the vertices of degree <= 11 (same generator, ~1.1M edges, n = 2e6).
    Rooted rows are not sampled here: every vertex of this graph (degree >= 8 by
    construction) reaches a hub within two steps, so no rooted enumeration fits a cap."""
    g = graphgen.config(4)
    out = pkg.evoke_orbits_edges(g.n, g.edges)
    _invariants(g, out, cliques=_golden_cliques(4, g))
    del out
    e = _unique_edges(g.n, g.edges)
    e = e[e[:, 0] != e[:, 1]]
    deg = np.bincount(e.ravel(), minlength=g.n)
    keep = deg <= 11
    e = e[keep[e[:, 0]] & keep[e[:, 1]]].astype(np.int32)
    assert e.shape[0] > 1_000_000
    _assert_equal(pkg.evoke_orbits_edges(g.n, e), oracle.orbits(g.n, e), "config4 core")


def test_four_vertex_mode_and_serial_mode(pkg):
    """EVOKE_FLAG_FOUR (the paper's EVOKE-4): columns 0..14 equal the oracle's,
    15..72 are zero; EVOKE_FLAG_SERIAL (passes one after the other) gives the same matrix
    as the concurrent default"""
    rng = np.random.default_rng(5)
    graphs = [graphgen.erdos_renyi(int(rng.integers(5, 14)), float(rng.uniform(0.2, 0.8)), 3000 + t)
              for t in range(40)] + [graphgen.config(1)]
    for g in graphs:
        ref = oracle.orbits(g.n, g.edges)
        got4 = pkg.evoke_orbits_edges(g.n, g.edges, four_only=True)
        _assert_equal(got4[:, :15], ref[:, :15], g.name + " four")
        assert (got4[:, 15:] == 0).all()
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges, serial=True), ref, g.name + " serial")
    g = graphgen.config(2)
    full = pkg.evoke_orbits_edges(g.n, g.edges)
    _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges, four_only=True)[:, :15], full[:, :15], "config2 four")
    _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges, serial=True), full, "config2 serial")


def test_ccd_matches_definition(pkg):
    """evoke_ccd: for each distinct count x of an orbit column, the number of
    vertices whose count is >= x -- checked against the definition written with numpy"""
    g = graphgen.config(2)
    out = pkg.evoke_orbits_edges(g.n, g.edges)
    for orbit in (0, 15, 17, 34, 70, 72):
        col = out[:, orbit]
        vals, cnts = pkg.evoke_ccd(out, orbit)
        uv = np.unique(col)
        assert np.array_equal(vals, uv), orbit
        # every distinct value: #{v : col[v] >= x} = n - #{v : col[v] < x}
        exp = (g.n - np.searchsorted(np.sort(col), uv, side="left")).astype(np.uint64)
        assert np.array_equal(cnts, exp), orbit
        for x in uv[:: max(1, uv.size // 40)]:  # the definition written out on a spread of values
            assert int(cnts[np.searchsorted(uv, x)]) == int((col >= x).sum()), (orbit, x)
        assert int(cnts[0]) == g.n


def test_sorted_full_lists_path(pkg, monkeypatch):
    """the sorted-full-list path (used on triangle-heavy graphs) forced on small graphs:
    same matrices as the oracle"""
    monkeypatch.setenv("EVOKE_SORT_FULL_MIN", "1")
    rng = np.random.default_rng(9)
    for t in range(40):
        g = graphgen.erdos_renyi(int(rng.integers(5, 14)), float(rng.uniform(0.3, 0.9)), 4000 + t)
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name + " sorted")
    for g in (graphgen.config(1), graphgen.complete(9)):
        _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), g.name + " sorted")


def test_scratch_tables_left_zero(pkg, monkeypatch):
    """The per-CTA tables kept between calls (zero-invariant scratch) are all zero again after
    every call: EVOKE_CHECK_ZERO makes the library verify it and fail otherwise.  Runs the
    paths that use them: heavy pair sources (dense and swept tables), hub-local heavy items,
    5-cycle big / mid / light endpoints, on graphs with hubs."""
    monkeypatch.setenv("EVOKE_CHECK_ZERO", "1")
    first = None
    for g in [graphgen.config(2), graphgen.rmat(15, 16, 0.57, 0.19, 0.19, 0.05, 9)]:
        a = pkg.evoke_orbits_edges(g.n, g.edges)
        b = pkg.evoke_orbits_edges(g.n, g.edges, serial=True)
        _assert_equal(b, a, f"{g.name} after reuse")
        first = a if first is None else first
    g = graphgen.config(2)
    pkg.evoke_release_scratch(0)  # freed: the next call allocates and zeroes it again
    _assert_equal(pkg.evoke_orbits_edges(g.n, g.edges), first, "after evoke_release_scratch")
    monkeypatch.setenv("EVOKE_NO_ZERO_POOL", "1")
    c = pkg.evoke_orbits_edges(g.n, g.edges)
    _assert_equal(c, first, "fresh zeroed tables")


# ------------------------------------------- non-induced closed forms on every vertex ---
@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_noninduced_degree_forms_every_vertex(pkg, cfg):
    """non-induced mode: the star-like columns theta0/1/2/6/7/22/23 equal
    their degree-only closed forms (tests/degree_forms.py, pinned against the brute force) on
    EVERY vertex of the config, hub rows included, modulo 2^64"""
    g = graphgen.config(cfg)
    out = pkg.evoke_orbits_edges(g.n, g.edges, induced=False)
    f = degree_forms(g.n, g.edges)
    for c in DEGREE_FORM_COLUMNS:
        bad = np.flatnonzero(out[:, c] != f[c])
        assert bad.size == 0, f"config {cfg} theta{c}: {bad.size} rows differ, first {bad[:5].tolist()}"


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_noninduced_four_vertex_orbits_every_vertex(pkg, cfg):
    """non-induced mode: ALL fifteen orbits with at most 4 vertices
    (theta0..theta14: wedges, triangles, 3-paths, 4-cycles, tailed triangles, diamonds,
    4-cliques) bit-exact on EVERY vertex of the config, hub rows included, against the
    oracle's Lemma-4vertexorbit counter (oracle.dm4_vertex: the paper's equations
    on plain definitions of T(u,v) and C4(u), pinned against the non-induced brute force)"""
    g = graphgen.config(cfg)
    out = pkg.evoke_orbits_edges(g.n, g.edges, induced=False)
    ref = oracle.dm4_vertex(g.n, g.edges)
    for c in range(15):
        bad = np.flatnonzero(out[:, c] != ref[:, c])
        assert bad.size == 0, f"config {cfg} theta{c}: {bad.size} rows differ, first {bad[:5].tolist()}"


@pytest.mark.parametrize("cfg", [2, 4])
def test_noninduced_five_cycles_at_the_hubs(pkg, cfg):
    """non-induced theta34 (the 5-cycles through a vertex, the 5-cycle pass's own output) on
    the 12 highest-degree vertices of the config and 40 drawn uniformly, against the oracle's
    definition walk (oracle.c5_rows: O(#4-paths from v), feasible at hubs of these sparse
    graphs where the rooted ESU is not; on the R-MAT configs every 4-path walk runs through
    the 6e4-degree hub and none finishes)"""
    g = graphgen.config(cfg)
    out = pkg.evoke_orbits_edges(g.n, g.edges, induced=False)
    deg = np.bincount(g.edges.ravel(), minlength=g.n)
    rng = np.random.default_rng(40 + cfg)
    roots = np.unique(np.concatenate([np.argsort(-deg, kind="stable")[:12], rng.choice(g.n, 40, replace=False)]))
    ref, st = oracle.c5_rows(g.n, g.edges, roots, cap=50_000_000_000)
    assert (st == 0).sum() >= 40, st.tolist()
    for r, c, s_ in zip(roots, ref, st):
        if s_ == 0:
            assert out[r, 34] == c, f"config {cfg} vertex {r} (degree {deg[r]}): got {out[r, 34]} exp {c}"


# ------------------------------------------------ clique columns on every vertex ---
def _clique_columns(cfg, g, out, kmax):
    """columns 3 / 14 / 72 of the induced matrix against the oracle's per-vertex clique counts
    (oracle.clique_counts_vertex: a clique is an induced copy of itself, so DIM(v, theta3) =
    T(v), DIM(v, theta14) = K4(v), DIM(v, theta72) = K5(v))"""
    ref = oracle.clique_counts_vertex(g.n, g.edges, kmax=kmax)
    for j, c in enumerate((3, 14, 72)[:kmax - 2]):
        bad = np.flatnonzero(out[:, c] != ref[:, j])
        assert bad.size == 0, f"config {cfg} theta{c}: {bad.size} rows differ, first {bad[:5].tolist()}"


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_clique_columns_every_vertex(pkg, cfg):
    """induced mode: the triangle, 4-clique and 5-clique orbits (theta3, theta14, theta72)
    bit-exact on EVERY vertex of the config, hub rows included, against an enumeration that
    shares nothing with the CUDA path (pinned in tests/test_oracle_pins.py)"""
    g = graphgen.config(cfg)
    _clique_columns(cfg, g, pkg.evoke_orbits_edges(g.n, g.edges), 5)


# ------------------------------------------------------- work-balanced sharding ---
@pytest.mark.parametrize("cfg", [2, 3])
def test_eight_shards_sum_to_full_and_balance(pkg, cfg):
    """8 shards (the 8-GPU decomposition, run one after the other on this device): the partial
    matrices sum (mod 2^64) to the one-shard matrix bit for bit, and every sharded pass's work
    estimate is split evenly (max shard / mean shard)"""
    g = graphgen.config(cfg)
    full = pkg.evoke_orbits_edges(g.n, g.edges)
    acc = np.zeros_like(full)
    own = []
    total = None
    for si in range(8):
        part, st = pkg.evoke_orbits_edges(g.n, g.edges, shard_index=si, num_shards=8, return_stats=True)
        acc += part
        own.append(st["work_shard"])
        total = st["work_total"] if total is None else total
        assert st["work_total"] == total
    _assert_equal(acc, full, f"config {cfg} 8 shards")
    for p in total:
        shares = [o[p] for o in own]
        assert sum(shares) == total[p], p
        if total[p] > 0:
            imb = max(shares) / (total[p] / 8)
            assert imb < 1.25, (p, imb, shares)


# ---------------------------------------------------------------- boundary contract ---
def test_device_pointer_error_leaves_out_untouched(pkg):
    import torch
    dev = torch.device("cuda:0")
    out = torch.full((4, 73), 7, dtype=torch.int64, device=dev)
    bad = torch.tensor([[0, 1], [1, 9]], dtype=torch.int32, device=dev)
    with pytest.raises(pkg.EvokeError):
        pkg.evoke_orbits_edges(4, bad, out=out)
    assert (out == 7).all()


def test_default_stream_inputs_are_ordered(pkg):
    """inputs still being produced on torch's default stream when the call starts (torch's
    default stream reaches the library as a NULL stream): the call must wait for them"""
    import torch
    dev = torch.device("cuda:0")
    g = graphgen.config(1)
    ref = oracle.orbits(g.n, g.edges)
    src = torch.from_numpy(g.edges).to(dev)
    torch.cuda.synchronize()
    for _ in range(3):
        torch.cuda._sleep(50_000_000)          # ~25 ms of queued work on the default stream
        edges = src.clone()                   # written only after the sleep
        out = pkg.evoke_orbits_edges(g.n, edges)
        torch.cuda.synchronize()
        _assert_equal(out.cpu().numpy(), ref, "default-stream ordering")


def test_release_scratch_returns_memory(pkg):
    import torch
    g = graphgen.config(2)
    pkg.evoke_orbits_edges(g.n, g.edges)
    torch.cuda.synchronize()
    free_before, _ = torch.cuda.mem_get_info()
    pkg.evoke_release_scratch(0)
    free_after, _ = torch.cuda.mem_get_info()
    assert free_after > free_before + (256 << 20), (free_before, free_after)


# ------------------------------------------------------------ config 5 (last: longest) ---
def test_config5_invariants(pkg):
    """R-MAT 23 (BASELINE configs[4], ~65M edges, the 8-GPU config) on one B200: orbit 0 =
    degree, per-pattern consistency mod 2^64, Sigma DIM3 = 3 #K3,
    Sigma DIM14 = 4 #K4 and Sigma DIM72 = 5 #K5 (golden totals from the oracle's bitmap
    clique counter), the rooted oracle's rows for sampled cheap roots, and in non-induced
    mode the degree-only closed forms on every vertex"""
    import time
    t0 = time.time()

    def lap(what):  # shown with pytest -s / on failure: where the minutes of this test go
        nonlocal t0
        print(f"[config5] {what}: {time.time() - t0:.1f} s", flush=True)
        t0 = time.time()

    def gpu_state(st):
        import torch
        free, total = torch.cuda.mem_get_info()
        top = sorted(st["ms_pass"].items(), key=lambda kv: -kv[1])[:4]
        return (f"{st['ms_total'] / 1e3:.1f} s on the GPU ({', '.join(f'{k} {v / 1e3:.1f}' for k, v in top)}); "
                f"device free {free / 2**30:.1f} of {total / 2**30:.1f} GiB, torch reserved "
                f"{torch.cuda.memory_reserved() / 2**30:.2f} GiB")

    g = graphgen.config(5)
    lap("generate")
    out, st = pkg.evoke_orbits_edges(g.n, g.edges, return_stats=True)
    lap("GPU call, induced: " + gpu_state(st))
    _invariants(g, out, cliques=_golden_cliques(5, g))
    lap("invariants")
    done = _sampled_rows(g, out, 40, 5, cap=5_000_000)
    assert done >= 3, done
    lap("sampled rows")
    # theta3 and theta14 on every vertex (the 1.1e12 5-cliques are left to the total above)
    _clique_columns(5, g, out, 4)
    lap("clique columns")
    del out
    # non-induced mode: the degree-only closed forms on every vertex, the hubs included
    # (as test_noninduced_degree_forms_every_vertex does for configs 2-4)
    out, st = pkg.evoke_orbits_edges(g.n, g.edges, induced=False, return_stats=True)
    lap("GPU call, non-induced: " + gpu_state(st))
    f = degree_forms(g.n, g.edges)
    lap("degree forms")
    for c in DEGREE_FORM_COLUMNS:
        bad = np.flatnonzero(out[:, c] != f[c])
        assert bad.size == 0, f"config 5 theta{c}: {bad.size} rows differ, first {bad[:5].tolist()}"
