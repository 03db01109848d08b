"""Every tier / table variant of the enumeration passes forced onto small graphs and compared
bit for bit with the CPU oracle (-m gpu, through the C ABI).

The library picks a code path per work unit by size (warp / small CTA / big CTA, shared or
global tables, 16- / 32- / 64-bit table fields); on the bench graphs the heavy variants run
only for a few hub units, where no enumerator can check the rows.  The EVOKE_* limits below
can only be LOWERED: lowering one moves units
onto the heavier variant, whose tables are sized for anything, so each variant runs here on
every unit of graphs the oracle solves completely.
"""
import numpy as np
import pytest

import graphgen
import oracle

pytestmark = pytest.mark.gpu

HEAVY_PAIR = {"EVOKE_PAIR_LIGHT_MAX": "0", "EVOKE_PAIR_MIDS_MAX": "0", "EVOKE_PAIR_MID_MAX": "0"}
C5_BIG = {"EVOKE_C5_LIGHT_REC": "0", "EVOKE_C5_MID_REC": "0"}
COMBOS = {
    "pair_u64_tables": {"EVOKE_PAIR_PACKED_LIM": "0"},                 # k_pairs_heavy<u64>
    "pair_dense_touched": dict(HEAVY_PAIR, EVOKE_PAIR_SWEEP="0"),      # k_pairs_heavy<u32, false>
    "pair_dense_swept": dict(HEAVY_PAIR, EVOKE_PAIR_SWEEP="1"),        # k_pairs_heavy<u32, true>
    "pair_mid": {"EVOKE_PAIR_LIGHT_MAX": "0", "EVOKE_PAIR_MIDS_MAX": "0"},  # k_pairs_main CTA tier
    "pair_small_mid": {"EVOKE_PAIR_LIGHT_MAX": "0"},                  # k_pairs_mids
    "pair_light_no_tiny": {"EVOKE_PAIR_TINY_MAX": "0"},                # light sources all in k_pairs_main
    "pair_dense_hot_partial": dict(HEAVY_PAIR, EVOKE_PAIR_HOT="16"),   # heavy tables, top 16 ranks shared
    "pair_dense_nohot": dict(HEAVY_PAIR, EVOKE_PAIR_HOT="0"),
    "hub_warp": {"EVOKE_HUB_MICRO_MAX": "0"},                         # hub_item_warp (no micro items)
    "hub_heavy_hash": {"EVOKE_HUB_WARP_MAX": "0"},                    # hub_item_cta<HUB_T_HASH>
    "hub_heavy_shared": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_HASH_MAX": "0"},  # <HUB_T_SHPOS>
    "hub_heavy_global": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_HASH_MAX": "0",
                         "EVOKE_HUB_SH_DENSE": "0"},                  # <HUB_T_GLPOS>
    "hub_heavy_hash_tight": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_HASH_MAX": "8"},  # mixed per item
    "hub_giant": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_GIANT": "40"},  # k_hub_heavy<1024> + <256>
    "hub_split_queue": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_SPLIT": "40"},  # long lists chunked over the CTA
    "hub_giant_positions": {"EVOKE_HUB_WARP_MAX": "0", "EVOKE_HUB_GIANT": "0", "EVOKE_HUB_HASH_MAX": "0"},
    "c5_light_global": {"EVOKE_C5_SHCAP": "64"},                       # k_c5_light, global regions
    "c5_mid": {"EVOKE_C5_LIGHT_REC": "0"},                             # k_c5_mid
    "c5_big_u32": dict(C5_BIG),                                        # k_c5_heavy<u32> + bitmaps
    "c5_big_u64": dict(C5_BIG, EVOKE_C5_WIDE="1"),
    "c5_big_nobits": dict(C5_BIG, EVOKE_C5_NO_BITS="1"),
    "c5_big_hot": dict(C5_BIG, EVOKE_C5_HOT_MIN_W="0"),              # hot-vertex cache of every rank
    "c5_big_hot_partial": dict(C5_BIG, EVOKE_C5_HOT_MIN_W="0", EVOKE_C5_HOT="16"),  # of the top 16 ranks
    "c5_light_by_work": {"EVOKE_C5_LIGHT_WORK": "40", "EVOKE_C5_MID_WORK": "200"},
    "tri_not_flat": {"EVOKE_TRI_NO_FLAT": "1"},                       # k_triangles (warp walks N+(a) item by item)
    "c5_giant": {"EVOKE_C5_GIANT_W": "300"},                          # k_c5_giant (whole-GPU endpoints)
    "c5_giant_all": {"EVOKE_C5_GIANT_W": "1"},                        # every endpoint a giant
    "all_heavy_sorted": dict(HEAVY_PAIR, **C5_BIG, EVOKE_PAIR_PACKED_LIM="0", EVOKE_HUB_WARP_MAX="0",
                             EVOKE_HUB_HASH_MAX="0", EVOKE_HUB_SH_DENSE="0", EVOKE_C5_WIDE="1", EVOKE_SORT_FULL_MIN="1"),
}


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_10616_b200 as p
    p.lib()
    return p


def _book(pages, p, seed):
    """book graph: the spine edge (0, 1) and `pages` vertices adjacent to both ends (T(0,1) =
    pages), plus seeded random page-page edges"""
    rng = np.random.default_rng(seed)
    e = [(0, 1)] + [(0, 2 + i) for i in range(pages)] + [(1, 2 + i) for i in range(pages)]
    e += [(2 + i, 2 + j) for i in range(pages) for j in range(i + 1, pages) if rng.random() < p]
    return graphgen.Graph(f"book{pages}_p{p}", pages + 2, np.array(e, dtype=np.int32))


@pytest.fixture(scope="module")
def corpus():
    rng = np.random.default_rng(21)
    gs = []
    for t in range(30):
        n = int(rng.integers(4, 14))
        gs.append(graphgen.erdos_renyi(n, float(rng.uniform(0.15, 0.95)), 12000 + t))
    gs += [_book(70, 0.0, 1), _book(80, 0.04, 2)]  # T(a,b) > 64: long chord parts (the CTA queue)
    gs += [graphgen.config(1), graphgen.erdos_renyi(40, 0.5, 1), graphgen.erdos_renyi(34, 0.9, 3),
           graphgen.erdos_renyi(500, 0.02, 31), graphgen.erdos_renyi(2500, 0.004, 32), graphgen.petersen(),
           graphgen.complete(9), graphgen.complete_bipartite(4, 9)]
    return [(g, oracle.orbits(g.n, g.edges)) for g in gs]


def _eq(got, exp, what):
    got = np.asarray(got).view(np.uint64)
    bad = np.argwhere(got != exp)
    assert bad.size == 0, f"{what}: {len(bad)} mismatches, first (vertex, orbit) {bad[:8].tolist()}"


@pytest.mark.parametrize("combo", sorted(COMBOS))
def test_forced_tier_matches_oracle(pkg, corpus, combo, monkeypatch):
    for k, v in COMBOS[combo].items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("EVOKE_CHECK_ZERO", "1")  # the tables kept between calls stay zero
    for g, ref in corpus:
        _eq(pkg.evoke_orbits_edges(g.n, g.edges), ref, f"{combo} {g.name}")
    # non-induced output of the same variant (DM, before the transform)
    for g, _ in corpus[:12]:
        _eq(pkg.evoke_orbits_edges(g.n, g.edges, induced=False), oracle.noninduced_bruteforce(g.n, g.edges),
            f"{combo} non-induced {g.name}")


@pytest.mark.parametrize("combo", ["all_heavy_sorted", "pair_u64_tables", "c5_big_u64"])
def test_forced_tier_tiled_graph(pkg, combo, monkeypatch):
    """the heavy variants over a ~0.5M-edge disjoint union of seeded tiles (many units per CTA,
    table reuse across units): full matrix against the per-tile oracle"""
    for k, v in COMBOS[combo].items():
        monkeypatch.setenv(k, v)
    tiles = [graphgen.erdos_renyi(30, 0.2, 55 * 1000 + i) for i in range(32)]
    refs = [oracle.orbits(t.n, t.edges) for t in tiles]
    pick = np.random.default_rng(55).integers(0, 32, size=6000)
    g, _ = graphgen.disjoint_union([tiles[i] for i in pick], "tiled-small")
    exp = np.concatenate([refs[i] for i in pick], axis=0)
    _eq(pkg.evoke_orbits_edges(g.n, g.edges), exp, f"{combo} tiled")


@pytest.mark.parametrize("combo", ["all_heavy_sorted", "hub_heavy_global", "c5_big_u32"])
def test_forced_tier_closed_forms(pkg, combo, monkeypatch):
    """hubs under the forced variants: K_{1,s}, K_{a,b} and K_n rows against their closed forms
    (SURVEY 8(c) table), computed by the oracle's own ESU on small instances of the same family"""
    for k, v in COMBOS[combo].items():
        monkeypatch.setenv(k, v)
    for g in [graphgen.star(40), graphgen.complete_bipartite(3, 30), graphgen.complete(14)]:
        _eq(pkg.evoke_orbits_edges(g.n, g.edges), oracle.orbits(g.n, g.edges), f"{combo} {g.name}")


@pytest.mark.parametrize("giant_w", ["1", "2000"])
def test_giant_endpoints_split_over_shards(pkg, giant_w, monkeypatch):
    """giant 5-cycle endpoints run on every shard with step 3 split by j-key and the constant
    terms on shard 0: the shard partials still sum (mod 2^64) to the one-shard matrix, which
    equals the oracle's"""
    monkeypatch.setenv("EVOKE_C5_GIANT_W", giant_w)
    monkeypatch.setenv("EVOKE_CHECK_ZERO", "1")
    for g in [graphgen.erdos_renyi(60, 0.3, 77), graphgen.complete(12), _book(80, 0.04, 2)]:
        ref = oracle.orbits(g.n, g.edges)
        _eq(pkg.evoke_orbits_edges(g.n, g.edges), ref, f"giants {g.name}")
        for ns in (2, 3, 8):
            acc = np.zeros((g.n, 73), dtype=np.uint64)
            for si in range(ns):
                acc += np.asarray(pkg.evoke_orbits_edges(g.n, g.edges, shard_index=si, num_shards=ns)).view(np.uint64)
            _eq(acc, ref, f"giants {g.name} shards={ns}")
