"""Developer parity sweep (GPU): small random graphs + config 1 vs the oracle; prints the
orbits that disagree.  Usage: python tools/dev_check.py [count]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import graphgen
import oracle
import paper_1911_10616_b200 as pkg


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(1)
    bad_orbits = {}
    nbad = 0
    for t in range(count):
        n = int(rng.integers(2, 14))
        p = float(rng.uniform(0.1, 0.9))
        g = graphgen.erdos_renyi(n, p, 1000 + t)
        ref = oracle.orbits(g.n, g.edges)
        for induced in (True, False):
            got = pkg.evoke_orbits_edges(g.n, g.edges, induced=induced)
            exp = ref if induced else oracle.noninduced_bruteforce(g.n, g.edges)
            d = np.argwhere(got != exp)
            if d.size:
                nbad += 1
                for (_, th) in d:
                    bad_orbits[(induced, int(th))] = bad_orbits.get((induced, int(th)), 0) + 1
    print("small graphs: cases with mismatches:", nbad, "orbits:", sorted(bad_orbits.items())[:60])
    for cfg in (1,):
        g = graphgen.config(cfg)
        ref = oracle.orbits(g.n, g.edges)
        got = pkg.evoke_orbits_edges(g.n, g.edges)
        d = np.argwhere(got != ref)
        print(f"config {cfg}: mismatching entries {len(d)}; orbits {sorted(set(int(x) for x in d[:,1]))}")
    for cfg in (2, 3):
        g = graphgen.config(cfg)
        t0 = time.time()
        out, st = pkg.evoke_orbits_edges(g.n, g.edges, return_stats=True)
        t1 = time.time()
        print(f"config {cfg}: wall {t1-t0:.3f}s stats", {k: v for k, v in st.items() if k != 'ms_pass'})
        print("   passes:", {k: round(v, 3) for k, v in st["ms_pass"].items()})


if __name__ == "__main__":
    main()
