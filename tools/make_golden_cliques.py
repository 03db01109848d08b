"""Write tests/golden/clique_totals.json: #triangles / #4-cliques / #5-cliques of the BASELINE
configs, counted by the CPU oracle (oracle.clique_totals, pinned in tests/test_oracle_pins.py)
and nothing else.  The GPU invariants Sigma DIM3 = 3 #K3, Sigma DIM14 = 4 #K4, Sigma DIM72 =
5 #K5 (cliques: PAPER.md P:702) read these values; each entry carries the SHA-256
of the generated edge list, which the test checks before using it.

    python tools/make_golden_cliques.py [config ...]      (default: 2 3 4 5)
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402

# largest clique size whose count the plain loop nest (oracle.clique_totals) finishes in
# minutes on an 8-core host; the bitmap counter (oracle.clique_totals_bits, pinned against it)
# counts up to 5 everywhere, and both must agree on every size the plain one reaches
KMAX = {2: 5, 3: 4, 4: 5, 5: 3}
OUT = os.path.join(ROOT, "tests", "golden", "clique_totals.json")


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data["_source"] = ("oracle.clique_totals_bits (cliques counted at their first vertex in degree order, "
                       "P:432-437, membership on a local bitmap of N>(a)), checked equal to the plain loop nest "
                       "oracle.clique_totals up to plain_counter_kmax; on graphgen.config(i); written by "
                       "tools/make_golden_cliques.py")
    for c in cfgs:
        g = graphgen.config(c)
        sha = hashlib.sha256(g.edges.tobytes()).hexdigest()
        t0 = time.time()
        plain = oracle.clique_totals(g.n, g.edges, kmax=KMAX[c])
        t3, t4, t5 = oracle.clique_totals_bits(g.n, g.edges, kmax=5)
        for a, b in zip(plain, (t3, t4, t5)):
            assert a is None or a == b, (c, plain, (t3, t4, t5))
        data[str(c)] = {"graph": g.name, "n": g.n, "m_raw": int(g.edges.shape[0]), "edges_sha256": sha,
                        "triangles": t3, "k4": t4, "k5": t5, "kmax": 5,
                        "plain_counter_kmax": KMAX[c]}
        print(c, data[str(c)], f"{time.time() - t0:.1f} s", flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
