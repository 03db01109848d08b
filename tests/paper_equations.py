"""The paper's printed orbit equations, evaluated literally on a tiny graph (test helper).

Used ONLY to pin the oracle's orbit catalog (tests/test_oracle_pins.py): the oracle's
non-induced brute force DM(v, theta) must equal these equations on every vertex of
random small graphs.  Every equation is transcribed from PAPER.md in its own notation:

* Lemma "4vertexorbit": DM(u, lambda_0..14)
* Lemma "4edgeorbit": E0..E11 on ordered edges
* Theorem B.1: DM(u, lambda_15..71) except 34 (and 72, not printed)

with the readings listed in DESIGN.md section "Readings" (R4 parenthesisation, R6 theta19,
R7 theta20/21, R9 theta35, R10 theta40/60, R11 D(u,v,w), R12 theta66, R13 theta69,
R14 TT, R15 summation ranges).  A reading marked LITERAL below is the printed form;
the tests check that the printed form of each erratum fails and the reading holds.
"""
from __future__ import annotations

from itertools import combinations
from math import comb


def C(x: int, k: int) -> int:
    return comb(x, k) if x >= k else 0


class G:
    def __init__(self, n, edges):
        self.n = n
        self.N = [set() for _ in range(n)]
        for a, b in edges:
            if a != b:
                self.N[a].add(b)
                self.N[b].add(a)

    def d(self, u):
        return len(self.N[u])

    def adj(self, a, b):
        return b in self.N[a]

    def T(self, u, v=None):
        if v is None:
            return sum(1 for a, b in combinations(sorted(self.N[u]), 2) if self.adj(a, b))
        return len(self.N[u] & self.N[v])

    def W(self, u, v):
        return len(self.N[u] & self.N[v])

    def triangles_at(self, u):
        """each triangle containing u once, as (v, x) unordered (R15)"""
        return [(v, x) for v, x in combinations(sorted(self.N[u]), 2) if self.adj(v, x)]

    def cliques4_at(self, u):
        out = []
        for v, x, y in combinations(sorted(self.N[u]), 3):
            if self.adj(v, x) and self.adj(v, y) and self.adj(x, y):
                out.append((v, x, y))
        return out

    def C4(self, u, v=None):
        if v is None:  # C4(u) = sum_{x != u} C(W(u,x), 2)
            return sum(C(self.W(u, x), 2) for x in range(self.n) if x != u)
        # C4(u,v) = sum_{x in N(u)\v} (W(x,v) - 1)  (4-cycles through edge uv)
        return sum(self.W(x, v) - 1 for x in self.N[u] if x != v)

    def K4(self, *vs):
        if len(vs) == 1:
            return len(self.cliques4_at(vs[0]))
        common = set(range(self.n))
        for v in vs:
            common &= self.N[v]
        common -= set(vs)
        if len(vs) == 2:
            a, b = vs
            return sum(1 for x, y in combinations(sorted(common), 2) if self.adj(x, y))
        return len(common)  # K4(t) for a triangle t


def edge_orbits(g: G, u: int, v: int) -> dict:
    """Lemma 4edgeorbit for the ordered edge <u,v>."""
    E = {}
    E[0] = g.d(u) - 1
    E[1] = g.T(u, v)
    E[2] = sum(g.d(x) - 1 for x in g.N[u] if x != v) - E[1]
    E[3] = (g.d(u) - 1) * (g.d(v) - 1) - E[1]
    E[4] = C(g.d(u) - 1, 2)
    E[5] = g.C4(u, v)
    E[6] = g.T(u) - E[1]
    tri = g.N[u] & g.N[v]
    E[7] = sum(g.d(x) - 2 for x in tri)  # R4: "-2" inside the sum
    E[8] = E[1] * (g.d(u) - 2)
    E[9] = sum(g.T(u, x) - 1 for x in tri)  # R4
    E[10] = C(E[1], 2)
    E[11] = g.K4(u, v)
    return E


def noninduced_equations(g: G, variant: dict | None = None) -> list[list[int]]:
    """DM(u, theta) for theta in 0..71 (34 -> None) by the paper's equations.

    ``variant`` switches individual equations back to the literal printed form
    (keys: 'theta19', 'theta20_21', 'theta40', 'D', 'theta66', 'theta69') so tests can
    show that each printed erratum fails on brute force while the reading holds."""
    variant = variant or {}
    n = g.n
    DM = [[0] * 73 for _ in range(n)]
    # --- 4-vertex orbits, Lemma 4vertexorbit -- needs two passes
    for u in range(n):
        d = g.d(u)
        DM[u][0] = d
        DM[u][1] = sum(g.d(v) - 1 for v in g.N[u])
        DM[u][2] = C(d, 2)
        DM[u][3] = g.T(u)
    for u in range(n):
        d = g.d(u)
        D = DM[u]
        D[4] = sum(DM[v][1] for v in g.N[u]) - 2 * D[2] - 2 * D[3]
        D[5] = D[1] * (d - 1) - 2 * D[3]
        D[6] = sum(C(g.d(v) - 1, 2) for v in g.N[u])
        D[7] = C(d, 3)
        D[8] = g.C4(u)
        D[9] = sum(DM[v][3] - g.T(u, v) for v in g.N[u])
        D[10] = sum(g.T(u, v) * (g.d(v) - 2) for v in g.N[u])
        D[11] = D[3] * (d - 2)
        D[12] = sum(g.T(v, x) - 1 for v, x in g.triangles_at(u))
        D[13] = sum(C(g.T(u, v), 2) for v in g.N[u])
        D[14] = g.K4(u)

    def Dv(v, i):
        return DM[v][i]

    for u in range(n):
        d = g.d(u)
        D = DM[u]
        Nu = sorted(g.N[u])
        tris = g.triangles_at(u)
        others = [v for v in range(n) if v != u]
        E = {v: edge_orbits(g, u, v) for v in Nu}          # <u,v>
        Er = {v: edge_orbits(g, v, u) for v in Nu}         # <v,u>
        D[15] = sum(Dv(v, 4) for v in Nu) - D[5] - 2 * D[11] - 2 * D[8]
        D[16] = D[4] * (d - 1) - D[10] - 2 * D[8]
        D[17] = C(D[1], 2) - D[3] - D[6] - D[8] - D[10]
        D[18] = sum(Dv(v, 6) for v in Nu) - 3 * D[7] - D[10]
        if variant.get("theta19"):  # literal: DM(u, lambda_u) is not defined; use DM(u, lambda_u=?)
            D[19] = sum(Dv(v, 5) for v in Nu) - D[4] - D[10]  # drops the garbled term
        else:  # R6: lambda_u -> lambda_5
            D[19] = sum(Dv(v, 5) for v in Nu) - D[4] - D[5] - D[10]
        # R7: the printed coefficients (2 for theta20, 1 for theta21) are swapped
        c20, c21 = (2, 1) if variant.get("theta20_21") else (1, 2)
        D[20] = sum((d - 1) * C(g.d(v) - 1, 2) for v in Nu) - c20 * D[10]
        D[21] = sum((g.d(v) - 1) * C(d - 1, 2) for v in Nu) - c21 * D[11]
        D[22] = sum(C(g.d(v) - 1, 3) for v in Nu)
        D[23] = C(d, 4)
        D[24] = sum(Dv(v, 10) for v in Nu) - D[10] - 2 * D[11] - 2 * D[12]
        D[25] = sum((g.d(v) - 2) * (g.d(x) - 2) for v, x in tris) - D[12]
        D[26] = sum((d - 2) * ((g.d(x) - 2) + (g.d(v) - 2)) for v, x in tris) - 2 * D[13]
        D[27] = sum(Dv(v, 9) for v in Nu) - D[11] - 2 * D[13]
        D[28] = sum((d - 1) * Dv(v, 3) for v in Nu) - 2 * D[3] - 2 * D[11] - 2 * D[12]
        D[29] = (sum(Dv(v, 1) + Dv(x, 1) for v, x in tris) - 4 * D[3] - D[10] - 2 * D[11]
                 - 2 * D[12] - 2 * D[13])
        D[30] = sum((g.d(v) - 1) * D[3] for v in Nu) - 2 * D[3] - D[10] - 2 * D[13]
        D[31] = sum((g.d(v) - 1) * Dv(v, 3) for v in Nu) - 2 * D[9] - D[10] - 2 * D[3]
        D[32] = sum(C(g.d(v) - 2, 2) + C(g.d(x) - 2, 2) for v, x in tris)
        D[33] = D[3] * C(d - 2, 2)
        D[34] = None
        D[35] = sum(Dv(v, 8) for v in Nu) - 2 * D[8] - D[13]  # R9: R_8, R_13 read as DM8, DM13
        D[36] = sum(C(g.W(u, v), 2) * (g.d(v) - 2) for v in others) - D[13]
        D[37] = sum(E[v][5] * (g.d(v) - 2) for v in Nu) - 2 * D[12]
        D[38] = D[8] * (d - 2) - D[13]
        D[39] = sum(Dv(v, 13) for v in Nu) - D[13] - 2 * D[12]
        if variant.get("theta40"):  # literal E9(u,v)
            D[40] = sum(E[v][9] * (g.d(v) - 3) for v in Nu)
        else:  # R10: E9(<v,u>)
            D[40] = sum(Er[v][9] * (g.d(v) - 3) for v in Nu)
        D[41] = sum(C(E[v][1], 2) * (g.d(v) - 3) for v in Nu)
        D[42] = sum(C(E[v][1], 2) * (d - 3) for v in Nu)
        D[43] = sum((Dv(v, 3) - 1) + (Dv(x, 3) - 1) for v, x in tris) - 2 * D[12] - 2 * D[13]
        D[44] = C(D[3], 2) - D[13]
        D[45] = sum(Dv(v, 12) for v in Nu) - 2 * D[13] - 3 * D[14]
        D[46] = sum(edge_orbits(g, v, x)[7] for v, x in tris) - D[11] - 3 * D[14]
        D[47] = D[12] * (d - 2) - 3 * D[14]
        D[48] = (sum((E[v][1] - 1) * (g.d(x) - 2) + (E[x][1] - 1) * (g.d(v) - 2) for v, x in tris)
                 - 6 * D[14])
        D[49] = sum(C(g.W(v, x) - 1, 2) for v, x in combinations(Nu, 2))
        D[50] = sum(C(g.W(u, v), 3) for v in others)

        def TT(a, b):  # R14
            return sum(g.T(x, b) - (1 if g.adj(a, b) else 0) for x in g.N[a] & g.N[b])

        D[51] = sum(TT(u, v) * (g.W(u, v) - 1) for v in others) - 2 * D[12]
        D[52] = sum(edge_orbits(g, v, x)[5] for v, x in tris) - 2 * D[13]
        D[53] = sum(E[v][5] + E[x][5] for v, x in tris) - 2 * D[13] - 2 * D[12]
        D[54] = sum(C(edge_orbits(g, v, x)[1] - 1, 2) for v, x in tris)
        D[55] = sum(C(E[v][1], 3) for v in Nu)
        D[56] = sum(Dv(v, 14) for v in Nu) - 3 * D[14]
        D[57] = sum(E[v][11] * (g.d(v) - 3) for v in Nu)
        D[58] = D[14] * (d - 3)
        D[59] = (sum(edge_orbits(g, x, v)[9] + edge_orbits(g, v, x)[9] for v, x in tris)
                 - 2 * D[13] - 6 * D[14])
        D[60] = sum(Er[v][9] * (E[v][1] - 1) for v in Nu) - 6 * D[14]  # printed E9(<v,u>)
        D[61] = sum((E[v][1] - 1) * (E[x][1] - 1) for v, x in tris) - 3 * D[14]

        def Dpair(a, b):  # D(u,v): diamonds with u, v off the chord = edges inside N(a) & N(b)
            cm = sorted(g.N[a] & g.N[b])
            return sum(1 for x, y in combinations(cm, 2) if g.adj(x, y))

        def Dtrip(a, b, c):
            if variant.get("D"):  # literal: u and w are the chord vertices
                # diamonds containing a, b, c with a and c on the chord
                if not g.adj(a, c):
                    return 0
                return C(len((g.N[a] & g.N[c]) - {b}), 1) if b in (g.N[a] & g.N[c]) else 0
            return len(g.N[a] & g.N[b] & g.N[c])  # R11

        D[62] = sum(Dpair(v, x) for v, x in combinations(Nu, 2)) - D[13]
        D[63] = sum(Dpair(u, v) * (g.W(u, v) - 2) for v in others)
        D[64] = sum(Dtrip(v, u, x) * (g.W(v, x) - 2) for v, x in combinations(Nu, 2))
        D[65] = sum(edge_orbits(g, v, x)[11] for v, x in tris) - 3 * D[14]
        k4s = g.cliques4_at(u)
        D[66] = sum(g.T(v, x) + g.T(v, y) + g.T(x, y) for v, x, y in k4s)
        if not variant.get("theta66"):
            D[66] -= 6 * D[14]  # R12
        D[67] = sum(E[v][11] * (E[v][1] - 2) for v in Nu)
        D[68] = sum(C(Dtrip(u, v, x), 2) for v in Nu for x in g.N[v] if x != u)
        s69 = sum(C(Dtrip(u, v, x), 2) for v, x in combinations(Nu, 2))
        if variant.get("theta69"):
            D[69] = s69
        else:
            D[69] = s69 // 2  # R13 (s69 is even: each 4-cycle of G[N(u)] has two diagonals)
        D[70] = sum(g.K4(v, x, y) - 1 for v, x, y in k4s)
        D[71] = sum(C(g.K4(u, v, x), 2) for v, x in tris)
        D[72] = None
    return DM


def theta27_alt(g: G, DM, u, coef=2):
    """Second printed form of theta27; R8: coefficients 2,2,2 (printed: 1,1,1)."""
    s = sum(g.W(u, v) * DM[v][3] for v in range(g.n) if v != u)
    return s - coef * DM[u][13] - coef * DM[u][9] - coef * DM[u][3]


def theta18_alt(g: G, DM, u):
    """Second printed form of theta18."""
    return sum(g.W(u, v) * C(g.d(v) - 1, 2) for v in range(g.n) if v != u) - DM[u][10]
