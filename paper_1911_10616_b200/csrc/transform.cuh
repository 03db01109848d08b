// transform.cuh -- host side: the non-induced -> induced transform of Appendix A
// (P:1103-1112).  A[i][j] = number of non-induced matches of orbit i that an induced
// match of orbit j contains, i.e. DM_{H(j)}(w_j, theta_i) on the pattern graph H(j) at a
// vertex w_j of orbit j.  A is generated here from the pattern catalog by
// enumerating every spanning connected edge subset of every pattern -- never transcribed
// (Fig. 11 is pinned by the tests and carries the R18 misprint).  With the orbits
// numbered by (pattern size, edge count) A is unit upper triangular, so A^-1 is an
// integer matrix obtained by back substitution.
//
// The pattern table below is the product's own hand entry of Fig. 2 in the reading R1
// of DESIGN.md (vertex labellings chosen independently of oracle/).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace evoke_host {

struct PatternDef {
  int k;
  const char* edges;  // "ab cd ..." vertex pairs
  int orbit[5];
};

// Fig. 2, reading R1: 30 connected patterns, 73 orbits.
static const PatternDef kPatterns[30] = {
    {2, "01", {0, 0}},
    {3, "01 02", {2, 1, 1}},
    {3, "01 02 12", {3, 3, 3}},
    {4, "02 23 31", {4, 4, 5, 5}},
    {4, "03 13 23", {6, 6, 6, 7}},
    {4, "02 21 13 30", {8, 8, 8, 8}},
    {4, "01 12 13 23", {9, 11, 10, 10}},
    {4, "02 03 12 13 23", {12, 12, 13, 13}},
    {4, "01 02 03 12 13 23", {14, 14, 14, 14}},
    {5, "31 10 02 24", {17, 16, 16, 15, 15}},
    {5, "01 12 23 24", {18, 20, 21, 19, 19}},
    {5, "04 14 24 34", {22, 22, 22, 22, 23}},
    {5, "02 13 23 24 34", {24, 24, 26, 26, 25}},
    {5, "01 12 23 24 34", {27, 28, 30, 29, 29}},
    {5, "02 12 23 24 34", {31, 31, 33, 32, 32}},
    {5, "02 24 41 13 30", {34, 34, 34, 34, 34}},
    {5, "01 12 13 24 34", {35, 38, 37, 37, 36}},
    {5, "01 12 13 14 23 24", {39, 42, 41, 40, 40}},
    {5, "01 23 04 14 24 34", {43, 43, 43, 43, 44}},
    {5, "01 12 13 23 24 34", {45, 47, 48, 48, 46}},
    {5, "03 04 13 14 23 24", {49, 49, 49, 50, 50}},
    {5, "01 02 13 23 24 34", {51, 51, 53, 53, 52}},
    {5, "03 04 13 14 23 24 34", {54, 54, 54, 55, 55}},
    {5, "01 12 13 14 23 24 34", {56, 58, 57, 57, 57}},
    {5, "02 23 31 40 41 42 43", {59, 59, 60, 60, 61}},
    {5, "01 02 13 14 23 24 34", {62, 63, 63, 64, 64}},
    {5, "01 02 12 13 14 23 24 34", {65, 67, 67, 66, 66}},
    {5, "01 02 03 04 12 23 34 41", {69, 68, 68, 68, 68}},
    {5, "02 03 04 12 13 14 23 24 34", {70, 70, 71, 71, 71}},
    {5, "01 02 03 04 12 13 14 23 24 34", {72, 72, 72, 72, 72}},
};

static inline int adj_mask(int k, const std::vector<std::pair<int, int>>& es, const int* perm) {
  int m = 0;
  for (auto& e : es) {
    int a = perm[e.first], b = perm[e.second];
    m |= 1 << (a * k + b);
    m |= 1 << (b * k + a);
  }
  return m;
}

static std::vector<std::pair<int, int>> parse_edges(const char* s) {
  std::vector<std::pair<int, int>> es;
  for (const char* p = s; *p;) {
    if (*p == ' ') { p++; continue; }
    es.push_back({p[0] - '0', p[1] - '0'});
    p += 2;
  }
  return es;
}

struct Transform {
  int64_t A[73][73];
  int64_t Ainv[73][73];
  std::vector<int> rp, col;
  std::vector<long long> val;
};

static Transform build_transform() {
  Transform T;
  std::memset(T.A, 0, sizeof(T.A));
  std::memset(T.Ainv, 0, sizeof(T.Ainv));
  // (k, symmetric adjacency mask over k*k bits) -> orbit per vertex position
  std::vector<std::vector<int>> label[6];
  for (int k = 2; k <= 5; k++) label[k].assign(1 << (k * k), std::vector<int>());
  for (int p = 0; p < 30; p++) {
    const PatternDef& P = kPatterns[p];
    auto es = parse_edges(P.edges);
    int perm[5] = {0, 1, 2, 3, 4};
    do {
      int m = adj_mask(P.k, es, perm);
      std::vector<int> orb(P.k);
      for (int a = 0; a < P.k; a++) orb[perm[a]] = P.orbit[a];
      auto& slot = label[P.k][m];
      if (slot.empty()) slot = orb;
      else if (slot != orb) throw std::runtime_error("pattern table: inconsistent orbits");
    } while (std::next_permutation(perm, perm + P.k));
  }
  for (int p = 0; p < 30; p++) {
    const PatternDef& P = kPatterns[p];
    auto es = parse_edges(P.edges);
    const int ne = (int)es.size();
    // one representative vertex per orbit of H(p)
    for (int w = 0; w < P.k; w++) {
      bool first = true;
      for (int w2 = 0; w2 < w; w2++) if (P.orbit[w2] == P.orbit[w]) first = false;
      if (!first) continue;
      const int j = P.orbit[w];
      for (int sub = 1; sub < (1 << ne); sub++) {
        std::vector<std::pair<int, int>> fs;
        for (int e = 0; e < ne; e++) if (sub >> e & 1) fs.push_back(es[e]);
        int ident[5] = {0, 1, 2, 3, 4};
        int m = adj_mask(P.k, fs, ident);
        const auto& orb = label[P.k][m];
        if (orb.empty()) continue;  // not a spanning connected subgraph
        T.A[orb[w]][j] += 1;
      }
    }
  }
  for (int i = 0; i < 73; i++)
    for (int j = 0; j < 73; j++)
      if ((i == j && T.A[i][j] != 1) || (j < i && T.A[i][j] != 0))
        throw std::runtime_error("transform: A is not unit upper triangular");
  for (int c = 0; c < 73; c++) {
    for (int i = 72; i >= 0; i--) {
      int64_t x = (i == c) ? 1 : 0;
      for (int j = i + 1; j < 73; j++) x -= T.A[i][j] * T.Ainv[j][c];
      T.Ainv[i][c] = x;
    }
  }
  T.rp.assign(74, 0);
  for (int i = 0; i < 73; i++) {
    for (int j = 0; j < 73; j++)
      if (T.Ainv[i][j]) { T.col.push_back(j); T.val.push_back(T.Ainv[i][j]); }
    T.rp[i + 1] = (int)T.col.size();
  }
  return T;
}

static const Transform& transform() {
  static std::once_flag once;
  static Transform* T = nullptr;
  std::call_once(once, [] { T = new Transform(build_transform()); });
  return *T;
}

}  // namespace evoke_host
