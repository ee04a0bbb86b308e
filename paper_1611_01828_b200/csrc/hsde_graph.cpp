// hsde_graph.cpp -- host side of the decomposition:
// chordality test, chordal extension and maximal-clique enumeration of a
// block's sparsity pattern, with the reference's exact orderings and
// tie-breaking so the cliques (and therefore the slot layout) are identical.
//
//   mcs_order            graphs.py:73-97   maximum cardinality search; heap on
//                                          (-weight, node): ties -> smallest node
//   verify_peo           graphs.py:100-110
//   min_degree_eliminate graphs.py:121-149 greedy minimum degree; heap on
//                                          (degree, node); fill in sorted order
//   elimination_cliques  graphs.py:167-184 candidates {v} + later neighbours,
//                                          by (-size, sorted members), kept if
//                                          not inside a kept clique of its anchor
//   clique order         graphs.py:217-220 by (min, sorted tuple)
#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <queue>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hsde.h"

namespace {

using Adj = std::vector<std::vector<int>>;  // sorted neighbour lists

Adj build_adj(int n, int64_t ne, const int32_t *ei, const int32_t *ej) {
  Adj adj(n);
  for (int64_t k = 0; k < ne; ++k) {
    const int i = ei[k], j = ej[k];
    if (i == j) continue;
    adj[i].push_back(j);
    adj[j].push_back(i);
  }
  for (auto &a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  return adj;
}

std::vector<int> mcs_order(const Adj &adj) {
  const int n = (int)adj.size();
  std::vector<int> weight(n, 0);
  std::vector<char> visited(n, 0);
  using E = std::pair<int, int>;  // (-weight, node): smallest first
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int v = 0; v < n; ++v) heap.push({0, v});
  std::vector<int> visit;
  visit.reserve(n);
  while (!heap.empty()) {
    const E top = heap.top();
    heap.pop();
    const int v = top.second;
    if (visited[v] || -top.first != weight[v]) continue;
    visited[v] = 1;
    visit.push_back(v);
    for (int u : adj[v])
      if (!visited[u]) {
        ++weight[u];
        heap.push({-weight[u], u});
      }
  }
  std::reverse(visit.begin(), visit.end());
  return visit;
}

bool verify_peo(const Adj &adj, const std::vector<int> &order) {
  const int n = (int)adj.size();
  std::vector<int> pos(n);
  for (int k = 0; k < n; ++k) pos[order[k]] = k;
  std::vector<int> later;
  for (int v : order) {
    later.clear();
    for (int u : adj[v])
      if (pos[u] > pos[v]) later.push_back(u);
    if (later.size() <= 1) continue;
    int parent = later[0];
    for (int u : later)
      if (pos[u] < pos[parent]) parent = u;
    const auto &pa = adj[parent];
    for (int u : later)
      if (u != parent && !std::binary_search(pa.begin(), pa.end(), u)) return false;
  }
  return true;
}

// greedy minimum-degree elimination; returns the fill edges (a < b) in the
// order they are added
// Bitset form of min_degree_fill_sets below, for n <= kBitsetMaxN: row v of
// an n x n bit matrix is v's current neighbourhood.  Scanning a row gives the
// neighbours in ascending order, and the fill for the pair loop (x < y over
// the sorted neighbours) is, per x, the word-parallel set nbrs & ~row(x) &
// (bits > x) -- the same pairs in the same order, in O(deg * n / 64) words
// per elimination instead of O(deg^2 log deg) set probes.
constexpr int kBitsetMaxN = 32768;

std::vector<std::pair<int, int>> min_degree_fill_bitset(const Adj &adj0) {
  const int n = (int)adj0.size();
  const size_t W = ((size_t)n + 63) / 64;
  std::vector<uint64_t> bits((size_t)n * W, 0);
  auto row = [&](int v) { return bits.data() + (size_t)v * W; };
  std::vector<int> deg(n, 0);
  for (int v = 0; v < n; ++v) {
    for (int u : adj0[v]) row(v)[u >> 6] |= 1ull << (u & 63);
    int d = 0;
    for (size_t w = 0; w < W; ++w) d += __builtin_popcountll(row(v)[w]);
    deg[v] = d;
  }
  using E = std::pair<int, int>;  // (degree, node)
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int v = 0; v < n; ++v) heap.push({deg[v], v});
  std::vector<char> eliminated(n, 0);
  std::vector<std::pair<int, int>> fill;
  std::vector<int> nbrs;
  std::vector<uint64_t> nb(W);
  while (!heap.empty()) {
    const E top = heap.top();
    heap.pop();
    const int v = top.second;
    if (eliminated[v] || top.first != deg[v]) continue;
    eliminated[v] = 1;
    uint64_t *rv = row(v);
    nbrs.clear();
    for (size_t w = 0; w < W; ++w) {
      nb[w] = rv[w];
      for (uint64_t x = rv[w]; x; x &= x - 1) nbrs.push_back((int)(w * 64 + __builtin_ctzll(x)));
    }
    for (int u : nbrs) {
      row(u)[v >> 6] &= ~(1ull << (v & 63));
      --deg[u];
    }
    for (int x : nbrs) {
      uint64_t *rx = row(x);
      const size_t w0 = (size_t)(x + 1) >> 6;
      for (size_t w = w0; w < W; ++w) {
        uint64_t miss = nb[w] & ~rx[w];
        if (w == w0) miss &= ~0ull << ((x + 1) & 63);
        for (; miss; miss &= miss - 1) {
          const int y = (int)(w * 64 + __builtin_ctzll(miss));
          rx[w] |= 1ull << (y & 63);
          row(y)[x >> 6] |= 1ull << (x & 63);
          ++deg[x];
          ++deg[y];
          fill.push_back({x, y});
        }
      }
    }
    for (int u : nbrs) heap.push({deg[u], u});
  }
  return fill;
}

std::vector<std::pair<int, int>> min_degree_fill_sets(const Adj &adj0) {
  const int n = (int)adj0.size();
  std::vector<std::set<int>> adj(n);
  for (int v = 0; v < n; ++v) adj[v].insert(adj0[v].begin(), adj0[v].end());
  using E = std::pair<int, int>;  // (degree, node)
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int v = 0; v < n; ++v) heap.push({(int)adj[v].size(), v});
  std::vector<char> eliminated(n, 0);
  std::vector<std::pair<int, int>> fill;
  std::vector<int> nbrs;
  while (!heap.empty()) {
    const E top = heap.top();
    heap.pop();
    const int v = top.second;
    if (eliminated[v] || top.first != (int)adj[v].size()) continue;
    eliminated[v] = 1;
    nbrs.assign(adj[v].begin(), adj[v].end());  // sorted
    for (int u : nbrs) adj[u].erase(v);
    for (size_t a = 0; a < nbrs.size(); ++a)
      for (size_t b = a + 1; b < nbrs.size(); ++b) {
        const int x = nbrs[a], y = nbrs[b];
        if (!adj[x].count(y)) {
          adj[x].insert(y);
          adj[y].insert(x);
          fill.push_back({x, y});
        }
      }
    for (int u : nbrs) heap.push({(int)adj[u].size(), u});
  }
  return fill;
}

std::vector<std::vector<int>> elimination_cliques(const Adj &adj, const std::vector<int> &order) {
  const int n = (int)adj.size();
  std::vector<int> pos(n);
  for (int k = 0; k < n; ++k) pos[order[k]] = k;
  std::vector<std::vector<int>> cands;
  cands.reserve(n);
  for (int v : order) {
    std::vector<int> c{v};
    for (int u : adj[v])
      if (pos[u] > pos[v]) c.push_back(u);
    std::sort(c.begin(), c.end());
    cands.push_back(std::move(c));
  }
  std::sort(cands.begin(), cands.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
    if (a.size() != b.size()) return a.size() > b.size();
    return a < b;
  });
  cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
  std::vector<std::vector<int>> kept;
  std::vector<std::vector<int>> by_node(n);  // kept cliques containing a node
  for (auto &c : cands) {
    const int anchor = c[0];
    bool inside = false;
    for (int ki : by_node[anchor]) {
      const auto &k = kept[ki];
      if (std::includes(k.begin(), k.end(), c.begin(), c.end())) {
        inside = true;
        break;
      }
    }
    if (inside) continue;
    const int id = (int)kept.size();
    kept.push_back(c);
    for (int u : c) by_node[u].push_back(id);
  }
  std::sort(kept.begin(), kept.end(), [](const std::vector<int> &a, const std::vector<int> &b) {
    if (a[0] != b[0]) return a[0] < b[0];
    return a < b;
  });
  return kept;
}

}  // namespace

struct hsde_pattern {
  int chordal = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> nodes;
  std::vector<int32_t> fi, fj;
};

extern "C" {

int hsde_pattern_decompose(int32_t n, int64_t n_edges, const int32_t *ei, const int32_t *ej, int32_t extend,
                           hsde_pattern_t **out) {
  if (!out || n < 1 || n_edges < 0 || (n_edges && (!ei || !ej))) return HSDE_ERR_ARG;
  for (int64_t k = 0; k < n_edges; ++k)
    if (ei[k] < 0 || ei[k] >= n || ej[k] < 0 || ej[k] >= n) return HSDE_ERR_ARG;
  hsde_pattern *p = new hsde_pattern();
  Adj adj = build_adj(n, n_edges, ei, ej);
  std::vector<int> order = mcs_order(adj);
  p->chordal = verify_peo(adj, order) ? 1 : 0;
  if (!p->chordal) {
    if (!extend) {
      delete p;
      return HSDE_ERR_ARG;  // NotChordal (graphs.py:269-270)
    }
    const auto fill = (int)adj.size() <= kBitsetMaxN ? min_degree_fill_bitset(adj) : min_degree_fill_sets(adj);
    for (const auto &f : fill) {
      p->fi.push_back(f.first);
      p->fj.push_back(f.second);
      adj[f.first].push_back(f.second);
      adj[f.second].push_back(f.first);
    }
    for (auto &a : adj) std::sort(a.begin(), a.end());
    order = mcs_order(adj);
    if (!verify_peo(adj, order)) {
      delete p;
      return HSDE_ERR_ARG;
    }
  }
  const auto cliques = elimination_cliques(adj, order);
  p->ptr.push_back(0);
  for (const auto &c : cliques) {
    p->nodes.insert(p->nodes.end(), c.begin(), c.end());
    p->ptr.push_back((int64_t)p->nodes.size());
  }
  *out = p;
  return HSDE_OK;
}

int hsde_pattern_sizes(const hsde_pattern_t *p, int64_t *n_cliques, int64_t *n_nodes, int64_t *n_fill,
                       int32_t *was_chordal) {
  if (!p) return HSDE_ERR_ARG;
  if (n_cliques) *n_cliques = (int64_t)p->ptr.size() - 1;
  if (n_nodes) *n_nodes = (int64_t)p->nodes.size();
  if (n_fill) *n_fill = (int64_t)p->fi.size();
  if (was_chordal) *was_chordal = p->chordal;
  return HSDE_OK;
}

int hsde_pattern_cliques(const hsde_pattern_t *p, int64_t *ptr, int32_t *nodes) {
  if (!p || !ptr || (!nodes && !p->nodes.empty())) return HSDE_ERR_ARG;
  std::copy(p->ptr.begin(), p->ptr.end(), ptr);
  std::copy(p->nodes.begin(), p->nodes.end(), nodes);
  return HSDE_OK;
}

int hsde_pattern_fill(const hsde_pattern_t *p, int32_t *fi, int32_t *fj) {
  if (!p || ((!fi || !fj) && !p->fi.empty())) return HSDE_ERR_ARG;
  std::copy(p->fi.begin(), p->fi.end(), fi);
  std::copy(p->fj.begin(), p->fj.end(), fj);
  return HSDE_OK;
}

void hsde_pattern_destroy(hsde_pattern_t *p) { delete p; }

// The report's pattern index (solver.py:443-452 restated on the compressed
// layout): for the sorted codes gi * n + gj of the aggregate pattern plus the
// diagonal, the block (1-based), the block-local (i, j) (1-based), and where
// the column-major flat id gj * n + gi sits in the sorted `covered` (pos_c,
// clamped) and whether it is there (hit).  One pass in code order: the row gi
// never decreases, so within every column gj the looked-up keys ascend and a
// per-column pointer into `covered` only moves forward -- O(nq + n_covered),
// sequential output.  starts[0..nblocks] are the block offsets.
int hsde_pattern_index(const int64_t *covered, int64_t n_covered, int64_t n, const int64_t *code, int64_t nq,
                       const int64_t *starts, int32_t nblocks, int64_t *block, int64_t *li, int64_t *lj,
                       int64_t *pos_c, uint8_t *hit) {
  if (n <= 0 || n_covered < 0 || nq < 0 || nblocks < 1 || !starts || (n_covered && !covered) ||
      (nq && (!code || !block || !li || !lj || !pos_c || !hit)))
    return HSDE_ERR_ARG;
  for (int64_t q = 0; q < nq; ++q)
    if (code[q] < 0 || code[q] >= n * n || (q && code[q] <= code[q - 1])) return HSDE_ERR_ARG;  // sorted, unique
  std::vector<int64_t> ptr(n + 1), cblock(n);
  for (int64_t c = 0, i = 0; c <= n; ++c) {  // first covered index of column c
    while (i < n_covered && covered[i] < c * n) ++i;
    ptr[c] = i;
  }
  const std::vector<int64_t> cend(ptr.begin() + 1, ptr.end());
  for (int64_t c = 0, b = 0; c < n; ++c) {  // block of every column / row index
    while (b + 1 < nblocks && starts[b + 1] <= c) ++b;
    cblock[c] = b;
  }
  int64_t r = 0;
  for (int64_t q = 0; q < nq; ++q) {
    while (code[q] >= (r + 1) * n) ++r;
    const int64_t c = code[q] - r * n, key = c * n + r;  // (gi, gj) = (r, c)
    int64_t i = ptr[c];
    const int64_t end = cend[c];
    while (i < end && covered[i] < key) ++i;
    ptr[c] = i;
    const int64_t pc = std::min(i, std::max<int64_t>(n_covered - 1, 0));
    pos_c[q] = pc;
    hit[q] = i < n_covered && covered[pc] == key;
    const int64_t br = cblock[r], bc = cblock[c];
    block[q] = br + 1;
    li[q] = r - starts[br] + 1;
    lj[q] = c - starts[bc] + 1;
  }
  return HSDE_OK;
}

}  // extern "C"
