// Host path/slice planner.  Not the hot path: the paper takes its
// paths and slices from CoTenGra ("Our code does not perform the search
// for optimal slices or paths"); this is a plain greedy planner so the build is
// self-contained:
//   1. absorb every rank<=2 tensor (kets, 1-qudit gates, bras) into a neighbour
//      (exact re-association, emitted as the first SSA steps);
//   2. randomised greedy pair selection (Gumbel noise, two score functions), best of
//      many seeded trials by total FLOP, run on host threads;
//   3. subtree reconfiguration: optimal re-contraction of <=F-subtree frontiers by
//      subset DP (the local optimisation of Huang et al.);
//   4. greedy slicing of labels on the largest intermediates, each pick followed by a
//      reconfiguration sweep of the sliced tree;
//   5. slice-loop order for the prefix cache (heaviest label outermost + local search).
// Deterministic given the seed.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <functional>
#include <limits>
#include <queue>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "jt_internal.hpp"

namespace jt {
namespace {

struct SplitMix {
  uint64_t s;
  explicit SplitMix(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

// ---------------------------------------------------------------- bitsets over labels
struct BitPool {
  int W = 1;
  std::vector<uint64_t> v;
  uint64_t* at(size_t i) { return v.data() + i * W; }
  const uint64_t* at(size_t i) const { return v.data() + i * W; }
  size_t add() {
    v.resize(v.size() + W, 0);
    return v.size() / W - 1;
  }
};

inline int pc(const uint64_t* a, int W) {
  int c = 0;
  for (int i = 0; i < W; ++i) c += __builtin_popcountll(a[i]);
  return c;
}
inline int pc_and_not(const uint64_t* a, const uint64_t* m, int W) {
  int c = 0;
  for (int i = 0; i < W; ++i) c += __builtin_popcountll(a[i] & ~m[i]);
  return c;
}
inline int pc_union_not(const uint64_t* a, const uint64_t* b, const uint64_t* m, int W) {
  int c = 0;
  for (int i = 0; i < W; ++i) c += __builtin_popcountll((a[i] | b[i]) & ~m[i]);
  return c;
}
inline int pc_xor_not(const uint64_t* a, const uint64_t* b, const uint64_t* m, int W) {
  int c = 0;
  for (int i = 0; i < W; ++i) c += __builtin_popcountll((a[i] ^ b[i]) & ~m[i]);
  return c;
}

// ---------------------------------------------------------------- contraction tree
struct TNode {
  int left = -1, right = -1, parent = -1;
};

struct Tree {
  int W = 1;
  int n_leaves = 0;
  std::vector<TNode> nodes;
  std::vector<uint64_t> lab;  // nodes.size() * W, output labels of each node
  int root = -1;
  uint64_t* L(int i) { return lab.data() + (size_t)i * W; }
  const uint64_t* L(int i) const { return lab.data() + (size_t)i * W; }
  bool leaf(int i) const { return nodes[i].left < 0; }
};

struct CostModel {
  double log2d = 1.0;
  std::vector<double> dpow;  // d^n
  int cap = std::numeric_limits<int>::max();  // max output width in labels
  double R = 0;  // roofline weight: FLOP/8 per element moved (0 = pure FLOP objective)
  // Kernel-aware roofline model (seconds), used when rf_bw > 0: a contraction that K3 can run
  // (qubits: small side 3..7 free bits, 2..8 contracted bits, big side >= 7 free bits) costs
  // max(flop / rf_tc, bytes / rf_bw), any other max(flop / rf_cuda, bytes / rf_bw); plus a
  // fixed per-launch gap.
  double rf_bw = 0, rf_cuda = 0, rf_tc = 0, rf_gap = 0, esize = 8;
  bool qubits = true;
  double node_cost(int n_union, int n_a, int n_b, int n_out) const {
    double c;
    if (rf_bw > 0) {
      const double flop = 8.0 * dpow[n_union];
      const double bytes = esize * (dpow[n_a] + dpow[n_b] + dpow[n_out]);
      double F = rf_cuda;
      if (qubits && rf_tc > 0) {
        const int k = n_a + n_b - n_union, fa = n_a - k, fb = n_b - k;
        const int small = std::min(fa, fb), big = std::max(fa, fb);
        if (small >= 3 && small <= 7 && k >= 2 && k <= 8 && big >= 7) F = rf_tc;
      }
      c = std::max(flop / F, bytes / rf_bw) + rf_gap;
    } else {
      c = dpow[n_union];
      if (R > 0) c = std::max(c, R * (dpow[n_a] + dpow[n_b] + dpow[n_out]));
    }
    if (n_out > cap) c *= 1e6;  // soft width cap (in labels)
    return c;
  }
};

double tree_cost(const Tree& T, const CostModel& cm, const uint64_t* mask, int* maxw) {
  double tot = 0;
  int mw = 0;
  for (size_t i = T.n_leaves; i < T.nodes.size(); ++i) {
    const TNode& n = T.nodes[i];
    if (n.left < 0) continue;
    int u = pc_union_not(T.L(n.left), T.L(n.right), mask, T.W);
    int o = pc_and_not(T.L((int)i), mask, T.W);
    tot += cm.node_cost(u, pc_and_not(T.L(n.left), mask, T.W), pc_and_not(T.L(n.right), mask, T.W), o);
    mw = std::max(mw, o);
  }
  for (int i = 0; i < T.n_leaves; ++i) mw = std::max(mw, pc_and_not(T.L(i), mask, T.W));
  if (maxw) *maxw = mw;
  return tot;
}

// post-order of internal nodes
void postorder(const Tree& T, std::vector<int>& out) {
  out.clear();
  std::vector<std::pair<int, int>> st;
  st.push_back({T.root, 0});
  while (!st.empty()) {
    auto& top = st.back();
    int v = top.first;
    if (T.leaf(v)) {
      st.pop_back();
      continue;
    }
    if (top.second == 0) {
      top.second = 1;
      st.push_back({T.nodes[v].left, 0});
    } else if (top.second == 1) {
      top.second = 2;
      st.push_back({T.nodes[v].right, 0});
    } else {
      out.push_back(v);
      st.pop_back();
    }
  }
}

// ---------------------------------------------------------------- greedy
struct GreedyResult {
  std::vector<std::pair<int, int>> pairs;  // over leaf ids then new ids n_leaves + s
  double cost = std::numeric_limits<double>::infinity();
};

GreedyResult greedy_once(const BitPool& leaves, int n_leaves, const CostModel& cm, int variant,
                         double temperature, uint64_t seed,
                         const std::vector<std::vector<int>>& carriers0) {
  const int W = leaves.W;
  SplitMix rng(seed);
  BitPool lab;
  lab.W = W;
  lab.v = leaves.v;
  lab.v.reserve((size_t)W * 2 * n_leaves);
  std::vector<int> size(n_leaves);
  std::vector<char> alive(n_leaves, 1);
  for (int i = 0; i < n_leaves; ++i) size[i] = pc(lab.at(i), W);
  std::vector<std::vector<int>> carriers = carriers0;  // label -> tensors holding it
  struct Cand {
    double score;
    int a, b;
    bool operator<(const Cand& o) const {
      if (score != o.score) return score > o.score;  // min-heap
      if (a != o.a) return a > o.a;
      return b > o.b;
    }
  };
  std::priority_queue<Cand> heap;
  std::vector<uint64_t> tmp(W);
  auto score = [&](int a, int b) {
    int so = 0;
    const uint64_t* A = lab.at(a);
    const uint64_t* B = lab.at(b);
    for (int i = 0; i < W; ++i) so += __builtin_popcountll(A[i] ^ B[i]);
    int sa = size[a], sb = size[b];
    double s;
    if (variant == 0) {
      int mx = std::max(sa, sb);
      s = (cm.dpow[so] - cm.dpow[sa] - cm.dpow[sb]) / cm.dpow[mx];
    } else {
      s = (double)(so - std::max(sa, sb));
    }
    if (temperature > 0) s -= temperature * std::log(-std::log(rng.uniform()));
    return s;
  };
  auto push_neighbours = [&](int t) {
    const uint64_t* A = lab.at(t);
    std::vector<int> nb;
    for (int w = 0; w < W; ++w) {
      uint64_t x = A[w];
      while (x) {
        int bit = __builtin_ctzll(x);
        x &= x - 1;
        int l = w * 64 + bit;
        for (int o : carriers[l])
          if (o != t && alive[o]) nb.push_back(o);
      }
    }
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    for (int o : nb) heap.push({score(std::min(t, o), std::max(t, o)), std::min(t, o), std::max(t, o)});
  };
  for (int t = 0; t < n_leaves; ++t) {
    const uint64_t* A = lab.at(t);
    for (int w = 0; w < W; ++w) {
      uint64_t x = A[w];
      while (x) {
        int bit = __builtin_ctzll(x);
        x &= x - 1;
        int l = w * 64 + bit;
        for (int o : carriers[l])
          if (o > t) heap.push({score(t, o), t, o});
      }
    }
  }
  GreedyResult res;
  int n_alive = n_leaves;
  double cost = 0;
  while (n_alive > 1) {
    int a = -1, b = -1;
    while (!heap.empty()) {
      Cand c = heap.top();
      heap.pop();
      if (alive[c.a] && alive[c.b]) {
        a = c.a;
        b = c.b;
        break;
      }
    }
    if (a < 0) {  // disconnected: contract the two smallest alive tensors
      std::vector<std::pair<int, int>> al;
      for (size_t i = 0; i < alive.size(); ++i)
        if (alive[i]) al.push_back({size[i], (int)i});
      std::sort(al.begin(), al.end());
      a = std::min(al[0].second, al[1].second);
      b = std::max(al[0].second, al[1].second);
    }
    size_t c = lab.add();
    const uint64_t* A = lab.at(a);
    const uint64_t* B = lab.at(b);
    uint64_t* C = lab.at(c);
    int un = 0;
    for (int i = 0; i < W; ++i) {
      C[i] = A[i] ^ B[i];
      un += __builtin_popcountll(A[i] | B[i]);
    }
    int so = pc(C, W);
    cost += cm.node_cost(un, size[a], size[b], so);
    alive[a] = alive[b] = 0;
    alive.push_back(1);
    size.push_back(so);
    for (int w = 0; w < W; ++w) {
      uint64_t x = C[w];
      while (x) {
        int bit = __builtin_ctzll(x);
        x &= x - 1;
        for (int& o : carriers[w * 64 + bit])
          if (o == a || o == b) o = (int)c;
      }
    }
    res.pairs.push_back({a, b});
    --n_alive;
    push_neighbours((int)c);
  }
  res.cost = cost;
  return res;
}

Tree tree_from_pairs(const BitPool& leaves, int n_leaves, const std::vector<std::pair<int, int>>& pairs) {
  Tree T;
  T.W = leaves.W;
  T.n_leaves = n_leaves;
  T.nodes.assign(n_leaves + pairs.size(), TNode());
  T.lab.assign(T.nodes.size() * T.W, 0);
  std::copy(leaves.v.begin(), leaves.v.begin() + (size_t)n_leaves * T.W, T.lab.begin());
  for (size_t s = 0; s < pairs.size(); ++s) {
    int v = n_leaves + (int)s;
    auto [a, b] = pairs[s];
    T.nodes[v].left = a;
    T.nodes[v].right = b;
    T.nodes[a].parent = v;
    T.nodes[b].parent = v;
    for (int i = 0; i < T.W; ++i) T.L(v)[i] = T.L(a)[i] ^ T.L(b)[i];
  }
  T.root = pairs.empty() ? 0 : n_leaves + (int)pairs.size() - 1;
  return T;
}

// ---------------------------------------------------------------- recursive bisection (f2)
// A contraction tree from recursive graph bisection (the partitioned paths of PAPER.md l.176 use
// hypergraph partitioning, CoTenGra/KaHyPar): split the tensor set into two parts with few labels
// between them (Fiduccia-Mattheyses refinement of a grown region, a few random starts, part
// sizes within a balance band), contract each part recursively, then the two results.  Every
// label sits on exactly two tensors, so the hypergraph is a multigraph with edge weight =
// shared labels.  Cut labels are the labels of the intermediate; its width is what slicing and
// the roofline objective trade off later.
GreedyResult partition_once(const BitPool& leaves, int n_leaves, const CostModel& cm,
                            const std::vector<std::vector<int>>& carriers, uint64_t seed, double imbalance) {
  SplitMix rng(seed);
  // leaf adjacency with multiplicities
  std::vector<std::vector<std::pair<int, int>>> adj(n_leaves);
  {
    std::vector<std::unordered_map<int, int>> m(n_leaves);
    for (const auto& c : carriers)
      if (c.size() == 2 && c[0] != c[1]) {
        ++m[c[0]][c[1]];
        ++m[c[1]][c[0]];
      }
    for (int u = 0; u < n_leaves; ++u) {
      for (auto& kv : m[u]) adj[u].push_back(kv);
      std::sort(adj[u].begin(), adj[u].end());
    }
  }
  std::vector<int> side(n_leaves, -1), pos(n_leaves, -1);
  GreedyResult res;
  int next_id = n_leaves;
  // bisect the node set S (side[] marks membership via pos[] >= 0 while active)
  auto bisect = [&](const std::vector<int>& S, std::vector<int>& A, std::vector<int>& B) {
    const int n = (int)S.size();
    for (int i = 0; i < n; ++i) pos[S[i]] = i;
    const double f = 0.5 - imbalance * 0.5 * rng.uniform();
    const int lo = std::max(1, (int)std::floor(n * f)), hi = n - lo;
    std::vector<char> best_side;
    int best_cut = std::numeric_limits<int>::max();
    const int starts = n > 64 ? 4 : 2;
    std::vector<char> sd(n);
    std::vector<int> gain(n);
    for (int st = 0; st < starts; ++st) {
      // grow region 0 from a random seed, preferring nodes most connected to it
      std::fill(sd.begin(), sd.end(), 1);
      std::vector<int> conn(n, 0);
      int size0 = 0;
      const int target = std::max(1, std::min(n - 1, lo));  // the smaller part
      int u = (int)(rng.next() % (uint64_t)n);
      while (size0 < target) {
        sd[u] = 0;
        ++size0;
        for (auto& e : adj[S[u]]) {
          const int j = pos[e.first];
          if (j >= 0 && j < n && S[j] == e.first && sd[j]) conn[j] += e.second;
        }
        int bu = -1, bc = -1;
        for (int j = 0; j < n; ++j)
          if (sd[j] && (conn[j] > bc || (conn[j] == bc && (rng.next() & 1)))) { bc = conn[j]; bu = j; }
        if (bu < 0) break;
        u = bu;
      }
      // FM passes: move the best-gain unlocked node keeping lo <= |part| <= hi, keep the best prefix
      auto cut_of = [&]() {
        int c = 0;
        for (int i = 0; i < n; ++i)
          for (auto& e : adj[S[i]]) {
            const int j = pos[e.first];
            if (j >= 0 && j < n && S[j] == e.first && sd[i] != sd[j]) c += e.second;
          }
        return c / 2;
      };
      int cut = cut_of();
      for (int pass = 0; pass < 4; ++pass) {
        for (int i = 0; i < n; ++i) {
          int g = 0;
          for (auto& e : adj[S[i]]) {
            const int j = pos[e.first];
            if (j >= 0 && j < n && S[j] == e.first) g += sd[j] != sd[i] ? e.second : -e.second;
          }
          gain[i] = g;
        }
        std::vector<char> locked(n, 0);
        std::vector<int> moves;
        int cur = cut, bestc = cut, bestk = 0, n0 = 0;
        for (int i = 0; i < n; ++i) n0 += sd[i] == 0;
        for (int k = 0; k < n; ++k) {
          int bi = -1, bg = std::numeric_limits<int>::min();
          for (int i = 0; i < n; ++i) {
            if (locked[i]) continue;
            const int n0n = n0 + (sd[i] == 0 ? -1 : 1);
            if (std::min(n0n, n - n0n) < lo) continue;
            if (gain[i] > bg) { bg = gain[i]; bi = i; }
          }
          if (bi < 0) break;
          locked[bi] = 1;
          n0 += sd[bi] == 0 ? -1 : 1;
          sd[bi] ^= 1;
          cur -= bg;
          moves.push_back(bi);
          for (auto& e : adj[S[bi]]) {
            const int j = pos[e.first];
            if (j >= 0 && j < n && S[j] == e.first && !locked[j]) gain[j] += sd[j] == sd[bi] ? -2 * e.second : 2 * e.second;
          }
          if (cur < bestc) { bestc = cur; bestk = (int)moves.size(); }
        }
        for (int k = (int)moves.size() - 1; k >= bestk; --k) sd[moves[k]] ^= 1;
        if (bestc >= cut) break;
        cut = bestc;
      }
      if (cut < best_cut) { best_cut = cut; best_side = sd; }
    }
    A.clear();
    B.clear();
    for (int i = 0; i < n; ++i) (best_side[i] ? B : A).push_back(S[i]);
    for (int i = 0; i < n; ++i) pos[S[i]] = -1;
  };
  std::function<int(const std::vector<int>&)> build = [&](const std::vector<int>& S) -> int {
    if (S.size() == 1) return S[0];
    std::vector<int> A, B;
    if (S.size() == 2) { A = {S[0]}; B = {S[1]}; }
    else bisect(S, A, B);
    if (A.empty() || B.empty()) {  // degenerate split: peel one node
      A.assign(S.begin(), S.end() - 1);
      B.assign(1, S.back());
    }
    const int a = build(A), b = build(B);
    res.pairs.push_back({a, b});
    return next_id++;
  };
  std::vector<int> all(n_leaves);
  for (int i = 0; i < n_leaves; ++i) all[i] = i;
  build(all);
  Tree T = tree_from_pairs(leaves, n_leaves, res.pairs);
  std::vector<uint64_t> nomask(leaves.W, 0);
  res.cost = tree_cost(T, cm, nomask.data(), nullptr);
  (void)side;
  return res;
}

// ---------------------------------------------------------------- subtree reconfiguration
bool reconf_node(Tree& T, int v, int F, const CostModel& cm, const uint64_t* mask) {
  const int W = T.W;
  auto ncost = [&](int u) {
    const TNode& n = T.nodes[u];
    return cm.node_cost(pc_union_not(T.L(n.left), T.L(n.right), mask, W), pc_and_not(T.L(n.left), mask, W),
                        pc_and_not(T.L(n.right), mask, W), pc_and_not(T.L(u), mask, W));
  };
  std::vector<int> frontier{v}, removed;
  while ((int)frontier.size() < F) {
    int best = -1;
    double bc = -1;
    for (size_t i = 0; i < frontier.size(); ++i) {
      int u = frontier[i];
      if (T.leaf(u)) continue;
      double c = ncost(u);
      if (c > bc) {
        bc = c;
        best = (int)i;
      }
    }
    if (best < 0) break;
    int u = frontier[best];
    removed.push_back(u);
    frontier[best] = T.nodes[u].left;
    frontier.push_back(T.nodes[u].right);
  }
  if (removed.size() <= 1) return false;
  double old = 0;
  for (int u : removed) old += ncost(u);
  const int f = (int)frontier.size();
  const int NS = 1 << f;
  std::vector<uint64_t> lab((size_t)NS * W, 0);
  std::vector<double> best(NS, std::numeric_limits<double>::infinity());
  std::vector<int> split(NS, 0);
  for (int S = 1; S < NS; ++S) {
    int low = __builtin_ctz(S);
    uint64_t* LS = lab.data() + (size_t)S * W;
    if (S == (1 << low)) {
      std::copy(T.L(frontier[low]), T.L(frontier[low]) + W, LS);
      best[S] = 0;
      continue;
    }
    const uint64_t* Lrest = lab.data() + (size_t)(S ^ (1 << low)) * W;
    const uint64_t* Llow = lab.data() + (size_t)(1 << low) * W;
    for (int i = 0; i < W; ++i) LS[i] = Lrest[i] ^ Llow[i];
    int out = pc_and_not(LS, mask, W);
    // enumerate S1 subset of S containing the low bit, S1 != S
    int rest = S ^ (1 << low);
    for (int sub = rest;; sub = (sub - 1) & rest) {
      int S1 = sub | (1 << low);
      if (S1 != S) {
        int S2 = S ^ S1;
        double c1 = best[S1], c2 = best[S2];
        if (c1 + c2 < best[S]) {
          const uint64_t* L1 = lab.data() + (size_t)S1 * W;
          const uint64_t* L2 = lab.data() + (size_t)S2 * W;
          int un = pc_union_not(L1, L2, mask, W);
          double c = c1 + c2 + cm.node_cost(un, pc_and_not(L1, mask, W), pc_and_not(L2, mask, W), out);
          if (c < best[S]) {
            best[S] = c;
            split[S] = S1;
          }
        }
      }
      if (sub == 0) break;
    }
  }
  if (!(best[NS - 1] < old * (1.0 - 1e-9))) return false;
  // rebuild, reusing the removed internal ids; v stays on top
  std::vector<int> pool(removed.rbegin(), removed.rend());  // removed[0] == v -> popped last
  std::function<int(int, bool)> build = [&](int S, bool top) -> int {
    if (__builtin_popcount(S) == 1) return frontier[__builtin_ctz(S)];
    int id;
    if (top) {
      id = v;
      pool.erase(std::find(pool.begin(), pool.end(), v));
    } else {
      id = pool.back();
      pool.pop_back();
      if (id == v) {  // never hand v to a non-top subset
        int other = pool.back();
        pool.pop_back();
        pool.push_back(v);
        id = other;
      }
    }
    int a = build(split[S], false);
    int b = build(S ^ split[S], false);
    T.nodes[id].left = a;
    T.nodes[id].right = b;
    T.nodes[a].parent = id;
    T.nodes[b].parent = id;
    for (int i = 0; i < W; ++i) T.L(id)[i] = T.L(a)[i] ^ T.L(b)[i];
    return id;
  };
  int parent = T.nodes[v].parent;
  build(NS - 1, true);
  T.nodes[v].parent = parent;
  return true;
}

void reconf_sweeps(Tree& T, int sweeps, int F, const CostModel& cm, const uint64_t* mask) {
  std::vector<int> order;
  for (int s = 0; s < sweeps; ++s) {
    postorder(T, order);
    bool any = false;
    for (int v : order) any |= reconf_node(T, v, F, cm, mask);
    if (!any) break;
  }
}

// Greedy slicing: repeatedly slice the label, taken from the current largest
// intermediates, that minimises (max width, cost) while over the width cap, else cost; each
// pick is followed by one reconfiguration sweep of the sliced tree.
// Executed cost of the one-copy prefix cache for the sliced labels `labs` taken as the loop
// order (labs[0] outermost): sum_v c(v) d^(maxpos(S(v)) + 1), S(v) = the labels of labs on the
// leaves under v (PAPER.md l.205-212 Eq. task_based with the prefix-cache multiplicity, a6).
double prefix_tree_cost(const Tree& T, const CostModel& cm, const uint64_t* mask, const std::vector<int>& labs,
                        const std::vector<int>& po) {
  const int W = T.W;
  const int k = (int)labs.size();
  std::vector<uint64_t> dep(T.nodes.size(), 0);
  for (int i = 0; i < T.n_leaves; ++i)
    for (int c = 0; c < k; ++c)
      if (T.L(i)[labs[c] / 64] & (uint64_t(1) << (labs[c] % 64))) dep[i] |= uint64_t(1) << c;
  double tot = 0;
  for (int v : po) {
    const TNode& n = T.nodes[v];
    dep[v] = dep[n.left] | dep[n.right];
    const int mp = dep[v] ? 63 - __builtin_clzll(dep[v]) : -1;
    tot += cm.node_cost(pc_union_not(T.L(n.left), T.L(n.right), mask, W), pc_and_not(T.L(n.left), mask, W),
                        pc_and_not(T.L(n.right), mask, W), pc_and_not(T.L(v), mask, W)) *
           cm.dpow[mp + 1];
  }
  return tot;
}

void slice_tree(Tree& T, const CostModel& cm, int kmax, int capw, int sweeps, int F, int NL,
                std::vector<uint64_t>& mask, std::vector<int>& chosen, int objective = 0) {
  const int W = T.W;
  if (kmax == 0 || T.n_leaves <= 1) return;
  std::vector<int> po;
  for (int iter = 0; iter < 62; ++iter) {
    int mw;
    tree_cost(T, cm, mask.data(), &mw);
    if (kmax >= 0 && (int)chosen.size() >= kmax) break;
    if (kmax < 0 && (capw < 0 || mw <= capw)) break;
    std::vector<char> cand(NL, 0);
    for (size_t v = 0; v < T.nodes.size(); ++v) {
      if (pc_and_not(T.L((int)v), mask.data(), W) >= mw - 1) {
        const uint64_t* A = T.L((int)v);
        for (int w = 0; w < W; ++w) {
          uint64_t x = A[w] & ~mask[w];
          while (x) {
            int bit = __builtin_ctzll(x);
            x &= x - 1;
            cand[w * 64 + bit] = 1;
          }
        }
      }
    }
    int bl = -1;
    double bc = 0;
    int bw = 0;
    const bool width_first = (capw < 0) || (mw > capw);
    if (objective == 1) postorder(T, po);
    std::vector<int> labs = chosen;
    labs.push_back(-1);
    for (int l = 0; l < NL; ++l) {
      if (!cand[l]) continue;
      mask[l / 64] |= uint64_t(1) << (l % 64);
      int nw;
      double c = tree_cost(T, cm, mask.data(), &nw);
      if (objective == 1 && chosen.size() < 62) {
        labs.back() = l;
        c = prefix_tree_cost(T, cm, mask.data(), labs, po);
      }
      mask[l / 64] &= ~(uint64_t(1) << (l % 64));
      bool better;
      if (bl < 0) better = true;
      else if (width_first) better = (nw < bw) || (nw == bw && c < bc);
      else better = (c < bc) || (c == bc && nw < bw);
      if (better) {
        bl = l;
        bc = c;
        bw = nw;
      }
    }
    if (bl < 0) break;
    mask[bl / 64] |= uint64_t(1) << (bl % 64);
    chosen.push_back(bl);
    if (sweeps > 0) {
      CostModel cmc = cm;
      if (capw > 0) cmc.cap = capw;
      reconf_sweeps(T, 1, F, cmc, mask.data());
    }
  }
}

// ---------------------------------------------------------------- absorption
struct Absorbed {
  std::vector<int64_t> pre_path;        // SSA steps over raw ids
  std::vector<int64_t> comp_ssa;        // SSA id of each composite tensor
  std::vector<std::vector<int64_t>> comp_labels;
};

Absorbed absorb(const jt_network& net) {
  const int64_t nt = (int64_t)net.tensors.size();
  Absorbed ab;
  std::vector<std::vector<int64_t>> labs(nt);
  for (int64_t t = 0; t < nt; ++t) labs[t] = net.tensors[t].labels;
  std::unordered_map<int64_t, std::vector<int64_t>> carriers;
  for (int64_t t = 0; t < nt; ++t)
    for (int64_t l : labs[t]) carriers[l].push_back(t);
  std::vector<char> alive(nt, 1);
  int64_t n_alive = nt;
  std::vector<int64_t> queue;
  for (int64_t t = 0; t < nt; ++t)
    if (labs[t].size() <= 2) queue.push_back(t);
  size_t qi = 0;
  while (qi < queue.size() && n_alive > 1) {
    int64_t t = queue[qi++];
    if (!alive[t] || labs[t].size() > 2) continue;
    // neighbour with the largest rank (ties: smallest id)
    int64_t best = -1;
    size_t br = 0;
    for (int64_t l : labs[t])
      for (int64_t o : carriers[l])
        if (o != t && alive[o] && (best < 0 || labs[o].size() > br || (labs[o].size() == br && o < best))) {
          best = o;
          br = labs[o].size();
        }
    if (best < 0) continue;  // isolated scalar: left to the main tree
    int64_t nid = (int64_t)labs.size();
    std::vector<int64_t> out;
    for (int64_t l : labs[t])
      if (std::find(labs[best].begin(), labs[best].end(), l) == labs[best].end()) out.push_back(l);
    for (int64_t l : labs[best])
      if (std::find(labs[t].begin(), labs[t].end(), l) == labs[t].end()) out.push_back(l);
    ab.pre_path.push_back(t);
    ab.pre_path.push_back(best);
    alive[t] = alive[best] = 0;
    alive.push_back(1);
    labs.push_back(out);
    for (int64_t l : out)
      for (auto& o : carriers[l])
        if (o == t || o == best) o = nid;
    --n_alive;
    if (out.size() <= 2) queue.push_back(nid);
  }
  for (size_t i = 0; i < alive.size(); ++i)
    if (alive[i]) {
      ab.comp_ssa.push_back((int64_t)i);
      ab.comp_labels.push_back(labs[i]);
    }
  return ab;
}

// Slice-loop order for the prefix cache (a6): labels by the cost that depends on them (heaviest
// outermost), then adjacent swaps while the executed prefix-cache cost decreases.
std::vector<int> loop_order(const Tree& best_tree, const CostModel& cm, const std::vector<uint64_t>& mask,
                            const std::vector<int>& chosen, int n_leaves) {
  const int k = (int)chosen.size();
  const int W = best_tree.W;
  std::vector<int> order(k);
  struct { int W; } leaves{W};
  if (k > 0) {
    const int NN = (int)best_tree.nodes.size();
    std::vector<uint64_t> dep(NN, 0);  // S(v) over chosen positions (chosen index)
    std::vector<double> ncost(NN, 0);
    std::vector<int> po;
    postorder(best_tree, po);
    for (int i = 0; i < n_leaves; ++i)
      for (int c = 0; c < k; ++c)
        if (best_tree.L(i)[chosen[c] / 64] & (uint64_t(1) << (chosen[c] % 64))) dep[i] |= uint64_t(1) << c;
    for (int v : po) {
      const TNode& n = best_tree.nodes[v];
      dep[v] = dep[n.left] | dep[n.right];
      ncost[v] = cm.node_cost(pc_union_not(best_tree.L(n.left), best_tree.L(n.right), mask.data(), leaves.W),
                              pc_and_not(best_tree.L(n.left), mask.data(), leaves.W),
                              pc_and_not(best_tree.L(n.right), mask.data(), leaves.W),
                              pc_and_not(best_tree.L(v), mask.data(), leaves.W));
    }
    std::vector<double> wt(k, 0);
    for (int v : po)
      for (int c = 0; c < k; ++c)
        if (dep[v] & (uint64_t(1) << c)) wt[c] += ncost[v];
    for (int c = 0; c < k; ++c) order[c] = c;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return wt[a] > wt[b]; });
    auto prefix_cost = [&](const std::vector<int>& ord) {
      std::vector<int> pos(k);
      for (int p = 0; p < k; ++p) pos[ord[p]] = p;
      double tot = 0;
      for (int v : po) {
        int mp = -1;
        for (int c = 0; c < k; ++c)
          if (dep[v] & (uint64_t(1) << c)) mp = std::max(mp, pos[c]);
        tot += ncost[v] * cm.dpow[mp + 1];
      }
      return tot;
    };
    double cur = prefix_cost(order);
    for (bool improved = true; improved;) {
      improved = false;
      for (int p = 0; p + 1 < k; ++p) {
        std::swap(order[p], order[p + 1]);
        double c = prefix_cost(order);
        if (c < cur * (1 - 1e-12)) {
          cur = c;
          improved = true;
        } else {
          std::swap(order[p], order[p + 1]);
        }
      }
    }
  }
  return order;
}

}  // namespace

void greedy_plan(const jt_network& net0, const jt_planner_opts& o, std::vector<int64_t>& path,
                 std::vector<int64_t>& sliced) {
  // batch labels (open wires) are fixed in every run: plan on the network without them
  jt_network stripped;
  const jt_network* np = &net0;
  if (!net0.batch_labels.empty()) {
    stripped = net0;
    std::unordered_set<int64_t> bl(net0.batch_labels.begin(), net0.batch_labels.end());
    for (auto& t : stripped.tensors) {
      std::vector<int64_t> keep;
      for (int64_t l : t.labels)
        if (!bl.count(l)) keep.push_back(l);
      t.labels = keep;
    }
    np = &stripped;
  }
  const jt_network& net = *np;
  const int64_t nt = (int64_t)net.tensors.size();
  Absorbed ab = absorb(net);
  const int n_leaves = (int)ab.comp_ssa.size();
  // compact labels
  std::unordered_map<int64_t, int> cid;
  std::vector<int64_t> raw_of;
  for (auto& ls : ab.comp_labels)
    for (int64_t l : ls)
      if (!cid.count(l)) {
        cid[l] = (int)raw_of.size();
        raw_of.push_back(l);
      }
  const int NL = (int)raw_of.size();
  BitPool leaves;
  leaves.W = std::max(1, (NL + 63) / 64);
  std::vector<std::vector<int>> carriers(NL);
  for (int i = 0; i < n_leaves; ++i) {
    size_t k = leaves.add();
    for (int64_t l : ab.comp_labels[i]) {
      int c = cid[l];
      leaves.at(k)[c / 64] |= uint64_t(1) << (c % 64);
      carriers[c].push_back(i);
    }
  }
  CostModel cm;
  cm.log2d = std::log2((double)net.d);
  cm.R = o.bytes_weight > 0 ? o.bytes_weight : 0.0;
  if (o.model_hbm_gbs > 0) {
    cm.rf_bw = o.model_hbm_gbs * 1e9;
    cm.rf_cuda = o.model_cuda_tflops > 0 ? o.model_cuda_tflops * 1e12 : 40e12;
    cm.rf_tc = o.model_tc_tflops > 0 ? o.model_tc_tflops * 1e12 : 0.0;
    cm.rf_gap = o.model_launch_us * 1e-6;
    cm.esize = o.model_esize > 0 ? o.model_esize : 8;
    cm.qubits = net.d == 2;
  }
  cm.dpow.resize(NL + 2);
  for (int i = 0; i <= NL + 1; ++i) cm.dpow[i] = std::pow((double)net.d, (double)i);

  const int trials = o.trials > 0 ? o.trials : 64;
  int nthreads = o.threads > 0 ? o.threads : (int)std::thread::hardware_concurrency();
  nthreads = std::max(1, std::min(nthreads, trials));
  const int F = o.reconf_leaves > 0 ? std::min(o.reconf_leaves, 10) : 8;
  const int sweeps = o.reconf_sweeps >= 0 ? o.reconf_sweeps : 2;
  std::vector<uint64_t> nomask(leaves.W, 0);

  Tree best_tree;
  std::vector<uint64_t> mask(leaves.W, 0);
  std::vector<int> chosen;
  const int capw = o.width_cap > 0 ? (int)std::floor(o.width_cap / cm.log2d + 1e-9) : -1;
  if (n_leaves == 1) {
    best_tree = tree_from_pairs(leaves, 1, {});
  } else {
    // trials: greedy, then reconfiguration of each trial's tree; best by total cost
    std::vector<double> tcost(trials, std::numeric_limits<double>::infinity());
    std::vector<std::vector<std::pair<int, int>>> tpairs(trials);
    const double temps[4] = {0.1, 0.25, 0.5, 1.0};
    std::atomic<int> next{0};
    auto t0 = std::chrono::steady_clock::now();
    auto worker = [&]() {
      for (;;) {
        int i = next.fetch_add(1);
        if (i >= trials) break;
        if (o.time_budget_s > 0 && i >= nthreads) {
          double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          if (el > o.time_budget_s) break;
        }
        int variant = i % 2;
        double temp = (i < 2) ? 0.0 : temps[(i / 2) % 4];
        const uint64_t sd = o.seed * 0x9E3779B97F4A7C15ULL + (uint64_t)i;
        // opts.partition: 1 = every other trial, 2 = every trial by recursive bisection (f2)
        const bool part = o.partition == 2 || (o.partition == 1 && (i % 2) == 1);
        const double imbs[4] = {0.0, 0.2, 0.4, 0.6};
        GreedyResult g = part ? partition_once(leaves, n_leaves, cm, carriers, sd, imbs[(i / 2) % 4])
                              : greedy_once(leaves, n_leaves, cm, variant, temp, sd, carriers);
        tcost[i] = g.cost;
        tpairs[i] = std::move(g.pairs);
      }
    };
    {
      std::vector<std::thread> th;
      for (int t = 0; t < nthreads; ++t) th.emplace_back(worker);
      for (auto& t : th) t.join();
    }
    // the best few greedy trees (parallel): reconfigure, slice, reconfigure the sliced tree;
    // keep the candidate with the lowest sliced cost N_sl * sum_v cost(v)
    std::vector<int> idx;
    for (int i = 0; i < trials; ++i)
      if (std::isfinite(tcost[i])) idx.push_back(i);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return tcost[a] < tcost[b] || (tcost[a] == tcost[b] && a < b); });
    int nre = std::min<int>((int)idx.size(), std::max(o.candidates > 0 ? o.candidates : 8, 1));
    std::vector<Tree> trees(nre);
    std::vector<std::vector<int>> chosen_c(nre);
    std::vector<std::vector<uint64_t>> mask_c(nre);
    std::vector<double> rcost(nre);
    std::atomic<int> nx{0};
    auto rworker = [&]() {
      for (;;) {
        int i = nx.fetch_add(1);
        if (i >= nre) break;
        trees[i] = tree_from_pairs(leaves, n_leaves, tpairs[idx[i]]);
        reconf_sweeps(trees[i], sweeps, F, cm, nomask.data());
        mask_c[i].assign(leaves.W, 0);
        slice_tree(trees[i], cm, o.n_sliced, capw, sweeps, F, NL, mask_c[i], chosen_c[i], o.slice_objective);
        if (o.slice_objective == 1) {   // compare candidates by their executed (prefix-cache) cost
          std::vector<int> po;
          postorder(trees[i], po);
          const std::vector<int> ord = loop_order(trees[i], cm, mask_c[i], chosen_c[i], n_leaves);
          std::vector<int> labs;
          for (int c : ord) labs.push_back(chosen_c[i][c]);
          rcost[i] = prefix_tree_cost(trees[i], cm, mask_c[i].data(), labs, po);
        } else {
          rcost[i] = tree_cost(trees[i], cm, mask_c[i].data(), nullptr) * cm.dpow[chosen_c[i].size()];
        }
      }
    };
    {
      std::vector<std::thread> th;
      for (int t = 0; t < std::min(nthreads, nre); ++t) th.emplace_back(rworker);
      for (auto& t : th) t.join();
    }
    int bi = 0;
    for (int i = 1; i < nre; ++i)
      if (rcost[i] < rcost[bi]) bi = i;
    best_tree = std::move(trees[bi]);
    mask = mask_c[bi];
    chosen = chosen_c[bi];
  }

  // ---- slice loop order: heaviest dependent FLOP outermost, then adjacent-swap search
  const int k = (int)chosen.size();
  std::vector<int> order = loop_order(best_tree, cm, mask, chosen, n_leaves);
  sliced.clear();
  for (int p = 0; p < k; ++p) sliced.push_back(raw_of[chosen[order[p]]]);

  // ---- emit the SSA path over raw ids: absorption steps, then the tree in post-order
  path = ab.pre_path;
  int64_t next_id = nt + (int64_t)ab.pre_path.size() / 2;
  std::vector<int64_t> ssa(best_tree.nodes.size(), -1);
  for (int i = 0; i < n_leaves; ++i) ssa[i] = ab.comp_ssa[i];
  std::vector<int> po;
  if (n_leaves > 1) postorder(best_tree, po);
  for (int v : po) {
    path.push_back(ssa[best_tree.nodes[v].left]);
    path.push_back(ssa[best_tree.nodes[v].right]);
    ssa[v] = next_id++;
  }
}

// Greedy slicing along a fixed path (jt_plan_slice).  The path is over raw
// tensor ids (validated by the caller); no absorption and no reconfiguration: the tree is exactly
// the given one.
void slice_fixed_path(const jt_network& net0, const std::vector<int64_t>& path, const jt_planner_opts& o,
                      std::vector<int64_t>& sliced) {
  jt_network stripped;
  const jt_network* np = &net0;
  if (!net0.batch_labels.empty()) {
    stripped = net0;
    std::unordered_set<int64_t> bl(net0.batch_labels.begin(), net0.batch_labels.end());
    for (auto& t : stripped.tensors) {
      std::vector<int64_t> keep;
      for (int64_t l : t.labels)
        if (!bl.count(l)) keep.push_back(l);
      t.labels = keep;
    }
    np = &stripped;
  }
  const jt_network& net = *np;
  const int nt = (int)net.tensors.size();
  std::unordered_map<int64_t, int> cid;
  std::vector<int64_t> raw_of;
  for (const auto& t : net.tensors)
    for (int64_t l : t.labels)
      if (!cid.count(l)) {
        cid[l] = (int)raw_of.size();
        raw_of.push_back(l);
      }
  const int NL = (int)raw_of.size();
  BitPool leaves;
  leaves.W = std::max(1, (NL + 63) / 64);
  for (int i = 0; i < nt; ++i) {
    size_t k = leaves.add();
    for (int64_t l : net.tensors[i].labels) {
      const int c = cid[l];
      leaves.at(k)[c / 64] |= uint64_t(1) << (c % 64);
    }
  }
  std::vector<std::pair<int, int>> pairs;
  for (size_t q = 0; q + 1 < path.size(); q += 2) pairs.push_back({(int)path[q], (int)path[q + 1]});
  Tree T = tree_from_pairs(leaves, nt, pairs);
  CostModel cm;
  cm.log2d = std::log2((double)net.d);
  cm.R = o.bytes_weight > 0 ? o.bytes_weight : 0.0;
  cm.dpow.resize(NL + 2);
  for (int i = 0; i <= NL + 1; ++i) cm.dpow[i] = std::pow((double)net.d, (double)i);
  const int capw = o.width_cap > 0 ? (int)std::floor(o.width_cap / cm.log2d + 1e-9) : -1;
  std::vector<uint64_t> mask(leaves.W, 0);
  std::vector<int> chosen;
  slice_tree(T, cm, o.n_sliced, capw, 0, 8, NL, mask, chosen, o.slice_objective);
  const std::vector<int> order = loop_order(T, cm, mask, chosen, nt);
  sliced.clear();
  for (size_t p = 0; p < order.size(); ++p) sliced.push_back(raw_of[chosen[order[p]]]);
}

}  // namespace jt
