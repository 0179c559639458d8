// Contraction tree, slicing semantics and cost counters of a plan.
//   tree:    PAPER.md l.94-115 (Eq. sequence, binary contraction tree)
//   slicing: l.116-139 (Eq. sliced_sum, fig. contraction_tree_slice_e)
//   costs:   l.140-146 (Eq. sliced_flops), l.205-212 (Eq. task_based_amplitude_flops)
#include <algorithm>
#include <cmath>
#include <fstream>
#include <unordered_set>

#include "jt_internal.hpp"

namespace jt {

void build_plan_tree(jt_plan& plan) {
  const jt_network& net = plan.net;
  if (!net.closed) fail(JT_EVALIDATION, "plan: network is not closed");
  const int64_t nt = (int64_t)net.tensors.size();
  const int64_t ns = (int64_t)plan.path.size() / 2;
  if ((int64_t)plan.path.size() != 2 * ns) fail(JT_EUSAGE, "plan: odd path length");
  if (ns != nt - 1) fail(JT_EVALIDATION, "plan: path must have n_tensors - 1 steps");
  // bonds: every label on exactly two tensors (closed network)
  std::unordered_map<int64_t, int> carriers;
  for (const auto& t : net.tensors)
    for (int64_t l : t.labels) carriers[l]++;
  // batch labels sit on exactly one tensor and are fixed in every run
  std::unordered_set<int64_t> batch(net.batch_labels.begin(), net.batch_labels.end());
  for (auto& kv : carriers)
    if (kv.second != (batch.count(kv.first) ? 1 : 2))
      fail(JT_EVALIDATION, "plan: label " + std::to_string(kv.first) + " is not a bond");
  if (plan.n_summed < 0 || plan.n_summed + net.batch_labels.size() != plan.sliced.size())
    fail(JT_EINTERNAL, "plan: loop labels != sliced + batch labels");
  plan.slice_pos.clear();
  for (size_t p = 0; p < plan.sliced.size(); ++p) {
    int64_t l = plan.sliced[p];
    const bool is_batch = (int)p >= plan.n_summed;
    if (!carriers.count(l) || (batch.count(l) != 0) != is_batch)
      fail(JT_EVALIDATION, "plan: sliced label " + std::to_string(l) + " is not a bond");
    if (plan.slice_pos.count(l)) fail(JT_EVALIDATION, "plan: duplicate sliced label");
    plan.slice_pos[l] = (int)p;
  }
  if (plan.sliced.size() > 62) fail(JT_EUSAGE, "plan: at most 62 sliced labels");
  const double log2d = std::log2((double)net.d);
  plan.n_sl = 1;
  plan.n_batch = 1;
  for (size_t p = 0; p < plan.sliced.size(); ++p) {
    if (plan.n_sl > (int64_t(1) << 62) / net.d) fail(JT_EUSAGE, "plan: too many slices");
    plan.n_sl *= net.d;
    if ((int)p >= plan.n_summed) plan.n_batch *= net.d;
  }
  plan.nodes.assign(nt + ns, PlanNode());
  for (int64_t t = 0; t < nt; ++t) {
    PlanNode& n = plan.nodes[t];
    for (int64_t l : net.tensors[t].labels) {
      auto it = plan.slice_pos.find(l);
      if (it == plan.slice_pos.end()) n.labels.push_back(l);
      else n.smask |= (uint64_t(1) << it->second);
    }
    n.log2size = log2d * (double)n.labels.size();
  }
  std::vector<char> live(nt + ns, 0);
  for (int64_t t = 0; t < nt; ++t) live[t] = 1;
  for (int64_t s = 0; s < ns; ++s) {
    int64_t a = plan.path[2 * s], b = plan.path[2 * s + 1];
    if (a < 0 || b < 0 || a >= nt + s || b >= nt + s || a == b || !live[a] || !live[b])
      fail(JT_EVALIDATION, "plan: step " + std::to_string(s) + " uses a dead or unknown id");
    live[a] = live[b] = 0;
    const int64_t v = nt + s;
    live[v] = 1;
    PlanNode& n = plan.nodes[v];
    PlanNode& A = plan.nodes[a];
    PlanNode& B = plan.nodes[b];
    n.left = a;
    n.right = b;
    A.parent = v;
    B.parent = v;
    std::unordered_set<int64_t> sb(B.labels.begin(), B.labels.end()), sa(A.labels.begin(), A.labels.end());
    size_t n_union = A.labels.size();
    for (int64_t l : A.labels)
      if (!sb.count(l)) n.labels.push_back(l);
    for (int64_t l : B.labels) {
      if (!sa.count(l)) {
        n.labels.push_back(l);
        n_union++;
      }
    }
    n.smask = A.smask | B.smask;
    n.flop = 8.0 * std::pow((double)net.d, (double)n_union);
    n.log2size = log2d * (double)n.labels.size();
    n.bytes8 = 8.0 * (std::exp2(A.log2size) + std::exp2(B.log2size) + std::exp2(n.log2size));
  }
  if (!plan.nodes.back().labels.empty()) fail(JT_EVALIDATION, "plan: root is not a scalar");
  for (auto& n : plan.nodes) {
    n.maxpos = -1;
    for (int p = 0; p < 64; ++p)
      if (n.smask & (uint64_t(1) << p)) n.maxpos = p;
  }
}

jt_cost plan_cost(const jt_plan& plan) {
  jt_cost c{};
  const int64_t nt = (int64_t)plan.net.tensors.size();
  c.n_sl = plan.n_sl / plan.n_batch;
  c.n_batch = plan.n_batch;
  c.n_sliced = (int32_t)plan.n_summed;
  c.n_steps = (int64_t)plan.path.size() / 2;
  const double d = plan.net.d;
  for (int64_t v = nt; v < (int64_t)plan.nodes.size(); ++v) {
    const PlanNode& n = plan.nodes[v];
    c.flop_sl += n.flop;
    if (!n.smask) c.flop_shared += n.flop;
    c.exact_reuse += n.flop * std::pow(d, (double)__builtin_popcountll(n.smask));
    c.prefix += n.flop * std::pow(d, (double)(n.maxpos + 1));
    c.max_width = std::max(c.max_width, n.log2size);
    c.bytes_sl += n.bytes8;
  }
  // per batch of amplitudes: every (slice, bitstring) run is one contraction of the multi-contraction
  c.e_flsl = (double)plan.n_sl * c.flop_sl;
  c.e_fltask = c.flop_shared + (double)plan.n_sl * (c.flop_sl - c.flop_shared);
  return c;
}

void slice_digits(const jt_plan& plan, int64_t s, std::vector<int>& dig) {
  const int k = (int)plan.sliced.size();
  dig.assign(k, 0);
  for (int p = k - 1; p >= 0; --p) {
    dig[p] = (int)(s % plan.net.d);
    s /= plan.net.d;
  }
}

double prefix_flop(const jt_plan& plan, int64_t begin, int64_t end) {
  const int64_t nt = (int64_t)plan.net.tensors.size();
  const int k = (int)plan.sliced.size();
  std::vector<double> F(k + 1, 0.0);  // F[j+1] = FLOP of nodes with maxpos >= j
  for (int64_t v = nt; v < (int64_t)plan.nodes.size(); ++v)
    for (int j = -1; j <= plan.nodes[v].maxpos; ++j) F[j + 1] += plan.nodes[v].flop;
  // slice s > begin recomputes the nodes with maxpos >= j, j = k-1-t where t = the number of
  // trailing zero base-d digits of s (the digits that rolled over); count the slices of
  // (begin, end) by t in closed form (multiples of d^t minus multiples of d^(t+1))
  const int64_t d = plan.net.d;
  if (end <= begin) return 0.0;
  double total = F[0];  // the first slice of the range: everything (j = -1)
  auto multiples = [&](int t) -> int64_t {  // multiples of d^t in [begin+1, end-1]
    int64_t q = 1;
    for (int i = 0; i < t; ++i) {
      if (q > (end - 1) / d) return 0;
      q *= d;
    }
    return (end - 1) / q - begin / q;
  };
  for (int t = 0; t <= k; ++t) {
    const int64_t cnt = t == k ? multiples(t) : multiples(t) - multiples(t + 1);
    const int j = std::max(-1, k - 1 - t);
    total += (double)cnt * F[j + 1];
  }
  return total;
}

}  // namespace jt

using namespace jt;

namespace jt {
void plan_export(const jt_plan* plan, const char* path) {
  std::ofstream f(path);
  if (!f) fail(JT_EUSAGE, std::string("cannot open ") + path);
  f << "{\"n_tensors\": " << plan->net.tensors.size() << ", \"n_wires\": " << plan->net.n_wires
    << ", \"d\": " << plan->net.d << ", \"ssa_path\": [";
  for (size_t s = 0; s < plan->path.size() / 2; ++s)
    f << (s ? ", " : "") << "[" << plan->path[2 * s] << ", " << plan->path[2 * s + 1] << "]";
  f << "], \"sliced_labels\": [";
  for (int p = 0; p < plan->n_summed; ++p) f << (p ? ", " : "") << plan->sliced[p];
  f << "], \"batch_labels\": [";
  for (size_t p = plan->n_summed; p < plan->sliced.size(); ++p) f << (p > (size_t)plan->n_summed ? ", " : "") << plan->sliced[p];
  f << "]}\n";
}
}  // namespace jt
