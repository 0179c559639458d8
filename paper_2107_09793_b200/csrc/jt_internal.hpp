// Internal host-side data structures of libjetb200 (not part of the ABI).
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/jetb200.h"

namespace jt {

struct Error : std::runtime_error {
  jt_status code;
  Error(jt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(jt_status code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& msg);

using cplx = std::complex<double>;

struct HostTensor {
  std::vector<int64_t> labels;  // axis order; row-major data, last label fastest
  std::vector<cplx> data;
};

}  // namespace jt

// kets, gate tensors, bras joined by shared labels.
struct jt_network {
  int32_t n_wires = 0;
  int32_t d = 2;
  std::vector<jt::HostTensor> tensors;
  std::vector<int64_t> cur;  // current open label of each wire
  int64_t n_labels = 0;
  int64_t n_gates = 0;
  bool closed = false;
  // batch of amplitudes: the bra of an open wire is the d x d
  // identity with labels (wire label, batch label); fixing the batch label to y gives <y|.
  std::vector<int64_t> batch_labels;  // one per open wire, in open-wire order
};

namespace jt {

// One node of the binary contraction tree (fig. contraction_tree_no_slice).
struct PlanNode {
  int64_t left = -1, right = -1, parent = -1;  // node ids; leaves have no children
  std::vector<int64_t> labels;                 // output labels, sliced labels removed
  uint64_t smask = 0;  // S(v): sliced positions carried by leaves under v
  int maxpos = -1;     // max position of S(v) in the loop order, -1 if S(v) = {}
  double flop = 0;     // 8 * prod of distinct dims of the step (sliced labels fixed)
  double log2size = 0; // log2 elements of the output
  double bytes8 = 0;   // algorithmic bytes of the step at 8 B/elem: |A|+|B|+|C|
};

}  // namespace jt

struct jt_plan {
  jt_network net;                       // closed network (copy, with leaf data)
  std::vector<int64_t> path;            // 2 * n_steps SSA ids
  std::vector<int64_t> sliced;          // loop labels, pos 0 outermost: the n_summed sliced
                                        // (summed) labels, then the network's batch labels
  int n_summed = 0;                     // sliced labels that are summed (user-visible k)
  int64_t n_batch = 1;                  // amplitudes per run = d^(batch labels)
  std::vector<jt::PlanNode> nodes;      // n_tensors leaves + n_steps internal; root = back()
  std::unordered_map<int64_t, int> slice_pos;
  int64_t n_sl = 1;                     // runs = N_sl (summed slices) x n_batch
};

namespace jt {

// plan.cpp
void build_plan_tree(jt_plan& plan);  // validates path/slices and fills nodes
jt_cost plan_cost(const jt_plan& plan);
double prefix_flop(const jt_plan& plan, int64_t begin, int64_t end);
// digits of slice index s in the loop order (pos 0 most significant)
void slice_digits(const jt_plan& plan, int64_t s, std::vector<int>& dig);

// planner.cpp
void greedy_plan(const jt_network& net, const jt_planner_opts& opts, std::vector<int64_t>& path,
                 std::vector<int64_t>& sliced);
void slice_fixed_path(const jt_network& net, const std::vector<int64_t>& path, const jt_planner_opts& opts,
                      std::vector<int64_t>& sliced);

}  // namespace jt
