// extern "C" boundary of libjetb200 (include/jetb200.h).  Every entry point converts
// exceptions into a jt_status and a thread-local message.
#include <cstring>
#include <string>

#include "jt_internal.hpp"

namespace jt {
jt_network* network_create(int32_t n_wires, int32_t d);
void network_add_gate(jt_network* net, int32_t k, const int32_t* wires, const double* u);
void network_close(jt_network* net, const int32_t* x, const int32_t* open_wires, int32_t n_open);
void network_export(const jt_network* net, const char* path);
void plan_export(const jt_plan* plan, const char* path);
int64_t workspace_bytes(const jt_plan& plan, jt_dtype dt);
void describe_exec(const jt_plan& plan, jt_dtype dt, const char* path);
void exec_memory(const jt_plan& plan, jt_dtype dt, jt_memory* out);
void debug_emulate_host(const jt_plan& plan, jt_dtype dt, int64_t b, int64_t e, double* h_vals, bool reuse);
jt_exec* exec_create(const jt_plan& plan, jt_dtype dt, int device, void* d_ws, int64_t ws_bytes, void* stream);
void exec_contract(jt_exec* ex, int64_t b, int64_t e, double* d_acc, double* h_vals, bool reuse);
void exec_contract_host(jt_exec* ex, int64_t b, int64_t e, double* h_acc);
void exec_invalidate(jt_exec* ex);
void debug_time_node(jt_exec* ex, int64_t idx, int reps, double* ms, double* bytes, double* flop, int* kind);
void exec_set_profiling(jt_exec* ex, bool on);
void upload_leaves(jt_exec* ex);
void exec_stats(const jt_exec* ex, jt_exec_stats* out);
void exec_stats_reset(jt_exec* ex);
void exec_destroy(jt_exec* ex);
void amplitude(const jt_plan& plan, jt_dtype dt, int device, double* out);
void permute(jt_dtype dt, const void* src, void* dst, int n, const int32_t* perm, void* stream);

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace jt

using namespace jt;

template <typename F>
static jt_status guarded(F&& f) {
  g_last_error.clear();
  try {
    f();
    return JT_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return JT_ERESOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return JT_EINTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return JT_EINTERNAL;
  }
}

#define NEED(p, name) \
  if (!(p)) fail(JT_EUSAGE, std::string(name) + ": null argument")

extern "C" {

const char* jt_last_error(void) { return g_last_error.c_str(); }
const char* jt_version(void) { return "jetb200 0.1 (sm_100a)"; }

jt_status jt_network_create(int32_t n_wires, int32_t d, jt_network** out) {
  return guarded([&] {
    NEED(out, "jt_network_create");
    *out = network_create(n_wires, d);
  });
}
jt_status jt_network_add_gate(jt_network* net, int32_t k, const int32_t* wires, const double* u) {
  return guarded([&] { network_add_gate(net, k, wires, u); });
}
jt_status jt_network_close(jt_network* net, const int32_t* x) {
  return guarded([&] { network_close(net, x, nullptr, 0); });
}
jt_status jt_network_close_batch(jt_network* net, const int32_t* x, const int32_t* open_wires, int32_t n_open) {
  return guarded([&] { network_close(net, x, open_wires, n_open); });
}
jt_status jt_network_info(const jt_network* net, int64_t* n_tensors, int64_t* n_labels) {
  return guarded([&] {
    NEED(net, "jt_network_info");
    if (n_tensors) *n_tensors = (int64_t)net->tensors.size();
    if (n_labels) *n_labels = net->n_labels;
  });
}
jt_status jt_network_export(const jt_network* net, const char* path) {
  return guarded([&] {
    NEED(net && path, "jt_network_export");
    network_export(net, path);
  });
}
void jt_network_destroy(jt_network* net) { delete net; }

jt_status jt_plan_create(const jt_network* net, const int64_t* ssa_path, int64_t n_steps,
                         const int64_t* sliced_labels, int32_t n_sliced, jt_plan** out) {
  return guarded([&] {
    NEED(net && out, "jt_plan_create");
    if (n_steps < 0 || n_sliced < 0) fail(JT_EUSAGE, "jt_plan_create: negative size");
    if (n_steps > 0) NEED(ssa_path, "jt_plan_create");
    if (n_sliced > 0) NEED(sliced_labels, "jt_plan_create");
    auto* p = new jt_plan();
    try {
      p->net = *net;
      p->path.assign(ssa_path, ssa_path + 2 * n_steps);
      p->sliced.assign(sliced_labels, sliced_labels + n_sliced);
      p->n_summed = n_sliced;
      p->sliced.insert(p->sliced.end(), net->batch_labels.begin(), net->batch_labels.end());
      build_plan_tree(*p);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

jt_status jt_plan_greedy(const jt_network* net, const jt_planner_opts* opts, jt_plan** out) {
  return guarded([&] {
    NEED(net && out, "jt_plan_greedy");
    if (!net->closed) fail(JT_EVALIDATION, "jt_plan_greedy: network is not closed");
    jt_planner_opts o{};
    if (opts) o = *opts;
    auto* p = new jt_plan();
    try {
      p->net = *net;
      greedy_plan(*net, o, p->path, p->sliced);
      p->n_summed = (int)p->sliced.size();
      p->sliced.insert(p->sliced.end(), net->batch_labels.begin(), net->batch_labels.end());
      build_plan_tree(*p);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

jt_status jt_plan_slice(const jt_network* net, const int64_t* ssa_path, int64_t n_steps, const jt_planner_opts* opts,
                        jt_plan** out) {
  return guarded([&] {
    NEED(net && out && opts, "jt_plan_slice");
    if (!net->closed) fail(JT_EVALIDATION, "jt_plan_slice: network is not closed");
    if (n_steps < 0) fail(JT_EUSAGE, "jt_plan_slice: negative size");
    if (n_steps > 0) NEED(ssa_path, "jt_plan_slice");
    auto* p = new jt_plan();
    try {
      p->net = *net;
      p->path.assign(ssa_path, ssa_path + 2 * n_steps);
      p->sliced.assign(net->batch_labels.begin(), net->batch_labels.end());
      p->n_summed = 0;
      build_plan_tree(*p);   // validates the path before the slicer walks it
      std::vector<int64_t> sl;
      slice_fixed_path(*net, p->path, *opts, sl);
      jt_plan* q = new jt_plan();
      q->net = *net;
      q->path = p->path;
      q->sliced = sl;
      q->n_summed = (int)sl.size();
      q->sliced.insert(q->sliced.end(), net->batch_labels.begin(), net->batch_labels.end());
      delete p;
      p = q;
      build_plan_tree(*p);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

jt_status jt_plan_sizes(const jt_plan* plan, int64_t* n_steps, int32_t* n_sliced) {
  return guarded([&] {
    NEED(plan, "jt_plan_sizes");
    if (n_steps) *n_steps = (int64_t)plan->path.size() / 2;
    if (n_sliced) *n_sliced = (int32_t)plan->n_summed;
  });
}
jt_status jt_plan_get(const jt_plan* plan, int64_t* ssa_path, int64_t* sliced_labels) {
  return guarded([&] {
    NEED(plan, "jt_plan_get");
    if (ssa_path) std::memcpy(ssa_path, plan->path.data(), plan->path.size() * sizeof(int64_t));
    if (sliced_labels) std::memcpy(sliced_labels, plan->sliced.data(), plan->n_summed * sizeof(int64_t));
  });
}
jt_status jt_plan_cost(const jt_plan* plan, jt_cost* out) {
  return guarded([&] {
    NEED(plan && out, "jt_plan_cost");
    *out = plan_cost(*plan);
  });
}
jt_status jt_plan_prefix_flop(const jt_plan* plan, int64_t begin, int64_t end, double* flop) {
  return guarded([&] {
    NEED(plan && flop, "jt_plan_prefix_flop");
    if (begin < 0 || end > plan->n_sl || begin > end) fail(JT_EUSAGE, "jt_plan_prefix_flop: bad range");
    *flop = prefix_flop(*plan, begin, end);
  });
}
jt_status jt_plan_export(const jt_plan* plan, const char* path) {
  return guarded([&] {
    NEED(plan && path, "jt_plan_export");
    plan_export(plan, path);
  });
}
void jt_plan_destroy(jt_plan* plan) { delete plan; }

jt_status jt_exec_workspace_bytes(const jt_plan* plan, jt_dtype dtype, int64_t* bytes) {
  return guarded([&] {
    NEED(plan && bytes, "jt_exec_workspace_bytes");
    *bytes = workspace_bytes(*plan, dtype);
  });
}
jt_status jt_exec_memory(const jt_plan* plan, jt_dtype dtype, jt_memory* out) {
  return guarded([&] {
    NEED(plan && out, "jt_exec_memory");
    exec_memory(*plan, dtype, out);
  });
}
jt_status jt_exec_describe(const jt_plan* plan, jt_dtype dtype, const char* path) {
  return guarded([&] {
    NEED(plan && path, "jt_exec_describe");
    describe_exec(*plan, dtype, path);
  });
}
jt_status jt_exec_create(const jt_plan* plan, jt_dtype dtype, int32_t device, void* d_ws, int64_t ws_bytes,
                         void* cuda_stream, jt_exec** out) {
  return guarded([&] {
    NEED(plan && out, "jt_exec_create");
    *out = exec_create(*plan, dtype, device, d_ws, ws_bytes, cuda_stream);
  });
}
jt_status jt_exec_contract(jt_exec* ex, int64_t b, int64_t e, double* d_acc, double* h_vals) {
  return guarded([&] {
    NEED(ex, "jt_exec_contract");
    exec_contract(ex, b, e, d_acc, h_vals, true);
  });
}
jt_status jt_exec_contract_noreuse(jt_exec* ex, int64_t b, int64_t e, double* d_acc, double* h_vals) {
  return guarded([&] {
    NEED(ex, "jt_exec_contract_noreuse");
    exec_contract(ex, b, e, d_acc, h_vals, false);
  });
}
jt_status jt_exec_contract_host(jt_exec* ex, int64_t b, int64_t e, double* h_acc) {
  return guarded([&] {
    NEED(ex && h_acc, "jt_exec_contract_host");
    exec_contract_host(ex, b, e, h_acc);
  });
}
jt_status jt_exec_upload_leaves(jt_exec* ex) {
  return guarded([&] {
    NEED(ex, "jt_exec_upload_leaves");
    upload_leaves(ex);
  });
}
jt_status jt_exec_set_profiling(jt_exec* ex, int32_t on) {
  return guarded([&] {
    NEED(ex, "jt_exec_set_profiling");
    exec_set_profiling(ex, on != 0);
  });
}
jt_status jt_exec_stats_get(const jt_exec* ex, jt_exec_stats* out) {
  return guarded([&] {
    NEED(ex && out, "jt_exec_stats_get");
    exec_stats(ex, out);
  });
}
jt_status jt_exec_stats_reset(jt_exec* ex) {
  return guarded([&] {
    NEED(ex, "jt_exec_stats_reset");
    exec_stats_reset(ex);
  });
}
jt_status jt_exec_invalidate(jt_exec* ex) {
  return guarded([&] {
    NEED(ex, "jt_exec_invalidate");
    exec_invalidate(ex);
  });
}
void jt_exec_destroy(jt_exec* ex) { exec_destroy(ex); }

jt_status jt_debug_emulate_host(const jt_plan* plan, jt_dtype dtype, int64_t b, int64_t e, double* h_vals,
                                int32_t reuse) {
  return guarded([&] {
    NEED(plan && (h_vals || b == e), "jt_debug_emulate_host");
    debug_emulate_host(*plan, dtype, b, e, h_vals, reuse != 0);
  });
}

jt_status jt_debug_time_node(jt_exec* ex, int64_t order_index, int32_t reps, double* ms, double* bytes,
                             double* flop, int32_t* kind) {
  return guarded([&] {
    NEED(ex && ms && bytes && flop && kind, "jt_debug_time_node");
    debug_time_node(ex, order_index, reps, ms, bytes, flop, kind);
  });
}

jt_status jt_amplitude(const jt_plan* plan, jt_dtype dtype, int32_t device, double* out) {
  return guarded([&] {
    NEED(plan && out, "jt_amplitude");
    amplitude(*plan, dtype, device, out);
  });
}

jt_status jt_permute(jt_dtype dtype, const void* d_src, void* d_dst, int32_t n_bits, const int32_t* perm,
                     void* cuda_stream) {
  return guarded([&] {
    NEED(d_src && d_dst && (perm || n_bits == 0), "jt_permute");
    if (dtype != JT_C64 && dtype != JT_C128) fail(JT_EUSAGE, "jt_permute: bad dtype");
    permute(dtype, d_src, d_dst, n_bits, perm, cuda_stream);
  });
}

}  // extern "C"
