/*
 * libjetb200 -- C ABI of the B200-native Jet hot path (arXiv 2107.09793).
 *
 * The calls follow the paper's problem statement:
 *   build a network from gates and a bitstring      PAPER.md l.72-85  (Sec. II.B.1)
 *   take a contraction path and a set of sliced indices
 *                                                   l.94-105 (Eq. sequence), l.116-133 (Eq. sliced_sum), l.176
 *   return the amplitude(s)                         l.83-85  (<a|U|0>)
 *
 * Conventions
 *   - Every call returns jt_status; nothing throws across the ABI.  On a non-zero
 *     status, jt_last_error() returns a thread-local message valid until the next
 *     jt_* call on that thread.  Codes: 0 OK, 2 usage (bad argument),
 *     3 validation (bad network / path / slices), 4 resource (device OOM, workspace
 *     too small, width over cap), 5 CUDA error, 6 internal.
 *   - Host inputs are copied; handles are opaque and freed by *_destroy.
 *   - Device memory and CUDA streams belong to the caller (PyTorch in the Python
 *     binding): the library never allocates device memory except in the
 *     self-contained convenience call jt_amplitude.
 *   - Complex numbers are interleaved (re, im) pairs of double (host) or of the
 *     execution dtype (device).
 *
 * Id conventions (shared by definition with the oracle):
 *   tensors: 0..n-1 = the |0> ket of wires 0..n-1 (l.81), then one tensor per gate in
 *            the order added, then (after jt_network_close) the bra of wire 0..n-1 (l.83).
 *   labels:  0..n-1 = the ket legs; then every gate creates one new label per wire, in
 *            the order of its `wires` argument ("w.k" scheme, numbered).
 *   A k-qudit gate tensor has labels (out_0..out_{k-1}, in_0..in_{k-1}) and data
 *   U[out][in] row-major, wires[0] most significant (reading A7, P:81 B_cfbe).
 *   SSA path: step s consumes ids (p[2s], p[2s+1]) and creates id n_tensors + s.
 *   Slice index <-> assignment: lexicographic, sliced_labels[0] most significant
 *   (reading A12); the same order is the prefix-cache loop order.
 */
#ifndef JETB200_H
#define JETB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t jt_status;
enum { JT_OK = 0, JT_EUSAGE = 2, JT_EVALIDATION = 3, JT_ERESOURCE = 4, JT_ECUDA = 5, JT_EINTERNAL = 6 };

typedef enum { JT_C64 = 0, JT_C128 = 1 } jt_dtype;

typedef struct jt_network jt_network;
typedef struct jt_plan jt_plan;
typedef struct jt_exec jt_exec;

/* Host planner options.  Zero-initialise and set what you need. */
typedef struct {
  uint64_t seed;          /* deterministic given the seed */
  int32_t trials;         /* greedy trials (randomised); <=0 -> 64 */
  int32_t threads;        /* host threads; <=0 -> hardware concurrency */
  int32_t n_sliced;       /* number of sliced labels k (N_sl = d^k); -1 -> slice until width <= width_cap */
  int32_t width_cap;      /* max intermediate size in log2(elements) after slicing; <=0 -> no cap */
  int32_t reconf_sweeps;  /* subtree-reconfiguration sweeps; <0 -> default 2 */
  int32_t reconf_leaves;  /* frontier size of the subset DP, <=10; <=0 -> 8 */
  double time_budget_s;   /* soft wall-clock budget for the greedy trials; <=0 -> none */
  double bytes_weight;    /* roofline objective: node cost = max(d^union, w (|A|+|B|+|C|)) with
                             w = peak FLOP/s * esize / (8 * HBM B/s); <=0 -> pure FLOP (d^union) */
  int32_t candidates;     /* greedy trees carried through reconfiguration + slicing; <=0 -> 8 */
  /* kernel-aware roofline objective (used when model_hbm_gbs > 0, overrides bytes_weight):
     node time = max(FLOP / rate, bytes / HBM) + launch gap, with rate = model_tc_tflops for
     contractions K3 can run and model_cuda_tflops otherwise */
  double model_hbm_gbs;
  double model_cuda_tflops;
  double model_tc_tflops;
  double model_launch_us;
  double model_esize;     /* bytes per element (8 = c64, 16 = c128) */
  /* slice selection objective ("we greedily selected our slices
     along a fixed contraction path to maximize shared work"): 0 -> sliced cost N_sl sum_v c(v);
     1 -> shared-work aware: the executed cost of the one-copy prefix cache,
     sum_v c(v) prod_{pos(l) <= maxpos(S(v))} d_l, with the candidate appended innermost */
  int32_t slice_objective;
  /* trial generator ("better path"): 0 = randomised greedy only; 1 = every other
     trial a recursive graph bisection (few labels between the parts, Fiduccia-Mattheyses, random
     balance band; PAPER.md l.176 uses hypergraph partitioning); 2 = every trial by bisection.
     Each trial's tree then goes through the same reconfiguration and slicing. */
  int32_t partition;
} jt_planner_opts;

/* Cost counters (PAPER.md l.140-146 Eq. sliced_flops, l.205-212 Eq. task_based;
   FLOP convention: 8 real FLOP x prod(distinct dims) per pairwise step, reading A11). */
typedef struct {
  int64_t n_sl;            /* N_sl = prod of sliced (summed) dims, per amplitude */
  double flop_sl;          /* FLOP of one slice */
  double flop_shared;      /* FLOP of nodes with S(v) = {} (f_sl = flop_shared / flop_sl) */
  double e_flsl;           /* N_sl * FLOP_sl */
  double e_fltask;         /* f_sl FLOP_sl + N_sl (1 - f_sl) FLOP_sl */
  double exact_reuse;      /* sum_v flop_v prod_{l in S(v)} d_l  (dedup by task name) */
  double prefix;           /* executed FLOP of the one-copy prefix cache over all slices */
  double max_width;        /* log2 elements of the largest intermediate of one slice */
  double bytes_sl;         /* algorithmic bytes of one slice at 8 B/elem: sum_v (|A|+|B|+|C|) */
  int64_t n_steps;         /* SSA path length */
  int32_t n_sliced;
  int64_t n_batch;         /* amplitudes per run (d^open wires, jt_network_close_batch); 1 otherwise.
                              e_flsl / e_fltask / exact_reuse / prefix count all n_sl x n_batch
                              contractions of the multi-contraction */
} jt_cost;

/* Execution statistics accumulated by jt_exec_contract. */
typedef struct {
  int64_t slices_done;
  int64_t node_launches;   /* contraction nodes executed */
  int64_t kernel_launches; /* every kernel launched (contractions, reductions, accumulate) */
  double flop_executed;    /* algorithmic FLOP of the executed nodes (compare with jt_cost.prefix) */
  double bytes_executed;   /* algorithmic bytes of the executed nodes, at the exec dtype size */
  /* filled only while profiling is on (jt_exec_set_profiling): CUDA-event time of every
     contraction launch (K2 or K3) on the exec stream, and the algorithmic bytes/FLOP of those
     launches */
  double k2_time_ms;
  int64_t k2_timed_launches;
  double k2_timed_bytes;
  double k2_timed_flop;
  double k3_time_ms;          /* ... the subset of those launches that ran on K3 (tcgen05) */
  int64_t k3_timed_launches;
  double k3_timed_bytes;
  double k3_timed_flop;
  int64_t h2d_bytes;       /* host->device bytes copied by jt_exec_create / jt_exec_upload_leaves */
  double k4_time_ms;          /* ... the subset of the timed launches that ran on K4 (c128 DMMA) */
  int64_t k4_timed_launches;
  double k4_timed_bytes;
  double k4_timed_flop;
  double k3g_time_ms;         /* ... the subset of the K3 launches that ran on K3g (both operands
                                 streamed; the tensor-bound GEMM-shaped nodes) */
  int64_t k3g_timed_launches;
  double k3g_timed_bytes;
  double k3g_timed_flop;
  double k2s_time_ms;         /* ... the subset of the timed launches that ran on K2s (streaming
                                 GETT for skinny c64 nodes, small operand in registers; not
                                 counted under K3) */
  int64_t k2s_timed_launches;
  double k2s_timed_bytes;
  double k2s_timed_flop;
} jt_exec_stats;

const char* jt_last_error(void);
const char* jt_version(void);

/* ---- network ----------------------------------------------------- */
/* n_wires >= 1, d >= 2.  Every wire starts in |0> (l.53, l.81). */
jt_status jt_network_create(int32_t n_wires, int32_t d, jt_network** out);
/* k in {1,2}; wires[k] distinct in [0,n_wires); u: d^k x d^k complex, row-major U[out][in],
   interleaved (re,im) doubles, wires[0] most significant; copied.  Error 3 after close. */
jt_status jt_network_add_gate(jt_network* net, int32_t k, const int32_t* wires, const double* u);
/* Attach <x_w| to every wire (l.83); x: n_wires digits in [0,d); copied; once. */
jt_status jt_network_close(jt_network* net, const int32_t* x);
/* Batch of amplitudes ("computing batches of amplitudes" as a
   multi-contraction with shared work).  Like jt_network_close, but every wire in
   open_wires[0..n_open) gets the d x d identity with labels (wire label, batch label) in
   place of its bra; the batch labels are new labels n_labels.. n_labels+n_open-1 in
   open-wire order and sit on that one tensor.  A plan of this network loops over
   (summed slice, batch digits) with the batch labels innermost; fixing batch label i to y_i
   turns the identity into <y_i|, so run r = sigma * n_batch + y computes s_sigma of the
   amplitude <x with x[open_wires[i]] = y_i|U|0>, y mixed radix with open_wires[0] most
   significant.  The prefix cache then recomputes only the nodes that depend on the batch
   digits (the bra-attached subtrees) per bitstring.  x digits of open wires are ignored.
   Errors: 2 for a repeated or out-of-range open wire. */
jt_status jt_network_close_batch(jt_network* net, const int32_t* x, const int32_t* open_wires, int32_t n_open);
/* Counts of the raw network (kets + gates + bras) and labels. */
jt_status jt_network_info(const jt_network* net, int64_t* n_tensors, int64_t* n_labels);
/* Neutral JSON file: wires, d, per tensor its labels and its data (row-major over those labels,
   interleaved re, im, 17 significant digits).  Tests compare it element by element with the
   oracle's own network build (row a1); the oracle never reads it as an input. */
jt_status jt_network_export(const jt_network* net, const char* path);
void jt_network_destroy(jt_network* net);

/* ---- plan (path + slices) ------------------------------- */
/* ssa_path: 2*n_steps ids; sliced_labels: n_sliced bond labels in loop order.  The network
   must be closed.  Validation (error 3): ids consumed once, one tensor left, sliced labels
   are bonds, no duplicates.  Batch labels of the network are appended to the loop order
   (innermost) automatically and are not listed by jt_plan_get. */
jt_status jt_plan_create(const jt_network* net, const int64_t* ssa_path, int64_t n_steps,
                         const int64_t* sliced_labels, int32_t n_sliced, jt_plan** out);
/* Host greedy planner: absorption of rank<=2 tensors, randomised greedy, subtree
   reconfiguration, greedy slicing, slice-loop order. */
jt_status jt_plan_greedy(const jt_network* net, const jt_planner_opts* opts, jt_plan** out);
/* Greedy slicing along a FIXED contraction path: the path is kept as given
   (same validation as jt_plan_create), labels are sliced one at a time by opts->slice_objective
   until opts->n_sliced labels or the width is <= opts->width_cap (in log2 elements), and the
   slice-loop order is chosen as in jt_plan_greedy.  trials / reconfiguration fields are ignored. */
jt_status jt_plan_slice(const jt_network* net, const int64_t* ssa_path, int64_t n_steps,
                        const jt_planner_opts* opts, jt_plan** out);
/* Sizes for jt_plan_get. */
jt_status jt_plan_sizes(const jt_plan* plan, int64_t* n_steps, int32_t* n_sliced);
/* Caller-sized buffers: ssa_path[2*n_steps], sliced_labels[n_sliced]. */
jt_status jt_plan_get(const jt_plan* plan, int64_t* ssa_path, int64_t* sliced_labels);
jt_status jt_plan_cost(const jt_plan* plan, jt_cost* out);
/* Prefix-cache FLOP of the slice range [begin,end) starting with a cold cache. */
jt_status jt_plan_prefix_flop(const jt_plan* plan, int64_t begin, int64_t end, double* flop);
/* Neutral JSON plan file (n_tensors, ssa_path, sliced_labels) for the oracle. */
jt_status jt_plan_export(const jt_plan* plan, const char* path);
void jt_plan_destroy(jt_plan* plan);

/* ---- execution on one B200 (the hot path) ----------------------------------------- */
/* Device workspace bytes for this plan and dtype (leaves + intermediates with lifetime
   reuse + prefix cache + split-K scratch + slice values). */
jt_status jt_exec_workspace_bytes(const jt_plan* plan, jt_dtype dtype, int64_t* bytes);
/* Memory report of the compiled plan (host only, fig. m10_memory: peak memory
   with and without deletion of intermediates, and the extra memory that shared work costs).
   All in bytes of the exec dtype.  Intermediates are deleted after their last use: the arena
   places every node output by first fit over its live interval in the execution order, so
   peak_live_bytes <= arena_bytes <= no_deletion_bytes.  A caller that wants several slice
   subsets in flight on one device can size them a priori: each extra executor needs
   total_bytes - leaf_bytes more (leaves can be shared read-only). */
typedef struct {
  int64_t total_bytes;             /* = jt_exec_workspace_bytes */
  int64_t leaf_bytes;              /* network leaves (full, unsliced data) */
  int64_t arena_bytes;             /* intermediates as placed (with deletion) */
  int64_t peak_live_bytes;         /* max over execution positions of the live intermediates */
  int64_t no_deletion_bytes;       /* every intermediate kept ("without deletion") */
  int64_t cache_bytes;             /* prefix-cache entries resident for the whole run (shared work) */
  int64_t peak_live_noshare_bytes; /* peak live if nothing were kept across slices (no shared work) */
  int64_t scratch_bytes;           /* split-K partial buffers */
} jt_memory;
jt_status jt_exec_memory(const jt_plan* plan, jt_dtype dtype, jt_memory* out);
/* Host only: write the compiled per-node launch plan (tiles, grid, split-K, bytes, FLOP,
   prefix-cache level) and the workspace layout as JSON (for analysis and DESIGN.md). */
jt_status jt_exec_describe(const jt_plan* plan, jt_dtype dtype, const char* path);
/* Caller owns d_ws (>= workspace bytes, 256-B aligned) and the stream (cudaStream_t or
   NULL for the legacy stream).  Uploads the leaves (H2D on the stream).  Error 4 if
   ws_bytes is too small; error 2 if d is not a power of two. */
jt_status jt_exec_create(const jt_plan* plan, jt_dtype dtype, int32_t device, void* d_ws,
                         int64_t ws_bytes, void* cuda_stream, jt_exec** out);
/* Contract slices [slice_begin, slice_end) in canonical order with the prefix cache,
   adding sum s_sigma into d_acc (device complex128, 2 doubles) in order -- async on the
   stream.  If h_slice_vals is non-NULL the call synchronises the stream and writes
   (end-begin) complex128 values s_sigma there (at most min(N_sl, 2^20) per call, else
   error 2).  The cache persists across calls.
   Batch plans (jt_network_close_batch): the index runs over N_sl x n_batch runs
   r = sigma * n_batch + y and d_acc holds n_batch complex128 (2 * n_batch doubles);
   run r adds into d_acc[2y], d_acc[2y+1]. */
jt_status jt_exec_contract(jt_exec* ex, int64_t slice_begin, int64_t slice_end, double* d_acc,
                           double* h_slice_vals);
/* Same with the prefix cache disabled: every node is recomputed for every slice (E-flsl). */
jt_status jt_exec_contract_noreuse(jt_exec* ex, int64_t slice_begin, int64_t slice_end,
                                   double* d_acc, double* h_slice_vals);
/* Host-buffer path: copies nothing else; equals jt_exec_contract + D2H of the sum.  h_acc
   receives the complex128 sum of the range (synchronous); n_batch complex128 for batch plans. */
jt_status jt_exec_contract_host(jt_exec* ex, int64_t slice_begin, int64_t slice_end, double* h_acc);
/* Re-upload the leaf tensors (the network data) from host memory through a pinned staging
   buffer, H2D on the stream (the per-step input copy of the end-to-end path). */
jt_status jt_exec_upload_leaves(jt_exec* ex);
/* Profiling: bracket every contraction launch (K2/K3/K3g/K4) with CUDA events on the exec stream; each
   jt_exec_contract call then synchronises and adds the event times to the stats. */
jt_status jt_exec_set_profiling(jt_exec* ex, int32_t on);
jt_status jt_exec_stats_get(const jt_exec* ex, jt_exec_stats* out);
jt_status jt_exec_stats_reset(jt_exec* ex);
/* Drop the prefix cache (next call recomputes everything). */
jt_status jt_exec_invalidate(jt_exec* ex);
void jt_exec_destroy(jt_exec* ex);

/* 1-GPU convenience, synchronous: allocates its own workspace. out = (re, im); for batch
   plans out holds n_batch complex128 amplitudes (2 * n_batch doubles), y-indexed. */
jt_status jt_amplitude(const jt_plan* plan, jt_dtype dtype, int32_t device, double* out);

/* TEST ONLY (never called by jt_exec_*): execute the compiled K2 descriptors, workspace
   layout and prefix-cache schedule for slices [b,e) on the host with the kernels' index
   arithmetic, writing s_sigma to h_vals (2*(e-b) doubles).  Lets CPU tests check the plan
   compiler and the scheduler against the oracle without a GPU; tiny plans only. */
jt_status jt_debug_emulate_host(const jt_plan* plan, jt_dtype dtype, int64_t b, int64_t e, double* h_vals,
                                int32_t reuse);

/* DEBUG ONLY: time `reps` back-to-back launches of the node at execution-order index
   `order_index` (CUDA events on the exec stream; inputs as currently in the workspace).
   Returns the mean ms per launch, the node's algorithmic bytes and FLOP, and its kernel kind
   (0 K2, 1 K3, 2 K3g, 3 K4).  For kernel tuning on real plan shapes. */
jt_status jt_debug_time_node(jt_exec* ex, int64_t order_index, int32_t reps, double* ms, double* bytes,
                             double* flop, int32_t* kind);

/* ---- K1 index permutation ("two (partial) tensor transposes") ------- */
/* dst[pi(i)] = src[i] for a tensor of 2^n_bits elements of the dtype, where the address
   bit b of src moves to bit perm[b] of dst (perm is a permutation of 0..n_bits-1).
   Device pointers, async on the stream; src and dst must not overlap. */
jt_status jt_permute(jt_dtype dtype, const void* d_src, void* d_dst, int32_t n_bits,
                     const int32_t* perm, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* JETB200_H */
