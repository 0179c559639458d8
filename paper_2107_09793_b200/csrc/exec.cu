// Slice executor: compiles a plan into per-node K2 launch
// descriptors (bit layouts, tiles, workspace offsets) and runs the sliced contraction with
// the one-copy prefix cache -- the paper's shared-work reuse: a node
// v depends only on the slice digits of S(v); with slices in lexicographic order, v is
// recomputed only when a digit at a position <= maxpos(S(v)) changes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>

#include "jt_internal.hpp"
#include "kernels.cuh"
#include "kernels_tc.cuh"
#include "kernels_tcg.cuh"
#include "kernels_dmma.cuh"
#include "kernels_stream.cuh"

#define JT_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      ::jt::fail(e_ == cudaErrorMemoryAllocation ? JT_ERESOURCE : JT_ECUDA,               \
                 std::string(#x) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

namespace jt {

namespace {

constexpr int64_t kAlign = 256;
inline int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// A tensor view: (bit label, element stride) per address bit, unsliced bits only.
struct View {
  std::vector<std::pair<int64_t, int64_t>> bits;
};

struct ExecNode {
  int kind = 0;  // 0: K2 CUDA-core GETT, 1: K3 tcgen05 (resident A), 2: K3g tcgen05 (streamed A),
                 // 3: K4 DMMA (c128), 4: K2s streaming GETT (skinny c64, A in registers)
  StreamArgs st{};
  std::vector<int64_t> stN, stK;  // K2s: B strides of the column bits and the K bits (emulator)
  TcArgs tc{};
  TcgArgs tcg{};
  std::vector<int64_t> tcgA_m, tcgA_k, tcgB_oN, tcgA_oM;  // K3g host strides (emulator)
  std::vector<int64_t> tcB_n, tcB_k;  // K3: B strides of the 7 row bits and the K bits (emulator)
  // K3g fed by a K1 bit-gather: the operand is first copied into the K3g layout (item bits
  // lowest); gA/gB = the source strides of the copy's bits (bit j of the copy <- stride), the
  // copies live in the scratch region at perm_off (B) and perm_off + permA_at (A)
  bool permA = false, permB = false;
  GatherArgs gA{}, gB{};
  int64_t perm_bytes = 0, permA_at = 0, perm_off = 0;
  int64_t v = -1;
  int64_t opA = -1, opB = -1;  // plan node ids (A has the fewer free bits)
  std::vector<std::pair<int, int64_t>> sliceA, sliceB;  // (slice position, element stride) for leaves
  GettArgs args{};
  int RM = 1, RN = 1, block = 32;
  int64_t grid_x = 1;  // persistent CTAs along the output tiles (set for the device at exec create)
  size_t smem = 0;
  int64_t out_off = 0;   // byte offset of the output in the workspace
  int64_t part_off = 0;  // byte offset of split-K partials
  int64_t n_out = 1;     // output elements
  double flop = 0, bytes = 0;
  int maxpos = -1;
  // bit keys the consumer (parent) contracts: the producer puts one of them at stride 1 in its
  // output when it can (consumer-ordered layout -> 16-B k-pair gathers in a K3 consumer)
  std::vector<int64_t> pref_low;
  // bit keys of this node's output that its parent contracts (shared with the sibling)
  std::vector<int64_t> consumer_k;
};

// Consumer-aware order (K3, default; JETB200_K3_CORDER=0 keeps stride order): the bits the parent
// contracts first within the small-operand (M) bits and within the tile-index (outer) bits, so the
// parent's K chunk sits right above the 7 row bits in this node's output and the parent's item
// is one long contiguous run (one or a few TMA-engine copies).  Both orders are free: the epilogue
// writes [rows][M][outer] whatever the bit order inside M and inside outer.
template <typename T, typename Key>
void consumer_first(std::vector<T>& v, const std::vector<int64_t>& ck, Key key) {
  const char* e = std::getenv("JETB200_K3_CORDER");
  if ((e && e[0] == '0') || ck.empty()) return;
  std::stable_partition(v.begin(), v.end(),
                        [&](const T& x) { return std::find(ck.begin(), ck.end(), key(x)) != ck.end(); });
}

// Move the first bit of `t` that the consumer contracts to the front (it gets stride 1 in the
// output view); the others keep their order.
void prefer_low(std::vector<int64_t>& t, const std::vector<int64_t>& pref) {
  for (size_t i = 0; i < t.size(); ++i)
    if (std::find(pref.begin(), pref.end(), t[i]) != pref.end()) {
      std::rotate(t.begin(), t.begin() + i, t.begin() + i + 1);
      return;
    }
}

struct Layout {
  int esize = 8;
  std::vector<ExecNode> order;        // execution order (internal nodes)
  std::vector<int64_t> leaf_off;      // byte offset of every leaf (full, unsliced data)
  std::vector<int64_t> node_off;      // byte offset of every node output (leaves: leaf_off)
  int64_t leaf_bytes = 0, inter_bytes = 0, scratch_bytes = 0;
  int64_t inter_base = 0, scratch_base = 0, vals_base = 0, acc_base = 0, state_base = 0, total = 0;
  int64_t vals_cap = 1;  // slice-value ring (per call, indexed from the call's first slice)
  // memory report (f3, PAPER.md l.291-298 fig. m10_memory)
  int64_t mem_no_deletion = 0, mem_peak_live = 0, mem_cache = 0, mem_peak_live_noshare = 0;
};

using GettFn = void (*)(GettArgs);
using TcFn = void (*)(TcArgs);

using TcgFn = void (*)(TcgArgs);
TcgFn pick_tcg(int tmt, bool tma) {
  switch (tmt * 2 + (tma ? 1 : 0)) {
    case 8: return gett_tcg_kernel<4, false>;
    case 9: return gett_tcg_kernel<4, true>;
    case 10: return gett_tcg_kernel<5, false>;
    case 11: return gett_tcg_kernel<5, true>;
    case 12: return gett_tcg_kernel<6, false>;
    case 13: return gett_tcg_kernel<6, true>;
    case 14: return gett_tcg_kernel<7, false>;
    case 15: return gett_tcg_kernel<7, true>;
  }
  fail(JT_EINTERNAL, "no tcg instance");
}

TcFn pick_tc(int tkc, bool tma) {
  switch (tkc * 2 + (tma ? 1 : 0)) {
    case 4: return gett_tc_kernel<2, false>;
    case 5: return gett_tc_kernel<2, true>;
    case 6: return gett_tc_kernel<3, false>;
    case 7: return gett_tc_kernel<3, true>;
    case 8: return gett_tc_kernel<4, false>;
    case 9: return gett_tc_kernel<4, true>;
  }
  fail(JT_EINTERNAL, "no tc instance");
}

using StreamFn = void (*)(StreamArgs);
StreamFn pick_stream(int tm, int kt) {
#define JT_SCASE(a, b) \
  if (tm == a && kt == b) return stream_gett_kernel<a, b>;
  JT_SCASE(0, 1) JT_SCASE(0, 2) JT_SCASE(0, 3) JT_SCASE(1, 1) JT_SCASE(1, 2) JT_SCASE(1, 3)
  JT_SCASE(2, 1) JT_SCASE(2, 2) JT_SCASE(2, 3)
#undef JT_SCASE
  fail(JT_EINTERNAL, "no stream instance");
}

GettFn pick_dmma(int SMT, int SNT, bool gauss) {
#define JT_DCASE(a, b) \
  if (SMT == a && SNT == b) return gauss ? gett_dmma_kernel<a, b, true> : gett_dmma_kernel<a, b, false>;
  JT_DCASE(1, 1) JT_DCASE(1, 2) JT_DCASE(1, 4) JT_DCASE(2, 1) JT_DCASE(2, 2) JT_DCASE(2, 4)
  JT_DCASE(4, 1) JT_DCASE(4, 2)
#undef JT_DCASE
  if (SMT == 4 && SNT == 4 && !gauss) return gett_dmma_kernel<4, 4, false>;
  fail(JT_EINTERNAL, "no dmma instance");
}

template <typename R>
GettFn pick_gett(int RM, int RN) {
#define JT_CASE(a, b) \
  if (RM == a && RN == b) return gett_kernel<R, a, b>;
  JT_CASE(1, 1) JT_CASE(1, 2) JT_CASE(1, 4) JT_CASE(2, 1) JT_CASE(2, 2) JT_CASE(2, 4)
  JT_CASE(4, 1) JT_CASE(4, 2) JT_CASE(4, 4)
#undef JT_CASE
  fail(JT_EINTERNAL, "no gett instance");
}

// Raise the dynamic shared-memory limit of every kernel the executor launches.  The attribute
// is per device, so it is set once per device id (the current device at the call) and every
// result is checked.
void set_smem_attrs() {
  static std::mutex mu;
  static std::vector<char> done;
  int dev = 0;
  JT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if ((int)done.size() <= dev) done.resize(dev + 1, 0);
  if (done[dev]) return;
  // the largest shared-memory carveout: without it the occupancy calculator assumes the default
  // carveout and reported ONE K3 CTA per SM for the 52-108 KB K3 CTAs that are sized to run two
  // per SM (measured: every C3 K3 launch had 148 CTAs, sm__warps_active 21.9% = 14 of 64 warps)
  auto set = [](const void* f, int bytes) {
    JT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    JT_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  };
  const int rms[3] = {1, 2, 4};
  for (int a : rms)
    for (int b : rms) {
      set(reinterpret_cast<const void*>(pick_gett<float>(a, b)), 200 * 1024);
      set(reinterpret_cast<const void*>(pick_gett<double>(a, b)), 200 * 1024);
      set(reinterpret_cast<const void*>(pick_dmma(a, b, false)), 200 * 1024);
      if (a * b <= 8) set(reinterpret_cast<const void*>(pick_dmma(a, b, true)), 200 * 1024);
    }
  for (int tkc = 2; tkc <= 4; ++tkc)
    for (int tma = 0; tma < 2; ++tma) set(reinterpret_cast<const void*>(pick_tc(tkc, tma != 0)), 222 * 1024);
  for (int tmt = 4; tmt <= 7; ++tmt)
    for (int tma = 0; tma < 2; ++tma) set(reinterpret_cast<const void*>(pick_tcg(tmt, tma != 0)), 222 * 1024);

  set(reinterpret_cast<const void*>(permute_kernel<float2, 0>), 200 * 1024);
  set(reinterpret_cast<const void*>(permute_kernel<float2, 1>), 200 * 1024);
  set(reinterpret_cast<const void*>(permute_kernel<float2, 2>), 200 * 1024);
  set(reinterpret_cast<const void*>(permute_kernel<double2, 0>), 200 * 1024);
  done[dev] = 1;
}

int ilog2_exact(int d) {
  int b = 0;
  while ((1 << b) < d) ++b;
  if ((1 << b) != d) fail(JT_EUSAGE, "exec: the GPU path needs a power-of-two qudit dimension d");
  return b;
}

// Bulk-copy (TMA engine, cp.async.bulk) landing of an item whose address bits have the given
// element strides: the bits sorted by stride land packed, bit b at byte 8 << rank(b).  The run of
// consecutive strides that starts at stride 1 is contiguous in global memory and moves as one
// copy; the item's remaining h bits (h <= 5) enumerate 2^h copies, copy j at element offset
// xoff[j] (the digits of j over those bits, in rank order) landing at j * copy bytes.  (A tensor
// map cannot take the item base as a coordinate: a dim-0 extent overlapping the higher strides
// faults with an illegal instruction on B200, profiles/r02_tma_probe.txt.)  Returns false when
// the item does not hold the operand's stride-1 bit or needs more than 32 copies.
bool tma_item_dims(const std::vector<int64_t>& strides, int* ncopy, int* copy_log2, int64_t* xoff,
                   std::vector<int>& rank) {
  std::vector<std::pair<int64_t, int>> bits;
  for (size_t i = 0; i < strides.size(); ++i) bits.push_back({strides[i], (int)i});
  std::sort(bits.begin(), bits.end());
  rank.assign(strides.size(), 0);
  for (size_t r = 0; r < bits.size(); ++r) rank[bits[r].second] = (int)r;
  if (bits[0].first != 1) return false;
  size_t low = 1;
  while (low < bits.size() && bits[low].first == bits[low - 1].first * 2) ++low;
  const int h = (int)(bits.size() - low);
  if (h > 5) return false;
  // copies below JETB200_TMA_MINCOPY bytes (default 2 KB) lose to the cp.async gathers: measured
  // on the C3 K3 nodes, 16 x 1 KB copies per item ran at 57-73% of HBM vs 70-91% gathered, while
  // 2-4 copies of 4-8 KB reached 100-103% (profiles/r02_nodes_C3_tma.txt); in the amplitude step
  // a 2-KB floor beat a 4-KB one (9.17 vs 9.27 s, profiles/r02_variants_pdl.txt)
  int64_t min_copy = 2048;
  if (const char* e = std::getenv("JETB200_TMA_MINCOPY")) min_copy = std::max<int64_t>(16, atoll(e));
  if ((int64_t(8) << low) < min_copy) return false;
  *ncopy = 1 << h;
  *copy_log2 = (int)low;
  if (xoff)
    for (int j = 0; j < *ncopy; ++j) {
      int64_t o = 0;
      for (int i = 0; i < h; ++i)
        if ((j >> i) & 1) o += bits[low + i].first;
      xoff[j] = o;
    }
  return true;
}

bool tma_enabled() {
  const char* e = std::getenv("JETB200_K3_TMA");
  return !(e && e[0] == '0');
}

// K3 eligibility and descriptor (c64 only): small A fully inside the tile with 3..7 free
// bits and 2..8 contracted bits, big B with >= 7 free bits (128-row MMA tiles).  Returns
// false if the contraction does not fit K3.
bool plan_tc(ExecNode& en, const View& va, const View& vb, int esize, View& out) {
  if (esize != 8) return false;
  std::map<int64_t, int64_t> sa, sb;
  for (auto& x : va.bits) sa[x.first] = x.second;
  for (auto& x : vb.bits) sb[x.first] = x.second;
  std::vector<std::pair<int64_t, int64_t>> M, N, K;  // (stride, bit)
  for (auto& x : va.bits) {
    if (sb.count(x.first)) K.push_back({sb[x.first], x.first});
    else M.push_back({x.second, x.first});
  }
  for (auto& x : vb.bits)
    if (!sa.count(x.first)) N.push_back({x.second, x.first});
  const int tm = (int)M.size(), kt = (int)K.size();
  // (1-2 free bits of A run through the padded-N path correctly but measured slower than K2 on
  // the C3 streaming nodes -- 8-KB gather items -- so K3 takes 3..7)
  int min_tm = 3;  // JETB200_K3_MINTM: sweep knob (1-2 free bits of A run on the padded-N path)
  if (const char* e = std::getenv("JETB200_K3_MINTM")) min_tm = std::max(1, std::min(3, atoi(e)));
  if (tm < min_tm || tm > 7 || kt < 2 || kt > 8 || (int)N.size() < 7) return false;
  const int swz = kt >= 4 ? 1 : 0;        // SWIZZLE_128B needs 32 TF32 (16 complex) per row
  const int tkc = swz ? 4 : kt;
  const int n_kc = 1 << (kt - tkc);
  // MMA N = 2 * 2^tm, padded to the M=128 minimum of 16 for 1-2 free bits of A (the padded Y
  // rows are zero and the padded accumulator columns are never stored)
  const int Kpc = 2 << tkc, Np = std::max(16, 2 << tm);
  const int yplane = Np * Kpc * 4;
  // TMEM: accumulators (2 when they fit beside >= 2 X stages) + X stages of 2*Kpc columns.
  // CTAs per SM: TMEM (512 columns) is per SM and the block scheduler does not see it, so the
  // shared-memory footprint enforces the CTA count the TMEM budget allows -- two CTAs of <= 256
  // columns each, or one CTA whose shared memory is padded past half of the SM.  (Two CTAs of
  // one grid sized for one per SM co-resided through shared memory, the second blocking in
  // tcgen05.alloc until the first finished: +2.2 s per C3 amplitude under PDL.)
  // pairN (JETB200_K3_PAIRN=1): N = 16 one-chunk tiles issue 2 MMAs per K step (see TcArgs.pairN)
  // on accumulators twice as wide
  bool pairN = false;
  if (const char* e = std::getenv("JETB200_K3_PAIRN"))
    pairN = e[0] == '1' && swz && n_kc == 1 && Np == 16 && (2 << tm) == Np;
  const int acc_w = pairN ? 2 * Np : Np;
  int acc_bufs = (2 * acc_w + 2 * 2 * Kpc <= 512) ? 2 : 1;
  // JETB200_K3_ACC=4: four accumulators when MMA N <= 16 (one-chunk tiles of tm = 3: the MMA can
  // run up to four tiles ahead of the epilogue)
  if (const char* e = std::getenv("JETB200_K3_ACC"))
    if (atoi(e) == 4 && Np <= 16) acc_bufs = 4;
  // CTAs per SM: two (each half the TMEM and shared memory) when the per-item MMA work is large
  // against the item's bytes -- N <= 16 tiles (tm = 3) or tiles of several K chunks -- else one
  // with the deeper rings.  Measured per node on C3 (profiles/r02_nodes_C3_ctas.txt): tm = 3 nodes
  // 0.65-0.76 -> 0.86-0.93 of HBM with two CTAs, tm = 4 single-chunk nodes 0.99 -> 0.89.
  // JETB200_K3_CTAS=1/2 forces the count.
  int ctas = (Np <= 16 || n_kc >= 2) ? 2 : 1;
  if (const char* e = std::getenv("JETB200_K3_CTAS")) ctas = std::max(1, std::min(2, atoi(e)));
  const bool two = ctas == 2 && acc_bufs * acc_w + 2 * 2 * Kpc <= 256;
  const int cols_budget = two ? 256 : 512;
  int xstages = std::min(4, (cols_budget - acc_bufs * acc_w) / (2 * Kpc));
  if (xstages < 2) return false;
  const int rbytes = 128 * (8 << tkc);
  const int64_t ybytes = 2LL * n_kc * yplane;
  const int64_t budget = (two ? 112 : 220) * 1024 - 1024 - ybytes;
  int rs_cap = two ? 6 : 12;  // JETB200_K3_RS: sweep knob for the raw ring depth (<= 16)
  if (const char* e = std::getenv("JETB200_K3_RS")) rs_cap = std::max(2, std::min(16, atoi(e)));
  const int rstages = (int)std::min<int64_t>(rs_cap, budget / rbytes);
  if (rstages < 2) return false;
  int64_t smem = ybytes + (int64_t)rstages * rbytes + 1024;
  if (!two) smem = std::max<int64_t>(smem, 116 * 1024);
  std::sort(M.begin(), M.end());
  std::sort(N.begin(), N.end());
  std::sort(K.begin(), K.end());
  std::vector<int64_t> tN, oN;
  for (size_t i = 0; i < N.size(); ++i) (i < 7 ? tN : oN).push_back(N[i].second);
  if ((int)oN.size() > 31) return false;
  prefer_low(tN, en.pref_low);
  consumer_first(M, en.consumer_k, [](const std::pair<int64_t, int64_t>& x) { return x.second; });
  consumer_first(oN, en.consumer_k, [](int64_t x) { return x; });
  TcArgs& t = en.tc;
  std::memset(&t, 0, sizeof(t));
  t.tm = tm;
  t.K = kt;
  t.tkc = tkc;
  t.n_kc = n_kc;
  t.swz = swz;
  t.nX = 7 + tkc;
  t.Np = Np;
  t.Kpc = Kpc;
  t.sbo_x = t.sbo_y = swz ? 1024 : (Kpc / 4) * 128;
  t.xbuf = 0;
  t.yplane = yplane;
  t.xstages = xstages;
  t.rstages = rstages;
  t.rbytes = rbytes;
  t.passes = 3;
  if (const char* e = std::getenv("JETB200_DEBUG_K3_PASSES"))  // diagnostic only: MMA-count sweep
    if (e[0] == '1') t.passes = 1;
  t.acc_bufs = acc_bufs;
  t.pairN = pairN ? 1 : 0;
  t.acc_w = acc_w;
  t.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  uint32_t cols = 32;
  while ((int)cols < acc_bufs * acc_w + xstages * 2 * Kpc) cols <<= 1;
  if (!two) cols = 512;
  t.tmem_cols = cols;
  // chunk-tile bits in B-stride order with their byte offsets in the raw landing stage:
  // row n, complex k at n*rb + ((k>>1) ^ (n & (chunks-1)))*16 + (k&1)*8 (XOR-combinable)
  const int rb = 8 << tkc, lg_chunks = tkc - 1;
  std::vector<std::pair<int64_t, int32_t>> tb;
  // the raw-row XOR swizzle uses the lg_chunks row bits with the SMALLEST B strides (a warp's
  // gather lanes vary those first), whatever row-bit order the output layout chose
  int swz_rank[7];
  {
    std::vector<std::pair<int64_t, int>> rs;
    for (int i = 0; i < 7; ++i) rs.push_back({sb[tN[i]], i});
    std::sort(rs.begin(), rs.end());
    for (int q = 0; q < 7; ++q) swz_rank[rs[q].second] = q;
    for (int q = 0; q < 3; ++q) t.swz_row[q] = (int8_t)rs[q].second;
  }
  for (int i = 0; i < 7; ++i)
    tb.push_back({sb[tN[i]], (rb << i) ^ (swz_rank[i] < lg_chunks ? (16 << swz_rank[i]) : 0)});
  for (int i = 0; i < tkc; ++i) tb.push_back({sb[K[i].second], i == 0 ? 8 : (16 << (i - 1))});
  std::sort(tb.begin(), tb.end());
  for (size_t j = 0; j < tb.size(); ++j) {
    t.gX[j] = tb[j].first;
    t.sX[j] = tb[j].second;
  }
  // 16-B k-pair gathers: the lowest chunk-tile bit is K bit 0 (raw offset 8) at stride 1; every
  // other bit of B then has an even stride, so pairs stay 16-B aligned on both sides
  {
    // opt-in: measured slower on C3 (12.3 s vs 10.3 s per amplitude with consumer-ordered
    // layouts, profiles/r01_bench_c3_vec*.json), so off unless JETB200_K3_VEC=1
    const char* e = getenv("JETB200_K3_VEC");
    t.vecB = (tb[0].first == 1 && tb[0].second == 8 && e && e[0] == '1') ? 1 : 0;
  }
  en.args.vecB = t.vecB;  // (reported by jt_exec_describe)
  // TMA-engine item load (default; JETB200_K3_TMA=0 keeps the cp.async gathers): the item's
  // 7 + tkc bits land packed in B-stride order, bit b at byte 8 << rank(b), moved as bulk copies
  // of the item's stride-1 run (tma_item_dims)
  {
    std::vector<int64_t> item;
    for (int i = 0; i < 7; ++i) item.push_back(sb[tN[i]]);
    for (int j = 0; j < tkc; ++j) item.push_back(sb[K[j].second]);
    std::vector<int> rank;
    int ncopy = 0, clog = 0;
    bool even = true;  // 16-B aligned copies: a sliced leaf's digit strides must be even
    for (auto& x : en.sliceB) even &= (x.second % 2) == 0;
    t.tma = (tma_enabled() && even && tma_item_dims(item, &ncopy, &clog, t.xoff, rank)) ? 1 : 0;
    if (t.tma) {
      t.ncopy = ncopy;
      t.copy_bytes = 8 << clog;
      for (int i = 0; i < 7; ++i) t.rofs_row[i] = 8 << rank[i];
      for (int j = 0; j < tkc; ++j) t.rofs_k[j] = 8 << rank[7 + j];
      t.vecB = 0;
      en.args.vecB = 0;
    }
  }
  for (int j = 0; j < kt - tkc; ++j) t.o_kB[j] = sb[K[tkc + j].second];
  for (int i = 0; i < tm; ++i) t.aM[i] = sa[M[i].second];
  for (int i = 0; i < kt; ++i) t.aK[i] = sa[K[i].second];
  t.n_outer = (int)oN.size();
  for (int j = 0; j < t.n_outer; ++j) t.o_sB[j] = sb[oN[j]];
  t.n_tiles = int64_t(1) << t.n_outer;
  en.tcB_n.clear();
  en.tcB_k.clear();
  for (int i = 0; i < 7; ++i) en.tcB_n.push_back(sb[tN[i]]);
  for (int i = 0; i < kt; ++i) en.tcB_k.push_back(sb[K[i].second]);
  en.kind = 1;
  en.smem = (size_t)smem;
  en.block = t.tma ? 448 : 416;
  en.n_out = t.n_tiles << (7 + tm);
  en.grid_x = t.n_tiles;
  en.args.splits = 1;
  en.args.n_tiles = t.n_tiles;
  // output layout: [M][7 rows][outer] (JETB200_K3_MLOW=1, tm >= 3 so a row's m values are
  // whole 16-B pairs) puts the small operand's new legs -- which the next absorption contracts --
  // lowest, next to the rows; default [rows][M][outer]
  {
    const char* e = std::getenv("JETB200_K3_MLOW");
    t.mlow = (e && e[0] == '1' && tm >= 3 && Np == 2 << tm) ? 1 : 0;
  }
  out.bits.clear();
  int64_t st = 1;
  if (t.mlow) {
    for (auto& b : M) { out.bits.push_back({b.second, st}); st <<= 1; }
    for (auto b : tN) { out.bits.push_back({b, st}); st <<= 1; }
  } else {
    for (auto b : tN) { out.bits.push_back({b, st}); st <<= 1; }
    for (auto& b : M) { out.bits.push_back({b.second, st}); st <<= 1; }
  }
  for (auto b : oN) { out.bits.push_back({b, st}); st <<= 1; }
  return true;
}

// K2s eligibility and descriptor (c64): A tiny (<= 2 free bits, 1..3 contracted bits), B with
// >= 10 free bits.  `kv` is the K2 output view of the same node ([tile-N][tile-M][outer], from
// plan_gett): K2s writes exactly that layout when the M bits are adjacent in it, so the consumer
// sees what K2 would have produced.  JETB200_K2S=0 keeps such nodes on K2.
bool plan_stream(ExecNode& en, const View& va, const View& vb, const View& kv, int esize) {
  if (esize != 8) return false;
  if (const char* e = std::getenv("JETB200_K2S"))
    if (e[0] == '0') return false;
  std::map<int64_t, int64_t> sa, sb;
  for (auto& x : va.bits) sa[x.first] = x.second;
  for (auto& x : vb.bits) sb[x.first] = x.second;
  std::vector<std::pair<int64_t, int64_t>> M, K;  // (stride in A / in B, bit)
  for (auto& x : va.bits) {
    if (sb.count(x.first)) K.push_back({sb[x.first], x.first});
    else M.push_back({x.second, x.first});
  }
  const int tm = (int)M.size(), kt = (int)K.size();
  const int ncols = (int)vb.bits.size() - kt;
  if (tm > 2 || kt < 1 || kt > 3 || ncols < 10 || ncols > kStreamMaxCols) return false;
  // the K2 layout: column bits (B free) in output order, the M bits adjacent at n_lo
  std::vector<int64_t> cols, mo;
  int n_lo = -1;
  for (size_t i = 0; i < kv.bits.size(); ++i) {
    const int64_t b = kv.bits[i].first;
    if (sa.count(b)) {
      if (n_lo < 0) n_lo = (int)i;
      else if ((int)i != n_lo + (int)mo.size()) return false;
      mo.push_back(b);
    } else {
      cols.push_back(b);
    }
  }
  if (tm == 0) n_lo = ncols;
  if ((int)cols.size() != ncols || (int)mo.size() != tm) return false;
  std::sort(K.begin(), K.end());  // lowest B stride first: K bit 0 is the pair bit when stride 1
  StreamArgs& t = en.st;
  std::memset(&t, 0, sizeof(t));
  t.n_cols = ncols;
  t.n_lo = n_lo;
  bool even = K[0].first == 1;
  for (int j = 0; j < ncols; ++j) {
    t.sN[j] = sb[cols[j]];
    even &= t.sN[j] % 2 == 0;
  }
  for (int j = 1; j < kt; ++j) even &= K[j].first % 2 == 0;
  for (auto& x : en.sliceB) even &= (x.second % 2) == 0;
  t.vec = even ? 1 : 0;
  for (int k = 0; k < (1 << kt); ++k) {
    int64_t o = 0;
    for (int j = 0; j < kt; ++j) if ((k >> j) & 1) o += K[j].first;
    t.kofs[k] = o;
  }
  for (int m = 0; m < (1 << tm); ++m)
    for (int k = 0; k < (1 << kt); ++k) {
      int64_t o = 0;
      for (int i = 0; i < tm; ++i) if ((m >> i) & 1) o += sa[mo[i]];
      for (int j = 0; j < kt; ++j) if ((k >> j) & 1) o += sa[K[j].second];
      t.aofs[m * (1 << kt) + k] = o;
    }
  en.stN.clear();
  en.stK.clear();
  for (int j = 0; j < ncols; ++j) en.stN.push_back(t.sN[j]);
  for (int j = 0; j < kt; ++j) en.stK.push_back(K[j].first);
  en.kind = 4;
  en.args.tm = tm;   // (reported by jt_exec_describe)
  en.args.tk = kt;
  en.args.tn = n_lo;
  en.args.n_outer = ncols - n_lo;
  en.args.splits = 1;
  en.args.n_tiles = int64_t(1) << ncols;
  en.smem = 0;
  en.block = 256;
  en.n_out = int64_t(1) << (ncols + tm);
  en.grid_x = 1;
  return true;
}

// K3g eligibility and descriptor (c64): both operands streamed; output tiles of 128 rows of B's
// free bits x 2^tmt (16..128) complex columns of A's free bits; K in chunks of 16 complex.
bool plan_tcg(ExecNode& en, const View& va, const View& vb, int esize, View& out) {
  if (esize != 8) return false;
  std::map<int64_t, int64_t> sa, sb;
  for (auto& x : va.bits) sa[x.first] = x.second;
  for (auto& x : vb.bits) sb[x.first] = x.second;
  std::vector<std::pair<int64_t, int64_t>> M, N, K;
  for (auto& x : va.bits) {
    if (sb.count(x.first)) K.push_back({sb[x.first], x.first});
    else M.push_back({x.second, x.first});
  }
  for (auto& x : vb.bits)
    if (!sa.count(x.first)) N.push_back({x.second, x.first});
  if ((int)M.size() < 4 || (int)N.size() < 7 || (int)K.size() < 4) return false;
  // tile columns: up to 128 complex (MMA N 256, one TMEM accumulator beside 4 X stages): the
  // producers' gather + split work per MMA FLOP drops by a third against 64 columns (two
  // accumulators); measured 124 -> 167-172 TFLOP/s on the C5 nodes.  JETB200_TCG_TMT caps it.
  int tmt_max = 7;
  if (const char* e = getenv("JETB200_TCG_TMT")) tmt_max = std::max(4, std::min(7, atoi(e)));
  const int tmt = std::min<int>((int)M.size(), tmt_max);
  const int MT = 1 << tmt, NP = 2 * MT;
  std::sort(M.begin(), M.end());
  std::sort(N.begin(), N.end());
  // K chunk: the 2 lowest-A-stride K bits, then the lowest-B-stride ones, to 4 bits
  std::vector<std::pair<int64_t, int64_t>> KA;
  for (auto& k : K) KA.push_back({sa[k.second], k.second});
  std::sort(KA.begin(), KA.end());
  std::sort(K.begin(), K.end());
  std::vector<int64_t> kc, ko;
  std::vector<int64_t> tN, oN, tM, oM;
  for (size_t i = 0; i < N.size(); ++i) (i < 7 ? tN : oN).push_back(N[i].second);
  for (size_t i = 0; i < M.size(); ++i) ((int)i < tmt ? tM : oM).push_back(M[i].second);
  // candidate K chunks, in order of preference: (gather path) the 2 lowest-A-stride K bits then
  // the lowest-B-stride ones; (TMA) the 4 lowest-B-stride, the 4 lowest-A-stride K bits.  With
  // TMA on, the first candidate whose B and A chunks are both <= 5-run boxes wins.
  auto chunk_from = [&](int na) {
    std::vector<int64_t> c;
    for (int i = 0; i < na; ++i) c.push_back(KA[i].second);
    for (auto& k : K)
      if ((int)c.size() < 4 && std::find(c.begin(), c.end(), k.second) == c.end()) c.push_back(k.second);
    return c;
  };
  auto chunk_boxes = [&](const std::vector<int64_t>& c) {  // TMA boxes per item, 1 << 20 if none
    std::vector<int64_t> ib, ia;
    for (int i = 0; i < 7; ++i) ib.push_back(sb[tN[i]]);
    for (int i = 0; i < tmt; ++i) ia.push_back(sa[tM[i]]);
    for (auto b : c) { ib.push_back(sb[b]); ia.push_back(sa[b]); }
    std::vector<int> r;
    int nb = 0, na = 0, cl = 0;
    if (!tma_item_dims(ib, &nb, &cl, nullptr, r) || !tma_item_dims(ia, &na, &cl, nullptr, r)) return 1 << 20;
    return nb + na;
  };
  kc = chunk_from(2);
  if (tma_enabled()) {
    int best = chunk_boxes(kc);
    for (int na : {0, 4, 1, 3}) {
      const int nb = chunk_boxes(chunk_from(na));
      if (nb < best) { best = nb; kc = chunk_from(na); }
    }
  }
  for (auto& k : K)
    if (std::find(kc.begin(), kc.end(), k.second) == kc.end()) ko.push_back(k.second);
  if (oN.size() + oM.size() > 31 || ko.size() > 32 || oN.size() > 32 || oM.size() > 32) return false;
  // K1-fed operands (default; JETB200_TCG_PERM=0 keeps the gathers): an operand whose chunk is
  // not a few long runs of its own layout is bit-gathered into the K3g layout first -- B as
  // [7 rows][4 chunk K][chunk-index K][outer N], A as [4 chunk K][tmt M][chunk-index K][outer M]
  // -- so each item is ONE contiguous TMA-engine copy (the copy costs 16 B per element, against
  // thousands of FLOP per element on these GEMM-shaped nodes)
  en.permA = en.permB = false;
  if (tma_enabled()) {
    const std::map<int64_t, int64_t> sb0 = sb, sa0 = sa;
    const char* e = getenv("JETB200_TCG_PERM");
    const bool allow = !(e && e[0] == '0');
    const bool force = e && std::string(e) == "force";  // tests: copy whenever an item is not one box
    auto item_ok = [&](const std::vector<int64_t>& strides, const std::vector<std::pair<int, int64_t>>& sl) {
      for (auto& x : sl)
        if (x.second % 2) return false;
      std::vector<int> r;
      int nc = 0, cl = 0;
      return tma_item_dims(strides, &nc, &cl, nullptr, r);
    };
    std::vector<int64_t> ib, ia;
    for (auto b : tN) ib.push_back(sb[b]);
    for (auto b : kc) ib.push_back(sb[b]);
    for (auto b : tM) ia.push_back(sa[b]);
    for (auto b : kc) ia.push_back(sa[b]);
    // only where the copy is cheap against the node: each B element meets 2^|M| columns of A, so
    // the copy's 16 B per element is <= ~10% of the MMA time at |M| >= 9 (likewise A with |N|)
    if (allow && (M.size() >= 9 || force) && !item_ok(ib, en.sliceB)) {
      std::vector<int64_t> order(tN.begin(), tN.end());
      order.insert(order.end(), kc.begin(), kc.end());
      order.insert(order.end(), ko.begin(), ko.end());
      order.insert(order.end(), oN.begin(), oN.end());
      if (order.size() == vb.bits.size() && order.size() <= 40) {
        en.permB = true;
        en.gB = GatherArgs{};
        en.gB.n_bits = (int)order.size();
        en.gB.is_a = 0;
        for (size_t j = 0; j < order.size(); ++j) {
          en.gB.s[j] = sb[order[j]];
          sb[order[j]] = int64_t(1) << j;
        }
      }
    }
    if (allow && (N.size() >= 9 || force) && !item_ok(ia, en.sliceA)) {
      std::vector<int64_t> order(kc.begin(), kc.end());
      order.insert(order.end(), tM.begin(), tM.end());
      order.insert(order.end(), ko.begin(), ko.end());
      order.insert(order.end(), oM.begin(), oM.end());
      if (order.size() == va.bits.size() && order.size() <= 40) {
        en.permA = true;
        en.gA = GatherArgs{};
        en.gA.n_bits = (int)order.size();
        en.gA.is_a = 1;
        for (size_t j = 0; j < order.size(); ++j) {
          en.gA.s[j] = sa[order[j]];
          sa[order[j]] = int64_t(1) << j;
        }
      }
    }
    // a copy pays only if it makes BOTH operands TMA-fed: otherwise the gather path runs anyway
    const bool okB = en.permB || item_ok(ib, en.sliceB), okA = en.permA || item_ok(ia, en.sliceA);
    if (!(okA && okB) && !force) {
      sb = sb0;
      sa = sa0;
      en.permA = en.permB = false;
    }
    const int64_t bB = en.permB ? align_up((int64_t(8) << en.gB.n_bits)) : 0;
    const int64_t bA = en.permA ? align_up((int64_t(8) << en.gA.n_bits)) : 0;
    en.permA_at = bB;
    en.perm_bytes = bA + bB;
  }
  // Y (expanded A, hi|lo planes) ring depth: the producers run ystages-1 items ahead of the MMAs
  // (2, 3 and 4 measured within 3% of each other on the C5 nodes: not the bound; 2 keeps the
  // deepest raw gather ring)
  int ystages = 2;
  if (const char* e = getenv("JETB200_TCG_YS")) ystages = std::max(2, std::min(4, atoi(e)));
  const int rb_b = 128 * 128, rb_a = MT * 128;
  int64_t ybytes = (int64_t)ystages * 2 * NP * 128;
  while (ystages > 2 && (220 * 1024 - 1024 - 16384 - ybytes) / (rb_b + rb_a) < 3) {
    --ystages;
    ybytes = (int64_t)ystages * 2 * NP * 128;
  }
  const int64_t ebytes = 16384;  // epilogue staging: two 8-KB buffers (8 complex columns x 128 rows)
  const int rstages = (int)std::min<int64_t>(6, (220 * 1024 - 1024 - ybytes - ebytes) / (rb_b + rb_a));
  if (rstages < 2) return false;
  TcgArgs& t = en.tcg;
  std::memset(&t, 0, sizeof(t));
  t.n_oN = (int)oN.size();
  t.n_oM = (int)oM.size();
  t.tmt = tmt;
  {
    const char* e = getenv("JETB200_TCG_BM");  // tuning knob: band height (log2 M tiles)
    t.lg_bm = std::min(e ? atoi(e) : 4, t.n_oM);
    if (t.lg_bm < 0) t.lg_bm = 0;
  }
  t.lg_kc = (int)ko.size();
  // FP32 accumulation in TMEM over very long K drifts (C5: 2^19-complex K, 7.9e-3 relative vs
  // the CUDA-core path, 1.07e-3 vs the P7 closed form): the accumulator restarts every
  // 2^JETB200_TCG_SEG chunks and the epilogue sums the segments in FP32 in order.  Measured on
  // the benched C5 plan (profiles/r02_c5_segments.txt), K3g vs K2 / worst P7 slice / K3g time:
  // seg 8: 1.8e-4 / 8.8e-5 / +2%; seg 6: 1.0e-4 / 8.6e-5 / +5%; seg 4: 4.2e-5 / 6.9e-5 / +13%.
  // Default 4 (256 complex per segment, the longest accumulation K3 itself does)
  {
    int seg = 4;
    if (const char* e = getenv("JETB200_TCG_SEG")) seg = std::max(0, atoi(e));
    t.lg_kcs = std::min(t.lg_kc, seg);
  }
  t.nXb = 11;
  t.nAb = tmt + 4;
  t.Np = NP;
  t.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  t.acc_bufs = NP <= 128 ? 2 : 1;   // 512 TMEM columns = accumulators + 4 X stages of 64
  // rotating accumulator regions (opt-in, JETB200_TCG_ROT=1): with 256 accumulator columns and K
  // segments, three 128-column regions + 2 X stages (kernels_tcg.cuh tcg::Rot) so the MMAs never
  // wait for a segment drain.  Correct (tests) but measured slower on the C5 nodes: 186-189 vs
  // 214-219 TFLOP/s single-accumulator (no-segment ceiling 242-250), i.e. the N = 128 MMAs and
  // the halved X ring cost more than the drains they hide (profiles/r02_nodes_C5_rot.txt)
  t.lg_xs = 2;
  {
    const char* e = getenv("JETB200_TCG_EPI");  // "warp": per-warp segment drains (A/B knob)
    t.epi_warp = (e && std::string(e) == "warp") ? 1 : 0;
  }
  {
    const char* e = getenv("JETB200_TCG_ROT");
    if (e && e[0] == '1' && NP == 256 && t.lg_kcs >= 1 && t.lg_kcs < t.lg_kc) {
      t.rot = 1;
      t.lg_xs = 1;
    }
  }
  t.tmem_cols = 512;
  t.ystages = ystages;
  t.rstages = rstages;
  t.rbytes_b = rb_b;
  t.rbytes_a = rb_a;
  for (int j = 0; j < t.n_oN; ++j) t.o_B[j] = sb[oN[j]];
  for (int j = 0; j < t.n_oM; ++j) t.o_A[j] = sa[oM[j]];
  for (int j = 0; j < t.lg_kc; ++j) {
    t.k_B[j] = sb[ko[j]];
    t.k_A[j] = sa[ko[j]];
  }
  auto raw_off_row = [](int i) { return (128 << i) ^ (i < 3 ? (16 << i) : 0); };
  auto raw_off_k = [](int j) { return j == 0 ? 8 : (16 << (j - 1)); };
  std::vector<std::pair<int64_t, int32_t>> bb, aa;
  for (int i = 0; i < 7; ++i) bb.push_back({sb[tN[i]], raw_off_row(i)});
  for (int j = 0; j < 4; ++j) bb.push_back({sb[kc[j]], raw_off_k(j)});
  for (int i = 0; i < tmt; ++i) aa.push_back({sa[tM[i]], raw_off_row(i)});
  for (int j = 0; j < 4; ++j) aa.push_back({sa[kc[j]], raw_off_k(j)});
  std::sort(bb.begin(), bb.end());
  std::sort(aa.begin(), aa.end());
  for (size_t j = 0; j < bb.size(); ++j) { t.gB[j] = bb[j].first; t.sB[j] = bb[j].second; }
  for (size_t j = 0; j < aa.size(); ++j) { t.gA[j] = aa[j].first; t.sA[j] = aa[j].second; }
  t.n_tiles = int64_t(1) << (t.n_oN + t.n_oM);
  // TMA chunk loads (default; JETB200_K3_TMA=0 keeps the cp.async gathers): B chunk = 7 row + 4
  // K bits, A chunk = tmt M + 4 K bits, each <= 5 stride runs holding the operand's stride-1 bit
  {
    std::vector<int64_t> ib, ia;
    for (int i = 0; i < 7; ++i) ib.push_back(sb[tN[i]]);
    for (int j = 0; j < 4; ++j) ib.push_back(sb[kc[j]]);
    for (int i = 0; i < tmt; ++i) ia.push_back(sa[tM[i]]);
    for (int j = 0; j < 4; ++j) ia.push_back(sa[kc[j]]);
    std::vector<int> rb_, ra_;
    int nb = 0, na = 0, cb = 0, ca = 0;
    bool even = true;
    if (!en.permB)
      for (auto& x : en.sliceB) even &= (x.second % 2) == 0;
    if (!en.permA)
      for (auto& x : en.sliceA) even &= (x.second % 2) == 0;
    t.tma = (tma_enabled() && even && tma_item_dims(ib, &nb, &cb, t.xoffB, rb_) &&
             tma_item_dims(ia, &na, &ca, t.xoffA, ra_)) ? 1 : 0;
    if (t.tma) {
      t.ncopyB = nb;
      t.copyB_bytes = 8 << cb;
      t.ncopyA = na;
      t.copyA_bytes = 8 << ca;
      for (int i = 0; i < 7; ++i) t.rofsB_n[i] = 8 << rb_[i];
      for (int j = 0; j < 4; ++j) t.rofsB_k[j] = 8 << rb_[7 + j];
      for (int i = 0; i < tmt; ++i) t.rofsA_m[i] = 8 << ra_[i];
      for (int j = 0; j < 4; ++j) t.rofsA_k[j] = 8 << ra_[tmt + j];
    }
  }
  // host copies for the emulator
  en.tcB_n.clear(); en.tcB_k.clear(); en.tcgA_m.clear(); en.tcgA_k.clear(); en.tcgB_oN.clear(); en.tcgA_oM.clear();
  for (int i = 0; i < 7; ++i) en.tcB_n.push_back(sb[tN[i]]);
  for (auto b : kc) { en.tcB_k.push_back(sb[b]); en.tcgA_k.push_back(sa[b]); }
  for (auto b : ko) { en.tcB_k.push_back(sb[b]); en.tcgA_k.push_back(sa[b]); }
  for (auto b : tM) en.tcgA_m.push_back(sa[b]);
  for (auto b : oN) en.tcgB_oN.push_back(sb[b]);
  for (auto b : oM) en.tcgA_oM.push_back(sa[b]);
  en.kind = 2;
  en.smem = (size_t)(ybytes + (int64_t)rstages * (rb_b + rb_a) + ebytes + 1024);
  en.block = t.tma ? 448 : 416;
  en.n_out = t.n_tiles << (7 + tmt);
  en.grid_x = t.n_tiles;
  en.args.splits = 1;
  en.args.n_tiles = t.n_tiles;
  out.bits.clear();
  int64_t st = 1;
  for (auto b : tN) { out.bits.push_back({b, st}); st <<= 1; }
  for (auto b : tM) { out.bits.push_back({b, st}); st <<= 1; }
  for (auto b : oN) { out.bits.push_back({b, st}); st <<= 1; }
  for (auto b : oM) { out.bits.push_back({b, st}); st <<= 1; }
  return true;
}

bool tc_enabled() {
  const char* e = std::getenv("JETB200_TC");
  return !(e && e[0] == '0');
}

View fill_gett(ExecNode& en, std::map<int64_t, int64_t>& sa, std::map<int64_t, int64_t>& sb,
               const std::vector<std::pair<int64_t, int64_t>>& M, const std::vector<std::pair<int64_t, int64_t>>& N,
               const std::vector<std::pair<int64_t, int64_t>>& K, const std::vector<char>& inM,
               const std::vector<char>& inN, const std::vector<char>& inK, int esize, bool dmma);

// K4 3M (Gauss) form: opt-in (JETB200_K4_3M=1).  Measured on the C4 nodes (one B200,
// profiles/r02_nodes_C4_k4_3m.txt): 26.7-30.6 TFLOP/s algorithmic in the 3M form (4x2 warp tiles,
// one 256-thread CTA per SM) vs 28.8-32.1 in the 4M form (4x4 warp tiles, two 128-thread CTAs) --
// the 4M kernel is already at 86% of the FP64 pipe, and the 3M form's smaller warp tiles double
// the operand loads per DMMA.
bool k4_gauss_enabled() {
  const char* e = std::getenv("JETB200_K4_3M");
  return e && e[0] == '1';
}

bool dmma_enabled() {
  const char* e = std::getenv("JETB200_DMMA");
  return !(e && e[0] == '0');
}

// Split the bits of a pairwise contraction into M (A only), N (B only) and K (shared), each
// sorted by stride (lowest first).  Every shared label is summed (no hyperedges).
void split_mnk(const View& va, const View& vb, std::map<int64_t, int64_t>& sa, std::map<int64_t, int64_t>& sb,
               std::vector<std::pair<int64_t, int64_t>>& M, std::vector<std::pair<int64_t, int64_t>>& N,
               std::vector<std::pair<int64_t, int64_t>>& K) {
  for (auto& x : va.bits) sa[x.first] = x.second;
  for (auto& x : vb.bits) sb[x.first] = x.second;
  for (auto& x : va.bits) {
    if (sb.count(x.first)) K.push_back({std::min(x.second, sb[x.first]), x.first});
    else M.push_back({x.second, x.first});
  }
  for (auto& x : vb.bits)
    if (!sa.count(x.first)) N.push_back({x.second, x.first});
  std::sort(M.begin(), M.end());
  std::sort(N.begin(), N.end());
  std::sort(K.begin(), K.end());
}

// K4 tile selection (c128 on DMMA): C tile 2^tm x 2^tn with tm, tn in [3, 7] and tm + tn <= 13
// (8x8 MMA sub-tiles, at most 4x4 per warp and 8 warps), tile-K 2^tk with tk in [2, 5], each
// operand's lowest 3 address bits (128-B runs) inside the tiles, two pipeline stages within
// 200 KB of shared memory.  Returns false when the contraction has no such tile (K2 runs it).
bool plan_dmma(ExecNode& en, const View& va, const View& vb, View& out) {
  std::map<int64_t, int64_t> sa, sb;
  std::vector<std::pair<int64_t, int64_t>> M, N, K;
  split_mnk(va, vb, sa, sb, M, N, K);
  if (M.size() < 3 || N.size() < 3 || K.size() < 2) return false;
  std::vector<char> inM(M.size(), 0), inN(N.size(), 0), inK(K.size(), 0);
  auto mark_low = [&](const View& vw) {
    std::vector<std::pair<int64_t, int64_t>> s;
    for (auto& x : vw.bits) s.push_back({x.second, x.first});
    std::sort(s.begin(), s.end());
    for (size_t i = 0; i < s.size() && i < 3; ++i) {
      for (size_t j = 0; j < M.size(); ++j) if (M[j].second == s[i].second) inM[j] = 1;
      for (size_t j = 0; j < N.size(); ++j) if (N[j].second == s[i].second) inN[j] = 1;
      for (size_t j = 0; j < K.size(); ++j) if (K[j].second == s[i].second) inK[j] = 1;
    }
  };
  mark_low(va);
  mark_low(vb);
  auto cnt = [](const std::vector<char>& v) { int c = 0; for (char x : v) c += x; return c; };
  auto grow = [&](std::vector<char>& in, int target) {
    for (size_t i = 0; i < in.size() && cnt(in) < target; ++i) in[i] = 1;
  };
  // default caps tile-N at 32 and tile-K at 16 complex: 128-thread CTAs of 240 registers and
  // 80 KB, two per SM whose barriers and load phases interleave (measured 29-32 TFLOP/s vs
  // 25-31 for one 256-thread CTA with 128x64x32 tiles, profiles/r01_nodes_C4_k4_tiles.txt);
  // JETB200_DMMA_TK / _TN override (sweeps)
  int tk_cap = 4, tn_cap = 5;
  if (const char* e = getenv("JETB200_DMMA_TK")) tk_cap = std::max(2, std::min(5, atoi(e)));
  if (const char* e = getenv("JETB200_DMMA_TN")) tn_cap = std::max(3, std::min(7, atoi(e)));
  grow(inK, std::min<int>((int)K.size(), tk_cap));
  grow(inM, std::min<int>((int)M.size(), 7));
  grow(inN, std::min<int>({(int)N.size(), std::max(3, 13 - cnt(inM)), tn_cap}));
  if (cnt(inN) > 7) return false;
  const int tm = cnt(inM), tn = cnt(inN), tk = cnt(inK);
  if (tm < 3 || tn < 3 || tk < 2 || tk > 5 || tm > 7 || tm + tn > 13) return false;
  // tile-K 32 complex when the two stages fit (fewer per-item barriers and address updates per
  // MMA), else 16
  auto smem_of = [&](int k) { return 2 * ((int64_t(1) << (tm + k)) + (int64_t(1) << (k + tn))) * 16; };
  int tkk = tk;
  for (int i = (int)K.size() - 1; i >= 0 && (tm + tkk > 12 || tkk + tn > 12 || smem_of(tkk) > 200 * 1024); --i)
    if (inK[i] && tkk > 4) {
      bool low = false;   // never drop a coalescing bit
      std::vector<std::pair<int64_t, int64_t>> s2;
      for (auto& x : va.bits) s2.push_back({x.second, x.first});
      std::sort(s2.begin(), s2.end());
      for (size_t q = 0; q < s2.size() && q < 3; ++q) low |= s2[q].second == K[i].second;
      s2.clear();
      for (auto& x : vb.bits) s2.push_back({x.second, x.first});
      std::sort(s2.begin(), s2.end());
      for (size_t q = 0; q < s2.size() && q < 3; ++q) low |= s2[q].second == K[i].second;
      if (!low) { inK[i] = 0; --tkk; }
    }
  if (tm + tkk > 12 || tkk + tn > 12 || smem_of(tkk) > 200 * 1024) return false;
  out = fill_gett(en, sa, sb, M, N, K, inM, inN, inK, 16, true);
  return true;
}

// Tile selection and argument fill for one contraction (K2).  Returns the output view.
View plan_gett(ExecNode& en, const View& va, const View& vb, int esize) {
  std::map<int64_t, int64_t> sa, sb;
  for (auto& x : va.bits) sa[x.first] = x.second;
  for (auto& x : vb.bits) sb[x.first] = x.second;
  std::vector<std::pair<int64_t, int64_t>> M, N, K;  // (stride key, bit)
  for (auto& x : va.bits) {
    if (sb.count(x.first)) K.push_back({std::min(x.second, sb[x.first]), x.first});
    else M.push_back({x.second, x.first});
  }
  for (auto& x : vb.bits)
    if (!sa.count(x.first)) N.push_back({x.second, x.first});
  std::sort(M.begin(), M.end());
  std::sort(N.begin(), N.end());
  std::sort(K.begin(), K.end());
  const int coal = esize == 8 ? 4 : 3;
  const int lim = esize == 8 ? 12 : 11;  // max tile bits per operand / C tile
  std::vector<char> inM(M.size(), 0), inN(N.size(), 0), inK(K.size(), 0);
  auto idx_of = [](const std::vector<std::pair<int64_t, int64_t>>& v, int64_t bit) {
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i].second == bit) return (int)i;
    return -1;
  };
  // mandatory: the lowest `coal` address bits of each operand
  auto mandatory = [&](const View& vw) {
    std::vector<std::pair<int64_t, int64_t>> s;
    for (auto& x : vw.bits) s.push_back({x.second, x.first});
    std::sort(s.begin(), s.end());
    for (size_t i = 0; i < s.size() && (int)i < coal; ++i) {
      int j;
      if ((j = idx_of(M, s[i].second)) >= 0) inM[j] = 1;
      else if ((j = idx_of(N, s[i].second)) >= 0) inN[j] = 1;
      else if ((j = idx_of(K, s[i].second)) >= 0) inK[j] = 1;
    }
  };
  mandatory(va);
  mandatory(vb);
  auto cnt = [](const std::vector<char>& v) { int c = 0; for (char x : v) c += x; return c; };
  auto add_first = [](std::vector<char>& in) {
    for (size_t i = 0; i < in.size(); ++i)
      if (!in[i]) { in[i] = 1; return true; }
    return false;
  };
  // K: all if small, else at least up to 4 bits
  const int kfull = esize == 8 ? 5 : 4;
  if ((int)K.size() <= kfull)
    for (auto& x : inK) x = 1;
  // M up to 6 (or all), N fills the C tile, then M again
  while (cnt(inM) < std::min<int>((int)M.size(), 6) && cnt(inM) + cnt(inN) < lim && add_first(inM)) {}
  while (cnt(inM) + cnt(inN) < lim && add_first(inN)) {}
  while (cnt(inM) + cnt(inN) < lim && add_first(inM)) {}
  // K: at least 4 bits, and more while one K step moves < 4096 elements (small C tiles,
  // e.g. big x big -> small reductions, need long K steps to amortise each barrier)
  while (cnt(inK) + std::max(cnt(inM), cnt(inN)) < lim &&
         (cnt(inK) < 4 || (1 << (cnt(inM) + cnt(inK))) + (1 << (cnt(inK) + cnt(inN))) < 4096) && add_first(inK)) {}
  // enforce operand tile limits by dropping non-mandatory bits from the high end
  auto drop_last = [](std::vector<char>& in, const std::vector<char>& keep) {
    for (int i = (int)in.size() - 1; i >= 0; --i)
      if (in[i] && !keep[i]) { in[i] = 0; return true; }
    return false;
  };
  std::vector<char> keepM(M.size(), 0), keepN(N.size(), 0), keepK(K.size(), 0);
  {  // recompute mandatory sets as keep masks
    std::vector<char> sM = inM, sN = inN, sK = inK;
    std::fill(inM.begin(), inM.end(), 0);
    std::fill(inN.begin(), inN.end(), 0);
    std::fill(inK.begin(), inK.end(), 0);
    mandatory(va);
    mandatory(vb);
    keepM = inM; keepN = inN; keepK = inK;
    inM = sM; inN = sN; inK = sK;
  }
  for (int guard = 0; guard < 200; ++guard) {
    int tm = cnt(inM), tn = cnt(inN), tk = cnt(inK);
    bool ok = tm + tk <= lim && tk + tn <= lim && tm + tn <= lim;
    // thread-layout limit: C tile / (RM*RN) <= 256
    int RM = std::min(4, 1 << tm), RN = std::min(4, 1 << tn);
    ok = ok && ((1 << (tm + tn)) / (RM * RN) <= 256);
    if (ok) break;
    if (tm + tk > lim || tk + tn > lim) {
      // JETB200_K2_KEEPK=1 (sweep knob): shrink the N tile before the K tile, so small K
      // reductions stay whole inside one item (measured slower on the C3 streaming nodes:
      // 3.04 vs 3.46 TB/s, so off by default)
      static const bool keepk = [] { const char* e = std::getenv("JETB200_K2_KEEPK"); return e && e[0] == '1'; }();
      if (keepk && tk + tn > lim && tn > tm && drop_last(inN, keepN)) continue;
      if (drop_last(inK, keepK)) continue;
    }
    if (tn >= tm) {
      if (drop_last(inN, keepN)) continue;
      if (drop_last(inM, keepM)) continue;
    } else {
      if (drop_last(inM, keepM)) continue;
      if (drop_last(inN, keepN)) continue;
    }
    if (drop_last(inK, keepK)) continue;
    fail(JT_EINTERNAL, "exec: cannot fit a contraction tile");
  }
  return fill_gett(en, sa, sb, M, N, K, inM, inN, inK, esize, false);
}

// Argument fill for one contraction tile choice (K2, or K4 when dmma): gather tables, outer
// and K-loop strides, thread layout, split-K and shared memory.  Returns the output view.
View fill_gett(ExecNode& en, std::map<int64_t, int64_t>& sa, std::map<int64_t, int64_t>& sb,
               const std::vector<std::pair<int64_t, int64_t>>& M, const std::vector<std::pair<int64_t, int64_t>>& N,
               const std::vector<std::pair<int64_t, int64_t>>& K, const std::vector<char>& inM,
               const std::vector<char>& inN, const std::vector<char>& inK, int esize, bool dmma) {
  std::vector<int64_t> tM, tN, tK, oM, oN, oK;
  for (size_t i = 0; i < M.size(); ++i) (inM[i] ? tM : oM).push_back(M[i].second);
  for (size_t i = 0; i < N.size(); ++i) (inN[i] ? tN : oN).push_back(N[i].second);
  prefer_low(tN, en.pref_low);
  for (size_t i = 0; i < K.size(); ++i) (inK[i] ? tK : oK).push_back(K[i].second);
  GettArgs& g = en.args;
  std::memset(&g, 0, sizeof(g));
  g.tm = (int)tM.size();
  g.tn = (int)tN.size();
  g.tk = (int)tK.size();
  g.nA = g.tm + g.tk;
  g.nB = g.tk + g.tn;
  if (g.nA > 12 || g.nB > 12) fail(JT_EINTERNAL, "exec: tile too large");
  // operand tiles in the operand's own bit order (stride ascending): tile bit j has global
  // stride g[j] and shared-memory stride 2^j; record where each M/K/N bit landed
  {
    std::vector<std::pair<int64_t, std::pair<int, int>>> ta;  // (stride, (role 0=M 1=K, index))
    for (int i = 0; i < g.tm; ++i) ta.push_back({sa[tM[i]], {0, i}});
    for (int i = 0; i < g.tk; ++i) ta.push_back({sa[tK[i]], {1, i}});
    std::sort(ta.begin(), ta.end());
    for (size_t j = 0; j < ta.size(); ++j) {
      g.gA[j] = ta[j].first;
      (ta[j].second.first == 0 ? g.pM : g.pKA)[ta[j].second.second] = (int8_t)j;
    }
    std::vector<std::pair<int64_t, std::pair<int, int>>> tb;
    for (int i = 0; i < g.tn; ++i) tb.push_back({sb[tN[i]], {0, i}});
    for (int i = 0; i < g.tk; ++i) tb.push_back({sb[tK[i]], {1, i}});
    std::sort(tb.begin(), tb.end());
    for (size_t j = 0; j < tb.size(); ++j) {
      g.gB[j] = tb[j].first;
      (tb[j].second.first == 0 ? g.pN : g.pKB)[tb[j].second.second] = (int8_t)j;
    }
  }
  // outer bits: N (B-stride order) then M (A-stride order) -> blockIdx.x bits
  std::vector<int64_t> outer;
  for (auto b : oN) outer.push_back(b);
  for (auto b : oM) outer.push_back(b);
  if ((int)outer.size() > 31) fail(JT_ERESOURCE, "exec: too many output tiles");
  if ((int)outer.size() > kMaxOuter || (int)oK.size() > kMaxOuter) fail(JT_EINTERNAL, "exec: too many bits");
  g.n_outer = (int)outer.size();
  for (int j = 0; j < g.n_outer; ++j) {
    g.o_sA[j] = sa.count(outer[j]) ? sa[outer[j]] : 0;
    g.o_sB[j] = sb.count(outer[j]) ? sb[outer[j]] : 0;
  }
  g.n_ok = (int)oK.size();
  if (g.n_ok > 40) fail(JT_ERESOURCE, "exec: contraction too large");
  for (int j = 0; j < g.n_ok; ++j) {
    g.ok_sA[j] = sa[oK[j]];
    g.ok_sB[j] = sb[oK[j]];
  }
  g.n_tiles = int64_t(1) << g.n_outer;
  g.k_iters = int64_t(1) << g.n_ok;
  int64_t splits = 1;
  if (dmma) {
    // K4 warp layout: 8x8 sub-tiles, up to 4x4 per warp, TY x TX warps (<= 8)
    en.kind = 3;
    en.RM = std::min(4, 1 << (g.tm - 3));
    en.RN = std::min(4, 1 << (g.tn - 3));
    // 3M (Gauss) form (opt-in, JETB200_K4_3M=1): three accumulators per sub-tile, so warp tiles
    // of <= 8 sub-tiles (4x2) and CTAs of <= 8 warps
    g.gauss = 0;
    if (k4_gauss_enabled()) {
      const int rn = std::min(2, 1 << (g.tn - 3));
      if (32 * ((1 << (g.tm - 3)) / en.RM) * ((1 << (g.tn - 3)) / rn) <= 256) {
        en.RN = rn;
        g.gauss = 1;
      }
    }
    g.TY = (1 << (g.tm - 3)) / en.RM;
    g.TX = (1 << (g.tn - 3)) / en.RN;
    g.KG = 1;
    en.block = 32 * g.TX * g.TY;
    // split-K to fill the machine: choose the split count (<= 512, <= K iterations / 4) with the
    // smallest wave-quantisation loss over ~148 x (CTAs per SM) slots, 0.2% per extra split for
    // the partial sums.  (Round 1 capped it at 8: the C4 width-30 plan's inner-product node --
    // 2 output tiles, K = 2^24 -- then ran 16 CTAs at 0.5 TFLOP/s, profiles/r02_nodes_C4_k4.txt.)
    const int cps = en.block >= 256 ? 1 : (en.block >= 128 ? 2 : 4);
    const double slots = 148.0 * cps;
    double best = 1e30;
    const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(512, g.k_iters / 4));
    for (int64_t s2 = 1; s2 <= smax; ++s2) {
      const double items = (double)(g.n_tiles * s2);
      const double waves = std::ceil(items / slots);
      const double loss = waves * slots / items * (1.0 + 0.002 * (double)(s2 - 1));
      if (loss < best - 1e-9) { best = loss; splits = s2; }
    }
    const int64_t cbytes = (g.n_tiles << (g.tm + g.tn)) * esize;
    while (splits > 1 && splits * cbytes > (int64_t(1) << 32)) --splits;
    g.splits = (int32_t)splits;
    g.vecA = g.vecB = 0;
    g.dbuf = 1;
    const int64_t stage = (int64_t(1) << g.nA) + (int64_t(1) << g.nB);
    en.smem = (size_t)(2 * stage * esize + 2 * 4 * (int64_t(1) << g.tk));
    en.n_out = g.n_tiles << (g.tm + g.tn);
    View vc;
    int64_t st = 1;
    for (auto b : tN) { vc.bits.push_back({b, st}); st <<= 1; }
    for (auto b : tM) { vc.bits.push_back({b, st}); st <<= 1; }
    for (auto b : outer) { vc.bits.push_back({b, st}); st <<= 1; }
    return vc;
  }
  en.RM = std::min(4, 1 << g.tm);
  en.RN = std::min(4, 1 << g.tn);
  g.TX = (1 << g.tn) / en.RN;
  g.TY = (1 << g.tm) / en.RM;
  const int TXY = g.TX * g.TY;
  g.KG = std::max(1, std::min(256 / TXY, 1 << g.tk));
  en.block = std::max(32, (TXY * g.KG + 31) / 32 * 32);
  // cross-CTA split-K when the grid is small and the K loop is long
  const int64_t target = 148 * 4;
  if (g.n_tiles < target && g.k_iters > 1) {
    splits = std::min<int64_t>(g.k_iters, (target + g.n_tiles - 1) / g.n_tiles);
    const int64_t cbytes = (g.n_tiles << (g.tm + g.tn)) * esize;
    const int64_t cap = int64_t(1) << 31;  // partial buffer <= 2 GiB
    while (splits > 1 && splits * cbytes > cap) splits /= 2;
  }
  g.splits = (int32_t)splits;
  // 16-B element-pair copies (c64) when tile bit 0 is unit-stride and every other stride is even
  auto vec_ok = [&](const int64_t* gt, int n, const int64_t* o, const int64_t* ok) {
    if (esize != 8 || n < 1 || gt[0] != 1) return 0;
    for (int j = 1; j < n; ++j) if (gt[j] & 1) return 0;
    for (int j = 0; j < g.n_outer; ++j) if (o[j] & 1) return 0;
    for (int j = 0; j < g.n_ok; ++j) if (ok[j] & 1) return 0;
    return 1;
  };
  g.vecA = vec_ok(g.gA, g.nA, g.o_sA, g.ok_sA);
  g.vecB = vec_ok(g.gB, g.nB, g.o_sB, g.ok_sB);
  g.dbuf = 1;
  const int64_t stage = (int64_t(1) << g.nA) + (int64_t(1) << g.nB);
  const int64_t red = g.KG > 1 ? (int64_t)(g.KG - 1) * (int64_t(1) << (g.tm + g.tn)) : 0;
  en.smem = (size_t)((2 * stage + red) * esize + 2 * 4 * (int64_t(1) << g.tk));
  en.n_out = g.n_tiles << (g.tm + g.tn);
  // output view: [tile N bits][tile M bits][outer bits]
  View vc;
  int64_t st = 1;
  for (auto b : tN) { vc.bits.push_back({b, st}); st <<= 1; }
  for (auto b : tM) { vc.bits.push_back({b, st}); st <<= 1; }
  for (auto b : outer) { vc.bits.push_back({b, st}); st <<= 1; }
  return vc;
}

Layout compile(const jt_plan& plan, int esize) {
  const bool use_tc = tc_enabled();
  const bool use_dmma = dmma_enabled();
  const char* fg = std::getenv("JETB200_TCG_FORCE");  // tests: route K3-eligible nodes to K3g
  const bool force_tcg = fg && fg[0] == '1';
  Layout L;
  L.esize = esize;
  const jt_network& net = plan.net;
  const int lb = ilog2_exact(net.d);
  const int64_t nt = (int64_t)net.tensors.size();
  const int64_t NN = (int64_t)plan.nodes.size();
  std::vector<View> views(NN);
  std::vector<std::vector<std::pair<int, int64_t>>> leaf_slices(nt);
  L.leaf_off.assign(nt, 0);
  L.node_off.assign(NN, -1);
  int64_t off = 0;
  for (int64_t t = 0; t < nt; ++t) {
    const auto& ls = net.tensors[t].labels;
    int64_t stride = 1;
    for (int i = (int)ls.size() - 1; i >= 0; --i) {  // row-major: last label fastest
      auto it = plan.slice_pos.find(ls[i]);
      if (it != plan.slice_pos.end()) {
        leaf_slices[t].push_back({it->second, stride});
      } else {
        for (int j = 0; j < lb; ++j) views[t].bits.push_back({ls[i] * lb + j, stride << j});
      }
      stride *= net.d;
    }
    L.leaf_off[t] = off;
    L.node_off[t] = off;
    off += align_up((int64_t)net.tensors[t].data.size() * esize);
  }
  L.leaf_bytes = off;
  // execution order: post-order, the child with the larger peak first (Sethi-Ullman style)
  std::vector<double> sz(NN), peak(NN);
  for (int64_t v = 0; v < NN; ++v) sz[v] = std::exp2(plan.nodes[v].log2size);
  for (int64_t v = 0; v < nt; ++v) peak[v] = 0;
  for (int64_t v = nt; v < NN; ++v) {
    const PlanNode& n = plan.nodes[v];
    double p1 = std::max({peak[n.left], sz[n.left] + peak[n.right], sz[n.left] + sz[n.right] + sz[v]});
    double p2 = std::max({peak[n.right], sz[n.right] + peak[n.left], sz[n.left] + sz[n.right] + sz[v]});
    peak[v] = std::min(p1, p2);
  }
  std::vector<int64_t> ord;
  {
    std::vector<std::pair<int64_t, int>> st;
    st.push_back({NN - 1, 0});
    while (!st.empty()) {
      auto& top = st.back();
      int64_t v = top.first;
      if (v < nt) { st.pop_back(); continue; }
      const PlanNode& n = plan.nodes[v];
      double p1 = std::max({peak[n.left], sz[n.left] + peak[n.right]});
      double p2 = std::max({peak[n.right], sz[n.right] + peak[n.left]});
      int64_t first = p1 <= p2 ? n.left : n.right, second = p1 <= p2 ? n.right : n.left;
      if (top.second == 0) { top.second = 1; st.push_back({first, 0}); }
      else if (top.second == 1) { top.second = 2; st.push_back({second, 0}); }
      else { ord.push_back(v); st.pop_back(); }
    }
  }
  // per node descriptors
  std::vector<int64_t> pos(NN, -1);
  for (size_t i = 0; i < ord.size(); ++i) pos[ord[i]] = (int64_t)i;
  for (int64_t v : ord) {
    const PlanNode& n = plan.nodes[v];
    ExecNode en;
    en.v = v;
    auto nfree = [&](int64_t x, int64_t y) {
      std::map<int64_t, int> s;
      for (auto& b : views[y].bits) s[b.first] = 1;
      int c = 0;
      for (auto& b : views[x].bits) c += !s.count(b.first);
      return c;
    };
    int fl = nfree(n.left, n.right), fr = nfree(n.right, n.left);
    en.opA = fl <= fr ? n.left : n.right;
    en.opB = fl <= fr ? n.right : n.left;
    // consumer-ordered output layouts: opt-in (JETB200_CONSUMER_LAYOUT=1); measured neutral to
    // slightly slower on C3 without the 16-B gathers (10.34 s vs 10.03 s)
    const char* cl = std::getenv("JETB200_CONSUMER_LAYOUT");
    if (n.parent >= 0) {
      const PlanNode& par = plan.nodes[n.parent];
      const int64_t sib = par.left == v ? par.right : par.left;
      for (int64_t l : n.labels)
        if (std::find(plan.nodes[sib].labels.begin(), plan.nodes[sib].labels.end(), l) != plan.nodes[sib].labels.end())
          for (int j = 0; j < lb; ++j) en.consumer_k.push_back(l * lb + j);
      if (cl && cl[0] == '1') en.pref_low = en.consumer_k;
    }
    if (en.opA < nt) en.sliceA = leaf_slices[en.opA];
    if (en.opB < nt) en.sliceB = leaf_slices[en.opB];
    if (en.sliceA.size() > 4 || en.sliceB.size() > 4) fail(JT_EUSAGE, "exec: more than 4 sliced labels on one leaf");
    View tv;
    if (use_tc && !force_tcg && plan_tc(en, views[en.opA], views[en.opB], esize, tv)) views[v] = tv;
    else if (use_tc && plan_tcg(en, views[en.opA], views[en.opB], esize, tv)) views[v] = tv;
    else if (esize == 16 && use_dmma && plan_dmma(en, views[en.opA], views[en.opB], tv)) views[v] = tv;
    else {
      views[v] = plan_gett(en, views[en.opA], views[en.opB], esize);
      if (use_tc) plan_stream(en, views[en.opA], views[en.opB], views[v], esize);  // K2 layout kept
    }
    en.maxpos = n.maxpos;
    en.flop = n.flop;
    en.bytes = n.bytes8 / 8.0 * esize;
    L.order.push_back(en);
  }
  // workspace: interval allocation of node outputs over execution positions.
  // A node whose parent is recomputed more often than itself (maxpos(v) < maxpos(parent))
  // is a prefix-cache entry and lives for the whole run.
  struct Buf { int64_t v, size, start, end, off; };
  std::vector<Buf> bufs;
  const int64_t INF = std::numeric_limits<int64_t>::max();
  for (const ExecNode& en : L.order) {
    const int64_t v = en.v;
    const PlanNode& n = plan.nodes[v];
    Buf b{v, align_up(en.n_out * esize), pos[v], 0, 0};
    if (n.parent < 0) { b.start = 0; b.end = INF; }
    else if (plan.nodes[n.parent].maxpos > n.maxpos) { b.start = 0; b.end = INF; }
    else b.end = pos[n.parent];
    bufs.push_back(b);
  }
  std::vector<size_t> bi(bufs.size());
  for (size_t i = 0; i < bi.size(); ++i) bi[i] = i;
  std::sort(bi.begin(), bi.end(), [&](size_t x, size_t y) {
    return bufs[x].size > bufs[y].size || (bufs[x].size == bufs[y].size && x < y);
  });
  std::vector<size_t> placed;
  int64_t inter = 0;
  for (size_t i : bi) {
    Buf& b = bufs[i];
    std::vector<std::pair<int64_t, int64_t>> occ;
    for (size_t j : placed) {
      const Buf& o = bufs[j];
      if (o.start <= b.end && b.start <= o.end) occ.push_back({o.off, o.off + o.size});
    }
    std::sort(occ.begin(), occ.end());
    int64_t cand = 0;
    for (auto& iv : occ) {
      if (cand + b.size <= iv.first) break;
      cand = std::max(cand, iv.second);
    }
    b.off = cand;
    inter = std::max(inter, cand + b.size);
    placed.push_back(i);
  }
  // memory report: every intermediate kept (no deletion); the peak of live intermediates over
  // the execution order (deletion after the last use); the prefix-cache entries resident for the
  // whole run; the same peak if nothing were kept across slices (no shared work)
  {
    std::vector<int64_t> delta(ord.size() + 1, 0), delta_ns(ord.size() + 1, 0);
    int64_t always = 0, always_ns = 0;
    for (const Buf& b : bufs) {
      L.mem_no_deletion += b.size;
      const PlanNode& n = plan.nodes[b.v];
      const bool cache = n.parent >= 0 && plan.nodes[n.parent].maxpos > n.maxpos;
      if (cache) L.mem_cache += b.size;
      if (b.end == INF) always += b.size;
      else { delta[b.start] += b.size; delta[b.end + 1] -= b.size; }
      const int64_t s0 = pos[b.v], e0 = n.parent < 0 ? (int64_t)ord.size() - 1 : pos[n.parent];
      if (n.parent < 0) always_ns += b.size;
      else { delta_ns[s0] += b.size; delta_ns[e0 + 1] -= b.size; }
    }
    int64_t cur = 0, cur_ns = 0;
    for (size_t q = 0; q < ord.size(); ++q) {
      cur += delta[q];
      cur_ns += delta_ns[q];
      L.mem_peak_live = std::max(L.mem_peak_live, cur + always);
      L.mem_peak_live_noshare = std::max(L.mem_peak_live_noshare, cur_ns + always_ns);
    }
  }
  L.inter_base = align_up(L.leaf_bytes);
  L.inter_bytes = inter;
  for (const Buf& b : bufs) L.node_off[b.v] = L.inter_base + b.off;
  L.scratch_base = align_up(L.inter_base + L.inter_bytes);
  int64_t scratch = 0;
  for (ExecNode& en : L.order) {
    if (en.args.splits > 1) scratch = std::max(scratch, align_up(en.n_out * esize * en.args.splits));
    scratch = std::max(scratch, en.perm_bytes);  // K1-fed K3g operand copies (used within the node)
    en.out_off = L.node_off[en.v];
    en.part_off = L.scratch_base;
    en.perm_off = L.scratch_base;
  }
  L.scratch_bytes = scratch;
  L.vals_base = align_up(L.scratch_base + L.scratch_bytes);
  L.vals_cap = 1;
  while (L.vals_cap < plan.n_sl && L.vals_cap < (int64_t(1) << 20)) L.vals_cap <<= 1;
  L.acc_base = align_up(L.vals_base + L.vals_cap * 16);
  L.state_base = align_up(L.acc_base + 16 * plan.n_batch);
  L.total = align_up(L.state_base + (int64_t)sizeof(SliceState));
  return L;
}


// ---------------------------------------------------------------- debug: host emulation
// Test-only (jt_debug_emulate_host): executes the compiled K2 descriptors, the workspace
// layout and the prefix-cache schedule on host memory with the kernel's exact index
// arithmetic, so descriptor/layout/scheduling bugs are caught by CPU tests.  Never used by
// jt_exec_* (there is no CPU execution path in the product).
template <typename R>
void emulate_gett(const GettArgs& p, char* ws, const ExecNode& en, const std::vector<std::pair<int64_t, int64_t>>& ab_off) {
  using C2 = typename V2<R>::t;
  (void)en;
  const C2* A = reinterpret_cast<const C2*>(ws + ab_off[0].first) + ab_off[0].second;
  const C2* B = reinterpret_cast<const C2*>(ws + ab_off[1].first) + ab_off[1].second;
  C2* C = reinterpret_cast<C2*>(ws + ab_off[2].first);
  C2* P = reinterpret_cast<C2*>(ws + ab_off[3].first);
  auto gofs = [](const int64_t* g, int n, int e) {
    int64_t o = 0;
    for (int j = 0; j < n; ++j) if ((e >> j) & 1) o += g[j];
    return o;
  };
  auto dep = [](int v, const int8_t* pos, int n) {
    int r = 0;
    for (int i = 0; i < n; ++i) r |= ((v >> i) & 1) << pos[i];
    return r;
  };
  std::vector<C2> sA(size_t(1) << p.nA), sB(size_t(1) << p.nB), acc(size_t(1) << (p.tm + p.tn));
  for (int64_t tile = 0; tile < p.n_tiles; ++tile)
    for (int split = 0; split < p.splits; ++split) {
      int64_t baseA = 0, baseB = 0;
      for (int j = 0; j < p.n_outer; ++j)
        if ((tile >> j) & 1) { baseA += p.o_sA[j]; baseB += p.o_sB[j]; }
      const int64_t it0 = (int64_t)split * p.k_iters / p.splits, it1 = (int64_t)(split + 1) * p.k_iters / p.splits;
      for (auto& x : acc) { x.x = 0; x.y = 0; }
      for (int64_t it = it0; it < it1; ++it) {
        int64_t oa = baseA, ob = baseB;
        for (int j = 0; j < p.n_ok; ++j)
          if ((it >> j) & 1) { oa += p.ok_sA[j]; ob += p.ok_sB[j]; }
        for (int e = 0; e < (1 << p.nA); ++e) sA[e] = A[oa + gofs(p.gA, p.nA, e)];
        for (int e = 0; e < (1 << p.nB); ++e) sB[e] = B[ob + gofs(p.gB, p.nB, e)];
        for (int k = 0; k < (1 << p.tk); ++k)
          for (int m = 0; m < (1 << p.tm); ++m)
            for (int n = 0; n < (1 << p.tn); ++n) {
              const C2 a = sA[dep(m, p.pM, p.tm) | dep(k, p.pKA, p.tk)];
              const C2 b = sB[dep(n, p.pN, p.tn) | dep(k, p.pKB, p.tk)];
              C2& c = acc[(m << p.tn) + n];
              c.x += a.x * b.x - a.y * b.y;
              c.y += a.x * b.y + a.y * b.x;
            }
      }
      C2* out = p.splits == 1 ? C : P;
      const int64_t base = ((int64_t)(p.splits == 1 ? 0 : split) * p.n_tiles + tile) << (p.tm + p.tn);
      for (size_t i = 0; i < acc.size(); ++i) out[base + i] = acc[i];
    }
  if (p.splits > 1) {
    const int64_t n = p.n_tiles << (p.tm + p.tn);
    for (int64_t i = 0; i < n; ++i) {
      C2 s = P[i];
      for (int k = 1; k < p.splits; ++k) { s.x += P[k * n + i].x; s.y += P[k * n + i].y; }
      C[i] = s;
    }
  }
}

// The packed landing of a bulk-copied item: element e sits at global base + xoff[e >> log2 copy
// elements] + (e & (copy elements - 1)).
std::vector<int64_t> landing(int64_t base, int ncopy, int copy_bytes, const int64_t* xoff, size_t n) {
  std::vector<int64_t> b(n);
  const int64_t ce = copy_bytes / 8;
  if ((int64_t)ncopy * ce != (int64_t)n) fail(JT_EINTERNAL, "emulate: bulk copies do not tile the item");
  for (size_t e = 0; e < n; ++e) b[e] = base + xoff[(int64_t)e / ce] + (int64_t)e % ce;
  return b;
}

// K2s: every column's B offsets from the descriptor (the kernel's four 9-bit tables are the
// GF(2)-linear bit -> stride map, recomputed here bit by bit), the 16-B pair alignment, and the
// output layout [n_lo columns][M][rest], with the kernel's FP32 complex arithmetic order
void emulate_stream(const StreamArgs& p, const ExecNode& en, char* ws, const std::vector<std::pair<int64_t, int64_t>>& off) {
  const float2* A = reinterpret_cast<const float2*>(ws + off[0].first) + off[0].second;
  const float2* B = reinterpret_cast<const float2*>(ws + off[1].first) + off[1].second;
  float2* C = reinterpret_cast<float2*>(ws + off[2].first);
  const int tm = en.args.tm, kt = en.args.tk, nm = 1 << tm, nk = 1 << kt;
  for (int k = 0; k < nk; ++k) {
    int64_t o = 0;
    for (int j = 0; j < kt; ++j) if ((k >> j) & 1) o += en.stK[j];
    if (o != p.kofs[k]) fail(JT_EINTERNAL, "emulate: K2s k offsets");
  }
  const int64_t ncol = int64_t(1) << p.n_cols, lo_mask = (int64_t(1) << p.n_lo) - 1;
  for (int64_t c = 0; c < ncol; ++c) {
    int64_t bo = 0;
    for (int h = 0; h < 4; ++h) {
      const int v = (int)((c >> (9 * h)) & 511);
      for (int b = 0; b < 9; ++b)
        if (((v >> b) & 1) && 9 * h + b < p.n_cols) bo += p.sN[9 * h + b];
    }
    float2 bv[8];
    for (int k = 0; k < nk; ++k) {
      if (p.vec && (k % 2) == 0 && ((off[1].second + bo + p.kofs[k]) % 2) != 0)
        fail(JT_EINTERNAL, "emulate: K2s 16-B pair misaligned");
      bv[k] = B[bo + p.kofs[k]];
    }
    float2* out = C + (c & lo_mask) + ((c >> p.n_lo) << (p.n_lo + tm));
    for (int m = 0; m < nm; ++m) {
      float re = 0.f, im = 0.f;
      for (int k = 0; k < nk; ++k) {
        const float2 x = A[p.aofs[m * nk + k]];
        re = std::fma(x.x, bv[k].x, re);
        re = std::fma(-x.y, bv[k].y, re);
        im = std::fma(x.x, bv[k].y, im);
        im = std::fma(x.y, bv[k].x, im);
      }
      out[(int64_t)m << p.n_lo] = make_float2(re, im);
    }
  }
}

void emulate_tc(const TcArgs& p, const ExecNode& en, char* ws, const std::vector<std::pair<int64_t, int64_t>>& off) {
  const float2* A = reinterpret_cast<const float2*>(ws + off[0].first) + off[0].second;
  const float2* B = reinterpret_cast<const float2*>(ws + off[1].first) + off[1].second;
  float2* C = reinterpret_cast<float2*>(ws + off[2].first);
  const int nm = 1 << p.tm, nk = 1 << p.K;
  std::vector<float2> a((size_t)nm * nk);
  for (int m = 0; m < nm; ++m)
    for (int k = 0; k < nk; ++k) {
      int64_t ao = 0;
      for (int i = 0; i < p.tm; ++i) if ((m >> i) & 1) ao += p.aM[i];
      for (int i = 0; i < p.K; ++i) if ((k >> i) & 1) ao += p.aK[i];
      a[(size_t)m * nk + k] = A[ao];
    }
  if (p.tma) {
    // the TMA-engine landing of every item, read back through rofs_row / rofs_k, must be the
    // item's B elements
    for (int64_t t = 0; t < p.n_tiles; ++t)
      for (int c = 0; c < p.n_kc; ++c) {
        int64_t base = 0;
        for (int j = 0; j < p.n_outer; ++j) if ((t >> j) & 1) base += p.o_sB[j];
        for (int j = 0; j < p.K - p.tkc; ++j) if ((c >> j) & 1) base += p.o_kB[j];
        const std::vector<int64_t> box = landing(base, p.ncopy, p.copy_bytes, p.xoff, (size_t)128 << p.tkc);
        for (int n = 0; n < 128; ++n)
          for (int k = 0; k < (1 << p.tkc); ++k) {
            int64_t want = base, ro = 0;
            for (int i = 0; i < 7; ++i) if ((n >> i) & 1) { want += en.tcB_n[i]; ro += p.rofs_row[i]; }
            for (int i = 0; i < p.tkc; ++i) if ((k >> i) & 1) { want += en.tcB_k[i]; ro += p.rofs_k[i]; }
            if (box[(size_t)(ro / 8)] != want) fail(JT_EINTERNAL, "emulate: K3 TMA landing mismatch");
          }
      }
  }
  for (int64_t t = 0; t < p.n_tiles; ++t) {
    int64_t base = 0;
    for (int j = 0; j < p.n_outer; ++j) if ((t >> j) & 1) base += p.o_sB[j];
    for (int n = 0; n < 128; ++n) {
      int64_t bn = base;
      for (int i = 0; i < 7; ++i) if ((n >> i) & 1) bn += en.tcB_n[i];
      for (int m = 0; m < nm; ++m) {
        double re = 0, im = 0;
        for (int k = 0; k < nk; ++k) {
          int64_t bo = bn;
          for (int i = 0; i < p.K; ++i) if ((k >> i) & 1) bo += en.tcB_k[i];
          const float2 x = a[(size_t)m * nk + k], y = B[bo];
          re += (double)x.x * y.x - (double)x.y * y.y;
          im += (double)x.x * y.y + (double)x.y * y.x;
        }
        C[(t << (7 + p.tm)) + (p.mlow ? ((int64_t)n << p.tm) + m : ((int64_t)m << 7) + n)] =
            make_float2((float)re, (float)im);
      }
    }
  }
}

void emulate_tcg(const TcgArgs& p, const ExecNode& en, char* ws, const std::vector<std::pair<int64_t, int64_t>>& off) {
  const float2* A = reinterpret_cast<const float2*>(ws + off[0].first) + off[0].second;
  const float2* B = reinterpret_cast<const float2*>(ws + off[1].first) + off[1].second;
  // K1-fed operands: the bit-gather into the K3g layout (dst bit j <- source stride s[j])
  std::vector<float2> pa, pb;
  auto gather = [](const float2* src, const GatherArgs& g, std::vector<float2>& dst) {
    dst.resize(size_t(1) << g.n_bits);
    for (size_t i = 0; i < dst.size(); ++i) {
      int64_t o = 0;
      for (int j = 0; j < g.n_bits; ++j) if ((i >> j) & 1) o += g.s[j];
      dst[i] = src[o];
    }
  };
  if (en.permB) { gather(B, en.gB, pb); B = pb.data(); }
  if (en.permA) { gather(A, en.gA, pa); A = pa.data(); }
  float2* C = reinterpret_cast<float2*>(ws + off[2].first);
  const int MT = 1 << p.tmt;
  const int64_t nk = int64_t(1) << (int)en.tcB_k.size();
  auto bits = [](int64_t v, const std::vector<int64_t>& st) {
    int64_t o = 0;
    for (size_t j = 0; j < st.size(); ++j) if ((v >> j) & 1) o += st[j];
    return o;
  };
  if (p.tma) {
    // TMA-engine landings of every (tile, chunk), read back through the rofs tables
    const std::vector<int64_t> kcB(en.tcB_k.begin(), en.tcB_k.begin() + 4), koB(en.tcB_k.begin() + 4, en.tcB_k.end());
    const std::vector<int64_t> kcA(en.tcgA_k.begin(), en.tcgA_k.begin() + 4), koA(en.tcgA_k.begin() + 4, en.tcgA_k.end());
    for (int64_t t = 0; t < p.n_tiles; ++t)
      for (int64_t c = 0; c < (int64_t(1) << p.lg_kc); ++c) {
        const int64_t bo = bits(t, en.tcgB_oN) + bits(c, koB), ao = bits(t >> p.n_oN, en.tcgA_oM) + bits(c, koA);
        const auto bb = landing(bo, p.ncopyB, p.copyB_bytes, p.xoffB, 2048);
        const auto ab = landing(ao, p.ncopyA, p.copyA_bytes, p.xoffA, (size_t)MT * 16);
        for (int k = 0; k < 16; ++k) {
          int32_t kb = 0, ka = 0;
          for (int j = 0; j < 4; ++j) if ((k >> j) & 1) { kb += p.rofsB_k[j]; ka += p.rofsA_k[j]; }
          for (int n = 0; n < 128; ++n) {
            int32_t r = kb;
            for (int i = 0; i < 7; ++i) if ((n >> i) & 1) r += p.rofsB_n[i];
            if (bb[r / 8] != bo + bits(n, en.tcB_n) + bits(k, kcB)) fail(JT_EINTERNAL, "emulate: K3g B landing mismatch");
          }
          for (int m = 0; m < MT; ++m) {
            int32_t r = ka;
            for (int i = 0; i < p.tmt; ++i) if ((m >> i) & 1) r += p.rofsA_m[i];
            if (ab[r / 8] != ao + bits(m, en.tcgA_m) + bits(k, kcA)) fail(JT_EINTERNAL, "emulate: K3g A landing mismatch");
          }
        }
      }
  }
  for (int64_t t = 0; t < p.n_tiles; ++t) {
    const int64_t bo = bits(t, en.tcgB_oN), ao = bits(t >> p.n_oN, en.tcgA_oM);
    for (int n = 0; n < 128; ++n)
      for (int m = 0; m < MT; ++m) {
        double re = 0, im = 0;
        for (int64_t k = 0; k < nk; ++k) {
          const float2 a = A[ao + bits(m, en.tcgA_m) + bits(k, en.tcgA_k)];
          const float2 b = B[bo + bits(n, en.tcB_n) + bits(k, en.tcB_k)];
          re += (double)a.x * b.x - (double)a.y * b.y;
          im += (double)a.x * b.y + (double)a.y * b.x;
        }
        C[(t << (7 + p.tmt)) + ((int64_t)m << 7) + n] = make_float2((float)re, (float)im);
      }
  }
}

template <typename R>
void emulate_host(const jt_plan& plan, int esize, int64_t b, int64_t e, double* h_vals, bool reuse) {
  using C2 = typename V2<R>::t;
  Layout L = compile(plan, esize);
  std::vector<char> ws(L.total, 0);
  const int64_t nt = (int64_t)plan.net.tensors.size();
  for (int64_t t = 0; t < nt; ++t) {
    const auto& data = plan.net.tensors[t].data;
    C2* dst = reinterpret_cast<C2*>(ws.data() + L.leaf_off[t]);
    for (size_t i = 0; i < data.size(); ++i) { dst[i].x = (R)data[i].real(); dst[i].y = (R)data[i].imag(); }
  }
  const int k = (int)plan.sliced.size(), d = plan.net.d;
  std::vector<int> dig(k), prev(k);
  int64_t last = -1;
  for (int64_t s = b; s < e; ++s) {
    int64_t x = s;
    for (int q = k - 1; q >= 0; --q) { dig[q] = (int)(x % d); x /= d; }
    int j = -1;
    if (reuse && last >= 0) {
      j = k;
      for (int q = 0; q < k; ++q)
        if (dig[q] != prev[q]) { j = q; break; }
    }
    for (const ExecNode& en : L.order) {
      if (en.maxpos < j) continue;
      int64_t offA = 0, offB = 0;
      for (auto& sl : en.sliceA) offA += (int64_t)dig[sl.first] * sl.second;
      for (auto& sl : en.sliceB) offB += (int64_t)dig[sl.first] * sl.second;
      std::vector<std::pair<int64_t, int64_t>> offs = {{L.node_off[en.opA], offA}, {L.node_off[en.opB], offB},
                                                       {en.out_off, 0}, {en.part_off, 0}};
      if (en.kind == 4) emulate_stream(en.st, en, ws.data(), offs);
      else if (en.kind == 2) emulate_tcg(en.tcg, en, ws.data(), offs);
      else if (en.kind == 1) emulate_tc(en.tc, en, ws.data(), offs);
      else emulate_gett<R>(en.args, ws.data(), en, offs);
    }
    const C2 r = *reinterpret_cast<const C2*>(ws.data() + L.order.back().out_off);
    h_vals[2 * (s - b)] = (double)r.x;
    h_vals[2 * (s - b) + 1] = (double)r.y;
    last = s;
    prev = dig;
  }
}

}  // namespace

void debug_emulate_host(const jt_plan& plan, jt_dtype dt, int64_t b, int64_t e, double* h_vals, bool reuse) {
  if (b < 0 || e > plan.n_sl || b > e) fail(JT_EUSAGE, "emulate: bad range");
  if (dt == JT_C64) emulate_host<float>(plan, 8, b, e, h_vals, reuse);
  else emulate_host<double>(plan, 16, b, e, h_vals, reuse);
}

namespace {
}  // namespace

}  // namespace jt

struct jt_exec {
  jt::Layout L;
  jt_dtype dtype = JT_C64;
  int device = 0;
  char* ws = nullptr;
  int64_t ws_bytes = 0;
  cudaStream_t stream = nullptr;
  int64_t n_sl = 1;       // runs: summed slices x batch
  int k = 0, d = 2;       // loop positions (summed + batch), qudit dimension
  int n_summed = 0;       // first batch position
  int64_t n_batch = 1;
  int64_t last = -1;  // last slice whose values are in the prefix cache, -1 = cold
  jt_exec_stats stats{};
  std::vector<char> host_leaves;   // leaf data converted to the exec dtype
  char* pinned = nullptr;          // pinned staging buffer for uploads
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // event pool for K2 timing
  size_t ev_used = 0;
  std::vector<std::pair<double, double>> ev_work;        // (bytes, flop) of each timed launch
  std::vector<int> ev_kind;                              // 0 = K2, 1 = K3
  bool use_graphs = true;
  bool pdl = true;  // programmatic dependent launch between the kernels of a slice
  bool pdl_small = false;  // PDL only for the small CUDA-core launches (K2, K2s, reductions, K6)
  std::vector<cudaGraphExec_t> graphs;   // per prefix-cache level j+1 (j = -1..k)
  std::vector<jt_exec_stats> graph_stats;
  double* graph_acc = nullptr;           // accumulator baked into the graphs
  jt_exec_stats* cur_stats = nullptr;
  void drop_graphs() {
    for (auto g : graphs)
      if (g) cudaGraphExecDestroy(g);
    graphs.clear();
    graph_stats.clear();
    graph_acc = nullptr;
  }
  ~jt_exec() {
    drop_graphs();
    for (auto& e : ev) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (pinned) cudaFreeHost(pinned);
  }
};

namespace jt {

void describe_exec(const jt_plan& plan, jt_dtype dt, const char* path) {
  Layout L = compile(plan, dt == JT_C64 ? 8 : 16);
  FILE* f = std::fopen(path, "w");
  if (!f) fail(JT_EUSAGE, std::string("cannot open ") + path);
  std::fprintf(f, "{\"total_bytes\": %lld, \"leaf_bytes\": %lld, \"inter_bytes\": %lld, \"scratch_bytes\": %lld, "
               "\"inter_base\": %lld, \"peak_live_bytes\": %lld, \"no_deletion_bytes\": %lld, \"cache_bytes\": %lld, \"nodes\": [",
               (long long)L.total, (long long)L.leaf_bytes, (long long)L.inter_bytes, (long long)L.scratch_bytes,
               (long long)L.inter_base, (long long)L.mem_peak_live, (long long)L.mem_no_deletion, (long long)L.mem_cache);
  for (size_t i = 0; i < L.order.size(); ++i) {
    const ExecNode& en = L.order[i];
    const GettArgs& g = en.args;
    std::fprintf(f, "%s{\"v\": %lld, \"maxpos\": %d, \"flop\": %.17g, \"bytes\": %.17g, \"n_out\": %lld, "
                 "\"tm\": %d, \"tn\": %d, \"tk\": %d, \"n_outer\": %d, \"n_ok\": %d, \"splits\": %d, "
                 "\"block\": %d, \"RM\": %d, \"RN\": %d, \"KG\": %d, \"smem\": %zu, \"vecA\": %d, \"vecB\": %d, \"dbuf\": %d, \"gauss\": %d, \"kind\": %d, \"tc_tm\": %d, \"tc_tk\": %d, \"tc_outer\": %d, \"out_off\": %lld, \"parent\": %lld, \"pos\": %zu",
                 i ? ", " : "", (long long)en.v, en.maxpos, en.flop, en.bytes, (long long)en.n_out, g.tm, g.tn, g.tk,
                 g.n_outer, g.n_ok, g.splits, en.block, en.RM, en.RN, g.KG, en.smem, g.vecA, g.vecB, g.dbuf, g.gauss, en.kind,
                 en.kind == 2 ? en.tcg.tmt : en.tc.tm, en.kind == 2 ? 4 + en.tcg.lg_kc : en.tc.K,
                 en.kind == 2 ? en.tcg.n_oN + en.tcg.n_oM : en.tc.n_outer, (long long)L.node_off[en.v],
                 (long long)plan.nodes[en.v].parent, i);
    if (en.kind == 1 || en.kind == 2) {  // big-operand strides of the tile rows and K bits
      std::fprintf(f, ", \"Bn\": [");
      for (size_t q = 0; q < en.tcB_n.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.tcB_n[q]);
      std::fprintf(f, "], \"Bk\": [");
      for (size_t q = 0; q < en.tcB_k.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.tcB_k[q]);
      std::fprintf(f, "], \"Am\": [");
      for (size_t q = 0; q < en.tcgA_m.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.tcgA_m[q]);
      std::fprintf(f, "], \"Ak\": [");
      for (size_t q = 0; q < en.tcgA_k.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.tcgA_k[q]);
      std::fprintf(f, "], \"ncopy\": %d, \"copy_bytes\": %d, \"rofs_row\": [%d, %d, %d, %d, %d, %d, %d]", en.kind == 1 ? en.tc.ncopy : en.tcg.ncopyB,
                   en.kind == 1 ? en.tc.copy_bytes : en.tcg.copyB_bytes, en.tc.rofs_row[0], en.tc.rofs_row[1],
                   en.tc.rofs_row[2], en.tc.rofs_row[3], en.tc.rofs_row[4], en.tc.rofs_row[5], en.tc.rofs_row[6]);
      std::fprintf(f, ", \"tkc\": %d, \"tma\": %d, \"permA\": %d, \"permB\": %d, \"rot\": %d", en.kind == 1 ? en.tc.tkc : 4,
                   en.kind == 1 ? en.tc.tma : en.tcg.tma, en.permA ? 1 : 0, en.permB ? 1 : 0, en.kind == 2 ? en.tcg.rot : 0);
    }
    if (en.kind == 4) {
      std::fprintf(f, ", \"st_vec\": %d, \"st_n_lo\": %d, \"st_cols\": %d, \"stN\": [", en.st.vec, en.st.n_lo, en.st.n_cols);
      for (size_t q = 0; q < en.stN.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.stN[q]);
      std::fprintf(f, "], \"stK\": [");
      for (size_t q = 0; q < en.stK.size(); ++q) std::fprintf(f, "%s%lld", q ? ", " : "", (long long)en.stK[q]);
      std::fprintf(f, "]");
    }
    std::fprintf(f, "}");
  }
  std::fprintf(f, "]}\n");
  std::fclose(f);
}

int64_t workspace_bytes(const jt_plan& plan, jt_dtype dt) {
  return compile(plan, dt == JT_C64 ? 8 : 16).total;
}

void exec_memory(const jt_plan& plan, jt_dtype dt, jt_memory* out) {
  const Layout L = compile(plan, dt == JT_C64 ? 8 : 16);
  jt_memory m{};
  m.total_bytes = L.total;
  m.leaf_bytes = L.leaf_bytes;
  m.arena_bytes = L.inter_bytes;
  m.peak_live_bytes = L.mem_peak_live;
  m.no_deletion_bytes = L.mem_no_deletion;
  m.cache_bytes = L.mem_cache;
  m.peak_live_noshare_bytes = L.mem_peak_live_noshare;
  m.scratch_bytes = L.scratch_bytes;
  *out = m;
}

void upload_leaves(jt_exec* ex) {
  // the pinned buffer is reused: wait for the previous upload to finish before refilling
  JT_CUDA(cudaStreamSynchronize(ex->stream));
  std::memcpy(ex->pinned, ex->host_leaves.data(), ex->host_leaves.size());
  JT_CUDA(cudaMemcpyAsync(ex->ws, ex->pinned, ex->host_leaves.size(), cudaMemcpyHostToDevice, ex->stream));
  ex->stats.h2d_bytes += (int64_t)ex->host_leaves.size();
}

jt_exec* exec_create(const jt_plan& plan, jt_dtype dt, int device, void* d_ws, int64_t ws_bytes, void* stream) {
  if (dt != JT_C64 && dt != JT_C128) fail(JT_EUSAGE, "exec: bad dtype");
  const int esize = dt == JT_C64 ? 8 : 16;
  Layout L = compile(plan, esize);
  if (!d_ws) fail(JT_EUSAGE, "exec: null workspace");
  if ((reinterpret_cast<uintptr_t>(d_ws) % kAlign) != 0) fail(JT_EUSAGE, "exec: workspace must be 256-B aligned");
  if (ws_bytes < L.total)
    fail(JT_ERESOURCE, "exec: workspace too small (" + std::to_string(ws_bytes) + " < " + std::to_string(L.total) + ")");
  JT_CUDA(cudaSetDevice(device));
  set_smem_attrs();
  int n_sm = 148;
  JT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
  for (ExecNode& en : L.order) {
    int nb = 1;
    if (en.kind == 2) {
      en.grid_x = std::min<int64_t>(en.tcg.n_tiles, n_sm);  // one CTA per SM (512 TMEM columns)
      continue;
    }
    if (en.kind == 4) {
      JT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &nb, reinterpret_cast<const void*>(pick_stream(en.args.tm, en.args.tk)), en.block, en.smem));
      if (nb < 1) fail(JT_EINTERNAL, "exec: a K2s block does not fit on an SM");
      en.grid_x = std::max<int64_t>(1, std::min<int64_t>(en.args.n_tiles / 512, (int64_t)nb * n_sm));
      continue;
    }
    if (en.kind == 1) {
      JT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &nb, reinterpret_cast<const void*>(pick_tc(en.tc.tkc, en.tc.tma != 0)), en.block, en.smem));
      const int nb_occ = nb;
      // The occupancy calculator reports 1 CTA per SM for the tcgen05 kernels whatever their
      // shared memory and block size (it assumes the whole TMEM per CTA); K3's shared-memory
      // footprint is sized so that exactly 512 / tmem_cols CTAs fit (plan_tc), so that count is
      // used (JETB200_K3_OCC=api keeps the calculator's answer).
      {
        const char* e = std::getenv("JETB200_K3_OCC");
        if (!(e && std::string(e) == "api")) nb = 512 / (int)en.tc.tmem_cols;
      }
      nb = std::min<int>(nb, 512 / (int)en.tc.tmem_cols);  // TMEM columns per SM
      if (nb < 1) fail(JT_EINTERNAL, "exec: a K3 tile does not fit on an SM");
      en.grid_x = std::min<int64_t>(en.tc.n_tiles, (int64_t)nb * n_sm);
      if (std::getenv("JETB200_DEBUG_GRID")) {
        cudaFuncAttributes fa{};
        const void* f = reinterpret_cast<const void*>(pick_tc(en.tc.tkc, en.tc.tma != 0));
        JT_CUDA(cudaFuncGetAttributes(&fa, f));
        int o0 = 0, o1 = 0;
        JT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o0, f, en.block, 0));
        JT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, f, 128, 0));
        std::fprintf(stderr, "K3 node %lld: smem %zu block %d occupancy %d tmem_cols %u -> %d CTAs/SM, grid %lld | "
                     "regs %d static smem %zu max dyn %d maxthr %d | occ(smem 0) %d occ(128 thr) %d\n",
                     (long long)en.v, en.smem, en.block, nb_occ, en.tc.tmem_cols, nb, (long long)en.grid_x, fa.numRegs,
                     fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.maxThreadsPerBlock, o0, o1);
      }
      continue;
    }
    const void* fn = en.kind == 3   ? reinterpret_cast<const void*>(pick_dmma(en.RM, en.RN, en.args.gauss != 0))
                     : dt == JT_C64 ? reinterpret_cast<const void*>(pick_gett<float>(en.RM, en.RN))
                                    : reinterpret_cast<const void*>(pick_gett<double>(en.RM, en.RN));
    JT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, en.block, en.smem));
    if (nb < 1) fail(JT_EINTERNAL, "exec: a contraction tile does not fit on an SM");
    const int64_t resident = (int64_t)nb * n_sm;
    en.grid_x = std::min<int64_t>(en.args.n_tiles, std::max<int64_t>(1, resident / en.args.splits));
  }
  // K3 TMA maps: B's item box at its workspace address (dim 0 declared 2^32 long: the item
  // base offset is the dim-0 coordinate; see plan_tc)
  auto* ex = new jt_exec();
  ex->L = std::move(L);
  ex->cur_stats = &ex->stats;
  {
    const char* e = std::getenv("JETB200_GRAPHS");
    ex->use_graphs = !(e && e[0] == '0') && stream != nullptr;  // no capture on the legacy stream
    // programmatic dependent launch: opt-in (JETB200_PDL=1).  Measured on the C3 amplitude with
    // the TMA-fed K3: 10.22 s with PDL vs 9.28 s without (gather K3: 10.08 vs 9.72 s), i.e. the
    // early-launched dependents cost more than the prologue overlap saves
    // (profiles/r02_variants_pdl.txt)
    const char* q = std::getenv("JETB200_PDL");
    ex->pdl = q && q[0] == '1';
    ex->pdl_small = q && std::string(q) == "small";  // JETB200_PDL=small: only K2 / K2s / K6 launches
  }
  const int32_t* dptr = reinterpret_cast<const int32_t*>(static_cast<char*>(d_ws) + ex->L.state_base +
                                                         offsetof(SliceState, digits));
  for (ExecNode& en : ex->L.order) {
    SliceView sv{};
    sv.digits = dptr;
    sv.nA = (int)en.sliceA.size();
    sv.nB = (int)en.sliceB.size();
    for (int i = 0; i < sv.nA; ++i) { sv.posA[i] = en.sliceA[i].first; sv.strA[i] = en.sliceA[i].second; }
    for (int i = 0; i < sv.nB; ++i) { sv.posB[i] = en.sliceB[i].first; sv.strB[i] = en.sliceB[i].second; }
    en.args.sv = sv;
    en.st.sv = sv;
    en.tc.sv = sv;
    en.tcg.sv = sv;
    en.gA.sv = sv;
    en.gB.sv = sv;
    if (en.permA) en.tcg.sv.nA = 0;  // the K1 copy already holds the slice
    if (en.permB) en.tcg.sv.nB = 0;
  }
  ex->dtype = dt;
  ex->device = device;
  ex->ws = static_cast<char*>(d_ws);
  ex->ws_bytes = ws_bytes;
  ex->stream = static_cast<cudaStream_t>(stream);
  ex->n_sl = plan.n_sl;
  ex->k = (int)plan.sliced.size();
  ex->d = plan.net.d;
  ex->n_summed = plan.n_summed;
  ex->n_batch = plan.n_batch;
  // leaves converted to the exec dtype, uploaded through a pinned staging buffer
  ex->host_leaves.assign(ex->L.leaf_bytes, 0);
  const int64_t nt = (int64_t)plan.net.tensors.size();
  for (int64_t t = 0; t < nt; ++t) {
    const auto& data = plan.net.tensors[t].data;
    char* dst = ex->host_leaves.data() + ex->L.leaf_off[t];
    for (size_t i = 0; i < data.size(); ++i) {
      if (esize == 8) {
        float2 f = make_float2((float)data[i].real(), (float)data[i].imag());
        std::memcpy(dst + i * 8, &f, 8);
      } else {
        double2 f = make_double2(data[i].real(), data[i].imag());
        std::memcpy(dst + i * 16, &f, 16);
      }
    }
  }
  try {
    JT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ex->pinned), std::max<int64_t>(ex->L.leaf_bytes, 16),
                          cudaHostAllocDefault));
    upload_leaves(ex);
    JT_CUDA(cudaStreamSynchronize(ex->stream));
  } catch (...) {
    delete ex;
    throw;
  }
  return ex;
}

// Launch with programmatic stream serialisation (PDL): the kernel may start while its
// predecessor drains and synchronises through griddepcontrol.wait.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  JT_CUDA(cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...));
}

void ev_begin(jt_exec* ex) {
  if (!ex->profiling) return;
  if (ex->ev_used == ex->ev.size()) {
    cudaEvent_t a, b;
    JT_CUDA(cudaEventCreate(&a));
    JT_CUDA(cudaEventCreate(&b));
    ex->ev.push_back({a, b});
  }
  JT_CUDA(cudaEventRecord(ex->ev[ex->ev_used].first, ex->stream));
}
void ev_end(jt_exec* ex, const ExecNode& en) {
  if (!ex->profiling) return;
  JT_CUDA(cudaEventRecord(ex->ev[ex->ev_used].second, ex->stream));
  ex->ev_work.push_back({en.bytes, en.flop});
  ex->ev_kind.push_back(en.kind);
  ex->ev_used++;
}

template <typename R>
void launch_node(jt_exec* ex, ExecNode& en) {
  using C2 = typename V2<R>::t;
  const Layout& L = ex->L;
  jt_exec_stats& st = *ex->cur_stats;
  if (en.kind == 2) {
    TcgArgs& t = en.tcg;
    t.A = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opA]);
    t.B = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opB]);
    t.C = reinterpret_cast<float2*>(ex->ws + en.out_off);
    ev_begin(ex);  // the node's time includes its K1 copies
    if (en.permB) {
      en.gB.src = t.B;
      en.gB.dst = reinterpret_cast<float2*>(ex->ws + en.perm_off);
      launch_pdl(view_gather_kernel, dim3(148 * 8), dim3(256), 0, ex->stream, ex->pdl, en.gB);
      st.kernel_launches++;
      t.B = en.gB.dst;
    }
    if (en.permA) {
      en.gA.src = t.A;
      en.gA.dst = reinterpret_cast<float2*>(ex->ws + en.perm_off + en.permA_at);
      launch_pdl(view_gather_kernel, dim3(148 * 8), dim3(256), 0, ex->stream, ex->pdl, en.gA);
      st.kernel_launches++;
      t.A = en.gA.dst;
    }
    launch_pdl(pick_tcg(t.tmt, t.tma != 0), dim3((unsigned)en.grid_x), dim3(en.block), en.smem, ex->stream, ex->pdl, t);
    ev_end(ex, en);
    st.kernel_launches++;
  } else if (en.kind == 4) {
    StreamArgs& t = en.st;
    t.A = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opA]);
    t.B = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opB]);
    t.C = reinterpret_cast<float2*>(ex->ws + en.out_off);
    ev_begin(ex);
    launch_pdl(pick_stream(en.args.tm, en.args.tk), dim3((unsigned)en.grid_x), dim3(en.block), en.smem, ex->stream,
               ex->pdl || ex->pdl_small, t);
    ev_end(ex, en);
    st.kernel_launches++;
  } else if (en.kind == 1) {
    TcArgs& t = en.tc;
    t.A = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opA]);
    t.B = reinterpret_cast<const float2*>(ex->ws + L.node_off[en.opB]);
    t.C = reinterpret_cast<float2*>(ex->ws + en.out_off);
    ev_begin(ex);
    launch_pdl(pick_tc(t.tkc, t.tma != 0), dim3((unsigned)en.grid_x), dim3(en.block), en.smem, ex->stream, ex->pdl, t);
    ev_end(ex, en);
    st.kernel_launches++;
  } else {
    GettArgs& g = en.args;
    g.A = ex->ws + L.node_off[en.opA];
    g.B = ex->ws + L.node_off[en.opB];
    g.C = ex->ws + en.out_off;
    g.P = ex->ws + en.part_off;
    dim3 grid((unsigned)en.grid_x, (unsigned)g.splits);
    GettFn fn = en.kind == 3 ? pick_dmma(en.RM, en.RN, g.gauss != 0) : pick_gett<R>(en.RM, en.RN);
    ev_begin(ex);
    launch_pdl(fn, grid, dim3(en.block), en.smem, ex->stream, ex->pdl || ex->pdl_small, g);
    ev_end(ex, en);
    st.kernel_launches++;
    if (g.splits > 1) {
      int64_t n = en.n_out;
      int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
      launch_pdl(reduce_splits_kernel<R>, dim3(blocks), dim3(256), 0, ex->stream, ex->pdl || ex->pdl_small,
                 reinterpret_cast<const C2*>(g.P), reinterpret_cast<C2*>(g.C), n, (int)g.splits);
      st.kernel_launches++;
    }
  }
  st.node_launches++;
  st.flop_executed += en.flop;
  st.bytes_executed += en.bytes;
}

// One slice at prefix-cache level j: advance the device slice state, every node with
// maxpos(S(v)) >= j, then the accumulate.
template <typename R>
void slice_sequence(jt_exec* ex, int j, double* d_acc) {
  using C2 = typename V2<R>::t;
  SliceState* state = reinterpret_cast<SliceState*>(ex->ws + ex->L.state_base);
  launch_pdl(advance_slice_kernel, dim3(1), dim3(32), 0, ex->stream, ex->pdl || ex->pdl_small, state, ex->k, ex->d);
  ex->cur_stats->kernel_launches++;
  for (ExecNode& en : ex->L.order)
    if (en.maxpos >= j) launch_node<R>(ex, en);
  const ExecNode& root = ex->L.order.back();
  launch_pdl(accumulate_kernel<R>, dim3(1), dim3(32), 0, ex->stream, ex->pdl || ex->pdl_small,
             reinterpret_cast<const C2*>(ex->ws + root.out_off), d_acc,
             reinterpret_cast<double2*>(ex->ws + ex->L.vals_base), (const SliceState*)state, ex->n_summed,
             ex->k - ex->n_summed, ex->d);
  ex->cur_stats->kernel_launches++;
  ex->cur_stats->slices_done++;
}

template <typename R>
void contract_range(jt_exec* ex, int64_t b, int64_t e, double* d_acc, bool reuse) {
  std::vector<int> dig(ex->k), prev(ex->k);
  auto digits = [&](int64_t s, std::vector<int>& out) {
    for (int p = ex->k - 1; p >= 0; --p) { out[p] = (int)(s % ex->d); s /= ex->d; }
  };
  if (ex->last >= 0) digits(ex->last, prev);
  const bool graphs = ex->use_graphs && !ex->profiling;
  if (graphs && ex->graph_acc != d_acc) {
    ex->drop_graphs();
    ex->graphs.assign(ex->k + 2, nullptr);
    ex->graph_stats.assign(ex->k + 2, jt_exec_stats{});
    ex->graph_acc = d_acc;
  }
  if (e > b) {
    set_slice_kernel<<<1, 32, 0, ex->stream>>>(reinterpret_cast<SliceState*>(ex->ws + ex->L.state_base), b - 1, b,
                                               ex->L.vals_cap - 1);
    ex->stats.kernel_launches++;
  }
  for (int64_t s = b; s < e; ++s) {
    digits(s, dig);
    int j;
    if (!reuse || ex->last < 0) {
      j = -1;
    } else {
      j = ex->k;  // nothing changed
      for (int p = 0; p < ex->k; ++p)
        if (dig[p] != prev[p]) { j = p; break; }
    }
    if (!graphs) {
      ex->cur_stats = &ex->stats;
      slice_sequence<R>(ex, j, d_acc);
    } else {
      cudaGraphExec_t& ge = ex->graphs[j + 1];
      if (!ge) {  // capture this level once
        cudaGraph_t g;
        ex->cur_stats = &ex->graph_stats[j + 1];
        JT_CUDA(cudaStreamBeginCapture(ex->stream, cudaStreamCaptureModeThreadLocal));
        slice_sequence<R>(ex, j, d_acc);
        JT_CUDA(cudaStreamEndCapture(ex->stream, &g));
        JT_CUDA(cudaGraphInstantiate(&ge, g, 0));
        JT_CUDA(cudaGraphDestroy(g));
      }
      JT_CUDA(cudaGraphLaunch(ge, ex->stream));
      const jt_exec_stats& gs = ex->graph_stats[j + 1];
      ex->stats.kernel_launches += gs.kernel_launches;
      ex->stats.node_launches += gs.node_launches;
      ex->stats.flop_executed += gs.flop_executed;
      ex->stats.bytes_executed += gs.bytes_executed;
      ex->stats.slices_done += gs.slices_done;
    }
    ex->last = s;
    prev = dig;
  }
  ex->cur_stats = &ex->stats;
  JT_CUDA(cudaGetLastError());
}

void exec_contract(jt_exec* ex, int64_t b, int64_t e, double* d_acc, double* h_vals, bool reuse) {
  if (b < 0 || e > ex->n_sl || b > e) fail(JT_EUSAGE, "exec: slice range out of bounds");
  if (!d_acc) fail(JT_EUSAGE, "exec: null accumulator");
  if (h_vals && e - b > ex->L.vals_cap)
    fail(JT_EUSAGE, "exec: at most " + std::to_string(ex->L.vals_cap) + " slice values per call");
  JT_CUDA(cudaSetDevice(ex->device));
  ex->ev_used = 0;
  ex->ev_work.clear();
  ex->ev_kind.clear();
  if (ex->dtype == JT_C64) contract_range<float>(ex, b, e, d_acc, reuse);
  else contract_range<double>(ex, b, e, d_acc, reuse);
  if (ex->profiling && ex->ev_used) {
    JT_CUDA(cudaStreamSynchronize(ex->stream));
    for (size_t i = 0; i < ex->ev_used; ++i) {
      float ms = 0;
      JT_CUDA(cudaEventElapsedTime(&ms, ex->ev[i].first, ex->ev[i].second));
      ex->stats.k2_time_ms += ms;
      ex->stats.k2_timed_launches++;
      ex->stats.k2_timed_bytes += ex->ev_work[i].first;
      ex->stats.k2_timed_flop += ex->ev_work[i].second;
      if (ex->ev_kind[i] == 3) {
        ex->stats.k4_time_ms += ms;
        ex->stats.k4_timed_launches++;
        ex->stats.k4_timed_bytes += ex->ev_work[i].first;
        ex->stats.k4_timed_flop += ex->ev_work[i].second;
      } else if (ex->ev_kind[i] == 4) {
        ex->stats.k2s_time_ms += ms;
        ex->stats.k2s_timed_launches++;
        ex->stats.k2s_timed_bytes += ex->ev_work[i].first;
        ex->stats.k2s_timed_flop += ex->ev_work[i].second;
      } else if (ex->ev_kind[i] >= 1) {
        if (ex->ev_kind[i] == 2) {
          ex->stats.k3g_time_ms += ms;
          ex->stats.k3g_timed_launches++;
          ex->stats.k3g_timed_bytes += ex->ev_work[i].first;
          ex->stats.k3g_timed_flop += ex->ev_work[i].second;
        }
        ex->stats.k3_time_ms += ms;
        ex->stats.k3_timed_launches++;
        ex->stats.k3_timed_bytes += ex->ev_work[i].first;
        ex->stats.k3_timed_flop += ex->ev_work[i].second;
      }
    }
  }
  if (h_vals && e > b) {
    JT_CUDA(cudaMemcpyAsync(h_vals, ex->ws + ex->L.vals_base, (e - b) * 16, cudaMemcpyDeviceToHost, ex->stream));
    JT_CUDA(cudaStreamSynchronize(ex->stream));
  }
}

void exec_contract_host(jt_exec* ex, int64_t b, int64_t e, double* h_acc) {
  double* d_acc = reinterpret_cast<double*>(ex->ws + ex->L.acc_base);
  JT_CUDA(cudaSetDevice(ex->device));
  JT_CUDA(cudaMemsetAsync(d_acc, 0, 16 * ex->n_batch, ex->stream));
  exec_contract(ex, b, e, d_acc, nullptr, true);
  JT_CUDA(cudaMemcpyAsync(h_acc, d_acc, 16 * ex->n_batch, cudaMemcpyDeviceToHost, ex->stream));
  JT_CUDA(cudaStreamSynchronize(ex->stream));
}

// DEBUG: time `reps` back-to-back launches of execution-order node `idx` (CUDA events on the
// exec stream); the node reads whatever its inputs currently hold.
void debug_time_node(jt_exec* ex, int64_t idx, int reps, double* ms_out, double* bytes, double* flop, int* kind) {
  if (idx < 0 || idx >= (int64_t)ex->L.order.size() || reps < 1) fail(JT_EUSAGE, "debug_time_node: bad index");
  ExecNode& en = ex->L.order[idx];
  ex->cur_stats = &ex->stats;
  const bool prof = ex->profiling;
  ex->profiling = false;
  cudaEvent_t a, b;
  JT_CUDA(cudaEventCreate(&a));
  JT_CUDA(cudaEventCreate(&b));
  auto one = [&]() {
    if (ex->dtype == JT_C64) launch_node<float>(ex, en);
    else launch_node<double>(ex, en);
  };
  one();
  JT_CUDA(cudaEventRecord(a, ex->stream));
  for (int r = 0; r < reps; ++r) one();
  JT_CUDA(cudaEventRecord(b, ex->stream));
  JT_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  JT_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  ex->profiling = prof;
  *ms_out = ms / reps;
  *bytes = en.bytes;
  *flop = en.flop;
  *kind = en.kind;
}

void exec_invalidate(jt_exec* ex) { ex->last = -1; }
void exec_set_graphs(jt_exec* ex, bool on) { ex->use_graphs = on; }
void exec_set_profiling(jt_exec* ex, bool on) { ex->profiling = on; }
void exec_stats(const jt_exec* ex, jt_exec_stats* out) { *out = ex->stats; }
void exec_stats_reset(jt_exec* ex) { ex->stats = jt_exec_stats{}; }
void exec_destroy(jt_exec* ex) { delete ex; }

void amplitude(const jt_plan& plan, jt_dtype dt, int device, double* out) {
  JT_CUDA(cudaSetDevice(device));
  int64_t bytes = workspace_bytes(plan, dt);
  void* ws = nullptr;
  JT_CUDA(cudaMalloc(&ws, bytes));
  jt_exec* ex = nullptr;
  try {
    ex = exec_create(plan, dt, device, ws, bytes, nullptr);
    exec_contract_host(ex, 0, plan.n_sl, out);
  } catch (...) {
    delete ex;
    cudaFree(ws);
    throw;
  }
  delete ex;
  JT_CUDA(cudaFree(ws));
}

// K1: dst[pi(i)] = src[i]; bit b of the source address moves to bit perm[b].
void permute(jt_dtype dt, const void* src, void* dst, int n, const int32_t* perm, void* stream) {
  if (n < 0 || n > 40) fail(JT_EUSAGE, "permute: n_bits out of range");
  std::vector<int> inv(n, -1);
  for (int b = 0; b < n; ++b) {
    if (perm[b] < 0 || perm[b] >= n || inv[perm[b]] >= 0) fail(JT_EUSAGE, "permute: not a permutation");
    inv[perm[b]] = b;
  }
  const int esize = dt == JT_C64 ? 8 : 16;
  set_smem_attrs();
  PermArgs p;
  std::memset(&p, 0, sizeof(p));
  p.src = src;
  p.dst = dst;
  // tile: the lowest input bits and the lowest output bits (as input bits)
  // tile = the lowest `half` input bits + the lowest `half` output bits, filled with further
  // low input bits to 2^12 (c64) / 2^11 (c128) elements: 32 KB per CTA keeps enough bytes in
  // flight per SM
  const int half = esize == 8 ? 5 : 4;
  const int tile_bits = esize == 8 ? 12 : 11;
  std::vector<char> in_tile(n, 0);
  for (int b = 0; b < std::min(n, half); ++b) in_tile[b] = 1;          // low input bits
  for (int o = 0; o < std::min(n, half); ++o) in_tile[inv[o]] = 1;     // low output bits
  for (int b = 0; b < n && std::count(in_tile.begin(), in_tile.end(), 1) < std::min(n, tile_bits); ++b)
    in_tile[b] = 1;
  std::vector<int> tbits, obits;
  for (int b = 0; b < n; ++b) (in_tile[b] ? tbits : obits).push_back(b);
  p.nt = (int)tbits.size();
  if (p.nt > 12) fail(JT_EINTERNAL, "permute: tile too large");
  for (int i = 0; i < p.nt; ++i) p.in_g[i] = int64_t(1) << tbits[i];
  std::vector<std::pair<int, int>> byout;  // (output position, tile index)
  for (int i = 0; i < p.nt; ++i) byout.push_back({perm[tbits[i]], i});
  std::sort(byout.begin(), byout.end());
  for (int i = 0; i < p.nt; ++i) {
    p.out_g[i] = int64_t(1) << byout[i].first;
    p.out_s[i] = 1 << byout[i].second;
  }
  p.n_outer = (int)obits.size();
  for (int j = 0; j < p.n_outer; ++j) {
    p.o_src[j] = int64_t(1) << obits[j];
    p.o_dst[j] = int64_t(1) << perm[obits[j]];
  }
  const int64_t nblk = int64_t(1) << p.n_outer;
  if (nblk > (int64_t(1) << 31) - 1) fail(JT_EUSAGE, "permute: tensor too large");
  const size_t smem = (size_t)(int64_t(1) << p.nt) * esize;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // element pairs stay together when bit 0 maps to bit 0 (and the tile holds >= 2 elements)
  const bool pair = esize == 8 && n >= 1 && perm[0] == 0 && p.nt >= 1 && p.in_g[0] == 1 && p.out_g[0] == 1;
  // otherwise (c64, bit 0 moves) input pairs and output pairs still move as 16 B (input bit 0
  // and output bit 0 are both tile bits)
  const bool split = esize == 8 && !pair && p.nt >= 2 && p.in_g[0] == 1 && p.out_g[0] == 1;
  if (esize == 8 && pair) permute_kernel<float2, 1><<<(unsigned)nblk, 256, smem, s>>>(p);
  else if (split) permute_kernel<float2, 2><<<(unsigned)nblk, 256, smem, s>>>(p);
  else if (esize == 8) permute_kernel<float2, 0><<<(unsigned)nblk, 256, smem, s>>>(p);
  else permute_kernel<double2, 0><<<(unsigned)nblk, 256, smem, s>>>(p);
  JT_CUDA(cudaGetLastError());
}

}  // namespace jt
