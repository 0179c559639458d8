// Device kernels of the hot path (sm_100a).
//
//   K2  gett_kernel     pairwise contraction C = sum_K A*B (Eq. sequence)
//                       of two bit-addressed tensors, tiled over *address bits*: every
//                       dimension is a power of two, so a tensor of 2^n elements is n
//                       address bits and a contraction is a GEMM whose M/N/K "indices"
//                       are arbitrary bit subsets.  A CTA stages an A tile (tile-M x
//                       tile-K bits) and a B tile (tile-K x tile-N bits) in shared memory
//                       through gather tables that enumerate each operand's lowest
//                       address bits fastest (coalesced 128-B runs), so the two transposes
//                       of the paper's transpose-transpose-GEMM (l.180) are fused into the
//                       loads.  The output tile is written as one contiguous block (the
//                       planner lays C out as [tile bits][outer bits]).  Complex FP32 (c64)
//                       or FP64 (c128) FMA on CUDA cores, in-CTA split-K over k-groups and
//                       optional cross-CTA split-K into a scratch buffer + K2r reduction.
//   K2r reduce_splits   deterministic sum of split-K partials (fixed order).
//   K6  accumulate      acc(c128) += s_sigma, store s_sigma ("sum_i s_i").
//   K1  permute_kernel  bit permutation of a 2^n tensor through a shared-memory tile that
//                       holds the low input bits and the low output bits (l.180, l.285).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace jt {

// Programmatic dependent launch: every kernel of the slice sequence is launched with
// programmatic stream serialisation, runs its parameter-only prologue, then waits for the
// previous kernel's memory (griddepcontrol.wait) before touching the workspace, and lets the
// next kernel start its own prologue (griddepcontrol.launch_dependents).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr int kMaxOuter = 48;
constexpr int kMaxTile = 14;

// K5 slice views, resolved on the device: a leaf operand carrying sliced labels is read at
// base + sum_i digit[pos_i] * stride_i, with the digits of the current slice in device
// memory (written by advance_slice_kernel), so a captured CUDA graph serves every slice.
struct SliceView {
  const int32_t* digits;
  int32_t nA, nB;
  int32_t posA[4], posB[4];
  int64_t strA[4], strB[4];
};

__device__ __forceinline__ int64_t slice_off(const SliceView& v, bool a) {
  int64_t o = 0;
  const int n = a ? v.nA : v.nB;
  for (int i = 0; i < n; ++i) o += (int64_t)v.digits[a ? v.posA[i] : v.posB[i]] * (a ? v.strA[i] : v.strB[i]);
  return o;
}

template <typename R> struct V2;
template <> struct V2<float> { using t = float2; };
template <> struct V2<double> { using t = double2; };

struct GettArgs {
  const void* A;
  const void* B;
  void* C;   // output (splits == 1)
  void* P;   // split-K partials (splits > 1), [split][tile][local]
  int64_t n_tiles;
  int64_t k_iters;
  int32_t n_outer, n_ok, splits;
  int32_t tm, tn, tk, nA, nB;
  int32_t TX, TY, KG;
  int32_t vecA, vecB;  // 1: tile bit 0 has global stride 1 -> 16-B copies of element pairs (c64)
  int32_t dbuf;        // unused (kept for the descriptor dump); the kernel always double-buffers
  int32_t gauss;       // K4: 1 = 3M (Gauss) complex product, 3 DMMAs per complex MAC (else 4M)
  int64_t o_sA[kMaxOuter], o_sB[kMaxOuter];    // outer M/N bit j: strides in A and B
  int64_t ok_sA[kMaxOuter], ok_sB[kMaxOuter];  // outer K bit j
  int64_t gA[kMaxTile], gB[kMaxTile];          // tile bit j of A (B), sorted by stride: global stride;
                                               // its shared-memory stride is 2^j (operand order)
  int8_t pM[kMaxTile], pKA[kMaxTile];          // tile-M bit i / tile-K bit i -> bit position in A's tile
  int8_t pKB[kMaxTile], pN[kMaxTile];          // tile-K bit i / tile-N bit i -> bit position in B's tile
  SliceView sv;
};

template <typename C2>
__device__ __forceinline__ void cmac(C2& acc, const C2 a, const C2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// cp.async.wait_group with a run-time count (0..11), for rings sized at launch
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::); break;
    case 4: asm volatile("cp.async.wait_group 4;\n" ::); break;
    case 5: asm volatile("cp.async.wait_group 5;\n" ::); break;
    case 6: asm volatile("cp.async.wait_group 6;\n" ::); break;
    case 7: asm volatile("cp.async.wait_group 7;\n" ::); break;
    case 8: asm volatile("cp.async.wait_group 8;\n" ::); break;
    case 9: asm volatile("cp.async.wait_group 9;\n" ::); break;
    case 10: asm volatile("cp.async.wait_group 10;\n" ::); break;
    default: asm volatile("cp.async.wait_group 11;\n" ::); break;
  }
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// deposit the bits of v at the given bit positions: sum_i bit_i(v) << pos[i]
__device__ __forceinline__ int deposit(int v, const int8_t* pos, int n) {
  int r = 0;
  for (int i = 0; i < n; ++i) r |= ((v >> i) & 1) << pos[i];
  return r;
}

// Shared-memory XOR swizzle of an operand tile index: folds bits 4-12 (c64) / 3-11 (c128)
// onto the 16-B slot bits of a 128-B row so that warp reads along any tile bit spread over
// the banks.  Linear over GF(2): swz(a | b) = swz(a) ^ swz(b) for disjoint a, b, so a row
// offset and a column offset can be swizzled separately and combined with XOR.  Bit 0 is
// untouched for c64, keeping 16-B element pairs contiguous.
template <typename C2>
__device__ __forceinline__ int swz(int i) {
  if (sizeof(C2) == 8) return i ^ ((((i >> 4) ^ (i >> 7) ^ (i >> 10)) & 7) << 1);
  return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9)) & 7);
}

// Copy one operand tile (2^n elements, tile bit j at global stride g[j], shared stride 2^j)
// into shared memory with cp.async; element pairs move as 16 B when g[0] == 1.
template <typename C2>
__device__ __forceinline__ void load_tile(C2* dst, const C2* src, int n, bool vec, const int64_t (*tg)[64],
                                          int tid, int nthr) {
  const int sz = 1 << n;
  if (sizeof(C2) == 16) {
    for (int e = tid; e < sz; e += nthr) cp_async16(dst + swz<C2>(e), src + tg[0][e & 63] + tg[1][e >> 6]);
  } else if (vec) {
    if ((nthr & 31) == 0) {  // 2*nthr is a multiple of 64: e & 63 is fixed per thread (swz is GF(2)-linear)
      const int lo = (2 * tid) & 63;
      const C2* s0 = src + tg[0][lo];
      const int d0 = swz<C2>(lo);
      for (int e = 2 * tid; e < sz; e += 2 * nthr) cp_async16(dst + (d0 ^ swz<C2>(e & ~63)), s0 + tg[1][e >> 6]);
    } else {
      for (int e = 2 * tid; e < sz; e += 2 * nthr) cp_async16(dst + swz<C2>(e), src + tg[0][e & 63] + tg[1][e >> 6]);
    }
  } else {
    for (int e = tid; e < sz; e += nthr) cp_async8(dst + swz<C2>(e), src + tg[0][e & 63] + tg[1][e >> 6]);
  }
}

// Persistent over output tiles: CTA x walks tiles x, x + gridDim.x, ...; within a tile it walks
// its split's K steps.  The (tile, K step) items form one flat sequence with a two-stage
// cp.async pipeline, so the next item's operand tiles stream in while this one computes.
template <typename R, int RM, int RN>
__global__ void __launch_bounds__(256) gett_kernel(const __grid_constant__ GettArgs p) {
  using C2 = typename V2<R>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t tgA[2][64], tgB[2][64];
  __shared__ int64_t dkA[kMaxOuter], dkB[kMaxOuter];  // K-loop step deltas by trailing-zero count
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  for (int t = tid; t < p.n_ok; t += nthr) {
    // it-1 -> it flips bits 0..t-1 (1 -> 0) and bit t (0 -> 1), t = ctz(it)
    int64_t da = p.ok_sA[t], db = p.ok_sB[t];
    for (int i = 0; i < t; ++i) { da -= p.ok_sA[i]; db -= p.ok_sB[i]; }
    dkA[t] = da;
    dkB[t] = db;
  }
  for (int i = tid; i < 64; i += nthr) {
    // global-offset tables: lo = tile bits 0..5, hi = tile bits 6..11 (stride order)
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0, gb = 0;
      for (int b = 0; b < 6; ++b) {
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nA) g += p.gA[bi];
          if (bi < p.nB) gb += p.gB[bi];
        }
      }
      tgA[h][i] = g;
      tgB[h][i] = gb;
    }
  }
  const int szA = 1 << p.nA, szB = 1 << p.nB, TK = 1 << p.tk;
  const int CT = 1 << (p.tm + p.tn);
  C2* sA0 = reinterpret_cast<C2*>(smem_raw);
  const int stage = szA + szB;  // elements per pipeline stage
  C2* red = sA0 + 2 * stage;    // k-group partials (KG > 1)
  int* posKA = reinterpret_cast<int*>(red + (p.KG > 1 ? (p.KG - 1) * CT : 0));
  int* posKB = posKA + TK;
  for (int kk = tid; kk < TK; kk += nthr) {
    posKA[kk] = swz<C2>(deposit(kk, p.pKA, p.tk));
    posKB[kk] = swz<C2>(deposit(kk, p.pKB, p.tk));
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const int split = blockIdx.y;
  const int64_t it0 = (int64_t)split * p.k_iters / p.splits;
  const int64_t it1 = (int64_t)(split + 1) * p.k_iters / p.splits;
  const int64_t nk = it1 - it0;
  const int64_t my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nk;
  const int TXY = p.TX * p.TY;
  const int kg = tid / TXY;
  const int txy = tid - kg * TXY;
  const int tx = txy % p.TX, ty = txy / p.TX;
  const bool active = kg < p.KG;
  // this thread's rows m = ty + r*TY and columns n = pairs (2tx, 2tx+1) + (c/2)*2TX (RN >= 2)
  auto col = [&](int c) { return RN >= 2 ? (2 * tx + (c & 1) + (c >> 1) * 2 * p.TX) : tx; };
  int offM[RM], offN[RN];
#pragma unroll
  for (int r = 0; r < RM; ++r) offM[r] = swz<C2>(deposit(ty + r * p.TY, p.pM, p.tm));
#pragma unroll
  for (int c = 0; c < RN; ++c) offN[c] = swz<C2>(deposit(col(c), p.pN, p.tn));
  const C2* __restrict__ A = reinterpret_cast<const C2*>(p.A) + slice_off(p.sv, true);
  const C2* __restrict__ B = reinterpret_cast<const C2*>(p.B) + slice_off(p.sv, false);
  // operand offsets of the next item to load: recomputed from the bits at a tile start, stepped
  // by one delta per K iteration otherwise (no per-item bit loops)
  int64_t ld_tile = blockIdx.x, ld_k = 0, ld_oa = 0, ld_ob = 0;
  auto tile_start = [&]() {
    const int64_t it = it0;
    ld_oa = 0;
    ld_ob = 0;
    for (int j = 0; j < p.n_outer; ++j)
      if ((ld_tile >> j) & 1) { ld_oa += p.o_sA[j]; ld_ob += p.o_sB[j]; }
    for (int j = 0; j < p.n_ok; ++j)
      if ((it >> j) & 1) { ld_oa += p.ok_sA[j]; ld_ob += p.ok_sB[j]; }
  };
  auto advance = [&]() {
    if (++ld_k == nk) {
      ld_k = 0;
      ld_tile += gridDim.x;
      tile_start();
    } else {
      const int t = __ffsll((unsigned long long)(it0 + ld_k)) - 1;
      ld_oa += dkA[t];
      ld_ob += dkB[t];
    }
  };
  C2 acc[RM][RN];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) { acc[r][c].x = 0; acc[r][c].y = 0; }
  if (total > 0) {
    tile_start();
    load_tile(sA0, A + ld_oa, p.nA, p.vecA, tgA, tid, nthr);
    load_tile(sA0 + szA, B + ld_ob, p.nB, p.vecB, tgB, tid, nthr);
    cp_async_commit();
  }
  for (int64_t w = 0; w < total; ++w) {
    const int buf = (int)(w & 1);
    if (w + 1 < total) {  // prefetch the next item into the other stage
      advance();
      C2* nxt = sA0 + (buf ^ 1) * stage;
      load_tile(nxt, A + ld_oa, p.nA, p.vecA, tgA, tid, nthr);
      load_tile(nxt + szA, B + ld_ob, p.nB, p.vecB, tgB, tid, nthr);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const C2* sA = sA0 + buf * stage;
    const C2* sB = sA + szA;
    if (active) {
      for (int kk = kg; kk < TK; kk += p.KG) {
        const int ka = posKA[kk], kb = posKB[kk];
        C2 a[RM], b[RN];
#pragma unroll
        for (int r = 0; r < RM; ++r) a[r] = sA[ka ^ offM[r]];
#pragma unroll
        for (int c = 0; c < RN; ++c) b[c] = sB[kb ^ offN[c]];
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
          for (int c = 0; c < RN; ++c) cmac(acc[r][c], a[r], b[c]);
      }
    }
    if (w % nk != nk - 1) {
      __syncthreads();  // this stage is refilled by the prefetch two items later
      continue;
    }
    // ---- epilogue of a tile
    const int64_t tile = blockIdx.x + (w / nk) * gridDim.x;
    if (p.KG > 1) {  // deterministic in-CTA reduction over k-groups
      if (active && kg > 0) {
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
          for (int c = 0; c < RN; ++c) red[(kg - 1) * CT + ((ty + r * p.TY) << p.tn) + col(c)] = acc[r][c];
      }
      __syncthreads();
      if (kg == 0) {
        for (int g = 1; g < p.KG; ++g) {
#pragma unroll
          for (int r = 0; r < RM; ++r)
#pragma unroll
            for (int c = 0; c < RN; ++c) {
              const C2 v = red[(g - 1) * CT + ((ty + r * p.TY) << p.tn) + col(c)];
              acc[r][c].x += v.x;
              acc[r][c].y += v.y;
            }
        }
      }
    }
    if (kg == 0 && txy < TXY) {
      C2* out = reinterpret_cast<C2*>(p.splits == 1 ? p.C : p.P);
      const int64_t base = ((int64_t)(p.splits == 1 ? 0 : split) * p.n_tiles + tile) << (p.tm + p.tn);
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        C2* row = out + base + ((int64_t)(ty + r * p.TY) << p.tn);
        if (RN >= 2 && sizeof(C2) == 8) {
#pragma unroll
          for (int c = 0; c < RN; c += 2) {
            const float4 v = make_float4((float)acc[r][c].x, (float)acc[r][c].y, (float)acc[r][c + 1].x,
                                         (float)acc[r][c + 1].y);
            *reinterpret_cast<float4*>(row + col(c)) = v;
          }
        } else {
#pragma unroll
          for (int c = 0; c < RN; ++c) row[col(c)] = acc[r][c];
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int c = 0; c < RN; ++c) { acc[r][c].x = 0; acc[r][c].y = 0; }
    __syncthreads();
  }
}

template <typename R>
__global__ void reduce_splits_kernel(const typename V2<R>::t* __restrict__ P, typename V2<R>::t* __restrict__ C,
                                     int64_t n, int splits) {
  pdl_wait();
  pdl_launch_dependents();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    typename V2<R>::t s = P[i];
    for (int k = 1; k < splits; ++k) {
      const typename V2<R>::t v = P[(int64_t)k * n + i];
      s.x += v.x;
      s.y += v.y;
    }
    C[i] = s;
  }
}

// Device slice state: the current slice index and its digits (loop order, pos 0 outermost).
struct SliceState {
  int64_t s;
  int64_t base;      // first slice of the current jt_exec_contract call
  int64_t vals_mask; // slice-value ring size - 1 (power of two)
  int32_t digits[64];
};

__global__ void set_slice_kernel(SliceState* st, int64_t s, int64_t base, int64_t vals_mask) {
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    st->s = s;
    st->base = base;
    st->vals_mask = vals_mask;
  }
}

// s += 1 and its mixed-radix digits (every sliced label has dimension d)
__global__ void advance_slice_kernel(SliceState* st, int k, int d) {
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    int64_t s = st->s + 1;
    st->s = s;
    for (int p = k - 1; p >= 0; --p) {
      st->digits[p] = (int32_t)(s % d);
      s /= d;
    }
  }
}

// acc[y] += s (complex128), y = the batch digits of the current run (positions bpos0..bpos0+nq-1,
// first most significant; y = 0 without a batch), in canonical order.
template <typename R>
__global__ void accumulate_kernel(const typename V2<R>::t* __restrict__ root, double* __restrict__ acc,
                                  double2* __restrict__ slicevals, const SliceState* __restrict__ st, int bpos0,
                                  int nq, int d) {
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double re = (double)root[0].x, im = (double)root[0].y;
    int64_t y = 0;
    for (int i = 0; i < nq; ++i) y = y * d + st->digits[bpos0 + i];
    acc[2 * y] += re;
    acc[2 * y + 1] += im;
    slicevals[(st->s - st->base) & st->vals_mask] = make_double2(re, im);
  }
}

struct PermArgs {
  const void* src;
  void* dst;
  int32_t n_outer, nt;
  int64_t o_src[kMaxOuter], o_dst[kMaxOuter];
  int64_t in_g[kMaxTile];   // tile bits in input order: src stride (smem stride = 2^i)
  int64_t out_g[kMaxTile];  // tile bits in output order: dst stride
  int32_t out_s[kMaxTile];  //   ... and smem stride
};

// MODE 0: one element per access.  MODE 1 (c64): address bit 0 stays bit 0, so element pairs
// move as 16 B on both sides.  MODE 2 (c64, bit 0 moves): 16-B loads of input-order pairs
// (input bit 0) and 16-B stores of output-order pairs (output bit 0), the two halves of a
// stored pair gathered from the tile with two 8-B shared loads.  The shared tile is
// XOR-swizzled (swz, 8-B units, bit 0 kept) so the output-order reads spread over banks.
template <typename E, int MODE>
__global__ void __launch_bounds__(256) permute_kernel(const __grid_constant__ PermArgs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* tileb = reinterpret_cast<E*>(smem_raw);
  __shared__ int64_t tin[2][64], tout[2][64];
  __shared__ int32_t tso[2][64];
  const int tid = threadIdx.x;
  for (int i = tid; i < 64; i += blockDim.x) {
    for (int h = 0; h < 2; ++h) {
      int64_t gi = 0, go = 0;
      int32_t so = 0;
      for (int b = 0; b < 6; ++b)
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nt) { gi += p.in_g[bi]; go += p.out_g[bi]; so += p.out_s[bi]; }
        }
      tin[h][i] = gi; tout[h][i] = go; tso[h][i] = so;
    }
  }
  __syncthreads();
  const int64_t blk = blockIdx.x;
  int64_t bs = 0, bd = 0;
  for (int j = 0; j < p.n_outer; ++j)
    if ((blk >> j) & 1) { bs += p.o_src[j]; bd += p.o_dst[j]; }
  const E* __restrict__ src = reinterpret_cast<const E*>(p.src);
  E* __restrict__ dst = reinterpret_cast<E*>(p.dst);
  const int sz = 1 << p.nt;
  if (MODE == 1) {
    for (int e = 2 * tid; e < sz; e += 2 * blockDim.x)
      *reinterpret_cast<float4*>(tileb + swz<E>(e)) = *reinterpret_cast<const float4*>(src + bs + tin[0][e & 63] + tin[1][e >> 6]);
    __syncthreads();
    for (int f = 2 * tid; f < sz; f += 2 * blockDim.x)
      *reinterpret_cast<float4*>(dst + bd + tout[0][f & 63] + tout[1][f >> 6]) =
          *reinterpret_cast<const float4*>(tileb + swz<E>(tso[0][f & 63] + tso[1][f >> 6]));
  } else if (MODE == 2) {
    for (int e = 2 * tid; e < sz; e += 2 * blockDim.x)
      *reinterpret_cast<float4*>(tileb + swz<E>(e)) = *reinterpret_cast<const float4*>(src + bs + tin[0][e & 63] + tin[1][e >> 6]);
    __syncthreads();
    const int s1 = tso[0][1];  // tile position of output bit 0
    for (int f = 2 * tid; f < sz; f += 2 * blockDim.x) {
      const int s0 = tso[0][f & 63] + tso[1][f >> 6];
      const E a = tileb[swz<E>(s0)], b = tileb[swz<E>(s0 + s1)];
      *reinterpret_cast<float4*>(dst + bd + tout[0][f & 63] + tout[1][f >> 6]) = make_float4(a.x, a.y, b.x, b.y);
    }
  } else {
    for (int e = tid; e < sz; e += blockDim.x) tileb[swz<E>(e)] = src[bs + tin[0][e & 63] + tin[1][e >> 6]];
    __syncthreads();
    for (int f = tid; f < sz; f += blockDim.x)
      dst[bd + tout[0][f & 63] + tout[1][f >> 6]] = tileb[swz<E>(tso[0][f & 63] + tso[1][f >> 6])];
  }
}

}  // namespace jt
