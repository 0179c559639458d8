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

constexpr int kMaxOuter = 48;
constexpr int kMaxTile = 14;

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
  int64_t o_sA[kMaxOuter], o_sB[kMaxOuter];    // outer M/N bit j: strides in A and B
  int64_t ok_sA[kMaxOuter], ok_sB[kMaxOuter];  // outer K bit j
  int64_t gA[kMaxTile], gB[kMaxTile];          // tile bit (sorted by operand stride): global stride
  int32_t sA[kMaxTile], sB[kMaxTile];          //   ... and shared-memory stride
};

template <typename C2>
__device__ __forceinline__ void cmac(C2& acc, const C2 a, const C2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

template <typename R, int RM, int RN>
__global__ void __launch_bounds__(256) gett_kernel(const __grid_constant__ GettArgs p) {
  using C2 = typename V2<R>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t tgA[2][64], tgB[2][64];
  __shared__ int32_t tsA[2][64], tsB[2][64];
  const int tid = threadIdx.x;
  for (int i = tid; i < 64; i += blockDim.x) {
    // lo tables: tile bits 0..5; hi tables: tile bits 6..11 (of the stride-sorted order)
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0, gb = 0;
      int32_t s = 0, sb = 0;
      for (int b = 0; b < 6; ++b) {
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nA) { g += p.gA[bi]; s += p.sA[bi]; }
          if (bi < p.nB) { gb += p.gB[bi]; sb += p.sB[bi]; }
        }
      }
      tgA[h][i] = g; tsA[h][i] = s;
      tgB[h][i] = gb; tsB[h][i] = sb;
    }
  }
  __syncthreads();
  C2* sAm = reinterpret_cast<C2*>(smem_raw);
  C2* sBm = sAm + (1 << p.nA);
  const int64_t tile = blockIdx.x;
  const int split = blockIdx.y;
  int64_t baseA = 0, baseB = 0;
  for (int j = 0; j < p.n_outer; ++j)
    if ((tile >> j) & 1) { baseA += p.o_sA[j]; baseB += p.o_sB[j]; }
  const int64_t it0 = (int64_t)split * p.k_iters / p.splits;
  const int64_t it1 = (int64_t)(split + 1) * p.k_iters / p.splits;
  const int TXY = p.TX * p.TY;
  const int kg = tid / TXY;
  const int txy = tid - kg * TXY;
  const int tx = txy % p.TX, ty = txy / p.TX;
  const bool active = kg < p.KG;
  C2 acc[RM][RN];
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) { acc[r][c].x = 0; acc[r][c].y = 0; }
  const C2* __restrict__ A = reinterpret_cast<const C2*>(p.A);
  const C2* __restrict__ B = reinterpret_cast<const C2*>(p.B);
  const int szA = 1 << p.nA, szB = 1 << p.nB, TK = 1 << p.tk;
  for (int64_t it = it0; it < it1; ++it) {
    int64_t oa = baseA, ob = baseB;
    for (int j = 0; j < p.n_ok; ++j)
      if ((it >> j) & 1) { oa += p.ok_sA[j]; ob += p.ok_sB[j]; }
    if (it != it0) __syncthreads();
    for (int e = tid; e < szA; e += blockDim.x)
      sAm[tsA[0][e & 63] + tsA[1][e >> 6]] = A[oa + tgA[0][e & 63] + tgA[1][e >> 6]];
    for (int e = tid; e < szB; e += blockDim.x)
      sBm[tsB[0][e & 63] + tsB[1][e >> 6]] = B[ob + tgB[0][e & 63] + tgB[1][e >> 6]];
    __syncthreads();
    if (active) {
      for (int kk = kg; kk < TK; kk += p.KG) {
        C2 a[RM], b[RN];
#pragma unroll
        for (int r = 0; r < RM; ++r) a[r] = sAm[(kk << p.tm) + ty + r * p.TY];
#pragma unroll
        for (int c = 0; c < RN; ++c) b[c] = sBm[(kk << p.tn) + tx + c * p.TX];
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
          for (int c = 0; c < RN; ++c) cmac(acc[r][c], a[r], b[c]);
      }
    }
  }
  const int CT = 1 << (p.tm + p.tn);
  if (p.KG > 1) {  // deterministic in-CTA reduction over k-groups
    __syncthreads();
    C2* red = sAm;
    if (active && kg > 0) {
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < RN; ++c)
          red[(kg - 1) * CT + ((ty + r * p.TY) << p.tn) + tx + c * p.TX] = acc[r][c];
    }
    __syncthreads();
    if (kg == 0) {
      for (int g = 1; g < p.KG; ++g) {
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
          for (int c = 0; c < RN; ++c) {
            const C2 v = red[(g - 1) * CT + ((ty + r * p.TY) << p.tn) + tx + c * p.TX];
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
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int c = 0; c < RN; ++c) out[base + ((ty + r * p.TY) << p.tn) + tx + c * p.TX] = acc[r][c];
  }
}

template <typename R>
__global__ void reduce_splits_kernel(const typename V2<R>::t* __restrict__ P, typename V2<R>::t* __restrict__ C,
                                     int64_t n, int splits) {
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

template <typename R>
__global__ void accumulate_kernel(const typename V2<R>::t* __restrict__ root, double* __restrict__ acc,
                                  double2* __restrict__ slicevals, int64_t idx) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double re = (double)root[0].x, im = (double)root[0].y;
    acc[0] += re;
    acc[1] += im;
    slicevals[idx] = make_double2(re, im);
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

template <typename E>
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
  for (int e = tid; e < sz; e += blockDim.x) tileb[e] = src[bs + tin[0][e & 63] + tin[1][e >> 6]];
  __syncthreads();
  for (int f = tid; f < sz; f += blockDim.x) dst[bd + tout[0][f & 63] + tout[1][f >> 6]] = tileb[tso[0][f & 63] + tso[1][f >> 6]];
}

}  // namespace jt
