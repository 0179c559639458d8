// K2s: streaming contraction for skinny c64 nodes (register-resident small operand).
//
// "Small tensor applied to a big tensor" where the small operand A is tiny
// (2^TM x 2^KT complex, TM <= 2, KT <= 3): C[m][n] = sum_k A[m][k] B[k][n] with N ~ 2^25 on the
// Sycamore m=14 path.  Arithmetic intensity is ~2-3 FLOP/B, so the node is a pure HBM stream
// (skinny contractions run on a CUDA-core kernel; roofline = HBM): every B byte is
// read once and every C byte written once (algorithmic bytes 8(|A|+|B|+|C|)).
//
//   A (<= 32 complex) is held in registers by every thread.
//   Thread <-> column n (an assignment of B's free bits, enumerated in the output's bit order):
//   lanes take consecutive n, so with B's lowest-stride free bits lowest in the output the 32
//   lanes of a warp read 32 neighbouring columns per k (coalesced) and write 32 neighbouring
//   outputs per m.  A column's B offset is the sum of four 512-entry shared tables (9 column bits
//   each, GF(2)-linear bit -> stride map); its 2^KT values are loaded as 8-B complex, or as 16-B
//   k-pairs when B's K bit 0 has stride 1.  Two columns per thread per iteration keep 2^(KT+1)
//   loads in flight.  FP32 complex MACs in k order (as K2's cmac).
//   Output layout: [n_lo column bits][M bits][remaining column bits] -- the K2 layout of the same
//   node ([tile-N][tile-M][outer]), so consumers see exactly what K2 would have produced.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace jt {

constexpr int kStreamMaxCols = 36;  // column bits covered by the four 9-bit tables

struct StreamArgs {
  const float2* A;
  const float2* B;
  float2* C;
  int32_t n_cols;                // column (free B) bits, in output order
  int32_t n_lo;                  // column bits below the M bits in the output
  int32_t vec;                   // 1: k-pair (K bit 0, B stride 1) loads as one 16-B load
  int64_t sN[kStreamMaxCols];    // B stride of column bit j
  int64_t kofs[8];               // B offset of k (all K bits)
  int64_t aofs[32];              // A offset of (m, k) at m * 2^KT + k
  SliceView sv;
};

template <int TM, int KT>
__global__ void __launch_bounds__(256, 2) stream_gett_kernel(const __grid_constant__ StreamArgs p) {
  constexpr int NM = 1 << TM, NK = 1 << KT;
  __shared__ int64_t tab[4][512];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4 * 512; i += blockDim.x) {
    const int h = i >> 9, v = i & 511;
    int64_t s = 0;
    for (int b = 0; b < 9; ++b)
      if (((v >> b) & 1) && 9 * h + b < p.n_cols) s += p.sN[9 * h + b];
    tab[h][v] = s;
  }
  __syncthreads();
  pdl_wait();  // A and B are written by the previous kernels of the sequence
  pdl_launch_dependents();
  const float2* __restrict__ A = p.A + slice_off(p.sv, true);
  const float2* __restrict__ B = p.B + slice_off(p.sv, false);
  float2 a[NM][NK];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int k = 0; k < NK; ++k) a[m][k] = A[p.aofs[m * NK + k]];
  int64_t ko[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) ko[k] = p.kofs[k];
  const int64_t ncol = int64_t(1) << p.n_cols;
  const int64_t lo_mask = (int64_t(1) << p.n_lo) - 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto col_off = [&](int64_t c) {
    return tab[0][c & 511] + tab[1][(c >> 9) & 511] + tab[2][(c >> 18) & 511] + tab[3][(c >> 27) & 511];
  };
  auto store = [&](int64_t c, const float2 (&b)[NK]) {
    float2* out = p.C + (c & lo_mask) + ((c >> p.n_lo) << (p.n_lo + TM));
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < NK; ++k) cmac(acc, a[m][k], b[k]);
      out[(int64_t)m << p.n_lo] = acc;
    }
  };
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x + tid; c0 < ncol; c0 += 2 * stride) {
    const int64_t c1 = c0 + stride;
    const bool two = c1 < ncol;
    const float2* b0p = B + col_off(c0);
    const float2* b1p = B + (two ? col_off(c1) : col_off(c0));
    float2 b0[NK], b1[NK];
    if (KT >= 1 && p.vec) {
#pragma unroll
      for (int k = 0; k < NK; k += 2) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(b0p + ko[k]));
        const float4 y = __ldg(reinterpret_cast<const float4*>(b1p + ko[k]));
        b0[k] = make_float2(x.x, x.y);
        b0[k + 1] = make_float2(x.z, x.w);
        b1[k] = make_float2(y.x, y.y);
        b1[k + 1] = make_float2(y.z, y.w);
      }
    } else {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        b0[k] = __ldg(b0p + ko[k]);
        b1[k] = __ldg(b1p + ko[k]);
      }
    }
    store(c0, b0);
    if (two) store(c1, b1);
  }
}

}  // namespace jt
