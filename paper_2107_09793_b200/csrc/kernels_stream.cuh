// K2s: streaming contraction for skinny c64 nodes (sm_100a, TMA-fed).
//
// "Small tensor applied to a big tensor" where the small operand A is tiny
// (2^TM x 2^KT complex, TM <= 3, KT <= 3): C[m][n] = sum_k A[m][k] B[k][n] with N ~ 2^25 on the
// Sycamore m=14 path.  Arithmetic intensity is ~2-3 FLOP/B, so the node is a pure HBM stream:
// every B byte is read once and every C byte written once (algorithmic bytes 8(|A|+|B|+|C|)).
//
//   tile  = 256 columns n (B's 8 lowest-stride free bits) x all 2^KT k: 2^(8+KT) elements
//           (<= 16 KB) moved by TMA-engine bulk copies of its contiguous runs, landing packed in
//           B-stride order (bit b at byte 8 << rank b)
//   warp 8     issues the copies (one per lane) into a ring of RS stages (full/empty mbarriers)
//   warps 0-7  one thread per column n: read its 2^KT values, multiply by A (registers),
//              write its 2^TM outputs as one contiguous run: C is laid out
//              [M bits][tile n bits][outer bits], so a warp stores 32 x 2^TM x 8 B contiguous
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels_tc.cuh"

namespace jt {

struct StreamArgs {
  const float2* A;
  const float2* B;
  float2* C;
  int64_t n_tiles;
  int32_t n_outer, rstages, rbytes;
  int64_t o_sB[kMaxOuter];    // B stride of outer (tile-index) bit j
  int32_t rofs_n[8], rofs_k[3];  // landing byte offset of tile column bit i / K bit j
  int32_t ncopy, copy_bytes;  // bulk copies per tile (its stride-1 run each), copy j at xoff[j]
  int64_t xoff[32];
  int64_t aM[3], aK[3];       // A strides of its M / K bits
  SliceView sv;
};

template <int TM, int KT>
__global__ void __launch_bounds__(288, 1) stream_gett_kernel(const __grid_constant__ StreamArgs p) {
  constexpr int NM = 1 << TM, NK = 1 << KT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  __shared__ float2 As[NM * NK];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* R = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  if (tid == 0) {
    for (int i = 0; i < p.rstages; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  pdl_launch_dependents();
  if (tid < NM * NK) {
    const int m = tid / NK, k = tid % NK;
    int64_t off = slice_off(p.sv, true);
#pragma unroll
    for (int i = 0; i < TM; ++i) off += ((m >> i) & 1) ? p.aM[i] : 0;
#pragma unroll
    for (int i = 0; i < KT; ++i) off += ((k >> i) & 1) ? p.aK[i] : 0;
    As[tid] = p.A[off];
  }
  __syncthreads();
  const int64_t my = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int RS = p.rstages;
  if (warp == 8) {
    // ===================== TMA issuer =====================
    const int64_t boff = slice_off(p.sv, false);
    const int64_t o_s0 = lane < p.n_outer ? p.o_sB[lane] : 0;
    const int64_t o_s1 = lane + 32 < p.n_outer ? p.o_sB[lane + 32] : 0;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < my; ++it) {
      const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
      int64_t tb = (((t >> lane) & 1) ? o_s0 : 0) + ((lane < 16 && ((t >> (lane + 32)) & 1)) ? o_s1 : 0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(0xffffffffu, tb, o);
      if (lane == 0) {
        if (it >= RS) tc::mbar_wait(&empty[st], ph ^ 1);
        tc::mbar_expect_tx(&full[st], (uint32_t)p.rbytes);
      }
      __syncwarp();
      if (lane < p.ncopy)
        tc::bulk_g2s(R + st * p.rbytes + lane * p.copy_bytes, p.B + (boff + tb + p.xoff[lane]), (uint32_t)p.copy_bytes,
                     &full[st]);
      if (++st == RS) { st = 0; ph ^= 1; }
    }
  } else {
    // ===================== compute: one column n per thread =====================
    float2 a[NM][NK];
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int k = 0; k < NK; ++k) a[m][k] = As[m * NK + k];
    int32_t noff = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) noff += ((tid >> i) & 1) ? p.rofs_n[i] : 0;
    int32_t koff[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      int32_t o = 0;
#pragma unroll
      for (int j = 0; j < KT; ++j) o += ((k >> j) & 1) ? p.rofs_k[j] : 0;
      koff[k] = o;
    }
    int st = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < my; ++it) {
      tc::mbar_wait(&full[st], ph);
      const unsigned char* raw = R + st * p.rbytes + noff;
      float2 b[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) b[k] = *reinterpret_cast<const float2*>(raw + koff[k]);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[st]);
      if (++st == RS) { st = 0; ph ^= 1; }
      float2 c[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        float re = 0.f, im = 0.f;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          re = fmaf(a[m][k].x, b[k].x, re);
          re = fmaf(-a[m][k].y, b[k].y, re);
          im = fmaf(a[m][k].x, b[k].y, im);
          im = fmaf(a[m][k].y, b[k].x, im);
        }
        c[m] = make_float2(re, im);
      }
      const int64_t t = (int64_t)blockIdx.x + it * gridDim.x;
      float2* out = p.C + (t << (8 + TM)) + ((int64_t)tid << TM);
      if constexpr (NM == 1) {
        out[0] = c[0];
      } else {
#pragma unroll
        for (int m = 0; m < NM; m += 2)
          *reinterpret_cast<float4*>(out + m) = make_float4(c[m].x, c[m].y, c[m + 1].x, c[m + 1].y);
      }
    }
  }
}

}  // namespace jt
