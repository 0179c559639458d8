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
//   warps 0-7  lane-linear (bank-conflict-free) reads of the packed tile; each element is
//              multiplied by A (registers), partial sums over the K bits held by lanes are
//              combined by a shuffle butterfly, those held by iterations in registers; C is laid
//              out [M bits][tile n bits][outer bits]
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
  // lane-linear read map of the packed tile (11 - (3 - KT) rank bits): lanes = ranks 0-4, warp
  // bits and iteration bits = the remaining ranks; *_kidx / *_nidx: the k-index / column-index
  // bit each of them carries (0 if none); lane_kmask / it_kmask: which lane / iteration bits are K
  int32_t warp_rank[3], warp_nidx[3];
  int32_t lane_kidx[5], lane_nidx[5], lane_kmask;
  int32_t it_rank[3], it_kidx[3], it_nidx[3], it_kmask;
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
    // ===================== compute =====================
    // The tile lands packed in B-stride order (2^(8+KT) elements, 11 bits at most).  Reads are
    // lane-linear and bank-conflict free: lane l reads rank bits 0-4 = l, the warp index gives
    // three further ranks (warp_rank), and the iteration index it gives the remaining ranks
    // (it_rank).  Each element (n, k) is multiplied by A[:, k]; the K bits held by lanes are
    // summed by a shuffle butterfly, those held by iterations in registers; the lanes whose
    // K bits are 0 then write their columns' outputs ([M][tile n][outer] layout).
    constexpr int NIT = 1 << (11 - 8);  // iterations per thread = (2^(8+KT) / 256) for KT = 3
    const int nit = 1 << KT;            // actual iterations (2^(8+KT) elements / 256 threads)
    int wpos = 0, nw = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if ((warp >> j) & 1) { wpos += 1 << p.warp_rank[j]; nw |= p.warp_nidx[j]; }
    int kl = 0, nl = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if ((lane >> i) & 1) { kl |= p.lane_kidx[i]; nl |= p.lane_nidx[i]; }
    int itpos[NIT], itk[NIT], itn[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      int ps = 0, kk = 0, nn = 0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if ((it >> b) & 1) { ps += 1 << p.it_rank[b]; kk |= p.it_kidx[b]; nn |= p.it_nidx[b]; }
      itpos[it] = ps;
      itk[it] = kk;
      itn[it] = nn;
    }
    const int lane_kmask = p.lane_kmask, it_kmask = p.it_kmask;
    float2 ak[NIT][NM];  // A[m][k] of this thread's element in iteration it (k is fixed per thread)
#pragma unroll
    for (int it = 0; it < NIT; ++it)
#pragma unroll
      for (int m = 0; m < NM; ++m) ak[it][m] = As[m * NK + ((kl | itk[it]) & (NK - 1))];
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t_it = 0; t_it < my; ++t_it) {
      tc::mbar_wait(&full[st], ph);
      const float2* raw = reinterpret_cast<const float2*>(R + st * p.rbytes) + lane + wpos;
      float2 acc[NIT][NM];
#pragma unroll
      for (int it = 0; it < NIT; ++it)
#pragma unroll
        for (int m = 0; m < NM; ++m) acc[it][m] = make_float2(0.f, 0.f);
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        if (it < nit) {
          const float2 b = raw[itpos[it]];
#pragma unroll
          for (int m = 0; m < NM; ++m) {
            const float2 x = ak[it][m];
            acc[it][m].x = fmaf(x.x, b.x, fmaf(-x.y, b.y, acc[it][m].x));
            acc[it][m].y = fmaf(x.x, b.y, fmaf(x.y, b.x, acc[it][m].y));
          }
        }
      }
      // iterations that differ only in K bits share a slot (it & ~it_kmask): fold them in order
#pragma unroll
      for (int it = 1; it < NIT; ++it)
        if (it < nit && (it & it_kmask) != 0)
#pragma unroll
          for (int s2 = 0; s2 < NIT; ++s2)
            if (s2 == (it & ~it_kmask))
#pragma unroll
              for (int m = 0; m < NM; ++m) {
                acc[s2][m].x += acc[it][m].x;
                acc[s2][m].y += acc[it][m].y;
              }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[st]);
      if (++st == RS) { st = 0; ph ^= 1; }
      // sum over the K bits held by lanes (butterfly), fixed order
#pragma unroll
      for (int i = 0; i < 5; ++i)
        if ((lane_kmask >> i) & 1)
#pragma unroll
          for (int it = 0; it < NIT; ++it)
            if (it < nit && (it & it_kmask) == 0)
#pragma unroll
              for (int m = 0; m < NM; ++m) {
                acc[it][m].x += __shfl_xor_sync(0xffffffffu, acc[it][m].x, 1 << i);
                acc[it][m].y += __shfl_xor_sync(0xffffffffu, acc[it][m].y, 1 << i);
              }
      if ((lane & lane_kmask) == 0) {
        const int64_t t = (int64_t)blockIdx.x + t_it * gridDim.x;
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
          if (it < nit && (it & it_kmask) == 0) {
            const int n = nl | nw | itn[it];
            float2* out = p.C + (t << (8 + TM)) + ((int64_t)n << TM);
            if constexpr (NM == 1) {
              out[0] = acc[it][0];
            } else {
#pragma unroll
              for (int m = 0; m < NM; m += 2)
                *reinterpret_cast<float4*>(out + m) =
                    make_float4(acc[it][m].x, acc[it][m].y, acc[it][m + 1].x, acc[it][m + 1].y);
            }
          }
        }
      }
    }
  }
}

}  // namespace jt
