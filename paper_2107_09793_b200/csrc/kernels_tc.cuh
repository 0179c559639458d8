// K3: complex64 pairwise contraction on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Used for "small tensor applied to a big tensor" contractions:
// C[m][n] = sum_k A[m][k] B[k][n] with A small (all its bits in the tile) and B big.  The
// complex product is one real GEMM (4M form) D = X * Y with
//   X[n][2k+t]  = (Re B[k][n], Im B[k][n])         -- B's interleaved complex data, K-major
//   Y[2k+t][2m+s]: s=0: ( Re A, -Im A ), s=1: ( Im A, Re A )   (t = 0, 1)
// so that D[n][2m] = Re C[m][n] and D[n][2m+1] = Im C[m][n]: the accumulator row n is the
// interleaved complex column n of C.  MMA_M = 128 rows of n (TMEM lanes), MMA_N = 2*2^tm
// columns, K' = 2*2^tk (TF32, 8 per instruction).  Precision: 3xTF32 -- every fp32 operand is
// split into hi = rna_tf32(x) and lo = x - hi, and D += Xhi*Yhi + Xhi*Ylo + Xlo*Yhi with FP32
// accumulation in TMEM (1xTF32 misses 1e-4 over a deep tree, 3xTF32 does not).
//
// Shared-memory operands use the UMMA K-major SWIZZLE_NONE canonical layout: core matrices of
// 8 rows x 16 B; LBO = 128 B (next core matrix along K), SBO = (K'/4) * 128 B (next 8 rows).
// Every tile bit contributes a fixed byte offset in that layout, so the gather into it uses
// the same lo/hi offset tables as K2.  One CTA = 256 threads; thread 0 issues the MMAs; all
// threads prefetch the next tile's B into registers while the current tile's epilogue
// (tcgen05.ld -> 256-B coalesced stores) runs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace jt {

constexpr int kTcMaxTile = 13;  // 7 row bits + up to 6 K bits

struct TcArgs {
  const float2* A;  // small operand (all bits in the tile)
  const float2* B;  // big operand
  float2* C;        // output, layout [7 row (n) bits][tm bits][outer bits]
  int64_t n_tiles;
  int32_t n_outer, tm, tk, nX;   // nX = 7 + tk tile bits of B
  int32_t Np, Kp;                // MMA N (2*2^tm padded to >= 16), K' (2*2^tk padded to >= 8)
  int32_t sbo;                   // bytes between 8-row core-matrix groups (X and Y)
  uint32_t idesc;                // instruction descriptor (kind::tf32, M=128, N=Np, F32 accum)
  uint32_t tmem_cols;
  int64_t o_sB[kMaxOuter];       // outer (row) bit j of B: stride
  int64_t gX[kTcMaxTile];        // B tile bit j (stride order): global stride
  int32_t sX[kTcMaxTile];        //   ... and byte offset in the X tile (canonical layout)
  int64_t aM[8], aK[8];          // A strides of its M bits / K bits
  SliceView sv;
};

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  // start address [0,14), LBO [16,30), SBO [32,46) in 16-B units; version 1 at [46,48);
  // base offset 0; layout SWIZZLE_NONE (0) at [61,64)
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "JT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra JT_WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace tc

// PER = elements of the B tile each thread carries between the prefetch and the smem store
// (2^(7+tk) / 256 = 2^(tk-1)).
template <int PER>
__global__ void __launch_bounds__(256, 1) gett_tc_kernel(const __grid_constant__ TcArgs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int64_t tg[2][64];
  __shared__ int32_t ts[2][64];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // smem carve: Xhi | Xlo | Yhi | Ylo, each operand tile = rows * Kp * 4 bytes
  const int xbytes = 128 * p.Kp * 4;
  const int ybytes = p.Np * p.Kp * 4;
  unsigned char* Xhi = smem_raw;
  unsigned char* Xlo = Xhi + xbytes;
  unsigned char* Yhi = Xlo + xbytes;
  unsigned char* Ylo = Yhi + ybytes;
  for (int i = tid; i < 64; i += blockDim.x) {
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0;
      int32_t s = 0;
      for (int b = 0; b < 6; ++b)
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nX) { g += p.gX[bi]; s += p.sX[bi]; }
        }
      tg[h][i] = g;
      ts[h][i] = s;
    }
  }
  // zero the operand tiles (padding rows/columns of K' and N' must be finite zeros)
  for (int i = tid; i < (2 * xbytes + 2 * ybytes) / 16; i += blockDim.x)
    reinterpret_cast<float4*>(smem_raw)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_base_sh)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_sh;
  // ---- Y = expanded small operand (hi/lo), built once: row = 2m+s, col = 2k+t
  {
    const int nm = 1 << p.tm, nk = 1 << p.tk;
    for (int idx = tid; idx < nm * nk; idx += blockDim.x) {
      const int m = idx % nm, k = idx / nm;
      int64_t off = 0;
      for (int i = 0; i < p.tm; ++i) if ((m >> i) & 1) off += p.aM[i];
      for (int i = 0; i < p.tk; ++i) if ((k >> i) & 1) off += p.aK[i];
      const float2 a = p.A[off + slice_off(p.sv, true)];
      const float vals[2][2] = {{a.x, -a.y}, {a.y, a.x}};  // [s][t]
      for (int s = 0; s < 2; ++s)
        for (int t = 0; t < 2; ++t) {
          const int row = 2 * m + s, kk = 2 * k + t;
          const int byte = (row & 7) * 16 + (row >> 3) * p.sbo + (kk >> 2) * 128 + (kk & 3) * 4;
          const float x = vals[s][t];
          const float hi = tc::tf32_hi(x);
          *reinterpret_cast<float*>(Yhi + byte) = hi;
          *reinterpret_cast<float*>(Ylo + byte) = x - hi;
        }
    }
  }
  float2 reg[PER];
  auto tile_base = [&](int64_t t) {
    int64_t o = 0;
    for (int j = 0; j < p.n_outer; ++j) if ((t >> j) & 1) o += p.o_sB[j];
    return o;
  };
  const int64_t boff = slice_off(p.sv, false);
  auto prefetch = [&](int64_t t) {
    const float2* src = p.B + boff + tile_base(t);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * 256;
      reg[i] = src[tg[0][e & 63] + tg[1][e >> 6]];
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = tid + i * 256;
      const int byte = ts[0][e & 63] + ts[1][e >> 6];
      const float hx = tc::tf32_hi(reg[i].x), hy = tc::tf32_hi(reg[i].y);
      *reinterpret_cast<float2*>(Xhi + byte) = make_float2(hx, hy);
      *reinterpret_cast<float2*>(Xlo + byte) = make_float2(reg[i].x - hx, reg[i].y - hy);
    }
  };
  int64_t t = blockIdx.x;
  if (t < p.n_tiles) {
    prefetch(t);
  }
  uint32_t phase = 0;
  for (; t < p.n_tiles; t += gridDim.x) {
    stash();
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const int64_t tn = t + gridDim.x;
    if (tn < p.n_tiles) prefetch(tn);  // in flight during the MMAs and the epilogue
    if (tid == 0) {
      const int ksteps = p.Kp / 8;
      for (int ks = 0; ks < ksteps; ++ks) {
        const uint64_t xh = tc::sdesc(Xhi + ks * 256, 128, p.sbo), xl = tc::sdesc(Xlo + ks * 256, 128, p.sbo);
        const uint64_t yh = tc::sdesc(Yhi + ks * 256, 128, p.sbo), yl = tc::sdesc(Ylo + ks * 256, 128, p.sbo);
        tc::mma_tf32(tmem, xh, yh, p.idesc, ks > 0 ? 1u : 0u);
        tc::mma_tf32(tmem, xh, yl, p.idesc, 1u);
        tc::mma_tf32(tmem, xl, yh, p.idesc, 1u);
      }
      tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, phase);
    phase ^= 1;
    tc::fence_after();
    // ---- epilogue: warp w reads TMEM lanes 32*(w%4)...; warps w and w+4 split the columns
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;  // n within the tile
    // column range of this warp: halves when Np >= 32, else warps 0-3 take all 16 columns
    const int cbeg = p.Np >= 32 ? half * (p.Np / 2) : (half ? p.Np : 0);
    const int cend = p.Np >= 32 ? (half + 1) * (p.Np / 2) : (half ? p.Np : p.Np);
    float2* out = p.C + (t << (7 + p.tm));
    const int nm = 1 << p.tm;
    for (int c0 = cbeg; c0 < cend; c0 += 16) {
      float v[16];
      tc::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int m = c0 / 2 + j;
        if (m < nm) out[row + ((int64_t)m << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
      }
    }
    tc::fence_before();
    __syncthreads();  // TMEM and the X tile are free for the next tile
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

}  // namespace jt
