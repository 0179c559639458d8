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

constexpr int kTcMaxTile = 12;  // 7 row bits + up to 5 K bits per chunk

struct TcArgs {
  const float2* A;  // small operand (all bits in the tile)
  const float2* B;  // big operand
  float2* C;        // output, layout [7 row (n) bits][tm bits][outer bits]
  int64_t n_tiles;
  int32_t n_outer, tm, K, tkc, n_kc, nX, swz;  // K contracted bits, tkc per chunk, n_kc = 2^(K-tkc)
  int32_t Np, Kpc;                             // MMA N (2*2^tm); TF32 per row per chunk (2*2^tkc)
  int32_t sbo_x, sbo_y;                        // bytes between 8-row core-matrix groups
  int32_t xbuf, yplane;                        // bytes of one X buffer / one Y chunk plane (hi or lo)
  uint32_t idesc;                              // kind::tf32, M=128, N=Np, F32 accumulate, K-major
  uint32_t tmem_cols;                          // 2 accumulators of Np columns
  int32_t xstages;                             // X stages (2 or 3): cp.async runs xstages-1 items ahead
  int64_t o_sB[kMaxOuter];                     // outer (row) bit j of B: stride
  int64_t o_kB[4];                             // chunk-index bit j of B: stride
  int64_t gX[kTcMaxTile];                      // B chunk-tile bit j (stride order): global stride
  int32_t sX[kTcMaxTile];                      //   ... and its byte offset in the X buffer (XOR-combined)
  int64_t aM[8], aK[8];                        // A strides of its M bits / K bits
  SliceView sv;
};

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// UMMA shared-memory descriptor: start address [0,14), LBO [16,30), SBO [32,46) in 16-B
// units, version 1 at [46,48), layout type at [61,64) (0 = none, 2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// 3xTF32 split by truncation: hi = x with the low 13 mantissa bits cleared (exactly a TF32
// value, so the MMA reads it exactly whatever its own rounding), lo = x - hi (exact in fp32);
// lo is then read at TF32 precision (relative error 2^-11 of lo, ~2^-22 of x).
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

}  // namespace tc

// Byte offset of A-operand element (row r, tf32 column kk) inside one X buffer / Y plane.
__device__ __forceinline__ int tc_off(int r, int kk, int sbo, int swz) {
  if (swz) return (r & 7) * 128 + (r >> 3) * 1024 + ((((kk >> 2) ^ (r & 7)) & 7) << 4) + (kk & 3) * 4;
  return (r & 7) * 16 + (r >> 3) * sbo + (kk >> 2) * 128 + (kk & 3) * 4;
}

// Warp-specialised K3.  Warps 0-3: epilogue (TMEM lane quarter w -> 256-B coalesced stores);
// warps 4-11: producers (B chunk tile -> shared stage by cp.async, lo split in place); warp 12:
// MMA issuer (one elected thread).  Two X stages and two TMEM accumulators, so the loads of
// item i+1, the MMAs of item i and the epilogue of the previous tile overlap.  Y (the expanded
// small operand) is built once and stays resident for every K chunk.
// PER = B-tile elements per producer thread = 2^(7+tkc) / 256.
template <int PER>
__global__ void __launch_bounds__(416, 1) gett_tc_kernel(const __grid_constant__ TcArgs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int64_t tg[2][64];
  __shared__ int32_t ts[2][64];
  __shared__ __align__(8) uint64_t full[3], empty[3], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 1024-B aligned carve: X stage s = [hi | lo], then Y planes [hi c=0..n_kc-1 | lo ...]
  unsigned char* base = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* X = base;
  unsigned char* Yhi = X + 2 * p.xstages * p.xbuf;
  unsigned char* Ylo = Yhi + p.n_kc * p.yplane;
  for (int i = tid; i < 64; i += blockDim.x) {
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0;
      int32_t s = 0;
      for (int b = 0; b < 6; ++b)
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nX) { g += p.gX[bi]; s ^= p.sX[bi]; }
        }
      tg[h][i] = g;
      ts[h][i] = s;
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_base_sh)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      tc::mbar_init(&full[i], 256);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- Y = expanded small operand (hi/lo) for every K chunk: row = 2m+s, col = 2k+t
  {
    const int nm = 1 << p.tm, nk = 1 << p.K, nkc = 1 << p.tkc;
    const int64_t aoff = slice_off(p.sv, true);
    for (int idx = tid; idx < nm * nk; idx += blockDim.x) {
      const int m = idx % nm, k = idx / nm;
      int64_t off = aoff;
      for (int i = 0; i < p.tm; ++i) if ((m >> i) & 1) off += p.aM[i];
      for (int i = 0; i < p.K; ++i) if ((k >> i) & 1) off += p.aK[i];
      const float2 a = p.A[off];
      const float vals[2][2] = {{a.x, -a.y}, {a.y, a.x}};  // [s][t]
      const int c = k / nkc, kl = k % nkc;
      for (int s = 0; s < 2; ++s)
        for (int t = 0; t < 2; ++t) {
          const int byte = c * p.yplane + tc_off(2 * m + s, 2 * kl + t, p.sbo_y, p.swz);
          const float x = vals[s][t];
          const float hi = tc::tf32_trunc(x);
          *reinterpret_cast<float*>(Yhi + byte) = hi;
          *reinterpret_cast<float*>(Ylo + byte) = x - hi;
        }
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_sh;
  const int64_t my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles * p.n_kc;
  auto tile_of = [&](int64_t it) { return (int64_t)blockIdx.x + (it / p.n_kc) * gridDim.x; };
  const uint32_t layout = p.swz ? 2u : 0u;
  const uint32_t lbo = p.swz ? 16u : 128u;
  const uint32_t kstep = p.swz ? 32u : 256u;  // descriptor advance per 8-TF32 K step

  if (warp >= 4 && warp < 12) {
    // ===================== producers =====================
    // cp.async (no registers, commit groups instead of scoreboards) lands each item's B data
    // straight into its X stage at the operand-layout position, XSTAGES-1 items ahead; the
    // thread then splits the elements it copied in place into hi (X_hi) and lo (X_lo).
    const int ptid = tid - 128;  // 0..255
    const int64_t boff = slice_off(p.sv, false);
    int bytes_of[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = ptid + i * 256;
      bytes_of[i] = ts[0][e & 63] ^ ts[1][e >> 6];
    }
    const int S = p.xstages;
    auto issue = [&](int64_t it) {
      const int s = (int)(it % S);
      const uint32_t ph = (uint32_t)((it / S) & 1);
      tc::mbar_wait(&empty[s], ph ^ 1);  // stage free (first use passes)
      const int64_t t = tile_of(it);
      const int c = (int)(it % p.n_kc);
      int64_t src = boff;
      for (int j = 0; j < p.n_outer; ++j) if ((t >> j) & 1) src += p.o_sB[j];
      for (int j = 0; j < p.K - p.tkc; ++j) if ((c >> j) & 1) src += p.o_kB[j];
      unsigned char* xhi = X + s * 2 * p.xbuf;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int e = ptid + i * 256;
        cp_async8(xhi + bytes_of[i], p.B + src + tg[0][e & 63] + tg[1][e >> 6]);
      }
    };
    const int64_t depth = S - 1;
    for (int64_t q = 0; q < depth; ++q) {
      if (q < items) issue(q);
      cp_async_commit();  // (possibly empty) group per slot keeps the group arithmetic uniform
    }
    for (int64_t it = 0; it < items; ++it) {
      // groups committed so far: depth + it; item it's group is the oldest of the last depth
      if (S == 3) cp_async_wait<1>();
      else cp_async_wait<0>();
      const int s = (int)(it % S);
      unsigned char* xhi = X + s * 2 * p.xbuf;
      unsigned char* xlo = xhi + p.xbuf;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const float2 v = *reinterpret_cast<const float2*>(xhi + bytes_of[i]);
        const float hx = tc::tf32_trunc(v.x), hy = tc::tf32_trunc(v.y);
        *reinterpret_cast<float2*>(xhi + bytes_of[i]) = make_float2(hx, hy);
        *reinterpret_cast<float2*>(xlo + bytes_of[i]) = make_float2(v.x - hx, v.y - hy);
      }
      tc::fence_proxy_async();
      tc::mbar_arrive(&full[s]);
      if (it + depth < items) issue(it + depth);
      cp_async_commit();
    }
  } else if (warp == 12) {
    // ===================== MMA issuer =====================
    const bool leader = lane == 0;
    int64_t tt = 0;
    const int S = p.xstages;
    for (int64_t it = 0; it < items; ++it) {
      const int s = (int)(it % S);
      const uint32_t ph = (uint32_t)((it / S) & 1);
      const int c = (int)(it % p.n_kc);
      const int b = (int)(tt & 1);
      const uint32_t tph = (uint32_t)((tt >> 1) & 1);
      if (c == 0) tc::mbar_wait(&tempty[b], tph ^ 1);  // accumulator drained (first use passes)
      tc::mbar_wait(&full[s], ph);
      tc::fence_after();
      if (leader) {
        const uint32_t d = tmem + (uint32_t)(b * p.Np);
        const uint32_t xh = tc::smem_u32(X + s * 2 * p.xbuf), xl = xh + p.xbuf;
        const uint32_t yh = tc::smem_u32(Yhi + c * p.yplane), yl = tc::smem_u32(Ylo + c * p.yplane);
        const int ksteps = p.Kpc / 8;
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint32_t o = ks * kstep;
          const uint64_t dxh = tc::sdesc(xh + o, lbo, p.sbo_x, layout), dxl = tc::sdesc(xl + o, lbo, p.sbo_x, layout);
          const uint64_t dyh = tc::sdesc(yh + o, lbo, p.sbo_y, layout), dyl = tc::sdesc(yl + o, lbo, p.sbo_y, layout);
          tc::mma_tf32(d, dxh, dyh, p.idesc, (c > 0 || ks > 0) ? 1u : 0u);
          tc::mma_tf32(d, dxh, dyl, p.idesc, 1u);
          tc::mma_tf32(d, dxl, dyh, p.idesc, 1u);
        }
        tc::mma_commit(&empty[s]);                      // stage s free once these MMAs finish
        if (c == p.n_kc - 1) tc::mma_commit(&tfull[b]);  // tile accumulated
      }
      __syncwarp();
      if (c == p.n_kc - 1) ++tt;
    }
  } else if (warp < 4) {
    // ===================== epilogue =====================
    const int row = warp * 32 + lane;
    const int nm = 1 << p.tm;
    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      const int b = (int)(tt & 1);
      const uint32_t tph = (uint32_t)((tt >> 1) & 1);
      tc::mbar_wait(&tfull[b], tph);
      tc::fence_after();
      const int64_t t = (int64_t)blockIdx.x + tt * gridDim.x;
      float2* out = p.C + (t << (7 + p.tm));
      for (int c0 = 0; c0 < p.Np; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * p.Np + c0), v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int m = c0 / 2 + j;
          if (m < nm) out[row + ((int64_t)m << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[b]);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

}  // namespace jt
