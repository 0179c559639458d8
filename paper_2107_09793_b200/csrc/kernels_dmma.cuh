// K4: complex128 pairwise contraction on the FP64 tensor cores (DMMA).
//
// "c128 -> K4 DMMA"; the contraction is C = sum_K A*B of PAPER.md l.92-105
// (Eq. sequence), GEMM-shaped at the GBS nodes (arithmetic intensity 30..400 FLOP/B, far above
// the FP64 ridge of ~6 FLOP/B at the measured 6.5 TB/s), so the FP64 pipe is the bound.
//
// Measured on B200 (scripts/fp64_probe.cu, profiles/r01_fp64_probe.txt): DFMA 36.2 TFLOP/s,
// mma.sync.m8n8k4.f64 37.0 TFLOP/s -- the same pipe rate, but one DMMA is 256 FMA per warp
// instruction with one 8-B operand per lane, where CUDA-core complex FMA (K2) needs a 16-B
// shared load per 4 DFMA and saturates the shared-memory port together with the FP64 pipe.
//
// Tiling, gather tables, cp.async double buffering, split-K and the output layout are K2's
// (GettArgs, kernels.cuh): the planner picks tile bit sets tile-M / tile-N / tile-K that hold
// each operand's lowest address bits, the operand tiles land in shared memory in their own bit
// order (XOR-swizzled) and the output tile is written as [tile-N bits][tile-M bits].  Only the
// compute differs: warps tile the C tile (TY x TX warps, each 8*SMT rows x 8*SNT columns of
// 8x8 sub-tiles); per K step of 4 complex every lane loads one complex of A (row lane/4,
// k lane%4) and one of B (k lane%4, column lane/4) -- exactly the m8n8k4 f64 fragments -- and
// the complex product is four real MMAs on the planar parts:
//   Cr += Ar*Br + (-Ai)*Bi,   Ci += Ar*Bi + Ai*Br.
// The accumulators (Cr, Ci fragments: row lane/4, columns 2*(lane%4)+{0,1}) stay in registers.
//
// GAUSS = true (SURVEY 8a a5 "3M"): the complex product as three real MMAs (Gauss's trick),
//   P += Ar*Br,  Q += Ai*Bi,  R += (Ar+Ai)*(Br+Bi);   Cr = P - Q,  Ci = R - P - Q
// -- 25% fewer DMMAs for the FP64-bound GBS nodes, at 1.5x the accumulator registers (so warp
// tiles of at most 8 sub-tiles).  Rounding: |dC| <~ 3 eps sum|a||b| per K step instead of
// 2 eps sum|a||b| (normwise; the amplitude parity bar is normwise, A13).  Opt-in
// (JETB200_K4_3M=1): measured slower than 4M on the C4 nodes (see k4_gauss_enabled, exec.cu).
#pragma once

#include "kernels.cuh"

namespace jt {

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Operand tile copy for CTAs of a multiple of 64 threads: thread tid copies elements
// e = tid + i*nthr, so e & 63 = tid & 63 is fixed -- its low gather offset and the low part of
// the (GF(2)-linear) shared-memory swizzle are hoisted; per element one table load remains.
__device__ __forceinline__ void load_tile_c128_g64(double2* dst, const double2* src, int n, const int64_t (*tg)[64],
                                                   int tid, int nthr) {
  const int sz = 1 << n;
  const int lo = tid & 63;
  const double2* s0 = src + tg[0][lo];
  const int d0 = swz<double2>(lo);
  for (int e = tid; e < sz; e += nthr) cp_async16(dst + (d0 ^ swz<double2>(e & ~63)), s0 + tg[1][e >> 6]);
}

__device__ __forceinline__ void load_tile_c128(double2* dst, const double2* src, int n, const int64_t (*tg)[64],
                                               int tid, int nthr) {
  if ((nthr & 63) == 0) load_tile_c128_g64(dst, src, n, tg, tid, nthr);
  else load_tile(dst, src, n, false, tg, tid, nthr);
}

// p.TY x p.TX warps (rows x columns of warp tiles), KG = 1.  2^tm = 8*SMT*TY, 2^tn = 8*SNT*TX,
// tile-K >= 4 complex.
template <int SMT, int SNT, bool GAUSS>
__global__ void __launch_bounds__(256) gett_dmma_kernel(const __grid_constant__ GettArgs p) {
  using C2 = double2;
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
  C2* sA0 = reinterpret_cast<C2*>(smem_raw);
  const int stage = szA + szB;
  int* posKA = reinterpret_cast<int*>(sA0 + 2 * stage);
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
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp % p.TY, wn = warp / p.TY;
  const int g4 = lane >> 2, t4 = lane & 3;
  int offM[SMT], offN[SNT];
#pragma unroll
  for (int i = 0; i < SMT; ++i) offM[i] = swz<C2>(deposit(wm * 8 * SMT + 8 * i + g4, p.pM, p.tm));
#pragma unroll
  for (int j = 0; j < SNT; ++j) offN[j] = swz<C2>(deposit(wn * 8 * SNT + 8 * j + g4, p.pN, p.tn));
  const C2* __restrict__ A = reinterpret_cast<const C2*>(p.A) + slice_off(p.sv, true);
  const C2* __restrict__ B = reinterpret_cast<const C2*>(p.B) + slice_off(p.sv, false);
  // operand offsets of the next item to load: recomputed from the bits at a tile start,
  // stepped by one delta per K iteration otherwise (no per-item bit loops)
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
  // 4M: cr, ci are Cr, Ci.  3M: cr = P, ci = Q, cs = R (cs unused by 4M; the compiler drops it)
  double cr[SMT][SNT][2], ci[SMT][SNT][2], cs[SMT][SNT][2];
#pragma unroll
  for (int i = 0; i < SMT; ++i)
#pragma unroll
    for (int j = 0; j < SNT; ++j)
      cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = cs[i][j][0] = cs[i][j][1] = 0.0;
  if (total > 0) {
    tile_start();
    load_tile_c128(sA0, A + ld_oa, p.nA, tgA, tid, nthr);
    load_tile_c128(sA0 + szA, B + ld_ob, p.nB, tgB, tid, nthr);
    cp_async_commit();
  }
  for (int64_t w = 0; w < total; ++w) {
    const int buf = (int)(w & 1);
    if (w + 1 < total) {
      advance();
      C2* nxt = sA0 + (buf ^ 1) * stage;
      load_tile_c128(nxt, A + ld_oa, p.nA, tgA, tid, nthr);
      load_tile_c128(nxt + szA, B + ld_ob, p.nB, tgB, tid, nthr);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const C2* sA = sA0 + buf * stage;
    const C2* sB = sA + szA;
#pragma unroll 2
    for (int k0 = 0; k0 < TK; k0 += 4) {
      const int ka = posKA[k0 + t4], kb = posKB[k0 + t4];
      C2 a[SMT], b[SNT];
#pragma unroll
      for (int i = 0; i < SMT; ++i) a[i] = sA[ka ^ offM[i]];
#pragma unroll
      for (int j = 0; j < SNT; ++j) b[j] = sB[kb ^ offN[j]];
      if (GAUSS) {
        // three passes (P, Q, R accumulators 2*SMT*SNT instructions apart)
        double sa[SMT], sb[SNT];
#pragma unroll
        for (int i = 0; i < SMT; ++i) sa[i] = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < SNT; ++j) sb[j] = b[j].x + b[j].y;
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(cr[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(ci[i][j], a[i].y, b[j].y);
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(cs[i][j], sa[i], sb[j]);
      } else {
        // four passes over the sub-tiles, so that the two MMAs into one accumulator are
        // 2*SMT*SNT instructions apart (DMMA latency hidden by independent accumulators)
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(cr[i][j], a[i].x, b[j].x);
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(ci[i][j], a[i].x, b[j].y);
#pragma unroll
        for (int i = 0; i < SMT; ++i) {
          const double nai = -a[i].y;
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(cr[i][j], nai, b[j].y);
        }
#pragma unroll
        for (int i = 0; i < SMT; ++i)
#pragma unroll
          for (int j = 0; j < SNT; ++j) dmma884(ci[i][j], a[i].y, b[j].x);
      }
    }
    if (w % nk != nk - 1) {
      __syncthreads();  // this stage is refilled by the prefetch two items later
      continue;
    }
    // ---- epilogue of a tile: row m = wm*8*SMT + 8i + lane/4, columns n, n+1 with
    // n = wn*8*SNT + 8j + 2*(lane%4): 32 contiguous bytes per lane, 128 B per row quad
    const int64_t tile = blockIdx.x + (w / nk) * gridDim.x;
    C2* out = reinterpret_cast<C2*>(p.splits == 1 ? p.C : p.P);
    const int64_t base = ((int64_t)(p.splits == 1 ? 0 : split) * p.n_tiles + tile) << (p.tm + p.tn);
#pragma unroll
    for (int i = 0; i < SMT; ++i) {
      C2* row = out + base + ((int64_t)(wm * 8 * SMT + 8 * i + g4) << p.tn);
#pragma unroll
      for (int j = 0; j < SNT; ++j) {
        const int n = wn * 8 * SNT + 8 * j + 2 * t4;
        if (GAUSS) {
          row[n] = make_double2(cr[i][j][0] - ci[i][j][0], cs[i][j][0] - cr[i][j][0] - ci[i][j][0]);
          row[n + 1] = make_double2(cr[i][j][1] - ci[i][j][1], cs[i][j][1] - cr[i][j][1] - ci[i][j][1]);
        } else {
          row[n] = make_double2(cr[i][j][0], ci[i][j][0]);
          row[n + 1] = make_double2(cr[i][j][1], ci[i][j][1]);
        }
        cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = cs[i][j][0] = cs[i][j][1] = 0.0;
      }
    }
    __syncthreads();
  }
}

}  // namespace jt
