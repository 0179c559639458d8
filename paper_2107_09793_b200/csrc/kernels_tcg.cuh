// K3g: general complex64 contraction on tcgen05 -- both operands streamed.
//
// Same 4M / 3xTF32 formulation as K3 (kernels_tc.cuh), for contractions where the "small"
// operand does not fit a resident tile: large GEMM-shaped nodes (e.g. Sycamore m=20:
// M = N = 2^6 tiles, K = 2^12..2^17) that are tensor-bound rather than HBM-bound.
//   output tile = 128 rows n (7 bits of B) x Mt = 2^tmt complex columns m (bits of A)
//   K loop over chunks of 16 complex (4 bits); the remaining contracted bits index the chunks
//   per item (tile, chunk): producers cp.async the B chunk (128 x 16) and the A chunk (Mt x 16)
//   into raw shared rings, then split B into hi/lo TF32 in TMEM (the MMA's A operand) and expand
//   A into the Y operand [[Re,-Im],[Im,Re]] hi/lo in shared memory (SWIZZLE_128B, K-major)
//   MMA warp: 4 K steps x 3 (hi*hi, hi*lo, lo*hi) tcgen05.mma kind::tf32 per item
//   epilogue warps: TMEM accumulator -> 256-B coalesced stores of the complex output tile (first
//   accumulation segment); later segments -> shared staging (8 complex columns x 128 rows, two
//   buffers) -> TMA-engine bulk FP32 add-reductions (cp.reduce.async.bulk .add.f32) of 8-KB runs,
//   in segment order (the issuing thread waits for the previous segment's group before the next)
#pragma once

#include "kernels_tc.cuh"

namespace jt {

struct TcgArgs {
  const float2* A;
  const float2* B;
  float2* C;                // layout [7 n bits][tmt m bits][outer N bits][outer M bits]
  int64_t n_tiles;          // 2^(n_oN + n_oM)
  int32_t n_oN, n_oM;       // outer bits of the tile index: N bits first (B strides), then M (A)
  int32_t tmt, lg_kc;       // M tile bits; K chunk-index bits (n_kc = 2^lg_kc)
  int32_t lg_kcs;           // chunks per accumulation segment (log2, <= lg_kc): the TMEM
                            // accumulator restarts every 2^lg_kcs chunks and the epilogue adds the
                            // segment sums into the output tile in order (long-K precision)
  int32_t nXb, nAb;         // tile bits of a B chunk (7 + 4) and of an A chunk (tmt + 4)
  int32_t Np;               // MMA N = 2 * 2^tmt
  uint32_t idesc, tmem_cols;
  int32_t rstages, rbytes_b, rbytes_a, acc_bufs;
  int32_t ystages;          // Y (expanded A) shared stages, 2..4
  int32_t lg_bm;            // tile raster: bands of 2^lg_bm M tiles (<= n_oM) walked N-major
  int64_t o_B[32], o_A[32]; // outer N bit strides in B / outer M bit strides in A
  int64_t k_B[32], k_A[32]; // chunk-index bit strides in B / in A
  int64_t gB[12], gA[12];   // chunk-tile bits (stride order): global strides
  int32_t sB[12], sA[12];   //   ... and raw byte offsets (XOR-combinable)
  int32_t tma;              // 1: chunks arrive by TMA (gett_tcg_kernel<TMT, true>)
  int32_t rot;              // 1: rotating accumulator regions (see tcg::Rot), 2 X stages
  int32_t lg_xs;            // log2 of the TMEM X stages (2, or 1 with rot)
  int32_t epi_warp;         // 1: later segments drained per warp (own staging, 256-B bulk adds)
  int32_t ncopyB, copyB_bytes, ncopyA, copyA_bytes;  // bulk copies per chunk (TcArgs::ncopy)
  int64_t xoffB[32], xoffA[32];
  int32_t rofsB_n[7], rofsB_k[4], rofsA_m[7], rofsA_k[4];  // TMA landing byte offsets per bit
  SliceView sv;
};

// K1 on the K3g path (the paper's transpose before the GEMM): an operand whose
// tile / chunk bits do not form a few long runs in its own layout is first copied into the
// layout K3g wants (item bits lowest, one contiguous run per item) by this bit-gather:
// dst[i] = src[slice offset + sum_j bit_j(i) * s[j]] for i < 2^n_bits.  Used only for the
// compute-bound K3g nodes, where the copy's 16 B/element is negligible against the MMA time.
struct GatherArgs {
  const float2* src;
  float2* dst;
  int32_t n_bits, is_a;
  int64_t s[40];
  SliceView sv;
};

__global__ void __launch_bounds__(256) view_gather_kernel(const __grid_constant__ GatherArgs p) {
  __shared__ int64_t tab[5][256];
  for (int i = threadIdx.x; i < 5 * 256; i += blockDim.x) {
    const int h = i >> 8, v = i & 255;
    int64_t o = 0;
    for (int b = 0; b < 8; ++b)
      if (((v >> b) & 1) && 8 * h + b < p.n_bits) o += p.s[8 * h + b];
    tab[h][v] = o;
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const float2* __restrict__ src = p.src + slice_off(p.sv, p.is_a != 0);
  const int64_t n = int64_t(1) << p.n_bits, stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll 4
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p.dst[i] = __ldg(src + tab[0][i & 255] + tab[1][(i >> 8) & 255] + tab[2][(i >> 16) & 255] +
                     tab[3][(i >> 24) & 255] + tab[4][(i >> 32) & 255]);
}

namespace tcg {
// sum over the set bits j < n of v of stride[j], computed lane-parallel and butterfly-reduced
__device__ __forceinline__ int64_t bits_sum(int64_t v, int n, const int64_t* stride, int lane) {
  int64_t part = 0;
  for (int j = lane; j < n; j += 32)
    if ((v >> j) & 1) part += stride[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  return part;
}
// Processing order -> canonical tile index (N bits low, M bits high).  Consecutive t (the
// CTAs of one wave) cover 2^lg_bm M tiles x ~148/2^lg_bm N tiles, so each B chunk is read
// from HBM once per band and served to the band's other CTAs from L2 (and each A chunk to
// the wave's N tiles), instead of once per M tile.
// Rotating accumulator regions (p.rot): the 256 accumulator columns of a tile are two halves of
// 128 (64 complex columns each, MMA N = 128), and three 128-column TMEM regions rotate between
// them.  The halves' accumulation segments are staggered by half a segment (half 0 restarts at
// chunk c = 0 mod S, half 1 at c = S/2 mod S), so at every boundary only ONE half needs a fresh
// region -- the spare one -- while its finished region drains: the MMAs never wait for the
// epilogue (the single-accumulator layout stalls them for every drain, 12-14% of the C5 nodes).
// Opt-in: measured slower than the single accumulator (N = 128 MMAs, 2 X stages; see exec.cu).
// MMA warp and epilogue run this same deterministic schedule: regions are handed back in event
// order (FIFO), use counts give the mbarrier parities.
struct Rot {
  int reg[2], fifo[4], head, tail, use[3];
  __device__ __forceinline__ void init() {
    reg[0] = 0; reg[1] = 1; fifo[0] = 2; head = 0; tail = 1;
    use[0] = 1; use[1] = 1; use[2] = 0;
  }
  // take the next region; *before = its uses so far (parity of the release to wait for)
  __device__ __forceinline__ int acquire(int* before) {
    const int r = fifo[head & 3];
    ++head;
    *before = use[r]++;
    return r;
  }
  __device__ __forceinline__ void release(int r) { fifo[tail & 3] = r; ++tail; }
};

__device__ __forceinline__ int64_t raster(int64_t t, const TcgArgs& p) {
  const int lb = p.lg_bm;
  const int64_t mlo = t & ((int64_t(1) << lb) - 1);
  const int64_t n = (t >> lb) & ((int64_t(1) << p.n_oN) - 1);
  const int64_t band = t >> (lb + p.n_oN);
  return n | (((band << lb) | mlo) << p.n_oN);
}
}  // namespace tcg

// TMA = true: warp 13 issues the B and A chunks of each item as TMA-engine bulk copies of their
// contiguous runs (one per lane) into the raw rings (rfull /
// rempty mbarriers); the producers only split X and expand Y (no gathers, no named barrier).
template <int TMT, bool TMA>
__global__ void __launch_bounds__(TMA ? 448 : 416, 1) gett_tcg_kernel(const __grid_constant__ TcgArgs p) {
  constexpr int MT = 1 << TMT;       // complex columns of the tile
  constexpr int NP = 2 * MT;         // MMA N
  constexpr int PERB = 2048 / 256;   // B chunk elements per producer thread
  constexpr int PERA = (MT * 16 + 255) / 256;
  constexpr int PAIRS = (MT * 8 + 255) / 256;  // (m, k-pair) units of the Y expansion per thread
  constexpr int KPC = 32;            // TF32 columns of one X row (16 complex)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int64_t tgb[2][64], tga[2][64];
  __shared__ int32_t tsb[2][64], tsa[2][64];
  __shared__ int64_t dkB[32], dkA[32];  // chunk c -> c+1 offset steps, by trailing ones of c
  __shared__ __align__(8) uint64_t full[4], xempty[4], yempty[4], tfull[4], tempty[4], rfull[8], rempty[8];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* base = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* Y = base;                            // ystages x [hi plane | lo plane], NP x 128 B each
  unsigned char* RB = Y + p.ystages * 2 * NP * 128;   // raw B ring
  unsigned char* RA = RB + p.rstages * p.rbytes_b;    // raw A ring
  float2* ES = reinterpret_cast<float2*>(RA + p.rstages * p.rbytes_a);  // epilogue staging, 2 x 8 KB
  for (int i = tid; i < 64; i += blockDim.x) {
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0, ga = 0;
      int32_t s = 0, sa = 0;
      for (int b = 0; b < 6; ++b)
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nXb) { g += p.gB[bi]; s ^= p.sB[bi]; }
          if (bi < p.nAb) { ga += p.gA[bi]; sa ^= p.sA[bi]; }
        }
      tgb[h][i] = g; tsb[h][i] = s;
      tga[h][i] = ga; tsa[h][i] = sa;
    }
  }
  if (tid < p.lg_kc) {
    int64_t b = p.k_B[tid], a = p.k_A[tid];
    for (int j = 0; j < tid; ++j) { b -= p.k_B[j]; a -= p.k_A[j]; }
    dkB[tid] = b;
    dkA[tid] = a;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tmem_base_sh)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&full[i], 256);
      tc::mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) tc::mbar_init(&yempty[i], 1);
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    if (TMA)
      for (int i = 0; i < p.rstages; ++i) {
        tc::mbar_init(&rfull[i], 1);
        tc::mbar_init(&rempty[i], 8);
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t xcol0 = p.rot ? 384u : (uint32_t)(p.acc_bufs * NP);  // rot: regions 0-383, X 384-511
  const int64_t my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles << p.lg_kc;
  const int64_t kc_mask = ((int64_t)1 << p.lg_kc) - 1;

  if (TMA && warp >= 4 && warp < 12) {
    // ===================== producers (TMA-fed) =====================
    const int ptid = tid - 128;
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;
    const int RS = p.rstages;
    int32_t rB = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i) rB += ((row >> i) & 1) ? p.rofsB_n[i] : 0;
    int32_t kB[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int k = half * 8 + q;
      int32_t o = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) o += ((k >> j) & 1) ? p.rofsB_k[j] : 0;
      kB[q] = o;
    }
    int32_t a0[PAIRS], a1[PAIRS];
#pragma unroll
    for (int q = 0; q < PAIRS; ++q) {
      const int u = (ptid + q * 256) & (MT * 8 - 1);
      const int m = u >> 3, kp = u & 7;
      int32_t o = 0;
#pragma unroll
      for (int i = 0; i < TMT; ++i) o += ((m >> i) & 1) ? p.rofsA_m[i] : 0;
#pragma unroll
      for (int j = 1; j < 4; ++j) o += ((kp >> (j - 1)) & 1) ? p.rofsA_k[j] : 0;
      a0[q] = o;
      a1[q] = o + p.rofsA_k[0];
    }
    int rst = 0, ys = 0;
    uint32_t rph = 0, yph = 0;
    for (int64_t it = 0; it < items; ++it) {
      const int xs = (int)(it & ((1 << p.lg_xs) - 1));
      tc::mbar_wait(&rfull[rst], rph);
      tc::mbar_wait(&xempty[xs], (uint32_t)(((it >> p.lg_xs) & 1) ^ 1));
      tc::mbar_wait(&yempty[ys], yph ^ 1u);
      tc::fence_after();
      // ---- X: this thread's row, half of the chunk -> hi/lo TF32 in TMEM
      {
        const unsigned char* raw = RB + rst * p.rbytes_b + rB;
        float hi[16], lo[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float2 v = *reinterpret_cast<const float2*>(raw + kB[q]);
          hi[2 * q] = tc::tf32_rna(v.x);
          lo[2 * q] = tc::tf32_lo(v.x, hi[2 * q]);
          hi[2 * q + 1] = tc::tf32_rna(v.y);
          lo[2 * q + 1] = tc::tf32_lo(v.y, hi[2 * q + 1]);
        }
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t col = xcol0 + (uint32_t)(xs * 2 * KPC + half * 16);
        tc::tmem_st<16>(lane_addr + col, hi);
        tc::tmem_st<16>(lane_addr + col + KPC, lo);
      }
      // ---- Y: expand the A chunk into [[Re,-Im],[Im,Re]] hi/lo (SWIZZLE_128B, K-major)
      {
        const unsigned char* raw = RA + rst * p.rbytes_a;
        unsigned char* yhi = Y + ys * 2 * NP * 128;
        unsigned char* ylo = yhi + NP * 128;
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) {
          const int u = ptid + q * 256;
          if (u < MT * 8) {
            const int m = u >> 3, kp = u & 7;
            const float2 e0 = *reinterpret_cast<const float2*>(raw + a0[q]);
            const float2 e1 = *reinterpret_cast<const float2*>(raw + a1[q]);
            const float hx = tc::tf32_rna(e0.x), hy = tc::tf32_rna(e0.y), hz = tc::tf32_rna(e1.x), hw = tc::tf32_rna(e1.y);
            const float lx = tc::tf32_lo(e0.x, hx), ly = tc::tf32_lo(e0.y, hy), lz = tc::tf32_lo(e1.x, hz),
                        lw = tc::tf32_lo(e1.y, hw);
            const int ra0 = 2 * m, ra1 = 2 * m + 1;
            const int b0 = (ra0 & 7) * 128 + (ra0 >> 3) * 1024 + ((kp ^ (ra0 & 7)) << 4);
            const int b1 = (ra1 & 7) * 128 + (ra1 >> 3) * 1024 + ((kp ^ (ra1 & 7)) << 4);
            *reinterpret_cast<float4*>(yhi + b0) = make_float4(hx, -hy, hz, -hw);
            *reinterpret_cast<float4*>(ylo + b0) = make_float4(lx, -ly, lz, -lw);
            *reinterpret_cast<float4*>(yhi + b1) = make_float4(hy, hx, hw, hz);
            *reinterpret_cast<float4*>(ylo + b1) = make_float4(ly, lx, lw, lz);
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&rempty[rst]);
      if (++rst == RS) { rst = 0; rph ^= 1; }
      tc::fence_proxy_async();
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&full[xs]);
      if (++ys == p.ystages) { ys = 0; yph ^= 1u; }
    }
  } else if (TMA && warp == 13) {
    // ===================== TMA issuer =====================
    const int64_t boff = slice_off(p.sv, false), aoff = slice_off(p.sv, true);
    const int64_t ob = lane < p.n_oN ? p.o_B[lane] : 0, oa = lane < p.n_oM ? p.o_A[lane] : 0;
    const int RS = p.rstages;
    int64_t ct = 0, cc = 0, tileB = 0, tileA = 0, kBo = 0, kAo = 0;
    auto tile_bases = [&]() {
      const int64_t t = tcg::raster((int64_t)blockIdx.x + ct * gridDim.x, p);
      int64_t b = ((t >> lane) & 1) ? ob : 0;
      int64_t a = (((t >> p.n_oN) >> lane) & 1) ? oa : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
      }
      tileB = boff + b;
      tileA = aoff + a;
    };
    tile_bases();
    int wst = 0;
    uint32_t wph = 0;
    for (int64_t it = 0; it < items; ++it) {
      if (lane == 0) {
        if (it >= RS) tc::mbar_wait(&rempty[wst], wph ^ 1);
        tc::mbar_expect_tx(&rfull[wst], (uint32_t)(p.rbytes_b + p.rbytes_a));
      }
      __syncwarp();
      if (lane < p.ncopyB)
        tc::bulk_g2s(RB + wst * p.rbytes_b + lane * p.copyB_bytes, p.B + (tileB + kBo + p.xoffB[lane]),
                     (uint32_t)p.copyB_bytes, &rfull[wst]);
      if (lane < p.ncopyA)
        tc::bulk_g2s(RA + wst * p.rbytes_a + lane * p.copyA_bytes, p.A + (tileA + kAo + p.xoffA[lane]),
                     (uint32_t)p.copyA_bytes, &rfull[wst]);
      if (++wst == RS) { wst = 0; wph ^= 1; }
      if (cc == kc_mask) {
        cc = 0;
        kBo = kAo = 0;
        ++ct;
        tile_bases();
      } else {
        const int tz = __ffsll(~cc) - 1;
        kBo += dkB[tz];
        kAo += dkA[tz];
        ++cc;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ===================== producers =====================
    const int ptid = tid - 128;
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;
    const int RS = p.rstages;
    const int64_t boff = slice_off(p.sv, false), aoff = slice_off(p.sv, true);
    int64_t goffB[PERB], goffA[PERA];
    int32_t soffB[PERB], soffA[PERA];
#pragma unroll
    for (int i = 0; i < PERB; ++i) {
      const int e = ptid + i * 256;
      goffB[i] = tgb[0][e & 63] + tgb[1][e >> 6];
      soffB[i] = tsb[0][e & 63] ^ tsb[1][e >> 6];
    }
#pragma unroll
    for (int i = 0; i < PERA; ++i) {
      const int e = (ptid + i * 256) & (MT * 16 - 1);
      goffA[i] = tga[0][e & 63] + tga[1][e >> 6];
      soffA[i] = tsa[0][e & 63] ^ tsa[1][e >> 6];
    }
    // copy cursor: tile ct of this CTA, chunk cc; tile bases re-summed (lane j holds outer
    // bit j's stride) only when the tile changes, chunk offsets stepped through dkB/dkA
    const int64_t ob = lane < p.n_oN ? p.o_B[lane] : 0, oa = lane < p.n_oM ? p.o_A[lane] : 0;
    int64_t ct = 0, cc = 0, tileB = 0, tileA = 0, kB = 0, kA = 0;
    auto tile_bases = [&]() {
      const int64_t t = tcg::raster((int64_t)blockIdx.x + ct * gridDim.x, p);
      int64_t b = ((t >> lane) & 1) ? ob : 0;
      int64_t a = (((t >> p.n_oN) >> lane) & 1) ? oa : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        b += __shfl_xor_sync(0xffffffffu, b, o);
        a += __shfl_xor_sync(0xffffffffu, a, o);
      }
      tileB = boff + b;
      tileA = aoff + a;
    };
    tile_bases();
    int wst = 0;  // raw stage the next copy lands in
    auto copy = [&](int64_t) {
      unsigned char* rb = RB + wst * p.rbytes_b;
      unsigned char* ra = RA + wst * p.rbytes_a;
      if (++wst == RS) wst = 0;
      const float2* sb = p.B + (tileB + kB);
      const float2* sa = p.A + (tileA + kA);
#pragma unroll
      for (int i = 0; i < PERB; ++i) cp_async8(rb + soffB[i], sb + goffB[i]);
#pragma unroll
      for (int i = 0; i < PERA; ++i)
        if (ptid + i * 256 < MT * 16) cp_async8(ra + soffA[i], sa + goffA[i]);
      if (cc == kc_mask) {
        cc = 0;
        kB = kA = 0;
        ++ct;
        tile_bases();
      } else {
        const int tz = __ffsll(~cc) - 1;  // trailing ones of cc
        kB += dkB[tz];
        kA += dkA[tz];
        ++cc;
      }
    };
    for (int q = 0; q < RS - 1; ++q) {
      if (q < items) copy(q);
      cp_async_commit();
    }
    int rst = 0;  // raw stage of item it
    int ys = 0;
    uint32_t yph = 0;  // Y stage of item it and its ring pass parity
    for (int64_t it = 0; it < items; ++it) {
      switch (RS) {
        case 2: cp_async_wait<0>(); break;
        case 3: cp_async_wait<1>(); break;
        case 4: cp_async_wait<2>(); break;
        case 5: cp_async_wait<3>(); break;
        default: cp_async_wait<4>(); break;
      }
      tc::bar_sync(1, 256);
      if (it + RS - 1 < items) copy(it + RS - 1);
      cp_async_commit();
      const int xs = (int)(it & ((1 << p.lg_xs) - 1));
      tc::mbar_wait(&xempty[xs], (uint32_t)(((it >> p.lg_xs) & 1) ^ 1));
      tc::mbar_wait(&yempty[ys], yph ^ 1u);
      tc::fence_after();
      // ---- X: this thread's row, half of the chunk -> hi/lo TF32 in TMEM
      {
        const unsigned char* raw = RB + rst * p.rbytes_b + row * 128;
        float hi[16], lo[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cc = half * 4 + j;
          const float4 v = *reinterpret_cast<const float4*>(raw + ((cc ^ (row & 7)) << 4));
          const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            hi[4 * j + q] = tc::tf32_rna(x[q]);
            lo[4 * j + q] = tc::tf32_lo(x[q], hi[4 * j + q]);
          }
        }
        const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t col = xcol0 + (uint32_t)(xs * 2 * KPC + half * 16);
        tc::tmem_st<16>(lane_addr + col, hi);
        tc::tmem_st<16>(lane_addr + col + KPC, lo);
      }
      // ---- Y: expand the A chunk into [[Re,-Im],[Im,Re]] hi/lo (SWIZZLE_128B, K-major)
      {
        const unsigned char* raw = RA + rst * p.rbytes_a;
        unsigned char* yhi = Y + ys * 2 * NP * 128;
        unsigned char* ylo = yhi + NP * 128;
#pragma unroll
        for (int q = 0; q < PAIRS; ++q) {
          const int u = ptid + q * 256;
          if (u < MT * 8) {
            const int m = u >> 3, kp = u & 7;
            const float4 a = *reinterpret_cast<const float4*>(raw + m * 128 + ((kp ^ (m & 7)) << 4));
            // split each value once (rna is odd-symmetric, so -x splits as (-hi, -lo)), then
            // permute / negate into row 2m = (Re, -Im) and row 2m+1 = (Im, Re) per k
            const float hx = tc::tf32_rna(a.x), hy = tc::tf32_rna(a.y), hz = tc::tf32_rna(a.z), hw = tc::tf32_rna(a.w);
            const float lx = tc::tf32_lo(a.x, hx), ly = tc::tf32_lo(a.y, hy), lz = tc::tf32_lo(a.z, hz),
                        lw = tc::tf32_lo(a.w, hw);
            const float h0[4] = {hx, -hy, hz, -hw}, l0[4] = {lx, -ly, lz, -lw};  // row 2m   (s = 0)
            const float h1[4] = {hy, hx, hw, hz}, l1[4] = {ly, lx, lw, lz};      // row 2m+1 (s = 1)
            const int ra0 = 2 * m, ra1 = 2 * m + 1;
            const int b0 = (ra0 & 7) * 128 + (ra0 >> 3) * 1024 + ((kp ^ (ra0 & 7)) << 4);
            const int b1 = (ra1 & 7) * 128 + (ra1 >> 3) * 1024 + ((kp ^ (ra1 & 7)) << 4);
            *reinterpret_cast<float4*>(yhi + b0) = make_float4(h0[0], h0[1], h0[2], h0[3]);
            *reinterpret_cast<float4*>(ylo + b0) = make_float4(l0[0], l0[1], l0[2], l0[3]);
            *reinterpret_cast<float4*>(yhi + b1) = make_float4(h1[0], h1[1], h1[2], h1[3]);
            *reinterpret_cast<float4*>(ylo + b1) = make_float4(l1[0], l1[1], l1[2], l1[3]);
          }
        }
      }
      tc::fence_proxy_async();
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&full[xs]);
      if (++rst == RS) rst = 0;
      if (++ys == p.ystages) { ys = 0; yph ^= 1u; }
    }
  } else if (warp == 12 && p.rot) {
    // ===================== MMA issuer (rotating accumulator regions) =====================
    const bool leader = lane == 0;
    const int64_t S = (int64_t)1 << p.lg_kcs, n_kc = (int64_t)1 << p.lg_kc;
    const uint32_t idesc_h = (p.idesc & ~(0x3Fu << 17)) | ((uint32_t)(128 >> 3) << 17);  // N = 128
    tcg::Rot R;
    R.init();
    bool acc_on[2] = {false, false};
    int ys = 0;
    int64_t it = 0;
    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      if (tt > 0)
        for (int h = 0; h < 2; ++h) {
          int before;
          R.reg[h] = R.acquire(&before);
          if (before > 0) tc::mbar_wait(&tempty[R.reg[h]], (uint32_t)((before & 1) ^ 1));
          acc_on[h] = false;
        }
      for (int64_t c = 0; c < n_kc; ++c, ++it) {
        for (int h = 0; h < 2; ++h) {
          const bool bnd = c > 0 && (h == 0 ? (c & (S - 1)) == 0 : (c & (S - 1)) == (S >> 1));
          if (!bnd) continue;
          if (leader) tc::mma_commit(&tfull[R.reg[h]]);  // the half's segment is complete
          R.release(R.reg[h]);
          int before;
          R.reg[h] = R.acquire(&before);
          if (before > 0) tc::mbar_wait(&tempty[R.reg[h]], (uint32_t)((before & 1) ^ 1));
          acc_on[h] = false;
        }
        const int xs = (int)(it & 1);
        tc::mbar_wait(&full[xs], (uint32_t)((it >> 1) & 1));
        tc::fence_after();
        if (leader) {
          const uint32_t xh = tmem + xcol0 + (uint32_t)(xs * 2 * KPC), xl = xh + KPC;
          const uint32_t yh = tc::smem_u32(Y + ys * 2 * NP * 128), yl = yh + NP * 128;
#pragma unroll
          for (int ks = 0; ks < KPC / 8; ++ks)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t d = tmem + (uint32_t)(R.reg[h] * 128);
              const uint64_t dyh = tc::sdesc(yh + h * 16384 + ks * 32, 16, 1024, 2);
              const uint64_t dyl = tc::sdesc(yl + h * 16384 + ks * 32, 16, 1024, 2);
              tc::mma_tf32_ts(d, xh + ks * 8, dyh, idesc_h, (acc_on[h] || ks > 0) ? 1u : 0u);
              tc::mma_tf32_ts(d, xh + ks * 8, dyl, idesc_h, 1u);
              tc::mma_tf32_ts(d, xl + ks * 8, dyh, idesc_h, 1u);
            }
          tc::mma_commit(&xempty[xs]);
          tc::mma_commit(&yempty[ys]);
        }
        __syncwarp();
        acc_on[0] = acc_on[1] = true;
        if (++ys == p.ystages) ys = 0;
      }
      for (int h = 0; h < 2; ++h) {  // tile end: both halves' last segments
        if (leader) tc::mma_commit(&tfull[R.reg[h]]);
        R.release(R.reg[h]);
      }
    }
  } else if (warp == 12) {
    // ===================== MMA issuer =====================
    const bool leader = lane == 0;
    int64_t tt = 0;
    int ys = 0;
    const int64_t seg_mask = ((int64_t)1 << p.lg_kcs) - 1;
    for (int64_t it = 0; it < items; ++it) {
      const int xs = (int)(it & ((1 << p.lg_xs) - 1));
      const int64_t c = it & seg_mask;  // chunk within the accumulation segment
      const int b = p.acc_bufs == 2 ? (int)(tt & 1) : 0;
      const uint32_t tph = p.acc_bufs == 2 ? (uint32_t)((tt >> 1) & 1) : (uint32_t)(tt & 1);
      if (c == 0) tc::mbar_wait(&tempty[b], tph ^ 1);
      tc::mbar_wait(&full[xs], (uint32_t)((it >> p.lg_xs) & 1));
      tc::fence_after();
      if (leader) {
        const uint32_t d = tmem + (uint32_t)(b * NP);
        const uint32_t xh = tmem + xcol0 + (uint32_t)(xs * 2 * KPC), xl = xh + KPC;
        const uint32_t yh = tc::smem_u32(Y + ys * 2 * NP * 128), yl = yh + NP * 128;
#pragma unroll
        for (int ks = 0; ks < KPC / 8; ++ks) {
          const uint64_t dyh = tc::sdesc(yh + ks * 32, 16, 1024, 2), dyl = tc::sdesc(yl + ks * 32, 16, 1024, 2);
          tc::mma_tf32_ts(d, xh + ks * 8, dyh, p.idesc, (c > 0 || ks > 0) ? 1u : 0u);
          tc::mma_tf32_ts(d, xh + ks * 8, dyl, p.idesc, 1u);
          tc::mma_tf32_ts(d, xl + ks * 8, dyh, p.idesc, 1u);
        }
        tc::mma_commit(&xempty[xs]);
        tc::mma_commit(&yempty[ys]);
        if (c == seg_mask) tc::mma_commit(&tfull[b]);
      }
      __syncwarp();
      if (c == seg_mask) ++tt;
      if (++ys == p.ystages) ys = 0;
    }
  } else if (warp < 4 && p.rot) {
    // ===================== epilogue (rotating accumulator regions) =====================
    // the MMA warp's schedule replayed: every segment event (tile, half, region) in order; the
    // first segment of a half stores its 64 complex columns directly, later ones are bulk-added
    const int row = warp * 32 + lane;
    const int64_t S = (int64_t)1 << p.lg_kcs, n_kc = (int64_t)1 << p.lg_kc;
    tcg::Rot R;
    R.init();
    int q = 0;
    int seg[2] = {0, 0};
    auto drain = [&](int64_t tt, int h, int r, int u) {
      tc::mbar_wait(&tfull[r], (uint32_t)((u - 1) & 1));
      tc::fence_after();
      const int64_t t = tcg::raster((int64_t)blockIdx.x + tt * gridDim.x, p);
      float2* out = p.C + (t << (7 + TMT)) + ((int64_t)(64 * h) << 7);
      const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(r * 128);
      if (seg[h]++ == 0) {
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 16) {
          float v[16];
          tc::tmem_ld16(tbase + (uint32_t)c0, v);
#pragma unroll
          for (int j = 0; j < 8; ++j) out[row + ((int64_t)(c0 / 2 + j) << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
        }
        tc::fence_before();
        tc::mbar_arrive(&tempty[r]);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // stores before the bulk adds
        return;
      }
      if (tid == 0) tc::bulk_wait<0>();  // this half's earlier segments complete
      float v[16];
      tc::tmem_ld16(tbase, v);
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 16, ++q) {
        float2* sb = ES + (q & 1) * 1024;
        tc::bar_sync(2, 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) sb[j * 128 + row] = make_float2(v[2 * j], v[2 * j + 1]);
        if (c0 + 16 < 128) tc::tmem_ld16(tbase + (uint32_t)(c0 + 16), v);
        else {
          tc::fence_before();
          tc::mbar_arrive(&tempty[r]);
        }
        tc::fence_proxy_async();
        tc::bar_sync(2, 128);
        if (tid == 0) {
          tc::bulk_s2g_add_f32(out + ((int64_t)(c0 / 2) << 7), sb, 8192);
          tc::bulk_commit();
          tc::bulk_wait_read<1>();
        }
      }
    };
    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      seg[0] = seg[1] = 0;
      if (tt > 0)
        for (int h = 0; h < 2; ++h) {
          int before;
          R.reg[h] = R.acquire(&before);
        }
      for (int64_t c = 1; c < n_kc; ++c)
        for (int h = 0; h < 2; ++h) {
          const bool bnd = h == 0 ? (c & (S - 1)) == 0 : (c & (S - 1)) == (S >> 1);
          if (!bnd) continue;
          const int r = R.reg[h];
          drain(tt, h, r, R.use[r]);
          R.release(r);
          int before;
          R.reg[h] = R.acquire(&before);
        }
      for (int h = 0; h < 2; ++h) {
        const int r = R.reg[h];
        drain(tt, h, r, R.use[r]);
        R.release(r);
      }
    }
    if (tid == 0) tc::bulk_wait<0>();
  } else if (warp < 4) {
    // ===================== epilogue =====================
    // one accumulator drain per K segment of 2^lg_kcs chunks.  The first segment of a tile is
    // stored directly (tcgen05.ld -> 256-B coalesced stores, then a generic->async proxy fence);
    // each later segment goes through shared staging ([8 columns][128 rows], two buffers) and is
    // added by thread 0 with 8-KB bulk FP32 add-reductions (cp.reduce.async.bulk .add.f32) -- no
    // read-modify-write round trip.  Before a later segment, thread 0 waits for every earlier
    // bulk group to complete, so the adds into one element happen in segment order (the same
    // FP32 sums as a read-modify-write).
    const int row = warp * 32 + lane;
    const int lg_seg = p.lg_kc - p.lg_kcs;
    int q = 0;  // staged chunk counter (staging buffer q & 1)
    for (int64_t st = 0; st < (my_tiles << lg_seg); ++st) {
      const int64_t tt = st >> lg_seg;
      const bool first = (st & (((int64_t)1 << lg_seg) - 1)) == 0;
      const int b = p.acc_bufs == 2 ? (int)(st & 1) : 0;
      const uint32_t tph = p.acc_bufs == 2 ? (uint32_t)((st >> 1) & 1) : (uint32_t)(st & 1);
      tc::mbar_wait(&tfull[b], tph);
      tc::fence_after();
      const int64_t t = tcg::raster((int64_t)blockIdx.x + tt * gridDim.x, p);
      float2* out = p.C + (t << (7 + TMT));
      const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * NP);
      if (first) {
#pragma unroll 1
        for (int c0 = 0; c0 < NP; c0 += 16) {
          float v[16];
          tc::tmem_ld16(tbase + (uint32_t)c0, v);
#pragma unroll
          for (int j = 0; j < 8; ++j) out[row + ((int64_t)(c0 / 2 + j) << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
        }
        tc::fence_before();
        tc::mbar_arrive(&tempty[b]);
        if (lg_seg > 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // stores before the bulk adds
        continue;
      }
      if (p.epi_warp) {
        // per-warp drain: the warp's 32 rows of 8 columns -> its own 2-KB staging buffer (two
        // per warp) -> 8 bulk FP32 adds of 256 B (one per column) by lane 0; no CTA barrier
        float2* wsb = ES + warp * 512;
        if (lane == 0) tc::bulk_wait<0>();  // this warp's earlier segments complete
        __syncwarp();
        float v[16];
        tc::tmem_ld16(tbase, v);
#pragma unroll 1
        for (int c0 = 0; c0 < NP; c0 += 16, ++q) {
          float2* sb = wsb + (q & 1) * 256;
          __syncwarp();  // lane 0 waited for this buffer's previous read
#pragma unroll
          for (int j = 0; j < 8; ++j) sb[j * 32 + lane] = make_float2(v[2 * j], v[2 * j + 1]);
          if (c0 + 16 < NP) tc::tmem_ld16(tbase + (uint32_t)(c0 + 16), v);
          else {
            tc::fence_before();
            tc::mbar_arrive(&tempty[b]);
          }
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              tc::bulk_s2g_add_f32(out + ((int64_t)(c0 / 2 + j) << 7) + warp * 32, sb + j * 32, 256);
            tc::bulk_commit();
            tc::bulk_wait_read<1>();
          }
        }
        continue;
      }
      if (tid == 0) tc::bulk_wait<0>();  // earlier segments' adds complete
      float v[16];
      tc::tmem_ld16(tbase, v);
#pragma unroll 1
      for (int c0 = 0; c0 < NP; c0 += 16, ++q) {
        float2* sb = ES + (q & 1) * 1024;
        tc::bar_sync(2, 128);  // staging buffer q & 1 free (thread 0 waited for its last read)
#pragma unroll
        for (int j = 0; j < 8; ++j) sb[j * 128 + row] = make_float2(v[2 * j], v[2 * j + 1]);
        if (c0 + 16 < NP) tc::tmem_ld16(tbase + (uint32_t)(c0 + 16), v);
        else {
          tc::fence_before();
          tc::mbar_arrive(&tempty[b]);  // accumulator drained into registers / staging
        }
        tc::fence_proxy_async();
        tc::bar_sync(2, 128);  // staging written
        if (tid == 0) {
          tc::bulk_s2g_add_f32(out + ((int64_t)(c0 / 2) << 7), sb, 8192);
          tc::bulk_commit();
          tc::bulk_wait_read<1>();  // the group before (the other buffer) has been read
        }
      }
    }
    if (tid == 0 || (p.epi_warp && lane == 0)) tc::bulk_wait<0>();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

}  // namespace jt
