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
// Y (the expanded small operand, hi and lo planes, every K chunk) stays resident in shared
// memory in the UMMA K-major layout (SWIZZLE_128B when a chunk holds 16 complex, else the
// SWIZZLE_NONE canonical layout: core matrices of 8 rows x 16 B, LBO 128 B, SBO (K'/4)*128 B).
// X (the streamed big operand) is split into hi/lo by producer warps and written to tensor
// memory, from which the MMA reads it (the "TS" form).  See gett_tc_kernel below for the
// warp roles; B items reach shared memory either on the TMA engine (cp.async.bulk copies of the
// item's contiguous runs, the default) or by per-element cp.async gathers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace jt {

constexpr int kTcMaxTile = 12;  // 7 row bits + up to 5 K bits per chunk

struct TcArgs {
  const float2* A;  // small operand (all bits in the tile)
  const float2* B;  // big operand
  float2* C;        // output, layout [7 row (n) bits][tm bits][outer bits], or [tm][7 rows][outer] (mlow)
  int64_t n_tiles;
  int32_t n_outer, tm, K, tkc, n_kc, nX, swz;  // K contracted bits, tkc per chunk, n_kc = 2^(K-tkc)
  int32_t Np, Kpc;                             // MMA N (2*2^tm); TF32 per row per chunk (2*2^tkc)
  int32_t sbo_x, sbo_y;                        // bytes between 8-row core-matrix groups
  int32_t xbuf, yplane;                        // bytes of one X buffer / one Y chunk plane (hi or lo)
  uint32_t idesc;                              // kind::tf32, M=128, N=Np, F32 accumulate, K-major
  uint32_t tmem_cols;                          // 2 accumulators of Np columns
  int32_t xstages;                             // TMEM X stages (hi|lo, 2*Kpc columns each)
  int32_t rstages;                             // raw shared landing stages (cp.async depth rstages-1)
  int32_t rbytes;                              // bytes of one raw stage (128 rows x 8*2^tkc)
  int32_t acc_bufs;                            // TMEM accumulators (1, 2 or 4; > 1: epilogue overlaps
                                               // the next tiles)
  int64_t o_sB[kMaxOuter];                     // outer (row) bit j of B: stride
  int64_t o_kB[4];                             // chunk-index bit j of B: stride
  int64_t gX[kTcMaxTile];                      // B chunk-tile bit j (stride order): global stride
  int32_t sX[kTcMaxTile];                      //   ... and its byte offset in the raw stage (XOR-combined)
  int64_t aM[8], aK[8];                        // A strides of its M bits / K bits
  int8_t swz_row[3];                           // row bits (lowest B stride first) that drive the raw-row swizzle
  int32_t vecB;                                // 1: chunk-tile bit 0 is a K bit at global stride 1
                                               //    -> gather k-pairs as 16-B copies
  int32_t tma;                                 // 1: items arrive by TMA bulk copies (gett_tc_kernel<TKC, true>)
  int32_t mlow;                                // output layout [M bits][7 row bits][outer] (else [rows][M][outer])
  int32_t pairN;                               // 1: N = 16 one-chunk tiles issue Xhi * [Yhi | Ylo] as ONE
                                               // N = 32 MMA (Ylo plane right after Yhi) plus Xlo * Yhi:
                                               // 2 MMAs per K step instead of 3; the epilogue adds the halves
  int32_t acc_w;                               // TMEM columns per accumulator (Np, or 2 * Np with pairN)
  int32_t passes;                              // MMA products per K step: 3 (3xTF32); 1 only for the
                                               // JETB200_DEBUG_K3_PASSES=1 diagnostic (hi*hi, wrong digits)
  int32_t ncopy, copy_bytes;                   // bulk copies per item (the stride-1 run each) and their size
  int64_t xoff[32];                            //   ... copy j reads at item base + xoff[j], lands at j * copy_bytes
  int32_t rofs_row[7], rofs_k[5];              // TMA landing: byte offset of row bit i / chunk K bit j
                                               //   (the box is packed in B-stride order: 8 << rank)
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
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const float (&v)[N]);
template <>
__device__ __forceinline__ void tmem_st<4>(uint32_t taddr, const float (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3])
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<16>(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra JT_WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x100000)  // suspend-time hint: sleep until the phase flips, don't spin
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
// Round-to-nearest TF32 (low 13 mantissa bits zero): hi = rna(x) is an exact TF32 value, so the
// MMA reads it exactly whatever its own handling of the low mantissa bits.  (Integer form of
// cvt.rna.tf32.f32, which ptxas expands with an Inf/NaN branch; the operands here are finite.)
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// 3xTF32 low part of a streamed operand: lo = x - rna(x) is exact in fp32 and |lo| <= 2^-11 |x|;
// it is NOT rounded here -- the tensor core reads the fp32 pattern at TF32 precision, which
// perturbs lo by < 2^-10 |lo| <= 2^-21 |x| (below the dropped lo*lo term's scale of 2^-22 |x y|
// only by a factor of 2, and 2^-21 is ~15x below fp32-accumulate rounding over a 16-term K step).
// Saves two integer ops per value on the producers' critical path.
__device__ __forceinline__ float tf32_lo(float x, float hi) { return x - hi; }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// One bulk copy global -> shared on the TMA engine (16-B aligned, size a multiple of 16 B),
// completing its bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Bulk (TMA-engine) shared -> global copy / element-wise FP32 add-reduction of `bytes` (16-B
// aligned, a multiple of 16), tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_add_f32(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace tc

// Byte offset of A-operand element (row r, tf32 column kk) inside one X buffer / Y plane.
__device__ __forceinline__ int tc_off(int r, int kk, int sbo, int swz) {
  if (swz) return (r & 7) * 128 + (r >> 3) * 1024 + ((((kk >> 2) ^ (r & 7)) & 7) << 4) + (kk & 3) * 4;
  return (r & 7) * 16 + (r >> 3) * sbo + (kk >> 2) * 128 + (kk & 3) * 4;
}

// Warp-specialised K3 with the streamed operand in tensor memory.
//   warps 0-3  epilogue: TMEM accumulator -> registers -> 256-B coalesced global stores
//   warps 4-11 producers: cp.async gathers each item's B rows into a raw shared stage
//              (rstages-1 items in flight, no registers held); after a producer barrier each
//              thread takes one row (its TMEM lane) and half of the K chunk, splits it into
//              hi/lo TF32 and writes both into a TMEM X stage with tcgen05.st
//   warp 12    MMA issuer: tcgen05.mma kind::tf32 with A = X from TMEM ([a_tmem], the "TS" form)
//              and B = Y (expanded small operand, resident in shared memory), 3xTF32
//   warp 13    (TMA = true) TMA issuer: each item's contiguous runs as cp.async.bulk copies (one
//              per lane) into the raw ring, landing packed in B-stride order;
//              the producers then only read their row from shared memory, split and store
// Barriers: xfull/xempty per TMEM X stage, tfull/tempty per accumulator, rfull/rempty per raw
// stage (TMA = true; without TMA the producers sync on a named barrier per item instead).
// TKC = K bits per chunk (row of the X stage = 2*2^TKC TF32 = hi or lo).
template <int TKC, bool TMA>
__global__ void __launch_bounds__(TMA ? 448 : 416, 1) gett_tc_kernel(const __grid_constant__ TcArgs p) {
  constexpr int PER = (128 << TKC) / 256;  // B elements each producer thread copies per item
  constexpr int NCOL = 1 << TKC;           // fp32 columns (of hi or lo) each producer thread writes
  constexpr int KPC = 2 << TKC;            // TF32 columns of one X row (hi or lo)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int64_t tg[2][64];
  __shared__ int32_t ts[2][64];
  __shared__ int64_t kc_off[16];  // B offset of K chunk c (n_kc <= 16)
  __shared__ __align__(8) uint64_t xfull[4], xempty[4], tfull[4], tempty[4], rfull[16], rempty[16];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 16) {
    int64_t o = 0;
    for (int j = 0; j < p.K - p.tkc; ++j) if ((tid >> j) & 1) o += p.o_kB[j];
    kc_off[tid] = o;
  }
  // 1024-B aligned carve: Y planes [hi c=0..n_kc-1 | lo ...], then the raw stages
  unsigned char* base = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* Yhi = base;
  unsigned char* Ylo = Yhi + p.n_kc * p.yplane;
  unsigned char* R = Ylo + p.n_kc * p.yplane;
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
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&xfull[i], 256);
      tc::mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    if (TMA)
      for (int i = 0; i < p.rstages; ++i) {
        tc::mbar_init(&rfull[i], 1);   // the issuer's expect_tx arrival + the TMA bytes
        tc::mbar_init(&rempty[i], 8);  // one arrival per producer warp
      }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // the operands are written by the previous kernels of the sequence
  pdl_launch_dependents();
  // ---- Y = expanded small operand (hi/lo) for every K chunk: row = 2m+s, col = 2k+t
  {
    const int nm = 1 << p.tm, nk = 1 << p.K, nkc = 1 << p.tkc;
    if (2 * nm < p.Np)  // padded MMA N: zero the Y rows past 2*nm
      for (int i = tid; i < 2 * p.n_kc * p.yplane / 16; i += blockDim.x)
        reinterpret_cast<float4*>(Yhi)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
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
          const float hi = tc::tf32_rna(x);
          *reinterpret_cast<float*>(Yhi + byte) = hi;
          *reinterpret_cast<float*>(Ylo + byte) = tc::tf32_rna(x - hi);
        }
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t xcol0 = (uint32_t)(p.acc_bufs * p.acc_w);  // first TMEM column of the X stages
  const int64_t my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles * p.n_kc;
  const uint32_t layout = p.swz ? 2u : 0u;
  const uint32_t lbo = p.swz ? 16u : 128u;
  const uint32_t kstep = p.swz ? 32u : 256u;  // Y descriptor advance per 8-TF32 K step

  if (TMA && warp >= 4 && warp < 12) {
    // ===================== producers (TMA-fed) =====================
    // the item landed as one box packed in B-stride order: element (row n, complex k) sits at
    // byte rofs(n) + kofs(k); each thread reads its row's half of the chunk, splits, stores to TMEM
    constexpr int NQ = 1 << (TKC - 1);  // complex per thread per item
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;
    int32_t roff = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i) roff += ((row >> i) & 1) ? p.rofs_row[i] : 0;
    int32_t koff[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = half * NQ + q;
      int32_t o = 0;
#pragma unroll
      for (int j = 0; j < TKC; ++j) o += ((k >> j) & 1) ? p.rofs_k[j] : 0;
      koff[q] = o;
    }
    const int RS = p.rstages, XS = p.xstages;
    int rst = 0, xs = 0;
    uint32_t rph = 0, xph = 0;
    for (int64_t it = 0; it < items; ++it) {
      tc::mbar_wait(&rfull[rst], rph);
      const unsigned char* raw = R + rst * p.rbytes + roff;
      float hi[NCOL], lo[NCOL];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 v = *reinterpret_cast<const float2*>(raw + koff[q]);
        hi[2 * q] = tc::tf32_rna(v.x);
        lo[2 * q] = tc::tf32_lo(v.x, hi[2 * q]);
        hi[2 * q + 1] = tc::tf32_rna(v.y);
        lo[2 * q + 1] = tc::tf32_lo(v.y, hi[2 * q + 1]);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&rempty[rst]);  // this warp is done with the raw stage
      if (++rst == RS) { rst = 0; rph ^= 1; }
      tc::mbar_wait(&xempty[xs], xph ^ 1);  // TMEM X stage free
      tc::fence_after();
      const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
      const uint32_t col = xcol0 + (uint32_t)(xs * 2 * KPC + half * NCOL);
      tc::tmem_st<NCOL>(lane_addr + col, hi);
      tc::tmem_st<NCOL>(lane_addr + col + KPC, lo);
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&xfull[xs]);
      if (++xs == XS) { xs = 0; xph ^= 1; }
    }
  } else if (TMA && warp == 13) {
    // ===================== TMA issuer =====================
    const int64_t boff = slice_off(p.sv, false);
    const int64_t o_s = lane < p.n_outer ? p.o_sB[lane] : 0;
    auto tile_base = [&](int64_t ct) {
      const int64_t t = (int64_t)blockIdx.x + ct * gridDim.x;
      int64_t tb = ((t >> lane) & 1) ? o_s : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(0xffffffffu, tb, o);
      return boff + tb;
    };
    const int RS = p.rstages;
    int64_t ct = 0, cbase = tile_base(0);
    int cc = 0, wst = 0;
    uint32_t wph = 0;
    for (int64_t it = 0; it < items; ++it) {
      if (lane == 0) {
        if (it >= RS) tc::mbar_wait(&rempty[wst], wph ^ 1);  // all producer warps released it
        tc::mbar_expect_tx(&rfull[wst], (uint32_t)p.rbytes);
      }
      __syncwarp();
      if (lane < p.ncopy)
        tc::bulk_g2s(R + wst * p.rbytes + lane * p.copy_bytes, p.B + (cbase + kc_off[cc] + p.xoff[lane]),
                     (uint32_t)p.copy_bytes, &rfull[wst]);
      if (++wst == RS) { wst = 0; wph ^= 1; }
      if (++cc == p.n_kc) {
        cc = 0;
        ++ct;
        cbase = tile_base(ct);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ===================== producers =====================
    const int ptid = tid - 128;  // 0..255
    const int64_t boff = slice_off(p.sv, false);
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;  // this thread's TMEM lane (row n of the tile)
    // swizzle key of this row: its row bits of lowest B stride (see plan_tc)
    const int rsw = ((row >> p.swz_row[0]) & 1) | (((row >> p.swz_row[1]) & 1) << 1) | (((row >> p.swz_row[2]) & 1) << 2);
    const int RS = p.rstages, XS = p.xstages;
    // raw row layout: 16-B chunk c of row n lives at chunk c ^ (n & (chunks-1))
    const int rb = 8 << TKC;            // raw bytes per row
    const int chunks = rb >> 4;
    // per-thread gather offsets are the same for every item: keep them in registers
    int64_t goff[PER];
    int32_t soff[PER];
    const bool vec = p.vecB != 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      // 16-B mode: the first PER/2 entries are element pairs (2q, 2q+1), q = ptid + i*256
      const int e = vec ? (i < PER / 2 ? 2 * (ptid + i * 256) : 0) : ptid + i * 256;
      goff[i] = tg[0][e & 63] + tg[1][e >> 6];
      soff[i] = ts[0][e & 63] ^ ts[1][e >> 6];
    }
    // copy cursor: the next item to gather (tile number ct of this CTA, K chunk cc); the tile
    // base offset is re-summed (lane j holds outer bit j's stride) only when the tile changes
    const int64_t o_s = lane < p.n_outer ? p.o_sB[lane] : 0;
    auto tile_base = [&](int64_t ct) {
      const int64_t t = (int64_t)blockIdx.x + ct * gridDim.x;
      int64_t tb = ((t >> lane) & 1) ? o_s : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(0xffffffffu, tb, o);
      return boff + tb;
    };
    int64_t ct = 0, cbase = tile_base(0);
    int cc = 0, wst = 0;  // wst = raw stage the next copy lands in
    auto copy = [&]() {
      unsigned char* raw = R + wst * p.rbytes;
      const float2* srcp = p.B + (cbase + kc_off[cc]);
      if (vec) {
#pragma unroll
        for (int i = 0; i < PER / 2; ++i) cp_async16(raw + soff[i], srcp + goff[i]);
      } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) cp_async8(raw + soff[i], srcp + goff[i]);
      }
      if (++wst == RS) wst = 0;
      if (++cc == p.n_kc) {
        cc = 0;
        ++ct;
        cbase = tile_base(ct);
      }
    };
    for (int q = 0; q < RS - 1; ++q) {
      if (q < items) copy();
      cp_async_commit();
    }
    int rst = 0, xs = 0;
    uint32_t xph = 0;
    for (int64_t it = 0; it < items; ++it) {
      // own copies of item it have landed (RS-1+it groups committed, RS-2 may stay pending)
      switch (RS) {
        case 2: cp_async_wait<0>(); break;
        case 3: cp_async_wait<1>(); break;
        case 4: cp_async_wait<2>(); break;
        case 5: cp_async_wait<3>(); break;
        default: cp_async_wait<4>(); break;
      }
      tc::bar_sync(1, 256);  // all producers' copies of item it landed; raw stage of it-1 is free
      if (it + RS - 1 < items) copy();
      cp_async_commit();
      tc::mbar_wait(&xempty[xs], xph ^ 1);  // TMEM X stage free
      tc::fence_after();
      const unsigned char* raw = R + rst * p.rbytes + row * rb;
      if (++rst == RS) rst = 0;
      float hi[NCOL], lo[NCOL];
#pragma unroll
      for (int j = 0; j < NCOL / 4; ++j) {
        const int cc = half * (NCOL / 4) + j;  // 16-B chunk of this row = 2 complex
        const float4 v = *reinterpret_cast<const float4*>(raw + ((cc ^ (rsw & (chunks - 1))) << 4));
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          hi[4 * j + q] = tc::tf32_rna(x[q]);
          lo[4 * j + q] = tc::tf32_lo(x[q], hi[4 * j + q]);
        }
      }
      const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
      const uint32_t col = xcol0 + (uint32_t)(xs * 2 * KPC + half * NCOL);
      tc::tmem_st<NCOL>(lane_addr + col, hi);
      tc::tmem_st<NCOL>(lane_addr + col + KPC, lo);
      tc::tmem_st_wait();
      tc::fence_before();
      tc::mbar_arrive(&xfull[xs]);
      if (++xs == XS) { xs = 0; xph ^= 1; }
    }
  } else if (warp == 12) {
    // ===================== MMA issuer =====================
    const bool leader = lane == 0;
    int64_t tt = 0;
    const int XS = p.xstages;
    int xs = 0, c = 0;
    uint32_t xph = 0;
    for (int64_t it = 0; it < items; ++it) {
      // accumulator b = tt mod acc_bufs (1, 2 or 4), its use count tt / acc_bufs -> phase
      const int lgb = p.acc_bufs >> 1;  // log2(acc_bufs) for 1, 2, 4
      const int b = (int)(tt & (p.acc_bufs - 1));
      const uint32_t tph = (uint32_t)((tt >> lgb) & 1);
      if (c == 0) tc::mbar_wait(&tempty[b], tph ^ 1);  // accumulator drained (first use passes)
      tc::mbar_wait(&xfull[xs], xph);
      tc::fence_after();
      if (leader) {
        const uint32_t d = tmem + (uint32_t)(b * p.acc_w);
        const uint32_t xh = tmem + xcol0 + (uint32_t)(xs * 2 * KPC), xl = xh + KPC;
        const uint32_t yh = tc::smem_u32(Yhi + c * p.yplane), yl = tc::smem_u32(Ylo + c * p.yplane);
        if (p.pairN) {
          // Xhi * [Yhi | Ylo] (N = 2 Np: the Ylo plane follows Yhi in shared memory) into columns
          // [0, 2 Np), Xlo * Yhi (N = Np) into [0, Np); the epilogue adds column j + Np to j
          const uint32_t idesc2 = (p.idesc & ~(0x3Fu << 17)) | ((uint32_t)((2 * p.Np) >> 3) << 17);
#pragma unroll
          for (int ks = 0; ks < KPC / 8; ++ks) {
            const uint64_t dyh = tc::sdesc(yh + ks * kstep, lbo, p.sbo_y, layout);
            tc::mma_tf32_ts(d, xh + ks * 8, dyh, idesc2, (c > 0 || ks > 0) ? 1u : 0u);
            tc::mma_tf32_ts(d, xl + ks * 8, dyh, p.idesc, 1u);  // after the N = 2 Np MMA: always accumulate
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < KPC / 8; ++ks) {
            const uint64_t dyh = tc::sdesc(yh + ks * kstep, lbo, p.sbo_y, layout);
            const uint64_t dyl = tc::sdesc(yl + ks * kstep, lbo, p.sbo_y, layout);
            tc::mma_tf32_ts(d, xh + ks * 8, dyh, p.idesc, (c > 0 || ks > 0) ? 1u : 0u);
            if (p.passes == 3) {
              tc::mma_tf32_ts(d, xh + ks * 8, dyl, p.idesc, 1u);
              tc::mma_tf32_ts(d, xl + ks * 8, dyh, p.idesc, 1u);
            }
          }
        }
        tc::mma_commit(&xempty[xs]);                     // TMEM X stage free once these finish
        if (c == p.n_kc - 1) tc::mma_commit(&tfull[b]);  // tile accumulated
      }
      __syncwarp();
      if (c == p.n_kc - 1) ++tt;
      if (++c == p.n_kc) c = 0;
      if (++xs == XS) { xs = 0; xph ^= 1; }
    }
  } else if (warp < 4) {
    // ===================== epilogue =====================
    const int row = warp * 32 + lane;
    const int nm = 1 << p.tm;
    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      // accumulator b = tt mod acc_bufs (1, 2 or 4), its use count tt / acc_bufs -> phase
      const int lgb = p.acc_bufs >> 1;  // log2(acc_bufs) for 1, 2, 4
      const int b = (int)(tt & (p.acc_bufs - 1));
      const uint32_t tph = (uint32_t)((tt >> lgb) & 1);
      tc::mbar_wait(&tfull[b], tph);
      tc::fence_after();
      const int64_t t = (int64_t)blockIdx.x + tt * gridDim.x;
      float2* out = p.C + (t << (7 + p.tm));
      for (int c0 = 0; c0 < p.Np; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * p.acc_w + c0), v);
        if (p.pairN) {  // + the Xhi * Ylo half
          float w[16];
          tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * p.acc_w + p.Np + c0), w);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int m = c0 / 2 + j;
          if (!p.mlow && m < nm) out[row + ((int64_t)m << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
        }
        if (p.mlow && c0 / 2 < nm) {  // [M][rows] layout: this row's m values are contiguous
          float4* o4 = reinterpret_cast<float4*>(out + ((int64_t)row << p.tm) + c0 / 2);
#pragma unroll
          for (int j = 0; j < 4; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
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
