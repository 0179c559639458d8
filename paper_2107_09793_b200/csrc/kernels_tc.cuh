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

constexpr int kTcMaxTile = 12;    // 7 row bits + up to 5 K bits per chunk
constexpr int kTcMaxStages = 12;  // K3 ring stages (raw smem + TMEM lo)
constexpr int kTcLag = 3;
constexpr int kTrBegin = 200;  // first traced item (steady state)         // K3 ring stages between the item being gathered and the oldest in use

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
  int32_t xstages;                             // ring stages (raw shared stage + Kpc TMEM lo columns)
  int32_t rstages;                             // items gathered ahead (<= xstages)
  int32_t rbytes;                              // bytes of one raw stage (128 rows x 8*2^tkc)
  int32_t acc_bufs;                            // TMEM accumulator buffers (2: epilogue overlaps next tile)
  int32_t ycat;                                // 1: Y planes hold [Yhi | Ylo] along N (2*Np rows): per K step
                                               //   D[:, 0:2Np] += X*[Yhi|Ylo] and += Xlo*[Yhi|Ylo] (2 MMAs
                                               //   instead of 3); the epilogue adds the two column halves
  int32_t nw;                                  // accumulator width in TMEM columns (Np, or 2*Np with ycat)
  int32_t dbg;  // DEBUG (JETB200_K3_DBG): 1 skip stores, 2 skip loads, 4 skip split+STTM, 8 skip MMAs, 16 skip LDTM,
                //   32 one xfull/tempty arrival per warp, 64 no fence.proxy.async (timing only)
  unsigned long long* trace;  // DEBUG (JETB200_K3_TRACE): clock64 stamps of CTA 0, items [kTrBegin, +64)
  int64_t o_sB[kMaxOuter];                     // outer (row) bit j of B: stride
  int64_t o_kB[4];                             // chunk-index bit j of B: stride
  int64_t gX[kTcMaxTile];                      // B chunk-tile bit j (stride order): global stride
  int32_t sX[kTcMaxTile];                      //   ... and its byte offset in the raw stage (XOR-combined)
  int32_t wpos[3];                             // positions (in gX order) of row bits 5, 6 and K bit tkc-1:
                                               //   the bits that select a producer warp's share
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
// The MMA / commit wrappers are executed by the WHOLE issuing warp with warp-uniform operands;
// elect.sync inside the asm picks the one lane that issues.  (Issuing from a divergent
// single-lane branch costs ~150 cycles per tcgen05.mma; warp-uniform issue ~20-60, i.e. the
// tensor core's own rate -- measured by scripts/mma_probe.cu.)
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
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
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// All MMAs of one item in ONE asm block with one elect.sync: every operand is moved to the
// uniform datapath before the first tcgen05.mma, so the MMAs issue back to back (separate asm
// statements interleave an R2UR/ELECT round trip with every MMA, ~100 cycles each).
// K3 ycat: per K step s, D += X_s * Ycat_s (A from shared memory) and D += Xlo_s * Ycat_s (A from
// tensor memory); `acc` enables accumulation for the first MMA (all later ones accumulate).
template <int KS>
__device__ __forceinline__ void mma_item_ycat(uint32_t d, uint32_t idesc, uint32_t acc, const uint64_t (&dx)[KS],
                                              const uint64_t (&dy)[KS], const uint32_t (&xl)[KS]);
#define JT_MMA_SS(D, A, B, P) "@e tcgen05.mma.cta_group::1.kind::tf32 [" D "], " A ", " B ", %1, " P ";\n\t"
#define JT_MMA_TS(D, A, B) "@e tcgen05.mma.cta_group::1.kind::tf32 [" D "], [" A "], " B ", %1, 1;\n\t"
template <>
__device__ __forceinline__ void mma_item_ycat<1>(uint32_t d, uint32_t idesc, uint32_t acc, const uint64_t (&dx)[1],
                                                 const uint64_t (&dy)[1], const uint32_t (&xl)[1]) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %2, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      JT_MMA_SS("%0", "%3", "%4", "p") JT_MMA_TS("%0", "%5", "%4") "}\n" ::"r"(d),
      "r"(idesc), "r"(acc), "l"(dx[0]), "l"(dy[0]), "r"(xl[0])
      : "memory");
}
template <>
__device__ __forceinline__ void mma_item_ycat<2>(uint32_t d, uint32_t idesc, uint32_t acc, const uint64_t (&dx)[2],
                                                 const uint64_t (&dy)[2], const uint32_t (&xl)[2]) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %2, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      JT_MMA_SS("%0", "%3", "%5", "p") JT_MMA_TS("%0", "%7", "%5")
      JT_MMA_SS("%0", "%4", "%6", "1") JT_MMA_TS("%0", "%8", "%6") "}\n" ::"r"(d),
      "r"(idesc), "r"(acc), "l"(dx[0]), "l"(dx[1]), "l"(dy[0]), "l"(dy[1]), "r"(xl[0]), "r"(xl[1])
      : "memory");
}
template <>
__device__ __forceinline__ void mma_item_ycat<4>(uint32_t d, uint32_t idesc, uint32_t acc, const uint64_t (&dx)[4],
                                                 const uint64_t (&dy)[4], const uint32_t (&xl)[4]) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %2, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      JT_MMA_SS("%0", "%3", "%7", "p") JT_MMA_TS("%0", "%11", "%7")
      JT_MMA_SS("%0", "%4", "%8", "1") JT_MMA_TS("%0", "%12", "%8")
      JT_MMA_SS("%0", "%5", "%9", "1") JT_MMA_TS("%0", "%13", "%9")
      JT_MMA_SS("%0", "%6", "%10", "1") JT_MMA_TS("%0", "%14", "%10") "}\n" ::"r"(d),
      "r"(idesc), "r"(acc), "l"(dx[0]), "l"(dx[1]), "l"(dx[2]), "l"(dx[3]), "l"(dy[0]), "l"(dy[1]), "l"(dy[2]),
      "l"(dy[3]), "r"(xl[0]), "r"(xl[1]), "r"(xl[2]), "r"(xl[3])
      : "memory");
}
// Classic 3xTF32 per K step (wide N): D += X*Yhi + X*Ylo + Xlo*Yhi, one K step per asm block.
__device__ __forceinline__ void mma_step3(uint32_t d, uint32_t idesc, uint32_t acc, uint64_t dx, uint64_t dyh,
                                          uint64_t dyl, uint32_t xl) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %2, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      JT_MMA_SS("%0", "%3", "%4", "p") JT_MMA_SS("%0", "%3", "%5", "1") JT_MMA_TS("%0", "%6", "%4") "}\n" ::"r"(d),
      "r"(idesc), "r"(acc), "l"(dx), "l"(dyh), "l"(dyl), "r"(xl)
      : "memory");
}
#undef JT_MMA_SS
#undef JT_MMA_TS
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
// 3xTF32 split by truncation: hi = x with the low 13 mantissa bits cleared (exactly a TF32
// value, so the MMA reads it exactly whatever its own rounding), lo = x - hi (exact in fp32);
// lo is then read at TF32 precision (relative error 2^-11 of lo, ~2^-22 of x).
// Round-to-nearest TF32 (low 13 mantissa bits zero).  The 3xTF32 split is hi = rna(x),
// lo = rna(x - hi): both are exact TF32 inputs, so |x - hi - lo| <= 2^-22 |x| and the MMA's
// own handling of the low mantissa bits never enters (a truncated split loses ~4x more).
// (Integer form of cvt.rna.tf32.f32, which ptxas expands with an Inf/NaN branch; the
// operands here are finite.)
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
// x - trunc_tf32(x): exact in fp32; the tensor core reads x itself as trunc_tf32(x) (it ignores
// the low 13 mantissa bits), so hi + lo = x exactly and lo is then read at TF32 precision
// (relative error 2^-10 of lo <= 2^-20 of x).
__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

}  // namespace tc

// Byte offset of A-operand element (row r, tf32 column kk) inside one X buffer / Y plane.
__device__ __forceinline__ int tc_off(int r, int kk, int sbo, int swz) {
  if (swz) return (r & 7) * 128 + (r >> 3) * 1024 + ((((kk >> 2) ^ (r & 7)) & 7) << 4) + (kk & 3) * 4;
  return (r & 7) * 16 + (r >> 3) * sbo + (kk >> 2) * 128 + (kk & 3) * 4;
}

// Warp-specialised K3 (v12): the raw landing stage IS the MMA's A operand for the hi part.
//   warps 4-11 producers: each warp cp.async-gathers its own share of every item (rows
//              quarter*32..+31, chunk half `half`) into a ring stage laid out as the UMMA K-major
//              swizzled operand (SW128/64/32 for 16/8/4 complex per K chunk); after its own
//              copies landed (cp.async.wait + __syncwarp) each thread reads its row half, forms
//              lo = x - trunc_tf32(x) and writes lo to the stage's TMEM columns (tcgen05.st)
//   warp 12    MMA issuer, per 8-TF32 K step: D += X*Yhi, D += X*Ylo with A = X straight from the
//              raw stage (the tensor core reads the top 19 bits of each fp32, i.e. hi =
//              trunc_tf32(x)), then D += Xlo*Yhi with A = lo from TMEM (the TS form); 3xTF32
//   warps 0-3  epilogue: TMEM accumulator -> registers -> 256-B coalesced global stores
// Barriers: xfull/xempty per ring stage (raw smem + TMEM lo), tfull/tempty per accumulator.
// Ring: p.xstages stages, p.rstages items gathered ahead (<= xstages).
// TKC = K bits per chunk (row of a stage = 2*2^TKC TF32).
template <int TKC>
__global__ void __launch_bounds__(416, 1) gett_tc_kernel(const __grid_constant__ TcArgs p) {
  constexpr int PER = (128 << TKC) / 256;  // B elements each producer thread copies per item
  constexpr int NCOL = 1 << TKC;           // lo fp32 columns each producer thread writes (half a row)
  constexpr int KPC = 2 << TKC;            // TF32 columns of one X row
  constexpr int RB = 8 << TKC;             // raw bytes per row
  constexpr int CHUNKS = RB >> 4;          // 16-B chunks per row
  constexpr int SWS = 4 - TKC;             // swizzle: chunk ^= (row >> SWS) & (CHUNKS-1)
  constexpr uint32_t ALAYOUT = TKC == 4 ? 2u : (TKC == 3 ? 4u : 6u);  // SW128 / SW64 / SW32
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int64_t tg[2][64];
  __shared__ int32_t ts[2][64];
  __shared__ int64_t kc_off[16];  // B byte offset of K chunk c (n_kc <= 16)
  __shared__ __align__(8) uint64_t xfull[kTcMaxStages], xempty[kTcMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto kwait = [&](uint64_t* bar, uint32_t ph) { tc::mbar_wait(bar, ph); };
  // DEBUG trace: role r (0/1 producer warps 4/11, 2 MMA warp, 3 epilogue warp 0), item i, slot k
  auto tr = [&](int r, int64_t i, int k) {
    if (p.trace && blockIdx.x == 0 && lane == 0 && i >= kTrBegin && i < kTrBegin + 64)
      p.trace[((r * 64) + (i - kTrBegin)) * 8 + k] = clock64();
  };
  if (tid < 16) {
    int64_t o = 0;
    for (int j = 0; j < p.K - p.tkc; ++j) if ((tid >> j) & 1) o += p.o_kB[j];
    kc_off[tid] = o * 8;
  }
  // 1024-B aligned carve: Y planes [hi c=0..n_kc-1 | lo ...], then the ring stages (1024-aligned)
  unsigned char* base = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* Yhi = base;
  unsigned char* Ylo = Yhi + p.n_kc * p.yplane;
  unsigned char* R = base + (((p.ycat ? 1 : 2) * p.n_kc * p.yplane + 1023) & ~1023);
  for (int i = tid; i < 64; i += blockDim.x) {
    for (int h = 0; h < 2; ++h) {
      int64_t g = 0;
      int32_t s = 0;
      for (int b = 0; b < 6; ++b)
        if ((i >> b) & 1) {
          const int bi = 6 * h + b;
          if (bi < p.nX) { g += p.gX[bi]; s ^= p.sX[bi]; }
        }
      tg[h][i] = g * 8;
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
    for (int i = 0; i < p.xstages; ++i) {
      tc::mbar_init(&xfull[i], (p.dbg & 32) ? 8 : 256);
      tc::mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], (p.dbg & 32) ? 4 : 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // the operands are written by the previous kernels of the sequence
  pdl_launch_dependents();
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
          const float x = vals[s][t];
          const float hi = tc::tf32_rna(x);
          if (p.ycat) {  // one plane per chunk: rows [0, Np) = Yhi, [Np, 2Np) = Ylo
            *reinterpret_cast<float*>(Yhi + c * p.yplane + tc_off(2 * m + s, 2 * kl + t, p.sbo_y, p.swz)) = hi;
            *reinterpret_cast<float*>(Yhi + c * p.yplane + tc_off(p.Np + 2 * m + s, 2 * kl + t, p.sbo_y, p.swz)) =
                tc::tf32_rna(x - hi);
          } else {
            const int byte = c * p.yplane + tc_off(2 * m + s, 2 * kl + t, p.sbo_y, p.swz);
            *reinterpret_cast<float*>(Yhi + byte) = hi;
            *reinterpret_cast<float*>(Ylo + byte) = tc::tf32_rna(x - hi);
          }
        }
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base_sh;
  const uint32_t xcol0 = (uint32_t)(p.acc_bufs * p.nw);  // first TMEM column of the lo stages
  const int64_t my_tiles = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles * p.n_kc;
  const uint32_t layout = p.swz ? 2u : 0u;
  const uint32_t lbo = p.swz ? 16u : 128u;
  const uint32_t kstep = p.swz ? 32u : 256u;  // Y descriptor advance per 8-TF32 K step

  if (warp >= 4 && warp < 12) {
    // ===================== producers =====================
    const int64_t boff = slice_off(p.sv, false) * 8;
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;  // this thread's TMEM lane (row n of the tile)
    const int S = p.xstages, D = p.rstages;
    const char* Bb = reinterpret_cast<const char*>(p.B);
    // Each producer warp gathers exactly the elements it converts later, so a warp only waits
    // for its own copies (cp.async.wait + __syncwarp) and never synchronises with the other
    // producer warps.  Its share is the tile with the three warp-select bits fixed; the other
    // bits, lowest strides first, index lane + 32 i (coalesced).  Byte offsets, in registers.
    int64_t goff[PER];
    int32_t soff[PER];
    {
      const int wbits[3] = {quarter & 1, quarter >> 1, half};
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        int sub = lane + i * 32, e = 0, sb = 0;
        for (int j = 0; j < p.nX; ++j) {
          int bit;
          if (j == p.wpos[0]) bit = wbits[0];
          else if (j == p.wpos[1]) bit = wbits[1];
          else if (j == p.wpos[2]) bit = wbits[2];
          else bit = (sub >> sb++) & 1;
          e |= bit << j;
        }
        goff[i] = tg[0][e & 63] + tg[1][e >> 6];
        soff[i] = ts[0][e & 63] ^ ts[1][e >> 6];
      }
    }
    // copy cursor: the next item to gather (tile number ct of this CTA, K chunk cc); the tile
    // base offset is re-summed (lane j holds outer bit j's stride) only when the tile changes
    const int64_t o_s = lane < p.n_outer ? p.o_sB[lane] * 8 : 0;
    auto tile_base = [&](int64_t ct) {
      const int64_t t = (int64_t)blockIdx.x + ct * gridDim.x;
      int64_t tb = ((t >> lane) & 1) ? o_s : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb += __shfl_xor_sync(0xffffffffu, tb, o);
      return boff + tb;
    };
    int64_t ct = 0, cbase = tile_base(0);
    int cc = 0, wst = 0;  // wst = ring stage the next copy lands in
    uint32_t wph = 0;     // use parity of that stage
    int64_t trit = -1;
    const int trr = warp == 4 ? 0 : (warp == 11 ? 1 : -1);
    auto copy = [&]() {
      kwait(&xempty[wst], wph ^ 1);  // the stage's previous item is consumed by the MMAs
      if (trr >= 0 && trit >= 0) tr(trr, trit, 6);
      unsigned char* raw = R + wst * p.rbytes;
      const char* src = Bb + (cbase + kc_off[cc]);
      if (!(p.dbg & 2)) {
#pragma unroll
        for (int i = 0; i < PER; ++i) cp_async8(raw + soff[i], src + goff[i]);
      }
      if (++wst == S) { wst = 0; wph ^= 1; }
      if (++cc == p.n_kc) {
        cc = 0;
        ++ct;
        cbase = tile_base(ct);
      }
    };
    for (int q = 0; q < D; ++q) {
      if (q < items) copy();
      cp_async_commit();
    }
    int rst = 0;  // ring stage of item it
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
    const int sw = (row >> SWS) & (CHUNKS - 1);
    for (int64_t it = 0; it < items; ++it) {
      if (trr >= 0) tr(trr, it, 0);
      cp_async_wait_dyn(D - 1);  // own copies of item it landed (D groups ahead were committed)
      __syncwarp();              // ... and every lane's copies of this warp's share
      if (trr >= 0) tr(trr, it, 1);
      if (!(p.dbg & 4)) {
        const unsigned char* raw = R + rst * p.rbytes + row * RB;
        float lo[NCOL];
#pragma unroll
        for (int j = 0; j < NCOL / 4; ++j) {
          const int ch = half * (NCOL / 4) + j;  // 16-B chunk of this row = 2 complex
          const float4 v = *reinterpret_cast<const float4*>(raw + ((ch ^ sw) << 4));
          lo[4 * j + 0] = tc::tf32_lo(v.x);
          lo[4 * j + 1] = tc::tf32_lo(v.y);
          lo[4 * j + 2] = tc::tf32_lo(v.z);
          lo[4 * j + 3] = tc::tf32_lo(v.w);
        }
        if (trr >= 0) tr(trr, it, 2);
        tc::tmem_st<NCOL>(lane_addr + xcol0 + (uint32_t)(rst * KPC + half * NCOL), lo);
        tc::tmem_st_wait();
      }
      if (trr >= 0) tr(trr, it, 3);
      if (!(p.dbg & 64)) tc::fence_proxy_async();  // this thread's cp.async data -> visible to the MMA (async proxy)
      tc::fence_before();
      if (p.dbg & 32) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&xfull[rst]);
      } else {
        tc::mbar_arrive(&xfull[rst]);
      }
      if (trr >= 0) tr(trr, it, 4);
      if (++rst == S) rst = 0;
      trit = it;
      if (it + D < items) copy();
      cp_async_commit();
      if (trr >= 0) tr(trr, it, 5);
    }
  } else if (warp == 12) {
    // ===================== MMA issuer =====================
    int64_t tt = 0;
    const int S = p.xstages;
    int xs = 0, c = 0;
    uint32_t xph = 0;
    for (int64_t it = 0; it < items; ++it) {
      const int b = p.acc_bufs == 2 ? (int)(tt & 1) : 0;
      const uint32_t tph = p.acc_bufs == 2 ? (uint32_t)((tt >> 1) & 1) : (uint32_t)(tt & 1);
      tr(2, it, 0);
      if (c == 0) kwait(&tempty[b], tph ^ 1);  // accumulator drained (first use passes)
      tr(2, it, 1);
      kwait(&xfull[xs], xph);
      tr(2, it, 2);
      tc::fence_after();
      if (!(p.dbg & 8)) {  // whole warp: the wrappers elect the issuing lane
        const uint32_t d = tmem + (uint32_t)(b * p.nw);
        const uint32_t xl = tmem + xcol0 + (uint32_t)(xs * KPC);
        const uint32_t xr = tc::smem_u32(R + xs * p.rbytes);
        const uint32_t yh = tc::smem_u32(Yhi + c * p.yplane), yl = tc::smem_u32(Ylo + c * p.yplane);
        constexpr int KS = KPC / 8;
        const uint32_t acc = c > 0 ? 1u : 0u;
        uint64_t dx[KS], dy[KS];
        uint32_t xls[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          dx[ks] = tc::sdesc(xr + ks * 32, 16, 8 * RB, ALAYOUT);
          dy[ks] = tc::sdesc(yh + ks * kstep, lbo, p.sbo_y, layout);
          xls[ks] = xl + ks * 8;
        }
        if (p.ycat) {  // D[:, 0:2Np] += (hi + lo) * [Yhi|Ylo]
          tc::mma_item_ycat<KS>(d, p.idesc, acc, dx, dy, xls);
        } else {  // D += hi*Yhi + hi*Ylo + lo*Yhi
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
            tc::mma_step3(d, p.idesc, (c > 0 || ks > 0) ? 1u : 0u, dx[ks], dy[ks],
                          tc::sdesc(yl + ks * kstep, lbo, p.sbo_y, layout), xls[ks]);
        }
        tc::mma_commit(&xempty[xs]);                     // ring stage free once these finish
        if (c == p.n_kc - 1) tc::mma_commit(&tfull[b]);  // tile accumulated
      } else if (lane == 0) {
        tc::mbar_arrive(&xempty[xs]);
        if (c == p.n_kc - 1) tc::mbar_arrive(&tfull[b]);
      }
      __syncwarp();
      tr(2, it, 3);
      if (c == p.n_kc - 1) ++tt;
      if (++c == p.n_kc) c = 0;
      if (++xs == S) { xs = 0; xph ^= 1; }
    }
  } else if (warp < 4) {
    // ===================== epilogue =====================
    const int row = warp * 32 + lane;
    const int nm = 1 << p.tm;
    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      const int b = p.acc_bufs == 2 ? (int)(tt & 1) : 0;
      const uint32_t tph = p.acc_bufs == 2 ? (uint32_t)((tt >> 1) & 1) : (uint32_t)(tt & 1);
      if (warp == 0) tr(3, tt, 0);
      kwait(&tfull[b], tph);
      if (warp == 0) tr(3, tt, 1);
      tc::fence_after();
      const int64_t t = (int64_t)blockIdx.x + tt * gridDim.x;
      float2* out = p.C + (t << (7 + p.tm));
      for (int c0 = 0; c0 < p.Np; c0 += 16) {
        float v[16];
        if (p.dbg & 16) {
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
        } else {
          const uint32_t a0 = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * p.nw + c0);
          tc::tmem_ld16(a0, v);
          if (p.ycat) {  // (hi + lo) x Yhi  +  (hi + lo) x Ylo
            float w[16];
            tc::tmem_ld16(a0 + (uint32_t)p.Np, w);
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) v[jj] += w[jj];
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int m = c0 / 2 + j;
          if (m < nm && !(p.dbg & 1)) out[row + ((int64_t)m << 7)] = make_float2(v[2 * j], v[2 * j + 1]);
        }
      }
      if (warp == 0) tr(3, tt, 2);
      tc::fence_before();
      if (p.dbg & 32) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[b]);
      } else {
        tc::mbar_arrive(&tempty[b]);
      }
      if (warp == 0) tr(3, tt, 3);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

}  // namespace jt
