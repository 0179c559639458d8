// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::tf32 (M=128) issued back to back by
// one thread, for several N, SS (A in shared memory) and TS (A in tensor memory) forms, with one
// accumulator and with independent accumulators.  Operand contents are irrelevant (zeros).
// Build/run on the GPU box:  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_probe
//                            scripts/mma_probe.cu && /tmp/mma_probe
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// mode 0: thread 0 issues (divergent warp), runtime accumulator rotation
// mode 1: the whole warp runs the loop, the MMA is predicated by elect.sync inside the asm
// mode 2: like 1 with a compile-time accumulator (no rotation), unrolled by 8
template <bool TS>
__global__ void probe(int n, int nacc, int reps, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t da = sdesc(su32(sm), 16, 1024, 2);
  const uint64_t db = sdesc(su32(sm + 32768), 16, 1024, 2);
  const uint32_t a_tmem = tm + 256;  // A operand columns for the TS form
  auto mma = [&](uint32_t d, uint32_t acc) {
    if (TS)
      asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                   "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc)
                   : "memory");
    else
      asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc)
                   : "memory");
  };
  auto mma1 = [&](uint32_t d, uint32_t acc) {  // plain, single thread
    if (TS)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                   "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc)
                   : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc)
                   : "memory");
  };
  if ((mode == 0 && threadIdx.x == 0) || (mode > 0 && warp == 0)) {
    unsigned long long t0 = 0, t1 = 0;
    for (int r = 0; r < 2; ++r) {  // r = 0 warm-up
      __syncwarp(mode == 0 ? 1u : 0xffffffffu);
      t0 = clock64();
      if (mode == 0) {
        for (int i = 0; i < reps; ++i) mma1(tm + (uint32_t)((i % nacc) * n), i >= nacc ? 1u : 0u);
      } else if (mode == 1) {
        for (int i = 0; i < reps; ++i) mma(tm + (uint32_t)((i % nacc) * n), i >= nacc ? 1u : 0u);
      } else {
        for (int i = 0; i < reps; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) mma(tm, (i + j) > 0 ? 1u : 0u);
        }
      }
      t1 = clock64();
      if (mode == 0 || (threadIdx.x & 31) == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}\n" ::"r"(
              su32(&bar)),
          "r"(r & 1)
          : "memory");
    }
    const unsigned long long t2 = clock64();
    if ((threadIdx.x & 31) == 0) {
      out[0] = t1 - t0;  // issue time of `reps` MMAs
      out[1] = t2 - t0;  // until all completed
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int reps = 96;
  printf("mode form  N  nacc  issue_cyc/mma  total_cyc/mma\n");
  for (int mode = 0; mode < 3; ++mode)
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {32, 64, 128, 256})
      for (int nacc : {1, 2}) {
        if (nacc * n > (ts ? 256 : 512)) continue;
        if (mode == 2 && nacc > 1) continue;
        if (ts) probe<true><<<1, 128, 65536>>>(n, nacc, reps, mode, d);
        else probe<false><<<1, 128, 65536>>>(n, nacc, reps, mode, d);
        unsigned long long h[2] = {0, 0};
        cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        printf("%d %s %4d %4d %10.1f %10.1f\n", mode, ts ? "TS" : "SS", n, nacc, (double)h[0] / reps, (double)h[1] / reps);
      }
  return 0;
}
