// TMA probe for the K3 item load (B200, sm_100a).
//
// A K3 item is 128 rows x 2^tkc K of the big operand B; its 7+tkc address bits form <= 5 runs
// of consecutive strides.  The item is loaded as ONE cp.async.bulk.tensor box whose dims are
// those runs, and the item's base offset (outer tile bits + K chunk + slice) goes into the
// dim-0 coordinate: dim 0 is declared 2^32 elements long, i.e. its extent overlaps the higher
// dims' strides.  This probe checks (1) that the driver accepts such a map and the loaded box is
// bit-exact for random run structures and offsets, (2) the streaming rate of 16-KB boxes from
// one elected thread per CTA with an mbarrier ring (148 CTAs, HBM-resident source).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe scripts/tma_probe.cu && ./tma_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e = (x);                                                                        \
    if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } \
  } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn) { printf("no cuTensorMapEncodeTiled\n"); exit(1); }
  return (EncodeFn)fn;
}

struct Args {
  CUtensorMap map;
  int rank;
  int64_t n_items;
  int64_t off_stride;  // element offset between consecutive items (dim-0 coordinate)
  double* out;         // checksum sink
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) probe_kernel(const __grid_constant__ Args a, int64_t coord_base,
                                                        unsigned long long* dst) {
  // single-box correctness: load one box at coordinate coord_base into smem, copy it out
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16384) : "memory");
    const int c0 = (int)coord_base;
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            su32(sm)),
        "l"(&a.map), "r"(c0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(su32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) dst[i] = reinterpret_cast<unsigned long long*>(sm)[i];
}

// streaming: every CTA walks items blockIdx.x, +gridDim.x, ... with a ring of RS stages
template <int RS>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[RS], empty[RS];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < RS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 3;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t my = a.n_items > blockIdx.x ? (a.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {  // producer
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < my; ++it) {
      if (it >= RS)
        asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}" ::"r"(
                         su32(&empty[s])),
                     "r"(ph ^ 1)
                     : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384) : "memory");
      const int c0 = (int)((blockIdx.x + it * gridDim.x) * a.off_stride);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
              su32(sm + s * 16384)),
          "l"(&a.map), "r"(c0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(su32(&full[s]))
          : "memory");
      if (++s == RS) { s = 0; ph ^= 1; }
    }
  } else if (tid >= 32) {  // 3 consumer warps: touch the stage, release it
    int s = 0;
    uint32_t ph = 0;
    double acc = 0;
    for (int64_t it = 0; it < my; ++it) {
      asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}" ::"r"(
                       su32(&full[s])),
                   "r"(ph)
                   : "memory");
      const double* d = reinterpret_cast<const double*>(sm + s * 16384);
      for (int i = tid - 32; i < 2048; i += 96) acc += d[i];
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      if (++s == RS) { s = 0; ph ^= 1; }
    }
    if (acc == 12345.678) a.out[0] = acc;
  }
}

int main() {
  EncodeFn enc = get_encode();
  const int64_t N = int64_t(1) << 29;  // 4 GB of 8-B elements
  unsigned long long* src;
  CK(cudaMalloc(&src, N * 8));
  {
    std::vector<unsigned long long> h(1 << 24);
    for (int64_t base = 0; base < N; base += (1 << 24)) {
      for (int64_t i = 0; i < (1 << 24); ++i) h[i] = (unsigned long long)(base + i);
      CK(cudaMemcpy(src + base, h.data(), (1 << 24) * 8, cudaMemcpyHostToDevice));
    }
  }
  unsigned long long* dst;
  CK(cudaMalloc(&dst, 2048 * 8));
  double* sink;
  CK(cudaMalloc(&sink, 64));
  std::mt19937_64 rng(7);
  int bad = 0, tests = 0;
  // random item structures: 11 bits split into 1..5 runs of consecutive strides (each run <= 8
  // bits so it is one TMA dim), run strides increasing with gaps, lowest stride 1
  for (int t = 0; t < 200; ++t) {
    int nr = 1 + rng() % 5;
    std::vector<int> len(nr, 0);
    int left = 11;
    for (int i = 0; i < nr; ++i) len[i] = 1;
    left -= nr;
    while (left > 0) {
      int i = rng() % nr;
      if (len[i] < 8) { ++len[i]; --left; }
    }
    if (len[0] < 1) continue;
    std::vector<int64_t> rstr(nr);
    int64_t s = 1;
    for (int i = 0; i < nr; ++i) {
      rstr[i] = s;
      s <<= len[i];
      s <<= (i + 1 < nr) ? (rng() % 3) : 0;  // gap bits (outer bits of the tensor)
    }
    cuuint64_t gdim[5], gstr[4];
    cuuint32_t box[5], est[5];
    for (int i = 0; i < 5; ++i) {
      gdim[i] = i < nr ? (cuuint64_t)1 << len[i] : 1;
      box[i] = i < nr ? (cuuint32_t)1 << len[i] : 1;
      est[i] = 1;
    }
    gdim[0] = (cuuint64_t)1 << 32;  // overlapping dim 0: offsets go into its coordinate
    for (int i = 1; i < 5; ++i) gstr[i - 1] = (cuuint64_t)(i < nr ? rstr[i] : rstr[nr - 1] << len[nr - 1]) * 8;
    Args a{};
    CUresult r = enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, src, gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed (%d) for nr=%d\n", (int)r, nr);
      ++bad;
      continue;
    }
    const int64_t span = s;
    const int64_t base = (int64_t)(rng() % (uint64_t)(N - span - 1)) & ~int64_t(1);
    probe_kernel<<<1, 128, 16384 + 1024>>>(a, base, dst);
    CK(cudaGetLastError());
    std::vector<unsigned long long> h(2048);
    CK(cudaMemcpy(h.data(), dst, 2048 * 8, cudaMemcpyDeviceToHost));
    for (int e = 0; e < 2048; ++e) {
      int64_t off = base;
      int bit = 0;
      for (int i = 0; i < nr; ++i)
        for (int j = 0; j < len[i]; ++j, ++bit)
          if ((e >> bit) & 1) off += rstr[i] << j;
      if (h[e] != (unsigned long long)off) { ++bad; if (bad < 5) printf("mismatch t=%d e=%d got %llu want %lld\n", t, e, h[e], (long long)off); break; }
    }
    ++tests;
  }
  printf("correctness: %d structures, %d bad\n", tests, bad);
  // streaming rate: 16-KB items (a 2-dim box 256 x 8 over contiguous data), item i at dim-0
  // coordinate i * 2048, 148 CTAs, ring depth RS
  {
    Args a{};
    cuuint64_t gd[5] = {(cuuint64_t)1 << 32, 8, 1, 1, 1}, gs[4] = {256 * 8, 2048 * 8, 2048 * 8, 2048 * 8};
    cuuint32_t bx[5] = {256, 8, 1, 1, 1}, est[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, src, gd, gs, bx, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("stream map encode: %d\n", (int)r);
    a.n_items = N / 2048;
    a.off_stride = 2048;
    a.out = sink;
    for (int rs : {4, 6, 8, 10}) {
      void (*k)(Args) = rs == 4 ? stream_kernel<4> : rs == 6 ? stream_kernel<6> : rs == 8 ? stream_kernel<8> : stream_kernel<10>;
      CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, rs * 16384 + 1024));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k<<<148, 128, rs * 16384 + 1024>>>(a);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) k<<<148, 128, rs * 16384 + 1024>>>(a);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("stream RS=%d: %.1f GB/s (read only, 4 GB x 5)\n", rs, 5.0 * N * 8 / (ms / 1e3) / 1e9);
    }
  }
  CK(cudaDeviceSynchronize());
  return bad ? 1 : 0;
}
