// TMA probe (B200, sm_100a): which forms of the K3 item load work, each variant in its own
// process (a faulting variant cannot take the others down):
//
//   v0  2-D tensor map, non-overlapping dims (256 x 8 contiguous), coordinate 0
//   v1  v0 + prefetch.tensormap on the __grid_constant__ map
//   v2  dim 0 declared 2^32 elements long (overlapping the dim-1 stride), coordinate 0
//   v3  v2 at a large dim-0 coordinate (the item base offset as the coordinate)
//   v4  v0 with the map passed through global memory instead of the kernel parameters
//   v5  non-tensor bulk copies (cp.async.bulk.shared::cluster.global), 8 x 2 KB per 16-KB item
//
// Each variant loads one 16-KB item and checks it bit-exactly, then (v0, v5) streams 4 GB of
// 16-KB items over 148 CTAs and reports GB/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe scripts/tma_probe.cu
//   for v in 0 1 2 3 4 5; do timeout 30 ./tma_probe $v; done
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                              \
  do {                                                                                                     \
    cudaError_t e = (x);                                                                                   \
    if (e != cudaSuccess) {                                                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                                     \
      fflush(stdout);                                                                                      \
      exit(1);                                                                                             \
    }                                                                                                      \
  } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Args {
  CUtensorMap map;
  const CUtensorMap* gmap;   // v4: the same map in global memory
  const unsigned long long* src;
  int variant;
  int64_t n_items;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(bar)),
               "r"(ph)
               : "memory");
}

__device__ __forceinline__ void issue(const Args& a, unsigned char* dst, int64_t base, uint64_t* bar) {
  if (a.variant == 5) {
    for (int j = 0; j < 8; ++j)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst + j * 2048)),
                   "l"(a.src + base + j * 256), "r"(2048), "r"(su32(bar))
                   : "memory");
    return;
  }
  const void* map = a.variant == 4 ? (const void*)a.gmap : (const void*)&a.map;
  const int c0 = (a.variant >= 2 && a.variant <= 3) ? (int)base : 0;
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(map), "r"(c0), "r"(0), "r"(su32(bar))
      : "memory");
}

__global__ void __launch_bounds__(128, 1) one_kernel(const __grid_constant__ Args a, int64_t base,
                                                      unsigned long long* dst) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (a.variant == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(&a.map) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16384) : "memory");
    issue(a, sm, base, &bar);
  }
  wait_parity(&bar, 0);
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) dst[i] = reinterpret_cast<unsigned long long*>(sm)[i];
}

template <int RS>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ Args a, double* sink) {
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
  if (tid == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int64_t it = 0; it < my; ++it) {
      if (it >= RS) wait_parity(&empty[s], ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(16384) : "memory");
      const int64_t base = (blockIdx.x + it * gridDim.x) * 2048;
      if (a.variant == 5) {
        issue(a, sm + s * 16384, base, &full[s]);
      } else {  // v0 streaming: the map covers the whole array as (256, n/256)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(sm + s * 16384)),
            "l"(&a.map), "r"(0), "r"((int)(base / 256)), "r"(su32(&full[s]))
            : "memory");
      }
      if (++s == RS) { s = 0; ph ^= 1; }
    }
  } else if (tid >= 32) {
    int s = 0;
    uint32_t ph = 0;
    double acc = 0;
    for (int64_t it = 0; it < my; ++it) {
      wait_parity(&full[s], ph);
      const double* d = reinterpret_cast<const double*>(sm + s * 16384);
      for (int i = tid - 32; i < 2048; i += 96) acc += d[i];
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      if (++s == RS) { s = 0; ph ^= 1; }
    }
    if (acc == 12345.678) sink[0] = acc;
  }
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fn;
  const int64_t N = int64_t(1) << 29;
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
  Args a{};
  a.variant = v;
  a.src = src;
  cuuint64_t gdim[2] = {256, 8}, gstr[1] = {256 * 8};
  cuuint32_t box[2] = {256, 8}, est[2] = {1, 1};
  if (v == 2 || v == 3) gdim[0] = (cuuint64_t)1 << 32;
  CUresult r = enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("v%d encode -> %d\n", v, (int)r);
  CUtensorMap* g;
  CK(cudaMalloc(&g, sizeof(CUtensorMap)));
  CK(cudaMemcpy(g, &a.map, sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  a.gmap = g;
  const int64_t base = v == 3 ? (int64_t(1) << 28) + 4096 : 0;
  CK(cudaFuncSetAttribute((const void*)one_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 1024));
  one_kernel<<<1, 128, 16384 + 1024>>>(a, base, dst);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> h(2048);
  CK(cudaMemcpy(h.data(), dst, 2048 * 8, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int e = 0; e < 2048; ++e) bad += h[e] != (unsigned long long)(base + e);
  printf("v%d one item: %s (%d bad)\n", v, bad ? "MISMATCH" : "ok", bad);
  if (v == 0 || v == 5) {
    if (v == 0) {
      cuuint64_t gd[2] = {256, (cuuint64_t)(N / 256)}, gs[1] = {256 * 8};
      enc(&a.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, gd, gs, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    a.n_items = N / 2048;
    double* sink;
    CK(cudaMalloc(&sink, 64));
    auto k = stream_kernel<8>;
    CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<148, 128, 8 * 16384 + 1024>>>(a, sink);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) k<<<148, 128, 8 * 16384 + 1024>>>(a, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("v%d stream: %.1f GB/s (read only, 4 GB x 5, 16-KB items, ring 8)\n", v, 5.0 * N * 8 / (ms / 1e3) / 1e9);
  }
  return bad ? 1 : 0;
}
