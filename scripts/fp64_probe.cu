// Microbenchmark: FP64 throughput on B200 through (a) DFMA on the CUDA cores and (b) the
// FP64 tensor-core MMA mma.sync.aligned.m8n8k4.row.col.f64 (DMMA), register-resident operands,
// many independent accumulators per warp, every SM busy.  Decides K4's design (SURVEY 8a a5:
// "c128 -> K4 DMMA").  Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_probe scripts/fp64_probe.cu && /tmp/fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dfma_probe(int reps, double* out) {
  double a[NACC];
  const double x = 1.0000001 + threadIdx.x * 1e-9, y = 0.9999999;
#pragma unroll
  for (int i = 0; i < NACC; ++i) a[i] = i;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) a[i] = fma(a[i], x, y);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma_probe(int reps, double* out) {
  double c[NACC][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
void run(const char* name, K kern, int blocks, int threads, int reps, double fma_per_thread_rep) {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(reps / 10, d);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(reps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * fma_per_thread_rep * reps * (double)blocks * threads;
  printf("%-28s blocks %5d threads %4d  %8.3f ms  %7.2f TFLOP/s  (%s)\n", name, blocks, threads, ms,
         flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {1, 2, 4}) {
    run("dfma nacc=8", dfma_probe<8>, sms * bps, 256, 20000, 8);
    run("dfma nacc=16", dfma_probe<16>, sms * bps, 256, 10000, 16);
    // one m8n8k4 = 256 FMA per warp = 8 FMA per thread
    run("dmma nacc=4", dmma_probe<4>, sms * bps, 256, 10000, 4 * 8);
    run("dmma nacc=8", dmma_probe<8>, sms * bps, 256, 5000, 8 * 8);
    run("dmma nacc=16", dmma_probe<16>, sms * bps, 256, 2500, 16 * 8);
  }
  run("dmma nacc=8 128thr", dmma_probe<8>, sms * 4, 128, 5000, 8 * 8);
  run("dmma nacc=8 512thr", dmma_probe<8>, sms * 2, 512, 5000, 8 * 8);
  return 0;
}
