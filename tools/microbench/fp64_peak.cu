// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) vs DMMA.8x8x4
// (fp64 tensor cores, mma.sync m8n8k4).  Reports TFLOP/s (FMA = 2 flop) over a
// long kernel so the clock settles; run with clocks sampled beside it.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

// half the warps of a CTA run the DFMA loop, half the DMMA loop: do the two
// fp64 paths share one pipe (total ~= either alone) or add up?
template <int ILP>
__global__ void mixed_loop(double* out, int iters_f, int iters_m, double a, double b) {
  if ((threadIdx.x / 32) & 1) {
    double aa = threadIdx.x * 1e-3, bb = 1.0 - threadIdx.x * 1e-4;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters_m; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(aa), "d"(bb));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
  } else {
    double acc[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
  }
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0, smemOptin = 0, clk = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"smem_per_sm\": %zu, \"clock_khz\": %d}\n",
         p.name, p.multiProcessorCount, l2, smemOptin, p.sharedMemPerMultiprocessor, clk);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      int iters = 20000;
      dfma_loop<8><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      dfma_loop<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 8 * (double)iters * blocks * tpb;
      printf("{\"kernel\": \"dfma\", \"tpb\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", tpb, ms, flop / ms / 1e9);
    }
    for (int tpb : {128, 256, 512}) {
      int blocks = sms * (1024 / tpb);
      int iters = 5000;
      dmma_loop<4><<<blocks, tpb>>>(out, 100);
      CK(cudaEventRecord(e0));
      dmma_loop<4><<<blocks, tpb>>>(out, iters);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 256 * 4 * (double)iters * blocks * (tpb / 32);
      printf("{\"kernel\": \"dmma_m8n8k4\", \"tpb\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", tpb, ms, flop / ms / 1e9);
    }
  }
  // mixed: per warp pair, DFMA work 2*16*iters_f*32 flop, DMMA 2*256*4*iters_m flop
  for (int rep = 0; rep < 2; ++rep) {
    for (int ratio : {1, 2, 4}) {
      int tpb = 512, blocks = sms * 2;
      int iters_m = 4000, iters_f = 4000 * ratio;
      mixed_loop<16><<<blocks, tpb>>>(out, 100, 100, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      mixed_loop<16><<<blocks, tpb>>>(out, iters_f, iters_m, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double wp = (double)blocks * tpb / 64;  // warp pairs
      double ff = 2.0 * 16 * iters_f * 32 * wp, fm = 2.0 * 256 * 4 * (double)iters_m * wp;
      printf("{\"kernel\": \"mixed\", \"ratio\": %d, \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
             ratio, ms, ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9);
    }
    for (int tpb : {256, 512}) {
      int blocks = sms * (2048 / tpb);
      int iters = 10000;
      dfma_loop<16><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-9);
      CK(cudaEventRecord(e0));
      dfma_loop<16><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = 2.0 * 16 * (double)iters * blocks * tpb;
      printf("{\"kernel\": \"dfma_ilp16\", \"tpb\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", tpb, ms, flop / ms / 1e9);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
