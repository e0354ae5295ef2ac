// microbench_fp64.cu -- B200 FP64 pipe probes used to pick the kernel design
// (DESIGN.md "Measured machine facts"): DFMA vs DMMA (mma.sync m8n8k4 f64)
// throughput and whether they overlap, and fp64 RED (atomicAdd) throughput.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1e-9);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a) {
  double d[8];
  for (int i = 0; i < 8; ++i) d[i] = 0;
  double b = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma(d[2 * i], d[2 * i + 1], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += d[i];
  if (s == 12345.678) out[0] = s;
}

// half the warps DFMA, half DMMA
__global__ void mixed_kernel(double* out, int iters, double a) {
  if ((threadIdx.x >> 5) & 1) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1e-9);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
  } else {
    double d[8];
    for (int i = 0; i < 8; ++i) d[i] = 0;
    double b = threadIdx.x * 1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dmma(d[2 * i], d[2 * i + 1], a, b);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += d[i];
    if (s == 12345.678) out[0] = s;
  }
}

__global__ void red_kernel(double* buf, long long n_mask, int per_thread, unsigned seed) {
  unsigned long long x = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + seed;
  for (int i = 0; i < per_thread; ++i) {
    x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
    long long idx = (long long)((x * 2685821657736338717ull) >> 20) & n_mask;
    atomicAdd(buf + idx, 1.0);
  }
}

// RED to addresses that are contiguous per warp (like a CSR row segment)
__global__ void red_coalesced_kernel(double* buf, long long n_mask, int per_thread) {
  long long base = (long long)(blockIdx.x * blockDim.x + threadIdx.x);
  for (int i = 0; i < per_thread; ++i) {
    long long idx = (base + (long long)i * gridDim.x * blockDim.x) & n_mask;
    atomicAdd(buf + idx, 1.0);
  }
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d L2 %d MB clock %d MHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20, clk / 1000);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep) printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(d, iters, 1.0000001); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl2 = 2.0 * 8 * 8 * 4 * 4 * iters * (double)blocks * threads / 32;
    if (rep) printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", fl2 / ms / 1e9, ms);
    cudaEventRecord(e0); mixed_kernel<<<blocks, threads>>>(d, iters, 1.0000001); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("mixed half DFMA/half DMMA: %.2f TFLOP/s (%.3f ms)\n", (fl + fl2) / 2 / ms / 1e9, ms);
  }
  for (long long mb : {32LL, 64LL, 2048LL}) {
    long long n = mb * 1024 * 1024 / 8;  // power of two
    double* buf; CK(cudaMalloc(&buf, n * 8)); CK(cudaMemset(buf, 0, n * 8));
    int per = 64;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); red_kernel<<<blocks * 4, 256>>>(buf, n - 1, per, 7 + rep); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double nops = (double)blocks * 4 * 256 * per;
      if (rep) printf("RED.F64 random, %lld MB buffer: %.1f G atom/s\n", mb, nops / ms / 1e6);
      cudaEventRecord(e0); red_coalesced_kernel<<<blocks * 4, 256>>>(buf, n - 1, per); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("RED.F64 coalesced, %lld MB buffer: %.1f G atom/s\n", mb, nops / ms / 1e6);
    }
    cudaFree(buf);
  }
  return 0;
}
