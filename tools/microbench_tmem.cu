// microbench_tmem.cu -- can TMEM serve as per-thread private scratch for a
// non-MMA kernel?  Each thread of a
// 128-thread warpgroup owns one TMEM lane (32x32b shape: warp w <-> lanes
// 32w..32w+31); we time tcgen05.st / tcgen05.ld round trips of N columns per
// thread against the same volume through shared memory, with 1 and 2 CTAs per
// SM, and the DFMA-chain latency (fixed-latency pipe) for the design notes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tmem tools/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NCOL>
__global__ void __launch_bounds__(128, 2) tmem_kernel(unsigned long long* cyc, double* out, int iters) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr_s)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + (uint32_t(warp * 32) << 16);
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCOL; c += 32) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(base + c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                   "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
                   "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < NCOL; c += 32) {
      uint32_t q[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                     "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]),
                     "=r"(q[16]), "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]),
                     "=r"(q[24]), "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
                   : "r"(base + c) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] += q[i];
    }
  }
  unsigned long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr_s), "n"(256));
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += r[i];
  if (s == 0x12345678u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the same volume through shared memory, SoA [col][thread] (conflict-free)
template <int NCOL>
__global__ void __launch_bounds__(128, 2) smem_kernel(unsigned long long* cyc, double* out, int iters) {
  extern __shared__ uint32_t sm[];
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 7 + i;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < NCOL; c += 32)
#pragma unroll
      for (int i = 0; i < 32; i += 2)
        *reinterpret_cast<uint2*>(&sm[((c + i) / 2) * 256 + 2 * threadIdx.x]) = make_uint2(r[i], r[i + 1]);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NCOL; c += 32)
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        uint32_t qx, qy;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(qx), "=r"(qy)
                     : "r"(smem_u32(&sm[((c + i) / 2) * 256 + 2 * threadIdx.x])));
        r[i] += qx; r[i + 1] += qy;
      }
    __syncwarp();
  }
  unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += r[i];
  if (s == 0x12345678u) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// dependent DFMA chain: latency of the fixed-latency FP64 pipe
__global__ void dfma_latency(unsigned long long* cyc, double* out, int iters) {
  double x = threadIdx.x * 1e-3;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 64; ++i) x = fma(x, 0.999, 1e-9);
  }
  unsigned long long t1 = clock64();
  if (x == 12345.678) out[0] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* d_cyc;
  double* d_out;
  const int maxb = 296;
  CK(cudaMalloc(&d_cyc, maxb * sizeof(unsigned long long)));
  CK(cudaMalloc(&d_out, 8));
  unsigned long long h[maxb];
  const int iters = 2000;
  auto report = [&](const char* name, int blocks, double bytes_per_cta_iter, double secs) {
    CK(cudaMemcpy(h, d_cyc, blocks * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    double per_sm = bytes_per_cta_iter * iters * (blocks / 148.0);
    printf("%-34s blocks %3d: %8.1f cycles/iter (max CTA), %7.1f B/clk/SM (clock64), %7.2f TB/s chip (events)\n",
           name, blocks, mx / iters, per_sm / mx, bytes_per_cta_iter * iters * blocks / secs / 1e12);
    return 0;
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocks : {148, 296}) {
    float ms;
    tmem_kernel<128><<<blocks, 128>>>(d_cyc, d_out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    tmem_kernel<128><<<blocks, 128>>>(d_cyc, d_out, iters);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
    report("tmem st+ld 128 cols/thread", blocks, 2.0 * 128 * 4 * 128, ms / 1e3);
    CK(cudaFuncSetAttribute(smem_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    smem_kernel<128><<<blocks, 128, 64 * 1024>>>(d_cyc, d_out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    smem_kernel<128><<<blocks, 128, 64 * 1024>>>(d_cyc, d_out, iters);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
    report("smem st+ld 128 words/thread", blocks, 2.0 * 128 * 4 * 128, ms / 1e3);
  }
  dfma_latency<<<1, 32>>>(d_cyc, d_out, 100);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, d_cyc, 8, cudaMemcpyDeviceToHost));
  printf("DFMA dependent-chain latency: %.2f cycles\n", double(h[0]) / (100 * 64));
  return 0;
}
