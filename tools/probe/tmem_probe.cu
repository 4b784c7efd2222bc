// TMEM read throughput per SM (tcgen05.ld 32x32b) against shared-memory LDS.128 (diagnostics).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/tmem_probe tools/probe/tmem_probe.cu
#include <cstdio>
#include <cstdint>

#define LD32(base, off, v)                                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                       \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),  \
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),       \
                 "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),     \
                 "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),     \
                 "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                          \
               : "r"((base) + (off)))

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tmem_k(int n, unsigned long long* cyc, unsigned* sink) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * (512 / (WARPS / 4)));
  uint32_t v[32], acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    LD32(base, 0, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    acc ^= v[0] ^ v[31];
    LD32(base, 32, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    acc ^= v[1] ^ v[30];
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) lds_k(int n, unsigned long long* cyc, unsigned* sink) {
  __shared__ float4 buf[WARPS * 32 * 8];
  for (int i = threadIdx.x; i < WARPS * 32 * 8; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float acc = 0.f;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4 f = buf[(k * WARPS * 32 + threadIdx.x + i) & (WARPS * 32 * 8 - 1)];
      acc += f.x + f.w;
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 1.2345f) sink[0] = 1;
}

int main() {
  unsigned long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, 4096 * 8);
  cudaMalloc(&sink, 4);
  const int n = 4096;
  unsigned long long h[148];
  {
    tmem_k<8><<<148, 256>>>(n, cyc, sink);
    tmem_k<8><<<148, 256>>>(n, cyc, sink);
    cudaDeviceSynchronize();
    printf("tmem_k<8>: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)n * 2 * 32 * 4 * 256;
    printf("TMEM 32x32b.x32, 8 warps: %.1f cycles, %.1f B/cycle/SM\n", (double)h[0], bytes / h[0]);
  }
  {
    tmem_k<16><<<148, 512>>>(n, cyc, sink);
    cudaDeviceSynchronize();
    printf("tmem_k<16>: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)n * 2 * 32 * 4 * 512;
    printf("TMEM 32x32b.x32, 16 warps: %.1f cycles, %.1f B/cycle/SM\n", (double)h[0], bytes / h[0]);
  }
  {
    lds_k<8><<<148, 256>>>(n, cyc, sink);
    lds_k<8><<<148, 256>>>(n, cyc, sink);
    cudaDeviceSynchronize();
    printf("lds_k: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)n * 16 * 16 * 256;
    printf("LDS.128, 8 warps: %.1f cycles, %.1f B/cycle/SM\n", (double)h[0], bytes / h[0]);
  }
  return 0;
}
