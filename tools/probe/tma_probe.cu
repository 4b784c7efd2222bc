// Bisect TMA / mbarrier usage of the fused setup kernel (diagnostics).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

struct Maps { CUtensorMap I; };

__global__ void probe(const __grid_constant__ Maps m, int mode, float* out, const CUtensorMap* gmap) {
  extern __shared__ __align__(128) unsigned char raw[];
  float* tile = reinterpret_cast<float*>(raw);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + 8192);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    if (mode >= 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (mode >= 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (mode >= 3) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(40 * 34 * 4) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"((uint32_t)__cvta_generic_to_shared(tile)),
          "l"(mode == 5 ? gmap : &m.I), "r"(mode == 6 || mode == 8 ? 0 : (mode == 7 ? -4 : (mode == 9 ? -16 : -1))), "r"(mode == 6 ? 0 : -1), "r"(mode == 4 ? -1 : 0), "r"(b)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra.uni WAIT_%=;\n\t}" ::"r"(b),
        "r"(0)
        : "memory");
    out[threadIdx.x] = tile[threadIdx.x + 41];
  }
}

int main() {
  const int nx = 16, ny = 18, nz = 20;
  float* d;
  cudaMalloc(&d, nx * ny * nz * 4);
  float* h = new float[nx * ny * nz];
  for (int i = 0; i < nx * ny * nz; ++i) h[i] = (float)i;
  cudaMemcpy(d, h, nx * ny * nz * 4, cudaMemcpyHostToDevice);
  float* out;
  cudaMalloc(&out, 1024 * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Maps m;
  memset(&m, 0, sizeof(m));
  const cuuint64_t dims[3] = {nx, ny, nz};
  const cuuint64_t strides[2] = {nx * 4, nx * ny * 4};
  const cuuint32_t box[3] = {40, 34, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&m.I, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &m.I, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  int modes[] = {6, 8, 7, 9, 3};
  for (int mode : modes) {
    probe<<<1, 128, 16384>>>(m, mode, out, gm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    float o[4];
    cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
    printf("  out %g %g %g %g\n", o[0], o[1], o[2], o[3]);
  }
  return 0;
}
