// Shared helpers for librwb (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "rwb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "librwb is written for Blackwell (sm_100a); compile with -gencode arch=compute_100a,code=sm_100a"
#endif

namespace rwb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);

#define RWB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t err__ = (call);                          \
    if (err__ != cudaSuccess) return ::rwb::cuda_fail(err__, #call); \
  } while (0)

// RWB_DEBUG_SYNC=1 in the environment: synchronise after every checked launch
// so an asynchronous fault is reported at the launch that caused it.
bool debug_sync();
// for launches that may be captured into a graph: never synchronise
#define RWB_LAUNCH_CHECK_CAPTURE(what)                   \
  do {                                                   \
    cudaError_t err__ = cudaGetLastError();              \
    if (err__ != cudaSuccess) return ::rwb::cuda_fail(err__, what); \
  } while (0)
#define RWB_LAUNCH_CHECK(what)                           \
  do {                                                   \
    cudaError_t err__ = cudaGetLastError();              \
    if (err__ == cudaSuccess && ::rwb::debug_sync()) err__ = cudaDeviceSynchronize(); \
    if (err__ != cudaSuccess) return ::rwb::cuda_fail(err__, what); \
  } while (0)

// Dense level shape, padded to 3 dims (leading dims of size 1).
struct Shape3 {
  int nz, ny, nx;
  __host__ __device__ long long count() const { return (long long)nz * ny * nx; }
};

int shape_from(int32_t ndim, const int64_t* size, Shape3* out);

// Launch configurations (occupancy-derived grids, >48 KB shared-memory opt-ins) are properties of
// one device, so they are cached per device ordinal: a process that drives several GPUs sets the
// function attributes on each of them.  Concurrent first uses may compute a value twice (same result).
constexpr int kMaxDevices = 64;
using DeviceCache = std::atomic<int>[kMaxDevices];
// current device ordinal into *dev (RWB_ERR_UNSUPPORTED beyond kMaxDevices)
int device_slot(int* dev);

// process-wide kernel launch counter (rwb_kernel_launches)
void count_launches(long long n);

inline unsigned ceil_div_u(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// Edge weight of the Grady random walker: max(exp(-beta*(a-b)^2), w_min) as
// max(2^((d * c) * d), w_min) with c = -beta log2(e), one MUFU.EX2 (.ftz: an
// output below 2^-126 is flushed to 0, then clamped to w_min anyway).  Relative
// error ~|beta d^2| * 2^-22, i.e. a few 1e-6 for every weight above
// w_min = 1e-6, far inside the 1e-4 probability bar; it is symmetric in (a, b),
// so both endpoints of an edge compute identical bits.
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float edge_weight(float a, float b, float beta, float wmin) {
  const float c = -beta * 1.44269504088896341f;
  const float d = a - b;
  return fmaxf(ex2_ftz((d * c) * d), wmin);
}

}  // namespace rwb
