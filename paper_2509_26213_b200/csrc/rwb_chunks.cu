// Chunk payloads <-> dense level tensors, for streaming chunked tensor files
// (the reference's PLCT format, pkg/src/chunkcast/tensorfile.py:1-13) through
// the GPU, and the plain factor-2 mean downsampling of build_lod(smooth=False).
//
// A chunk payload is the full chunk box, row-major, last dimension fastest,
// lanes innermost (ElementType.payload_shape, model.py:78-80); border chunks
// are clipped to the tensor and zero-padded (chunk_logical_region,
// model.py:158-170; _ChunkWriter / import_raw, tensorfile.py:108-165).
//   scatter: payloads of a batch of chunks -> their clipped regions of the dense tensor
//   gather:  dense tensor -> payloads (zero padding outside the tensor)
// Elements are opaque `elem_bytes`-byte items (scalar width x lanes), so one
// kernel serves every element type.  These sit on the PCIe / disk path
// (~50 GB/s), two orders below HBM; one element per thread is plenty.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rwb.h"
#include "rwb_common.cuh"

namespace rwb {
namespace {

struct ChunkGeo {
  int nd;                 // padded to 4 dims (leading 1s)
  long long size[4];
  long long chunk[4];
  long long grid[4];      // chunks per dimension
  long long box;          // elements per chunk
};

int make_chunk_geo(int32_t ndim, const int64_t* size, const int64_t* chunk, ChunkGeo* g) {
  if (ndim < 1 || ndim > 4 || !size || !chunk) return fail(RWB_ERR_INVALID, "chunks: ndim must be 1..4");
  g->nd = 4;
  g->box = 1;
  for (int d = 0; d < 4; ++d) {
    const int s = d - (4 - ndim);
    g->size[d] = s >= 0 ? size[s] : 1;
    g->chunk[d] = s >= 0 ? chunk[s] : 1;
    if (g->size[d] < 1 || g->chunk[d] < 1) return fail(RWB_ERR_INVALID, "chunks: sizes must be positive");
    g->grid[d] = (g->size[d] + g->chunk[d] - 1) / g->chunk[d];
    g->box *= g->chunk[d];
  }
  return RWB_OK;
}

template <typename T>
__device__ __forceinline__ void copy_elem(unsigned char* dst, const unsigned char* src, int eb) {
  const int n = eb / (int)sizeof(T);
  for (int i = 0; i < n; ++i) reinterpret_cast<T*>(dst)[i] = reinterpret_cast<const T*>(src)[i];
}

__device__ __forceinline__ void move_elem(unsigned char* dst, const unsigned char* src, int eb) {
  if ((eb & 7) == 0)
    copy_elem<unsigned long long>(dst, src, eb);
  else if ((eb & 3) == 0)
    copy_elem<unsigned int>(dst, src, eb);
  else if ((eb & 1) == 0)
    copy_elem<unsigned short>(dst, src, eb);
  else
    copy_elem<unsigned char>(dst, src, eb);
}

__device__ __forceinline__ void zero_elem(unsigned char* dst, int eb) {
  for (int i = 0; i < eb; ++i) dst[i] = 0;
}

// blockIdx.y: chunk of the batch; x-blocks stride over the chunk box
template <bool GATHER>
__global__ void __launch_bounds__(256) chunks_kernel(ChunkGeo g, int eb, unsigned char* __restrict__ payloads,
                                                     unsigned char* __restrict__ dense,
                                                     const long long* __restrict__ ids, long long first,
                                                     long long n) {
  const long long c = (long long)blockIdx.y + (long long)blockIdx.z * gridDim.y;
  if (c >= n) return;
  long long id = ids ? ids[c] : first + c;
  long long org[4];
  for (int d = 3; d >= 0; --d) {
    org[d] = (id % g.grid[d]) * g.chunk[d];
    id /= g.grid[d];
  }
  unsigned char* pay = payloads + c * g.box * eb;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < g.box; e += (long long)gridDim.x * blockDim.x) {
    long long r = e, gi = 0;
    bool in = true;
    long long coord[4];
    for (int d = 3; d >= 0; --d) {
      coord[d] = org[d] + r % g.chunk[d];
      r /= g.chunk[d];
      in = in && coord[d] < g.size[d];
    }
    for (int d = 0; d < 4; ++d) gi = gi * g.size[d] + coord[d];
    if (GATHER) {
      if (in)
        move_elem(pay + e * eb, dense + gi * eb, eb);
      else
        zero_elem(pay + e * eb, eb);
    } else if (in) {
      move_elem(dense + gi * eb, pay + e * eb, eb);
    }
  }
}

template <bool GATHER>
int run_chunks(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t elem_bytes, void* payloads,
               const int64_t* chunk_ids, int64_t first, int64_t n, void* dense, void* stream) {
  ChunkGeo g;
  int rc = make_chunk_geo(ndim, size, chunk, &g);
  if (rc) return rc;
  if (elem_bytes < 1 || elem_bytes > 64) return fail(RWB_ERR_INVALID, "chunks: elem_bytes must be 1..64");
  if (n < 0) return fail(RWB_ERR_INVALID, "chunks: negative chunk count");
  if (n == 0) return RWB_OK;
  if (!payloads || !dense) return fail(RWB_ERR_INVALID, "chunks: null pointer");
  const long long total = g.grid[0] * g.grid[1] * g.grid[2] * g.grid[3];
  if (!chunk_ids && (first < 0 || first + n > total)) return fail(RWB_ERR_INVALID, "chunks: chunk range outside the grid");
  cudaStream_t st = (cudaStream_t)stream;
  const long long bx = (g.box + 255) / 256;
  const unsigned gx = (unsigned)(bx < 64 ? bx : 64);
  const long long ny = n < 65535 ? n : 65535;
  const long long nz = (n + ny - 1) / ny;
  chunks_kernel<GATHER><<<dim3(gx, (unsigned)ny, (unsigned)nz), 256, 0, st>>>(
      g, elem_bytes, (unsigned char*)payloads, (unsigned char*)dense, (const long long*)chunk_ids, first, n);
  RWB_LAUNCH_CHECK(GATHER ? "chunks_gather" : "chunks_scatter");
  count_launches(1);
  return RWB_OK;
}

// f32(pairwise means along z, then y, then x) of each 2^d block, a trailing odd
// element passing through (downsample_mean / _pairwise_mean, ops.py:611-676;
// float64 arithmetic: assemble_region hands the means float64 blocks, ops.py:426-464).
// sel[k] = 0: dimension k is not downsampled (downsample_mean(dims=...), ops.py:614-616).
__global__ void __launch_bounds__(256) downsample_mean_kernel(const float* __restrict__ src, long long fz, long long fy,
                                                              long long fx, float* __restrict__ dst, long long cz,
                                                              long long cy, long long cx, int sz, int sy, int sx) {
  const long long n = cz * cy * cx;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (long long)gridDim.x * blockDim.x) {
    const long long jx = o % cx, jy = (o / cx) % cy, jz = o / (cx * cy);
    const long long bz = sz ? 2 * jz : jz, by = sy ? 2 * jy : jy, bx = sx ? 2 * jx : jx;
    const int nz = (sz && bz + 1 < fz) ? 2 : 1, ny = (sy && by + 1 < fy) ? 2 : 1, nx = (sx && bx + 1 < fx) ? 2 : 1;
    double v[2][2][2];
    for (int a = 0; a < nz; ++a)
      for (int b = 0; b < ny; ++b)
        for (int c = 0; c < nx; ++c) v[a][b][c] = src[((bz + a) * fy + (by + b)) * fx + (bx + c)];
    double m1[2][2], m2[2];
    for (int b = 0; b < ny; ++b)
      for (int c = 0; c < nx; ++c) m1[b][c] = nz == 2 ? __dmul_rn(__dadd_rn(v[0][b][c], v[1][b][c]), 0.5) : v[0][b][c];
    for (int c = 0; c < nx; ++c) m2[c] = ny == 2 ? __dmul_rn(__dadd_rn(m1[0][c], m1[1][c]), 0.5) : m1[0][c];
    dst[o] = (float)(nx == 2 ? __dmul_rn(__dadd_rn(m2[0], m2[1]), 0.5) : m2[0]);
  }
}

}  // namespace
}  // namespace rwb

extern "C" int rwb_chunks_scatter(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t elem_bytes,
                                  const void* payloads, const int64_t* chunk_ids, int64_t first, int64_t n,
                                  void* dense, void* stream) {
  return rwb::run_chunks<false>(ndim, size, chunk, elem_bytes, const_cast<void*>(payloads), chunk_ids, first, n,
                                dense, stream);
}

extern "C" int rwb_chunks_gather(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t elem_bytes,
                                 const void* dense, const int64_t* chunk_ids, int64_t first, int64_t n,
                                 void* payloads, void* stream) {
  return rwb::run_chunks<true>(ndim, size, chunk, elem_bytes, payloads, chunk_ids, first, n,
                               const_cast<void*>(dense), stream);
}

extern "C" int rwb_downsample_mean_dims_f32(int32_t ndim, const int64_t* size, uint32_t dims_mask, const float* src,
                                            float* dst, void* stream) {
  if (ndim < 1 || ndim > 3 || !size || !src || !dst) return rwb::fail(RWB_ERR_INVALID, "downsample_mean: bad arguments");
  if (dims_mask >> ndim) return rwb::fail(RWB_ERR_INVALID, "downsample_mean: dims outside the tensor");
  long long f[3] = {1, 1, 1};
  int sel[3] = {0, 0, 0};
  for (int d = 0; d < ndim; ++d) {
    if (size[d] < 1) return rwb::fail(RWB_ERR_INVALID, "downsample_mean: sizes must be positive");
    f[3 - ndim + d] = size[d];
    sel[3 - ndim + d] = (dims_mask >> d) & 1;
  }
  // unselected (and unit leading) dims keep their size
  const long long c[3] = {sel[0] ? (f[0] + 1) / 2 : f[0], sel[1] ? (f[1] + 1) / 2 : f[1], sel[2] ? (f[2] + 1) / 2 : f[2]};
  const long long n = c[0] * c[1] * c[2];
  const long long blocks = (n + 255) / 256;
  rwb::downsample_mean_kernel<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, (cudaStream_t)stream>>>(
      src, f[0], f[1], f[2], dst, c[0], c[1], c[2], sel[0], sel[1], sel[2]);
  RWB_LAUNCH_CHECK("downsample_mean_kernel");
  rwb::count_launches(1);
  return RWB_OK;
}

extern "C" int rwb_downsample_mean_f32(int32_t ndim, const int64_t* size, const float* src, float* dst,
                                       void* stream) {
  return rwb_downsample_mean_dims_f32(ndim, size, ndim >= 1 && ndim <= 3 ? (1u << ndim) - 1u : 0u, src, dst, stream);
}

// ---------------------------------------------------------------------------
// Constant-chunk table (build_const_chunk_table, ops.py:777-816): one element per chunk of a
// scalar tensor, the chunk's value if every element of its logical (clipped) region equals the
// first one (element type ==, so NaN never matches), else the sentinel (NaN for floats, the
// type's maximum for integers, ops.py:770-774).  One CTA per chunk.
namespace rwb {
namespace {

template <typename T>
__device__ __forceinline__ T sentinel_of();
template <> __device__ __forceinline__ uint8_t sentinel_of<uint8_t>() { return 0xFF; }
template <> __device__ __forceinline__ int16_t sentinel_of<int16_t>() { return 0x7FFF; }
template <> __device__ __forceinline__ uint16_t sentinel_of<uint16_t>() { return 0xFFFF; }
template <> __device__ __forceinline__ float sentinel_of<float>() { return __int_as_float(0x7FC00000); }
template <> __device__ __forceinline__ double sentinel_of<double>() { return __longlong_as_double(0x7FF8000000000000LL); }

template <typename T>
__global__ void __launch_bounds__(256) const_table_kernel(ChunkGeo g, const T* __restrict__ src, T* __restrict__ table,
                                                          long long n) {
  __shared__ int all_eq;
  for (long long c = blockIdx.x; c < n; c += gridDim.x) {
    long long id = c, org[4], ext[4], cnt = 1;
    for (int d = 3; d >= 0; --d) {
      org[d] = (id % g.grid[d]) * g.chunk[d];
      id /= g.grid[d];
      ext[d] = min(g.chunk[d], g.size[d] - org[d]);
      cnt *= ext[d];
    }
    const long long base = ((org[0] * g.size[1] + org[1]) * g.size[2] + org[2]) * g.size[3] + org[3];
    const T first = src[base];
    if (threadIdx.x == 0) all_eq = 1;
    __syncthreads();
    bool eq = true;
    for (long long e = threadIdx.x; e < cnt && eq; e += blockDim.x) {
      long long r = e, off[4];
      for (int d = 3; d >= 0; --d) {
        off[d] = r % ext[d];
        r /= ext[d];
      }
      const long long gi = (((org[0] + off[0]) * g.size[1] + org[1] + off[1]) * g.size[2] + org[2] + off[2]) * g.size[3] +
                           org[3] + off[3];
      eq = src[gi] == first;
    }
    if (!eq) all_eq = 0;  // benign race: every writer stores 0
    __syncthreads();
    if (threadIdx.x == 0) table[c] = all_eq ? first : sentinel_of<T>();
    __syncthreads();
  }
}

}  // namespace
}  // namespace rwb

extern "C" int rwb_const_chunk_table(int32_t ndim, const int64_t* size, const int64_t* chunk, int32_t scalar_code,
                                     const void* src, void* table, void* stream) {
  rwb::ChunkGeo g;
  int rc = rwb::make_chunk_geo(ndim, size, chunk, &g);
  if (rc) return rc;
  if (!src || !table) return rwb::fail(RWB_ERR_INVALID, "const_chunk_table: null pointer");
  const long long n = g.grid[0] * g.grid[1] * g.grid[2] * g.grid[3];
  const unsigned blocks = (unsigned)(n < 65535 ? n : 65535);
  cudaStream_t st = (cudaStream_t)stream;
  switch (scalar_code) {
    case 0: rwb::const_table_kernel<uint8_t><<<blocks, 256, 0, st>>>(g, (const uint8_t*)src, (uint8_t*)table, n); break;
    case 1: rwb::const_table_kernel<int16_t><<<blocks, 256, 0, st>>>(g, (const int16_t*)src, (int16_t*)table, n); break;
    case 2: rwb::const_table_kernel<uint16_t><<<blocks, 256, 0, st>>>(g, (const uint16_t*)src, (uint16_t*)table, n); break;
    case 3: rwb::const_table_kernel<float><<<blocks, 256, 0, st>>>(g, (const float*)src, (float*)table, n); break;
    case 4: rwb::const_table_kernel<double><<<blocks, 256, 0, st>>>(g, (const double*)src, (double*)table, n); break;
    default: return rwb::fail(RWB_ERR_INVALID, "const_chunk_table: scalar code must be 0..4 (u8, i16, u16, f32, f64)");
  }
  RWB_LAUNCH_CHECK("const_table_kernel");
  rwb::count_launches(1);
  return RWB_OK;
}

// ---------------------------------------------------------------------------
// Nearest-neighbour pan/zoom resampling of a 2-D image or an axis-aligned slice of a 3-D level
// (the reference's viewer path: _resample_nn, slice_view, image_view, render.py:640-741).  Frame
// pixel (p0, p1) samples source element floor((p + 0.5) * scale + offset) per axis, computed in
// float64 like the reference (numpy float64 arange), background 0 outside the source.
namespace rwb {
namespace {

__global__ void __launch_bounds__(256) resample_nn_kernel(const unsigned char* __restrict__ src, long long st0,
                                                          long long st1, long long base, long long n0, long long n1,
                                                          int eb, unsigned char* __restrict__ frame, long long f0,
                                                          long long f1, double s0, double s1, double o0, double o1) {
  const long long n = f0 * f1;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long p0 = e / f1, p1 = e % f1;
    const long long a0 = (long long)floor(__dadd_rn(__dmul_rn(__dadd_rn((double)p0, 0.5), s0), o0));
    const long long a1 = (long long)floor(__dadd_rn(__dmul_rn(__dadd_rn((double)p1, 0.5), s1), o1));
    unsigned char* out = frame + e * eb;
    if (a0 >= 0 && a0 < n0 && a1 >= 0 && a1 < n1)
      move_elem(out, src + (base + a0 * st0 + a1 * st1) * eb, eb);
    else
      zero_elem(out, eb);
  }
}

}  // namespace
}  // namespace rwb

extern "C" int rwb_resample_nn(int32_t src_ndim, const int64_t* src_size, int32_t slice_dim, int64_t slice_index,
                               int32_t elem_bytes, const void* src, const int64_t* frame_size, const double* scale,
                               const double* offset, void* frame, void* stream) {
  if (!src_size || !frame_size || !scale || !offset || !src || !frame)
    return rwb::fail(RWB_ERR_INVALID, "resample_nn: null pointer");
  if (elem_bytes < 1 || elem_bytes > 64) return rwb::fail(RWB_ERR_INVALID, "resample_nn: elem_bytes must be 1..64");
  long long n0, n1, st0, st1, base = 0;
  if (src_ndim == 2 && slice_dim < 0) {
    n0 = src_size[0], n1 = src_size[1], st0 = n1, st1 = 1;
  } else if (src_ndim == 3 && slice_dim >= 0 && slice_dim < 3) {
    const long long s[3] = {src_size[0], src_size[1], src_size[2]};
    const long long stride[3] = {s[1] * s[2], s[2], 1};
    if (slice_index < 0 || slice_index >= s[slice_dim]) return rwb::fail(RWB_ERR_INVALID, "resample_nn: slice index");
    base = slice_index * stride[slice_dim];
    const int d0 = slice_dim == 0 ? 1 : 0, d1 = slice_dim == 2 ? 1 : 2;  // the remaining axes, in order
    n0 = s[d0], n1 = s[d1], st0 = stride[d0], st1 = stride[d1];
  } else {
    return rwb::fail(RWB_ERR_INVALID, "resample_nn: a 2-D image (slice_dim < 0) or a 3-D slice");
  }
  const long long f0 = frame_size[0], f1 = frame_size[1];
  if (f0 < 1 || f1 < 1 || n0 < 1 || n1 < 1) return rwb::fail(RWB_ERR_INVALID, "resample_nn: sizes must be positive");
  const long long blocks = (f0 * f1 + 255) / 256;
  rwb::resample_nn_kernel<<<(unsigned)(blocks < 8192 ? blocks : 8192), 256, 0, (cudaStream_t)stream>>>(
      (const unsigned char*)src, st0, st1, base, n0, n1, elem_bytes, (unsigned char*)frame, f0, f1, scale[0],
      scale[1], offset[0], offset[1]);
  RWB_LAUNCH_CHECK("resample_nn_kernel");
  rwb::count_launches(1);
  return RWB_OK;
}
