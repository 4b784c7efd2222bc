// Per-voxel operators of the hierarchical random walker: LOD step, seed
// projection, coarse-to-fine upsampling, edge weights, labels.
//
// All of them are HBM-bound streaming kernels (a few bytes per voxel).  One
// thread per OUTPUT voxel, x fastest so warps read/write contiguous rows;
// neighbourhood re-reads are served by L1 (x/y neighbours are in the same or
// adjacent warps).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "rwb_common.cuh"

namespace rwb {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }

int device_slot(int* dev) {
  RWB_CUDA(cudaGetDevice(dev));
  if (*dev < 0 || *dev >= kMaxDevices) return fail(RWB_ERR_UNSUPPORTED, "device ordinal beyond the launch caches");
  return RWB_OK;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t err, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ")";
  return RWB_ERR_CUDA;
}

bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("RWB_DEBUG_SYNC");
    return e && *e && *e != '0';
  }();
  return on;
}

int shape_from(int32_t ndim, const int64_t* size, Shape3* out) {
  if (ndim < 1 || ndim > 3 || size == nullptr) return fail(RWB_ERR_INVALID, "ndim must be 1..3");
  int64_t s[3] = {1, 1, 1};
  for (int i = 0; i < ndim; ++i) {
    if (size[i] < 1 || size[i] > (1ll << 30)) return fail(RWB_ERR_INVALID, "dimension size out of range");
    s[3 - ndim + i] = size[i];
  }
  if (s[0] * s[1] * s[2] > (1ll << 40)) return fail(RWB_ERR_INVALID, "level too large");
  if (s[0] > 65535 || s[1] > 65535 * 8) return fail(RWB_ERR_INVALID, "dimension too large for the 3-D launch grid");
  out->nz = (int)s[0];
  out->ny = (int)s[1];
  out->nx = (int)s[2];
  return RWB_OK;
}

// 3-D launch geometry for per-voxel kernels: block 32 (x) x 8 (y), grid over
// (x tiles, y tiles, z) — no 64-bit index division in the kernels.
constexpr int BX = 32, BY = 8;
static inline dim3 grid3(const Shape3& s) { return dim3((s.nx + BX - 1) / BX, (s.ny + BY - 1) / BY, s.nz); }
static const dim3 kBlock3(BX, BY, 1);

#define VOXEL3(S, X, Y, Z)                    \
  const int X = blockIdx.x * BX + threadIdx.x; \
  const int Y = blockIdx.y * BY + threadIdx.y; \
  const int Z = blockIdx.z;                    \
  if (X >= (S).nx || Y >= (S).ny) return

// ---------------------------------------------------------------------------
// LOD step: f32(mean2(f32(conv3_clamp(x)))) with the reference's float64
// operation order (ops.py:533-548 then ops.py:664-676): every 1-D pass is
// acc = 0; acc += k0*a; acc += k1*b; acc += k2*c (products by powers of two
// are exact, so fma == mul+add here), dims in order z, y, x; the conv result
// is rounded to f32 before the pairwise means.

__device__ __forceinline__ double conv3(double a, double b, double c) {
  double acc = 0.0;
  acc += 0.25 * a;
  acc += 0.5 * b;
  acc += 0.25 * c;
  return acc;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

template <bool HAS_Z, bool HAS_Y>
__global__ void __launch_bounds__(256) lod_down_kernel(const float* __restrict__ src, Shape3 fs,
                                                       float* __restrict__ dst, Shape3 cs) {
  VOXEL3(cs, jx, jy, jz);
  const long long o = ((long long)jz * cs.ny + jy) * cs.nx + jx;
  // fine index windows 2j-1 .. 2j+2, clamped
  int zi[4], yi[4], xi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    zi[k] = clampi(2 * jz - 1 + k, 0, fs.nz - 1);
    yi[k] = clampi(2 * jy - 1 + k, 0, fs.ny - 1);
    xi[k] = clampi(2 * jx - 1 + k, 0, fs.nx - 1);
  }
  const int ncz = HAS_Z ? ((2 * jz + 1 < fs.nz) ? 2 : 1) : 1;
  const int ncy = HAS_Y ? ((2 * jy + 1 < fs.ny) ? 2 : 1) : 1;
  const int ncx = (2 * jx + 1 < fs.nx) ? 2 : 1;
  const long long sxy = (long long)fs.ny * fs.nx;

  // conv along z for the 2 child planes at every (y, x) of the 4x4 window
  double A[2][4][4];
#pragma unroll
  for (int cz = 0; cz < 2; ++cz)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (!HAS_Y && a != 1) { A[cz][a][b] = 0.0; continue; }
        if (HAS_Z) {
          const float* col = src + (long long)yi[a] * fs.nx + xi[b];
          double v0 = __ldg(col + zi[cz] * sxy);
          double v1 = __ldg(col + zi[cz + 1] * sxy);
          double v2 = __ldg(col + zi[cz + 2] * sxy);
          A[cz][a][b] = conv3(v0, v1, v2);
        } else {
          A[cz][a][b] = (double)__ldg(src + (long long)yi[a] * fs.nx + xi[b]);
        }
      }
  float C[2][2][2];
#pragma unroll
  for (int cz = 0; cz < 2; ++cz)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      double B[4];
#pragma unroll
      for (int b = 0; b < 4; ++b)
        B[b] = HAS_Y ? conv3(A[cz][cy][b], A[cz][cy + 1][b], A[cz][cy + 2][b]) : A[cz][1][b];
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) C[cz][cy][cx] = (float)conv3(B[cx], B[cx + 1], B[cx + 2]);
    }
  // pairwise means, dims z, y, x
  double m0[2][2];
#pragma unroll
  for (int cy = 0; cy < 2; ++cy)
#pragma unroll
    for (int cx = 0; cx < 2; ++cx)
      m0[cy][cx] = ncz == 2 ? ((double)C[0][cy][cx] + (double)C[1][cy][cx]) * 0.5 : (double)C[0][cy][cx];
  double m1[2];
#pragma unroll
  for (int cx = 0; cx < 2; ++cx) m1[cx] = ncy == 2 ? (m0[0][cx] + m0[1][cx]) * 0.5 : m0[0][cx];
  double m2 = ncx == 2 ? (m1[0] + m1[1]) * 0.5 : m1[0];
  dst[o] = (float)m2;
}

// ---------------------------------------------------------------------------
// seed projection: fg if any child fg and none bg; bg symmetric; else 0

__global__ void __launch_bounds__(256) project_seeds_kernel(const uint8_t* __restrict__ fine, Shape3 fs,
                                                            uint8_t* __restrict__ coarse, Shape3 cs) {
  VOXEL3(cs, jx, jy, jz);
  const long long o = ((long long)jz * cs.ny + jy) * cs.nx + jx;
  bool fg = false, bg = false;
  for (int z = 2 * jz; z < min(2 * jz + 2, fs.nz); ++z)
    for (int y = 2 * jy; y < min(2 * jy + 2, fs.ny); ++y)
      for (int x = 2 * jx; x < min(2 * jx + 2, fs.nx); ++x) {
        uint8_t s = fine[((long long)z * fs.ny + y) * fs.nx + x];
        fg |= (s == 1);
        bg |= (s == 2);
      }
  coarse[o] = (fg && !bg) ? 1 : ((bg && !fg) ? 2 : 0);
}

// ---------------------------------------------------------------------------
// cell-centred multilinear prolongation (parent coordinate g/2 - 1/4, clamped)

// One thread per PARENT voxel j: it reads the clamped 3x3x3 parent
// neighbourhood once and writes the (up to) 2x2x2 fine voxels 2j, 2j+1 that
// fall inside the fine window [fo, fo+fw) (taps 1/4, 3/4; x first, then y,
// then z).  ~1/8 of the address arithmetic of a per-fine-voxel kernel, which
// was instruction-bound.  The parent is addressed through a window
// [po, po+pw) of the full parent of size ps; the fine output through the
// window's own dense layout.  Full-level and windowed calls run this same
// code, so every caller gets bit-identical values.
__global__ void __launch_bounds__(256) upsample_kernel(const float* __restrict__ parent, Shape3 ps, Shape3 po,
                                                       Shape3 pw, float* __restrict__ fine, Shape3 fs, Shape3 fo,
                                                       Shape3 fw, Shape3 j0) {
  const int jx = j0.nx + blockIdx.x * BX + threadIdx.x;
  const int jy = j0.ny + blockIdx.y * BY + threadIdx.y;
  const int jz = j0.nz + blockIdx.z;
  if (jx >= ps.nx || jy >= ps.ny || jz >= ps.nz) return;
  const long long psxy = (long long)pw.ny * pw.nx;
  // window-relative taps, clamped into the parent window: a tap outside it only feeds fine
  // voxels outside the fine window (the host checked that the window's taps are covered), and
  // reading it would run past the window buffer
  auto in_w = [](int v, int n) { return min(max(v, 0), n - 1); };
  const int xm = in_w(max(jx - 1, 0) - po.nx, pw.nx), xc = in_w(jx - po.nx, pw.nx);
  const int xp = in_w(min(jx + 1, ps.nx - 1) - po.nx, pw.nx);
  const int zz[3] = {in_w(max(jz - 1, 0) - po.nz, pw.nz), in_w(jz - po.nz, pw.nz),
                     in_w(min(jz + 1, ps.nz - 1) - po.nz, pw.nz)};
  const int yy[3] = {in_w(max(jy - 1, 0) - po.ny, pw.ny), in_w(jy - po.ny, pw.ny),
                     in_w(min(jy + 1, ps.ny - 1) - po.ny, pw.ny)};
  // x-interpolated parent rows: lo -> fine 2j (0.25 P[j-1] + 0.75 P[j]), hi -> 2j+1 (0.75 P[j] + 0.25 P[j+1])
  float lo[3][3], hi[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float* row = parent + zz[a] * psxy + (long long)yy[b] * pw.nx;
      const float c = __ldg(row + xc), m = __ldg(row + xm), p = __ldg(row + xp);
      lo[a][b] = __fmaf_rn(0.25f, m, __fmul_rn(0.75f, c));
      hi[a][b] = __fmaf_rn(0.75f, c, __fmul_rn(0.25f, p));
    }
  // then y and z; a fine dimension of size 1 takes its single row unweighted
  const bool fy2 = fs.ny > 1, fz2 = fs.nz > 1;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const int gz = 2 * jz + dz;
    if (gz >= fs.nz || gz < fo.nz || gz >= fo.nz + fw.nz) continue;
    const int za = dz ? 1 : 0, zb = dz ? 2 : 1;
    const float wa = fz2 ? (dz ? 0.75f : 0.25f) : 0.f, wb = fz2 ? (dz ? 0.25f : 0.75f) : 1.f;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int gy = 2 * jy + dy;
      if (gy >= fs.ny || gy < fo.ny || gy >= fo.ny + fw.ny) continue;
      const int ya = dy ? 1 : 0, yb = dy ? 2 : 1;
      const float va = fy2 ? (dy ? 0.75f : 0.25f) : 0.f, vb = fy2 ? (dy ? 0.25f : 0.75f) : 1.f;
      float f[2];
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const float(*xs)[3] = dx ? hi : lo;
        const float ra = __fmaf_rn(va, xs[za][ya], __fmul_rn(vb, xs[za][yb]));
        const float rb = __fmaf_rn(va, xs[zb][ya], __fmul_rn(vb, xs[zb][yb]));
        f[dx] = __fmaf_rn(wa, ra, __fmul_rn(wb, rb));
      }
      const int gx = 2 * jx;
      float* out = fine + ((long long)(gz - fo.nz) * fw.ny + (gy - fo.ny)) * fw.nx + (gx - fo.nx);
      const bool in0 = gx >= fo.nx && gx < fo.nx + fw.nx;
      const bool in1 = gx + 1 < fs.nx && gx + 1 >= fo.nx && gx + 1 < fo.nx + fw.nx;
      if (in0 && in1 && (((uintptr_t)out) & 7) == 0) {
        *reinterpret_cast<float2*>(out) = make_float2(f[0], f[1]);
      } else {
        if (in0) out[0] = f[0];
        if (in1) out[1] = f[1];
      }
    }
  }
}

// Whole-level upsampling, UQ parent x-voxels (2 UQ fine x) per thread: the 9
// parent rows a thread needs are x-interpolated once and reused by its 2x2
// fine rows, and every fine row segment is written with 16 B stores.
// Same expressions as upsample_kernel, so the results are bit-identical.
// Requires fine nx == 2 * parent nx, nx % (2 UQ) == 0 (16 B aligned row segments).
constexpr int UQ = 2;  // parent x-voxels per thread
constexpr int UZ = 8;  // parent planes marched per thread
// `fine` = fine plane fz0 (a z-window [fz0, fz1) of the level, full in y and x).
__global__ void __launch_bounds__(256, 4) upsample4_kernel(const float* __restrict__ parent, Shape3 ps,
                                                        float* __restrict__ fine, Shape3 fs, int fz0, int fz1) {
  const int jx0 = (blockIdx.x * BX + threadIdx.x) * UQ;
  const int jy = blockIdx.y * BY + threadIdx.y;
  const int jz0 = (fz0 >> 1) + blockIdx.z * UZ;
  if (jx0 >= ps.nx || jy >= ps.ny) return;
  const long long psxy = (long long)ps.ny * ps.nx;
  const int yy[3] = {max(jy - 1, 0), jy, min(jy + 1, ps.ny - 1)};
  int xx[UQ + 2];
#pragma unroll
  for (int k = 0; k < UQ + 2; ++k) xx[k] = min(max(jx0 - 1 + k, 0), ps.nx - 1);
  // x-interpolated rows of the parent planes jz-1, jz, jz+1 (clamped): a window slid along z
  float lo[3][3][UQ], hi[3][3][UQ];
  auto load_plane = [&](int pz, float (&l)[3][UQ], float (&h)[3][UQ]) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const float* row = parent + pz * psxy + (long long)yy[b] * ps.nx;
      float v[UQ + 2];
#pragma unroll
      for (int k = 0; k < UQ + 2; ++k) v[k] = __ldg(row + xx[k]);
#pragma unroll
      for (int i = 0; i < UQ; ++i) {
        l[b][i] = __fmaf_rn(0.25f, v[i], __fmul_rn(0.75f, v[i + 1]));
        h[b][i] = __fmaf_rn(0.75f, v[i + 1], __fmul_rn(0.25f, v[i + 2]));
      }
    }
  };
  load_plane(max(jz0 - 1, 0), lo[0], hi[0]);
  load_plane(min(jz0, ps.nz - 1), lo[1], hi[1]);
  const bool fy2 = fs.ny > 1, fz2 = fs.nz > 1;
#pragma unroll
  for (int s = 0; s < UZ; ++s) {
    const int jz = jz0 + s;
    if (jz >= ps.nz || 2 * jz >= fz1) break;
    load_plane(min(jz + 1, ps.nz - 1), lo[2], hi[2]);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz) {
      const int gz = 2 * jz + dz;
      if (gz >= fs.nz || gz < fz0 || gz >= fz1) continue;
      const int za = dz ? 1 : 0, zb = dz ? 2 : 1;
      const float wa = fz2 ? (dz ? 0.75f : 0.25f) : 0.f, wb = fz2 ? (dz ? 0.25f : 0.75f) : 1.f;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        const int gy = 2 * jy + dy;
        if (gy >= fs.ny) continue;
        const int ya = dy ? 1 : 0, yb = dy ? 2 : 1;
        const float va = fy2 ? (dy ? 0.75f : 0.25f) : 0.f, vb = fy2 ? (dy ? 0.25f : 0.75f) : 1.f;
        float f[2 * UQ];
#pragma unroll
        for (int i = 0; i < UQ; ++i)
#pragma unroll
          for (int dx = 0; dx < 2; ++dx) {
            const float(*xs)[3][UQ] = dx ? hi : lo;
            const float ra = __fmaf_rn(va, xs[za][ya][i], __fmul_rn(vb, xs[za][yb][i]));
            const float rb = __fmaf_rn(va, xs[zb][ya][i], __fmul_rn(vb, xs[zb][yb][i]));
            f[2 * i + dx] = __fmaf_rn(wa, ra, __fmul_rn(wb, rb));
          }
        float4* out = reinterpret_cast<float4*>(fine + ((long long)(gz - fz0) * fs.ny + gy) * fs.nx + 2 * jx0);
#pragma unroll
        for (int q = 0; q < UQ / 2; ++q) out[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
      }
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
      for (int i = 0; i < UQ; ++i) {
        lo[0][b][i] = lo[1][b][i], hi[0][b][i] = hi[1][b][i];
        lo[1][b][i] = lo[2][b][i], hi[1][b][i] = hi[2][b][i];
      }
  }
}

static void launch_upsample(const float* parent, Shape3 ps, Shape3 po, Shape3 pw, float* fine, Shape3 fs, Shape3 fo,
                            Shape3 fw, cudaStream_t st) {
  // parent voxels whose fine children intersect the window
  Shape3 j0{fo.nz >> 1, fo.ny >> 1, fo.nx >> 1};
  Shape3 j1{(fo.nz + fw.nz + 1) >> 1, (fo.ny + fw.ny + 1) >> 1, (fo.nx + fw.nx + 1) >> 1};
  dim3 grid((j1.nx - j0.nx + BX - 1) / BX, (j1.ny - j0.ny + BY - 1) / BY, j1.nz - j0.nz);
  upsample_kernel<<<grid, kBlock3, 0, st>>>(parent, ps, po, pw, fine, fs, fo, fw, j0);
}

// ---------------------------------------------------------------------------
// forward edge weights, lanes-last

__global__ void __launch_bounds__(256) edge_weights_kernel(const float* __restrict__ vol, Shape3 s, int ndim,
                                                           float beta, float wmin, float* __restrict__ w) {
  VOXEL3(s, x, y, z);
  const long long o = ((long long)z * s.ny + y) * s.nx + x;
  float c = vol[o];
  const long long sxy = (long long)s.ny * s.nx;
  float* out = w + o * ndim;
  int lane = 0;
  if (ndim == 3) out[lane++] = (z + 1 < s.nz) ? edge_weight(c, __ldg(vol + o + sxy), beta, wmin) : 0.0f;
  if (ndim >= 2) out[lane++] = (y + 1 < s.ny) ? edge_weight(c, __ldg(vol + o + s.nx), beta, wmin) : 0.0f;
  out[lane] = (x + 1 < s.nx) ? edge_weight(c, __ldg(vol + o + 1), beta, wmin) : 0.0f;
}

__global__ void __launch_bounds__(256) labels_kernel(const float* __restrict__ prob, long long n,
                                                     uint8_t* __restrict__ labels) {
  long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (o < n) labels[o] = prob[o] > 0.5f ? 1 : 0;
}

}  // namespace rwb

using namespace rwb;

static int coarse_of(const Shape3& f, Shape3* c) {
  c->nz = (f.nz + 1) / 2;
  c->ny = (f.ny + 1) / 2;
  c->nx = (f.nx + 1) / 2;
  return RWB_OK;
}

extern "C" int rwb_abi_version(void) { return RWB_ABI_VERSION; }

extern "C" const char* rwb_last_error(void) { return g_last_error.c_str(); }

extern "C" int64_t rwb_kernel_launches(void) { return (int64_t)g_launches.load(); }

extern "C" int rwb_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  RWB_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  RWB_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (prop.major != 10) return fail(RWB_ERR_UNSUPPORTED, "librwb is built for sm_100a (B200); found sm_" +
                                                             std::to_string(prop.major) + std::to_string(prop.minor));
  return RWB_OK;
}

// 3-D LOD step, separable and staged through shared memory: a CTA owns a
// coarse 8 (y) x 32 (x) column block and marches LZC coarse planes.  Per
// coarse plane: (1) z-conv of the two child fine planes at every (y, x) of the
// fine window incl. the 1-voxel clamp halo (18 x 66), each thread carrying two
// fine values per column from the previous plane, so every fine voxel is read
// once; (2) y-conv of the 16 child rows; (3) per output, the x-conv of its 8
// children and the pairwise means.  Every intermediate is computed from the
// same operands in the same order as lod_down_kernel (A = conv_z, B = conv_y(A),
// C = f32(conv_x(B))), so the result is bit-identical; each conv is evaluated
// once per fine position instead of up to 8 times.
constexpr int LCX = 32, LCY = 8, LZC = 8;                // coarse tile and planes per CTA
constexpr int LFX = 2 * LCX + 2, LFY = 2 * LCY + 2;      // fine window 66 x 18
constexpr int LCOLS = LFX * LFY;                          // fine columns per CTA (1188)
constexpr int LTH = LCX * LCY;                            // threads (one output each)
constexpr int LCPT = (LCOLS + LTH - 1) / LTH;             // columns per thread (5)

__global__ void __launch_bounds__(LTH) lod_down3_kernel(const float* __restrict__ src, Shape3 fs,
                                                        float* __restrict__ dst, Shape3 cs) {
  __shared__ double A[2][LFY][LFX];
  __shared__ __align__(16) double B[2][2 * LCY][LFX];
  const int tid = threadIdx.x;
  const int cx0 = blockIdx.x * LCX, cy0 = blockIdx.y * LCY, cz0 = blockIdx.z * LZC;
  const int fx0 = 2 * cx0 - 1, fy0 = 2 * cy0 - 1;
  const long long sxy = (long long)fs.ny * fs.nx;
  // this thread's fine columns (clamped level offsets) and the two fine values carried between planes
  long long colo[LCPT];
  bool colv[LCPT];
  float c1[LCPT], c2[LCPT];
#pragma unroll
  for (int k = 0; k < LCPT; ++k) {
    const int c = tid + k * LTH;
    colv[k] = c < LCOLS;
    const int ty = colv[k] ? c / LFX : 0, tx = colv[k] ? c % LFX : 0;
    colo[k] = (long long)clampi(fy0 + ty, 0, fs.ny - 1) * fs.nx + clampi(fx0 + tx, 0, fs.nx - 1);
    c1[k] = c2[k] = 0.f;
  }
  const int oy = tid / LCX, ox = tid % LCX;
  const int jy = cy0 + oy, jx = cx0 + ox;
  const int zend = min(cz0 + LZC, cs.nz);
  // fine planes 2jz+1, 2jz+2 of the current coarse plane, loaded one plane ahead
  float n1[LCPT], n2[LCPT];
  auto load_next = [&](int jz) {
    const long long z2 = (long long)clampi(2 * jz + 1, 0, fs.nz - 1) * sxy;
    const long long z3 = (long long)clampi(2 * jz + 2, 0, fs.nz - 1) * sxy;
#pragma unroll
    for (int k = 0; k < LCPT; ++k) {
      n1[k] = colv[k] ? __ldg(src + colo[k] + z2) : 0.f;
      n2[k] = colv[k] ? __ldg(src + colo[k] + z3) : 0.f;
    }
  };
  {
    const long long z0 = (long long)clampi(2 * cz0 - 1, 0, fs.nz - 1) * sxy;
    const long long z1 = (long long)clampi(2 * cz0, 0, fs.nz - 1) * sxy;
#pragma unroll
    for (int k = 0; k < LCPT; ++k) {
      c1[k] = colv[k] ? __ldg(src + colo[k] + z0) : 0.f;
      c2[k] = colv[k] ? __ldg(src + colo[k] + z1) : 0.f;
    }
    load_next(cz0);
  }
  for (int jz = cz0; jz < zend; ++jz) {
    // (1) z-conv: fine planes 2jz-1 .. 2jz+2 (clamped); the first two carried from jz-1
    float v2[LCPT], v3[LCPT];
#pragma unroll
    for (int k = 0; k < LCPT; ++k) v2[k] = n1[k], v3[k] = n2[k];
    if (jz + 1 < zend) load_next(jz + 1);  // in flight during this plane's convolutions
#pragma unroll
    for (int k = 0; k < LCPT; ++k) {
      if (!colv[k]) continue;
      const int c = tid + k * LTH, ty = c / LFX, tx = c % LFX;
      A[0][ty][tx] = conv3(c1[k], c2[k], v2[k]);
      A[1][ty][tx] = conv3(c2[k], v2[k], v3[k]);
      c1[k] = v2[k];
      c2[k] = v3[k];
    }
    __syncthreads();
    // (2) y-conv of the 16 child rows of both child planes: one thread per (plane,
    // column) slides down the 18 A rows, so every A value is read once
    if (tid < 2 * LFX) {
      const int cz = tid / LFX, tx = tid % LFX;
      double a0 = A[cz][0][tx], a1 = A[cz][1][tx];
#pragma unroll
      for (int r = 0; r < 2 * LCY; ++r) {
        const double a2 = A[cz][r + 2][tx];
        B[cz][r][tx] = conv3(a0, a1, a2);
        a0 = a1;
        a1 = a2;
      }
    }
    __syncthreads();
    // (3) x-conv of this output's 8 children, then the pairwise means (z, y, x)
    if (jy < cs.ny && jx < cs.nx) {
      float C[2][2][2];
#pragma unroll
      for (int cz = 0; cz < 2; ++cz)
#pragma unroll
        for (int cy = 0; cy < 2; ++cy) {
          // two 16-byte loads (2 ox doubles apart: 16-byte aligned) instead of four 8-byte ones
          const double2* b = reinterpret_cast<const double2*>(&B[cz][2 * oy + cy][2 * ox]);
          const double2 bl = b[0], bh = b[1];
          const double b0 = bl.x, b1 = bl.y, b2 = bh.x, b3 = bh.y;
          C[cz][cy][0] = (float)conv3(b0, b1, b2);
          C[cz][cy][1] = (float)conv3(b1, b2, b3);
        }
      const int ncz = (2 * jz + 1 < fs.nz) ? 2 : 1;
      const int ncy = (2 * jy + 1 < fs.ny) ? 2 : 1;
      const int ncx = (2 * jx + 1 < fs.nx) ? 2 : 1;
      double m0[2][2];
#pragma unroll
      for (int cy = 0; cy < 2; ++cy)
#pragma unroll
        for (int cx = 0; cx < 2; ++cx)
          m0[cy][cx] = ncz == 2 ? ((double)C[0][cy][cx] + (double)C[1][cy][cx]) * 0.5 : (double)C[0][cy][cx];
      double m1[2];
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) m1[cx] = ncy == 2 ? (m0[0][cx] + m0[1][cx]) * 0.5 : m0[0][cx];
      const double m2 = ncx == 2 ? (m1[0] + m1[1]) * 0.5 : m1[0];
      dst[((long long)jz * cs.ny + jy) * cs.nx + jx] = (float)m2;
    }
    __syncthreads();  // A and B are rewritten by the next plane
  }
}

extern "C" int rwb_lod_down_f32(int32_t ndim, const int64_t* size, const float* src, float* dst, void* stream) {
  Shape3 fs, cs;
  int rc = shape_from(ndim, size, &fs);
  if (rc) return rc;
  if (!src || !dst) return fail(RWB_ERR_INVALID, "null pointer");
  coarse_of(fs, &cs);
  if (ndim == 1) cs.ny = fs.ny, cs.nz = fs.nz;
  if (ndim == 2) cs.nz = fs.nz;
  cudaStream_t st = (cudaStream_t)stream;
  if (ndim == 3)
    lod_down3_kernel<<<dim3((cs.nx + LCX - 1) / LCX, (cs.ny + LCY - 1) / LCY, (cs.nz + LZC - 1) / LZC), LTH, 0, st>>>(
        src, fs, dst, cs);
  else if (ndim == 2)
    lod_down_kernel<false, true><<<grid3(cs), kBlock3, 0, st>>>(src, fs, dst, cs);
  else
    lod_down_kernel<false, false><<<grid3(cs), kBlock3, 0, st>>>(src, fs, dst, cs);
  RWB_LAUNCH_CHECK("lod_down_kernel");
  count_launches(1);
  return RWB_OK;
}

// Seed projection, 8 coarse x-voxels per thread: each fine row segment (16
// bytes) is one 16 B load, the 8 results one 8 B store.  Requires fine nx a
// multiple of 16 (coarse nx = fine nx / 2).
__global__ void __launch_bounds__(256) project_seeds8_kernel(const uint8_t* __restrict__ fine, Shape3 fs,
                                                             uint8_t* __restrict__ coarse, Shape3 cs) {
  const int jx0 = (blockIdx.x * BX + threadIdx.x) * 8;
  const int jy = blockIdx.y * BY + threadIdx.y;
  const int jz = blockIdx.z;
  if (jx0 >= cs.nx || jy >= cs.ny) return;
  // byte-parallel: per 32-bit word (4 fine x), OR over the 2 x 2 (z, y) rows of "byte == 1" / "== 2"
  // masks (0xff per byte), then fold the x pairs; all four rows' loads are issued first
  uint4 q[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int z = 2 * jz + (k >> 1), y = 2 * jy + (k & 1);
    q[k] = (z < fs.nz && y < fs.ny)
               ? *reinterpret_cast<const uint4*>(fine + ((long long)z * fs.ny + y) * fs.nx + 2 * jx0)
               : make_uint4(0u, 0u, 0u, 0u);
  }
  unsigned F[4] = {0u, 0u, 0u, 0u}, B[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned w[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      F[i] |= __vcmpeq4(w[i], 0x01010101u);
      B[i] |= __vcmpeq4(w[i], 0x02020202u);
    }
  }
  // word i holds coarse voxels 2i (fine bytes 0, 1) and 2i + 1 (bytes 2, 3): fold the pairs into
  // bytes 0 and 2, value 1 (fg only), 2 (bg only) or 0
  unsigned v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned f = (F[i] | (F[i] >> 8)) & 0x00010001u, g = (B[i] | (B[i] >> 8)) & 0x00010001u;
    v[i] = (f & ~g) | ((g & ~f) << 1);
  }
  const unsigned lo = (v[0] & 0xffu) | ((v[0] >> 16) << 8) | ((v[1] & 0xffu) << 16) | ((v[1] >> 16) << 24);
  const unsigned hi = (v[2] & 0xffu) | ((v[2] >> 16) << 8) | ((v[3] & 0xffu) << 16) | ((v[3] >> 16) << 24);
  *reinterpret_cast<uint2*>(coarse + ((long long)jz * cs.ny + jy) * cs.nx + jx0) = make_uint2(lo, hi);
}

extern "C" int rwb_project_seeds_u8(int32_t ndim, const int64_t* size, const uint8_t* fine, uint8_t* coarse,
                                    void* stream) {
  Shape3 fs, cs;
  int rc = shape_from(ndim, size, &fs);
  if (rc) return rc;
  if (!fine || !coarse) return fail(RWB_ERR_INVALID, "null pointer");
  coarse_of(fs, &cs);
  if (ndim < 3) cs.nz = fs.nz;
  if (ndim < 2) cs.ny = fs.ny;
  if (fs.nx % 16 == 0 && cs.nx * 2 == fs.nx && ((uintptr_t)fine & 15) == 0 && ((uintptr_t)coarse & 7) == 0) {
    dim3 grid((cs.nx / 8 + BX - 1) / BX, (cs.ny + BY - 1) / BY, cs.nz);
    project_seeds8_kernel<<<grid, kBlock3, 0, (cudaStream_t)stream>>>(fine, fs, coarse, cs);
  } else {
    project_seeds_kernel<<<grid3(cs), kBlock3, 0, (cudaStream_t)stream>>>(fine, fs, coarse, cs);
  }
  RWB_LAUNCH_CHECK("project_seeds_kernel");
  count_launches(1);
  return RWB_OK;
}

extern "C" int rwb_upsample_f32(int32_t ndim, const int64_t* parent_size, const float* parent,
                                const int64_t* fine_size, float* fine, void* stream) {
  Shape3 ps, fs, chk;
  int rc = shape_from(ndim, parent_size, &ps);
  if (rc) return rc;
  rc = shape_from(ndim, fine_size, &fs);
  if (rc) return rc;
  if (!parent || !fine) return fail(RWB_ERR_INVALID, "null pointer");
  coarse_of(fs, &chk);
  if (ndim < 3) chk.nz = fs.nz;
  if (ndim < 2) chk.ny = fs.ny;
  if (chk.nz != ps.nz || chk.ny != ps.ny || chk.nx != ps.nx)
    return fail(RWB_ERR_INVALID, "fine size is not a 2x refinement of the parent size");
  if (fs.nx == 2 * ps.nx && fs.nx % (2 * UQ) == 0 && ((uintptr_t)fine & 15) == 0) {
    dim3 grid((ps.nx / UQ + BX - 1) / BX, (ps.ny + BY - 1) / BY, (ps.nz + UZ - 1) / UZ);
    upsample4_kernel<<<grid, kBlock3, 0, (cudaStream_t)stream>>>(parent, ps, fine, fs, 0, fs.nz);
  } else {
    launch_upsample(parent, ps, Shape3{0, 0, 0}, ps, fine, fs, Shape3{0, 0, 0}, fs, (cudaStream_t)stream);
  }
  RWB_LAUNCH_CHECK("upsample_kernel");
  count_launches(1);
  return RWB_OK;
}

static int shape_raw(int32_t ndim, const int64_t* v, bool allow_zero_origin, Shape3* out) {
  int64_t s[3] = {allow_zero_origin ? 0 : 1, allow_zero_origin ? 0 : 1, allow_zero_origin ? 0 : 1};
  if (!v) return fail(RWB_ERR_INVALID, "null shape");
  for (int i = 0; i < ndim; ++i) {
    if (v[i] < (allow_zero_origin ? 0 : 1) || v[i] > (1ll << 30)) return fail(RWB_ERR_INVALID, "window out of range");
    s[3 - ndim + i] = v[i];
  }
  out->nz = (int)s[0];
  out->ny = (int)s[1];
  out->nx = (int)s[2];
  return RWB_OK;
}

extern "C" int rwb_upsample_window_f32(int32_t ndim, const int64_t* parent_size, const int64_t* parent_origin,
                                       const int64_t* parent_window, const float* parent, const int64_t* fine_size,
                                       const int64_t* fine_origin, const int64_t* fine_window, float* fine,
                                       void* stream) {
  if (ndim < 1 || ndim > 3) return fail(RWB_ERR_INVALID, "ndim must be 1..3");
  Shape3 ps, po, pw, fs, fo, fw, chk;
  int rc = shape_raw(ndim, parent_size, false, &ps);
  if (!rc) rc = shape_raw(ndim, parent_origin, true, &po);
  if (!rc) rc = shape_raw(ndim, parent_window, false, &pw);
  if (!rc) rc = shape_raw(ndim, fine_size, false, &fs);
  if (!rc) rc = shape_raw(ndim, fine_origin, true, &fo);
  if (!rc) rc = shape_raw(ndim, fine_window, false, &fw);
  if (rc) return rc;
  if (!parent || !fine) return fail(RWB_ERR_INVALID, "null pointer");
  coarse_of(fs, &chk);
  const int fd[3] = {fs.nz, fs.ny, fs.nx}, cd[3] = {chk.nz, chk.ny, chk.nx}, pd[3] = {ps.nz, ps.ny, ps.nx};
  const int pod[3] = {po.nz, po.ny, po.nx}, pwd[3] = {pw.nz, pw.ny, pw.nx};
  const int fod[3] = {fo.nz, fo.ny, fo.nx}, fwd[3] = {fw.nz, fw.ny, fw.nx};
  for (int d = 3 - ndim; d < 3; ++d) {
    if (cd[d] != pd[d]) return fail(RWB_ERR_INVALID, "fine size is not a 2x refinement of the parent size");
    if (fod[d] + fwd[d] > fd[d] || pod[d] + pwd[d] > pd[d]) return fail(RWB_ERR_INVALID, "window outside the level");
    // parent rows the taps of the fine window touch must lie inside the parent window
    int g0 = fod[d], g1 = fod[d] + fwd[d] - 1;
    int lo = (g0 & 1) ? g0 / 2 : (g0 / 2 > 0 ? g0 / 2 - 1 : 0);
    int hi = (g1 & 1) ? (g1 / 2 + 1 < pd[d] ? g1 / 2 + 1 : pd[d] - 1) : g1 / 2;
    if (fd[d] == 1) lo = hi = 0;
    if (lo < pod[d] || hi >= pod[d] + pwd[d]) return fail(RWB_ERR_INVALID, "parent window does not cover the taps");
  }
  const bool whole_parent = po.nz == 0 && po.ny == 0 && po.nx == 0 && pw.nz == ps.nz && pw.ny == ps.ny && pw.nx == ps.nx;
  const bool z_slab = fo.ny == 0 && fo.nx == 0 && fw.ny == fs.ny && fw.nx == fs.nx;
  if (whole_parent && z_slab && fs.nx == 2 * ps.nx && fs.nx % (2 * UQ) == 0 && ((uintptr_t)fine & 15) == 0) {
    const int pz0 = fo.nz >> 1, pz1 = (fo.nz + fw.nz + 1) >> 1;
    dim3 grid((ps.nx / UQ + BX - 1) / BX, (ps.ny + BY - 1) / BY, (pz1 - pz0 + UZ - 1) / UZ);
    upsample4_kernel<<<grid, kBlock3, 0, (cudaStream_t)stream>>>(parent, ps, fine, fs, fo.nz, fo.nz + fw.nz);
  } else {
    launch_upsample(parent, ps, po, pw, fine, fs, fo, fw, (cudaStream_t)stream);
  }
  RWB_LAUNCH_CHECK("upsample_kernel (window)");
  count_launches(1);
  return RWB_OK;
}

extern "C" int rwb_edge_weights_f32(int32_t ndim, const int64_t* size, const float* volume, float beta,
                                    float min_weight, float* weights, void* stream) {
  Shape3 s;
  int rc = shape_from(ndim, size, &s);
  if (rc) return rc;
  if (!volume || !weights) return fail(RWB_ERR_INVALID, "null pointer");
  if (!(beta >= 0.0f) || !(min_weight >= 0.0f)) return fail(RWB_ERR_INVALID, "beta and min_weight must be >= 0");
  edge_weights_kernel<<<grid3(s), kBlock3, 0, (cudaStream_t)stream>>>(volume, s, ndim, beta,
                                                                                     min_weight, weights);
  RWB_LAUNCH_CHECK("edge_weights_kernel");
  count_launches(1);
  return RWB_OK;
}

extern "C" int rwb_labels_u8(int64_t n, const float* prob, uint8_t* labels, void* stream) {
  if (n < 0) return fail(RWB_ERR_INVALID, "negative length");
  if (n == 0) return RWB_OK;
  if (!prob || !labels) return fail(RWB_ERR_INVALID, "null pointer");
  labels_kernel<<<ceil_div_u(n, 256), 256, 0, (cudaStream_t)stream>>>(prob, n, labels);
  RWB_LAUNCH_CHECK("labels_kernel");
  count_launches(1);
  return RWB_OK;
}
