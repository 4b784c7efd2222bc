// Brick-batched Jacobi-PCG random-walker solve of one pyramid level.
//
// Every brick of a level is an independent Dirichlet problem (oracle/rw.py,
// DESIGN.md §3).  All listed bricks are solved together, in lockstep, with
// per-brick CG scalars: one launch per CG pass covers every unconverged
// brick, so the GPU stays full while bricks converge at different
// iteration counts.
//
// The system is solved in Jacobi-scaled form: with s_i = diag_i^-1/2,
// A' = S L_UU S has unit diagonal, off-diagonals -w'_ij = -w_ij s_i s_j, and
// CG on A' y = S b is Jacobi-PCG on L_UU x = b with x = S y.  The scaled
// forward weights w' are zero on every edge that leaves the brick or touches
// a Dirichlet node, so the block-diagonal operator needs no brick masks in
// the iteration and no preconditioner array.
//
// Workspace (brick-local, each brick padded to the full brick box, brick
// `slot` at offset slot*bvol, x fastest):
//   y, r, p[2], q, w'x, w'y, w'z, s   (f32)   -> 36 B/voxel (3D), 32 B (2D)
// Per CG iteration and unknown, HBM traffic is
//   pass 1: read r, p_in, w'x, w'y, w'z; write p_out, q   (28 B; 2D: 24 B)
//   pass 2: read y, r, p_out, q;        write y, r        (24 B)
// = 52 B (3D) / 48 B (2D) of algorithmic bytes.
//
// Per-brick reductions are deterministic: each CTA writes one partial, the
// last CTA of a brick to finish (atomic ticket) sums the partials in a fixed
// order in float64.  Results are therefore independent of which other bricks
// share the launch (multi-GPU sharding gives bit-identical bytes).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace rwb {

constexpr int TX = 32;  // threads along x (one warp per row segment)
constexpr int TY = 8;   // threads along y
constexpr int TZ = 8;   // z extent marched by each thread
constexpr int NTHREADS = TX * TY;

struct Work {
  float *y, *r, *p0, *p1, *q, *wx, *wy, *wz, *sc;
  double* rr;  // [2][nb]
  double* pq;  // [nb]
  double* bb;  // [nb]
  int* state;  // [nb]
  int* iters;  // [nb]
  unsigned* unk;     // [nb] unknowns per brick
  unsigned* ticket;  // [nb]
  float2* part;      // [nb*tiles]
  int* alist;        // [nb] compacted active slots
  int* base_it;      // [1]  iteration count at the start of the current graph chunk
  int* n_active;     // [1]
  unsigned long long* unknowns;  // [1]
  int* stat_i;       // [8] device stats scratch
  unsigned long long* stamp;  // [2] %globaltimer (ns) around the solve launches
  int* next;                  // [1] dynamic brick counter of the resident 3-D engine
};

// ---------------------------------------------------------------------------
// brick/tile addressing

struct TileCtx {
  int slot, brick, tile;
  int hz, hy, hx;       // brick coords
  int gz0, gy0, gx0;    // global coords of brick-local (0,0,0)
  int lz0, lz1, ly, lx; // this thread's column and z range (local)
  bool col;             // column inside the brick box
};

template <int TZv = TZ>
__device__ __forceinline__ TileCtx tile_ctx(const Geo& g, const int* __restrict__ list, int slot, int tile) {
  TileCtx c;
  c.slot = slot;
  c.tile = tile;
  c.brick = list ? list[slot] : slot;
  c.hx = c.brick % g.gx;
  int t = c.brick / g.gx;
  c.hy = t % g.gy;
  c.hz = t / g.gy;
  c.gz0 = g.oz + c.hz * g.bz;
  c.gy0 = g.oy + c.hy * g.by;
  c.gx0 = g.ox + c.hx * g.bx;
  int ttx = tile % g.tx;
  int tt = tile / g.tx;
  int tty = tt % g.ty;
  int ttz = tt / g.ty;
  c.lx = ttx * TX + threadIdx.x;
  c.ly = tty * TY + threadIdx.y;
  c.lz0 = ttz * TZv;
  c.lz1 = min(c.lz0 + TZv, g.bz);
  c.col = c.lx < g.bx && c.ly < g.by;
  return c;
}

// one CTA per (slot, tile) for the non-iterative kernels
__device__ __forceinline__ TileCtx tile_ctx(const Geo& g, const int* __restrict__ list) {
  int slot = blockIdx.x / g.tiles;
  return tile_ctx(g, list, slot, blockIdx.x - slot * g.tiles);
}

// setup kernels: one voxel per thread (tiles of a single z plane) for more
// independent loads in flight; `setup_tiles(g)` tiles per brick
constexpr int STZ = 4;  // z extent marched per setup thread
__device__ __host__ __forceinline__ int setup_tiles(const Geo& g) { return ((g.bz + STZ - 1) / STZ) * g.ty * g.tx; }

__device__ __forceinline__ TileCtx setup_ctx(const Geo& g, const int* __restrict__ list) {
  const int st = setup_tiles(g);
  int slot = blockIdx.x / st;
  return tile_ctx<STZ>(g, list, slot, blockIdx.x - slot * st);
}

// block-wide sum of two floats -> thread 0
__device__ __forceinline__ float2 block_sum2(float a, float b) {
  __shared__ float2 warp_part[NTHREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if ((tid & 31) == 0) warp_part[tid >> 5] = make_float2(a, b);
  __syncthreads();
  float2 s = make_float2(0.f, 0.f);
  if (tid == 0) {
#pragma unroll
    for (int w = 0; w < NTHREADS / 32; ++w) {
      s.x += warp_part[w].x;
      s.y += warp_part[w].y;
    }
  }
  return s;
}

// Publish this CTA's partial; the last CTA of the brick reduces all partials
// (fixed order, float64).  Must be called by all threads of the CTA.  Returns
// true in exactly one thread (thread 0 of the brick's last CTA), which then
// holds the brick totals in *sum0 / *sum1.  Ends with a CTA barrier so the
// shared scratch can be reused by the next work item.
__device__ __forceinline__ bool brick_reduce(const Geo& g, const Work& w, int slot, int tile, float a, float b,
                                             double* sum0, double* sum1, int ntiles = -1) {
  const int tiles = ntiles > 0 ? ntiles : g.tiles;
  __shared__ bool last;
  float2 s = block_sum2(a, b);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  bool mine = false;
  if (tiles == 1) {
    if (tid == 0) {
      *sum0 = (double)s.x;
      *sum1 = (double)s.y;
      mine = true;
    }
    __syncthreads();
    return mine;
  }
  if (tid == 0) {
    w.part[(long long)slot * tiles + tile] = s;
    __threadfence();
    unsigned t = atomicAdd(&w.ticket[slot], 1u);
    last = (t == (unsigned)tiles - 1);
  }
  __syncthreads();
  if (last && tid < 32) {
    __threadfence();
    double sa = 0.0, sb = 0.0;
    const float2* p = w.part + (long long)slot * tiles;
    for (int i = tid; i < tiles; i += 32) {
      float2 v = __ldcg(p + i);
      sa += (double)v.x;
      sb += (double)v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
      sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (tid == 0) {
      *sum0 = sa;
      *sum1 = sb;
      w.ticket[slot] = 0;
      mine = true;
    }
  }
  __syncthreads();
  return mine;
}

// ---------------------------------------------------------------------------
// setup

__device__ __forceinline__ float seed_value(uint8_t s) { return s == 1 ? 1.0f : 0.0f; }

// Shared by both setups (bit-identical systems).  s = diag^-1/2 by MUFU.RSQ
// (~1 ulp; the float64 oracle is matched to the solve tolerance, not bits);
// r0 = s (b + acc - diag x0); y0 = x0 / s = x0 diag s.
__device__ __forceinline__ float jacobi_scale(float d) {  // d >= w_min > 0: no denormal path needed
  float s;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(d));
  return s;
}
__device__ __forceinline__ float initial_residual(float si, float b, float acc, float diag, float x0) {
  return si * fmaf(-diag, x0, b + acc);
}
__device__ __forceinline__ float initial_y(float x0, float si, float diag) { return x0 * (diag * si); }

// Neighbour addressing of one voxel for the setup kernels: the six neighbours in
// the order -z,+z,-y,+y,-x,+x, whether each is in the level and in the brick,
// and clamped (always valid) level / brick-local indices, so every neighbour
// load can be issued unconditionally and in parallel.
struct Nbrs {
  long long g[6];   // level index (clamped to the voxel itself when outside)
  long long l[6];   // brick-local index (clamped likewise)
  bool lev[6];      // neighbour inside the level
  bool brk[6];      // ... and inside this brick
};

__device__ __forceinline__ Nbrs neighbours(const Geo& g, long long gi, long long li, int gz, int gy, int gx, int lz,
                                           int ly, int lx) {
  Nbrs n;
  const long long sbz = (long long)g.by * g.bx;
  const long long dg[6] = {-g.sxy, g.sxy, -(long long)g.nx, (long long)g.nx, -1, 1};
  const long long dl[6] = {-sbz, sbz, -(long long)g.bx, (long long)g.bx, -1, 1};
  const bool lev[6] = {g.is3d && gz > 0, g.is3d && gz + 1 < g.nz, gy > 0, gy + 1 < g.ny, gx > 0, gx + 1 < g.nx};
  const bool brk[6] = {lz > 0, lz + 1 < g.bz, ly > 0, ly + 1 < g.by, lx > 0, lx + 1 < g.bx};
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    n.lev[e] = lev[e];
    n.brk[e] = lev[e] && brk[e];
    n.g[e] = lev[e] ? gi + dg[e] : gi;
    n.l[e] = n.brk[e] ? li + dl[e] : li;
  }
  return n;
}

// K1: scale s = diag^-1/2 for unknowns, 0 for seeds / padding / isolated voxels.
// The diagonal sums the six edge weights in the order -z,+z,-y,+y,-x,+x
// (the brick-resident engine and the oracle use the same order).
__global__ void __launch_bounds__(NTHREADS) setup_scale_kernel(Geo g, Work w, const int* __restrict__ list,
                                                               const float* __restrict__ I,
                                                               const uint8_t* __restrict__ S, float beta,
                                                               float wmin) {
  TileCtx c = setup_ctx(g, list);
  if (!c.col) return;
  const int gy = c.gy0 + c.ly, gx = c.gx0 + c.lx;
  const bool colin = gy >= 0 && gy < g.ny && gx >= 0 && gx < g.nx;
  const long long sbz = (long long)g.by * g.bx;
  float* __restrict__ sc = w.sc;
  const long long lbase = (long long)c.slot * g.bvol + (long long)c.ly * g.bx + c.lx;
#pragma unroll
  for (int k = 0; k < STZ; ++k) {
    const int lz = c.lz0 + k;
    if (lz >= c.lz1) break;
    const long long li = lbase + (long long)lz * sbz;
    const int gz = c.gz0 + lz;
    float s = 0.f;
    if (colin && gz >= 0 && gz < g.nz) {
      const long long gi = (long long)gz * g.sxy + (long long)gy * g.nx + gx;
      const Nbrs n = neighbours(g, gi, li, gz, gy, gx, lz, c.ly, c.lx);
      const float ci = __ldg(I + gi);
      float In[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) In[e] = __ldg(I + n.g[e]);
      if (__ldg(S + gi) == 0) {
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < 6; ++e) d += n.lev[e] ? edge_weight(ci, In[e], beta, wmin) : 0.f;
        s = d > 0.f ? jacobi_scale(d) : 0.f;
      }
    }
    sc[li] = s;
  }
}



// K2: scaled forward weights, r0 = S(b - L x0), y0 = x0 / s, (p = 0); per-brick
// ||S b||^2 and ||r0||^2 and the brick's initial decision.
__global__ void __launch_bounds__(NTHREADS) setup_system_kernel(Geo g, Work w, const int* __restrict__ list,
                                                                const float* __restrict__ I,
                                                                const uint8_t* __restrict__ S,
                                                                const float* __restrict__ bound, float beta,
                                                                float wmin, float tol2, int max_iter,
                                                                int write_p) {
  TileCtx c = setup_ctx(g, list);
  float acc_bb = 0.f, acc_rr = 0.f;
  unsigned n_unknown = 0;
  if (c.col) {
    const int gy = c.gy0 + c.ly, gx = c.gx0 + c.lx;
    const bool colin = gy >= 0 && gy < g.ny && gx >= 0 && gx < g.nx;
    const long long sbz = (long long)g.by * g.bx;
    const float* __restrict__ sc = w.sc;
    float* __restrict__ wx = w.wx;
    float* __restrict__ wy = w.wy;
    float* __restrict__ wz = w.wz;
    float* __restrict__ rv = w.r;
    float* __restrict__ yv = w.y;
    const long long lbase = (long long)c.slot * g.bvol + (long long)c.ly * g.bx + c.lx;
#pragma unroll
    for (int k = 0; k < STZ; ++k) {
      const int lz = c.lz0 + k;
      if (lz >= c.lz1) break;
      const long long li = lbase + (long long)lz * sbz;
      const int gz = c.gz0 + lz;
      const float si = sc[li];
      float wf[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, r = 0.f, y = 0.f;
      if (si > 0.f && colin && gz >= 0 && gz < g.nz) {
        ++n_unknown;
        const long long gi = (long long)gz * g.sxy + (long long)gy * g.nx + gx;
        const Nbrs n = neighbours(g, gi, li, gz, gy, gx, lz, c.ly, c.lx);
        const float ci = __ldg(I + gi);
        const float x0 = bound ? __ldg(bound + gi) : 0.f;
        float In[6], Bn[6], Sc[6];
        uint8_t Sn[6];
#pragma unroll
        for (int e = 0; e < 6; ++e) {  // all neighbour loads issued together
          In[e] = __ldg(I + n.g[e]);
          Sn[e] = __ldg(S + n.g[e]);
          Bn[e] = bound ? __ldg(bound + n.g[e]) : 0.f;
          Sc[e] = sc[n.l[e]];
        }
        float diag = 0.f, b = 0.f, acc = 0.f;
#pragma unroll
        for (int e = 0; e < 6; ++e) {
          if (!n.lev[e]) continue;
          const float wt = edge_weight(ci, In[e], beta, wmin);
          diag += wt;
          const float sn = n.brk[e] ? Sc[e] : 0.f;
          if (sn > 0.f) {  // coupled unknown of this brick
            acc = fmaf(wt, Bn[e], acc);
            wf[e] = wt * si * sn;
          } else {  // Dirichlet: seed, or outside the brick
            b = fmaf(wt, Sn[e] ? seed_value(Sn[e]) : Bn[e], b);
          }
        }
        r = initial_residual(si, b, acc, diag, x0);
        y = initial_y(x0, si, diag);
        const float sb = si * b;
        acc_bb = fmaf(sb, sb, acc_bb);
        acc_rr = fmaf(r, r, acc_rr);
      } else if (colin && gz >= 0 && gz < g.nz) {
        // not an unknown: y holds the voxel's final value (seed value, else bound),
        // which no CG path changes (its r, p, s, w stay exactly 0)
        const long long gi = (long long)gz * g.sxy + (long long)gy * g.nx + gx;
        const uint8_t sv = __ldg(S + gi);
        y = sv ? seed_value(sv) : (bound ? __ldg(bound + gi) : 0.f);
      }
      wx[li] = wf[5];
      wy[li] = wf[3];
      if (g.is3d) wz[li] = wf[1];
      rv[li] = r;
      yv[li] = y;
      if (write_p) w.p0[li] = 0.f;  // only the streaming passes read p
    }
  }
  {
    __shared__ unsigned cta_unknown;
    if (threadIdx.x == 0 && threadIdx.y == 0) cta_unknown = 0;
    __syncthreads();
    if (n_unknown) atomicAdd(&cta_unknown, n_unknown);
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0 && cta_unknown) {
      atomicAdd(w.unknowns, (unsigned long long)cta_unknown);
      atomicAdd(w.unk + c.slot, cta_unknown);
    }
  }
  double bb, rr;
  if (brick_reduce(g, w, c.slot, c.tile, acc_bb, acc_rr, &bb, &rr, setup_tiles(g))) {
    w.bb[c.slot] = bb;
    w.rr[c.slot] = rr;  // parity 0
    int st = ST_ACTIVE;
    if (bb <= 0.0)
      st = ST_ZERO;  // no Dirichlet coupling: the exact solution is 0
    else if (rr <= (double)tol2 * bb)
      st = ST_CONVERGED;
    else if (max_iter <= 0)
      st = ST_MAXITER;
    w.state[c.slot] = st;
    w.iters[c.slot] = 0;
  }
}

// ---------------------------------------------------------------------------
// Fused setup, one CTA per brick (brick x, y extents <= 32, x a multiple of 4):
// thread (xq, ly) owns a row quad of 4 x-voxels and marches z.  The two setup
// kernels above compute all six edge weights of every voxel twice (12
// exponentials) and exchange the scale factors through HBM; here each voxel
// computes its forward x/y/z and backward y weights (4 exponentials; backward
// x comes from the quad neighbour, backward z from the previous plane), the
// scale factors and Dirichlet values of plane a are computed one plane ahead
// of the system of plane a-1 and reach the y / quad-edge neighbours through
// shared memory.  Same arithmetic, same summation order (-z,+z,-y,+y,-x,+x) and
// the same reduction order for ||S b||^2 and ||r0||^2 as setup_scale /
// setup_system, so the outputs are bit-identical.
//
// Inputs arrive by TMA: for every plane, one elected thread loads the tile of
// intensity, bound and seeds that covers the brick's plane plus its one-voxel
// x/y halo (the x start rounded down to 16 B: TMA tile boxes must start 16 B
// aligned), out-of-level parts zero-filled by the tensor map, into a ring of
// SR stages, each completing on its own mbarrier, SR-4 planes ahead of use.
// Quads make every shared-memory access and global store 16 B wide and spread
// the per-plane bookkeeping over 4 voxels; two CTAs fit on an SM.
constexpr int FB = 32;                 // max brick extent in x and y for the fused setup
constexpr int SQ = 4;                  // x voxels per thread
constexpr int SQN = FB / SQ;           // quads per row
constexpr int STH = SQN * FB;          // threads per CTA
constexpr int SR = 6;                  // ring stages (planes)
constexpr int SRX = 40, SRY = FB + 2;  // f32 tile box: x [gx0-4, gx0+36), y [gy0-1, gy0+33)
constexpr int SRXS = 64;               // u8 seed tile box: x [gx0-16, gx0+48)
constexpr int SRX0 = 4, SRXS0 = 16;    // tile column of x = gx0
constexpr int SR_F32 = ((SRX * SRY * 4 + 127) / 128) * 128;  // bytes per f32 stage (128 B aligned)
constexpr int SR_U8 = ((SRXS * SRY + 127) / 128) * 128;
constexpr int SPX = 4, SPW = FB + 8;   // padded Sc / Dv rows: column SPX + x, halo at SPX-1 and SPX+bx
constexpr int SETUP_MAX_TILES = 256;   // (bz / STZ) * (by / TY) tiles of the two-kernel reduction order

struct SetupSmem {
  float I[SR][SR_F32 / 4];
  float B[SR][SR_F32 / 4];
  unsigned char S[SR][SR_U8];
  unsigned long long bar[SR];
  // per plane (2 alternating): scale factors and Dirichlet values (seed value,
  // else bound) with a one-voxel halo; Sc's halo stays 0 (cross-brick = never coupled)
  __align__(16) float Sc[2][SRY][SPW];
  __align__(16) float Dv[2][SRY][SPW];
  float2 rowpart[FB];             // per-row sums of the current 4-plane chunk
  float2 tpart[SETUP_MAX_TILES];  // per setup-tile sums, in setup_system_kernel's tile order
  unsigned red_unk[STH / 32];
};

struct SetupMaps {
  CUtensorMap I, B, S;  // 3-D tiled maps over the level (x fastest)
};

__device__ __forceinline__ void setup_tma_plane(const SetupMaps& m, SetupSmem& sm, bool has_b, int stage, int gx0,
                                                int y, int z) {
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar[stage]);
  const uint32_t bytes = (has_b ? 2u : 1u) * (SRX * SRY * 4) + SRXS * SRY;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  int x = gx0 - SRX0;
  auto load = [&](const CUtensorMap* map, void* dst) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
  };
  load(&m.I, sm.I[stage]);
  if (has_b) load(&m.B, sm.B[stage]);
  x = gx0 - SRXS0;
  load(&m.S, sm.S[stage]);
}

__device__ __forceinline__ void setup_wait(SetupSmem& sm, int stage, uint32_t parity) {
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&sm.bar[stage]);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra.uni WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float q4(const float4& v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

__global__ void __launch_bounds__(STH, 2) setup_brick_kernel(const __grid_constant__ SetupMaps maps, Geo g, Work w,
                                                             const int* __restrict__ list, bool has_b, float beta,
                                                             float wmin, float tol2, int max_iter, int write_p) {
  extern __shared__ __align__(128) unsigned char setup_smem_raw[];
  SetupSmem& sm = *reinterpret_cast<SetupSmem*>(setup_smem_raw);
  const int slot = blockIdx.x;
  const int brick = list ? list[slot] : slot;
  const int hx = brick % g.gx, hy = (brick / g.gx) % g.gy, hz = brick / (g.gx * g.gy);
  const int gz0 = g.oz + hz * g.bz, gy0 = g.oy + hy * g.by, gx0 = g.ox + hx * g.bx;
  const int tid = threadIdx.x;
  const int xq = tid % SQN, ly = tid / SQN;
  const int lx0 = xq * SQ;  // brick-local x of voxel 0 of the quad
  const int gy = gy0 + ly;
  const bool col = lx0 < g.bx && ly < g.by;  // quads lie wholly inside or outside (bx % 4 == 0)
  const bool rowin = gy >= 0 && gy < g.ny;
  const bool fxm = lx0 == 0, fxp = lx0 + SQ == g.bx, fym = ly == 0, fyp = ly + 1 == g.by;  // brick-face lanes
  const bool eym = gy > 0, eyp = gy + 1 < g.ny;
  bool colin[SQ], exm[SQ], exp_[SQ];
#pragma unroll
  for (int i = 0; i < SQ; ++i) {
    const int gx = gx0 + lx0 + i;
    colin[i] = col && rowin && gx >= 0 && gx < g.nx;
    exm[i] = gx > 0;
    exp_[i] = gx + 1 < g.nx;
  }
  const long long sbz = (long long)g.by * g.bx;
  const long long lcol = (long long)slot * g.bvol + (long long)ly * g.bx + lx0;
  auto wgt = [&](float a, float b) { return edge_weight(a, b, beta, wmin); };
  // plane p in [-1, bz] lives in stage (p + 1) % SR, use (p + 1) / SR; tile row ty = voxel y gy0-1+ty
  auto stage_of = [](int p) { return (p + 1) % SR; };
  auto rowI = [&](int p, int dy) { return &sm.I[stage_of(p)][(ly + 1 + dy) * SRX + SRX0 + lx0]; };
  auto rowB = [&](int p, int dy) { return &sm.B[stage_of(p)][(ly + 1 + dy) * SRX + SRX0 + lx0]; };
  auto ldI4 = [&](int p, int dy) { return *reinterpret_cast<const float4*>(rowI(p, dy)); };
  auto ldB4 = [&](int p, int dy) {
    return has_b ? *reinterpret_cast<const float4*>(rowB(p, dy)) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto ldS4 = [&](int p, int dy) {  // the quad's 4 seed bytes
    return *reinterpret_cast<const unsigned*>(&sm.S[stage_of(p)][(ly + 1 + dy) * SRXS + SRXS0 + lx0]);
  };
  auto sbyte = [](unsigned s4, int i) { return (s4 >> (8 * i)) & 0xffu; };
  auto dval1 = [](unsigned s, float b) { return s ? seed_value((uint8_t)s) : b; };  // Dirichlet value
  auto dval4 = [&](int p, int dy) {
    const unsigned s4 = ldS4(p, dy);
    const float4 b4 = ldB4(p, dy);
    return make_float4(dval1(sbyte(s4, 0), b4.x), dval1(sbyte(s4, 1), b4.y), dval1(sbyte(s4, 2), b4.z),
                       dval1(sbyte(s4, 3), b4.w));
  };
  auto dval_x = [&](int p, int dx) {  // x halo voxel (dx = -1 or 4) of the quad's row
    const unsigned s = sm.S[stage_of(p)][(ly + 1) * SRXS + SRXS0 + lx0 + dx];
    return dval1(s, has_b ? rowB(p, 0)[dx] : 0.f);
  };
  auto wait_plane = [&](int p) { setup_wait(sm, stage_of(p), (uint32_t)(((p + 1) / SR) & 1)); };
  const int last = g.bz;  // planes -1 .. bz are loaded

  if (tid == 0) {
    for (int s = 0; s < SR; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&sm.bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int p = -1; p <= min(last, SR - 4); ++p) setup_tma_plane(maps, sm, has_b, stage_of(p), gx0, gy0 - 1, gz0 + p);
  }
  for (int i = tid; i < 2 * SRY * SPW; i += STH) {
    (&sm.Sc[0][0][0])[i] = 0.f;
    (&sm.Dv[0][0][0])[i] = 0.f;
  }
  __syncthreads();
  wait_plane(-1);
  wait_plane(0);

  // system-step (plane z = a-1) registers: its weights, scale factors and
  // Dirichlet values of the own quad at z-1 and z
  float z_wxf[SQ], z_wyf[SQ], z_wzf[SQ], z_wxb[SQ], z_wyb[SQ], z_wzb[SQ];
  float sc_zm[SQ], sc_z[SQ], dv_zm[SQ], dv_z[SQ];
  float acc_bb[SQ], acc_rr[SQ];
  {
    const float4 dm = dval4(-1, 0);
#pragma unroll
    for (int i = 0; i < SQ; ++i) {
      z_wxf[i] = z_wyf[i] = z_wzf[i] = z_wxb[i] = z_wyb[i] = z_wzb[i] = 0.f;
      sc_zm[i] = sc_z[i] = dv_zm[i] = 0.f;
      dv_z[i] = q4(dm, i);
      acc_bb[i] = acc_rr[i] = 0.f;
    }
  }
  unsigned n_unknown = 0;
  // ||S b||^2 and ||r0||^2 are reduced in exactly the order of setup_system_kernel
  // (per voxel over a 4-plane chunk, xor tree over the 32 x of a row, 8 rows in
  // sequence per tile, tiles in float64 by brick_reduce), so both setups give
  // the same bits and the CG that starts from them the same trajectory.
  const int ty8 = (g.by + TY - 1) / TY;
  int pending_chunk = -1;
  auto tile_sums = [&]() {  // after a barrier: rows of the flushed chunk -> its tiles
    if (pending_chunk >= 0 && tid < ty8) {
      float2 s = make_float2(0.f, 0.f);
      for (int r8 = 0; r8 < TY; ++r8) {
        s.x += sm.rowpart[tid * TY + r8].x;
        s.y += sm.rowpart[tid * TY + r8].y;
      }
      sm.tpart[pending_chunk * ty8 + tid] = s;
    }
    if (pending_chunk >= 0) __syncthreads();  // rowpart free for the next flush (uniform branch)
    pending_chunk = -1;
  };

#pragma unroll 2
  for (int a = 0; a <= g.bz; ++a) {
    tile_sums();
    const int gza = gz0 + a;
    const bool pa_in = a < g.bz;
    const bool zin = gza >= 0 && gza < g.nz;
    // refill: plane a+SR-3 replaces plane a-3, whose last reader (step a-1) every thread has left
    if (tid == 0 && a + SR - 3 <= last)
      setup_tma_plane(maps, sm, has_b, stage_of(a + SR - 3), gx0, gy0 - 1, gz0 + a + SR - 3);
    if (a + 1 <= last) wait_plane(a + 1);
    // ---------------- phase 1: weights, scale and Dirichlet values of plane a ----------------
    float sca[SQ], wxf[SQ], wyf[SQ], wzf[SQ], wxb[SQ], wyb[SQ], wzb[SQ];
    const float4 dva4 = dval4(a, 0);
    float dva[SQ] = {dva4.x, dva4.y, dva4.z, dva4.w};
#pragma unroll
    for (int i = 0; i < SQ; ++i) sca[i] = wxf[i] = wyf[i] = wzf[i] = wxb[i] = wyb[i] = wzb[i] = 0.f;
    if (pa_in) {
      const int ab = a & 1;
      if (col && rowin && zin) {
        const float4 I4 = ldI4(a, 0), Iy4 = ldI4(a, 1), Iym4 = ldI4(a, -1), Iz4 = ldI4(a + 1, 0);
        const float Ixr = rowI(a, 0)[SQ], Ixl = rowI(a, 0)[-1];
        const unsigned s4 = ldS4(a, 0);
        const bool haszp = g.is3d && gza + 1 < g.nz, haszm = g.is3d && gza > 0;
        float4 Izm4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a == 0 && haszm) Izm4 = ldI4(-1, 0);
        // branch-free: every lane computes all four voxels (tile values are
        // finite, zero outside the level) and masks the voxels outside the level
#pragma unroll
        for (int i = 0; i < SQ; ++i) {
          const float Ii = q4(I4, i);
          const float Ixp = i + 1 < SQ ? q4(I4, i + 1) : Ixr;
          const float fx = wgt(Ii, Ixp);
          wxf[i] = colin[i] && exp_[i] ? fx : 0.f;
          wyf[i] = colin[i] && eyp ? wgt(Ii, q4(Iy4, i)) : 0.f;
          wzf[i] = colin[i] && haszp ? wgt(Ii, q4(Iz4, i)) : 0.f;
          wxb[i] = colin[i] && exm[i] ? (i > 0 ? wxf[i - 1] : wgt(Ii, Ixl)) : 0.f;
          wyb[i] = colin[i] && eym ? wgt(Ii, q4(Iym4, i)) : 0.f;
          wzb[i] = colin[i] && haszm ? (a > 0 ? z_wzf[i] : wgt(Ii, q4(Izm4, i))) : 0.f;
          const float d = ((((wzb[i] + wzf[i]) + wyb[i]) + wyf[i]) + wxb[i]) + wxf[i];
          sca[i] = (colin[i] && sbyte(s4, i) == 0 && d > 0.f) ? jacobi_scale(d) : 0.f;
        }
        *reinterpret_cast<float4*>(&sm.Sc[ab][ly + 1][SPX + lx0]) = make_float4(sca[0], sca[1], sca[2], sca[3]);
      }
      *reinterpret_cast<float4*>(&sm.Dv[ab][ly + 1][SPX + lx0]) = dva4;
      if (fxm) sm.Dv[ab][ly + 1][SPX - 1] = dval_x(a, -1);  // x / y halo of the brick face lanes
      if (fxp) sm.Dv[ab][ly + 1][SPX + g.bx] = dval_x(a, SQ);
      if (fym) *reinterpret_cast<float4*>(&sm.Dv[ab][0][SPX + lx0]) = dval4(a, -1);
      if (fyp) *reinterpret_cast<float4*>(&sm.Dv[ab][ly + 2][SPX + lx0]) = dval4(a, 1);
    }
    // ---------------- phase 2: the system of plane z = a-1 ----------------
    const int z = a - 1;
    if (z >= 0) {
      const bool vrow = col && rowin && gz0 + z >= 0 && gz0 + z < g.nz;
      const long long li = lcol + (long long)z * sbz;
      float wfx[SQ], wfy[SQ], wfz[SQ], r[SQ], y[SQ], scw[SQ];
      const int zb = z & 1;
      const float4 scm = *reinterpret_cast<const float4*>(&sm.Sc[zb][ly][SPX + lx0]);
      const float4 scp = *reinterpret_cast<const float4*>(&sm.Sc[zb][ly + 2][SPX + lx0]);
      const float4 dvm = *reinterpret_cast<const float4*>(&sm.Dv[zb][ly][SPX + lx0]);
      const float4 dvp = *reinterpret_cast<const float4*>(&sm.Dv[zb][ly + 2][SPX + lx0]);
      const float scl = sm.Sc[zb][ly + 1][SPX + lx0 - 1], scr = sm.Sc[zb][ly + 1][SPX + lx0 + SQ];
      const float dvl = sm.Dv[zb][ly + 1][SPX + lx0 - 1], dvr = sm.Dv[zb][ly + 1][SPX + lx0 + SQ];
      const float4 xb4 = ldB4(z, 0);
#pragma unroll
      for (int i = 0; i < SQ; ++i) {
        const bool vz = vrow && colin[i];
        scw[i] = vz ? sc_z[i] : 0.f;
        // branch-free: computed for every voxel, kept for the unknowns (sc > 0)
        const bool unk = vz && sc_z[i] > 0.f;
        n_unknown += unk;
        {
          const float si = sc_z[i], x0 = q4(xb4, i);
          float diag = 0.f, b = 0.f, acc = 0.f;
          // One neighbour, branch-free: a missing neighbour has weight 0 (phase
          // 1), which adds exact zeros, so the non-zero terms are summed in the
          // same order as setup_system_kernel's skipping loop.  A coupled
          // neighbour is an unknown, so its Dirichlet value is its bound.
          auto visit = [&](float wt, float sn, float dv) {
            diag += wt;
            const bool coupled = sn > 0.f;
            acc = coupled ? fmaf(wt, dv, acc) : acc;
            b = coupled ? b : fmaf(wt, dv, b);
            return coupled ? wt * si * sn : 0.f;
          };
          visit(z_wzb[i], z > 0 ? sc_zm[i] : 0.f, dv_zm[i]);
          const float fz = visit(z_wzf[i], z + 1 < g.bz ? sca[i] : 0.f, dva[i]);
          visit(z_wyb[i], q4(scm, i), q4(dvm, i));
          const float fy = visit(z_wyf[i], q4(scp, i), q4(dvp, i));
          visit(z_wxb[i], i > 0 ? sc_z[i - 1] : scl, i > 0 ? dv_z[i - 1] : dvl);
          const float fx = visit(z_wxf[i], i + 1 < SQ ? sc_z[i + 1] : scr, i + 1 < SQ ? dv_z[i + 1] : dvr);
          const float ri = initial_residual(si, b, acc, diag, x0);
          const float sb = si * b;
          wfx[i] = unk ? fx : 0.f;
          wfy[i] = unk ? fy : 0.f;
          wfz[i] = unk ? fz : 0.f;
          r[i] = unk ? ri : 0.f;
          // not an unknown: y holds the voxel's final value (seed value, else bound)
          y[i] = unk ? initial_y(x0, si, diag) : (vz ? dv_z[i] : 0.f);
          acc_bb[i] = unk ? fmaf(sb, sb, acc_bb[i]) : acc_bb[i];
          acc_rr[i] = unk ? fmaf(ri, ri, acc_rr[i]) : acc_rr[i];
        }
      }
      if (z % STZ == STZ - 1 || z == g.bz - 1) {  // chunk complete: row sums in the xor-tree order
        float bb[SQ], rr[SQ];
#pragma unroll
        for (int i = 0; i < SQ; ++i) {
          bb[i] = acc_bb[i];
          rr[i] = acc_rr[i];
#pragma unroll
          for (int o = SQN / 2; o > 0; o >>= 1) {  // x ^ 16, 8, 4 = quad ^ 4, 2, 1
            bb[i] += __shfl_xor_sync(0xffffffffu, bb[i], o);
            rr[i] += __shfl_xor_sync(0xffffffffu, rr[i], o);
          }
          acc_bb[i] = acc_rr[i] = 0.f;
        }
        // x ^ 2, then x ^ 1, inside the quad
        const float b0 = bb[0] + bb[2], b1 = bb[1] + bb[3], r0 = rr[0] + rr[2], r1 = rr[1] + rr[3];
        if (xq == 0) sm.rowpart[ly] = make_float2(b0 + b1, r0 + r1);
        pending_chunk = z / STZ;
      }
      if (col) {
        *reinterpret_cast<float4*>(w.wx + li) = make_float4(wfx[0], wfx[1], wfx[2], wfx[3]);
        *reinterpret_cast<float4*>(w.wy + li) = make_float4(wfy[0], wfy[1], wfy[2], wfy[3]);
        if (g.is3d) *reinterpret_cast<float4*>(w.wz + li) = make_float4(wfz[0], wfz[1], wfz[2], wfz[3]);
        *reinterpret_cast<float4*>(w.r + li) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<float4*>(w.y + li) = make_float4(y[0], y[1], y[2], y[3]);
        *reinterpret_cast<float4*>(w.sc + li) = make_float4(scw[0], scw[1], scw[2], scw[3]);
        if (write_p) *reinterpret_cast<float4*>(w.p0 + li) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    // rotate: plane a becomes plane z of the next system step
#pragma unroll
    for (int i = 0; i < SQ; ++i) {
      z_wxf[i] = wxf[i], z_wyf[i] = wyf[i], z_wzf[i] = wzf[i];
      z_wxb[i] = wxb[i], z_wyb[i] = wyb[i], z_wzb[i] = wzb[i];
      sc_zm[i] = sc_z[i];
      sc_z[i] = sca[i];
      dv_zm[i] = dv_z[i];
      dv_z[i] = dva[i];
    }
    __syncthreads();
  }
  // per-brick ||S b||^2, ||r0||^2 (brick_reduce's order) and the brick's initial decision
  tile_sums();
  const unsigned nu = __reduce_add_sync(0xffffffffu, n_unknown);
  if ((tid & 31) == 0) sm.red_unk[tid >> 5] = nu;
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    const int tiles = ((g.bz + STZ - 1) / STZ) * ty8;
    double sbb = 0.0, srr = 0.0;
    if (tiles == 1) {
      sbb = (double)sm.tpart[0].x;
      srr = (double)sm.tpart[0].y;
    } else {
      for (int i = lane; i < tiles; i += 32) {
        sbb += (double)sm.tpart[i].x;
        srr += (double)sm.tpart[i].y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
        srr += __shfl_xor_sync(0xffffffffu, srr, o);
      }
    }
    const unsigned su = __reduce_add_sync(0xffffffffu, lane < STH / 32 ? sm.red_unk[lane] : 0u);
    if (lane == 0) {
      if (su) atomicAdd(w.unknowns, (unsigned long long)su);
      w.unk[slot] = su;
      w.bb[slot] = sbb;
      w.rr[slot] = srr;  // parity 0
      int st = ST_ACTIVE;
      if (sbb <= 0.0)
        st = ST_ZERO;
      else if (srr <= (double)tol2 * sbb)
        st = ST_CONVERGED;
      else if (max_iter <= 0)
        st = ST_MAXITER;
      w.state[slot] = st;
      w.iters[slot] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Fused setup for 2-D levels with 64^2 tiles (config 3), one CTA per tile:
// the tile plus its one-pixel halo of intensity, seeds and bound is read once
// into shared memory (coalesced rows), each thread builds the system of a 4 x 4
// pixel block (the mapping of the tile-resident engine), and ||S b||^2, ||r0||^2
// are reduced in setup_system_kernel's order (per-pixel values, xor tree over
// the 32 x of a setup tile row, 8 rows in sequence, tiles in float64), so the
// result is bit-identical to the two-kernel setup.
constexpr int ST2 = 64, SH2 = ST2 + 2;  // tile edge, with halo
constexpr int SQ2 = 4, SQN2 = ST2 / SQ2, STH2 = SQN2 * SQN2;

__global__ void __launch_bounds__(STH2, 2) setup_tile2d_kernel(Geo g, Work w, const int* __restrict__ list,
                                                            const float* __restrict__ I,
                                                            const uint8_t* __restrict__ S,
                                                            const float* __restrict__ B, float beta, float wmin,
                                                            float tol2, int max_iter, int write_p) {
  __shared__ float sI[SH2][SH2];
  __shared__ float sDv[SH2][SH2];  // Dirichlet value: seed value, else bound
  __shared__ unsigned char sS[SH2][SH2];
  __shared__ float rowpart[2][ST2][2];  // [x tile][row] (bb, rr)
  __shared__ float2 tpart[16];
  __shared__ unsigned red_unk[STH2 / 32];
  const int slot = blockIdx.x;
  const int brick = list ? list[slot] : slot;
  const int hx = brick % g.gx, hy = brick / g.gx;
  const int gy0 = g.oy + hy * ST2, gx0 = g.ox + hx * ST2;
  const int tid = threadIdx.x;
  const int xq = tid % SQN2, yq = tid / SQN2;
  auto wgt = [&](float a, float b) { return edge_weight(a, b, beta, wmin); };
  // ---- tile + halo into shared memory ----
  auto load_px = [&](int ty, int tx) {
    const int gy = gy0 - 1 + ty, gx = gx0 - 1 + tx;
    float iv = 0.f, dv = 0.f;
    unsigned char sv = 0;
    if (gy >= 0 && gy < g.ny && gx >= 0 && gx < g.nx) {
      const long long gi = (long long)gy * g.nx + gx;
      iv = __ldg(I + gi);
      sv = __ldg(S + gi);
      dv = sv ? seed_value(sv) : (B ? __ldg(B + gi) : 0.f);
    }
    sI[ty][tx] = iv;
    sS[ty][tx] = sv;
    sDv[ty][tx] = dv;
  };
  if ((g.nx & 3) == 0 && (gx0 & 3) == 0 && gx0 >= 0 && gx0 + ST2 <= g.nx) {
    // interior columns as 16 B loads (4 pixels of I and B, 4 seeds per 32-bit word), halo
    // columns and out-of-level rows element-wise
    for (int e = tid; e < SH2 * (ST2 / 4); e += STH2) {
      const int ty = e / (ST2 / 4), q = e % (ST2 / 4);
      const int gy = gy0 - 1 + ty;
      float4 iv = make_float4(0.f, 0.f, 0.f, 0.f), bv = iv;
      uchar4 sv = make_uchar4(0, 0, 0, 0);
      if (gy >= 0 && gy < g.ny) {
        const long long gi = (long long)gy * g.nx + gx0 + 4 * q;
        iv = __ldg(reinterpret_cast<const float4*>(I + gi));
        sv = __ldg(reinterpret_cast<const uchar4*>(S + gi));
        if (B) bv = __ldg(reinterpret_cast<const float4*>(B + gi));
      }
      const float ivs[4] = {iv.x, iv.y, iv.z, iv.w}, bvs[4] = {bv.x, bv.y, bv.z, bv.w};
      const unsigned char svs[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int tx = 1 + 4 * q + k;
        sI[ty][tx] = ivs[k];
        sS[ty][tx] = svs[k];
        sDv[ty][tx] = svs[k] ? seed_value(svs[k]) : bvs[k];
      }
    }
    for (int e = tid; e < 2 * SH2; e += STH2) load_px(e >> 1, (e & 1) ? SH2 - 1 : 0);
  } else {
    for (int e = tid; e < SH2 * SH2; e += STH2) load_px(e / SH2, e % SH2);
  }
  __syncthreads();
  // ---- weights and scales of the thread's 4 x 4 pixels ----
  float wyb[SQ2][SQ2], wyf[SQ2][SQ2], wxb[SQ2][SQ2], wxf[SQ2][SQ2], sc[SQ2][SQ2];
  bool in[SQ2][SQ2];
#pragma unroll
  for (int i = 0; i < SQ2; ++i)
#pragma unroll
    for (int k = 0; k < SQ2; ++k) {
      const int ly = SQ2 * yq + i, lx = SQ2 * xq + k;
      const int gy = gy0 + ly, gx = gx0 + lx;
      const int ty = ly + 1, tx = lx + 1;
      in[i][k] = ly < g.by && lx < g.bx && gy >= 0 && gy < g.ny && gx >= 0 && gx < g.nx;
      const float c = sI[ty][tx];
      wyb[i][k] = in[i][k] && gy > 0 ? wgt(c, sI[ty - 1][tx]) : 0.f;
      wyf[i][k] = in[i][k] && gy + 1 < g.ny ? wgt(c, sI[ty + 1][tx]) : 0.f;
      wxb[i][k] = in[i][k] && gx > 0 ? wgt(c, sI[ty][tx - 1]) : 0.f;
      wxf[i][k] = in[i][k] && gx + 1 < g.nx ? wgt(c, sI[ty][tx + 1]) : 0.f;
      // the two-kernel order -z, +z, -y, +y, -x, +x (the z terms are absent: adding nothing)
      const float d = ((wyb[i][k] + wyf[i][k]) + wxb[i][k]) + wxf[i][k];
      sc[i][k] = (in[i][k] && sS[ty][tx] == 0 && d > 0.f) ? jacobi_scale(d) : 0.f;
    }
  // the intensities are consumed: their buffer becomes the scale tile (halo 0: never coupled)
  float(*sSc)[SH2] = sI;
  __syncthreads();
  for (int e = tid; e < SH2 * SH2; e += STH2) {
    const int ty = e / SH2, tx = e % SH2;
    if (ty == 0 || tx == 0 || ty == SH2 - 1 || tx == SH2 - 1) sSc[ty][tx] = 0.f;
  }
#pragma unroll
  for (int i = 0; i < SQ2; ++i)
#pragma unroll
    for (int k = 0; k < SQ2; ++k) sSc[SQ2 * yq + i + 1][SQ2 * xq + k + 1] = sc[i][k];
  __syncthreads();
  // ---- system ----
  float vbb[SQ2][SQ2], vrr[SQ2][SQ2];
  unsigned n_unknown = 0;
#pragma unroll
  for (int i = 0; i < SQ2; ++i) {
    const int ly = SQ2 * yq + i;
    float wfx[SQ2], wfy[SQ2], rr[SQ2], yy[SQ2], ss[SQ2];
#pragma unroll
    for (int k = 0; k < SQ2; ++k) {
      const int lx = SQ2 * xq + k, ty = ly + 1, tx = lx + 1;
      const float si = sc[i][k];
      const bool unk = si > 0.f;
      n_unknown += unk;
      float diag = 0.f, b = 0.f, acc = 0.f;
      auto visit = [&](float wt, float sn, float dv) {
        diag += wt;
        const bool coupled = sn > 0.f;
        acc = coupled ? fmaf(wt, dv, acc) : acc;
        b = coupled ? b : fmaf(wt, dv, b);
        return coupled ? wt * si * sn : 0.f;
      };
      visit(wyb[i][k], sSc[ty - 1][tx], sDv[ty - 1][tx]);
      const float fy = visit(wyf[i][k], sSc[ty + 1][tx], sDv[ty + 1][tx]);
      visit(wxb[i][k], sSc[ty][tx - 1], sDv[ty][tx - 1]);
      const float fx = visit(wxf[i][k], sSc[ty][tx + 1], sDv[ty][tx + 1]);
      const float x0 = B ? sDv[ty][tx] : 0.f;  // an unknown's bound (its Dirichlet value)
      const float ri = initial_residual(si, b, acc, diag, x0);
      const float sb = si * b;
      wfx[k] = unk ? fx : 0.f;
      wfy[k] = unk ? fy : 0.f;
      rr[k] = unk ? ri : 0.f;
      yy[k] = unk ? initial_y(x0, si, diag) : (in[i][k] ? sDv[ty][tx] : 0.f);
      ss[k] = in[i][k] ? si : 0.f;
      vbb[i][k] = unk ? fmaf(sb, sb, 0.f) : 0.f;
      vrr[i][k] = unk ? fmaf(ri, ri, 0.f) : 0.f;
    }
    if (ly < g.by && SQ2 * xq < g.bx) {
      const long long li = (long long)slot * g.bvol + (long long)ly * g.bx + SQ2 * xq;
      *reinterpret_cast<float4*>(w.wx + li) = make_float4(wfx[0], wfx[1], wfx[2], wfx[3]);
      *reinterpret_cast<float4*>(w.wy + li) = make_float4(wfy[0], wfy[1], wfy[2], wfy[3]);
      *reinterpret_cast<float4*>(w.r + li) = make_float4(rr[0], rr[1], rr[2], rr[3]);
      *reinterpret_cast<float4*>(w.y + li) = make_float4(yy[0], yy[1], yy[2], yy[3]);
      *reinterpret_cast<float4*>(w.sc + li) = make_float4(ss[0], ss[1], ss[2], ss[3]);
      if (write_p) *reinterpret_cast<float4*>(w.p0 + li) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  // ---- ||S b||^2, ||r0||^2 in the two-kernel order ----
#pragma unroll
  for (int i = 0; i < SQ2; ++i) {
    float bq[SQ2], rq[SQ2];
#pragma unroll
    for (int k = 0; k < SQ2; ++k) {
      bq[k] = vbb[i][k];
      rq[k] = vrr[i][k];
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {  // x ^ 16, 8, 4 = quad ^ 4, 2, 1 (within a 32-pixel setup tile row)
        bq[k] += __shfl_xor_sync(0xffffffffu, bq[k], o);
        rq[k] += __shfl_xor_sync(0xffffffffu, rq[k], o);
      }
    }
    if ((xq & 7) == 0) {  // x ^ 2, then x ^ 1, inside the quad
      rowpart[xq >> 3][SQ2 * yq + i][0] = (bq[0] + bq[2]) + (bq[1] + bq[3]);
      rowpart[xq >> 3][SQ2 * yq + i][1] = (rq[0] + rq[2]) + (rq[1] + rq[3]);
    }
  }
  const unsigned nu = __reduce_add_sync(0xffffffffu, n_unknown);
  if ((tid & 31) == 0) red_unk[tid >> 5] = nu;
  __syncthreads();
  // setup tiles of 32 x 8 pixels, index tty * 2 + ttx (setup_ctx order)
  if (tid < 16) {
    const int tty = tid >> 1, ttx = tid & 1;
    float2 s = make_float2(0.f, 0.f);
    for (int r8 = 0; r8 < TY; ++r8) {
      s.x += rowpart[ttx][tty * TY + r8][0];
      s.y += rowpart[ttx][tty * TY + r8][1];
    }
    tpart[tid] = s;
  }
  __syncthreads();
  if (tid < 32) {
    const int tiles = ((g.by + TY - 1) / TY) * ((g.bx + TX - 1) / TX);
    double sbb = 0.0, srr = 0.0;
    if (tiles == 1) {
      sbb = (double)tpart[0].x;
      srr = (double)tpart[0].y;
    } else {
      for (int i = tid; i < tiles; i += 32) {
        sbb += (double)tpart[i].x;
        srr += (double)tpart[i].y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sbb += __shfl_xor_sync(0xffffffffu, sbb, o);
        srr += __shfl_xor_sync(0xffffffffu, srr, o);
      }
    }
    const unsigned su = __reduce_add_sync(0xffffffffu, tid < STH2 / 32 ? red_unk[tid] : 0u);
    if (tid == 0) {
      if (su) atomicAdd(w.unknowns, (unsigned long long)su);
      w.unk[slot] = su;
      w.bb[slot] = sbb;
      w.rr[slot] = srr;
      int st = ST_ACTIVE;
      if (sbb <= 0.0)
        st = ST_ZERO;
      else if (srr <= (double)tol2 * sbb)
        st = ST_CONVERGED;
      else if (max_iter <= 0)
        st = ST_MAXITER;
      w.state[slot] = st;
      w.iters[slot] = 0;
    }
  }
}

// Tensor maps for the fused setup; false when the level's layout does not
// meet TMA's rules (16 B aligned bases, row pitches and box x starts) — the
// caller then uses the two-kernel setup.
static bool make_setup_maps(const Geo& g, const float* I, const uint8_t* S, const float* B, SetupMaps* m) {
  if (g.bx > FB || g.by > FB || g.bx % SQ || ((g.bz + STZ - 1) / STZ) * ((g.by + TY - 1) / TY) > SETUP_MAX_TILES)
    return false;
  if (g.ox % 16 || (g.gx > 1 && g.bx % 16)) return false;  // every brick's x start 16-voxel aligned
  if (g.nx % 16 || ((uintptr_t)I & 15) || ((uintptr_t)S & 15) || ((uintptr_t)B & 15)) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  auto enc = [&](CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esz, int boxx) {
    const cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nz};
    const cuuint64_t strides[2] = {(cuuint64_t)g.nx * esz, (cuuint64_t)g.nx * g.ny * esz};
    const cuuint32_t box[3] = {(cuuint32_t)boxx, (cuuint32_t)SRY, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  std::memset(m, 0, sizeof(*m));
  if (!enc(&m->I, I, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, SRX)) return false;
  if (B && !enc(&m->B, B, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, SRX)) return false;
  if (!enc(&m->S, S, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, SRXS)) return false;
  return true;
}

// ---------------------------------------------------------------------------
// CG passes.  Persistent grid: CTAs stride over the work items
// (active brick, tile) of the compacted active list; the list is rebuilt
// between graph chunks, so converged bricks stop costing launches.

__global__ void __launch_bounds__(NTHREADS) cg_pass1_kernel(Geo g, Work w, int nb, const int* __restrict__ list,
                                                            int j) {
  const int n_items = *w.n_active * g.tiles;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ pin = par ? w.p1 : w.p0;
  float* __restrict__ pout = par ? w.p0 : w.p1;
  const float* __restrict__ R = w.r;
  const long long sbz = (long long)g.by * g.bx;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item / g.tiles];
    if (w.state[slot] != ST_ACTIVE) continue;  // uniform per CTA
    TileCtx c = tile_ctx(g, list, slot, item % g.tiles);
    const double rr = w.rr[(long long)par * nb + slot];
    const double rr_prev = w.rr[(long long)(par ^ 1) * nb + slot];
    const float beta = (it == 0 || rr_prev <= 0.0) ? 0.f : (float)(rr / rr_prev);
    float acc = 0.f;
    if (c.col) {
      const long long lbase = (long long)slot * g.bvol + (long long)c.ly * g.bx + c.lx;
      const bool hx0 = c.lx > 0, hx1 = c.lx + 1 < g.bx, hy0 = c.ly > 0, hy1 = c.ly + 1 < g.by;
      auto pn_at = [&](long long i) { return __ldg(R + i) + beta * __ldg(pin + i); };
      long long li = lbase + (long long)c.lz0 * sbz;
      float pm = (g.is3d && c.lz0 > 0) ? pn_at(li - sbz) : 0.f;
      float wzm = (g.is3d && c.lz0 > 0) ? __ldg(w.wz + li - sbz) : 0.f;
      float pc = pn_at(li);
      for (int lz = c.lz0; lz < c.lz1; ++lz, li += sbz) {
        const bool up = g.is3d && lz + 1 < g.bz;
        float pp = up ? pn_at(li + sbz) : 0.f;
        float wzc = up ? __ldg(w.wz + li) : 0.f;
        float s = wzc * pp + wzm * pm;
        if (hx1) s += __ldg(w.wx + li) * pn_at(li + 1);
        if (hx0) s += __ldg(w.wx + li - 1) * pn_at(li - 1);
        if (hy1) s += __ldg(w.wy + li) * pn_at(li + g.bx);
        if (hy0) s += __ldg(w.wy + li - g.bx) * pn_at(li - g.bx);
        float q = pc - s;
        pout[li] = pc;
        w.q[li] = q;
        acc += pc * q;
        pm = pc;
        pc = pp;
        wzm = wzc;
      }
    }
    double pq, unused;
    if (brick_reduce(g, w, slot, c.tile, acc, 0.f, &pq, &unused)) w.pq[slot] = pq;
  }
}

__global__ void __launch_bounds__(NTHREADS) cg_pass2_kernel(Geo g, Work w, int nb, const int* __restrict__ list,
                                                            int j, float tol2, int max_iter) {
  const int n_items = *w.n_active * g.tiles;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ P = par ? w.p0 : w.p1;  // pass-1 output
  const long long sbz = (long long)g.by * g.bx;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item / g.tiles];
    if (w.state[slot] != ST_ACTIVE) continue;
    TileCtx c = tile_ctx(g, list, slot, item % g.tiles);
    const double rr = w.rr[(long long)par * nb + slot];
    const double pq = w.pq[slot];
    const float alpha = pq != 0.0 ? (float)(rr / pq) : 0.f;
    float acc = 0.f;
    if (c.col) {
      long long li = (long long)slot * g.bvol + (long long)c.ly * g.bx + c.lx + (long long)c.lz0 * sbz;
      for (int lz = c.lz0; lz < c.lz1; ++lz, li += sbz) {
        float y = w.y[li] + alpha * __ldg(P + li);
        float r = w.r[li] - alpha * __ldg(w.q + li);
        w.y[li] = y;
        w.r[li] = r;
        acc += r * r;
      }
    }
    double rr_new, unused;
    if (brick_reduce(g, w, slot, c.tile, acc, 0.f, &rr_new, &unused)) {
      w.rr[(long long)(par ^ 1) * nb + slot] = rr_new;
      // decide here so the next pass-1 launch already skips finished bricks
      if (rr_new <= (double)tol2 * w.bb[slot]) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_CONVERGED;
      } else if (it + 1 >= max_iter) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_MAXITER;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Column-marching CG passes (the default streaming passes).  A work item is a
// column tile of a brick: TX x TY threads, each marching the brick's whole
// extent along the march axis (3-D: z, planes of by*bx; 2-D: y, rows of bx,
// thread row ty taking a segment of ceil(by / TY) rows), so an item carries
// 4x (3-D 32^3) to 8x (2-D 64^2) the voxels of a cg_pass1/2 tile and its
// start-up (slot, state, scalars) and brick reduction are amortised over
// them.  Pass 1 keeps a two-plane-deep register pipeline (the loads of plane
// m+2 are issued before plane m is computed) and takes the x neighbours of
// p = r + beta p from the neighbouring lanes (a warp is one 32-voxel row
// segment); pass 2 streams four planes per step.  Same arithmetic, same
// per-brick fixed-order float64 reductions (over the brick's column items).
struct ColCtx {
  int slot, col, lx, ly, m0, m1;  // ly: 3-D row (2-D: 0); [m0, m1): march range of this thread
  bool in;                        // column inside the brick box
};

__device__ __host__ __forceinline__ int col_items(const Geo& g) {
  return g.is3d ? ((g.bx + TX - 1) / TX) * ((g.by + TY - 1) / TY) : (g.bx + TX - 1) / TX;
}

__device__ __forceinline__ ColCtx col_ctx(const Geo& g, int slot, int col) {
  ColCtx c;
  c.slot = slot;
  c.col = col;
  const int ntx = (g.bx + TX - 1) / TX;
  c.lx = (col % ntx) * TX + threadIdx.x;
  if (g.is3d) {
    c.ly = (col / ntx) * TY + threadIdx.y;
    c.m0 = 0;
    c.m1 = g.bz;
    c.in = c.lx < g.bx && c.ly < g.by;
  } else {
    const int my = (g.by + TY - 1) / TY;
    c.ly = 0;
    c.m0 = min(threadIdx.y * my, g.by);
    c.m1 = min(c.m0 + my, g.by);
    c.in = c.lx < g.bx && c.m0 < c.m1;
  }
  return c;
}

__global__ void __launch_bounds__(NTHREADS) cg_pass1_col_kernel(Geo g, Work w, int nb, int j) {
  const int ncol = col_items(g);
  const int n_items = *w.n_active * ncol;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ pin = par ? w.p1 : w.p0;
  float* __restrict__ pout = par ? w.p0 : w.p1;
  float* __restrict__ Q = w.q;
  const float* __restrict__ R = w.r;
  const float* __restrict__ WM = g.is3d ? w.wz : w.wy;  // weight along the march axis
  const long long sm_ = g.is3d ? (long long)g.by * g.bx : (long long)g.bx;
  const int nm = g.is3d ? g.bz : g.by;
  const int lane = threadIdx.x;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item / ncol];
    if (w.state[slot] != ST_ACTIVE) continue;  // uniform per CTA
    const ColCtx c = col_ctx(g, slot, item % ncol);
    const double rr = w.rr[(long long)par * nb + slot];
    const double rr_prev = w.rr[(long long)(par ^ 1) * nb + slot];
    const float beta = (it == 0 || rr_prev <= 0.0) ? 0.f : (float)(rr / rr_prev);
    float acc = 0.f;
    // every lane of a row segment runs the march (shuffles need the whole warp); lanes outside
    // the brick box load nothing and store nothing
    const bool in = c.in;
    const bool hx0 = in && c.lx > 0, hx1 = in && c.lx + 1 < g.bx;
    const bool hy0 = g.is3d && in && c.ly > 0, hy1 = g.is3d && in && c.ly + 1 < g.by;
    const bool ex0 = hx0 && lane == 0, ex1 = hx1 && lane == TX - 1;  // x neighbours outside the warp
    const long long base = (long long)slot * g.bvol + (long long)c.ly * g.bx + c.lx;
    auto ld = [&](const float* a, long long i, bool ok) { return ok ? __ldg(a + i) : 0.f; };
    int m = c.m0;
    long long li = base + (long long)m * sm_;
    const bool any = in && m < c.m1;
    // pipeline: (r, p) of planes m+1 and m+2 in flight; pm = pn(m - 1), pc = pn(m)
    float pm = 0.f, wmm = 0.f;
    if (any && m > 0) {
      pm = ld(R, li - sm_, true) + beta * ld(pin, li - sm_, true);
      wmm = ld(WM, li - sm_, true);
    }
    float pc = any ? ld(R, li, true) + beta * ld(pin, li, true) : 0.f;
    bool ok1 = any && m + 1 < nm, ok2 = any && m + 2 < nm;
    float r1 = ld(R, li + sm_, ok1), p1 = ld(pin, li + sm_, ok1);
    float r2 = ld(R, li + 2 * sm_, ok2), p2 = ld(pin, li + 2 * sm_, ok2);
    const int mend = __reduce_max_sync(0xffffffffu, any ? c.m1 : -1);  // warp-uniform trip count
    for (; m < mend; ++m, li += sm_) {
      const bool act = any && m < c.m1;
      const bool ok3 = act && m + 3 < nm;
      const float r3 = ld(R, li + 3 * sm_, ok3), p3 = ld(pin, li + 3 * sm_, ok3);
      const bool up = act && m + 1 < nm;
      const float pp = up ? r1 + beta * p1 : 0.f;
      const float wmc = ld(WM, li, up);
      float s = wmc * pp + wmm * pm;
      const float wxr = ld(w.wx, li, act && hx1), wxl = ld(w.wx, li - 1, act && hx0);
      float xr = __shfl_down_sync(0xffffffffu, pc, 1), xl = __shfl_up_sync(0xffffffffu, pc, 1);
      if (act && ex1) xr = __ldg(R + li + 1) + beta * __ldg(pin + li + 1);
      if (act && ex0) xl = __ldg(R + li - 1) + beta * __ldg(pin + li - 1);
      if (act && hx1) s += wxr * xr;
      if (act && hx0) s += wxl * xl;
      if (g.is3d) {
        if (act && hy1) s += __ldg(w.wy + li) * (__ldg(R + li + g.bx) + beta * __ldg(pin + li + g.bx));
        if (act && hy0) s += __ldg(w.wy + li - g.bx) * (__ldg(R + li - g.bx) + beta * __ldg(pin + li - g.bx));
      }
      if (act) {
        const float q = pc - s;
        pout[li] = pc;
        Q[li] = q;
        acc += pc * q;
      }
      pm = pc;
      pc = pp;
      wmm = wmc;
      r1 = r2, p1 = p2, r2 = r3, p2 = p3;
    }
    double pq, unused;
    if (brick_reduce(g, w, slot, c.col, acc, 0.f, &pq, &unused, ncol)) w.pq[slot] = pq;
  }
}

// 3-D pass 1 with the operands staged through shared memory: per plane, r and p of the tile's 8
// rows plus one halo row each side, w'x, w'y (with the row below), w'z — 45 rows of 32 floats —
// copied by cp.async (4 B per lane, zero-filled outside the brick) KS planes ahead of the march,
// so every thread has KS - 1 planes of loads in flight without holding them in registers.  The
// arithmetic (operand values and order) is cg_pass1_col_kernel's.
constexpr int KS = 8;           // stages (a plane of compute is ~0.1 us: 6 planes in flight cover the DRAM latency)
struct StgPlane {
  float r[TY + 2][TX], p[TY + 2][TX], wx[TY][TX], wy[TY + 1][TX], wz[TY][TX];
};

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(ok ? src : dst), "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

// VEC: 16-byte copies (brick rows a multiple of 4 floats), 360 per plane over the CTA's 256 threads
template <bool VEC>
__global__ void __launch_bounds__(NTHREADS, 3) cg_pass1_stg_kernel(Geo g, Work w, int nb, int j) {
  __shared__ __align__(16) StgPlane st[KS];
  const int ncol = col_items(g);
  const int n_items = *w.n_active * ncol;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ pin = par ? w.p1 : w.p0;
  float* __restrict__ pout = par ? w.p0 : w.p1;
  float* __restrict__ Q = w.q;
  const float* __restrict__ R = w.r;
  const long long sbz = (long long)g.by * g.bx;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int ntx = (g.bx + TX - 1) / TX;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item / ncol];
    if (w.state[slot] != ST_ACTIVE) continue;  // uniform per CTA
    const int col = item % ncol;
    const int x0 = (col % ntx) * TX, y0 = (col / ntx) * TY;
    const int lx = x0 + lane, ly = y0 + warp;
    const double rr = w.rr[(long long)par * nb + slot];
    const double rr_prev = w.rr[(long long)(par ^ 1) * nb + slot];
    const float beta = (it == 0 || rr_prev <= 0.0) ? 0.f : (float)(rr / rr_prev);
    const long long sbase = (long long)slot * g.bvol;
    const bool xin = lx < g.bx;
    // this warp's copy rows (fixed per item): r, p and w'y of brick row y0 - 1 + warp (stage rows
    // warp), w'x and w'z of row y0 + warp; warps 0-1 also r, p of rows y0 + 7 + warp (stage rows
    // 8 + warp), warp 0 also w'y of row y0 + 7 (stage row 8)
    // VEC: chunk q of this thread = plane row k = c / 8 (StgPlane order), 4 floats at x0 + 4 (c % 8)
    const float* vsrc[2];
    uint32_t vdst[2];
    bool vok[2];
    if (VEC) {
      const int tid = warp * TX + lane;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = tid + NTHREADS * q, k = c >> 3, xs = x0 + 4 * (c & 7);
        const float* arr;
        int row;
        if (k < TY + 2) {
          arr = R, row = y0 - 1 + k;
        } else if (k < 2 * (TY + 2)) {
          arr = pin, row = y0 - 1 + k - (TY + 2);
        } else if (k < 2 * (TY + 2) + TY) {
          arr = w.wx, row = y0 + k - 2 * (TY + 2);
        } else if (k < 2 * (TY + 2) + 2 * TY + 1) {
          arr = w.wy, row = y0 - 1 + k - 2 * (TY + 2) - TY;
        } else {
          arr = w.wz, row = y0 + k - 2 * (TY + 2) - 2 * TY - 1;
        }
        vok[q] = k < 45 && row >= 0 && row < g.by && xs < g.bx;
        vsrc[q] = arr + sbase + (long long)(vok[q] ? row : 0) * g.bx + (vok[q] ? xs : 0);
        vdst[q] = (uint32_t)__cvta_generic_to_shared(&st[0].r[0][0]) + 4u * (uint32_t)(k * TX + 4 * (c & 7));
        if (k >= 45) vdst[q] = 0xffffffffu;  // no such chunk
      }
    }
    const int ra = y0 - 1 + warp, rb = y0 + 7 + warp;
    const bool oka = xin && ra >= 0 && ra < g.by, okb = xin && warp < 2 && rb < g.by;
    const bool okc = xin && y0 + warp < g.by, okd = xin && warp == 0 && y0 + 7 < g.by;
    const long long ga = sbase + (long long)ra * g.bx + lx;
    const long long gb = ga + 8LL * g.bx;
    auto issue = [&](int m) {
      const bool inm = m < g.bz;
      if (VEC) {
        const uint32_t so = (uint32_t)((m % KS) * sizeof(StgPlane));
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (vdst[q] != 0xffffffffu) cp_async16(vdst[q] + so, vsrc[q] + (inm ? (long long)m * sbz : 0), inm && vok[q]);
        return;
      }
      StgPlane& sp = st[m % KS];
      const long long o = ga + (long long)m * sbz;
      cp_async4(&sp.r[warp][lane], R + o, inm && oka);
      cp_async4(&sp.p[warp][lane], pin + o, inm && oka);
      cp_async4(&sp.wy[warp][lane], w.wy + o, inm && oka);
      cp_async4(&sp.wx[warp][lane], w.wx + o + g.bx, inm && okc);
      cp_async4(&sp.wz[warp][lane], w.wz + o + g.bx, inm && okc);
      if (warp < 2) {
        const long long ob = gb + (long long)m * sbz;
        cp_async4(&sp.r[TY + warp][lane], R + ob, inm && okb);
        cp_async4(&sp.p[TY + warp][lane], pin + ob, inm && okb);
        if (warp == 0) cp_async4(&sp.wy[TY][lane], w.wy + ob, inm && okd);
      }
    };
#pragma unroll
    for (int m = 0; m < KS - 1; ++m) {
      issue(m);
      cp_async_commit();
    }
    const bool in = xin && ly < g.by;
    const bool hx0 = in && lx > 0, hx1 = in && lx + 1 < g.bx;
    const bool hy0 = in && ly > 0, hy1 = in && ly + 1 < g.by;
    const bool ex0 = hx0 && lane == 0, ex1 = hx1 && lane == TX - 1;
    long long li = sbase + (long long)ly * g.bx + lx;
    float acc = 0.f, pm = 0.f, wzm = 0.f, pc = 0.f;
    // the march, unrolled by the ring size so every stage index (and shared-memory offset) is a
    // constant; pointers advance by one plane per step
    const float* vnext[2] = {nullptr, nullptr};  // VEC: the sources of plane m + KS - 1, advanced per plane
    if (VEC) {
#pragma unroll
      for (int q = 0; q < 2; ++q) vnext[q] = vsrc[q] + (long long)(KS - 1) * sbz;
    }
    const float* pR = R + li;
    const float* ppin = pin + li;
    const float* pwx = w.wx + li;
    float* ppo = pout + li;
    float* pq_ = Q + li;
    for (int m0 = 0; m0 < g.bz; m0 += KS) {
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const int m = m0 + k;
        if (m >= g.bz) break;
        cp_async_wait<KS - 3>();  // planes m and m + 1 have landed (this thread's copies)
        __syncthreads();          // ... everyone's; and everyone is done with plane m - 1's stage
        if (VEC) {                // refills plane m - 1's stage (zero-filled past the brick)
          const uint32_t so = (uint32_t)(((k + KS - 1) % KS) * sizeof(StgPlane));
          const bool inm = m + KS - 1 < g.bz;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (vdst[q] != 0xffffffffu) cp_async16(vdst[q] + so, inm ? vnext[q] : vsrc[q], inm && vok[q]);
            vnext[q] += sbz;
          }
        } else {
          issue(m + KS - 1);
        }
        cp_async_commit();
        const StgPlane& sc = st[k];
        const StgPlane& sn = st[(k + 1) % KS];
        if (m == 0) pc = sc.r[warp + 1][lane] + beta * sc.p[warp + 1][lane];
        const bool up = m + 1 < g.bz;
        const float pp = up ? sn.r[warp + 1][lane] + beta * sn.p[warp + 1][lane] : 0.f;
        const float wzc = up ? sc.wz[warp][lane] : 0.f;
        float s = wzc * pp + wzm * pm;
        const float wxo = sc.wx[warp][lane];
        float xr = __shfl_down_sync(0xffffffffu, pc, 1), xl = __shfl_up_sync(0xffffffffu, pc, 1);
        float wxl = __shfl_up_sync(0xffffffffu, wxo, 1);
        if (ex1) xr = __ldg(pR + 1) + beta * __ldg(ppin + 1);
        if (ex0) {
          xl = __ldg(pR - 1) + beta * __ldg(ppin - 1);
          wxl = __ldg(pwx - 1);
        }
        if (hx1) s += wxo * xr;
        if (hx0) s += wxl * xl;
        if (hy1) s += sc.wy[warp + 1][lane] * (sc.r[warp + 2][lane] + beta * sc.p[warp + 2][lane]);
        if (hy0) s += sc.wy[warp][lane] * (sc.r[warp][lane] + beta * sc.p[warp][lane]);
        if (in) {
          const float q = pc - s;
          *ppo = pc;
          *pq_ = q;
          acc += pc * q;
        }
        pm = pc;
        pc = pp;
        wzm = wzc;
        pR += sbz, ppin += sbz, pwx += sbz, ppo += sbz, pq_ += sbz;
      }
    }
    cp_async_wait<0>();
    double pq, unused;
    if (brick_reduce(g, w, slot, col, acc, 0.f, &pq, &unused, ncol)) w.pq[slot] = pq;
  }
}

// 2-D pass 1 for bricks of up to 64 x 64 with rows a multiple of 4 floats (config 3's 64^2):
// one brick per item, its r, p, w'x, w'y staged whole into shared memory by 16-byte cp.async
// (64 KB; three CTAs per SM overlap one brick's loads with the others' compute), p = r + beta p
// formed once in place, then the 5-point product from shared memory.  Arithmetic order as
// cg_pass1_col_kernel's (march-axis y terms first, then x).
constexpr int B2 = 64;
struct Brick2Smem {
  float r[B2 * B2], p[B2 * B2], wx[B2 * B2], wy[B2 * B2];
};

__global__ void __launch_bounds__(NTHREADS, 3) cg_pass1_brick2d_kernel(Geo g, Work w, int nb, int j) {
  extern __shared__ __align__(16) unsigned char smem2[];
  Brick2Smem& sm = *reinterpret_cast<Brick2Smem*>(smem2);
  const int n_items = *w.n_active;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ pin = par ? w.p1 : w.p0;
  float* __restrict__ pout = par ? w.p0 : w.p1;
  const int tid = threadIdx.y * TX + threadIdx.x;
  const int bx = g.bx, by = g.by, n = bx * by, nq = n >> 2;  // bx % 4 == 0
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item];
    if (w.state[slot] != ST_ACTIVE) continue;  // uniform per CTA
    const long long sbase = (long long)slot * g.bvol;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem2);
    for (int c = tid; c < 4 * nq; c += NTHREADS) {  // brick-local arrays are contiguous: bx*by floats
      const int a = c / nq, o = 4 * (c - a * nq);
      const float* src = (a == 0 ? w.r : a == 1 ? pin : a == 2 ? w.wx : w.wy) + sbase + o;
      cp_async16(s0 + 4u * (uint32_t)(a * B2 * B2 + o), src, true);
    }
    cp_async_commit();
    const double rr = w.rr[(long long)par * nb + slot];
    const double rr_prev = w.rr[(long long)(par ^ 1) * nb + slot];
    const float beta = (it == 0 || rr_prev <= 0.0) ? 0.f : (float)(rr / rr_prev);
    cp_async_wait<0>();
    __syncthreads();
    for (int i = tid; i < n; i += NTHREADS) {  // p = r + beta p, in place of r
      const float pc = sm.r[i] + beta * sm.p[i];
      sm.r[i] = pc;
      pout[sbase + i] = pc;
    }
    __syncthreads();
    float acc = 0.f;
    for (int i = tid; i < n; i += NTHREADS) {
      const int y = i / bx, x = i - y * bx;
      const float pc = sm.r[i];
      const float pp = y + 1 < by ? sm.r[i + bx] : 0.f;
      const float wmc = y + 1 < by ? sm.wy[i] : 0.f;
      const float pm = y > 0 ? sm.r[i - bx] : 0.f;
      const float wmm = y > 0 ? sm.wy[i - bx] : 0.f;
      float s = wmc * pp + wmm * pm;
      if (x + 1 < bx) s += sm.wx[i] * sm.r[i + 1];
      if (x > 0) s += sm.wx[i - 1] * sm.r[i - 1];
      const float q = pc - s;
      w.q[sbase + i] = q;
      acc += pc * q;
    }
    double pq, unused;
    if (brick_reduce(g, w, slot, 0, acc, 0.f, &pq, &unused, 1)) w.pq[slot] = pq;
    __syncthreads();  // the staging buffer is refilled by the next item
  }
}

__global__ void __launch_bounds__(NTHREADS) cg_pass2_col_kernel(Geo g, Work w, int nb, int j, float tol2,
                                                                int max_iter) {
  const int ncol = col_items(g);
  const int n_items = *w.n_active * ncol;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float* __restrict__ P = par ? w.p0 : w.p1;  // pass-1 output
  const float* __restrict__ Q = w.q;
  float* __restrict__ Y = w.y;
  float* __restrict__ Rw = w.r;
  const long long sm_ = g.is3d ? (long long)g.by * g.bx : (long long)g.bx;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item / ncol];
    if (w.state[slot] != ST_ACTIVE) continue;
    const ColCtx c = col_ctx(g, slot, item % ncol);
    const double rr = w.rr[(long long)par * nb + slot];
    const double pq = w.pq[slot];
    const float alpha = pq != 0.0 ? (float)(rr / pq) : 0.f;
    float acc = 0.f;
    if (c.in) {
      long long li = (long long)slot * g.bvol + (long long)c.ly * g.bx + c.lx + (long long)c.m0 * sm_;
      int m = c.m0;
      for (; m + 4 <= c.m1; m += 4, li += 4 * sm_) {
        float y[4], r[4], pv[4], qv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          y[k] = Y[li + k * sm_];
          r[k] = Rw[li + k * sm_];
          pv[k] = __ldg(P + li + k * sm_);
          qv[k] = __ldg(Q + li + k * sm_);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          y[k] += alpha * pv[k];
          r[k] -= alpha * qv[k];
          Y[li + k * sm_] = y[k];
          Rw[li + k * sm_] = r[k];
          acc += r[k] * r[k];
        }
      }
      for (; m < c.m1; ++m, li += sm_) {
        const float y = Y[li] + alpha * __ldg(P + li);
        const float r = Rw[li] - alpha * __ldg(Q + li);
        Y[li] = y;
        Rw[li] = r;
        acc += r * r;
      }
    }
    double rr_new, unused;
    if (brick_reduce(g, w, slot, c.col, acc, 0.f, &rr_new, &unused, ncol)) {
      w.rr[(long long)(par ^ 1) * nb + slot] = rr_new;
      if (rr_new <= (double)tol2 * w.bb[slot]) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_CONVERGED;
      } else if (it + 1 >= max_iter) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_MAXITER;
      }
    }
  }
}

// Pass 2 over whole bricks as float4 streams (brick volume a multiple of 4): one brick per item,
// the CTA's 256 threads each keep four float4 of y, r, p, q in flight per step.
__global__ void __launch_bounds__(NTHREADS) cg_pass2_vec_kernel(Geo g, Work w, int nb, int j, float tol2, int max_iter) {
  const int n_items = *w.n_active;
  const int par = j & 1;
  const int it = *w.base_it + j;
  const float4* __restrict__ P = reinterpret_cast<const float4*>(par ? w.p0 : w.p1);  // pass-1 output
  const float4* __restrict__ Q = reinterpret_cast<const float4*>(w.q);
  float4* __restrict__ Y = reinterpret_cast<float4*>(w.y);
  float4* __restrict__ Rw = reinterpret_cast<float4*>(w.r);
  const int tid = threadIdx.y * TX + threadIdx.x;
  const int n4 = (int)(g.bvol >> 2);
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[item];
    if (w.state[slot] != ST_ACTIVE) continue;
    const double rr = w.rr[(long long)par * nb + slot];
    const double pq = w.pq[slot];
    const float alpha = pq != 0.0 ? (float)(rr / pq) : 0.f;
    const long long b4 = (long long)slot * n4;
    float acc = 0.f;
    int i = tid;
    for (; i + 3 * NTHREADS < n4; i += 4 * NTHREADS) {
      float4 y[4], r[4], pv[4], qv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y[k] = Y[b4 + i + k * NTHREADS];
        r[k] = Rw[b4 + i + k * NTHREADS];
        pv[k] = __ldg(P + b4 + i + k * NTHREADS);
        qv[k] = __ldg(Q + b4 + i + k * NTHREADS);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y[k] = make_float4(y[k].x + alpha * pv[k].x, y[k].y + alpha * pv[k].y, y[k].z + alpha * pv[k].z,
                           y[k].w + alpha * pv[k].w);
        r[k] = make_float4(r[k].x - alpha * qv[k].x, r[k].y - alpha * qv[k].y, r[k].z - alpha * qv[k].z,
                           r[k].w - alpha * qv[k].w);
        Y[b4 + i + k * NTHREADS] = y[k];
        Rw[b4 + i + k * NTHREADS] = r[k];
        acc += r[k].x * r[k].x;
        acc += r[k].y * r[k].y;
        acc += r[k].z * r[k].z;
        acc += r[k].w * r[k].w;
      }
    }
    for (; i < n4; i += NTHREADS) {
      float4 y = Y[b4 + i], r = Rw[b4 + i];
      const float4 pv = __ldg(P + b4 + i), qv = __ldg(Q + b4 + i);
      y = make_float4(y.x + alpha * pv.x, y.y + alpha * pv.y, y.z + alpha * pv.z, y.w + alpha * pv.w);
      r = make_float4(r.x - alpha * qv.x, r.y - alpha * qv.y, r.z - alpha * qv.z, r.w - alpha * qv.w);
      Y[b4 + i] = y;
      Rw[b4 + i] = r;
      acc += r.x * r.x;
      acc += r.y * r.y;
      acc += r.z * r.z;
      acc += r.w * r.w;
    }
    double rr_new, unused;
    if (brick_reduce(g, w, slot, 0, acc, 0.f, &rr_new, &unused, 1)) {
      w.rr[(long long)(par ^ 1) * nb + slot] = rr_new;
      if (rr_new <= (double)tol2 * w.bb[slot]) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_CONVERGED;
      } else if (it + 1 >= max_iter) {
        w.iters[slot] = it + 1;
        w.state[slot] = ST_MAXITER;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Whole-level (single-brick) solve as ONE cooperative persistent kernel: every
// iteration's two passes are separated by grid-wide barriers instead of kernel
// launches, and the level's working set (~36 B/voxel, 75 MB at 128^3) stays in
// the 126 MB L2.  Loads of the vectors written inside the kernel are plain
// (L1-cacheable) loads: the grid barrier's gpu-scope fence invalidates L1, and
// within a pass they are read-only.  Work items (kCoopTZ planes of a tile) are
// spread evenly over the blocks.  After each barrier every block reduces all
// per-block partials in the same fixed order (float64; every thread one wide
// load, then a fixed tree), so all blocks take the same decisions and the
// result is deterministic.  (A single-sweep Chronopoulos-Gear variant needs
// r, s, w double-buffered — 11 vectors, 92 MB at 128^3 — and fell out of L2:
// 38 GB of DRAM traffic per solve instead of 0.14 GB; it was slower.)
#ifndef RWB_COOP_TZ
#define RWB_COOP_TZ 4
#endif
constexpr int kCoopTZ = RWB_COOP_TZ;  // z planes per work item of the cooperative sweeps
constexpr int kCoopMaxBlocks = 4096;  // partial slots of the cooperative whole-level solve

__device__ __forceinline__ double coop_total(const float* part, int n, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  double a = 0.0;
  for (int i = tid; i < n; i += NTHREADS) a += (double)__ldcg(part + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  __syncthreads();  // sh free from its previous use
  if ((tid & 31) == 0) sh[tid >> 5] = a;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int wv = 0; wv < NTHREADS / 32; ++wv) t += sh[wv];
  return t;
}

#ifdef RWB_TRACE
__device__ long long g_coop_trace[2][64][8];  // [block 0 / last block][iteration][phase] clock64
extern "C" int rwb_coop_trace_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_coop_trace, sizeof(g_coop_trace));
}
#define CTRACE(k)                                                                                       \
  do {                                                                                                  \
    if (threadIdx.x == 0 && threadIdx.y == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && it < 64) \
      g_coop_trace[blockIdx.x == 0 ? 0 : 1][it][k] = clock64();                                        \
  } while (0)
#else
#define CTRACE(k) \
  do {            \
  } while (0)
#endif

__global__ void __launch_bounds__(NTHREADS) coop_cg_kernel(Geo g, Work w, float* part_pq, float* part_rr, int n_items,
                                                           float tol2, int max_iter) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[NTHREADS / 32];
  const long long sbz = (long long)g.by * g.bx;
  const double bb = w.bb[0];
  double rr = w.rr[0];
  int state = ST_ACTIVE;
  if (bb <= 0.0)
    state = ST_ZERO;
  else if (rr <= (double)tol2 * bb)
    state = ST_CONVERGED;
  else if (max_iter <= 0)
    state = ST_MAXITER;
  int it = 0;
  double rr_prev = 0.0;
  while (state == ST_ACTIVE) {
    CTRACE(0);
    const int par = it & 1;
    const float* pin = par ? w.p1 : w.p0;
    float* pout = par ? w.p0 : w.p1;
    const float beta = (it == 0) ? 0.f : (float)(rr / rr_prev);
    // pass 1: p <- r + beta p ; q = A'p ; p.q
    float acc = 0.f;
    {
      const float* __restrict__ R = w.r;
      const float* __restrict__ PI = pin;
      float* __restrict__ PO = pout;
      float* __restrict__ Q = w.q;
      const float* __restrict__ WX = w.wx;
      const float* __restrict__ WY = w.wy;
      const float* __restrict__ WZ = w.wz;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        TileCtx c = tile_ctx<kCoopTZ>(g, nullptr, 0, item);
        if (!c.col) continue;
        const long long lbase = (long long)c.ly * g.bx + c.lx;
        const bool hx0 = c.lx > 0, hx1 = c.lx + 1 < g.bx, hy0 = c.ly > 0, hy1 = c.ly + 1 < g.by;
        auto pn_at = [&](long long i) { return R[i] + beta * PI[i]; };
        long long li = lbase + (long long)c.lz0 * sbz;
        float pm = (g.is3d && c.lz0 > 0) ? pn_at(li - sbz) : 0.f;
        float wzm = (g.is3d && c.lz0 > 0) ? __ldg(WZ + li - sbz) : 0.f;
        float pc = pn_at(li);
        auto plane = [&](int lz) {
          const bool up = g.is3d && lz + 1 < g.bz;
          float pp = up ? pn_at(li + sbz) : 0.f;
          float wzc = up ? __ldg(WZ + li) : 0.f;
          float s = wzc * pp + wzm * pm;
          if (hx1) s += __ldg(WX + li) * pn_at(li + 1);
          if (hx0) s += __ldg(WX + li - 1) * pn_at(li - 1);
          if (hy1) s += __ldg(WY + li) * pn_at(li + g.bx);
          if (hy0) s += __ldg(WY + li - g.bx) * pn_at(li - g.bx);
          const float q = pc - s;
          PO[li] = pc;
          Q[li] = q;
          acc += pc * q;
          pm = pc;
          pc = pp;
          wzm = wzc;
          li += sbz;
        };
        if (c.lz1 - c.lz0 == kCoopTZ) {  // full items: unrolled, so the loads of all planes batch up
#pragma unroll
          for (int k = 0; k < kCoopTZ; ++k) plane(c.lz0 + k);
        } else {
          for (int lz = c.lz0; lz < c.lz1; ++lz) plane(lz);
        }
      }
    }
    {
      const float2 sblk = block_sum2(acc, 0.f);
      if (threadIdx.x == 0 && threadIdx.y == 0) part_pq[blockIdx.x] = sblk.x;
    }
    CTRACE(1);
    grid.sync();
    CTRACE(2);
    const double pq = coop_total(part_pq, gridDim.x, sh);
    CTRACE(3);
    const float alpha = pq != 0.0 ? (float)(rr / pq) : 0.f;
    // pass 2: y += alpha p ; r -= alpha q ; r.r
    float acc2 = 0.f;
    {
      float* __restrict__ Y = w.y;
      float* __restrict__ R = w.r;
      const float* __restrict__ PO = pout;
      const float* __restrict__ Q = w.q;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        TileCtx c = tile_ctx<kCoopTZ>(g, nullptr, 0, item);
        if (!c.col) continue;
        long long li = (long long)c.ly * g.bx + c.lx + (long long)c.lz0 * sbz;
        auto plane = [&]() {
          const float y = Y[li] + alpha * PO[li];
          const float r = R[li] - alpha * Q[li];
          Y[li] = y;
          R[li] = r;
          acc2 += r * r;
          li += sbz;
        };
        if (c.lz1 - c.lz0 == kCoopTZ) {
#pragma unroll
          for (int k = 0; k < kCoopTZ; ++k) plane();
        } else {
          for (int lz = c.lz0; lz < c.lz1; ++lz) plane();
        }
      }
    }
    {
      const float2 sblk = block_sum2(acc2, 0.f);
      if (threadIdx.x == 0 && threadIdx.y == 0) part_rr[blockIdx.x] = sblk.x;
    }
    CTRACE(4);
    grid.sync();
    CTRACE(5);
    const double rr_new = coop_total(part_rr, gridDim.x, sh);
    CTRACE(6);
    ++it;
    if (rr_new <= (double)tol2 * bb)
      state = ST_CONVERGED;
    else if (it >= max_iter)
      state = ST_MAXITER;
    rr_prev = rr;
    rr = rr_new;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) {
    w.state[0] = state;
    w.iters[0] = state == ST_ZERO ? 0 : it;
    // the epilogue reads y from the buffer pass 2 last wrote: nothing else to do
  }
}

// Single CTA: advance the iteration base by k and rebuild the compacted list
// of active slots (stable order).
__global__ void __launch_bounds__(1024) advance_kernel(Work w, int nb, int k) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int start = 0; start < nb; start += 1024) {
    int s = start + threadIdx.x;
    int a = (s < nb && w.state[s] == ST_ACTIVE) ? 1 : 0;
    unsigned m = __ballot_sync(0xffffffffu, a);
    int pre = __popc(m & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    int off = 0;
    for (int i = 0; i < wid; ++i) off += warp_tot[i];
    if (a) w.alist[base + off + pre] = s;
    // the settled slots fill the list from its end: alist[nb-1-i], i = their rank
    if (s < nb && !a) w.alist[nb - 1 - (start - base - off - pre + threadIdx.x)] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int i = 0; i < 32; ++i) t += warp_tot[i];
      base += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *w.n_active = base;
    *w.base_it += k;
  }
}

__global__ void finalize_kernel(Work w, int nb) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nb && w.state[s] == ST_ACTIVE) {
    w.state[s] = ST_MAXITER;
    w.iters[s] = *w.base_it;
  }
}

// prob = seed value | s*y | 0 (zero-rhs brick) | bound (isolated voxel)
// prob / labels of one tile of a brick from the brick-local solution
__device__ __forceinline__ void epilogue_tile(const Geo& g, const Work& w, const TileCtx& c, float* __restrict__ prob,
                                              uint8_t* __restrict__ labels) {
  if (!c.col) return;
  const int gy = c.gy0 + c.ly, gx = c.gx0 + c.lx;
  if (gy < 0 || gy >= g.ny || gx < 0 || gx >= g.nx) return;
  const int st = w.state[c.slot];
  const long long sbz = (long long)g.by * g.bx;
  long long li = (long long)c.slot * g.bvol + (long long)c.ly * g.bx + c.lx + (long long)c.lz0 * sbz;
  for (int lz = c.lz0; lz < c.lz1; ++lz, li += sbz) {
    const int gz = c.gz0 + lz;
    if (gz < 0 || gz >= g.nz) continue;
    long long gi = (long long)gz * g.sxy + (long long)gy * g.nx + gx;
    const float s = w.sc[li];
    const float y = w.y[li];  // an unknown's scaled solution, else the final value (setup)
    const float p = s > 0.f ? (st == ST_ZERO ? 0.f : s * y) : y;
    prob[gi] = p;
    if (labels) labels[gi] = p > 0.5f ? 1 : 0;
  }
}

__global__ void __launch_bounds__(NTHREADS) epilogue_kernel(Geo g, Work w, const int* __restrict__ list,
                                                            float* __restrict__ prob, uint8_t* __restrict__ labels) {
  epilogue_tile(g, w, tile_ctx(g, list), prob, labels);
}

// Epilogue of the bricks the setup already settled (zero rhs, converged at
// start): the brick-resident engine writes its own bricks' results.  The
// settled slots sit at the end of the active list (advance_kernel).
__global__ void __launch_bounds__(NTHREADS) settled_epilogue_kernel(Geo g, Work w, const int* __restrict__ list, int nb,
                                                                    float* __restrict__ prob,
                                                                    uint8_t* __restrict__ labels) {
  const int n_items = (nb - *w.n_active) * g.tiles;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int slot = w.alist[nb - 1 - item / g.tiles];
    epilogue_tile(g, w, tile_ctx(g, list, slot, item % g.tiles), prob, labels);
  }
}

// stat_i: [0] converged [1] maxiter [2] zero-rhs [3] max iterations [4..5] u64 sum of iterations
//         [6..7] u64 sum over bricks of unknowns x iterations
__global__ void __launch_bounds__(1024) stats_kernel(Work w, int nb) {
  // integer sums: order-free, so warp reductions and one shared atomic per warp
  __shared__ int sh[4];
  __shared__ unsigned long long sum, usum;
  if (threadIdx.x < 4) sh[threadIdx.x] = 0;
  if (threadIdx.x == 0) sum = usum = 0;
  __syncthreads();
  int c1 = 0, c2 = 0, c3 = 0, mx = 0;
  unsigned long long sm = 0, um = 0;
  for (int s = threadIdx.x; s < nb; s += blockDim.x) {
    const int st = w.state[s];
    c1 += st == ST_CONVERGED;
    c2 += st == ST_MAXITER;
    c3 += st == ST_ZERO;
    const int it = st == ST_ZERO ? 0 : w.iters[s];
    mx = max(mx, it);
    sm += (unsigned long long)it;
    um += (unsigned long long)it * w.unk[s];
  }
  c1 = __reduce_add_sync(0xffffffffu, c1);
  c2 = __reduce_add_sync(0xffffffffu, c2);
  c3 = __reduce_add_sync(0xffffffffu, c3);
  mx = __reduce_max_sync(0xffffffffu, mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    um += __shfl_xor_sync(0xffffffffu, um, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sh[0], c1);
    atomicAdd(&sh[1], c2);
    atomicAdd(&sh[2], c3);
    atomicMax(&sh[3], mx);
    atomicAdd(&sum, sm);
    atomicAdd(&usum, um);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) w.stat_i[i] = sh[i];
    *reinterpret_cast<unsigned long long*>(w.stat_i + 4) = sum;
    *reinterpret_cast<unsigned long long*>(w.stat_i + 6) = usum;
  }
}

// ---------------------------------------------------------------------------
// host side

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static int make_geo(const rwb_geometry_t* geom, Geo* g) {
  if (!geom) return fail(RWB_ERR_INVALID, "null geometry");
  if (geom->ndim != 2 && geom->ndim != 3) return fail(RWB_ERR_INVALID, "solver supports ndim 2 or 3");
  Shape3 s;
  int rc = shape_from(geom->ndim, geom->size, &s);
  if (rc) return rc;
  int64_t b[3] = {1, 1, 1}, o[3] = {0, 0, 0};
  for (int i = 0; i < geom->ndim; ++i) {
    b[3 - geom->ndim + i] = geom->brick[i];
    o[3 - geom->ndim + i] = geom->origin[i];
  }
  for (int i = 0; i < 3; ++i) {
    if (b[i] < 1 || b[i] > (1 << 20)) return fail(RWB_ERR_INVALID, "brick size out of range");
    if (o[i] > 0 || o[i] <= -b[i]) return fail(RWB_ERR_INVALID, "origin must lie in (-brick, 0]");
  }
  g->nz = s.nz, g->ny = s.ny, g->nx = s.nx;
  g->bz = (int)b[0], g->by = (int)b[1], g->bx = (int)b[2];
  g->oz = (int)o[0], g->oy = (int)o[1], g->ox = (int)o[2];
  g->gz = (int)((s.nz - o[0] + b[0] - 1) / b[0]);
  g->gy = (int)((s.ny - o[1] + b[1] - 1) / b[1]);
  g->gx = (int)((s.nx - o[2] + b[2] - 1) / b[2]);
  g->tz = (g->bz + TZ - 1) / TZ;
  g->ty = (g->by + TY - 1) / TY;
  g->tx = (g->bx + TX - 1) / TX;
  g->tiles = g->tz * g->ty * g->tx;
  g->bvol = (long long)g->bz * g->by * g->bx;
  g->sxy = (long long)g->ny * g->nx;
  g->is3d = geom->ndim == 3;
  return RWB_OK;
}


enum { L_Y, L_R, L_P0, L_P1, L_Q, L_WX, L_WY, L_WZ, L_SC, L_RR, L_PQ, L_BB, L_STATE, L_ITERS, L_UNK, L_TICKET,
       L_ALIST, L_PART, L_MISC, L_MG, L_N };

struct Layout {
  size_t off[L_N];
  size_t total;
};

static Layout layout(const Geo& g, long long nb) {
  Layout L;
  const size_t vox = (size_t)nb * (size_t)g.bvol * sizeof(float);
  const size_t sizes[L_N] = {vox, vox, vox, vox, vox, vox, vox, g.is3d ? vox : 0, vox,
                             2 * nb * sizeof(double), nb * sizeof(double), nb * sizeof(double),
                             nb * sizeof(int), nb * sizeof(int), nb * sizeof(unsigned), nb * sizeof(unsigned), nb * sizeof(int),
                             std::max((size_t)nb * std::max(g.tiles, setup_tiles(g)) * sizeof(float2),
                                      (size_t)2 * kCoopMaxBlocks * sizeof(float)),
                             128,
                             // whole-level geometry: the multigrid solver's vectors and aggregate levels
                             (g.gz == 1 && g.gy == 1 && g.gx == 1) ? mg_workspace_bytes(g.bz, g.by, g.bx) : 0};
  size_t o = 0;
  for (int i = 0; i < L_N; ++i) {
    L.off[i] = o;
    o = align_up(o + sizes[i], 256);
  }
  L.total = o;
  return L;
}

static Work carve(const Layout& L, char* base, const Geo& g) {
  Work w;
  float** f[9] = {&w.y, &w.r, &w.p0, &w.p1, &w.q, &w.wx, &w.wy, &w.wz, &w.sc};
  for (int i = 0; i < 9; ++i) *f[i] = reinterpret_cast<float*>(base + L.off[L_Y + i]);
  if (!g.is3d) w.wz = nullptr;
  w.rr = reinterpret_cast<double*>(base + L.off[L_RR]);
  w.pq = reinterpret_cast<double*>(base + L.off[L_PQ]);
  w.bb = reinterpret_cast<double*>(base + L.off[L_BB]);
  w.state = reinterpret_cast<int*>(base + L.off[L_STATE]);
  w.iters = reinterpret_cast<int*>(base + L.off[L_ITERS]);
  w.unk = reinterpret_cast<unsigned*>(base + L.off[L_UNK]);
  w.ticket = reinterpret_cast<unsigned*>(base + L.off[L_TICKET]);
  w.alist = reinterpret_cast<int*>(base + L.off[L_ALIST]);
  w.part = reinterpret_cast<float2*>(base + L.off[L_PART]);
  char* misc = base + L.off[L_MISC];
  w.base_it = reinterpret_cast<int*>(misc);
  w.n_active = reinterpret_cast<int*>(misc + 4);
  w.unknowns = reinterpret_cast<unsigned long long*>(misc + 8);
  w.stat_i = reinterpret_cast<int*>(misc + 16);
  w.stamp = reinterpret_cast<unsigned long long*>(misc + 48);
  w.next = reinterpret_cast<int*>(misc + 64);
  return w;
}

// Small device -> host readbacks (active-brick counts, per-level stats) go
// through MAPPED pinned memory written by a one-warp kernel, not through
// cudaMemcpyAsync: a copy puts the stream on the copy engine, and the stream's
// next operations then queue behind unrelated bulk copies on that engine (e.g.
// the overlapped result downloads of api.segment_many), stalling the solver.
struct PinnedScratch {
  int* host = nullptr;
  int* dev = nullptr;  // device alias of `host`
  ~PinnedScratch() {
    if (host) cudaFreeHost(host);
  }
};
static thread_local PinnedScratch t_pinned;

static int pinned(int** out, int** dev_alias = nullptr) {
  if (!t_pinned.host) {
    RWB_CUDA(cudaHostAlloc(&t_pinned.host, 64, cudaHostAllocMapped | cudaHostAllocPortable));  // [0] n_active, [2..9] stats, [10..11] unknowns
    RWB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t_pinned.dev), t_pinned.host, 0));
  }
  *out = t_pinned.host;
  if (dev_alias) *dev_alias = t_pinned.dev;
  return RWB_OK;
}

__global__ void readback_kernel(int* __restrict__ dst, const int* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// n 32-bit words from device memory into the mapped scratch at word `at`, then wait for the stream
static int readback(cudaStream_t st, const void* src, int at, int n) {
  int *host = nullptr, *dev = nullptr;
  int rc = pinned(&host, &dev);
  if (rc) return rc;
  readback_kernel<<<1, 32, 0, st>>>(dev + at, static_cast<const int*>(src), n);
  RWB_LAUNCH_CHECK("readback_kernel");
  RWB_CUDA(cudaStreamSynchronize(st));
  return RWB_OK;
}

// persistent grids of the CG passes: [0] the plane-tile passes (and the default for other users),
// [1] the staged 3-D pass 1, [2] the column-marching passes, [3] the whole-brick 2-D pass 1,
// [4] the whole-brick float4 pass 2
static int persistent_grid(int* grid, int* grids3 = nullptr) {
  static DeviceCache cache[5];
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int cached = cache[0][dev].load(std::memory_order_relaxed);
  if (!cached) {
    int sms = 0, per[5] = {0, 0, 0, 0, 0};
    RWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[0], cg_pass1_kernel, NTHREADS, 0));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[1], cg_pass2_kernel, NTHREADS, 0));
    int per_b = 0;
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[2], cg_pass1_stg_kernel<false>, NTHREADS, 0));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_b, cg_pass1_stg_kernel<true>, NTHREADS, 0));
    per[2] = std::min(per[2], per_b);
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[3], cg_pass1_col_kernel, NTHREADS, 0));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per[4], cg_pass2_col_kernel, NTHREADS, 0));
    cache[1][dev].store(sms * std::max(1, per[2]), std::memory_order_relaxed);
    int per2d = 0;
    RWB_CUDA(cudaFuncSetAttribute(cg_pass1_brick2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(Brick2Smem)));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2d, cg_pass1_brick2d_kernel, NTHREADS,
                                                           sizeof(Brick2Smem)));
    cache[3][dev].store(sms * std::max(1, per2d), std::memory_order_relaxed);
    int perv = 0;
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perv, cg_pass2_vec_kernel, NTHREADS, 0));
    cache[4][dev].store(sms * std::max(1, perv), std::memory_order_relaxed);
    cache[2][dev].store(sms * std::max(1, std::min(per[3], per[4])), std::memory_order_relaxed);
    cached = sms * std::max(1, std::min(per[0], per[1]));
    cache[0][dev].store(cached, std::memory_order_relaxed);
  }
  *grid = cached;
  if (grids3) {
    grids3[0] = cached;
    grids3[1] = cache[1][dev].load(std::memory_order_relaxed);
    grids3[2] = cache[2][dev].load(std::memory_order_relaxed);
    grids3[3] = cache[3][dev].load(std::memory_order_relaxed);
    grids3[4] = cache[4][dev].load(std::memory_order_relaxed);
  }
  return RWB_OK;
}

static int launch_chunk(const Geo& g, const Work& w, int nb, const int* list, int k, float tol2, int max_iter,
                        int grid, cudaStream_t st) {
  // counted by the caller (graph replays count 2k+1 kernels each)
  dim3 block(TX, TY);
  static const bool tiles_env = [] {  // RWB_CG_TILES=1: the plane-tile passes (diagnostics)
    const char* e = std::getenv("RWB_CG_TILES");
    return e && e[0] == '1';
  }();
  static const bool vec2_off = [] {  // RWB_CG_VEC2=0: the column-marching pass 2 (diagnostics)
    const char* e = std::getenv("RWB_CG_VEC2");
    return e && e[0] == '0';
  }();
  int grids[5];
  if (int rc = persistent_grid(&grid, grids)) return rc;
  for (int j = 0; j < k; ++j) {
    if (tiles_env) {
      cg_pass1_kernel<<<grids[0], block, 0, st>>>(g, w, nb, list, j);
      cg_pass2_kernel<<<grids[0], block, 0, st>>>(g, w, nb, list, j, tol2, max_iter);
    } else {
      if (g.is3d && g.bx % 4 == 0)
        cg_pass1_stg_kernel<true><<<grids[1], block, 0, st>>>(g, w, nb, j);
      else if (g.is3d)
        cg_pass1_stg_kernel<false><<<grids[1], block, 0, st>>>(g, w, nb, j);
      else if (g.bx % 4 == 0 && g.bx <= B2 && g.by <= B2)
        cg_pass1_brick2d_kernel<<<grids[3], block, sizeof(Brick2Smem), st>>>(g, w, nb, j);
      else
        cg_pass1_col_kernel<<<grids[2], block, 0, st>>>(g, w, nb, j);
      if (g.bvol % 4 == 0 && !vec2_off)
        cg_pass2_vec_kernel<<<grids[4], block, 0, st>>>(g, w, nb, j, tol2, max_iter);
      else
        cg_pass2_col_kernel<<<grids[2], block, 0, st>>>(g, w, nb, j, tol2, max_iter);
    }
  }
  advance_kernel<<<1, 1024, 0, st>>>(w, nb, k);
  RWB_LAUNCH_CHECK_CAPTURE("cg iteration kernels");
  return RWB_OK;
}

// Copy the per-level stats to the host (synchronises the stream).
// Copy the per-level stats to the host (synchronises the stream).  The copies
// land in PINNED scratch: a copy into pageable memory is staged by the driver
// and can queue behind unrelated bulk copies on other streams (e.g. the
// overlapped downloads of api.segment_many), stalling this stream for them.
__global__ void stamp_kernel(unsigned long long* dst, int* zero = nullptr) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
  if (zero) *zero = 0;
}

// RWB_SOLVE_STATS_DEVICE: `stats` is device-accessible memory (device memory or
// mapped pinned host memory); one thread fills it after the level's stats
// kernel, with no host synchronisation.  cg_ms = `host_ms` when given (>= 0),
// else the %globaltimer span around the solve launches.
__global__ void stats_to_struct_kernel(Work w, int nb, int sweeps, int path, float host_ms,
                                       rwb_solve_stats_t* __restrict__ out) {
  if (threadIdx.x != 0) return;
  const int* hs = w.stat_i;
  rwb_solve_stats_t s;
  s.bricks = nb;
  s.converged = hs[0];
  s.not_converged = hs[1];
  s.zero_rhs = hs[2];
  s.iterations_max = hs[3];
  s.iterations_sum = (int64_t)*reinterpret_cast<const unsigned long long*>(hs + 4);
  s.unknowns = (int64_t)*w.unknowns;
  s.sweeps = sweeps ? sweeps : hs[3];
  s.cg_ms = host_ms >= 0.f ? host_ms : (float)((double)(w.stamp[1] - w.stamp[0]) * 1e-6);
  s.path = path;
  s.reserved = 0;
  s.unknown_iterations = (int64_t)*reinterpret_cast<const unsigned long long*>(hs + 6);
  *out = s;
}

static int read_stats(const Work& w, int nb, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1, int sweeps, int path,
                      rwb_solve_stats_t* stats, float cg_ms = -1.f, bool on_device = false) {
  if (on_device) {
    stats_to_struct_kernel<<<1, 32, 0, st>>>(w, nb, sweeps, path, cg_ms, stats);
    RWB_LAUNCH_CHECK("stats_to_struct_kernel");
    count_launches(1);
    return RWB_OK;
  }
  int* host = nullptr;
  int rc = pinned(&host);
  if (rc) return rc;
  int* hs = host + 2;                                                   // 8 ints
  readback_kernel<<<1, 32, 0, st>>>(t_pinned.dev + 2, w.stat_i, 8);
  rc = readback(st, w.unknowns, 10, 2);
  if (rc) return rc;
  unsigned long long unk;
  std::memcpy(&unk, host + 10, sizeof(unk));
  float ms = cg_ms >= 0.f ? cg_ms : 0.f;
  if (cg_ms < 0.f && ev0 && ev1) RWB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  stats->bricks = nb;
  stats->converged = hs[0];
  stats->not_converged = hs[1];
  stats->zero_rhs = hs[2];
  stats->iterations_max = hs[3];
  unsigned long long s64;
  std::memcpy(&s64, hs + 4, sizeof(s64));
  stats->iterations_sum = (int64_t)s64;
  stats->unknowns = (int64_t)unk;
  stats->sweeps = sweeps ? sweeps : hs[3];
  unsigned long long ui;
  std::memcpy(&ui, hs + 6, sizeof(ui));
  stats->unknown_iterations = (int64_t)ui;
  stats->cg_ms = ms;
  stats->path = path;
  return RWB_OK;
}

static int coop_grid(int* grid) {
  static DeviceCache cache;
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int cached = cache[dev].load(std::memory_order_relaxed);
  if (!cached) {
    int sms = 0, per = 0, coop = 0;
    RWB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop) return fail(RWB_ERR_UNSUPPORTED, "device does not support cooperative launches");
    RWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, coop_cg_kernel, NTHREADS, 0));
    if (const char* e = std::getenv("RWB_COOP_BLOCKS_PER_SM"))  // diagnostics: fewer, fatter blocks
      per = std::max(1, std::min(per, std::atoi(e)));
    cached = std::min(sms * std::max(per, 1), kCoopMaxBlocks);
    cache[dev].store(cached, std::memory_order_relaxed);
  }
  *grid = cached;
  return RWB_OK;
}

}  // namespace rwb

using namespace rwb;

static bool use_resident(const Geo& g, long long total, int flags) {
  if (flags & RWB_SOLVE_STREAMING) return false;
  // a whole 2-D level of one 64^2 tile (config 3's coarsest) is one tile-resident CTA: CTA-local
  // reductions instead of the whole-level kernels' grid barriers (1.4 -> ~0.3 ms)
  if (total == 1) return resident2d_supported(g) && !(flags & RWB_SOLVE_MG);
  return resident3d_supported(g) || resident2d_supported(g);
}

extern "C" size_t rwb_solve_workspace_bytes(const rwb_geometry_t* geom, int64_t n_bricks, int32_t flags) {
  Geo g;
  if (make_geo(geom, &g)) return 0;
  long long total = (long long)g.gz * g.gy * g.gx;
  long long nb = n_bricks < 0 ? total : n_bricks;
  (void)flags;  // every path builds the brick-local system with the streaming setup kernels
  return layout(g, nb).total;
}

static int solve_level_impl(const rwb_geometry_t* geom, const float* intensity, const uint8_t* seeds,
                            const float* bound, const int32_t* brick_list, int64_t n_bricks,
                            const rwb_solve_params_t* params, float* prob, uint8_t* labels, void* workspace,
                            size_t workspace_bytes, rwb_solve_stats_t* stats, void* stream);

// Reentrant and stream-ordered: every piece of a call's device state lives in the caller's
// workspace, host-side scratch (the mapped readback words) is per thread, launch caches are per
// device (atomics), and the streaming path captures its graph in cudaStreamCaptureModeThreadLocal
// on a private stream, so concurrent callers on distinct streams and workspaces (the reference
// Engine's worker pool, engine.py:398-400, 866-875) run without a process-wide lock.
extern "C" int rwb_solve_level(const rwb_geometry_t* geom, const float* intensity, const uint8_t* seeds,
                               const float* bound, const int32_t* brick_list, int64_t n_bricks,
                               const rwb_solve_params_t* params, float* prob, uint8_t* labels, void* workspace,
                               size_t workspace_bytes, rwb_solve_stats_t* stats, void* stream) {
  return solve_level_impl(geom, intensity, seeds, bound, brick_list, n_bricks, params, prob, labels, workspace,
                          workspace_bytes, stats, stream);
}

static int solve_level_impl(const rwb_geometry_t* geom, const float* intensity, const uint8_t* seeds,
                            const float* bound, const int32_t* brick_list, int64_t n_bricks,
                            const rwb_solve_params_t* params, float* prob, uint8_t* labels, void* workspace,
                            size_t workspace_bytes, rwb_solve_stats_t* stats, void* stream) {
  Geo g;
  int rc = make_geo(geom, &g);
  if (rc) return rc;
  if (!intensity || !seeds || !prob || !params || !workspace) return fail(RWB_ERR_INVALID, "null pointer");
  const long long total = (long long)g.gz * g.gy * g.gx;
  const long long nbl = brick_list ? n_bricks : total;
  if (nbl < 0 || nbl > total) return fail(RWB_ERR_INVALID, "n_bricks out of range");
  if (!bound && total > 1) return fail(RWB_ERR_INVALID, "bound may be NULL only for a single-brick level");
  if (!(params->tol >= 0.f) || !(params->beta >= 0.f) || !(params->min_weight >= 0.f) || params->max_iter < 0)
    return fail(RWB_ERR_INVALID, "invalid solve parameters");
  if (nbl * (long long)std::max(g.tiles, setup_tiles(g)) >= (1ll << 31))
    return fail(RWB_ERR_INVALID, "too many bricks for one launch");
  const Layout L = layout(g, nbl);
  if (workspace_bytes < L.total)
    return fail(RWB_ERR_WORKSPACE, "workspace too small: need " + std::to_string(L.total) + " bytes");
  const bool dev_stats = params->flags & RWB_SOLVE_STATS_DEVICE;
  if (stats && !dev_stats) std::memset(stats, 0, sizeof(*stats));
  if (stats && dev_stats) RWB_CUDA(cudaMemsetAsync(stats, 0, sizeof(*stats), (cudaStream_t)stream));
  if (nbl == 0) return RWB_OK;
  const int nb = (int)nbl;
  cudaStream_t st = (cudaStream_t)stream;
  Work w = carve(L, (char*)workspace, g);
  const int* list = brick_list;
  const float tol2 = params->tol * params->tol;
  const int max_iter = params->max_iter;
  int k = params->check_every > 0 ? params->check_every : 16;
  k += k & 1;  // parity of the global iteration must match the captured j
  int grid = 0;
  rc = persistent_grid(&grid);
  if (rc) return rc;

  const unsigned sgrid = (unsigned)((long long)nb * g.tiles);
  const unsigned setup_grid = (unsigned)((long long)nb * setup_tiles(g));
  dim3 block(TX, TY);
  const bool resident = use_resident(g, total, params->flags);
  const bool setup_only = params->flags & RWB_SOLVE_SETUP_ONLY, no_setup = params->flags & RWB_SOLVE_NO_SETUP;
  if ((setup_only || no_setup) && (!resident || (setup_only && no_setup)))
    return fail(RWB_ERR_INVALID, "SETUP_ONLY / NO_SETUP: one of them, and only where the brick-resident engine runs");
  SetupMaps maps;
  if (no_setup) {
    // the workspace already holds this level's system (an earlier SETUP_ONLY call, same arguments)
  } else {
  // zero the scalar region (rr .. misc) in one memset
  RWB_CUDA(cudaMemsetAsync((char*)workspace + L.off[L_RR], 0, L.total - L.off[L_RR], st));
  if (!(params->flags & RWB_SOLVE_SETUP2) && !g.is3d && g.by == ST2 && g.bx == ST2) {
    setup_tile2d_kernel<<<nb, STH2, 0, st>>>(g, w, list, intensity, seeds, bound, params->beta, params->min_weight,
                                             tol2, max_iter, resident ? 0 : 1);
    RWB_LAUNCH_CHECK("2-D tile setup kernel");
  } else if (!(params->flags & RWB_SOLVE_SETUP2) && make_setup_maps(g, intensity, seeds, bound, &maps)) {
    static DeviceCache smem_set;
    int dev = 0;
    if ((rc = device_slot(&dev))) return rc;
    if (!smem_set[dev].load(std::memory_order_relaxed)) {
      RWB_CUDA(cudaFuncSetAttribute(setup_brick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sizeof(SetupSmem)));
      smem_set[dev].store(1, std::memory_order_relaxed);
    }
    setup_brick_kernel<<<nb, STH, sizeof(SetupSmem), st>>>(maps, g, w, list, bound != nullptr, params->beta,
                                                                   params->min_weight, tol2, max_iter,
                                                                   resident ? 0 : 1);
    RWB_LAUNCH_CHECK("fused setup kernel");
  } else {
    setup_scale_kernel<<<setup_grid, block, 0, st>>>(g, w, list, intensity, seeds, params->beta, params->min_weight);
    setup_system_kernel<<<setup_grid, block, 0, st>>>(g, w, list, intensity, seeds, bound, params->beta,
                                                      params->min_weight, tol2, max_iter, resident ? 0 : 1);
  }
  advance_kernel<<<1, 1024, 0, st>>>(w, nb, 0);
  RWB_LAUNCH_CHECK("setup kernels");
  count_launches(3);
  if (resident) {
    // bricks the setup settled are finished here; the engine writes its own bricks' results
    settled_epilogue_kernel<<<grid, block, 0, st>>>(g, w, list, nb, prob, labels);
    RWB_LAUNCH_CHECK("settled epilogue");
    count_launches(1);
  }
  }
  if (setup_only) return RWB_OK;

  if (resident) {
    // every CG iteration of a brick on chip: one 4-CTA cluster per 32^3 brick (cluster=8/16: 8- or 16-CTA variants)
    ResidentArgs ra;
    ra.wx = w.wx;
    ra.wy = w.wy;
    ra.wz = w.wz;
    ra.r0 = w.r;
    ra.y = w.y;
    ra.bb = w.bb;
    ra.alist = w.alist;
    ra.n_active = w.n_active;
    ra.state = w.state;
    ra.iters = w.iters;
    ra.next = w.next;
    ra.tol2 = tol2;
    ra.max_iter = max_iter;
    ra.sc = w.sc;
    ra.prob = prob;
    ra.labels = labels;
    ra.list = list;
    ra.nz = g.nz, ra.ny = g.ny, ra.nx = g.nx;
    ra.oz = g.oz, ra.oy = g.oy, ra.ox = g.ox;
    ra.gy = g.gy, ra.gx = g.gx;
    ra.coarse = !(params->flags & RWB_SOLVE_NO_COARSE);
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    RWB_CUDA(cudaEventCreate(&ev0));
    RWB_CUDA(cudaEventCreate(&ev1));
    RWB_CUDA(cudaEventRecord(ev0, st));
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp, w.next);  // also re-arms the brick counter
    if (g.is3d)
      rc = launch_resident3d(ra, nb, (params->flags & RWB_SOLVE_CLUSTER4) ? 4 : (params->flags & RWB_SOLVE_CLUSTER16) ? 16 : ((params->flags & RWB_SOLVE_SPLIT_Z) ? 512 : 8),
                             st);
    else
      rc = launch_resident2d(ra, nb, st);
    if (rc) {
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      return rc;
    }
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp + 1);
    count_launches(2);
    RWB_CUDA(cudaEventRecord(ev1, st));
    stats_kernel<<<1, 1024, 0, st>>>(w, nb);
    RWB_LAUNCH_CHECK("resident solve epilogue");
    count_launches(2);
    if (stats) {
      rc = read_stats(w, nb, st, ev0, ev1, 0, RWB_PATH_RESIDENT, stats, -1.f, dev_stats);
      if (rc) return rc;
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return RWB_OK;
  }

  // multigrid for large whole levels (128^3: 6.5 vs 13.3 ms); below ~2^19 voxels Jacobi-PCG is
  // faster (64^3: 1.6 vs 1.9 ms, 64^2: 0.6 vs 0.8 ms; tools/mg_small_probe.py)
  constexpr long long kMgMinVoxels = 1LL << 19;
  const bool use_mg = !(params->flags & RWB_SOLVE_NO_MG) && ((params->flags & RWB_SOLVE_MG) || g.bvol >= kMgMinVoxels);
  if (total == 1 && use_mg) {
    // whole-level solve: multigrid-preconditioned CG, all iterations in one cooperative launch
    MgArgs ma;
    std::memset(&ma, 0, sizeof(ma));
    mg_carve(&ma, (char*)workspace + L.off[L_MG], g.bz, g.by, g.bx);
    ma.nz = g.bz, ma.ny = g.by, ma.nx = g.bx;
    ma.wx = w.wx;
    ma.wy = w.wy;
    ma.wz = w.wz;
    ma.sc = w.sc;
    ma.y = w.y;
    ma.r[0] = w.r;
    ma.r[1] = w.p1;
    ma.p = w.p0;
    ma.q = w.q;
    ma.bb = w.bb;
    ma.rr0 = w.rr;
    ma.state = w.state;
    ma.iters = w.iters;
    ma.tol2 = tol2;
    ma.max_iter = max_iter;
    ma.omega = 0.8f;
    ma.bottom_sweeps = 8;  // an exact (dense-inverse) bottom solve was tried: no fewer iterations
    ma.intensity = intensity;
    ma.seeds = seeds;
    ma.beta = params->beta;
    ma.min_weight = params->min_weight;
    ma.trace = mg_trace_buffer();
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    RWB_CUDA(cudaEventCreate(&ev0));
    RWB_CUDA(cudaEventCreate(&ev1));
    RWB_CUDA(cudaEventRecord(ev0, st));
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp);
    rc = launch_mgcg(ma, st);
    if (rc) {
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      return rc;
    }
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp + 1);
    count_launches(2);
    RWB_CUDA(cudaEventRecord(ev1, st));
    epilogue_kernel<<<sgrid, block, 0, st>>>(g, w, list, prob, labels);
    stats_kernel<<<1, 1024, 0, st>>>(w, nb);
    RWB_LAUNCH_CHECK("multigrid solve");
    count_launches(2);
    if (stats) {
      rc = read_stats(w, nb, st, ev0, ev1, 0, RWB_PATH_MULTIGRID, stats, -1.f, dev_stats);
      if (rc) return rc;
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return RWB_OK;
  }

  if (total == 1 && !(params->flags & RWB_SOLVE_NO_COOP)) {
    // whole-level solve: all iterations in one cooperative launch
    int cgrid = 0;
    rc = coop_grid(&cgrid);
    if (rc) return rc;
    // work items of kCoopTZ planes, spread evenly: every block gets the same number
    int n_items = ((g.bz + kCoopTZ - 1) / kCoopTZ) * g.ty * g.tx;
    const int rounds = (n_items + cgrid - 1) / cgrid;
    cgrid = (n_items + rounds - 1) / rounds;
    float* part_pq = reinterpret_cast<float*>(w.part);
    float* part_rr = part_pq + kCoopMaxBlocks;
    float tol2v = tol2;
    int max_iter_v = max_iter;
    void* args[] = {&g, &w, &part_pq, &part_rr, &n_items, &tol2v, &max_iter_v};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    RWB_CUDA(cudaEventCreate(&ev0));
    RWB_CUDA(cudaEventCreate(&ev1));
    RWB_CUDA(cudaEventRecord(ev0, st));
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp);
    RWB_CUDA(cudaLaunchCooperativeKernel((const void*)coop_cg_kernel, dim3(cgrid), block, args, 0, st));
    stamp_kernel<<<1, 1, 0, st>>>(w.stamp + 1);
    count_launches(2);
    RWB_CUDA(cudaEventRecord(ev1, st));
    epilogue_kernel<<<sgrid, block, 0, st>>>(g, w, list, prob, labels);
    stats_kernel<<<1, 1024, 0, st>>>(w, nb);
    RWB_LAUNCH_CHECK("cooperative solve");
    count_launches(3);
    if (stats) {
      rc = read_stats(w, nb, st, ev0, ev1, 0, RWB_PATH_COOPERATIVE, stats, -1.f, dev_stats);
      if (rc) return rc;
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return RWB_OK;
  }

  int* host = nullptr;
  rc = pinned(&host);
  if (rc) return rc;
  rc = readback(st, w.n_active, 0, 1);
  if (rc) return rc;
  int active = host[0];

  cudaGraphExec_t exec = nullptr;
  const bool use_graph = !(params->flags & RWB_SOLVE_NO_GRAPH);
  if (use_graph && active > 0) {
    cudaStream_t cap;
    RWB_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      rc = launch_chunk(g, w, nb, list, k, tol2, max_iter, grid, cap);
      cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
      if (e2 != cudaSuccess) e = e2;
      if (rc == RWB_OK && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
    }
    cudaStreamDestroy(cap);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "graph capture of the CG iterations");
  }

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  RWB_CUDA(cudaEventCreate(&ev0));
  RWB_CUDA(cudaEventCreate(&ev1));
  float cg_ms = 0.f;
  int sweeps = 0;
  while (active > 0 && sweeps < max_iter) {
    RWB_CUDA(cudaEventRecord(ev0, st));
    if (exec) {
      cudaError_t e = cudaGraphLaunch(exec, st);
      if (e != cudaSuccess) {
        cudaGraphExecDestroy(exec);
        return cuda_fail(e, "cudaGraphLaunch");
      }
    } else {
      rc = launch_chunk(g, w, nb, list, k, tol2, max_iter, grid, st);
      if (rc) return rc;
    }
    sweeps += k;
    count_launches(2 * k + 1);
    cudaError_t e = cudaEventRecord(ev1, st);
    if (e == cudaSuccess) {
      readback_kernel<<<1, 32, 0, st>>>(t_pinned.dev, w.n_active, 1);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev0, ev1);
    if (e != cudaSuccess) {
      if (exec) cudaGraphExecDestroy(exec);
      cudaEventDestroy(ev0);
      cudaEventDestroy(ev1);
      return cuda_fail(e, "convergence poll");
    }
    cg_ms += ms;
    active = host[0];
  }
  if (exec) cudaGraphExecDestroy(exec);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);

  finalize_kernel<<<(nb + 255) / 256, 256, 0, st>>>(w, nb);
  epilogue_kernel<<<sgrid, block, 0, st>>>(g, w, list, prob, labels);
  stats_kernel<<<1, 1024, 0, st>>>(w, nb);
  RWB_LAUNCH_CHECK("epilogue kernels");
  count_launches(3);
  if (stats) {
    rc = read_stats(w, nb, st, nullptr, nullptr, sweeps, RWB_PATH_STREAMING, stats, cg_ms, dev_stats);
    if (rc) return rc;
  }
  return RWB_OK;
}
