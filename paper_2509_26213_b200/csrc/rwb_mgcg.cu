// Whole-level (coarsest) random-walker solve: multigrid-preconditioned CG, all iterations in ONE
// cooperative kernel.
//
// Why: the coarsest level of a hierarchy (128^3 at configs 2 and 4) is one Dirichlet problem with
// 2M unknowns; Jacobi-PCG needs ~550 iterations there, each a chain of grid-wide dependencies, and
// its cost (13 ms at 24 us per iteration) is replicated on every GPU of a multi-GPU run.  A V-cycle
// preconditioner cuts the iterations ~10x for 3 fine sweeps per iteration, and its coarse levels
// are tiny.
//
// The system is the one the setup kernels build for the single brick (rwb_solve.cu): A' = S L_UU S
// with unit diagonal on the unknowns, forward weights w' (0 across Dirichlet nodes and the level
// border), s = 0 off the unknowns, r0 / y0 / ||S b||^2.  CG runs on A' y = S b exactly as the
// Jacobi-PCG kernel does (same stop rule ||r|| <= tol ||S b||), with z = M r from:
//
//   hierarchy  level c+1 aggregates the 2x2x2 blocks of level c (ceil sizes).  Inside each block
//              only the largest set of children joined by STRONG edges (w_ij >= 0.01 min(d_i, d_j))
//              is prolongated to (cmask); the other children get no coarse correction.  Without
//              the mask, a block straddling a w_min boundary (the rim of an unseeded blob) injects
//              the outside's correction into the blob, whose error mode is invisible to the
//              residual (it couples through w_min edges only): the solve then "converges" with
//              ~3e-3 error inside the blob (config 1, seeds S2).  Galerkin operator of the masked
//              piecewise-constant prolongation P: face weights = sums of the strong-side fine
//              weights between included children, diagonal = leak + the six face weights, where
//              leak = the included children's Dirichlet couplings plus their weights to excluded
//              cells (assembled WITHOUT cancellation; the textbook "sum of diagonals - internal
//              weights" cancels catastrophically in fp32 for w_min pockets).  Every level is a
//              diagonally dominant M-matrix (SPD); aggregates without included children have
//              dinv = 0.
//   V(1,1)     pre-smooth x_c = w D^-1 b_c (one damped-Jacobi step from 0), restrict the residual
//              b_{c+1} = P^T (b_c - A_c x_c), recurse; bottom = damped-Jacobi sweeps; correct
//              x_c += P x_{c+1}, post-smooth one damped-Jacobi step.  Symmetric and positive
//              definite (w = 0.8 < 1, Jacobi on a diagonally dominant M-matrix), a fixed linear
//              operator: a valid CG preconditioner, deterministic (no atomics, fixed-order sums).
//
// Execution: levels with more than kMgSmemCells aggregates run grid-wide (2 z x 2 y rows x 32 x
// per warp item, neighbours through L1: after a grid barrier's acquire the SM's L1 holds no stale
// lines, so vectors written by other CTAs in this launch are read with ordinary cached loads; only
// the setup's read-only arrays use the non-coherent path).  The small levels are built and cycled
// REDUNDANTLY by every CTA in its own shared memory (bit-identical in every CTA), so the coarse
// solve needs no grid barrier at all: per iteration 2 * grid_levels + 1 barriers.  The pre-smoothed
// x_c is never stored (recomputed from b where a neighbour needs it), the CG update r <- r - alpha q
// / y <- y + alpha p is fused into the next restriction (r double buffered), and q = A'z + beta q
// replaces A'p.  Reductions: per-thread float64, fixed-order warp / block / grid sums; every block
// reduces all block partials itself, so all blocks take the same decisions.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"

namespace rwb {

constexpr int MG_THREADS = 1024;
constexpr int MG_WARPS = MG_THREADS / 32;
constexpr int kMgSmemCells = 512;  // aggregate levels at or below this many cells live in shared memory
                                   // (4096: 8% slower at 128^3, the shared-memory carve-out starves L1)
constexpr size_t kMgSmemMax = 200 * 1024;  // the shared-memory levels' arrays

constexpr int kMgBottomCells = 64;  // stop coarsening at or below this many cells
constexpr int kMgSmemArrays = 8;    // dinv, wx, wy, wz, b, x, t (residual / bottom buffer / leak), cmask
constexpr float kMgStrong = 0.01f;  // strong edge: w_ij >= kMgStrong * min(d_i, d_j)

struct Dims {
  int nz, ny, nx;
  __device__ __host__ int cells() const { return nz * ny * nx; }
};

__device__ __forceinline__ int at(const Dims& d, int z, int y, int x) { return (z * d.ny + y) * d.nx + x; }

__device__ __forceinline__ void cell_of(const Dims& d, int i, int& z, int& y, int& x) {
  x = i % d.nx;
  const int t = i / d.nx;
  y = t % d.ny;
  z = t / d.ny;
}

// the same for the shared-memory levels' per-iteration loops (cells < 2^22): quotients from a float
// reciprocal with one correction step instead of the ~20-instruction integer division sequence
__device__ __forceinline__ int fdivmod(int i, int n, float rn, int& r) {
  int q = __float2int_rz((float)i * rn);
  r = i - q * n;
  if (r < 0) {
    --q;
    r += n;
  } else if (r >= n) {
    ++q;
    r -= n;
  }
  return q;
}
__device__ __forceinline__ void cell_of_fast(const Dims& d, int i, int& z, int& y, int& x) {
  const int t = fdivmod(i, d.nx, 1.f / (float)d.nx, x);
  z = fdivmod(t, d.ny, 1.f / (float)d.ny, y);
}

// child bit of cell (z, y, x) of level c in the cmask of its aggregate on level c+1
__device__ __forceinline__ int child_bit(int z, int y, int x) { return ((z & 1) << 2) | ((y & 1) << 1) | (x & 1); }

// ---------------------------------------------------------------------------
// grid barrier (one counter, monotonically increasing within the launch) and reductions

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// publish this block's partial (slot k): fixed-order xor trees, warps' sums in order (warp 0)
__device__ __forceinline__ void put_partial(double* part, int k, double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = sh[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) part[k * kMgMaxBlocks + blockIdx.x] = t;
  }
  // sh is rewritten only after the grid barrier that must follow
}
// ... and, after a grid barrier, the sum of all blocks' partials: every warp reduces them itself in
// the same fixed order (no block synchronisation), so every thread of every block holds the same bits
__device__ __forceinline__ double grid_total(const double* part, int k) {
  const int lane = threadIdx.x & 31;
  double v = 0.0;
  for (int b = lane; b < (int)gridDim.x; b += 32) v += part[k * kMgMaxBlocks + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// 7-point stencil helpers.  W(k, i) = forward weight of dim k (0 = x, 1 = y, 2 = z) at cell i;
// sum_j w_ij v(j) over the in-level neighbours of (z, y, x).

template <class WF, class VF>
__device__ __forceinline__ float nbr_sum(const Dims& d, int i, int z, int y, int x, WF W, VF v, float s) {
  const int sz = d.nx * d.ny;
  if (x + 1 < d.nx) s = fmaf(W(0, i), v(i + 1, z, y, x + 1), s);
  if (x > 0) s = fmaf(W(0, i - 1), v(i - 1, z, y, x - 1), s);
  if (y + 1 < d.ny) s = fmaf(W(1, i), v(i + d.nx, z, y + 1, x), s);
  if (y > 0) s = fmaf(W(1, i - d.nx), v(i - d.nx, z, y - 1, x), s);
  if (z + 1 < d.nz) s = fmaf(W(2, i), v(i + sz, z + 1, y, x), s);
  if (z > 0) s = fmaf(W(2, i - sz), v(i - sz, z - 1, y, x), s);
  return s;
}

// children mask of aggregate (Z, Y, X) over level f: the largest strongly connected set of live
// children (d > 0); ties -> the set holding the lowest child index
template <class DG, class WF>
__device__ unsigned agg_mask(const Dims& f, int Z, int Y, int X, DG dgf, WF W) {
  float d[8];
  unsigned live = 0, adj[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    adj[k] = 0;
    d[k] = 0.f;
    const int z = 2 * Z + (k >> 2), y = 2 * Y + ((k >> 1) & 1), x = 2 * X + (k & 1);
    if (z < f.nz && y < f.ny && x < f.nx) {
      d[k] = dgf(at(f, z, y, x));
      if (d[k] > 0.f) live |= 1u << k;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!((live >> k) & 1)) continue;
    const int z = 2 * Z + (k >> 2), y = 2 * Y + ((k >> 1) & 1), x = 2 * X + (k & 1);
    const int i = at(f, z, y, x);
#pragma unroll
    for (int dim = 0; dim < 3; ++dim) {
      const int bit = 1 << dim;  // x: 1, y: 2, z: 4
      if (k & bit) continue;
      const int o = k | bit;
      if (!((live >> o) & 1)) continue;
      if (W(dim, i) >= kMgStrong * fminf(d[k], d[o])) {
        adj[k] |= 1u << o;
        adj[o] |= 1u << k;
      }
    }
  }
  unsigned best = 0, rem = live;
  while (rem) {
    unsigned comp = rem & (0u - rem);
    for (;;) {
      unsigned nc = comp;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if ((comp >> k) & 1) nc |= adj[k];
      if (nc == comp) break;
      comp = nc;
    }
    if (__popc(comp) > __popc(best)) best = comp;
    rem &= ~comp;
  }
  return best;
}

// Galerkin aggregate (Z, Y, X) of the next level with children mask M: leak = included children's
// leaks + their weights to excluded cells, forward face weights = weights between included children
// across the +x / +y / +z faces (float64 sums of non-negative terms).  MB(z, y, x) = cell's mask bit.
template <class LK, class WF, class MB>
__device__ void aggregate_cell(const Dims& f, int Z, int Y, int X, unsigned M, LK leakf, WF W, MB mbit,
                               float& cleak, float& cwx, float& cwy, float& cwz) {
  double lk = 0.0, fw[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < 8; ++k) {
    if (!((M >> k) & 1)) continue;
    const int z = 2 * Z + (k >> 2), y = 2 * Y + ((k >> 1) & 1), x = 2 * X + (k & 1);
    const int i = at(f, z, y, x);
    lk += (double)leakf(i);
    const int c[3] = {x, y, z};
    const int n[3] = {f.nx, f.ny, f.nz};
    const int st[3] = {1, f.nx, f.nx * f.ny};
#pragma unroll
    for (int dim = 0; dim < 3; ++dim) {
      if (c[dim] > 0) {  // backward edge
        const float w = W(dim, i - st[dim]);
        if (w > 0.f && !mbit(dim == 2 ? z - 1 : z, dim == 1 ? y - 1 : y, dim == 0 ? x - 1 : x)) lk += (double)w;
      }
      if (c[dim] + 1 < n[dim]) {  // forward edge
        const float w = W(dim, i);
        if (w > 0.f) {
          if (!mbit(dim == 2 ? z + 1 : z, dim == 1 ? y + 1 : y, dim == 0 ? x + 1 : x))
            lk += (double)w;
          else if (k & (1 << dim))
            fw[dim] += (double)w;  // the child on the + face: the edge leaves the aggregate
        }
      }
    }
  }
  cleak = (float)lk;
  cwx = (float)fw[0];
  cwy = (float)fw[1];
  cwz = (float)fw[2];
}

// 1 / (leak + the six face weights) of cell i of a level, 0 where that is 0 (nothing included)
template <class WF>
__device__ __forceinline__ float aggregate_dinv(const Dims& d, int i, float leak, WF W) {
  int z, y, x;
  cell_of(d, i, z, y, x);
  double dg = (double)leak + W(0, i) + W(1, i) + W(2, i);
  if (x > 0) dg += W(0, i - 1);
  if (y > 0) dg += W(1, i - d.nx);
  if (z > 0) dg += W(2, i - d.nx * d.ny);
  return dg > 0.0 ? (float)(1.0 / dg) : 0.f;
}

__device__ __forceinline__ void stamp(const MgArgs& a, int it, int k) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && it < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[it * 16 + k] = t;
  }
}

// ---------------------------------------------------------------------------
// grid-wide work items: a SEG-lane segment of a warp covers SEG x-columns of a (2 z) x (2 y) block
// of rows (4 cells per lane); a warp takes 32 / SEG consecutive items per step (uniform trip count).
// SEG = 16 balances the warps of a 128^3 level to ~1.5% (32768 items over 4736 warps) where
// SEG = 32 leaves up to 25% of them idle in the last round; SEG = 32 reads whole 128-byte rows.

struct Item {
  int z0, y0, x;
  bool ok;  // x inside the level and the item exists
};
template <int SEG>
__device__ __forceinline__ int n_items(const Dims& d) {
  return ((d.nz + 1) >> 1) * ((d.ny + 1) >> 1) * ((d.nx + SEG - 1) / SEG);
}
template <int SEG>
__device__ __forceinline__ Item item_of(const Dims& d, int base, int ni) {
  const int lane = threadIdx.x & 31;
  const int item = base + lane / SEG;
  const int nxs = (d.nx + SEG - 1) / SEG, nyh = (d.ny + 1) >> 1;
  Item it;
  const int xs = item % nxs;
  const int t = item / nxs;
  it.y0 = 2 * (t % nyh);
  it.z0 = 2 * (t / nyh);
  it.x = xs * SEG + lane % SEG;
  it.ok = item < ni && it.x < d.nx;
  return it;
}

// f(i, z, y) for each of the item's (up to) 4 cells, in (dz, dy) order.  Each phase evaluates a
// cell's own value and its 6 neighbours as independent loads (through L1) and finishes the cell
// before the next: the phases are latency-bound at 64 registers per thread, so memory-level
// parallelism and short live ranges beat fewer loads (variants that computed the 4 cells' values
// first and shared x +- 1 through lane shuffles were 1.1-1.4x slower).
template <class F>
__device__ __forceinline__ void for_cells(const Dims& d, const Item& t, F f) {
  if (!t.ok) return;
#pragma unroll
  for (int dz = 0; dz < 2; ++dz) {
    const int z = t.z0 + dz;
    if (z >= d.nz) break;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      const int y = t.y0 + dy;
      if (y >= d.ny) break;
      f(at(d, z, y, t.x), z, y);
    }
  }
}

// ---------------------------------------------------------------------------
// shared-memory levels (every CTA holds its own, identical copy)

struct SLv {
  Dims d;
  float *dinv, *wx, *wy, *wz, *b, *x, *t;
  uint8_t* cm;  // cmask of this level's aggregates (children on the level below)
  __device__ __forceinline__ float w(int k, int i) const { return (k == 0 ? wx : k == 1 ? wy : wz)[i]; }
};

// ---------------------------------------------------------------------------
// the kernel

template <int SEG>
__global__ void __launch_bounds__(MG_THREADS, 1) mgcg_kernel(const __grid_constant__ MgArgs a) {
  extern __shared__ float smem[];
  __shared__ double red[MG_WARPS];
  const float omega = a.omega;
  const int warp_g = blockIdx.x * MG_WARPS + (threadIdx.x >> 5);
  const int warps = gridDim.x * MG_WARPS;
  const int gl = a.grid_levels;
  const int gtid = blockIdx.x * MG_THREADS + threadIdx.x;
  const int gstride = gridDim.x * MG_THREADS;
  unsigned bar = 0;
  const Dims fd{a.nz, a.ny, a.nx};
  auto dims = [&](int c) { return c == 0 ? fd : Dims{a.lv[c].nz, a.lv[c].ny, a.lv[c].nx}; };
  stamp(a, 0, 14);  // launch

  // fine weights: written before the launch (non-coherent path); grid-level weights: this launch
  auto Wf = [&](int k, int i) { return __ldg((k == 0 ? a.wx : k == 1 ? a.wy : a.wz) + i); };
  auto Wg = [&](int c) {
    const MgLevel& L = a.lv[c];
    return [&L](int k, int i) { return (k == 0 ? L.wx : k == 1 ? L.wy : L.wz)[i]; };
  };
  // mask bit of cell (z, y, x) of level c (its aggregate lives on level c+1, cmask in global memory)
  auto mbit_g = [&](int c) {
    const uint8_t* cm = a.lv[c + 1].cmask;
    const Dims cd = dims(c + 1);
    return [cm, cd](int z, int y, int x) { return (cm[at(cd, z >> 1, y >> 1, x >> 1)] >> child_bit(z, y, x)) & 1; };
  };

  // ---- shared-memory level layout: level c's arrays follow those of levels gl .. c-1
  auto S = [&](int c) {
    float* p = smem;
    for (int k = gl; k < c; ++k) p += a.lv[k].nz * a.lv[k].ny * a.lv[k].nx * kMgSmemArrays;
    SLv L;
    L.d = Dims{a.lv[c].nz, a.lv[c].ny, a.lv[c].nx};
    const int n = L.d.cells();
    L.dinv = p;
    L.wx = p + n;
    L.wy = p + 2 * n;
    L.wz = p + 3 * n;
    L.b = p + 4 * n;
    L.x = p + 5 * n;
    L.t = p + 6 * n;
    L.cm = reinterpret_cast<uint8_t*>(p + 7 * n);
    return L;
  };

  // ---- build the Galerkin hierarchy.  Fine cells' leak = s_i^2 * (weights to seeded neighbours),
  // the Dirichlet coupling of the scaled system, from the same edge weights the setup used.
  auto fine_leak = [&](int j) -> float {
    const float s = __ldg(a.sc + j);
    if (!(s > 0.f)) return 0.f;
    int z, y, x;
    cell_of(fd, j, z, y, x);
    const float Ii = __ldg(a.intensity + j);
    float acc = 0.f;
    const int sz = fd.nx * fd.ny;
    if (x > 0 && a.seeds[j - 1]) acc += edge_weight(Ii, __ldg(a.intensity + j - 1), a.beta, a.min_weight);
    if (x + 1 < fd.nx && a.seeds[j + 1]) acc += edge_weight(Ii, __ldg(a.intensity + j + 1), a.beta, a.min_weight);
    if (y > 0 && a.seeds[j - fd.nx]) acc += edge_weight(Ii, __ldg(a.intensity + j - fd.nx), a.beta, a.min_weight);
    if (y + 1 < fd.ny && a.seeds[j + fd.nx])
      acc += edge_weight(Ii, __ldg(a.intensity + j + fd.nx), a.beta, a.min_weight);
    if (z > 0 && a.seeds[j - sz]) acc += edge_weight(Ii, __ldg(a.intensity + j - sz), a.beta, a.min_weight);
    if (z + 1 < fd.nz && a.seeds[j + sz]) acc += edge_weight(Ii, __ldg(a.intensity + j + sz), a.beta, a.min_weight);
    return acc * s * s;
  };
  auto fine_dg = [&](int j) { return __ldg(a.sc + j) > 0.f ? 1.f : 0.f; };

  // grid-wide: the masks of levels 1 .. gl (level gl's mask is read by the grid-wide passes of level
  // gl-1) and the aggregates of levels 1 .. gl-1
  for (int c = 1; c <= gl; ++c) {
    const Dims pd = dims(c - 1), cd = dims(c);
    const int n = cd.cells();
    uint8_t* cm = a.lv[c].cmask;
    for (int i = gtid; i < n; i += gstride) {
      int Z, Y, X;
      cell_of(cd, i, Z, Y, X);
      if (c == 1) {
        cm[i] = (uint8_t)agg_mask(pd, Z, Y, X, fine_dg, Wf);
      } else {
        const MgLevel& P = a.lv[c - 1];
        cm[i] = (uint8_t)agg_mask(
            pd, Z, Y, X, [&](int j) { return P.dinv[j] > 0.f ? 1.f / P.dinv[j] : 0.f; }, Wg(c - 1));
      }
    }
    grid_barrier(a.barrier, bar);
    if (c == gl) break;  // level gl itself is built in shared memory by every CTA
    const MgLevel& C = a.lv[c];
    for (int i = gtid; i < n; i += gstride) {
      int Z, Y, X;
      cell_of(cd, i, Z, Y, X);
      float lk, wx, wy, wz;
      if (c == 1) {
        aggregate_cell(pd, Z, Y, X, cm[i], fine_leak, Wf, mbit_g(0), lk, wx, wy, wz);
      } else {
        const MgLevel& P = a.lv[c - 1];
        aggregate_cell(pd, Z, Y, X, cm[i], [&](int j) { return P.leak[j]; }, Wg(c - 1), mbit_g(c - 1), lk, wx, wy,
                       wz);
      }
      C.leak[i] = lk;
      C.wx[i] = wx;
      C.wy[i] = wy;
      C.wz[i] = wz;
    }
    grid_barrier(a.barrier, bar);
    for (int i = gtid; i < n; i += gstride) C.dinv[i] = aggregate_dinv(cd, i, C.leak[i], Wg(c));
    grid_barrier(a.barrier, bar);
  }
  // every CTA: the shared-memory levels gl .. nlev-1 (built once, resident for the whole solve)
  for (int c = gl; c < a.nlev; ++c) {
    const SLv C = S(c);
    const Dims pd = dims(c - 1);
    const int n = C.d.cells();
    if (c > gl) {  // masks of the shared-memory aggregates (level gl's came from the grid phase)
      const SLv P = S(c - 1);
      for (int i = threadIdx.x; i < n; i += MG_THREADS) {
        int Z, Y, X;
        cell_of(C.d, i, Z, Y, X);
        C.cm[i] = (uint8_t)agg_mask(
            pd, Z, Y, X, [&](int j) { return P.dinv[j] > 0.f ? 1.f / P.dinv[j] : 0.f; },
            [&](int k, int j) { return P.w(k, j); });
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += MG_THREADS) {
      int Z, Y, X;
      cell_of(C.d, i, Z, Y, X);
      float lk, wx, wy, wz;
      if (c == gl) {
        const unsigned M = a.lv[gl].cmask[i];
        if (c == 1) {
          aggregate_cell(pd, Z, Y, X, M, fine_leak, Wf, mbit_g(0), lk, wx, wy, wz);
        } else {
          const MgLevel& P = a.lv[c - 1];
          aggregate_cell(pd, Z, Y, X, M, [&](int j) { return P.leak[j]; }, Wg(c - 1), mbit_g(c - 1), lk, wx, wy,
                         wz);
        }
      } else {
        const SLv P = S(c - 1);  // the parent's leak is kept in its t while building
        const uint8_t* cm = C.cm;
        const Dims cd = C.d;
        aggregate_cell(
            pd, Z, Y, X, C.cm[i], [&](int j) { return P.t[j]; }, [&](int k, int j) { return P.w(k, j); },
            [cm, cd](int z, int y, int x) { return (cm[at(cd, z >> 1, y >> 1, x >> 1)] >> child_bit(z, y, x)) & 1; },
            lk, wx, wy, wz);
      }
      C.t[i] = lk;
      C.wx[i] = wx;
      C.wy[i] = wy;
      C.wz[i] = wz;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += MG_THREADS)
      C.dinv[i] = aggregate_dinv(C.d, i, C.t[i], [&](int k, int j) { return C.w(k, j); });
    __syncthreads();
  }

  // ---- CG state
  const double bb = *a.bb;
  double rr = *a.rr0;
  int state = ST_ACTIVE;
  if (bb <= 0.0)
    state = ST_ZERO;
  else if (rr <= (double)a.tol2 * bb)
    state = ST_CONVERGED;
  else if (a.max_iter <= 0)
    state = ST_MAXITER;
  int it = 0;
  double rz_old = 0.0, alpha = 0.0;
  int cur = 0;  // r[cur] holds the current residual

  stamp(a, 0, 15);  // hierarchy built
  while (state == ST_ACTIVE) {
    stamp(a, it, 0);
    // ===== DOWN 0 (fused with the CG update of the previous iteration):
    //   r_new = r - alpha q, y += alpha p (alpha = 0 on the first pass: r = r0), ||r_new||^2,
    //   b_1 = P^T (r_new - A' w r_new)   (D = I on the unknowns; r = 0 elsewhere)
    {
      const float* R = a.r[cur];
      float* RN = a.r[cur ^ 1];
      const float* Q = a.q;
      const float al = (float)alpha;
      const bool upd = it > 0;
      auto rn = [&](int j, int, int, int) { return upd ? fmaf(-al, Q[j], R[j]) : R[j]; };
      const Dims cd = dims(1);
      const uint8_t* cm = a.lv[1].cmask;
      float* BN = a.lv[1].b;
      double acc = 0.0;
      const int ni = n_items<SEG>(fd);
      for (int base = (32 / SEG) * warp_g; base < ni; base += (32 / SEG) * warps) {
        const Item t = item_of<SEG>(fd, base, ni);
        const unsigned M = t.ok ? cm[at(cd, t.z0 >> 1, t.y0 >> 1, t.x >> 1)] : 0u;
        float sum = 0.f;
        for_cells(fd, t, [&](int i, int z, int y) {
          const float r_i = rn(i, z, y, t.x);
          if (upd) {
            RN[i] = r_i;
            a.y[i] = fmaf(al, a.p[i], a.y[i]);
          }
          acc += (double)r_i * (double)r_i;
          if ((M >> child_bit(z, y, t.x)) & 1)
            sum += fmaf(1.f - omega, r_i, omega * nbr_sum(fd, i, z, y, t.x, Wf, rn, 0.f));
        });
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        if (t.ok && !(t.x & 1)) BN[at(cd, t.z0 >> 1, t.y0 >> 1, t.x >> 1)] = sum;
      }
      if (upd) put_partial(a.part, 0, acc, red);
      if (upd) cur ^= 1;
    }
    stamp(a, it, 1);
    grid_barrier(a.barrier, bar);
    stamp(a, it, 2);
    if (it > 0) {
      rr = grid_total(a.part, 0);
      if (rr <= (double)a.tol2 * bb) {
        state = ST_CONVERGED;
        break;
      }
      if (it >= a.max_iter) {
        state = ST_MAXITER;
        break;
      }
    }

    // ===== DOWN c = 1 .. gl-1 (grid-wide): b_{c+1} = P^T (b_c - A_c w D^-1 b_c)
    for (int c = 1; c < gl; ++c) {
      const MgLevel& L = a.lv[c];
      const Dims d = dims(c), cd = dims(c + 1);
      const float* B = L.b;
      const float* DI = L.dinv;
      float* BN = a.lv[c + 1].b;
      const uint8_t* cm = a.lv[c + 1].cmask;
      auto W = Wg(c);
      auto v = [&](int j, int, int, int) { return DI[j] * B[j]; };
      const int ni = n_items<SEG>(d);
      for (int base = (32 / SEG) * warp_g; base < ni; base += (32 / SEG) * warps) {
        const Item t = item_of<SEG>(d, base, ni);
        const unsigned M = t.ok ? cm[at(cd, t.z0 >> 1, t.y0 >> 1, t.x >> 1)] : 0u;
        float sum = 0.f;
        for_cells(d, t, [&](int i, int z, int y) {
          if ((M >> child_bit(z, y, t.x)) & 1)
            sum += fmaf(1.f - omega, B[i], omega * nbr_sum(d, i, z, y, t.x, W, v, 0.f));
        });
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        if (t.ok && !(t.x & 1)) BN[at(cd, t.z0 >> 1, t.y0 >> 1, t.x >> 1)] = sum;
      }
      grid_barrier(a.barrier, bar);
    }

    stamp(a, it, 3);
    // ===== every CTA: the shared-memory levels, down, bottom, up (identical in every CTA)
    {
      {
        const SLv L = S(gl);
        const float* src = a.lv[gl].b;
        for (int i = threadIdx.x; i < L.d.cells(); i += MG_THREADS) L.b[i] = src[i];
        __syncthreads();
      }
      for (int c = gl; c + 1 < a.nlev; ++c) {
        const SLv L = S(c);
        const SLv N = S(c + 1);
        auto v = [&](int j, int, int, int) { return L.dinv[j] * L.b[j]; };
        auto W = [&](int k, int j) { return L.w(k, j); };
        for (int i = threadIdx.x; i < L.d.cells(); i += MG_THREADS) {
          int z, y, x;
          cell_of_fast(L.d, i, z, y, x);
          L.t[i] = fmaf(1.f - omega, L.b[i], omega * nbr_sum(L.d, i, z, y, x, W, v, 0.f));
        }
        __syncthreads();
        for (int I = threadIdx.x; I < N.d.cells(); I += MG_THREADS) {
          int Z, Y, X;
          cell_of_fast(N.d, I, Z, Y, X);
          const unsigned M = N.cm[I];
          float s = 0.f;
          for (int k = 0; k < 8; ++k)
            if ((M >> k) & 1) s += L.t[at(L.d, 2 * Z + (k >> 2), 2 * Y + ((k >> 1) & 1), 2 * X + (k & 1))];
          N.b[I] = s;
        }
        __syncthreads();
      }
      {  // bottom: damped-Jacobi sweeps from x = w D^-1 b
        const SLv L = S(a.nlev - 1);
        auto W = [&](int k, int j) { return L.w(k, j); };
        const int n = L.d.cells();
        for (int i = threadIdx.x; i < n; i += MG_THREADS) L.x[i] = omega * L.dinv[i] * L.b[i];
        __syncthreads();
        float* src = L.x;
        float* dst = L.t;
        const int sweeps = a.bottom_sweeps;
        for (int s = 1; s < sweeps; ++s) {
          for (int i = threadIdx.x; i < n; i += MG_THREADS) {
            int z, y, x;
            cell_of_fast(L.d, i, z, y, x);
            const float sm = nbr_sum(L.d, i, z, y, x, W, [&](int j, int, int, int) { return src[j]; }, L.b[i]);
            dst[i] = fmaf(1.f - omega, src[i], omega * L.dinv[i] * sm);
          }
          __syncthreads();
          float* tmp = src;
          src = dst;
          dst = tmp;
        }
        if (src != L.x) {
          for (int i = threadIdx.x; i < n; i += MG_THREADS) L.x[i] = src[i];
          __syncthreads();
        }
      }
      for (int c = a.nlev - 2; c >= gl; --c) {  // up: x'_c = w D^-1 b + P x_{c+1}; one Jacobi step
        const SLv L = S(c);
        const SLv N = S(c + 1);
        auto W = [&](int k, int j) { return L.w(k, j); };
        for (int i = threadIdx.x; i < L.d.cells(); i += MG_THREADS) {
          int z, y, x;
          cell_of_fast(L.d, i, z, y, x);
          const int I = at(N.d, z >> 1, y >> 1, x >> 1);
          const float xc = ((N.cm[I] >> child_bit(z, y, x)) & 1) ? N.x[I] : 0.f;
          L.t[i] = fmaf(omega * L.dinv[i], L.b[i], xc);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < L.d.cells(); i += MG_THREADS) {
          int z, y, x;
          cell_of_fast(L.d, i, z, y, x);
          const float sm = nbr_sum(L.d, i, z, y, x, W, [&](int j, int, int, int) { return L.t[j]; }, L.b[i]);
          L.x[i] = fmaf(1.f - omega, L.t[i], omega * L.dinv[i] * sm);
        }
        __syncthreads();
      }
    }
    stamp(a, it, 4);
    stamp(a, it, 5);
    const float* xgl = S(gl).x;  // this CTA's copy of level gl's corrected solution

    // ===== UP c = gl-1 .. 1 (grid-wide): x_c = post_smooth(w D^-1 b_c + P x_{c+1})
    for (int c = gl - 1; c >= 1; --c) {
      const MgLevel& L = a.lv[c];
      const Dims d = dims(c), pd = dims(c + 1);
      const float* B = L.b;
      const float* DI = L.dinv;
      const float* XP = c + 1 == gl ? xgl : a.lv[c + 1].x;
      const uint8_t* cm = a.lv[c + 1].cmask;
      float* XO = L.x;
      auto W = Wg(c);
      auto xp = [&](int j, int z, int y, int x) {  // mask and value loaded independently
        const int I = at(pd, z >> 1, y >> 1, x >> 1);
        const float xc = XP[I] * (float)((cm[I] >> child_bit(z, y, x)) & 1);
        return fmaf(omega * DI[j], B[j], xc);
      };
      const int ni = n_items<SEG>(d);
      for (int base = (32 / SEG) * warp_g; base < ni; base += (32 / SEG) * warps) {
        const Item t = item_of<SEG>(d, base, ni);
        for_cells(d, t, [&](int i, int z, int y) {
          const float sm = nbr_sum(d, i, z, y, t.x, W, xp, B[i]);
          XO[i] = fmaf(1.f - omega, xp(i, z, y, t.x), omega * DI[i] * sm);
        });
      }
      grid_barrier(a.barrier, bar);
    }

    stamp(a, it, 6);
    // ===== UP 0: z = post_smooth(w r + P x_1); r.z.  D = I on the unknowns; off them r = 0, the
    // weights are 0 and no aggregate includes the cell, so z = 0 there without a test.
    {
      const float* R = a.r[cur];
      const float* XP = gl == 1 ? xgl : a.lv[1].x;
      const uint8_t* cm = a.lv[1].cmask;
      const Dims pd = dims(1);
      auto xp = [&](int j, int z, int y, int x) {  // mask and value loaded independently
        const int I = at(pd, z >> 1, y >> 1, x >> 1);
        const float xc = XP[I] * (float)((cm[I] >> child_bit(z, y, x)) & 1);
        return fmaf(omega, R[j], xc);
      };
      double acc = 0.0;
      const int ni = n_items<SEG>(fd);
      for (int base = (32 / SEG) * warp_g; base < ni; base += (32 / SEG) * warps) {
        const Item t = item_of<SEG>(fd, base, ni);
        for_cells(fd, t, [&](int i, int z, int y) {
          const float r_i = R[i];
          const float sm = nbr_sum(fd, i, z, y, t.x, Wf, xp, r_i);
          const float zi = fmaf(1.f - omega, xp(i, z, y, t.x), omega * sm);
          a.z[i] = zi;
          acc += (double)r_i * (double)zi;
        });
      }
      put_partial(a.part, 1, acc, red);
    }
    stamp(a, it, 7);
    grid_barrier(a.barrier, bar);
    stamp(a, it, 8);

    // ===== CG: beta, p = z + beta p, q = A'z + beta q, p.q
    {
      const double rz = grid_total(a.part, 1);
      const double beta = it > 0 && rz_old != 0.0 ? rz / rz_old : 0.0;
      rz_old = rz;
      const float be = (float)beta;
      const bool first = it == 0;
      const float* Z = a.z;
      auto zv = [&](int j, int, int, int) { return Z[j]; };
      double acc = 0.0;
      const int ni = n_items<SEG>(fd);
      for (int base = (32 / SEG) * warp_g; base < ni; base += (32 / SEG) * warps) {
        const Item t = item_of<SEG>(fd, base, ni);
        for_cells(fd, t, [&](int i, int z, int y) {
          const float zi = Z[i];
          // A'z = z - sum_j w'_ij z_j  (unit diagonal; 0 off the unknowns)
          const float az = zi - nbr_sum(fd, i, z, y, t.x, Wf, zv, 0.f);
          const float pi = first ? zi : fmaf(be, a.p[i], zi);
          const float qi = first ? az : fmaf(be, a.q[i], az);
          a.p[i] = pi;
          a.q[i] = qi;
          acc += (double)pi * (double)qi;
        });
      }
      put_partial(a.part, 2, acc, red);
    }
    stamp(a, it, 9);
    grid_barrier(a.barrier, bar);
    stamp(a, it, 10);
    {
      const double pq = grid_total(a.part, 2);
      alpha = pq != 0.0 ? rz_old / pq : 0.0;
    }
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.state[0] = state;
    a.iters[0] = state == ST_ZERO ? 0 : it;
  }
  // the solution is in y (the epilogue reads it); r[cur] is the last residual
}

// ---------------------------------------------------------------------------
// host side

static int mg_levels(int nz, int ny, int nx, Dims* d, int* grid_levels) {
  int n = 0;
  d[n++] = Dims{nz, ny, nx};
  while (n < kMgMaxLevels && (n < 2 || d[n - 1].cells() > kMgBottomCells)) {
    const Dims& p = d[n - 1];
    d[n++] = Dims{(p.nz + 1) / 2, (p.ny + 1) / 2, (p.nx + 1) / 2};
    if (d[n - 1].cells() == 1) break;
  }
  int gl = 1;
  static const int smem_cells = [] {  // RWB_MG_SMEM_CELLS: diagnostics override of kMgSmemCells
    const char* e = std::getenv("RWB_MG_SMEM_CELLS");
    return e ? std::max(1, std::atoi(e)) : kMgSmemCells;
  }();
  while (gl < n && d[gl].cells() > smem_cells) ++gl;
  // the shared-memory levels must fit (thin levels shrink only 2x per level)
  auto smem = [&](int g0) {
    size_t c = 0;
    for (int k = g0; k < n; ++k) c += (size_t)d[k].cells();
    return c * kMgSmemArrays * sizeof(float);
  };
  while (gl < n && smem(gl) > kMgSmemMax) ++gl;
  *grid_levels = gl;
  return n;
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t mg_workspace_bytes(int nz, int ny, int nx) {
  if ((long long)nz * ny * nx > INT_MAX) return 0;
  Dims d[kMgMaxLevels];
  int gl = 1;
  const int n = mg_levels(nz, ny, nx, d, &gl);
  size_t total = align256((size_t)d[0].cells() * 4);  // z
  for (int c = 1; c < gl; ++c) total += 7 * align256((size_t)d[c].cells() * 4) + align256((size_t)d[c].cells());
  if (gl < n) total += align256((size_t)d[gl].cells() * 4) + align256((size_t)d[gl].cells());  // b, cmask of gl
  total += align256(3 * kMgMaxBlocks * sizeof(double)) + 256;  // partials + barrier
  return total;
}

void mg_carve(MgArgs* a, char* base, int nz, int ny, int nx) {
  Dims d[kMgMaxLevels];
  int gl = 1;
  const int n = mg_levels(nz, ny, nx, d, &gl);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    char* p = base + o;
    o += align256(bytes);
    return p;
  };
  a->z = reinterpret_cast<float*>(take((size_t)d[0].cells() * 4));
  std::memset(a->lv, 0, sizeof(a->lv));
  for (int c = 0; c < n; ++c) {
    a->lv[c].nz = d[c].nz;
    a->lv[c].ny = d[c].ny;
    a->lv[c].nx = d[c].nx;
  }
  for (int c = 1; c < gl; ++c) {
    const size_t b = (size_t)d[c].cells() * 4;
    MgLevel& L = a->lv[c];
    L.leak = reinterpret_cast<float*>(take(b));
    L.dinv = reinterpret_cast<float*>(take(b));
    L.wx = reinterpret_cast<float*>(take(b));
    L.wy = reinterpret_cast<float*>(take(b));
    L.wz = reinterpret_cast<float*>(take(b));
    L.b = reinterpret_cast<float*>(take(b));
    L.x = reinterpret_cast<float*>(take(b));
    L.cmask = reinterpret_cast<uint8_t*>(take((size_t)d[c].cells()));
  }
  if (gl < n) {
    a->lv[gl].b = reinterpret_cast<float*>(take((size_t)d[gl].cells() * 4));
    a->lv[gl].cmask = reinterpret_cast<uint8_t*>(take((size_t)d[gl].cells()));
  }
  a->part = reinterpret_cast<double*>(take(3 * kMgMaxBlocks * sizeof(double)));
  a->barrier = reinterpret_cast<unsigned*>(take(256));
  a->nlev = n;
  a->grid_levels = gl;
}

static size_t mg_smem_bytes(const MgArgs& a) {
  size_t cells = 0;
  for (int c = a.grid_levels; c < a.nlev; ++c) cells += (size_t)a.lv[c].nz * a.lv[c].ny * a.lv[c].nx;
  return cells * kMgSmemArrays * sizeof(float);
}

// x-segment width of the grid-wide work items (RWB_MG_SEG=32 selects whole-warp rows; diagnostics)
static int mg_seg() {
  static const int seg = [] {
    const char* e = std::getenv("RWB_MG_SEG");
    return e && std::atoi(e) == 32 ? 32 : 16;
  }();
  return seg;
}

int launch_mgcg(const MgArgs& a, cudaStream_t st) {
  static DeviceCache cache;  // cooperative grid (one CTA per SM)
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  if ((long long)a.nz * a.ny * a.nx > INT_MAX) return fail(RWB_ERR_UNSUPPORTED, "multigrid level too large");
  if (a.grid_levels >= a.nlev) return fail(RWB_ERR_UNSUPPORTED, "multigrid hierarchy has no shared-memory level");
  const size_t smem = mg_smem_bytes(a);
  if (smem > kMgSmemMax) return fail(RWB_ERR_UNSUPPORTED, "multigrid shared-memory levels too large");
  const void* fn = mg_seg() == 32 ? (const void*)mgcg_kernel<32> : (const void*)mgcg_kernel<16>;
  // the attribute is set for the largest footprint the hierarchy rule allows, once per device
  constexpr int kSmemMax = (int)(kMgSmemMax);
  int grid = cache[dev].load(std::memory_order_relaxed);
  if (!grid) {
    int sms = 0, per = 0, coop = 0;
    RWB_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop) return fail(RWB_ERR_UNSUPPORTED, "device does not support cooperative launches");
    RWB_CUDA(cudaFuncSetAttribute(mgcg_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
    RWB_CUDA(cudaFuncSetAttribute(mgcg_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax));
    RWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mgcg_kernel<16>, MG_THREADS, kSmemMax));
    if (per < 1) return fail(RWB_ERR_UNSUPPORTED, "multigrid kernel does not fit one CTA per SM");
    grid = std::min(sms, kMgMaxBlocks);
    cache[dev].store(grid, std::memory_order_relaxed);
  }
  RWB_CUDA(cudaMemsetAsync(a.barrier, 0, sizeof(unsigned), st));
  void* args[] = {const_cast<MgArgs*>(&a)};
  RWB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(MG_THREADS), args, smem, st));
  count_launches(1);
  return RWB_OK;
}

unsigned long long* mg_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static const bool on = std::getenv("RWB_MG_TRACE") != nullptr;
  if (on && !buf && cudaMalloc(&buf, 8 * 16 * sizeof(unsigned long long)) != cudaSuccess) buf = nullptr;
  return buf;
}

}  // namespace rwb

// diagnostics: the %globaltimer stamps of the last multigrid solve (RWB_MG_TRACE set), 128 values
extern "C" int rwb_mg_trace_dump(unsigned long long* out) {
  unsigned long long* buf = rwb::mg_trace_buffer();
  if (!buf) return -1;
  return (int)cudaMemcpy(out, buf, 8 * 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
