// Shared solver definitions (streaming solver rwb_solve.cu, brick-resident
// solver rwb_resident.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rwb {

enum BrickState : int { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_ZERO = 3 };

// Level + brick-grid geometry, padded to 3 dims (2-D levels have nz = bz = 1).
struct Geo {
  int nz, ny, nx;  // level
  int bz, by, bx;  // brick box
  int oz, oy, ox;  // brick grid origin
  int gz, gy, gx;  // brick grid
  int tz, ty, tx;  // streaming tiles per brick
  int tiles;
  long long bvol;  // bz*by*bx
  long long sxy;   // ny*nx
  int is3d;
};

// The brick-resident CG engine works on the brick-local system the streaming
// setup kernels build (slot-major, each brick box contiguous, x fastest).
struct ResidentArgs {
  const float* wx;        // scaled forward weights (0 across brick faces / at Dirichlet nodes)
  const float* wy;
  const float* wz;
  const float* r0;        // initial scaled residual
  const float* y;         // y0 = x0 / s (unknowns), the final value (other voxels)
  const float* sc;        // Jacobi scale s (0: not an unknown)
  const double* bb;       // per slot ||S b||^2
  const int* alist;       // compacted slots still active after the setup
  const int* n_active;
  int* state;             // per slot
  int* iters;             // per slot
  int* next;              // dynamic brick counter (zero at launch)
  int coarse;             // coarse-corrected PCG (4-CTA engine: 8^3 aggregates, 2-D engine: 8^2) instead of Jacobi-PCG
  float tol2;
  int max_iter;
  // results straight into the level: prob = s y (unknowns) or y, labels = prob > 0.5
  float* prob;
  uint8_t* labels;        // may be null
  const int* list;        // slot -> brick id (null: identity)
  int nz, ny, nx;         // level
  int oz, oy, ox;         // brick grid origin
  int gy, gx;             // brick grid extents in y, x
};

int resident3d_supported(const Geo& g);
// 2-D levels with 64^2 bricks: one CTA per tile (rwb_resident2d.cu)
int resident2d_supported(const Geo& g);
int launch_resident2d(const ResidentArgs& a, int max_bricks, cudaStream_t st);
// variant: 8 = 8-CTA clusters (4 planes per CTA), 16 = 16-CTA clusters (2 planes per CTA, 2 CTAs/SM)
int launch_resident3d(const ResidentArgs& a, int max_bricks, int variant, cudaStream_t st);
// 4-CTA clusters, 8 planes per CTA, scaled weights in tensor memory (rwb_resident4.cu)
int launch_resident3d_q4(const ResidentArgs& a, int max_bricks, cudaStream_t st);

// ---------------------------------------------------------------------------
// Whole-level (coarsest) solve: multigrid-preconditioned CG in one cooperative kernel
// (rwb_mgcg.cu).  The fine level is the Jacobi-scaled system the setup kernels build (unit
// diagonal, scaled forward weights w', s = 0 off the unknowns); the preconditioner is one V(1,1)
// cycle of a Galerkin hierarchy of strength-masked 2x2x2 aggregates.
constexpr int kMgMaxLevels = 16;
constexpr int kMgMaxBlocks = 1024;

struct MgLevel {
  int nz, ny, nx;
  uint8_t* cmask;  // per aggregate: bit (dz*4 + dy*2 + dx) = that child of the level below is prolongated to
  float* leak;  // Dirichlet coupling of the aggregate; diag = leak + the 6 face weights
  float* dinv;  // 1/diag, 0 for aggregates without unknowns
  float* wx;    // forward weights (negated off-diagonals) of the Galerkin operator
  float* wy;
  float* wz;
  float* b;     // restricted residual of the V-cycle
  float* x;     // corrected, post-smoothed level solution of the V-cycle
};

struct MgArgs {
  int nz, ny, nx;                  // fine level (= the whole-level brick)
  const float* wx;                 // fine scaled weights, Jacobi scale
  const float* wy;
  const float* wz;
  const float* sc;
  float* y;                        // solution (scaled); final value on non-unknowns
  float* r[2];                     // residual, double-buffered (r[0] = the setup's r0)
  float* p;
  float* q;
  float* z;                        // preconditioned residual
  const double* bb;                // ||S b||^2
  const double* rr0;               // ||r0||^2
  int* state;
  int* iters;
  double* part;                    // [3][kMgMaxBlocks] per-block partials (rr, rz, pq)
  unsigned* barrier;               // grid-barrier counter, zero at launch
  int nlev;                        // levels (fine = 0)
  int grid_levels;                 // levels 0..grid_levels-1 run grid-wide; the rest in every CTA's shared memory
  MgLevel lv[kMgMaxLevels];
  const float* intensity;          // the level's intensities and seeds: the fine cells' Dirichlet
  const uint8_t* seeds;            // couplings (leak) are computed exactly from them
  float beta, min_weight;
  float tol2;
  int max_iter;
  float omega;                     // damped-Jacobi smoothing factor
  int bottom_sweeps;               // Jacobi sweeps on the coarsest aggregate level
  unsigned long long* trace;       // diagnostics: %globaltimer at the phase boundaries of iterations 0..7 (or null)
};

// bytes of the multigrid workspace beyond the streaming solver's (z + coarse levels + partials)
size_t mg_workspace_bytes(int nz, int ny, int nx);
// lay out the multigrid workspace at `base` (mg_workspace_bytes bytes) and fill a.lv / levels
void mg_carve(MgArgs* a, char* base, int nz, int ny, int nx);
int launch_mgcg(const MgArgs& a, cudaStream_t st);
unsigned long long* mg_trace_buffer();  // RWB_MG_TRACE diagnostics buffer, else null

}  // namespace rwb
