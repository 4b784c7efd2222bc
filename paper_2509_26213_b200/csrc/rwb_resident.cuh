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
// 4-CTA clusters, 8 planes per CTA, weights in shared memory (rwb_resident4.cu)
int launch_resident3d_q4(const ResidentArgs& a, int max_bricks, cudaStream_t st);

}  // namespace rwb
