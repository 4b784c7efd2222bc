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

struct ResidentArgs {
  Geo g;
  const int* list;  // brick indices per slot, or null (slot == brick)
  int nb;           // slots
  const float* I;
  const uint8_t* S;
  const float* bound;
  float* prob;
  uint8_t* labels;
  float beta, wmin, tol2;
  int max_iter;
  int* state;    // [nb]
  int* iters;    // [nb]
  int* counter;  // work counter, zero before launch
  unsigned long long* unknowns;
};

int resident3d_supported(const Geo& g);
int launch_resident3d(const ResidentArgs& a, cudaStream_t st);

}  // namespace rwb
