// Brick-resident Jacobi-PCG: one 32^3 brick per 8-CTA thread-block cluster,
// the whole solve on chip.
//
// The streaming solver (rwb_solve.cu) moves 52 B per voxel per CG iteration
// through HBM.  A 32^3 brick's complete CG state — y, r, p, q and its six
// scaled edge weights, 10 floats per voxel = 1.25 MiB — fits in the register
// files of 8 SMs (8 x 256 KB), so here a cluster of 8 CTAs owns one brick:
// CTA `c` holds z-planes [4c, 4c+4), each of its 256 threads a 4(x) x 4(z)
// block of voxels in registers.  HBM is touched once per brick: the inputs
// (intensity, seeds, parent bound, each with a one-voxel halo) are staged into
// shared memory — for the NEXT brick, with cp.async, while the current brick
// iterates — and the epilogue writes probabilities and labels (~14 B/voxel
// in total instead of 52 B/voxel/iteration).
//
// The iteration is the single-reduction CG of Chronopoulos & Gear (1989):
// with w = A'r and s = A'p carried as vectors, both dot products of an
// iteration, gamma = r.r and delta = w.r, are reduced together, and
//   beta = gamma_new / gamma,  alpha = gamma_new / (delta - beta gamma_new / alpha),
//   p = r + beta p,  s = w + beta s,  y += alpha p,  r -= alpha s,  w = A'r.
// Latency, not bandwidth, bounds an on-chip brick solve (each iteration is a
// chain of neighbour exchange -> SpMV -> cluster-wide reduction), and this
// form has one cluster-wide reduction per iteration instead of two.
//
// Neighbour exchange per iteration (no cluster-wide barrier inside the loop):
//   x: warp shuffles (lanes of a row are x-consecutive quads)
//   y: r planes in shared memory (LDS.128 of the rows above / below)
//   z: in-thread, except the slab faces: each CTA PUSHES its two r face
//      planes into its z-neighbours' shared memory with `st.async ...
//      mbarrier::complete_tx` (DSMEM stores that complete on the receiver's
//      mbarrier).
// Reduction: every warp shuffle-reduces its partials and lanes 0..7 st.async
// them into slot [rank][warp] of all 8 CTAs; each CTA waits on its own
// mbarrier and every warp sums the 64 partials with the same fixed shuffle
// tree, so all CTAs take identical CG decisions (deterministic, independent
// of brick scheduling).
//
// Same Jacobi-scaled system as the streaming kernels (identical scale factors
// and scaled weights); the CG scalars are fp32 here (float64 there).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"

namespace cg = cooperative_groups;

namespace rwb {

constexpr int RB = 32;          // brick edge
constexpr int RCL = 8;          // CTAs per cluster (per brick)
constexpr int RPZ = RB / RCL;   // z planes per CTA
constexpr int RQ = 4;           // x voxels per thread
constexpr int RQN = RB / RQ;    // quads per row
constexpr int RT = RQN * RB;    // threads per CTA (256)
constexpr int RW = RT / 32;     // warps per CTA
constexpr int RV = RQ * RPZ;    // voxels per thread (16)
constexpr int NPART = RCL * RW; // pushed partials per reduction (64)
constexpr int TZS = RPZ + 2;    // staged tile: slab + 1-voxel halo
constexpr int TYS = RB + 2;
constexpr int TXS = RB + 2;
constexpr int TILE = TZS * TYS * TXS;
constexpr unsigned char OUTSIDE = 255;  // staged seed marker: voxel outside the level

static_assert(RPZ == 4 && RQ == 4, "register blocking assumes 4x4 voxels per thread");

}  // namespace rwb

#ifdef RWB_TRACE
// phase timestamps of cluster 0 (diagnostics build only)
__device__ long long g_rwb_trace[8][64][8];
__device__ long long g_rwb_btrace[8][16][10];
#define TRACE(k)                                                                                   \
  do {                                                                                             \
    if (tid == 0 && blockIdx.x < RCL && trace_it < 64) g_rwb_trace[rank][trace_it][k] = clock64(); \
  } while (0)
#define BTRACE(k)                                                                                   \
  do {                                                                                              \
    if (tid == 0 && blockIdx.x < RCL && btrace_n < 16) g_rwb_btrace[rank][btrace_n][k] = clock64(); \
  } while (0)
#else
#define TRACE(k) \
  do {           \
  } while (0)
#define BTRACE(k) \
  do {            \
  } while (0)
#endif

namespace rwb {

struct ResidentSmem {
  float tI[2][TZS][TYS][TXS];           // staged intensity (double buffer: current / next brick)
  float tB[2][TZS][TYS][TXS];           // staged parent bound
  unsigned char tS[2][TZS][TYS][TXS];   // staged seeds (OUTSIDE = not in the level)
  float4 rp[RPZ][RB][RQN];              // r planes of this slab (y neighbours of the SpMV)
  float4 rface[2][2][RB][RQN];          // received r faces [parity][0 = from below, 1 = from above]
  float4 sc[RPZ][RB][RQN];              // scale factors of the slab (setup exchange, epilogue)
  __align__(16) float red[2][3][NPART]; // pushed partials [parity][gamma, delta, bb][rank*RW + warp]
  unsigned long long barF[2];           // mbarriers: r faces from the z neighbours, per parity
  unsigned long long barR[2];           // mbarriers: dot-product partials, per parity
};

// ---- PTX helpers ----------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra.uni WAIT_%=;\n\t}" ::"r"(a),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void st_async_f32(uint32_t remote, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(remote),
               "r"(__float_as_uint(v)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void st_async_v4(uint32_t remote, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote),
               "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
               "r"(__float_as_uint(v.w)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float lane_of(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ float4 f4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }

__device__ __forceinline__ float seedval(unsigned char s) { return s == 1 ? 1.f : 0.f; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of the 64 pushed partials: lane l loads partials 2l, 2l+1 (one LDS.64)
// and the warp reduces them with a fixed shuffle tree, so every warp of every
// CTA gets the bit-identical total without a broadcast through shared memory.
__device__ __forceinline__ float sum64(const float* red) {
  const float2 v = reinterpret_cast<const float2*>(red)[threadIdx.x & 31];
  return warp_sum(v.x + v.y);
}

// Stage the slab of brick `brick` (+ one-voxel halo) into buffer `buf`:
// intensity and bound with cp.async (complete at the next wait_group), seeds
// with plain loads (byte granularity) when `seeds_now`.
__device__ __forceinline__ void stage_issue(const ResidentArgs& a, ResidentSmem& sm, int buf, int brick, int lz0,
                                            bool seeds_now) {
  const Geo& g = a.g;
  const int hx = brick % g.gx, hy = (brick / g.gx) % g.gy, hz = brick / (g.gx * g.gy);
  const int z0 = g.oz + hz * RB + lz0 - 1, y0 = g.oy + hy * RB - 1, x0 = g.ox + hx * RB - 1;
  for (int idx = threadIdx.x; idx < TILE; idx += RT) {
    const int tz = idx / (TYS * TXS), rem = idx - tz * (TYS * TXS);
    const int ty = rem / TXS, tx = rem - ty * TXS;
    const int z = z0 + tz, y = y0 + ty, x = x0 + tx;
    const bool in = z >= 0 && z < g.nz && y >= 0 && y < g.ny && x >= 0 && x < g.nx;
    if (in) {
      const long long gi = (long long)z * g.sxy + (long long)y * g.nx + x;
      cp_async4(&sm.tI[buf][tz][ty][tx], a.I + gi);
      cp_async4(&sm.tB[buf][tz][ty][tx], a.bound + gi);
      if (seeds_now) sm.tS[buf][tz][ty][tx] = __ldg(a.S + gi);
    } else {
      sm.tI[buf][tz][ty][tx] = 0.f;
      sm.tB[buf][tz][ty][tx] = 0.f;
      sm.tS[buf][tz][ty][tx] = OUTSIDE;
    }
  }
  cp_async_commit();
}

__device__ __forceinline__ void stage_seeds(const ResidentArgs& a, ResidentSmem& sm, int buf, int brick, int lz0) {
  const Geo& g = a.g;
  const int hx = brick % g.gx, hy = (brick / g.gx) % g.gy, hz = brick / (g.gx * g.gy);
  const int z0 = g.oz + hz * RB + lz0 - 1, y0 = g.oy + hy * RB - 1, x0 = g.ox + hx * RB - 1;
  for (int idx = threadIdx.x; idx < TILE; idx += RT) {
    const int tz = idx / (TYS * TXS), rem = idx - tz * (TYS * TXS);
    const int ty = rem / TXS, tx = rem - ty * TXS;
    const int z = z0 + tz, y = y0 + ty, x = x0 + tx;
    if (z >= 0 && z < g.nz && y >= 0 && y < g.ny && x >= 0 && x < g.nx)
      sm.tS[buf][tz][ty][tx] = __ldg(a.S + (long long)z * g.sxy + (long long)y * g.nx + x);
  }
}

__global__ void __cluster_dims__(RCL, 1, 1) __launch_bounds__(RT, 1) resident3d_kernel(ResidentArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ResidentSmem& sm = *reinterpret_cast<ResidentSmem*>(smem_raw);
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int ly = tid / RQN;  // row
  const int xq = tid % RQN;  // quad within the row
  const int lz0 = rank * RPZ;
  const Geo& g = a.g;
  const float bw = a.beta, wmin = a.wmin;
  const ResidentSmem* below = rank > 0 ? cluster.map_shared_rank(&sm, rank - 1) : nullptr;
  const ResidentSmem* above = rank < RCL - 1 ? cluster.map_shared_rank(&sm, rank + 1) : nullptr;
  const int nfaces = (rank > 0) + (rank < RCL - 1);
  const uint32_t face_bytes = (uint32_t)(RB * RQN * sizeof(float4));
  const int cid = blockIdx.x / RCL, ncl = gridDim.x / RCL;

  if (tid == 0) {
    mbar_init(&sm.barF[0], 1);
    mbar_init(&sm.barF[1], 1);
    mbar_init(&sm.barR[0], 1);
    mbar_init(&sm.barR[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // remote addresses this thread pushes to
  uint32_t face_dn_dst[2] = {0, 0}, face_up_dst[2] = {0, 0}, bar_dn[2] = {0, 0}, bar_up[2] = {0, 0};
  uint32_t red_dst[2] = {0, 0}, barR_dst[2] = {0, 0};
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    if (rank > 0) {  // my plane 0 goes to the CTA below, as its "from above" face
      face_dn_dst[par] = mapa_u32(smem_u32(&sm.rface[par][1][ly][xq]), rank - 1);
      bar_dn[par] = mapa_u32(smem_u32(&sm.barF[par]), rank - 1);
    }
    if (rank < RCL - 1) {  // my last plane goes to the CTA above, as its "from below" face
      face_up_dst[par] = mapa_u32(smem_u32(&sm.rface[par][0][ly][xq]), rank + 1);
      bar_up[par] = mapa_u32(smem_u32(&sm.barF[par]), rank + 1);
    }
    if (lane < RCL) {  // lane t delivers this warp's partials to CTA t
      red_dst[par] = mapa_u32(smem_u32(&sm.red[par][0][rank * RW + warp]), lane);
      barR_dst[par] = mapa_u32(smem_u32(&sm.barR[par]), lane);
    }
  }
  cluster.sync();
  unsigned gk = 0;  // iterations run by this cluster so far (drives the mbarrier parities)
#ifdef RWB_TRACE
  int btrace_n = 0;
#endif

  // static round-robin brick assignment; brick n+1 is staged while brick n iterates
  int buf = 0;
  if (cid < a.nb) stage_issue(a, sm, 0, a.list ? a.list[cid] : cid, lz0, true);
  for (int slot = cid; slot < a.nb; slot += ncl, buf ^= 1) {
    BTRACE(0);
    const int brick = a.list ? a.list[slot] : slot;
    const int next = slot + ncl;
    if (next < a.nb) {
      stage_issue(a, sm, buf ^ 1, a.list ? a.list[next] : next, lz0, false);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    BTRACE(1);
    const int hx = brick % g.gx;
    const int hy = (brick / g.gx) % g.gy;
    const int hz = brick / (g.gx * g.gy);
    const int gz0 = g.oz + hz * RB + lz0, gy = g.oy + hy * RB + ly, gx0 = g.ox + hx * RB + xq * RQ;
    const float(*tI)[TYS][TXS] = sm.tI[buf];
    const float(*tB)[TYS][TXS] = sm.tB[buf];
    const unsigned char(*tS)[TYS][TXS] = sm.tS[buf];
    // staged-tile coordinates of voxel (z, i) of this thread: (z+1, ly+1, xq*4+i+1)
    const int cy = ly + 1, cx0 = xq * RQ + 1;
    // the six edge weights (0 = no edge), order -z,+z,-y,+y,-x,+x
    auto weights6 = [&](int z, int i, float* wn) {
      const int cz = z + 1, cx = cx0 + i;
      const float c = tI[cz][cy][cx];
      const int nz[6] = {cz - 1, cz + 1, cz, cz, cz, cz};
      const int ny[6] = {cy, cy, cy - 1, cy + 1, cy, cy};
      const int nx[6] = {cx, cx, cx, cx, cx - 1, cx + 1};
#pragma unroll
      for (int e = 0; e < 6; ++e)
        wn[e] = tS[nz[e]][ny[e]][nx[e]] != OUTSIDE ? edge_weight(c, tI[nz[e]][ny[e]][nx[e]], bw, wmin) : 0.f;
    };

    // ---------------- setup 1: scale factors s = diag^-1/2 ----------------
    float scl[RV];
#pragma unroll
    for (int z = 0; z < RPZ; ++z)
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        scl[v] = 0.f;
        if (tS[z + 1][cy][cx0 + i] != 0) continue;  // seed or outside the level
        float wn[6];
        weights6(z, i, wn);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < 6; ++e) d += wn[e];
        scl[v] = d > 0.f ? 1.0f / sqrtf(d) : 0.f;
      }
#pragma unroll
    for (int z = 0; z < RPZ; ++z) sm.sc[z][ly][xq] = f4(scl[z * RQ], scl[z * RQ + 1], scl[z * RQ + 2], scl[z * RQ + 3]);
    BTRACE(2);
    cluster.sync();
    BTRACE(3);

    // ---------------- setup 2: scaled weights, r0 = S(b - L x0), y0 = x0 / s ----------------
    float y[RV], r[RV], p[RV], sv[RV], w[RV];
    float wxf[RV], wyf[RV], wzf[RV], wyb[RV], wxb[RPZ], wzb[RQ];
    float bb_part = 0.f, rr_part = 0.f;
    unsigned n_unk = 0;
#pragma unroll
    for (int z = 0; z < RPZ; ++z) {
      const float4 sy_up = ly + 1 < RB ? sm.sc[z][ly + 1][xq] : f4(0, 0, 0, 0);
      const float4 sy_dn = ly > 0 ? sm.sc[z][ly - 1][xq] : f4(0, 0, 0, 0);
      const float4 sz_up = z + 1 < RPZ ? sm.sc[z + 1][ly][xq] : (above ? above->sc[0][ly][xq] : f4(0, 0, 0, 0));
      const float4 sz_dn = z > 0 ? sm.sc[z - 1][ly][xq] : (below ? below->sc[RPZ - 1][ly][xq] : f4(0, 0, 0, 0));
      float sx_l = __shfl_up_sync(0xffffffffu, scl[z * RQ + RQ - 1], 1);
      float sx_r = __shfl_down_sync(0xffffffffu, scl[z * RQ], 1);
      if (xq == 0) sx_l = 0.f;
      if (xq == RQN - 1) sx_r = 0.f;
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        const float si = scl[v];
        float nsc[6];
        nsc[0] = lane_of(sz_dn, i);
        nsc[1] = lane_of(sz_up, i);
        nsc[2] = lane_of(sy_dn, i);
        nsc[3] = lane_of(sy_up, i);
        nsc[4] = i > 0 ? scl[v - 1] : sx_l;
        nsc[5] = i < RQ - 1 ? scl[v + 1] : sx_r;
        float wp[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        y[v] = 0.f;
        r[v] = 0.f;
        if (si > 0.f) {
          ++n_unk;
          const int cz = z + 1, cx = cx0 + i;
          const int nz[6] = {cz - 1, cz + 1, cz, cz, cz, cz};
          const int ny[6] = {cy, cy, cy - 1, cy + 1, cy, cy};
          const int nx[6] = {cx, cx, cx, cx, cx - 1, cx + 1};
          const float x0 = tB[cz][cy][cx];
          float wn[6];
          weights6(z, i, wn);
          float diag = 0.f, b = 0.f, acc = 0.f;
#pragma unroll
          for (int e = 0; e < 6; ++e) {
            diag += wn[e];
            if (wn[e] == 0.f) continue;
            const float bn = tB[nz[e]][ny[e]][nx[e]];
            if (nsc[e] > 0.f) {  // coupled unknown of this brick
              wp[e] = wn[e] * si * nsc[e];
              acc += wn[e] * bn;
            } else {  // Dirichlet: seed, or outside the brick
              const unsigned char s = tS[nz[e]][ny[e]][nx[e]];
              b += wn[e] * (s ? seedval(s) : bn);
            }
          }
          r[v] = si * (b + acc - diag * x0);
          y[v] = x0 / si;
          const float sb = si * b;
          bb_part += sb * sb;
          rr_part += r[v] * r[v];
        }
        if (z == 0) wzb[i] = wp[0];
        wzf[v] = wp[1];
        wyb[v] = wp[2];
        wyf[v] = wp[3];
        if (i == 0) wxb[z] = wp[4];
        wxf[v] = wp[5];
      }
    }
    {
      const unsigned nu = __reduce_add_sync(0xffffffffu, n_unk);
      if (lane == 0 && nu) atomicAdd(a.unknowns, (unsigned long long)nu);
    }
    BTRACE(4);
    BTRACE(5);

    // ---------------- CG (Chronopoulos-Gear) ----------------
    // pass 0 computes w0 = A'r0 and reduces gamma0 = r0.r0, delta0 = w0.r0 and
    // ||S b||^2; pass k >= 1 first applies update k, then the same SpMV + reduction.
    const uint32_t tx_faces = nfaces * face_bytes;
    float gamma = 0.f, alpha = 0.f, beta = 0.f, thresh = 0.f;
    int state = ST_ACTIVE, it = 0;
#ifdef RWB_TRACE
    int trace_it = (int)gk;
#endif
#pragma unroll
    for (int v = 0; v < RV; ++v) {
      p[v] = 0.f;
      sv[v] = 0.f;
      w[v] = 0.f;
    }
    for (int pass = 0;; ++pass) {
      TRACE(0);
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
      if (tid == 0) {
        if (tx_faces) mbar_expect_tx(&sm.barF[par], tx_faces);
        mbar_expect_tx(&sm.barR[par], 3 * NPART * 4);
      }
      if (pass > 0) {
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          p[v] = fmaf(beta, p[v], r[v]);
          sv[v] = fmaf(beta, sv[v], w[v]);
          y[v] = fmaf(alpha, p[v], y[v]);
          r[v] = fmaf(-alpha, sv[v], r[v]);
        }
      }
      // publish r: planes for the y neighbours, faces for the z neighbours
#pragma unroll
      for (int z = 0; z < RPZ; ++z) sm.rp[z][ly][xq] = f4(r[z * RQ], r[z * RQ + 1], r[z * RQ + 2], r[z * RQ + 3]);
      if (rank > 0)
        st_async_v4(par ? face_dn_dst[1] : face_dn_dst[0], f4(r[0], r[1], r[2], r[3]), par ? bar_dn[1] : bar_dn[0]);
      if (rank < RCL - 1)
        st_async_v4(par ? face_up_dst[1] : face_up_dst[0],
                    f4(r[(RPZ - 1) * RQ], r[(RPZ - 1) * RQ + 1], r[(RPZ - 1) * RQ + 2], r[(RPZ - 1) * RQ + 3]),
                    par ? bar_up[1] : bar_up[0]);
      __syncthreads();
      TRACE(1);
      // w = A'r: interior planes first, the two face planes once their neighbours arrived
      float g4[RPZ] = {0.f, 0.f, 0.f, 0.f}, d4[RPZ] = {0.f, 0.f, 0.f, 0.f};
      auto spmv_plane = [&](int z, const float4& rzu, const float4& rzd) {
        const float4 ru = ly + 1 < RB ? sm.rp[z][ly + 1][xq] : f4(0, 0, 0, 0);
        const float4 rd = ly > 0 ? sm.rp[z][ly - 1][xq] : f4(0, 0, 0, 0);
        const float rl = __shfl_up_sync(0xffffffffu, r[z * RQ + RQ - 1], 1);
        const float rr_ = __shfl_down_sync(0xffffffffu, r[z * RQ], 1);
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const int v = z * RQ + i;
          const float rxl = i > 0 ? r[v - 1] : rl;
          const float rxr = i < RQ - 1 ? r[v + 1] : rr_;
          const float wxl = i > 0 ? wxf[v - 1] : wxb[z];
          const float wzl = z > 0 ? wzf[v - RQ] : wzb[i];
          float acc = wxf[v] * rxr;
          acc = fmaf(wxl, rxl, acc);
          acc = fmaf(wyf[v], lane_of(ru, i), acc);
          acc = fmaf(wyb[v], lane_of(rd, i), acc);
          acc = fmaf(wzf[v], lane_of(rzu, i), acc);
          acc = fmaf(wzl, lane_of(rzd, i), acc);
          w[v] = r[v] - acc;
          g4[z] = fmaf(r[v], r[v], g4[z]);
          d4[z] = fmaf(w[v], r[v], d4[z]);
        }
      };
#pragma unroll
      for (int z = 1; z < RPZ - 1; ++z)
        spmv_plane(z, f4(r[(z + 1) * RQ], r[(z + 1) * RQ + 1], r[(z + 1) * RQ + 2], r[(z + 1) * RQ + 3]),
                   f4(r[(z - 1) * RQ], r[(z - 1) * RQ + 1], r[(z - 1) * RQ + 2], r[(z - 1) * RQ + 3]));
      if (tx_faces) mbar_wait(&sm.barF[par], ph);
      TRACE(2);
      spmv_plane(0, f4(r[RQ], r[RQ + 1], r[RQ + 2], r[RQ + 3]),
                 below ? sm.rface[par][0][ly][xq] : f4(0, 0, 0, 0));
      spmv_plane(RPZ - 1, above ? sm.rface[par][1][ly][xq] : f4(0, 0, 0, 0),
                 f4(r[(RPZ - 2) * RQ], r[(RPZ - 2) * RQ + 1], r[(RPZ - 2) * RQ + 2], r[(RPZ - 2) * RQ + 3]));
      TRACE(3);
      {
        const float gw = warp_sum((g4[0] + g4[1]) + (g4[2] + g4[3]));
        const float dw = warp_sum((d4[0] + d4[1]) + (d4[2] + d4[3]));
        const float bw_ = pass == 0 ? warp_sum(bb_part) : 0.f;
        if (lane < RCL) {
          const uint32_t dst = par ? red_dst[1] : red_dst[0], bar = par ? barR_dst[1] : barR_dst[0];
          st_async_f32(dst, gw, bar);
          st_async_f32(dst + NPART * 4, dw, bar);
          st_async_f32(dst + 2 * NPART * 4, bw_, bar);
        }
      }
      TRACE(4);
      mbar_wait(&sm.barR[par], ph);
      TRACE(5);
      ++gk;
      const float g_new = sum64(sm.red[par][0]);
      const float delta = sum64(sm.red[par][1]);
      if (pass == 0) {
        const double bb = (double)sum64(sm.red[par][2]);
        thresh = (float)((double)a.tol2 * bb);
        if (bb <= 0.0) {
          state = ST_ZERO;  // no Dirichlet coupling: the exact solution is 0
          break;
        }
        if ((double)g_new <= (double)a.tol2 * bb) {
          state = ST_CONVERGED;
          break;
        }
        if (a.max_iter <= 0) {
          state = ST_MAXITER;
          break;
        }
        beta = 0.f;
        alpha = delta != 0.f ? __fdividef(g_new, delta) : 0.f;
      } else {
        ++it;
        if (g_new <= thresh) {
          state = ST_CONVERGED;
          break;
        }
        if (it >= a.max_iter) {
          state = ST_MAXITER;
          break;
        }
        // fast reciprocals: the scalars only need to be identical in every CTA
        beta = __fdividef(g_new, gamma);
        const float den = delta - beta * __fdividef(g_new, alpha);
        alpha = den != 0.f ? __fdividef(g_new, den) : 0.f;
      }
      gamma = g_new;
      TRACE(6);
#ifdef RWB_TRACE
      ++trace_it;
#endif
    }
    BTRACE(6);

    // ---------------- epilogue: x = s*y | seed value | bound ----------------
#pragma unroll
    for (int z = 0; z < RPZ; ++z) {
      const int gz = gz0 + z;
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        const unsigned char s = tS[z + 1][cy][cx0 + i];
        if (s == OUTSIDE) continue;
        float x;
        if (scl[v] > 0.f)
          x = state == ST_ZERO ? 0.f : scl[v] * y[v];
        else
          x = s ? seedval(s) : tB[z + 1][cy][cx0 + i];
        const long long gi = (long long)gz * g.sxy + (long long)gy * g.nx + (gx0 + i);
        a.prob[gi] = x;
        if (a.labels) a.labels[gi] = x > 0.5f ? 1 : 0;
      }
    }
    if (rank == 0 && tid == 0) {
      a.state[slot] = state;
      a.iters[slot] = state == ST_ZERO ? 0 : it;
    }
    BTRACE(7);
    // every DSMEM read of this brick (sc) is done before any CTA starts the
    // next one; the staged seeds of the next brick are loaded after it
    cluster.sync();
    if (next < a.nb) stage_seeds(a, sm, buf ^ 1, a.list ? a.list[next] : next, lz0);
    BTRACE(8);
#ifdef RWB_TRACE
    ++btrace_n;
#endif
  }
}

#ifdef RWB_TRACE
extern "C" int rwb_trace_dump(long long* out) {  // 8*64*8 int64
  return (int)cudaMemcpyFromSymbol(out, g_rwb_trace, sizeof(g_rwb_trace));
}
extern "C" int rwb_btrace_dump(long long* out) {  // 8*16*10 int64
  return (int)cudaMemcpyFromSymbol(out, g_rwb_btrace, sizeof(g_rwb_btrace));
}
#endif

int resident3d_supported(const Geo& g) { return g.is3d && g.bz == RB && g.by == RB && g.bx == RB; }

int launch_resident3d(const ResidentArgs& a, cudaStream_t st) {
  static thread_local int clusters = 0;
  const int smem = (int)sizeof(ResidentSmem);
  if (!a.bound) return fail(RWB_ERR_INVALID, "the brick-resident solver needs a bound");
  if (!clusters) {
    RWB_CUDA(cudaFuncSetAttribute(resident3d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(RCL * 1024, 1, 1);
    cfg.blockDim = dim3(RT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = RCL;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    RWB_CUDA(cudaOccupancyMaxActiveClusters(&n, resident3d_kernel, &cfg));
    if (n <= 0) return fail(RWB_ERR_UNSUPPORTED, "no 8-CTA cluster fits on this device");
    clusters = n;
  }
  const int grid_clusters = clusters < a.nb ? clusters : a.nb;
  resident3d_kernel<<<grid_clusters * RCL, RT, smem, st>>>(a);
  RWB_LAUNCH_CHECK("resident3d_kernel");
  count_launches(1);
  return RWB_OK;
}

}  // namespace rwb
