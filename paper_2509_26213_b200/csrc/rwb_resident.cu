// Brick-resident Jacobi-PCG: one 32^3 brick per 8-CTA thread-block cluster,
// the whole solve on chip.
//
// The streaming solver (rwb_solve.cu) moves 52 B per voxel per CG iteration
// through HBM.  A 32^3 brick's complete CG state — y, r, p, q and its six
// scaled edge weights, 10 floats per voxel = 1.25 MiB — fits in the register
// files of 8 SMs (8 x 256 KB), so here a cluster of 8 CTAs owns one brick:
// CTA `c` holds z-planes [4c, 4c+4), each of its 256 threads a 4(x) x 4(z)
// block of voxels in registers.  HBM is touched once per brick: the setup
// reads intensity, seeds and the parent bound (plus a one-voxel halo), the
// epilogue writes probabilities and labels (~14 B/voxel in total instead of
// 52 B/voxel/iteration).
//
// Neighbour exchange per iteration (no cluster-wide barrier inside the loop):
//   x: warp shuffles (lanes of a row are x-consecutive quads)
//   y: p planes in shared memory (LDS.128 of the rows above / below)
//   z: in-thread, except the slab faces: every iteration each CTA PUSHES its
//      two r face planes into its z-neighbours' shared memory with
//      `st.async ... mbarrier::complete_tx` (DSMEM stores that complete on
//      the receiver's mbarrier); the receiver keeps its neighbours' p face
//      values in registers and advances them itself, p_face <- r_face + beta
//      p_face, so p never crosses CTAs.
// Reductions: warp shuffles -> CTA partial -> one thread st.async's it into
// slot `rank` of all 8 CTAs (again completing on their mbarriers) -> every
// CTA waits on its own mbarrier and sums the 8 partials in the same order
// (float64), so all CTAs take identical CG decisions (deterministic).
// Per iteration: two local mbarrier waits (pq; rr + faces) instead of
// cluster barriers with their release/acquire fences.
//
// The arithmetic is the same Jacobi-scaled CG as the streaming kernels
// (identical scale factors and scaled weights); only the summation order of
// the dot products differs.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"

namespace cg = cooperative_groups;

namespace rwb {

constexpr int RB = 32;              // brick edge
constexpr int RCL = 8;              // CTAs per cluster (per brick)
constexpr int RPZ = RB / RCL;       // z planes per CTA
constexpr int RQ = 4;               // x voxels per thread
constexpr int RQN = RB / RQ;        // quads per row
constexpr int RT = RQN * RB;        // threads per CTA (256)
constexpr int RV = RQ * RPZ;        // voxels per thread (16)

static_assert(RPZ == 4 && RQ == 4, "register blocking assumes 4x4 voxels per thread");

struct ResidentSmem {
  float4 p[RPZ][RB][RQN];       // p planes of this slab (y neighbours)
  float4 rface[2][2][RB][RQN];  // received r faces [parity][0 = from below, 1 = from above]
  float4 rown[2][RB][RQN];      // setup: own r0 faces (read once by the neighbours)
  float4 sc[RPZ][RB][RQN];      // setup: scale factors of the slab
  float red[2][2][RCL];         // pushed partials [0 = pq, 1 = rr][parity][rank]
  float red_setup[2][RCL];      // setup partials [0 = bb, 1 = rr0][rank]
  float warp_part[2][RT / 32];
  unsigned long long barA[2];   // mbarriers: pq partials, per parity
  unsigned long long barB[2];   // mbarriers: rr partials + r faces, per parity
  int brick;
};

// ---- PTX helpers: mbarriers and DSMEM st.async -----------------------------------

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
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
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

__device__ __forceinline__ float lane_of(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ float4 f4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }

// CTA-wide sum (fixed order) -> thread 0 (uses warp_part[phase]; caller syncs before reuse)
__device__ __forceinline__ float cta_sum(ResidentSmem& sm, float v, int phase) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sm.warp_part[phase][threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < RT / 32; ++w) s += sm.warp_part[phase][w];
  }
  return s;
}

// setup: CTA partial pushed to slot `rank` of every CTA's red_setup[phase] (plain DSMEM
// stores; the caller's cluster barrier publishes them)
__device__ __forceinline__ void cluster_push(cg::cluster_group& cluster, ResidentSmem& sm, float v, int phase,
                                             int par, int rank) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sm.warp_part[phase][threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < RCL) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < RT / 32; ++w) s += sm.warp_part[phase][w];
    float* dst = cluster.map_shared_rank(&sm.red_setup[phase][rank], (unsigned)threadIdx.x);
    *dst = s;
  }
  (void)par;
}

__device__ __forceinline__ double setup_total(const ResidentSmem& sm, int phase) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < RCL; ++i) s += (double)sm.red_setup[phase][i];
  return s;
}

__device__ __forceinline__ double pushed_total(const ResidentSmem& sm, int phase, int par) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < RCL; ++i) s += (double)sm.red[phase][par][i];
  return s;
}

__device__ __forceinline__ float seedval(uint8_t s) { return s == 1 ? 1.f : 0.f; }

__global__ void __cluster_dims__(RCL, 1, 1) __launch_bounds__(RT, 1)
    resident3d_kernel(ResidentArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ResidentSmem& sm = *reinterpret_cast<ResidentSmem*>(smem_raw);
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int ly = tid / RQN;  // row
  const int xq = tid % RQN;  // quad within the row
  const int lz0 = rank * RPZ;
  const Geo& g = a.g;
  const float bw = a.beta, wmin = a.wmin;
  const ResidentSmem* below = rank > 0 ? cluster.map_shared_rank(&sm, rank - 1) : nullptr;
  const ResidentSmem* above = rank < RCL - 1 ? cluster.map_shared_rank(&sm, rank + 1) : nullptr;
  const long long offs[6] = {-g.sxy, g.sxy, -(long long)g.nx, (long long)g.nx, -1, 1};
  const int nfaces = (rank > 0) + (rank < RCL - 1);
  const uint32_t face_bytes = (uint32_t)(RB * RQN * sizeof(float4));

  if (tid == 0) {
    mbar_init(&sm.barA[0], 1);
    mbar_init(&sm.barA[1], 1);
    mbar_init(&sm.barB[0], 1);
    mbar_init(&sm.barB[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // remote addresses this thread pushes to
  uint32_t red_dst[2][2] = {{0, 0}, {0, 0}}, barA_dst[2] = {0, 0}, barB_dst[2] = {0, 0};
  uint32_t face_dn_dst[2] = {0, 0}, face_up_dst[2] = {0, 0}, bar_dn[2] = {0, 0}, bar_up[2] = {0, 0};
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    if (rank > 0) {  // my plane 0 goes to the CTA below, as its "from above" face
      face_dn_dst[par] = mapa_u32(smem_u32(&sm.rface[par][1][ly][xq]), rank - 1);
      bar_dn[par] = mapa_u32(smem_u32(&sm.barB[par]), rank - 1);
    }
    if (rank < RCL - 1) {  // my last plane goes to the CTA above, as its "from below" face
      face_up_dst[par] = mapa_u32(smem_u32(&sm.rface[par][0][ly][xq]), rank + 1);
      bar_up[par] = mapa_u32(smem_u32(&sm.barB[par]), rank + 1);
    }
    if (tid < RCL) {  // thread t < 8 delivers the CTA partials to CTA t
      red_dst[0][par] = mapa_u32(smem_u32(&sm.red[0][par][rank]), tid);
      red_dst[1][par] = mapa_u32(smem_u32(&sm.red[1][par][rank]), tid);
      barA_dst[par] = mapa_u32(smem_u32(&sm.barA[par]), tid);
      barB_dst[par] = mapa_u32(smem_u32(&sm.barB[par]), tid);
    }
  }
  cluster.sync();
  unsigned gk = 0;  // iterations run by this cluster so far (drives mbarrier parities)

  while (true) {
    if (rank == 0 && tid == 0) {
      int b = atomicAdd(a.counter, 1);
#pragma unroll
      for (int r = 0; r < RCL; ++r) *cluster.map_shared_rank(&sm.brick, (unsigned)r) = b;
    }
    cluster.sync();
    const int slot = sm.brick;
    if (slot >= a.nb) break;
    const int brick = a.list ? a.list[slot] : slot;
    const int hx = brick % g.gx;
    const int hy = (brick / g.gx) % g.gy;
    const int hz = brick / (g.gx * g.gy);
    const int gz0 = g.oz + hz * RB + lz0, gy = g.oy + hy * RB + ly, gx0 = g.ox + hx * RB + xq * RQ;
    const bool row_in = gy >= 0 && gy < g.ny;
    auto in_level = [&](int z, int i) {
      const int gz = gz0 + z, gx = gx0 + i;
      return row_in && gz >= 0 && gz < g.nz && gx >= 0 && gx < g.nx;
    };
    auto gidx = [&](int z, int i) { return (long long)(gz0 + z) * g.sxy + (long long)gy * g.nx + (gx0 + i); };
    // the six edge weights of voxel gi in the level (0 = no edge), order -z,+z,-y,+y,-x,+x
    auto weights6 = [&](int z, int i, float c, long long gi, float* wn) {
      const int gz = gz0 + z, gx = gx0 + i;
      wn[0] = gz > 0 ? edge_weight(c, __ldg(a.I + gi - g.sxy), bw, wmin) : 0.f;
      wn[1] = gz + 1 < g.nz ? edge_weight(c, __ldg(a.I + gi + g.sxy), bw, wmin) : 0.f;
      wn[2] = gy > 0 ? edge_weight(c, __ldg(a.I + gi - g.nx), bw, wmin) : 0.f;
      wn[3] = gy + 1 < g.ny ? edge_weight(c, __ldg(a.I + gi + g.nx), bw, wmin) : 0.f;
      wn[4] = gx > 0 ? edge_weight(c, __ldg(a.I + gi - 1), bw, wmin) : 0.f;
      wn[5] = gx + 1 < g.nx ? edge_weight(c, __ldg(a.I + gi + 1), bw, wmin) : 0.f;
    };

    // ---------------- setup 1: scale factors s = diag^-1/2 ----------------
    float scl[RV];
#pragma unroll
    for (int z = 0; z < RPZ; ++z)
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        scl[v] = 0.f;
        if (!in_level(z, i)) continue;
        const long long gi = gidx(z, i);
        if (__ldg(a.S + gi) != 0) continue;
        float wn[6];
        weights6(z, i, __ldg(a.I + gi), gi, wn);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < 6; ++e) d += wn[e];
        scl[v] = d > 0.f ? 1.0f / sqrtf(d) : 0.f;
      }
#pragma unroll
    for (int z = 0; z < RPZ; ++z) sm.sc[z][ly][xq] = f4(scl[z * RQ], scl[z * RQ + 1], scl[z * RQ + 2], scl[z * RQ + 3]);
    cluster.sync();

    // ---------------- setup 2: scaled weights, r0 = S(b - L x0), y0 = x0 / s ----------------
    float y[RV], r[RV], p[RV], q[RV];
    float wxf[RV], wyf[RV], wzf[RV], wyb[RV], wxb[RPZ], wzb[RQ];
    float bb_part = 0.f, rr_part = 0.f;
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
          const long long gi = gidx(z, i);
          const float x0 = a.bound ? __ldg(a.bound + gi) : 0.f;
          float wn[6];
          weights6(z, i, __ldg(a.I + gi), gi, wn);
          float diag = 0.f, b = 0.f, acc = 0.f;
#pragma unroll
          for (int e = 0; e < 6; ++e) {
            diag += wn[e];
            if (wn[e] == 0.f) continue;
            if (nsc[e] > 0.f) {  // coupled unknown of this brick
              wp[e] = wn[e] * si * nsc[e];
              acc += wn[e] * (a.bound ? __ldg(a.bound + gi + offs[e]) : 0.f);
            } else {  // Dirichlet: seed, or outside the brick
              const uint8_t s = __ldg(a.S + gi + offs[e]);
              b += wn[e] * (s ? seedval(s) : (a.bound ? __ldg(a.bound + gi + offs[e]) : 0.f));
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
      unsigned n_unk = 0;
#pragma unroll
      for (int v = 0; v < RV; ++v) n_unk += scl[v] > 0.f;
      n_unk = __reduce_add_sync(0xffffffffu, n_unk);
      if ((tid & 31) == 0 && n_unk) atomicAdd(a.unknowns, (unsigned long long)n_unk);
    }
    cluster_push(cluster, sm, bb_part, 0, 1, rank);
    cluster_push(cluster, sm, rr_part, 1, 1, rank);
    // p_0 = r_0: publish p_0 planes and the r0 faces (read once by the neighbours)
#pragma unroll
    for (int v = 0; v < RV; ++v) p[v] = r[v];
#pragma unroll
    for (int z = 0; z < RPZ; ++z) sm.p[z][ly][xq] = f4(p[z * RQ], p[z * RQ + 1], p[z * RQ + 2], p[z * RQ + 3]);
    sm.rown[0][ly][xq] = f4(r[0], r[1], r[2], r[3]);
    sm.rown[1][ly][xq] = f4(r[(RPZ - 1) * RQ], r[(RPZ - 1) * RQ + 1], r[(RPZ - 1) * RQ + 2], r[(RPZ - 1) * RQ + 3]);
    cluster.sync();
    const double bb = setup_total(sm, 0);
    double rr = setup_total(sm, 1);
    // neighbours' p_0 faces (= their r0 faces), then advanced locally every iteration
    float4 pf_dn = below ? below->rown[1][ly][xq] : f4(0, 0, 0, 0);
    float4 pf_up = above ? above->rown[0][ly][xq] : f4(0, 0, 0, 0);
    int state = ST_ACTIVE, it = 0;
    if (bb <= 0.0)
      state = ST_ZERO;
    else if (rr <= (double)a.tol2 * bb)
      state = ST_CONVERGED;
    else if (a.max_iter <= 0)
      state = ST_MAXITER;

    // ---------------- CG iterations ----------------
    while (state == ST_ACTIVE) {
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
      if (tid == 0) {
        mbar_expect_tx(&sm.barA[par], RCL * 4);
        mbar_expect_tx(&sm.barB[par], RCL * 4 + nfaces * face_bytes);
      }
      // q = A' p
      float pq_part = 0.f;
#pragma unroll
      for (int z = 0; z < RPZ; ++z) {
        const float4 pu = ly + 1 < RB ? sm.p[z][ly + 1][xq] : f4(0, 0, 0, 0);
        const float4 pd = ly > 0 ? sm.p[z][ly - 1][xq] : f4(0, 0, 0, 0);
        const float4 pzu =
            z + 1 < RPZ ? f4(p[(z + 1) * RQ], p[(z + 1) * RQ + 1], p[(z + 1) * RQ + 2], p[(z + 1) * RQ + 3]) : pf_up;
        const float4 pzd = z > 0 ? f4(p[(z - 1) * RQ], p[(z - 1) * RQ + 1], p[(z - 1) * RQ + 2], p[(z - 1) * RQ + 3])
                                 : pf_dn;
        const float pl = __shfl_up_sync(0xffffffffu, p[z * RQ + RQ - 1], 1);
        const float pr = __shfl_down_sync(0xffffffffu, p[z * RQ], 1);
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const int v = z * RQ + i;
          const float pxl = i > 0 ? p[v - 1] : pl;
          const float pxr = i < RQ - 1 ? p[v + 1] : pr;
          const float wxl = i > 0 ? wxf[v - 1] : wxb[z];
          const float wzl = z > 0 ? wzf[v - RQ] : wzb[i];
          float s = wxf[v] * pxr;
          s = fmaf(wxl, pxl, s);
          s = fmaf(wyf[v], lane_of(pu, i), s);
          s = fmaf(wyb[v], lane_of(pd, i), s);
          s = fmaf(wzf[v], lane_of(pzu, i), s);
          s = fmaf(wzl, lane_of(pzd, i), s);
          q[v] = p[v] - s;
          pq_part = fmaf(p[v], q[v], pq_part);
        }
      }
      {
        const float s = cta_sum(sm, pq_part, 0);
        const float tot = __shfl_sync(0xffffffffu, s, 0);  // warp 0 holds thread 0's sum
        if (tid < RCL) st_async_f32(par ? red_dst[0][1] : red_dst[0][0], tot, par ? barA_dst[1] : barA_dst[0]);
      }
      mbar_wait(&sm.barA[par], ph);
      const double pq = pushed_total(sm, 0, par);
      const float alpha = pq != 0.0 ? (float)(rr / pq) : 0.f;
      float rr_part = 0.f;
#pragma unroll
      for (int v = 0; v < RV; ++v) {
        y[v] = fmaf(alpha, p[v], y[v]);
        r[v] = fmaf(-alpha, q[v], r[v]);
        rr_part = fmaf(r[v], r[v], rr_part);
      }
      if (rank > 0)
        st_async_v4(par ? face_dn_dst[1] : face_dn_dst[0], f4(r[0], r[1], r[2], r[3]), par ? bar_dn[1] : bar_dn[0]);
      if (rank < RCL - 1)
        st_async_v4(par ? face_up_dst[1] : face_up_dst[0],
                    f4(r[(RPZ - 1) * RQ], r[(RPZ - 1) * RQ + 1], r[(RPZ - 1) * RQ + 2], r[(RPZ - 1) * RQ + 3]),
                    par ? bar_up[1] : bar_up[0]);
      {
        const float s = cta_sum(sm, rr_part, 1);
        const float tot = __shfl_sync(0xffffffffu, s, 0);
        if (tid < RCL) st_async_f32(par ? red_dst[1][1] : red_dst[1][0], tot, par ? barB_dst[1] : barB_dst[0]);
      }
      mbar_wait(&sm.barB[par], ph);
      const double rr_new = pushed_total(sm, 1, par);
      ++it;
      ++gk;
      if (rr_new <= (double)a.tol2 * bb) {
        state = ST_CONVERGED;
        break;
      }
      if (it >= a.max_iter) {
        state = ST_MAXITER;
        break;
      }
      const float beta = (float)(rr_new / rr);
      rr = rr_new;
      if (rank > 0) {
        const float4 rn = sm.rface[par][0][ly][xq];
        pf_dn = f4(fmaf(beta, pf_dn.x, rn.x), fmaf(beta, pf_dn.y, rn.y), fmaf(beta, pf_dn.z, rn.z),
                   fmaf(beta, pf_dn.w, rn.w));
      }
      if (rank < RCL - 1) {
        const float4 rn = sm.rface[par][1][ly][xq];
        pf_up = f4(fmaf(beta, pf_up.x, rn.x), fmaf(beta, pf_up.y, rn.y), fmaf(beta, pf_up.z, rn.z),
                   fmaf(beta, pf_up.w, rn.w));
      }
#pragma unroll
      for (int v = 0; v < RV; ++v) p[v] = fmaf(beta, p[v], r[v]);
#pragma unroll
      for (int z = 0; z < RPZ; ++z) sm.p[z][ly][xq] = f4(p[z * RQ], p[z * RQ + 1], p[z * RQ + 2], p[z * RQ + 3]);
      __syncthreads();
    }

    // ---------------- epilogue: x = s*y | seed value | bound ----------------
#pragma unroll
    for (int z = 0; z < RPZ; ++z)
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        if (!in_level(z, i)) continue;
        const long long gi = gidx(z, i);
        float x;
        if (scl[v] > 0.f) {
          x = state == ST_ZERO ? 0.f : scl[v] * y[v];
        } else {
          const uint8_t s = __ldg(a.S + gi);
          x = s ? seedval(s) : (a.bound ? __ldg(a.bound + gi) : 0.f);
        }
        a.prob[gi] = x;
        if (a.labels) a.labels[gi] = x > 0.5f ? 1 : 0;
      }
    if (rank == 0 && tid == 0) {
      a.state[slot] = state;
      a.iters[slot] = state == ST_ZERO ? 0 : it;
    }
    // every DSMEM read of this brick is done before any CTA starts the next one
    cluster.sync();
  }
}

int resident3d_supported(const Geo& g) { return g.is3d && g.bz == RB && g.by == RB && g.bx == RB; }

int launch_resident3d(const ResidentArgs& a, cudaStream_t st) {
  static thread_local int clusters = 0;
  const int smem = (int)sizeof(ResidentSmem);
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
  int grid_clusters = clusters < a.nb ? clusters : a.nb;
  resident3d_kernel<<<grid_clusters * RCL, RT, smem, st>>>(a);
  RWB_LAUNCH_CHECK("resident3d_kernel");
  count_launches(1);
  return RWB_OK;
}

}  // namespace rwb
