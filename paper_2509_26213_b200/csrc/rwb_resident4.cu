// Brick-resident Jacobi-PCG engine, 4-CTA variant: one 32^3 brick per 4-CTA
// cluster, each CTA a slab of 8 z-planes (8192 voxels), every CG iteration on chip.
//
// Why a second engine (rwb_resident.cu holds the 8-CTA one): an 8-CTA brick
// iteration takes ~1950 cycles of which only ~650 are instruction issue; the
// rest is the latency chain of the iteration (SpMV -> warp sums -> DSMEM push
// -> wait -> scalars -> update), which does not grow with the voxels per SM.
// Giving each SM twice the voxels amortises that chain over twice the work,
// and 4-CTA clusters also place better (33 clusters = 132 SMs, against 15 x 8
// = 120 SMs for 8-CTA clusters).  The register file cannot hold 8192 voxels'
// vectors AND weights, so the split is:
//   registers:      y, r, p, s, w of the thread's 4(x) x 8(z) voxels (160 floats)
//   tensor memory:  the scaled weights (per plane w'y, w'y of the row below, w'z,
//                   w'x; plus the left w'x per plane and the w'z plane below),
//                   written once per brick with tcgen05.st and read every
//                   iteration with tcgen05.ld — each thread owns one TMEM lane
//                   (32x32b shape), ~900 B/cycle/SM of read bandwidth against
//                   128 B/cycle for shared memory, which bound the SpMV when the
//                   weights lived there (3770 -> 2800 cycles per iteration)
//   shared memory:  the staged slab of the next brick (bulk copies) and the r
//                   planes (y neighbours), as in the 8-CTA engine.
// The iteration, exchange protocol, reduction order and scalar recurrences are
// those of the 8-CTA engine (see there), with 4 partials per reduction; y += alpha p
// is deferred into the next iteration's SpMV.  Bricks are handed out dynamically
// (global counter drawn one brick ahead); the staging buffer is refilled with the
// next brick's slab as soon as the current one is in registers and TMEM.
//
// Coarse correction (CC, the default; RWB_SOLVE_NO_COARSE = Jacobi-PCG): the preconditioner is
// M = I + w P D_c^-1 P^T on the Jacobi-scaled system, P = the indicator of the brick's 64
// aggregates of 8^3 voxels (one 8-plane aggregate layer per CTA, so a thread's 4 x 8 voxels lie
// in one aggregate), D_c = diag(P^T A' P) assembled without cancellation as the aggregate's
// sum of tau = m - sigma (m = unknown, sigma = its scaled weights) plus the weights leaving it,
// w = 0.8.  The additive term corrects the smooth error of a brick that Jacobi leaves for the
// Krylov space: brick iterations x0.62 in a float64 model, x0.66 measured at config 4.  Per
// iteration, u = r + c (c = w g / d per aggregate, g = P^T r): A'u = A'r + c_own tau - the
// aggregate-face differences w' (c_nb - c_own) (weights already in registers), delta = w.r +
// c_own sum(w), gamma = r.r + c . g; the cluster exchange carries each CTA's 16 aggregate sums
// of w and of r next to the two partials, so every CTA forms P^T s = P^T w + beta P^T s and the
// next g = P^T r - alpha P^T s from exact sums (a drifting g recurrence stalled at tol 1e-7),
// warps 1 and 2 update the 64 coarse values.  p is updated with u unmasked: off the unknowns
// r = w = s = 0 stay exact, only p and y drift there, and the epilogue writes the staged
// Dirichlet value (y0, prefetched) instead.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include "rwb_common.cuh"
#include "rwb_ptx.cuh"
#include "rwb_resident.cuh"

namespace cg = cooperative_groups;

#ifdef RWB_TRACE
__device__ long long g_q4_trace[4][64][8];  // phase clocks of cluster 0 (diagnostics build only)
#define Q4TRACE(k)                                                                          \
  do {                                                                                      \
    if (tid == 0 && blockIdx.x < 4 && trace_it < 64) g_q4_trace[rank][trace_it][k] = clock64(); \
  } while (0)
extern "C" int rwb_q4_trace_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_q4_trace, sizeof(g_q4_trace));
}
__device__ long long g_q4_pro[4][64][8];  // per brick of cluster 0: loop top, slab staged, loop start, epilogue done,
                                          // TMEM / registers loaded, exchange pushed, exchange received
#define Q4PRO(k)                                                                          \
  do {                                                                                    \
    if (tid == 0 && blockIdx.x < 4 && trace_b < 64) g_q4_pro[rank][trace_b][k] = clock64(); \
  } while (0)
extern "C" int rwb_q4_pro_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_q4_pro, sizeof(g_q4_pro));
}
#else
#define Q4TRACE(k) \
  do {             \
  } while (0)
#define Q4PRO(k) \
  do {           \
  } while (0)
#endif

namespace rwb {
namespace q4 {
constexpr int RB = 32;                 // brick edge
constexpr int RQ = 4;                  // x voxels per thread
constexpr int RQN = RB / RQ;           // quads per row
constexpr int PLANE = RB * RB;
constexpr int RPZ = 8;                 // z planes per CTA
constexpr int RCL = RB / RPZ;          // CTAs per cluster (4)
constexpr int RT = RQN * RB;           // threads per z-group (one per row quad)
constexpr int SLAB = RPZ * PLANE;      // voxels per CTA (8192)
constexpr int NPART = RCL;
constexpr int MAXW = 16;               // warps per CTA at most
// TZT z planes per thread: 8 -> 256 threads x 32 voxels, 4 -> 512 threads x 16 voxels
template <int TZT>
struct Cfg {
  static constexpr int NZG = RPZ / TZT;             // thread z-groups
  static constexpr int RTT = RT * NZG;              // threads per CTA
  static constexpr int RW = RTT / 32;               // warps
  static constexpr int RV = RQ * TZT;               // voxels per thread
  static constexpr int COLS = 512 / (RW / 4);       // TMEM columns per thread (warps sharing a lane quarter)
  static constexpr int TAIL = 16 * TZT;             // column of the per-plane left w'x values
  static constexpr int WZB = TAIL + 8;              // column of the w'z plane below the thread's first plane
  static constexpr int TAU = WZB + 8;               // columns of tau = m - sigma per voxel (coarse correction)
  static constexpr int WYE = TAU + 4 * TZT;         // columns of the w'y across the thread's aggregate y face
  static_assert(WYE + 4 * TZT <= COLS, "TMEM row");
};
}  // namespace q4

struct Q4Smem {
  float sx[q4::SLAB];                       // scaled weights of the slab
  float sy[q4::SLAB];
  float sz[q4::PLANE + q4::SLAB];           // w'z incl. the plane below the slab
  float sr[q4::SLAB];                       // staged r0; then the Jacobi scales for the epilogue
  float sv[q4::SLAB];                       // staged y0
  float4 rp[q4::RPZ][q4::RB + 2][q4::RQN];  // r planes (y neighbours of the SpMV), row y at y + 1; rows 0 and
                                            // RB + 1 stay zero (no neighbour past the brick's y faces)
  float4 rface[2][2][q4::RB][q4::RQN];      // received faces [parity][0 = from below, 1 = from above]
  __align__(16) float red[2][2][q4::NPART]; // pushed partials [parity][r.r, delta][rank]
  float2 wpart[q4::MAXW];
  float cgs[2][2];                          // c . g per iteration parity (two warps' halves): r.u = r.r + c . g
  unsigned long long barR[2];               // faces + partials, per parity
  unsigned long long barL;                  // slab staging
  uint32_t tmem;                            // TMEM base address (512 columns)
  unsigned long long barJ[2];               // next brick index, per parity
  int jn[2];
  // coarse correction (8^3 aggregates of the brick, index rank*16 + ay*4 + ax; see the header)
  __align__(16) float aggw[2][64];          // received aggregate sums per parity: P^T w, or P^T r0 at brick start
  __align__(16) float aggr[2][64];          // received aggregate sums per parity: P^T r of the iteration's r
  __align__(16) float aggd[64];             // received aggregate diagonals (brick start)
  float cc[64];                             // c per aggregate
  float cst[3][64];                         // g = P^T r, P^T s, 1/d (updated by warp 1)
  float wagg[3][8][4];                      // per warp: 4 aggregate half sums (w, r; or r0 / d at brick start)
};

// Bulk-copy `slot`'s slab of this CTA into shared memory (one thread; completes on barL).
__device__ __forceinline__ void q4_stage(const ResidentArgs& a, Q4Smem& sm, int slot, int rank) {
  using namespace q4;
  const long long base = (long long)slot * (RB * RB * RB) + (long long)rank * SLAB;
  const uint32_t slab_bytes = SLAB * 4;
  const uint32_t zbytes = rank > 0 ? slab_bytes + PLANE * 4 : slab_bytes;
  mbar_expect_tx(&sm.barL, 4 * slab_bytes + zbytes);
  bulk_g2s(sm.sx, a.wx + base, slab_bytes, &sm.barL);
  bulk_g2s(sm.sy, a.wy + base, slab_bytes, &sm.barL);
  if (rank > 0)
    bulk_g2s(sm.sz, a.wz + base - PLANE, zbytes, &sm.barL);
  else
    bulk_g2s(sm.sz + PLANE, a.wz + base, zbytes, &sm.barL);
  bulk_g2s(sm.sr, a.r0 + base, slab_bytes, &sm.barL);
  bulk_g2s(sm.sv, a.y + base, slab_bytes, &sm.barL);
}

__device__ __forceinline__ void q4_prefetch(const ResidentArgs& a, int slot, int rank, bool y0) {
  using namespace q4;
  const long long base = (long long)slot * (RB * RB * RB) + (long long)rank * SLAB;
  prefetch_l2(a.sc + base, SLAB * 4);
  if (y0) prefetch_l2(a.y + base, SLAB * 4);  // the Dirichlet values the coarse-corrected epilogue writes
}

constexpr float kCcOmega = 0.8f;  // damping of the coarse correction

template <int TZT, bool CC>
__global__ void __launch_bounds__(q4::Cfg<TZT>::RTT, 1) resident3d_q4_kernel(ResidentArgs a) {
  using namespace q4;
  using C = Cfg<TZT>;
  constexpr int NZG = C::NZG, RTT = C::RTT, RW = C::RW, RV = C::RV;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Q4Smem& sm = *reinterpret_cast<Q4Smem*>(smem_raw);
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int zg = tid / RT;          // z-group: planes [pz0, pz0 + TZT) of the slab
  const int ly = (tid % RT) / RQN;  // row
  const int xq = tid % RQN;         // quad within the row
  const int pz0 = zg * TZT;
  const bool below = rank > 0, above = rank < RCL - 1;
  const bool first_zg = zg == 0, last_zg = zg == NZG - 1;
  const int nfaces = (int)below + (int)above;
  const uint32_t tx_faces = nfaces * (uint32_t)(RB * RQN * sizeof(float4));
  const int cid = blockIdx.x / RCL, ncl = gridDim.x / RCL;
  const int n_act = *a.n_active;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.barR[i], 1);
      mbar_init(&sm.barJ[i], 1);
    }
    mbar_init(&sm.barL, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (rank == 0)  // the CTA holding plane 0 has no plane below
    for (int i = tid; i < PLANE; i += RTT) sm.sz[i] = 0.f;
  for (int i = tid; i < RPZ * 2 * RQN; i += RTT) {  // the zero rows past the y faces
    const int pz = i / (2 * RQN), e = (i / RQN) & 1, x = i % RQN;
    sm.rp[pz][e ? RB + 1 : 0][x] = f4(0.f, 0.f, 0.f, 0.f);
  }
  // pushes (remote addresses formed where used: registers are the scarce resource here):
  // plane 0 goes to the CTA below as its "from above" face, plane 7 to the CTA above as its
  // "from below" face, lane t of warp 0 delivers the CTA's partials to CTA t
  auto push_dn = [&](int par, float4 v) {
    st_async_v4(mapa_u32(smem_u32(&sm.rface[par][1][ly][xq]), rank - 1), v, mapa_u32(smem_u32(&sm.barR[par]), rank - 1));
  };
  auto push_up = [&](int par, float4 v) {
    st_async_v4(mapa_u32(smem_u32(&sm.rface[par][0][ly][xq]), rank + 1), v, mapa_u32(smem_u32(&sm.barR[par]), rank + 1));
  };
  auto push_parts = [&](int par, float g, float d) {
    const uint32_t dst = mapa_u32(smem_u32(&sm.red[par][0][rank]), lane), bar = mapa_u32(smem_u32(&sm.barR[par]), lane);
    st_async_f32(dst, g, bar);
    st_async_f32(dst + NPART * 4, d, bar);
  };
  constexpr uint32_t tx_parts = 2 * NPART * 4;
  static_assert(!CC || TZT == 8, "the coarse correction maps one 8^3 aggregate layer per CTA (8 planes per thread)");
  // this thread's aggregate and its neighbours across the aggregate faces it touches
  const int ax = xq >> 1, ay = ly >> 3;
  const int agg = rank * 16 + ay * 4 + ax;
  const int agg_x = (xq & 1) ? (ax < 3 ? agg + 1 : agg) : (ax > 0 ? agg - 1 : agg);
  const bool ydn = (ly & 7) == 0, yup = (ly & 7) == 7;
  const int agg_y = ydn ? (ay > 0 ? agg - 4 : agg) : (yup ? (ay < 3 ? agg + 4 : agg) : agg);
  const uint32_t tx_agg = CC ? RCL * 16 * 4 : 0;  // aggregate sums received per exchange
  // warp 0 lanes 0..15: the CTA's 16 aggregate sums (halves from the warp pairs covering their 8 rows),
  // one float4 (4 aggregates of a row band) to each CTA of the cluster
  auto push_agg = [&](int par, float* dst, const float (*wg)[4]) {
    const int dest = lane >> 2, by = lane & 3;
    const float4 v = f4(wg[2 * by][0] + wg[2 * by + 1][0], wg[2 * by][1] + wg[2 * by + 1][1],
                        wg[2 * by][2] + wg[2 * by + 1][2], wg[2 * by][3] + wg[2 * by + 1][3]);
    st_async_v4(mapa_u32(smem_u32(dst + rank * 16 + by * 4), dest), v, mapa_u32(smem_u32(&sm.barR[par]), dest));
  };
  // sum over the 16 threads of an aggregate inside the warp (quad pairs, the warp's 4 rows): lanes 0, 2, 4, 6
  auto agg_warp_sum = [&](float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
  };
  if (warp == 0) tmem_alloc(&sm.tmem, 512);
  tmem_fence_before();
  cluster.sync();
  tmem_fence_after();
  // this thread's TMEM row: lane quarter of its warp, column block by warp / 4
  const uint32_t tb = sm.tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * C::COLS);
  unsigned gk = 0, usesL = 0, uJ = 0;

  // dynamic brick scheduling as in the 8-CTA engine: bricks cid and cid + ncl static, then a
  // global counter drawn one brick ahead by rank 0 and pushed into the cluster's CTAs
  if (cid < n_act && tid == 0) {
    q4_stage(a, sm, a.alist[cid], rank);
    q4_prefetch(a, a.alist[cid], rank, CC);
  }
#ifdef RWB_TRACE
  int trace_b = 0;
#endif
  for (int j = cid, jn = cid + ncl, jnn; j < n_act; j = jn, jn = jnn) {
    Q4PRO(0);
    const int slot = a.alist[j];
    const bool draw = jn < n_act;
    const int parJ = uJ & 1;
    int jd = 0;
    if (draw && tid == 0) {
      mbar_expect_tx(&sm.barJ[parJ], 4);
      if (rank == 0) jd = 2 * ncl + atomicAdd(a.next, 1);
    }
    // the unknowns of this thread's voxels (s > 0), from the scales prefetched into L2 when the
    // brick was staged; the loads overlap the staging wait
    float4 s4c[CC ? TZT : 1];
    if (CC) {
      const long long sb = (long long)slot * (RB * RB * RB) + (long long)rank * SLAB;
#pragma unroll
      for (int z = 0; z < TZT; ++z)
        s4c[z] = __ldg(reinterpret_cast<const float4*>(a.sc + sb + (pz0 + z) * PLANE + ly * RB + xq * RQ));
    }
    mbar_wait(&sm.barL, usesL & 1);
    ++usesL;
    Q4PRO(1);

    // the slab's weights into this thread's TMEM row: per plane z, columns 16z.. hold w'y of
    // the quad, w'y of the row below, w'z and w'x of the quad; columns TAIL.. the w'x left of
    // the quad for each plane, WZB.. the w'z plane below the thread's first plane
    float dpart = 0.f;  // coarse correction: this thread's share of its aggregate's diagonal d_I
    {
      float tt[16];
      float tau[2][16];  // tau = m - sigma per voxel (m = 1 on unknowns, sigma = sum of the 6 scaled weights)
      float wye[2][16];  // w'y across the aggregate's y face the thread's row touches (row below / above)
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const int o = (pz0 + z) * PLANE + ly * RB + xq * RQ;
        const float4 wx4 = *reinterpret_cast<const float4*>(&sm.sx[o]);
        const float4 wy4 = *reinterpret_cast<const float4*>(&sm.sy[o]);
        const float4 wz4 = *reinterpret_cast<const float4*>(&sm.sz[PLANE + o]);
        const float4 wyb4 = ly > 0 ? *reinterpret_cast<const float4*>(&sm.sy[o - RB]) : f4(0, 0, 0, 0);
        const float v[16] = {wy4.x, wy4.y, wy4.z, wy4.w, wyb4.x, wyb4.y, wyb4.z, wyb4.w,
                             wz4.x, wz4.y, wz4.z, wz4.w, wx4.x, wx4.y, wx4.z, wx4.w};
        tmem_st16(tb + 16 * z, v);
        tt[z] = xq > 0 ? sm.sx[o - 1] : 0.f;
        if (CC) {
          // d_I = sum over the aggregate of tau + the weights of the edges leaving it (no cancellation)
          const float4 wzd4 = *reinterpret_cast<const float4*>(&sm.sz[o]);  // w'z of the plane below
          const float4 s4 = s4c[CC ? z : 0];
#pragma unroll
          for (int i = 0; i < RQ; ++i) {
            const float wxl = i > 0 ? lane_of(wx4, i - 1) : tt[z];
            const float sig = ((lane_of(wx4, i) + wxl) + (lane_of(wy4, i) + lane_of(wyb4, i))) +
                              (lane_of(wz4, i) + lane_of(wzd4, i));
            const float t = (lane_of(s4, i) > 0.f ? 1.f : 0.f) - sig;
            tau[(z * RQ + i) >> 4][(z * RQ + i) & 15] = t;
            wye[(z * RQ + i) >> 4][(z * RQ + i) & 15] = ydn ? lane_of(wyb4, i) : lane_of(wy4, i);
            dpart += t;
            if (ydn) dpart += lane_of(wyb4, i);
            if (yup) dpart += lane_of(wy4, i);
            if (z == 0) dpart += lane_of(wzd4, i);
            if (z == TZT - 1) dpart += lane_of(wz4, i);
          }
          dpart += (xq & 1) ? lane_of(wx4, 3) : tt[z];
        }
      }
      if (CC) {
        tmem_st16(tb + C::TAU, tau[0]);
        tmem_st16(tb + C::TAU + 16, tau[1]);
        tmem_st16(tb + C::WYE, wye[0]);
        tmem_st16(tb + C::WYE + 16, wye[1]);
      }
#pragma unroll
      for (int z = TZT; z < 8; ++z) tt[z] = 0.f;
      const float4 wzb4 = *reinterpret_cast<const float4*>(&sm.sz[pz0 * PLANE + ly * RB + xq * RQ]);
      tt[8] = wzb4.x, tt[9] = wzb4.y, tt[10] = wzb4.z, tt[11] = wzb4.w;
      tt[12] = tt[13] = tt[14] = tt[15] = 0.f;
      tmem_st16(tb + C::TAIL, tt);
    }
    float y[RV], r[RV], p[RV], sv[RV], w[RV];
#pragma unroll
    for (int z = 0; z < TZT; ++z) {
      const int o = (pz0 + z) * PLANE + ly * RB + xq * RQ;
      const float4 fr = *reinterpret_cast<const float4*>(&sm.sr[o]);
      const float4 fv = *reinterpret_cast<const float4*>(&sm.sv[o]);
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        r[v] = lane_of(fr, i);
        y[v] = lane_of(fv, i);
        p[v] = sv[v] = w[v] = 0.f;
      }
    }
    const float thresh = (float)((double)a.tol2 * a.bb[slot]);
    if (draw && rank == 0 && tid == 0) {
#pragma unroll 1
      for (int c = 0; c < RCL; ++c)
        st_async_f32(mapa_u32(smem_u32(&sm.jn[parJ]), c), __int_as_float(jd), mapa_u32(smem_u32(&sm.barJ[parJ]), c));
    }

    float alpha = 0.f, rgamma = 0.f, ralpha = 0.f;  // 1/gamma, 1/alpha one iteration ahead
    int state = ST_ACTIVE, it = 0;
    float4 rf_dn = f4(0, 0, 0, 0), rf_up = f4(0, 0, 0, 0);
    float4 sf_dn = f4(0, 0, 0, 0), sf_up = f4(0, 0, 0, 0);
    const float4 z4 = f4(0, 0, 0, 0);
    auto plane4 = [&](const float* v, int z) { return f4(v[z * RQ], v[z * RQ + 1], v[z * RQ + 2], v[z * RQ + 3]); };
    Q4PRO(4);
#pragma unroll
    for (int z = 0; z < TZT; ++z) sm.rp[pz0 + z][ly + 1][xq] = plane4(r, z);
    {
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
      if (tid == 0) mbar_expect_tx(&sm.barR[par], tx_faces + tx_parts + 2 * tx_agg);
      if (below && first_zg) push_dn(par, plane4(r, 0));
      if (above && last_zg) push_up(par, plane4(r, TZT - 1));
      if (warp == 0 && lane < RCL) push_parts(par, 0.f, 0.f);
      if (CC) {  // the aggregates' P^T r0 and d_I, all 64 to every CTA
        float gpart = 0.f;
#pragma unroll
        for (int v = 0; v < RV; ++v) gpart += r[v];
        const float gv = agg_warp_sum(gpart), dv = agg_warp_sum(dpart);
        if ((lane & 0x19) == 0) {
          sm.wagg[0][warp][lane >> 1] = gv;
          sm.wagg[1][warp][lane >> 1] = dv;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(RTT) : "memory");
        if (warp == 0 && lane < 16)  // the two arrays from two warps, in parallel
          push_agg(par, sm.aggw[par], sm.wagg[0]);
        else if (warp == 1 && lane < 16)
          push_agg(par, sm.aggd, sm.wagg[1]);
      }
      Q4PRO(5);
      mbar_wait(&sm.barR[par], ph);
      Q4PRO(6);
      ++gk;
      if (below && first_zg) rf_dn = sm.rface[par][0][ly][xq];
      if (above && last_zg) rf_up = sm.rface[par][1][ly][xq];
      if (CC && (warp == 1 || warp == 2)) {  // coarse state: g = P^T r0, P^T s = 0, c = w g / d
        const int I = lane + 32 * (warp - 1);
        const float g = sm.aggw[par][I], d = sm.aggd[I];
        const float di = d > 1e-6f ? 1.f / d : 0.f;
        sm.cst[0][I] = g;
        sm.cst[1][I] = 0.f;
        sm.cst[2][I] = di;
        const float c = kCcOmega * g * di;
        sm.cc[I] = c;
        const float cg = warp_sum(c * g);
        if (lane == 0) sm.cgs[0][warp - 1] = cg;
      }
      tmem_wait_st();
      __syncthreads();  // r planes published; every thread has left the staged slab
    }
    // the staging buffer is free: bring in the next brick's slab while this one iterates
    if (draw && tid == 0) {
      q4_stage(a, sm, a.alist[jn], rank);
      q4_prefetch(a, a.alist[jn], rank, CC);  // its scales (unknown mask, epilogue) and y0
    }

#ifdef RWB_TRACE
    int trace_it = (int)gk;
#endif
    Q4PRO(2);
    for (int pass = 0;; ++pass) {
      Q4TRACE(0);
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
      if (tid == 0) mbar_expect_tx(&sm.barR[par], tx_faces + tx_parts + 2 * tx_agg);
      // u = r + c (c of the voxel's aggregate): the SpMV runs on r, and the c part enters as
      // c_own * tau plus the differences (c_neighbour - c_own) across the aggregate faces
      float c_own = 0.f, dxc = 0.f, dyc = 0.f, dzd = 0.f, dzu = 0.f, wsa = 0.f, wsb = 0.f, rsa = 0.f, rsb = 0.f;
      if (CC) {
        c_own = sm.cc[agg];
        dxc = sm.cc[agg_x] - c_own;
        dyc = sm.cc[agg_y] - c_own;
        dzd = below ? sm.cc[agg - 16] - c_own : 0.f;
        dzu = above ? sm.cc[agg + 16] - c_own : 0.f;
      }
      // the x-face difference on the side the thread's quad touches (the other side's term is 0)
      const float dxl = (xq & 1) ? 0.f : dxc, dxr = (xq & 1) ? dxc : 0.f;
      // w = A'r with the scaled weights from tensor memory
      float gp[2] = {0.f, 0.f}, dp[2] = {0.f, 0.f};
      float4 wzl4;  // w'z of the plane below the slab
      {
        float t4[4];
        tmem_ld4(tb + C::WZB, t4);
        tmem_wait_ld4(t4);
        wzl4 = f4(t4[0], t4[1], t4[2], t4[3]);
      }
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const int pz = pz0 + z;
        // plane z's weights, loaded once plane z-1 is done (the empty asm ties the address to its
        // result, so the compiler cannot hoist all eight loads up front and run out of registers)
        float ta[12];
        uint32_t ad = tb + 16 * z;
        if (z > 0) asm volatile("" : "+r"(ad) : "f"(w[z * RQ - 1]));
#ifdef RWB_EXP_NOTMEM  // diagnostics only: the SpMV without its TMEM latency (wrong weights)
#pragma unroll
        for (int k = 0; k < 12; ++k) ta[k] = 0.01f * (float)(k + 1) + 1e-9f * (float)ad;
#else
        tmem_ld8(ad, ta);
        tmem_ld4p(ad + 8, ta + 8);
        tmem_wait_ld12(ta);
#endif
        const float4 wy4 = f4(ta[0], ta[1], ta[2], ta[3]);
        const float4 wyb4 = f4(ta[4], ta[5], ta[6], ta[7]);
        const float4 wz4 = f4(ta[8], ta[9], ta[10], ta[11]);
        const float4 ru = sm.rp[pz][ly + 2][xq];
        const float4 rd = sm.rp[pz][ly][xq];
        const float4 rzu = z + 1 < TZT ? plane4(r, z + 1) : (pz + 1 < RPZ ? sm.rp[pz + 1][ly + 1][xq] : rf_up);
        const float4 rzd = z > 0 ? plane4(r, z - 1) : (pz > 0 ? sm.rp[pz - 1][ly + 1][xq] : rf_dn);
        const float rl = __shfl_up_sync(0xffffffffu, r[z * RQ + RQ - 1], 1);
        const float rr_ = __shfl_down_sync(0xffffffffu, r[z * RQ], 1);
        float acc[RQ];
#pragma unroll
        for (int i = 0; i < RQ; i += 2) {
          fma2(acc[i], acc[i + 1], lane_of(wy4, i), lane_of(wy4, i + 1), lane_of(ru, i), lane_of(ru, i + 1), 0.f, 0.f);
          fma2(acc[i], acc[i + 1], lane_of(wyb4, i), lane_of(wyb4, i + 1), lane_of(rd, i), lane_of(rd, i + 1), acc[i],
               acc[i + 1]);
          fma2(acc[i], acc[i + 1], lane_of(wz4, i), lane_of(wz4, i + 1), lane_of(rzu, i), lane_of(rzu, i + 1), acc[i],
               acc[i + 1]);
          fma2(acc[i], acc[i + 1], lane_of(wzl4, i), lane_of(wzl4, i + 1), lane_of(rzd, i), lane_of(rzd, i + 1), acc[i],
               acc[i + 1]);
        }
        float tx[13];  // w'x of the quad and the one left of it (+ tau, + the y-face w'y), once the y / z terms are done
        uint32_t adx = tb + 16 * z + 12, adl = tb + C::TAIL + z;
        asm volatile("" : "+r"(adx), "+r"(adl) : "f"(acc[0]), "f"(acc[2]));
#ifdef RWB_EXP_NOTMEM
#pragma unroll
        for (int k = 0; k < 9; ++k) tx[k] = 0.01f * (float)(k + 1) + 1e-9f * (float)(adx + adl);
#else
        tmem_ld4p(adx, tx);
        tmem_ld1(adl, tx[4]);
        if (CC) {
          tmem_ld4p(tb + C::TAU + RQ * z, tx + 5);
          tmem_ld4p(tb + C::WYE + RQ * z, tx + 9);
          tmem_wait_ld13(tx);
        } else {
          tmem_wait_ld5(tx);
        }
#endif
        const float4 wx4 = f4(tx[0], tx[1], tx[2], tx[3]);
        const float wxl0 = tx[4];
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const int v = z * RQ + i;
          const float rxl = i > 0 ? r[v - 1] : rl;
          const float rxr = i < RQ - 1 ? r[v + 1] : rr_;
          const float wxl = i > 0 ? lane_of(wx4, i - 1) : wxl0;
          acc[i] = fmaf(lane_of(wx4, i), rxr, acc[i]);
          acc[i] = fmaf(wxl, rxl, acc[i]);
        }
        // coarse part of A'u: c_own tau - sum over the aggregate faces of w' (c_neighbour - c_own)
        if (CC) {
#pragma unroll
          for (int i = 0; i < RQ; ++i) acc[i] = fmaf(tx[9 + i], dyc, acc[i]);
          if (z == 0) {
#pragma unroll
            for (int i = 0; i < RQ; ++i) acc[i] = fmaf(lane_of(wzl4, i), dzd, acc[i]);
          }
          if (z == TZT - 1) {
#pragma unroll
            for (int i = 0; i < RQ; ++i) acc[i] = fmaf(lane_of(wz4, i), dzu, acc[i]);
          }
          acc[0] = fmaf(wxl0, dxl, acc[0]);
          acc[RQ - 1] = fmaf(lane_of(wx4, RQ - 1), dxr, acc[RQ - 1]);
        }
#pragma unroll
        for (int i = 0; i < RQ; i += 2) {
          const int v = z * RQ + i;
          fma2(w[v], w[v + 1], -1.f, -1.f, acc[i], acc[i + 1], r[v], r[v + 1]);
          if (CC) {
            fma2(w[v], w[v + 1], c_own, c_own, tx[5 + i], tx[6 + i], w[v], w[v + 1]);
            fma2(wsa, wsb, 1.f, 1.f, w[v], w[v + 1], wsa, wsb);
            fma2(rsa, rsb, 1.f, 1.f, r[v], r[v + 1], rsa, rsb);
          }
          fma2(gp[0], gp[1], r[v], r[v + 1], r[v], r[v + 1], gp[0], gp[1]);
          fma2(dp[0], dp[1], w[v], w[v + 1], r[v], r[v + 1], dp[0], dp[1]);
        }
        wzl4 = wz4;
      }
      Q4TRACE(1);
      if (below && first_zg) push_dn(par, plane4(w, 0));
      if (above && last_zg) push_up(par, plane4(w, TZT - 1));
      {
        const float gs = gp[0] + gp[1];
        // u = r + c_own on the unknowns (r = w = 0 off them): delta = w.u = w.r + c_own sum(w),
        // gamma = r.u = r.r + c_own sum(r)
        const float ds = CC ? fmaf(c_own, wsa + wsb, dp[0] + dp[1]) : dp[0] + dp[1];
        const float gw = warp_sum(gs);
        const float dw = warp_sum(ds);
        if (lane == 0) sm.wpart[warp] = make_float2(gw, dw);
        if (CC) {
          const float wv = agg_warp_sum(wsa + wsb), rv = agg_warp_sum(rsa + rsb);
          if ((lane & 0x19) == 0) {
            sm.wagg[0][warp][lane >> 1] = wv;
            sm.wagg[2][warp][lane >> 1] = rv;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(RTT) : "memory");
        if (warp == 0) {
          float gc = 0.f, dc = 0.f;
#pragma unroll
          for (int wv = 0; wv < RW; ++wv) {
            const float2 v = sm.wpart[wv];
            gc += v.x;
            dc += v.y;
          }
          if (lane < RCL) push_parts(par, gc, dc);
        } else if (CC && warp == 1 && lane < 16) {  // the aggregate sums in parallel with warp 0's partials
          push_agg(par, sm.aggw[par], sm.wagg[0]);
          push_agg(par, sm.aggr[par], sm.wagg[2]);
        }
      }
      // the previous iteration's y += alpha p, deferred off the update -> publish -> barrier chain
      // into the exchange wait (nothing reads y until the epilogue; the SpMV is issue-bound)
      if (pass > 0) {
#pragma unroll
        for (int v = 0; v < RV; v += 2) fma2(y[v], y[v + 1], alpha, alpha, p[v], p[v + 1], y[v], y[v + 1]);
      }
      Q4TRACE(2);
      mbar_wait(&sm.barR[par], ph);
      Q4TRACE(3);
      ++gk;
      const float g_new = sum_parts<NPART>(sm.red[par][0]);  // r.r (the stop rule)
      const float delta = sum_parts<NPART>(sm.red[par][1]);
      // r.u = r.r + c . g, g = P^T r (one step from this iteration's exact aggregate sums)
      const float gam = CC ? g_new + (sm.cgs[pass & 1][0] + sm.cgs[pass & 1][1]) : g_new;
      float beta;
      if (pass == 0) {
        beta = 0.f;
        alpha = delta != 0.f ? gam * rcp_ftz(delta) : 0.f;
        if (a.max_iter <= 0) {
          state = ST_MAXITER;
          break;
        }
      } else {
        if (g_new <= thresh) {
          state = ST_CONVERGED;
          break;
        }
        if (it >= a.max_iter) {
          state = ST_MAXITER;
          break;
        }
        beta = gam * rgamma;
        const float den = delta - beta * (gam * ralpha);
        alpha = den != 0.f ? gam * rcp_ftz(den) : 0.f;
      }
      rgamma = rcp_ftz(gam);
      ralpha = rcp_ftz(alpha);
      if (CC && (warp == 1 || warp == 2)) {  // next c: P^T s = P^T w + beta P^T s, g -= alpha P^T s, c = w g / d
        const int I = lane + 32 * (warp - 1);
        // P^T r of the next residual from this iteration's exact P^T r (no drift over iterations)
        const float ps = fmaf(beta, sm.cst[1][I], sm.aggw[par][I]);
        const float g = fmaf(-alpha, ps, sm.aggr[par][I]);
        const float c = kCcOmega * g * sm.cst[2][I];
        sm.cst[1][I] = ps;
        sm.cst[0][I] = g;
        sm.cc[I] = c;
        const float cg = warp_sum(c * g);
        if (lane == 0) sm.cgs[(pass + 1) & 1][warp - 1] = cg;
      }
      Q4TRACE(4);
#pragma unroll
      for (int v = 0; v < RV; v += 2) {
        // p = u + beta p, u = r + c_own (unmasked: p drifts off the unknowns, where only y reads it,
        // and the epilogue writes the staged Dirichlet value there instead)
        if (CC)
          fma2(p[v], p[v + 1], beta, beta, p[v], p[v + 1], r[v] + c_own, r[v + 1] + c_own);
        else
          fma2(p[v], p[v + 1], beta, beta, p[v], p[v + 1], r[v], r[v + 1]);
        fma2(sv[v], sv[v + 1], beta, beta, sv[v], sv[v + 1], w[v], w[v + 1]);
        fma2(r[v], r[v + 1], -alpha, -alpha, sv[v], sv[v + 1], r[v], r[v + 1]);
      }
      ++it;
      if (below && first_zg) {
        const float4 wn = sm.rface[par][0][ly][xq];
        sf_dn = f4(fmaf(beta, sf_dn.x, wn.x), fmaf(beta, sf_dn.y, wn.y), fmaf(beta, sf_dn.z, wn.z), fmaf(beta, sf_dn.w, wn.w));
        rf_dn = f4(fmaf(-alpha, sf_dn.x, rf_dn.x), fmaf(-alpha, sf_dn.y, rf_dn.y), fmaf(-alpha, sf_dn.z, rf_dn.z),
                   fmaf(-alpha, sf_dn.w, rf_dn.w));
      }
      if (above && last_zg) {
        const float4 wn = sm.rface[par][1][ly][xq];
        sf_up = f4(fmaf(beta, sf_up.x, wn.x), fmaf(beta, sf_up.y, wn.y), fmaf(beta, sf_up.z, wn.z), fmaf(beta, sf_up.w, wn.w));
        rf_up = f4(fmaf(-alpha, sf_up.x, rf_up.x), fmaf(-alpha, sf_up.y, rf_up.y), fmaf(-alpha, sf_up.z, rf_up.z),
                   fmaf(-alpha, sf_up.w, rf_up.w));
      }
#pragma unroll
      for (int z = 0; z < TZT; ++z) sm.rp[pz0 + z][ly + 1][xq] = plane4(r, z);
      Q4TRACE(5);
      __syncthreads();
      Q4TRACE(6);
#ifdef RWB_TRACE
      ++trace_it;
#endif
    }
    Q4PRO(7);
    // epilogue: probabilities and labels straight into the level
    {
      const long long sbase = (long long)slot * (RB * RB * RB) + (long long)rank * SLAB;
      const int brick = a.list ? a.list[slot] : slot;
      const int hx = brick % a.gx, hy = (brick / a.gx) % a.gy, hz = brick / (a.gx * a.gy);
      const int gy = a.oy + hy * RB + ly, gx0 = a.ox + hx * RB + xq * RQ;
      const bool row_in = gy >= 0 && gy < a.ny;
      const bool quad_in = gx0 >= 0 && gx0 + RQ <= a.nx;
      // all planes' scales (and Dirichlet values) first: one load latency for the brick, not one
      // per plane (the stores below would otherwise keep each plane's loads behind the last store)
      float4 s4v[TZT], y0v[CC ? TZT : 1];
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const long long o = sbase + (pz0 + z) * PLANE + ly * RB + xq * RQ;
        s4v[z] = __ldg(reinterpret_cast<const float4*>(a.sc + o));
        if (CC) y0v[CC ? z : 0] = __ldcg(reinterpret_cast<const float4*>(a.y + o));
      }
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const int gz = a.oz + hz * RB + rank * RPZ + pz0 + z;
        if (!row_in || gz < 0 || gz >= a.nz) continue;
        const float4 s4 = s4v[z];
        const float4 y04 = CC ? y0v[CC ? z : 0] : f4(0.f, 0.f, 0.f, 0.f);
        float pv[RQ];
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const float s = lane_of(s4, i), yv = y[z * RQ + i];
          pv[i] = s > 0.f ? s * yv : (CC ? lane_of(y04, i) : yv);
        }
        const long long gi = ((long long)gz * a.ny + gy) * a.nx + gx0;
        if (quad_in && (gi & 3) == 0) {
          *reinterpret_cast<float4*>(a.prob + gi) = f4(pv[0], pv[1], pv[2], pv[3]);
          if (a.labels)
            *reinterpret_cast<uchar4*>(a.labels + gi) = make_uchar4(pv[0] > 0.5f, pv[1] > 0.5f, pv[2] > 0.5f, pv[3] > 0.5f);
        } else {
#pragma unroll
          for (int i = 0; i < RQ; ++i) {
            if (gx0 + i < 0 || gx0 + i >= a.nx) continue;
            a.prob[gi + i] = pv[i];
            if (a.labels) a.labels[gi + i] = pv[i] > 0.5f ? 1 : 0;
          }
        }
      }
    }
    if (rank == 0 && tid == 0) {
      a.state[slot] = state;
      a.iters[slot] = it;
    }
    Q4PRO(3);
#ifdef RWB_TRACE
    ++trace_b;
#endif
    jnn = n_act;
    if (draw) {
      mbar_wait(&sm.barJ[parJ], (uJ >> 1) & 1);
      jnn = sm.jn[parJ];
      ++uJ;
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(sm.tmem, 512);
}

template <int TZT, bool CC>
static int launch_q4(const ResidentArgs& a, int max_bricks, cudaStream_t st) {
  using namespace q4;
  constexpr int RTT = Cfg<TZT>::RTT;
  auto kern = resident3d_q4_kernel<TZT, CC>;
  static DeviceCache cache;
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int clusters = cache[dev].load(std::memory_order_relaxed);
  const int smem = (int)sizeof(Q4Smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = RCL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.blockDim = dim3(RTT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (!clusters) {
    RWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cfg.gridDim = dim3(RCL * 1024, 1, 1);
    int n = 0;
    RWB_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    if (n <= 0) return fail(RWB_ERR_UNSUPPORTED, "no 4-CTA brick cluster fits on this device");
    clusters = n;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  const int grid_clusters = clusters < max_bricks ? clusters : max_bricks;
  if (grid_clusters <= 0) return RWB_OK;
  cfg.gridDim = dim3(grid_clusters * RCL, 1, 1);
  RWB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  count_launches(1);
  return RWB_OK;
}

int launch_resident3d_q4(const ResidentArgs& a, int max_bricks, cudaStream_t st) {
  static const int threads = [] {  // diagnostics: RWB_Q4_THREADS=512 (4 planes per thread)
    const char* e = getenv("RWB_Q4_THREADS");
    return e ? atoi(e) : 256;
  }();
  static const bool cc_env = [] {  // RWB_Q4_CC=0: plain Jacobi-PCG everywhere (diagnostics)
    const char* e = getenv("RWB_Q4_CC");
    return !(e && atoi(e) == 0);
  }();
  if (threads == 512) return launch_q4<4, false>(a, max_bricks, st);
  return (cc_env && a.coarse) ? launch_q4<8, true>(a, max_bricks, st) : launch_q4<8, false>(a, max_bricks, st);
}

}  // namespace rwb
