// Brick-resident Jacobi-PCG engine: one 32^3 brick per 8-CTA thread-block
// cluster, every CG iteration on chip.
//
// The streaming solver (rwb_solve.cu) moves 52 B per voxel per CG iteration
// through HBM.  A 32^3 brick's complete CG state — y, r, p, s, w and its six
// scaled edge weights, ~10 floats per voxel = 1.25 MiB — fits in the register
// files of 8 SMs (8 x 256 KB), so a cluster of 8 CTAs owns one brick: CTA `c`
// holds z-planes [4c, 4c+4), each of its 256 threads a 4(x) x 4(z) block of
// voxels in registers.
//
// The system itself (scaled weights, r0, y0, ||S b||^2, per-brick decisions)
// is built by the high-occupancy streaming setup kernels into the brick-local
// workspace; this kernel only iterates.  A brick's slab inputs are contiguous
// in that layout, so each CTA stages them with five 1-D bulk copies
// (`cp.async.bulk` global -> shared, completing on an mbarrier) — for the NEXT
// brick, double-buffered, while the current brick iterates — and writes y back
// with coalesced float4 stores; the streaming epilogue kernel turns y into
// probabilities and labels.  HBM traffic per brick voxel: 20 B in, 4 B out,
// once per solve, instead of 52 B per iteration.
//
// The iteration is the single-reduction CG of Chronopoulos & Gear (1989):
// with w = A'r and s = A'p carried as vectors, both dot products of an
// iteration, gamma = r.r and delta = w.r, are reduced together, and
//   beta = gamma_new / gamma,  alpha = gamma_new / (delta - beta gamma_new / alpha),
//   p = r + beta p,  s = w + beta s,  y += alpha p,  r -= alpha s,  w = A'r.
// An on-chip brick solve is bound by the latency of each iteration's chain
// (neighbour exchange -> SpMV -> cluster-wide reduction); this form has one
// cluster-wide reduction per iteration instead of two.
//
// Neighbour exchange per iteration (no cluster-wide barrier inside the loop):
//   x: warp shuffles (lanes of a row are x-consecutive quads)
//   y: r planes in shared memory (LDS.128 of the rows above / below)
//   z: in-thread, except the slab faces: each CTA PUSHES its two r face planes
//      into its z-neighbours' shared memory with `st.async ...
//      mbarrier::complete_tx` (DSMEM stores completing on the receiver's
//      mbarrier).
// Reduction: every warp shuffle-reduces its partials, warp 0 adds the warps'
// sums in a fixed order and its lanes 0..7 st.async the CTA's pair into slot
// [rank] of all 8 CTAs; each CTA waits on its own mbarrier and every thread
// adds the 8 pairs in the same fixed tree (broadcast loads, no shuffles), so
// all CTAs take identical CG decisions (deterministic, independent of brick
// scheduling and of which other bricks are solved).  The scalar recurrences
// use approximate reciprocals, 1/gamma and 1/alpha computed one iteration
// ahead, so only one MUFU.RCP sits on the critical path.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"
#include "rwb_ptx.cuh"

namespace cg = cooperative_groups;

namespace rwb {

constexpr int RB = 32;           // brick edge
constexpr int RQ = 4;            // x voxels per thread
constexpr int RQN = RB / RQ;     // quads per row
constexpr int RT = RQN * RB;     // threads per CTA z-group (one thread per row quad of a plane set)
constexpr int PLANE = RB * RB;   // floats per plane

// Decompositions of a 32^3 brick (RPZ z-planes per CTA, TZT z-planes per thread):
//   <4,4>: 8-CTA clusters, 256 threads x 16 voxels, 1 CTA per SM, double-buffered
//          staging (the next brick prefetched while iterating);
//   <4,2>: 8-CTA clusters, 512 threads x 8 voxels: twice the warps per SM to hide
//          the latency of each phase, the middle planes exchanged through smem;
//   <2,2>: 16-CTA clusters (non-portable size), 256 threads x 8 voxels, two CTAs
//          of DIFFERENT bricks per SM.
template <int RPZ_, int TZT_>
struct RCfg {
  static constexpr int RPZ = RPZ_;               // z planes per CTA
  static constexpr int TZT = TZT_;               // z planes per thread
  static constexpr int NZG = RPZ / TZT;          // thread z-groups per CTA
  static constexpr int RTT = RT * NZG;           // threads per CTA
  static constexpr int RW = RTT / 32;            // warps per CTA
  static constexpr int RCL = RB / RPZ;           // CTAs per cluster (per brick)
  static constexpr int RV = RQ * TZT;            // voxels per thread
  static constexpr int NPART = RCL;              // pushed partials per reduction (one per CTA)
  static constexpr int SLAB = RPZ * PLANE;
  static constexpr int MINB = RPZ == 2 ? 2 : 1;  // CTAs per SM
  static constexpr int NBUF = MINB == 1 ? 2 : 1; // staging buffers (2: next brick prefetched)
};

}  // namespace rwb

#ifdef RWB_TRACE
// phase timestamps of cluster 0 (diagnostics build only)
__device__ long long g_rwb_trace[8][64][8];
__device__ long long g_rwb_btrace[8][16][10];
__device__ unsigned long long g_rwb_end[64];  // %globaltimer at each cluster's last brick (launch 0 only)
#define TRACE(k)                                                                                      \
  do {                                                                                                \
    if (tid == 0 && blockIdx.x < 8 && rank < 8 && trace_it < 64) g_rwb_trace[rank][trace_it][k] = clock64(); \
  } while (0)
#define BTRACE(k)                                                                                      \
  do {                                                                                                 \
    if (tid == 0 && blockIdx.x < 8 && rank < 8 && btrace_n < 16) g_rwb_btrace[rank][btrace_n][k] = clock64(); \
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

template <int RPZ, int TZT>
struct ResidentSmem {
  using C = RCfg<RPZ, TZT>;
  float sx[C::NBUF][C::SLAB];              // staged scaled weights (double buffer: current / next brick)
  float sy[C::NBUF][C::SLAB];
  float sz[C::NBUF][PLANE + C::SLAB];      // z weights incl. the plane below the slab
  float sr[C::NBUF][C::SLAB];              // staged r0
  float sv[C::NBUF][C::SLAB];              // staged y0
  float4 rp[RPZ][RB][RQN];                 // r planes of this slab (y neighbours of the SpMV)
  float4 rface[2][2][RB][RQN];             // received faces [parity][0 = from below, 1 = from above]
  __align__(16) float red[2][2][C::NPART];  // pushed partials [parity][gamma, delta][rank]
  float2 wpart[C::RW];                      // this CTA's per-warp (gamma, delta) before the CTA sum
  unsigned long long barF[2];            // mbarriers: r faces from the z neighbours, per parity
  unsigned long long barR[2];            // mbarriers: dot-product partials, per parity
  unsigned long long barL[2];            // mbarriers: bulk staging, per buffer
  unsigned long long barS[2];            // mbarriers: Jacobi scales staged into sr[] for the epilogue
  unsigned long long barJ[2];            // mbarriers: the cluster's next brick index, per parity
  int jn[2];                             // ... pushed by rank 0 into every CTA
};

// Stage the slab of `slot` into buffer `buf` (one thread issues; completes on barL[buf]).
template <int RPZ, int TZT>
__device__ __forceinline__ void stage_slab(const ResidentArgs& a, ResidentSmem<RPZ, TZT>& sm, int buf, int slot,
                                           int rank) {
  constexpr int SLAB = RCfg<RPZ, TZT>::SLAB;
  const long long base = (long long)slot * (RB * RB * RB) + (long long)rank * SLAB;
  const uint32_t slab_bytes = SLAB * 4;
  const uint32_t zbytes = rank > 0 ? slab_bytes + PLANE * 4 : slab_bytes;
  mbar_expect_tx(&sm.barL[buf], 4 * slab_bytes + zbytes);
  bulk_g2s(sm.sx[buf], a.wx + base, slab_bytes, &sm.barL[buf]);
  bulk_g2s(sm.sy[buf], a.wy + base, slab_bytes, &sm.barL[buf]);
  if (rank > 0)
    bulk_g2s(sm.sz[buf], a.wz + base - PLANE, zbytes, &sm.barL[buf]);
  else
    bulk_g2s(sm.sz[buf] + PLANE, a.wz + base, zbytes, &sm.barL[buf]);
  bulk_g2s(sm.sr[buf], a.r0 + base, slab_bytes, &sm.barL[buf]);
  bulk_g2s(sm.sv[buf], a.y + base, slab_bytes, &sm.barL[buf]);
}

template <int RPZ, int TZT>
__global__ void __launch_bounds__(RCfg<RPZ, TZT>::RTT, RCfg<RPZ, TZT>::MINB) resident3d_kernel(ResidentArgs a) {
  using C = RCfg<RPZ, TZT>;
  constexpr int RCL = C::RCL, RV = C::RV, NPART = C::NPART, NBUF = C::NBUF, RTT = C::RTT, NZG = C::NZG;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ResidentSmem<RPZ, TZT>& sm = *reinterpret_cast<ResidentSmem<RPZ, TZT>*>(smem_raw);
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int zg = tid / RT;          // thread z-group: planes [zg*TZT, zg*TZT + TZT) of the slab
  const int ly = (tid % RT) / RQN;  // row
  const int xq = tid % RQN;         // quad within the row
  const int pz0 = zg * TZT;
  const bool below = rank > 0, above = rank < RCL - 1;
  const bool first_zg = zg == 0, last_zg = zg == NZG - 1;
  const int nfaces = (int)below + (int)above;
  const uint32_t face_bytes = (uint32_t)(RB * RQN * sizeof(float4));
  const uint32_t tx_faces = nfaces * face_bytes;
  const int cid = blockIdx.x / RCL, ncl = gridDim.x / RCL;
  const int n_act = *a.n_active;

  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.barF[i], 1);
      mbar_init(&sm.barR[i], 1);
      mbar_init(&sm.barL[i], 1);
      mbar_init(&sm.barS[i], 1);
      mbar_init(&sm.barJ[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (rank == 0)  // the CTA holding plane 0 has no plane below: zero it once
    for (int i = tid; i < PLANE; i += RTT)
#pragma unroll
      for (int b = 0; b < NBUF; ++b) sm.sz[b][i] = 0.f;
  // remote addresses this thread pushes to
  uint32_t face_dn_dst[2] = {0, 0}, face_up_dst[2] = {0, 0}, bar_dn[2] = {0, 0}, bar_up[2] = {0, 0};
  uint32_t red_dst[2] = {0, 0}, barR_dst[2] = {0, 0};
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    if (below && first_zg) {  // slab plane 0 goes to the CTA below, as its "from above" face
      face_dn_dst[par] = mapa_u32(smem_u32(&sm.rface[par][1][ly][xq]), rank - 1);
      bar_dn[par] = mapa_u32(smem_u32(&sm.barR[par]), rank - 1);
    }
    if (above && last_zg) {  // the last slab plane goes to the CTA above, as its "from below" face
      face_up_dst[par] = mapa_u32(smem_u32(&sm.rface[par][0][ly][xq]), rank + 1);
      bar_up[par] = mapa_u32(smem_u32(&sm.barR[par]), rank + 1);
    }
    if (warp == 0 && lane < RCL) {  // lane t of warp 0 delivers this CTA's partials to CTA t
      red_dst[par] = mapa_u32(smem_u32(&sm.red[par][0][rank]), lane);
      barR_dst[par] = mapa_u32(smem_u32(&sm.barR[par]), lane);
    }
  }
  cluster.sync();  // barriers initialised and the zero plane written before any remote access
  unsigned gk = 0;  // CG passes run by this cluster so far (drives the exchange-barrier parities)
  unsigned uses0 = 0, uses1 = 0;  // completed uses of each staging buffer (barL parities)
  unsigned usesS0 = 0, usesS1 = 0;  // ... and of the scale copies (barS parities)
#ifdef RWB_TRACE
  int btrace_n = 0;
#endif

  // Bricks are handed out dynamically: a cluster's first two bricks are static (cid, cid + ncl),
  // every further one comes from a global counter.  Rank 0 draws the brick after next at the start
  // of a brick, pushes the index into the cluster's CTAs once the brick's registers are loaded
  // (the atomic's latency is hidden behind the slab wait), and every CTA picks it up at the end of
  // the brick, so the next brick's slab is always staged while this one iterates.  The end of a
  // launch then idles at most about one brick's time instead of the spread of static shares.
  unsigned uJ = 0;
  int buf = 0;
  if (cid < n_act && tid == 0) stage_slab<RPZ, TZT>(a, sm, 0, a.alist[cid], rank);
  for (int j = cid, jn = cid + ncl, jnn; j < n_act; j = jn, jn = jnn, buf ^= (NBUF - 1)) {
    BTRACE(0);
    const int slot = a.alist[j];
    const bool draw = jn < n_act;  // cluster-uniform: once past the end, every later draw is too
    const int parJ = uJ & 1;
    int jd = 0;
    if (draw && tid == 0) {
      mbar_expect_tx(&sm.barJ[parJ], 4);
      if (rank == 0) jd = 2 * ncl + atomicAdd(a.next, 1);
    }
    if (NBUF == 2 && draw && tid == 0) stage_slab<RPZ, TZT>(a, sm, buf ^ 1, a.alist[jn], rank);
    if (buf) {
      mbar_wait(&sm.barL[1], uses1 & 1);
      ++uses1;
    } else {
      mbar_wait(&sm.barL[0], uses0 & 1);
      ++uses0;
    }
    BTRACE(1);

    // ---------------- registers from the staged slab ----------------
    float y[RV], r[RV], p[RV], sv[RV], w[RV];
    float wxf[RV], wyf[RV], wzf[RV], wyb[RV], wxb[TZT], wzb[RQ];
#pragma unroll
    for (int z = 0; z < TZT; ++z) {
      const int pz = pz0 + z;
      const int o = pz * PLANE + ly * RB + xq * RQ;
      const float4 fx = *reinterpret_cast<const float4*>(&sm.sx[buf][o]);
      const float4 fy = *reinterpret_cast<const float4*>(&sm.sy[buf][o]);
      const float4 fz = *reinterpret_cast<const float4*>(&sm.sz[buf][PLANE + o]);
      const float4 fyb = ly > 0 ? *reinterpret_cast<const float4*>(&sm.sy[buf][o - RB]) : f4(0, 0, 0, 0);
      const float4 fr = *reinterpret_cast<const float4*>(&sm.sr[buf][o]);
      const float4 fv = *reinterpret_cast<const float4*>(&sm.sv[buf][o]);
      wxb[z] = xq > 0 ? sm.sx[buf][o - 1] : 0.f;
      if (z == 0) {  // -z weights of the thread's first plane (sz[0] is the plane below the slab)
        const float4 fzb = *reinterpret_cast<const float4*>(&sm.sz[buf][o]);
#pragma unroll
        for (int i = 0; i < RQ; ++i) wzb[i] = lane_of(fzb, i);
      }
#pragma unroll
      for (int i = 0; i < RQ; ++i) {
        const int v = z * RQ + i;
        wxf[v] = lane_of(fx, i);
        wyf[v] = lane_of(fy, i);
        wzf[v] = lane_of(fz, i);
        wyb[v] = lane_of(fyb, i);
        r[v] = lane_of(fr, i);
        y[v] = lane_of(fv, i);
        p[v] = 0.f;
        sv[v] = 0.f;
        w[v] = 0.f;
      }
    }
    const float thresh = (float)((double)a.tol2 * a.bb[slot]);
    if (draw && rank == 0 && tid == 0) {
#pragma unroll 1
      for (int c = 0; c < RCL; ++c)
        st_async_f32(mapa_u32(smem_u32(&sm.jn[parJ]), c), __int_as_float(jd), mapa_u32(smem_u32(&sm.barJ[parJ]), c));
    }
    BTRACE(2);

    // ---------------- CG (Chronopoulos-Gear) ----------------
    // One cluster-wide exchange per iteration: right after the SpMV w = A'r each
    // CTA pushes its dot partials AND its two face planes of w.  A CTA keeps its
    // own copies of the neighbours' face values of r and s (r0 exchanged once per
    // brick) and advances them with the same fmaf as their owner,
    //   s_face <- w_face + beta s_face,   r_face <- r_face - alpha s_face,
    // so they stay bit-identical and the next SpMV needs no second exchange.
    // (Pushing r faces as well would double the DSMEM volume, which at ~20 B/cycle
    // per SM is what bounds the exchange.)
    float gamma = 0.f, alpha = 0.f, rgamma = 0.f, ralpha = 0.f;
    int state = ST_ACTIVE, it = 0;
    float4 rf_dn = f4(0, 0, 0, 0), rf_up = f4(0, 0, 0, 0);  // neighbours' r at my faces
    float4 sf_dn = f4(0, 0, 0, 0), sf_up = f4(0, 0, 0, 0);  // ... and their s
    const float4 z4 = f4(0, 0, 0, 0);
    auto plane4 = [&](const float* v, int z) { return f4(v[z * RQ], v[z * RQ + 1], v[z * RQ + 2], v[z * RQ + 3]); };
    // publish r0: planes for the y / cross-group z neighbours, faces through a one-time exchange
#pragma unroll
    for (int z = 0; z < TZT; ++z) sm.rp[pz0 + z][ly][xq] = plane4(r, z);
    {
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
      if (tid == 0) mbar_expect_tx(&sm.barR[par], tx_faces + 2 * NPART * 4);
      if (below && first_zg) st_async_v4(par ? face_dn_dst[1] : face_dn_dst[0], plane4(r, 0), par ? bar_dn[1] : bar_dn[0]);
      if (above && last_zg)
        st_async_v4(par ? face_up_dst[1] : face_up_dst[0], plane4(r, TZT - 1), par ? bar_up[1] : bar_up[0]);
      // complete the phase's partial slots with zeros (this exchange carries no dot products)
      if (warp == 0 && lane < RCL) {
        const uint32_t dst = par ? red_dst[1] : red_dst[0], bar = par ? barR_dst[1] : barR_dst[0];
        st_async_f32(dst, 0.f, bar);
        st_async_f32(dst + NPART * 4, 0.f, bar);
      }
      mbar_wait(&sm.barR[par], ph);
      ++gk;
      if (first_zg && below) rf_dn = sm.rface[par][0][ly][xq];
      if (last_zg && above) rf_up = sm.rface[par][1][ly][xq];
      __syncthreads();  // own r planes published; every thread has left the staged slab
    }
    // the staged r0 is in registers: fetch the slab's Jacobi scales into its place
    // while the brick iterates (the epilogue at the end needs them)
    if (tid == 0) {
      const long long base = (long long)slot * (RB * RB * RB) + (long long)rank * C::SLAB;
      mbar_expect_tx(&sm.barS[buf], C::SLAB * 4);
      bulk_g2s(sm.sr[buf], a.sc + base, C::SLAB * 4, &sm.barS[buf]);
    }
#ifdef RWB_TRACE
    int trace_it = (int)gk;
#endif
    for (int pass = 0;; ++pass) {
      TRACE(0);
      const int par = gk & 1;
      const uint32_t ph = (gk >> 1) & 1;
#ifdef RWB_NOFACE  // diagnostics only: time an iteration without the face traffic (wrong results)
      if (tid == 0) mbar_expect_tx(&sm.barR[par], 2 * NPART * 4);
#else
      if (tid == 0) mbar_expect_tx(&sm.barR[par], tx_faces + 2 * NPART * 4);
#endif
      // w = A'r
      float gp[TZT][2], dp[TZT][2];  // dot partials per plane, per x-pair lane
#pragma unroll
      for (int z = 0; z < TZT; ++z) gp[z][0] = gp[z][1] = dp[z][0] = dp[z][1] = 0.f;
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const int pz = pz0 + z;
        const float4 ru = ly + 1 < RB ? sm.rp[pz][ly + 1][xq] : z4;
        const float4 rd = ly > 0 ? sm.rp[pz][ly - 1][xq] : z4;
        const float4 rzu = z + 1 < TZT ? plane4(r, z + 1) : (pz + 1 < RPZ ? sm.rp[pz + 1][ly][xq] : rf_up);
        const float4 rzd = z > 0 ? plane4(r, z - 1) : (pz > 0 ? sm.rp[pz - 1][ly][xq] : rf_dn);
        const float rl = __shfl_up_sync(0xffffffffu, r[z * RQ + RQ - 1], 1);
        const float rr_ = __shfl_down_sync(0xffffffffu, r[z * RQ], 1);
        // y / z terms on x-pairs (FFMA2), then the x terms per voxel
        float acc[RQ];
#pragma unroll
        for (int i = 0; i < RQ; i += 2) {
          const int v = z * RQ + i;
          const float wzl0 = z > 0 ? wzf[v - RQ] : wzb[i], wzl1 = z > 0 ? wzf[v + 1 - RQ] : wzb[i + 1];
          fma2(acc[i], acc[i + 1], wyf[v], wyf[v + 1], lane_of(ru, i), lane_of(ru, i + 1), 0.f, 0.f);
          fma2(acc[i], acc[i + 1], wyb[v], wyb[v + 1], lane_of(rd, i), lane_of(rd, i + 1), acc[i], acc[i + 1]);
          fma2(acc[i], acc[i + 1], wzf[v], wzf[v + 1], lane_of(rzu, i), lane_of(rzu, i + 1), acc[i], acc[i + 1]);
          fma2(acc[i], acc[i + 1], wzl0, wzl1, lane_of(rzd, i), lane_of(rzd, i + 1), acc[i], acc[i + 1]);
        }
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const int v = z * RQ + i;
          const float rxl = i > 0 ? r[v - 1] : rl;
          const float rxr = i < RQ - 1 ? r[v + 1] : rr_;
          const float wxl = i > 0 ? wxf[v - 1] : wxb[z];
          acc[i] = fmaf(wxf[v], rxr, acc[i]);
          acc[i] = fmaf(wxl, rxl, acc[i]);
        }
#pragma unroll
        for (int i = 0; i < RQ; i += 2) {
          const int v = z * RQ + i;
          fma2(w[v], w[v + 1], -1.f, -1.f, acc[i], acc[i + 1], r[v], r[v + 1]);  // w = r - acc (exact product)
          fma2(gp[z][0], gp[z][1], r[v], r[v + 1], r[v], r[v + 1], gp[z][0], gp[z][1]);
          fma2(dp[z][0], dp[z][1], w[v], w[v + 1], r[v], r[v + 1], dp[z][0], dp[z][1]);
        }
      }
      TRACE(1);
      // push the faces of w, then the dot partials, all onto the peers' barR[par]
      #ifndef RWB_NOFACE
      if (below && first_zg)
        st_async_v4(par ? face_dn_dst[1] : face_dn_dst[0], plane4(w, 0), par ? bar_dn[1] : bar_dn[0]);
      if (above && last_zg)
        st_async_v4(par ? face_up_dst[1] : face_up_dst[0], plane4(w, TZT - 1), par ? bar_up[1] : bar_up[0]);
#endif
      {
        float gs = 0.f, ds = 0.f;
#pragma unroll
        for (int z = 0; z < TZT; ++z) {
          gs += gp[z][0] + gp[z][1];
          ds += dp[z][0] + dp[z][1];
        }
        // warp sums -> CTA sum (fixed order) -> one st.async pair per CTA into every CTA
        const float gw = warp_sum(gs);
        const float dw = warp_sum(ds);
        if (lane == 0) sm.wpart[warp] = make_float2(gw, dw);
        asm volatile("bar.sync 1, %0;" ::"n"(RTT) : "memory");
        if (warp == 0) {
          float gc = 0.f, dc = 0.f;
#pragma unroll
          for (int wv = 0; wv < C::RW; ++wv) {
            const float2 v = sm.wpart[wv];
            gc += v.x;
            dc += v.y;
          }
          if (lane < RCL) {
            const uint32_t dst = par ? red_dst[1] : red_dst[0], bar = par ? barR_dst[1] : barR_dst[0];
            st_async_f32(dst, gc, bar);
            st_async_f32(dst + NPART * 4, dc, bar);
          }
        }
      }
      TRACE(2);
      mbar_wait(&sm.barR[par], ph);
      TRACE(3);
      ++gk;
      const float g_new = sum_parts<NPART>(sm.red[par][0]);
      const float delta = sum_parts<NPART>(sm.red[par][1]);
      float beta;
      if (pass == 0) {
        // the setup already settled zero-rhs and converged-at-start bricks
        beta = 0.f;
        alpha = delta != 0.f ? g_new * rcp_ftz(delta) : 0.f;
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
        // fast reciprocals, 1/gamma and 1/alpha taken off the critical path in the
        // previous iteration: the scalars only need to be identical in every CTA
        beta = g_new * rgamma;
        const float den = delta - beta * (g_new * ralpha);
        alpha = den != 0.f ? g_new * rcp_ftz(den) : 0.f;
      }
      gamma = g_new;
      rgamma = rcp_ftz(g_new);
      ralpha = rcp_ftz(alpha);
      TRACE(4);
      // update k: p = r + beta p, s = w + beta s, y += alpha p, r -= alpha s (and the neighbour faces)
#pragma unroll
      for (int v = 0; v < RV; v += 2) {  // packed pairs: the same fmaf, two per FFMA2
        fma2(p[v], p[v + 1], beta, beta, p[v], p[v + 1], r[v], r[v + 1]);
        fma2(sv[v], sv[v + 1], beta, beta, sv[v], sv[v + 1], w[v], w[v + 1]);
        fma2(y[v], y[v + 1], alpha, alpha, p[v], p[v + 1], y[v], y[v + 1]);
        fma2(r[v], r[v + 1], -alpha, -alpha, sv[v], sv[v + 1], r[v], r[v + 1]);
      }
      ++it;
      if (first_zg && below) {
        const float4 wn = sm.rface[par][0][ly][xq];
        sf_dn = f4(fmaf(beta, sf_dn.x, wn.x), fmaf(beta, sf_dn.y, wn.y), fmaf(beta, sf_dn.z, wn.z), fmaf(beta, sf_dn.w, wn.w));
        rf_dn = f4(fmaf(-alpha, sf_dn.x, rf_dn.x), fmaf(-alpha, sf_dn.y, rf_dn.y), fmaf(-alpha, sf_dn.z, rf_dn.z),
                   fmaf(-alpha, sf_dn.w, rf_dn.w));
      }
      if (last_zg && above) {
        const float4 wn = sm.rface[par][1][ly][xq];
        sf_up = f4(fmaf(beta, sf_up.x, wn.x), fmaf(beta, sf_up.y, wn.y), fmaf(beta, sf_up.z, wn.z), fmaf(beta, sf_up.w, wn.w));
        rf_up = f4(fmaf(-alpha, sf_up.x, rf_up.x), fmaf(-alpha, sf_up.y, rf_up.y), fmaf(-alpha, sf_up.z, rf_up.z),
                   fmaf(-alpha, sf_up.w, rf_up.w));
      }
      // publish the new r planes (previous readers finished before the wait: their
      // partials were part of it)
#pragma unroll
      for (int z = 0; z < TZT; ++z) sm.rp[pz0 + z][ly][xq] = plane4(r, z);
      __syncthreads();
      TRACE(5);
      TRACE(6);
#ifdef RWB_TRACE
      ++trace_it;
#endif
    }
    BTRACE(6);
    // ---------------- epilogue: probabilities and labels straight into the level ----------------
    {
      if (buf) {
        mbar_wait(&sm.barS[1], usesS1 & 1);
        ++usesS1;
      } else {
        mbar_wait(&sm.barS[0], usesS0 & 1);
        ++usesS0;
      }
      const int brick = a.list ? a.list[slot] : slot;
      const int hx = brick % a.gx, hy = (brick / a.gx) % a.gy, hz = brick / (a.gx * a.gy);
      const int gy = a.oy + hy * RB + ly, gx0 = a.ox + hx * RB + xq * RQ;
      const bool row_in = gy >= 0 && gy < a.ny;
      const bool quad_in = gx0 >= 0 && gx0 + RQ <= a.nx;
#pragma unroll
      for (int z = 0; z < TZT; ++z) {
        const int gz = a.oz + hz * RB + rank * RPZ + pz0 + z;
        if (!row_in || gz < 0 || gz >= a.nz) continue;
        const float4 s4 = *reinterpret_cast<const float4*>(&sm.sr[buf][(pz0 + z) * PLANE + ly * RB + xq * RQ]);
        float pv[RQ];
#pragma unroll
        for (int i = 0; i < RQ; ++i) {
          const float s = lane_of(s4, i), yv = y[z * RQ + i];
          pv[i] = s > 0.f ? s * yv : yv;
        }
        const long long gi = ((long long)gz * a.ny + gy) * a.nx + gx0;
        if (quad_in && (gi & 3) == 0) {
          *reinterpret_cast<float4*>(a.prob + gi) = f4(pv[0], pv[1], pv[2], pv[3]);
          if (a.labels)
            *reinterpret_cast<uchar4*>(a.labels + gi) =
                make_uchar4(pv[0] > 0.5f, pv[1] > 0.5f, pv[2] > 0.5f, pv[3] > 0.5f);
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
    // the staging buffer just read is refilled for a later brick: every thread
    // must be past its register loads first
    __syncthreads();
    if (NBUF == 1 && draw && tid == 0) stage_slab<RPZ, TZT>(a, sm, 0, a.alist[jn], rank);
    jnn = n_act;
    if (draw) {
      mbar_wait(&sm.barJ[parJ], (uJ >> 1) & 1);
      jnn = sm.jn[parJ];
      ++uJ;
    }
    BTRACE(7);
    BTRACE(8);
#ifdef RWB_TRACE
    ++btrace_n;
#endif
  }
#ifdef RWB_TRACE
  if (rank == 0 && tid == 0 && cid < 64) {
    unsigned long long tnow;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
    g_rwb_end[cid] = tnow;
  }
#endif
}

#ifdef RWB_TRACE
extern "C" int rwb_trace_dump(long long* out) {  // 8*64*8 int64
  return (int)cudaMemcpyFromSymbol(out, g_rwb_trace, sizeof(g_rwb_trace));
}
extern "C" int rwb_end_dump(unsigned long long* out) {  // 64 uint64
  return (int)cudaMemcpyFromSymbol(out, g_rwb_end, sizeof(g_rwb_end));
}
extern "C" int rwb_btrace_dump(long long* out) {  // 8*16*10 int64
  return (int)cudaMemcpyFromSymbol(out, g_rwb_btrace, sizeof(g_rwb_btrace));
}
#endif

int resident3d_supported(const Geo& g) { return g.is3d && g.bz == RB && g.by == RB && g.bx == RB; }

template <int RPZ, int TZT>
static int launch_resident(const ResidentArgs& a, int max_bricks, cudaStream_t st) {
  using C = RCfg<RPZ, TZT>;
  static DeviceCache cache;
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int clusters = cache[dev].load(std::memory_order_relaxed);
  auto kern = resident3d_kernel<RPZ, TZT>;
  const int smem = (int)sizeof(ResidentSmem<RPZ, TZT>);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C::RCL;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.blockDim = dim3(C::RTT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  if (!clusters) {
    RWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (C::RCL > 8) RWB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cfg.gridDim = dim3(C::RCL * 1024, 1, 1);
    int n = 0;
    RWB_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
    if (n <= 0) return fail(RWB_ERR_UNSUPPORTED, "no brick cluster fits on this device");
    clusters = n;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  const int grid_clusters = clusters < max_bricks ? clusters : max_bricks;
  if (grid_clusters <= 0) return RWB_OK;
  cfg.gridDim = dim3(grid_clusters * C::RCL, 1, 1);
  RWB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  count_launches(1);
  return RWB_OK;
}

int launch_resident3d(const ResidentArgs& a, int max_bricks, int variant, cudaStream_t st) {
  switch (variant) {
    case 4: return launch_resident3d_q4(a, max_bricks, st);
    case 16: return launch_resident<2, 2>(a, max_bricks, st);
    case 512: return launch_resident<4, 2>(a, max_bricks, st);
    default: return launch_resident<4, 4>(a, max_bricks, st);
  }
}

}  // namespace rwb
