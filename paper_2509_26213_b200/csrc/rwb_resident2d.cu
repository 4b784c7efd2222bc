// Tile-resident Jacobi-PCG engine for 2-D levels with 64^2 bricks (config 3):
// one CTA per tile, every CG iteration on chip.
//
// A 64 x 64 tile's whole CG state — y, r, p, s, w and the scaled forward
// weights, ~8 floats per pixel = 128 KiB — fits in ONE SM's register file, so
// unlike the 3-D engine (rwb_resident.cu, 8-CTA clusters, DSMEM exchange) a
// tile needs no cluster: 256 threads, each a 4(x) x 4(y) block of pixels.
// Neighbours: x by warp shuffles (a half-warp is one 64-pixel row band), y
// through the tile's r published in shared memory.  The iteration is the same
// Chronopoulos-Gear single-reduction CG as the 3-D engine (w = A'r and s = A'p
// carried), with the two dot products reduced CTA-wide in a fixed order
// (warp shuffle tree, 8 warp sums added in sequence): deterministic and
// independent of which other tiles are solved.
//
// Inputs are the brick-local system the setup kernels build (slot-major, tile
// contiguous, x fastest): scaled weights w'x, w'y, r0, y0 (y0 holds the final
// value of every non-unknown), and the Jacobi scales s; per tile 20 B/pixel
// in, and the probabilities (4 B) and labels (1 B) out, straight into the
// level — HBM traffic per pixel per SOLVE, where the streaming solver moves
// 48 B per pixel per ITERATION.
#include <cuda_runtime.h>

#include <cstdlib>

#include "rwb_common.cuh"
#include "rwb_resident.cuh"

namespace rwb {

constexpr int T2 = 64;            // tile edge
constexpr int Q2 = 4;             // pixels per thread along x and along y
constexpr int QN2 = T2 / Q2;      // thread quads per row / per column (16)
constexpr int TH2 = QN2 * QN2;    // threads per CTA (256)
constexpr int NW2 = TH2 / 32;     // warps
constexpr int PV2 = Q2 * Q2;      // pixels per thread

struct Resident2dSmem {
  float4 rp[T2][QN2];   // the tile's r (y neighbours of the SpMV)
  float4 wpart[2][NW2];  // per-warp (r.r, delta, r.u), double-buffered by iteration parity
  // coarse correction: 8 x 8 aggregates of 8 x 8 pixels (2 x 2 thread quads), index ay * 8 + ax
  float aggw[64], aggr[64];  // this iteration's P^T w, P^T r (P^T r0, d at the tile's start)
  float cc[64];              // c per aggregate
  float cps[64], cdi[64];    // P^T s, 1 / d
};
constexpr int NA2 = 8;           // aggregates per tile row / column
// omega 0.5 (the 3-D engine uses 0.8): tools/tile_cc_model.py, float64, stop at tol 1e-6 — on the
// random tiles of test_resident2d_tiles_match_oracle the max error vs the exact solution is 1.2e-4
// at 0.8 and 7.2e-5 at 0.5 (Jacobi-PCG: 7.9e-5), iterations x0.83 at both; on phantom tiles x0.53
// (0.8) and x0.57 (0.5)
constexpr float kCc2Omega = 0.5f;

__device__ __forceinline__ float q4l(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ float rcp_ftz2(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// CC: Jacobi + additive coarse correction M = I + w P D_c^-1 P^T on the tile's 8 x 8 aggregates
// (the 3-D engine's, csrc/rwb_resident4.cu header, CTA-local here: each aggregate's 4 threads share
// a warp, so its sums are two shuffles and one shared-memory store)
template <bool CC>
__global__ void __launch_bounds__(TH2, 1) resident2d_kernel(ResidentArgs a) {
  __shared__ Resident2dSmem sm;
  const int tid = threadIdx.x;
  const int xq = tid % QN2, yq = tid / QN2;  // lanes 0..15 / 16..31 of a warp: two row bands
  const int lane = tid & 31, warp = tid >> 5;
  const int n_act = *a.n_active;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const int tile_vox = T2 * T2;
  const int ax = xq >> 1, ay = yq >> 1, agg = ay * NA2 + ax;
  const int agg_x = (xq & 1) ? (ax < NA2 - 1 ? agg + 1 : agg) : (ax > 0 ? agg - 1 : agg);
  const int agg_y = (yq & 1) ? (ay < NA2 - 1 ? agg + NA2 : agg) : (ay > 0 ? agg - NA2 : agg);
  // the 4 threads of an aggregate: lanes xq, xq^1 of both quad rows of the warp
  auto agg_sum = [&](float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
  };
  const bool agg_lead = (lane & 17) == 0;

  for (int j = blockIdx.x; j < n_act; j += gridDim.x) {
    const int slot = a.alist[j];
    const long long base = (long long)slot * tile_vox;
    // ---- registers from the brick-local system (coalesced 16 B loads) ----
    float y[PV2], r[PV2], p[PV2], sv[PV2], w[PV2], wxf[PV2], wyf[PV2], wxb[Q2], wyb[Q2];
#pragma unroll
    for (int i = 0; i < Q2; ++i) {
      const long long o = base + (long long)(Q2 * yq + i) * T2 + Q2 * xq;
      const float4 fx = __ldg(reinterpret_cast<const float4*>(a.wx + o));
      const float4 fy = __ldg(reinterpret_cast<const float4*>(a.wy + o));
      const float4 fr = __ldg(reinterpret_cast<const float4*>(a.r0 + o));
      const float4 fv = __ldg(reinterpret_cast<const float4*>(a.y + o));
      wxb[i] = xq > 0 ? __ldg(a.wx + o - 1) : 0.f;
#pragma unroll
      for (int k = 0; k < Q2; ++k) {
        const int v = i * Q2 + k;
        wxf[v] = q4l(fx, k);
        wyf[v] = q4l(fy, k);
        r[v] = q4l(fr, k);
        y[v] = q4l(fv, k);
        p[v] = sv[v] = w[v] = 0.f;
      }
    }
    {
      const float4 fyb = yq > 0 ? __ldg(reinterpret_cast<const float4*>(a.wy + base + (long long)(Q2 * yq - 1) * T2 +
                                                                        Q2 * xq))
                                : z4;
#pragma unroll
      for (int k = 0; k < Q2; ++k) wyb[k] = q4l(fyb, k);
    }
    const float thresh = (float)((double)a.tol2 * a.bb[slot]);
    // coarse correction: tau = m - sigma per pixel, the aggregate diagonals and P^T r0
    float tau[CC ? PV2 : 1];
    if (CC) {
      float dpart = 0.f, gpart = 0.f;
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(a.sc + base + (long long)(Q2 * yq + i) * T2 + Q2 * xq));
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const int v = i * Q2 + k;
          const float wxl = k > 0 ? wxf[v - 1] : wxb[i];
          const float wyl = i > 0 ? wyf[v - Q2] : wyb[k];
          const float t = (q4l(s4, k) > 0.f ? 1.f : 0.f) - ((wxf[v] + wxl) + (wyf[v] + wyl));
          tau[v] = t;
          dpart += t;
          gpart += r[v];
          if (i == 0 && !(yq & 1)) dpart += wyl;            // edges leaving the aggregate
          if (i == Q2 - 1 && (yq & 1)) dpart += wyf[v];
          if (k == 0 && !(xq & 1)) dpart += wxl;
          if (k == Q2 - 1 && (xq & 1)) dpart += wxf[v];
        }
      }
      const float dv = agg_sum(dpart), gv = agg_sum(gpart);
      if (agg_lead) {
        sm.cdi[agg] = dv > 1e-6f ? 1.f / dv : 0.f;
        sm.aggr[agg] = gv;
        sm.cps[agg] = 0.f;
      }
      __syncthreads();
      if (tid < 64) sm.cc[tid] = kCc2Omega * sm.aggr[tid] * sm.cdi[tid];
    }
    auto publish = [&]() {
#pragma unroll
      for (int i = 0; i < Q2; ++i)
        sm.rp[Q2 * yq + i][xq] = make_float4(r[i * Q2], r[i * Q2 + 1], r[i * Q2 + 2], r[i * Q2 + 3]);
    };
    publish();
    __syncthreads();

    float alpha = 0.f, rgamma = 0.f, ralpha = 0.f;  // 1/gamma, 1/alpha one iteration ahead
    int state = ST_ACTIVE, it = 0;
    for (int pass = 0;; ++pass) {
      // ---- w = A'u (u = r + c of the pixel's aggregate), partial dots ----
      const float4 rd = yq > 0 ? sm.rp[Q2 * yq - 1][xq] : z4;
      const float4 ru = yq + 1 < QN2 ? sm.rp[Q2 * yq + Q2][xq] : z4;
      float gs = 0.f, ds = 0.f, rs = 0.f, ws = 0.f;
      float c_own = 0.f, dxc = 0.f, dyc = 0.f;
      if (CC) {
        c_own = sm.cc[agg];
        dxc = sm.cc[agg_x] - c_own;
        dyc = sm.cc[agg_y] - c_own;
      }
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const float rl = __shfl_up_sync(0xffffffffu, r[i * Q2 + Q2 - 1], 1);
        const float rr_ = __shfl_down_sync(0xffffffffu, r[i * Q2], 1);
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const int v = i * Q2 + k;
          const float rxl = k > 0 ? r[v - 1] : rl;
          const float rxr = k < Q2 - 1 ? r[v + 1] : rr_;
          const float wxl = k > 0 ? wxf[v - 1] : wxb[i];
          const float ryd = i > 0 ? r[v - Q2] : q4l(rd, k);
          const float ryu = i < Q2 - 1 ? r[v + Q2] : q4l(ru, k);
          const float wyl = i > 0 ? wyf[v - Q2] : wyb[k];
          float acc = wyf[v] * ryu;
          acc = fmaf(wyl, ryd, acc);
          acc = fmaf(wxf[v], rxr, acc);
          acc = fmaf(wxl, rxl, acc);
          w[v] = r[v] - acc;
          if (CC) {  // + c_own tau - the aggregate-face differences
            float kk = c_own * tau[v];
            if (i == 0 && !(yq & 1)) kk = fmaf(-wyl, dyc, kk);
            if (i == Q2 - 1 && (yq & 1)) kk = fmaf(-wyf[v], dyc, kk);
            if (k == 0 && !(xq & 1)) kk = fmaf(-wxl, dxc, kk);
            if (k == Q2 - 1 && (xq & 1)) kk = fmaf(-wxf[v], dxc, kk);
            w[v] += kk;
          }
          gs = fmaf(r[v], r[v], gs);
          ds = fmaf(w[v], r[v], ds);
          if (CC) {
            rs += r[v];
            ws += w[v];
          }
        }
      }
      // ---- CTA reduction (fixed order); CC: gamma = r.u = r.r + c P^T r, delta = w.u = w.r + c P^T w ----
      float us = gs;
      if (CC) {
        const float pr = agg_sum(rs), pw = agg_sum(ws);
        if (agg_lead) {
          sm.aggr[agg] = pr;
          sm.aggw[agg] = pw;
        }
        us = fmaf(c_own, rs, gs);
        ds = fmaf(c_own, ws, ds);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gs += __shfl_xor_sync(0xffffffffu, gs, o);
        ds += __shfl_xor_sync(0xffffffffu, ds, o);
        if (CC) us += __shfl_xor_sync(0xffffffffu, us, o);
      }
      const int par = pass & 1;
      if (lane == 0) sm.wpart[par][warp] = make_float4(gs, ds, us, 0.f);
      __syncthreads();  // partials visible; every thread has read rp and cc (its SpMV is done)
      float rr = 0.f, delta = 0.f, g_new = 0.f;
#pragma unroll
      for (int wv = 0; wv < NW2; ++wv) {
        const float4 v = sm.wpart[par][wv];
        rr += v.x;
        delta += v.y;
        g_new += v.z;
      }
      if (!CC) g_new = rr;
      float beta;
      if (pass == 0) {
        beta = 0.f;
        alpha = delta != 0.f ? g_new * rcp_ftz2(delta) : 0.f;
        if (a.max_iter <= 0) {
          state = ST_MAXITER;
          break;
        }
      } else {
        if (rr <= thresh) {
          state = ST_CONVERGED;
          break;
        }
        if (it >= a.max_iter) {
          state = ST_MAXITER;
          break;
        }
        beta = g_new * rgamma;
        const float den = delta - beta * (g_new * ralpha);
        alpha = den != 0.f ? g_new * rcp_ftz2(den) : 0.f;
      }
      rgamma = rcp_ftz2(g_new);
      ralpha = rcp_ftz2(alpha);
      // ---- update: p = u + beta p, s = w + beta s, y += alpha p, r -= alpha s ----
      if (CC && tid < 64) {  // the next c from P^T r' = P^T r - alpha (P^T w + beta P^T s)
        const float ps = fmaf(beta, sm.cps[tid], sm.aggw[tid]);
        sm.cps[tid] = ps;
        sm.cc[tid] = kCc2Omega * fmaf(-alpha, ps, sm.aggr[tid]) * sm.cdi[tid];
      }
#pragma unroll
      for (int v = 0; v < PV2; ++v) {
        p[v] = fmaf(beta, p[v], CC ? r[v] + c_own : r[v]);  // u off the unknowns is harmless: y0 is
                                                            // restored there in the epilogue
        sv[v] = fmaf(beta, sv[v], w[v]);
        y[v] = fmaf(alpha, p[v], y[v]);
        r[v] = fmaf(-alpha, sv[v], r[v]);
      }
      ++it;
      publish();  // the barrier above proved every reader of the previous r has finished
      __syncthreads();
    }
    // ---- epilogue: probabilities and labels straight into the level ----
    {
      const int brick = a.list ? a.list[slot] : slot;
      const int hx = brick % a.gx, hy = brick / a.gx;
      const int gx0 = a.ox + hx * T2 + Q2 * xq;
      const bool quad_in = gx0 >= 0 && gx0 + Q2 <= a.nx;
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const int gy = a.oy + hy * T2 + Q2 * yq + i;
        if (gy < 0 || gy >= a.ny) continue;
        const long long o = base + (long long)(Q2 * yq + i) * T2 + Q2 * xq;
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(a.sc + o));
        const float4 y0 = CC ? __ldg(reinterpret_cast<const float4*>(a.y + o)) : z4;
        float pv[Q2];
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const float s = q4l(s4, k), yv = CC && !(s > 0.f) ? q4l(y0, k) : y[i * Q2 + k];
          pv[k] = s > 0.f ? s * yv : yv;
        }
        const long long gi = (long long)gy * a.nx + gx0;
        if (quad_in && (gi & 3) == 0) {
          *reinterpret_cast<float4*>(a.prob + gi) = make_float4(pv[0], pv[1], pv[2], pv[3]);
          if (a.labels)
            *reinterpret_cast<uchar4*>(a.labels + gi) =
                make_uchar4(pv[0] > 0.5f, pv[1] > 0.5f, pv[2] > 0.5f, pv[3] > 0.5f);
        } else {
#pragma unroll
          for (int k = 0; k < Q2; ++k) {
            if (gx0 + k < 0 || gx0 + k >= a.nx) continue;
            a.prob[gi + k] = pv[k];
            if (a.labels) a.labels[gi + k] = pv[k] > 0.5f ? 1 : 0;
          }
        }
      }
    }
    if (tid == 0) {
      a.state[slot] = state;
      a.iters[slot] = it;
    }
    __syncthreads();  // sm.rp is rewritten by the next tile
  }
}

int resident2d_supported(const Geo& g) { return !g.is3d && g.by == T2 && g.bx == T2; }

int launch_resident2d(const ResidentArgs& a, int max_bricks, cudaStream_t st) {
  static DeviceCache cache[2];
  static const bool cc_off = [] {
    const char* e = std::getenv("RWB_R2_CC");
    return e && e[0] == '0';
  }();
  const bool cc = a.coarse && !cc_off;
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int grid = cache[cc][dev].load(std::memory_order_relaxed);
  if (!grid) {
    int sms = 0, per = 0;
    RWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, cc ? resident2d_kernel<true> : resident2d_kernel<false>,
                                                           TH2, 0));
    if (per <= 0) return fail(RWB_ERR_UNSUPPORTED, "2-D tile engine does not fit on this device");
    grid = sms * per;
    cache[cc][dev].store(grid, std::memory_order_relaxed);
  }
  const int g = grid < max_bricks ? grid : max_bricks;
  if (g <= 0) return RWB_OK;
  if (cc)
    resident2d_kernel<true><<<g, TH2, 0, st>>>(a);
  else
    resident2d_kernel<false><<<g, TH2, 0, st>>>(a);
  RWB_LAUNCH_CHECK("resident2d_kernel");
  count_launches(1);
  return RWB_OK;
}

}  // namespace rwb
