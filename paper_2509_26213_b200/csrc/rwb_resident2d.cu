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
#include "rwb_ptx.cuh"
#include "rwb_resident.cuh"

namespace rwb {

constexpr int T2 = 64;            // tile edge
constexpr int Q2 = 4;             // pixels per thread along x and along y
constexpr int QN2 = T2 / Q2;      // thread quads per row / per column (16)
constexpr int TH2 = QN2 * QN2;    // threads per CTA (256)
constexpr int NW2 = TH2 / 32;     // warps
constexpr int PV2 = Q2 * Q2;      // pixels per thread

struct Resident2dSmem {
  float4 rp[T2][QN2];    // the tile's r (Jacobi) or u = M r (CC): the y neighbours of the SpMV
  float4 wpart[2][NW2];  // per-warp (r.r, w.u, r.u), double-buffered by iteration parity
};
constexpr int NA2 = 8;  // aggregates per tile row / column
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

// CC: PCG with M = I + w P D_c^-1 P^T on the tile's 8 x 8 aggregates of 8 x 8 pixels (one damped
// Jacobi sweep of the Galerkin coarse system, the 3-D engine's correction, csrc/rwb_resident4.cu).
// An aggregate is 2 x 2 thread quads inside one warp, so P^T r is a 2-shuffle warp sum and every
// thread forms its own aggregate's c = w (P^T r) / d: u = M r is explicit (u = r + c on the
// unknowns, 0 elsewhere), the SpMV runs on u (w = A'u) and publishes u instead of r, and the
// iteration is plain Chronopoulos-Gear PCG (gamma = r.u, delta = w.u; r.r drives the stop rule) —
// no coarse state in shared memory, no extra barrier.
template <bool CC>
__global__ void __launch_bounds__(TH2, 1) resident2d_kernel(ResidentArgs a) {
  __shared__ Resident2dSmem sm;
  const int tid = threadIdx.x;
  const int xq = tid % QN2, yq = tid / QN2;  // lanes 0..15 / 16..31 of a warp: two row bands
  const int lane = tid & 31, warp = tid >> 5;
  const int n_act = *a.n_active;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const int tile_vox = T2 * T2;
  // the 4 threads of an aggregate: lanes xq, xq^1 of the warp's two quad rows (fixed order)
  auto agg_sum = [&](float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    return v;
  };

  for (int j = blockIdx.x; j < n_act; j += gridDim.x) {
    const int slot = a.alist[j];
    const long long base = (long long)slot * tile_vox;
    // ---- registers from the brick-local system (coalesced 16 B loads) ----
    float y[PV2], r[PV2], p[PV2], sv[PV2], w[PV2], wxf[PV2], wyf[PV2], wxb[Q2], wyb[Q2];
    float u[CC ? PV2 : 1];
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
    // coarse correction: the unknown mask, the aggregate's Galerkin diagonal d = sum over its
    // pixels of (m - sigma) + the weights leaving it, and u0
    unsigned mbits = 0;
    float cw = 0.f;  // w / d of the thread's aggregate
    auto form_u = [&]() {
      float rs4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) rs4[k] = (r[k] + r[k + 4]) + (r[k + 8] + r[k + 12]);
      const float c = cw * agg_sum((rs4[0] + rs4[1]) + (rs4[2] + rs4[3]));
#pragma unroll
      for (int v = 0; v < PV2; ++v) u[v] = (mbits >> v) & 1u ? r[v] + c : 0.f;
    };
    if (CC) {
      float dpart = 0.f;
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(a.sc + base + (long long)(Q2 * yq + i) * T2 + Q2 * xq));
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const int v = i * Q2 + k;
          const float wxl = k > 0 ? wxf[v - 1] : wxb[i];
          const float wyl = i > 0 ? wyf[v - Q2] : wyb[k];
          const bool m = q4l(s4, k) > 0.f;
          mbits |= (m ? 1u : 0u) << v;
          dpart += (m ? 1.f : 0.f) - ((wxf[v] + wxl) + (wyf[v] + wyl));
          if (i == 0 && !(yq & 1)) dpart += wyl;  // edges leaving the aggregate
          if (i == Q2 - 1 && (yq & 1)) dpart += wyf[v];
          if (k == 0 && !(xq & 1)) dpart += wxl;
          if (k == Q2 - 1 && (xq & 1)) dpart += wxf[v];
        }
      }
      const float d = agg_sum(dpart);
      cw = d > 1e-6f ? kCc2Omega / d : 0.f;
      form_u();
    }
    auto publish = [&]() {
      const float* q = CC ? u : r;
#pragma unroll
      for (int i = 0; i < Q2; ++i)
        sm.rp[Q2 * yq + i][xq] = make_float4(q[i * Q2], q[i * Q2 + 1], q[i * Q2 + 2], q[i * Q2 + 3]);
    };
    publish();
    __syncthreads();

    float alpha = 0.f, rgamma = 0.f, ralpha = 0.f;  // 1/gamma, 1/alpha one iteration ahead
    int state = ST_ACTIVE, it = 0;
    for (int pass = 0;; ++pass) {
      // ---- w = A'q (q = u with CC, else r), partial dots ----
      const float* q = CC ? u : r;
      const float4 qd = yq > 0 ? sm.rp[Q2 * yq - 1][xq] : z4;
      const float4 qu = yq + 1 < QN2 ? sm.rp[Q2 * yq + Q2][xq] : z4;
      float rs2[2] = {0.f, 0.f}, ds2[2] = {0.f, 0.f}, us2[2] = {0.f, 0.f};  // two chains each (latency)
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const float ql = __shfl_up_sync(0xffffffffu, q[i * Q2 + Q2 - 1], 1);
        const float qr = __shfl_down_sync(0xffffffffu, q[i * Q2], 1);
#pragma unroll
        for (int k = 0; k < Q2; k += 2) {  // pixel pairs (k, k+1) on the packed f32x2 FMA
          const int v = i * Q2 + k;
          float acc0, acc1;
          const float qyd0 = i > 0 ? q[v - Q2] : q4l(qd, k), qyd1 = i > 0 ? q[v + 1 - Q2] : q4l(qd, k + 1);
          const float qyu0 = i < Q2 - 1 ? q[v + Q2] : q4l(qu, k), qyu1 = i < Q2 - 1 ? q[v + 1 + Q2] : q4l(qu, k + 1);
          const float wyl0 = i > 0 ? wyf[v - Q2] : wyb[k], wyl1 = i > 0 ? wyf[v + 1 - Q2] : wyb[k + 1];
          fma2(acc0, acc1, wyf[v], wyf[v + 1], qyu0, qyu1, 0.f, 0.f);
          fma2(acc0, acc1, wyl0, wyl1, qyd0, qyd1, acc0, acc1);
          // x neighbours straddle the pairs: scalar
          acc0 = fmaf(wxf[v], q[v + 1], acc0);
          acc0 = fmaf(k > 0 ? wxf[v - 1] : wxb[i], k > 0 ? q[v - 1] : ql, acc0);
          acc1 = fmaf(wxf[v + 1], k + 1 < Q2 - 1 ? q[v + 2] : qr, acc1);
          acc1 = fmaf(wxf[v], q[v], acc1);
          fma2(w[v], w[v + 1], -1.f, -1.f, acc0, acc1, q[v], q[v + 1]);
          fma2(rs2[0], rs2[1], r[v], r[v + 1], r[v], r[v + 1], rs2[0], rs2[1]);
          fma2(ds2[0], ds2[1], w[v], w[v + 1], q[v], q[v + 1], ds2[0], ds2[1]);
          if (CC) fma2(us2[0], us2[1], r[v], r[v + 1], q[v], q[v + 1], us2[0], us2[1]);
        }
      }
      // ---- CTA reduction (fixed order): transpose-reduce the three warp sums (6 shuffles, not
      // 15; lanes 0-7 end with r.r, 8-15 with w.q, 16-23 with r.u), then a depth-3 tree over warps
      const int par = pass & 1;
      {
        const float rs = rs2[0] + rs2[1], ds = ds2[0] + ds2[1], us = CC ? us2[0] + us2[1] : 0.f;
        const bool hi = lane & 16, b3 = lane & 8;
        const float x0 = (hi ? us : rs) + __shfl_xor_sync(0xffffffffu, hi ? rs : us, 16);
        const float x1 = (hi ? 0.f : ds) + __shfl_xor_sync(0xffffffffu, hi ? ds : 0.f, 16);
        float t = (b3 ? x1 : x0) + __shfl_xor_sync(0xffffffffu, b3 ? x0 : x1, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        if ((lane & 7) == 0 && lane < 24) reinterpret_cast<float*>(&sm.wpart[par][warp])[lane >> 3] = t;
      }
      __syncthreads();  // partials visible; every thread has read rp (its SpMV is done)
      float4 wp[NW2];
#pragma unroll
      for (int wv = 0; wv < NW2; ++wv) wp[wv] = sm.wpart[par][wv];
      static_assert(NW2 == 8, "warp-sum tree");
      const float rr = ((wp[0].x + wp[1].x) + (wp[2].x + wp[3].x)) + ((wp[4].x + wp[5].x) + (wp[6].x + wp[7].x));
      const float delta = ((wp[0].y + wp[1].y) + (wp[2].y + wp[3].y)) + ((wp[4].y + wp[5].y) + (wp[6].y + wp[7].y));
      const float g_new =
          CC ? ((wp[0].z + wp[1].z) + (wp[2].z + wp[3].z)) + ((wp[4].z + wp[5].z) + (wp[6].z + wp[7].z)) : rr;
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
      // ---- update: p = q + beta p, s = w + beta s, y += alpha p, r -= alpha s ----
#pragma unroll
      for (int v = 0; v < PV2; v += 2) {
        fma2(p[v], p[v + 1], beta, beta, p[v], p[v + 1], q[v], q[v + 1]);
        fma2(sv[v], sv[v + 1], beta, beta, sv[v], sv[v + 1], w[v], w[v + 1]);
        fma2(y[v], y[v + 1], alpha, alpha, p[v], p[v + 1], y[v], y[v + 1]);
        fma2(r[v], r[v + 1], -alpha, -alpha, sv[v], sv[v + 1], r[v], r[v + 1]);
      }
      ++it;
      if (CC) form_u();
      publish();  // the barrier above proved every reader of the previous q has finished
      __syncthreads();
    }
    // ---- epilogue: probabilities and labels straight into the level ----
    {
      const int brick = a.list ? a.list[slot] : slot;
      const int hx = brick % a.gx, hy = brick / a.gx;
      const int gx0 = a.ox + hx * T2 + Q2 * xq;
      const bool quad_in = gx0 >= 0 && gx0 + Q2 <= a.nx;
      // all rows' scales first: one load latency per tile, not one per row
      float4 s4v[Q2];
#pragma unroll
      for (int i = 0; i < Q2; ++i)
        s4v[i] = __ldg(reinterpret_cast<const float4*>(a.sc + base + (long long)(Q2 * yq + i) * T2 + Q2 * xq));
#pragma unroll
      for (int i = 0; i < Q2; ++i) {
        const int gy = a.oy + hy * T2 + Q2 * yq + i;
        if (gy < 0 || gy >= a.ny) continue;
        const float4 s4 = s4v[i];
        float pv[Q2];
#pragma unroll
        for (int k = 0; k < Q2; ++k) {
          const float s = q4l(s4, k), yv = y[i * Q2 + k];
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
