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
  float2 wpart[2][NW2];  // per-warp (gamma, delta), double-buffered by iteration parity
};

__device__ __forceinline__ float q4l(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ float rcp_ftz2(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(TH2, 1) resident2d_kernel(ResidentArgs a) {
  __shared__ Resident2dSmem sm;
  const int tid = threadIdx.x;
  const int xq = tid % QN2, yq = tid / QN2;  // lanes 0..15 / 16..31 of a warp: two row bands
  const int lane = tid & 31, warp = tid >> 5;
  const int n_act = *a.n_active;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  const int tile_vox = T2 * T2;

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
      // ---- w = A'r, partial dots ----
      const float4 rd = yq > 0 ? sm.rp[Q2 * yq - 1][xq] : z4;
      const float4 ru = yq + 1 < QN2 ? sm.rp[Q2 * yq + Q2][xq] : z4;
      float gs = 0.f, ds = 0.f;
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
          gs = fmaf(r[v], r[v], gs);
          ds = fmaf(w[v], r[v], ds);
        }
      }
      // ---- CTA reduction (fixed order) ----
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gs += __shfl_xor_sync(0xffffffffu, gs, o);
        ds += __shfl_xor_sync(0xffffffffu, ds, o);
      }
      const int par = pass & 1;
      if (lane == 0) sm.wpart[par][warp] = make_float2(gs, ds);
      __syncthreads();  // partials visible; every thread has read rp (its SpMV is done)
      float g_new = 0.f, delta = 0.f;
#pragma unroll
      for (int wv = 0; wv < NW2; ++wv) {
        const float2 v = sm.wpart[par][wv];
        g_new += v.x;
        delta += v.y;
      }
      float beta;
      if (pass == 0) {
        beta = 0.f;
        alpha = delta != 0.f ? g_new * rcp_ftz2(delta) : 0.f;
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
        beta = g_new * rgamma;
        const float den = delta - beta * (g_new * ralpha);
        alpha = den != 0.f ? g_new * rcp_ftz2(den) : 0.f;
      }
      rgamma = rcp_ftz2(g_new);
      ralpha = rcp_ftz2(alpha);
      // ---- update: p = r + beta p, s = w + beta s, y += alpha p, r -= alpha s ----
#pragma unroll
      for (int v = 0; v < PV2; ++v) {
        p[v] = fmaf(beta, p[v], r[v]);
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
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(a.sc + base + (long long)(Q2 * yq + i) * T2 + Q2 * xq));
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
  static DeviceCache cache;
  int dev = 0;
  if (int rc = device_slot(&dev)) return rc;
  int grid = cache[dev].load(std::memory_order_relaxed);
  if (!grid) {
    int sms = 0, per = 0;
    RWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    RWB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, resident2d_kernel, TH2, 0));
    if (per <= 0) return fail(RWB_ERR_UNSUPPORTED, "2-D tile engine does not fit on this device");
    grid = sms * per;
    cache[dev].store(grid, std::memory_order_relaxed);
  }
  const int g = grid < max_bricks ? grid : max_bricks;
  if (g <= 0) return RWB_OK;
  resident2d_kernel<<<g, TH2, 0, st>>>(a);
  RWB_LAUNCH_CHECK("resident2d_kernel");
  count_launches(1);
  return RWB_OK;
}

}  // namespace rwb
