// Volume raycaster over an LOD pyramid — SURVEY.md §8(f)4, the march of the reference's
// `render.py:352-433` (`_march_pass`) and its compositing (`render.py:527-541`), one thread per pixel.
//
// The reference splits a frame into an entry-exit node (`entry_exit_points`, `render.py:203-249`:
// per pixel the ray's entry / exit distance in the volume box and its footprint terms, stored as
// float32) and a march in float64 from rays re-derived with `_pixel_rays`.  The host side
// (`render.raycast_frame`) computes exactly those per-pixel records with the reference's numpy
// expressions; this kernel marches them: one sample per step at t — the level whose finest spacing
// does not exceed the footprint fp0 + fps*t (+ bias, `select_level`), the nearest voxel
// floor(pos / spacing) clamped (`brick_of`), the grey-ramp transfer function, then DVR (opacity
// corrected to the step, 1 - (1 - a)^(dt / ds0), front to back, early termination at alpha 0.99)
// or MOP (maximum opacity); step dt = sample_distance_factor x the sampled level's finest spacing.
// Every float64 operation is the reference's, in its order, with explicit round-to-nearest
// intrinsics (no FMA contraction numpy does not do).  The reference's progressive preview pass only
// changes when a tile's bricks are fetched, never the final frame, which is this uninterrupted
// march (its constant-chunk tables return the payloads' values).  Output: premultiplied RGBA,
// float32, or u8 = rint(clip(x, 0, 1) * 255).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "rwb_common.cuh"

namespace rwb {
namespace {

constexpr int kMaxLevels = 24;
constexpr double kEarlyTermination = 0.99;  // render.py EARLY_TERMINATION_ALPHA

struct RayLevels {
  const float* data[kMaxLevels];
  int size[kMaxLevels][3];
  double spacing[kMaxLevels][3];
  double minsp[kMaxLevels];
  int n;
};

struct RayParams {
  long long n_px;
  int mop;  // 0 = DVR, 1 = MOP
  double sdf, bias, tf_lo, tf_hi;
};

// rays: per pixel 10 doubles — origin (3) and unit direction (3) from `_pixel_rays`, then the
// entry-exit record (t_entry, t_exit, fp0, fps) as float32 values widened (t_entry = +inf: miss)
template <bool U8>
__global__ void __launch_bounds__(128) raycast_kernel(const __grid_constant__ RayLevels lv,
                                                      const __grid_constant__ RayParams p,
                                                      const double* __restrict__ rays, void* out) {
  const long long px = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (px >= p.n_px) return;
  const double* r = rays + 10 * px;
  const double org[3] = {r[0], r[1], r[2]}, dir[3] = {r[3], r[4], r[5]};
  double t = r[6];
  const double t_exit = r[7], fp0 = r[8], fps = r[9];
  if (!isfinite(t)) t = INFINITY;
  const double ds0 = lv.minsp[0];
  double acc_c = 0.0, acc_a = 0.0, mop_a = 0.0, mop_c = 0.0;
  bool alive = true;
  while (alive && t <= t_exit) {
    const double fp = __dadd_rn(fp0, __dmul_rn(fps, t));
    int sel = -1;  // searchsorted(minsps, fp, side="right") - 1
    for (int k = 0; k < lv.n; ++k) sel += lv.minsp[k] <= fp ? 1 : 0;
    int l = (int)floor(__dadd_rn((double)sel, p.bias));
    l = l < 0 ? 0 : (l > lv.n - 1 ? lv.n - 1 : l);
    long long off = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double pos = __dadd_rn(org[d], __dmul_rn(t, dir[d]));
      long long i = (long long)floor(__ddiv_rn(pos, lv.spacing[l][d]));
      i = i < 0 ? 0 : (i > lv.size[l][d] - 1 ? lv.size[l][d] - 1 : i);
      off = off * lv.size[l][d] + i;
    }
    const double v = (double)__ldg(lv.data[l] + off);
    const double dt = __dmul_rn(p.sdf, lv.minsp[l]);
    // grey ramp: rgba = (a, a, a, a)
    const double a = fmin(fmax(__ddiv_rn(__dsub_rn(v, p.tf_lo), __dsub_rn(p.tf_hi, p.tf_lo)), 0.0), 1.0);
    if (!p.mop) {
      const double corrected = __dsub_rn(1.0, pow(__dsub_rn(1.0, a), __ddiv_rn(dt, ds0)));
      const double weight = __dmul_rn(__dsub_rn(1.0, acc_a), corrected);
      acc_c = __dadd_rn(acc_c, __dmul_rn(weight, a));
      acc_a = __dadd_rn(acc_a, weight);
      alive = acc_a < kEarlyTermination;
    } else if (a > mop_a) {
      mop_a = a;
      mop_c = a;
    }
    t = __dadd_rn(t, dt);
  }
  double rgba[4];
  if (!p.mop) {
    rgba[0] = rgba[1] = rgba[2] = acc_c;
    rgba[3] = acc_a;
  } else {
    rgba[0] = rgba[1] = rgba[2] = __dmul_rn(mop_a, mop_c);
    rgba[3] = mop_a;
  }
  if (U8) {
    uchar4 q;
    unsigned char* c = reinterpret_cast<unsigned char*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = (unsigned char)rint(__dmul_rn(fmin(fmax(rgba[k], 0.0), 1.0), 255.0));
    reinterpret_cast<uchar4*>(out)[px] = q;
  } else {
    reinterpret_cast<float4*>(out)[px] = make_float4((float)rgba[0], (float)rgba[1], (float)rgba[2], (float)rgba[3]);
  }
}

}  // namespace
}  // namespace rwb

extern "C" int rwb_raycast(int32_t n_levels, const float* const* levels, const int64_t* sizes, const double* spacing,
                           int64_t n_px, const double* rays, int32_t compositing, double sample_distance_factor,
                           double lod_bias, double tf_lo, double tf_hi, int32_t out_u8, void* out, void* stream) {
  using namespace rwb;
  if (n_levels < 1 || n_levels > kMaxLevels || !levels || !sizes || !spacing || n_px < 0 || !rays || !out)
    return fail(RWB_ERR_INVALID, "raycast: bad arguments");
  if (!(sample_distance_factor > 0.0) || !(tf_hi > tf_lo) || compositing < 0 || compositing > 1)
    return fail(RWB_ERR_INVALID, "raycast: bad step, transfer function or compositing");
  RayLevels lv;
  std::memset(&lv, 0, sizeof(lv));
  lv.n = n_levels;
  for (int k = 0; k < n_levels; ++k) {
    if (!levels[k]) return fail(RWB_ERR_INVALID, "raycast: null level");
    lv.data[k] = levels[k];
    double mn = INFINITY;
    for (int d = 0; d < 3; ++d) {
      if (sizes[3 * k + d] < 1 || !(spacing[3 * k + d] > 0.0))
        return fail(RWB_ERR_INVALID, "raycast: level sizes and spacings must be positive");
      lv.size[k][d] = (int)sizes[3 * k + d];
      lv.spacing[k][d] = spacing[3 * k + d];
      mn = spacing[3 * k + d] < mn ? spacing[3 * k + d] : mn;
    }
    lv.minsp[k] = mn;
  }
  if (n_px == 0) return RWB_OK;
  RayParams p;
  p.n_px = n_px;
  p.mop = compositing;
  p.sdf = sample_distance_factor, p.bias = lod_bias, p.tf_lo = tf_lo, p.tf_hi = tf_hi;
  const unsigned grid = (unsigned)((n_px + 127) / 128);
  if (out_u8)
    raycast_kernel<true><<<grid, 128, 0, (cudaStream_t)stream>>>(lv, p, rays, out);
  else
    raycast_kernel<false><<<grid, 128, 0, (cudaStream_t)stream>>>(lv, p, rays, out);
  RWB_LAUNCH_CHECK("raycast_kernel");
  count_launches(1);
  return RWB_OK;
}
