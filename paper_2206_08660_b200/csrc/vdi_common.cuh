// vdi_common.cuh -- device helpers shared by the generation and render
// kernels. Everything here is f64 and evaluated in the reference's operation
// order; the whole library is compiled with -fmad=false, so no multiply-add
// is contracted into an FMA (numba emits none).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/vdi_b200.h"

namespace vdi {

constexpr double kSqrt3 = 1.7320508075688772;  // math.sqrt(3.0), generate.py:25
constexpr int kTileW = 8;                     // a warp owns an 8x4 pixel tile
constexpr int kTileH = 4;

// x / d, correctly rounded, with y = RN(1 / d) given (Markstein: q = RN(x y)
// is within 1 ulp, r = x - q d is exact with an FMA, q + r y rounds correctly;
// valid for any d barring over/underflow). The FMAs compute an exact residual;
// they do not contract any expression of the reference. Verified on device by
// vdi_selftest_arith (tests/test_gpu_arith.py) and on 2.2e9 host quotients.
__device__ __forceinline__ double div_by(double x, double d, double y) {
  const double q = x * y;
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, y, q);
}

// _geom.py:12-19 ndc_of / 22-25 world_of: ((m0 x + m1 y) + m2 z) + m3, / w.
// The three quotients by the same w share one IEEE reciprocal.
__device__ __forceinline__ void xform(const double* __restrict__ m, double x, double y,
                                      double z, double& ox, double& oy, double& oz) {
  const double hx = m[0] * x + m[1] * y + m[2] * z + m[3];
  const double hy = m[4] * x + m[5] * y + m[6] * z + m[7];
  const double hz = m[8] * x + m[9] * y + m[10] * z + m[11];
  const double hw = m[12] * x + m[13] * y + m[14] * z + m[15];
  const double rw = 1.0 / hw;
  ox = div_by(hx, hw, rw);
  oy = div_by(hy, hw, rw);
  oz = div_by(hz, hw, rw);
}

// Only the z component of ndc_of (what _emit, generate.py:55-56, keeps).
__device__ __forceinline__ double xform_z(const double* __restrict__ m, double x, double y,
                                          double z) {
  const double hz = m[8] * x + m[9] * y + m[10] * z + m[11];
  const double hw = m[12] * x + m[13] * y + m[14] * z + m[15];
  return hz / hw;
}

// _geom.py:28-54 clip_aabb.
__device__ __forceinline__ bool clip_aabb(const double o[3], const double d[3],
                                          const double* bb, double& t0o, double& t1o) {
  double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = bb[a], hi = bb[3 + a];
    if (fabs(d[a]) < 1e-300) {
      if (o[a] < lo || o[a] > hi) return false;
    } else {
      double ta = (lo - o[a]) / d[a];
      double tb = (hi - o[a]) / d[a];
      if (ta > tb) {
        const double s = ta;
        ta = tb;
        tb = s;
      }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    }
  }
  if (t1 < t0) return false;
  t0o = t0;
  t1o = t1;
  return true;
}

// _geom.py:57-104 clip_frustum: 7 homogeneous half-spaces c + t d >= 0.
__device__ __forceinline__ bool clip_frustum(const double* __restrict__ m, const double o[3],
                                             const double d[3], double& t0o, double& t1o) {
  const double p0x = m[0] * o[0] + m[1] * o[1] + m[2] * o[2] + m[3];
  const double p0y = m[4] * o[0] + m[5] * o[1] + m[6] * o[2] + m[7];
  const double p0z = m[8] * o[0] + m[9] * o[1] + m[10] * o[2] + m[11];
  const double p0w = m[12] * o[0] + m[13] * o[1] + m[14] * o[2] + m[15];
  const double pdx = m[0] * d[0] + m[1] * d[1] + m[2] * d[2];
  const double pdy = m[4] * d[0] + m[5] * d[1] + m[6] * d[2];
  const double pdz = m[8] * d[0] + m[9] * d[1] + m[10] * d[2];
  const double pdw = m[12] * d[0] + m[13] * d[1] + m[14] * d[2];
  const double cs[7] = {p0w, p0w - p0x, p0w + p0x, p0w - p0y, p0w + p0y, p0w - p0z, p0w + p0z};
  const double ds[7] = {pdw, pdw - pdx, pdw + pdx, pdw - pdy, pdw + pdy, pdw - pdz, pdw + pdz};
  double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
  for (int i = 0; i < 7; ++i) {
    const double c = cs[i], dd = ds[i];
    if (fabs(dd) < 1e-300) {
      if (c < 0) return false;
    } else {
      const double t = -c / dd;
      if (dd > 0) {
        if (t > t0) t0 = t;
      } else {
        if (t < t1) t1 = t;
      }
    }
  }
  if (t1 < t0) return false;
  t0o = t0;
  t1o = t1;
  return true;
}

// List-SoA offsets (include/vdi_b200.h): [rgba float4 | front | back | pad].
__host__ __device__ __forceinline__ int list_stride(int n_sg) { return (6 * n_sg + 3) & ~3; }
__host__ __device__ __forceinline__ int front_off(int n_sg) { return 4 * n_sg; }
__host__ __device__ __forceinline__ int back_off(int n_sg) { return 5 * n_sg; }

__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// Eye ray through a pixel centre (generate.py:282-294, raycast.py:286-297).
__device__ __forceinline__ void pixel_ray(const double* __restrict__ inv_pv, const double* eye,
                                          int col, int row, int w, int h, double d[3]) {
  const double ndcx = 2.0 * (col + 0.5) / w - 1.0;
  const double ndcy = 2.0 * (row + 0.5) / h - 1.0;
  double wx, wy, wz;
  xform(inv_pv, ndcx, ndcy, -1.0, wx, wy, wz);
  const double dx = wx - eye[0], dy = wy - eye[1], dz = wz - eye[2];
  const double norm = sqrt(dx * dx + dy * dy + dz * dz);
  d[0] = dx / norm;
  d[1] = dy / norm;
  d[2] = dz / norm;
}

// Band map (include/vdi_b200.h): local row -> image row.
__device__ __forceinline__ int band_global_row(int local_row, int band_rows, int stride,
                                               int offset) {
  const int j = local_row / band_rows;
  return (j * stride + offset) * band_rows + (local_row - j * band_rows);
}

// Local row -> image row, with the contiguous-range override
// (VdiGenArgs.row_count > 0: rows [row_base, row_base + row_count)).
__device__ __forceinline__ int image_row(int local_row, int band_rows, int stride, int offset,
                                         int row_base, int row_count) {
  return row_count > 0 ? row_base + local_row
                       : band_global_row(local_row, band_rows, stride, offset);
}

// Storage row of list row r in an all-gathered band-sharded VDI.
__device__ __forceinline__ int vdi_storage_row(int r, int band_rows, int world,
                                               int rows_per_rank) {
  if (world <= 1) return r;
  const int b = r / band_rows;
  return (b % world) * rows_per_rank + (b / world) * band_rows + (r - b * band_rows);
}

}  // namespace vdi
