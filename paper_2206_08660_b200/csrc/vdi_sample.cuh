// vdi_sample.cuh -- the volume sampler shared by generation (vdi_gen.cu) and
// the direct volume renderer (vdi_dvr.cu): trilinear interpolation
// (volume.py:180-205 _trilinear) and transfer-function classification
// (volume.py:164-177 _lut_classify), f64 in the reference's order.
//
// trilinear<VT>(c, ...) reads, from any constant block `c`: c.a.volume,
// c.a.nx/ny/nz, c.a.brick_max, c.a.brick_log2, c.a.ess_max, c.ess, c.bnx,
// c.bny (the generation and DVR argument blocks share these names), and for
// kVoxelSub variants c.sub_*.
#pragma once

#include "vdi_common.cuh"

namespace vdi {

template <int VT>
struct Voxel;
template <>
struct Voxel<VDI_VOXEL_F32> {
  using type = float;
  static __device__ __forceinline__ double get(const void* p, long long i, const double*) {
    return (double)__ldg(reinterpret_cast<const float*>(p) + i);
  }
};
template <>
struct Voxel<VDI_VOXEL_U8> {
  using type = unsigned char;
  // volume.py:48-50 normalises with an f32 division by 255; the 256 exact
  // quotients live in shared memory, already widened to f64.
  static __device__ __forceinline__ double get(const void* p, long long i, const double* tab) {
    return tab[__ldg(reinterpret_cast<const unsigned char*>(p) + i)];
  }
};
template <>
struct Voxel<VDI_VOXEL_U16> {
  using type = unsigned short;
  static __device__ __forceinline__ double get(const void* p, long long i, const double*) {
    return (double)__fdiv_rn((float)__ldg(reinterpret_cast<const unsigned short*>(p) + i),
                             65535.0f);
  }
};

// Corner records (vdi_volume_cells): the 8 voxels of cell i in one load.
template <int BT>
struct Cell;
template <>
struct Cell<VDI_VOXEL_U8> {
  static __device__ __forceinline__ void get(const void* cells, long long i, const double* tab,
                                             double v[8]) {
    const uint2 r = __ldg(reinterpret_cast<const uint2*>(cells) + i);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      v[b] = tab[(r.x >> (8 * b)) & 0xffu];
      v[4 + b] = tab[(r.y >> (8 * b)) & 0xffu];
    }
  }
};
template <>
struct Cell<VDI_VOXEL_U16> {
  static __device__ __forceinline__ void get(const void* cells, long long i, const double*,
                                             double v[8]) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(cells) + i);
    const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      v[2 * b] = (double)__fdiv_rn((float)(w[b] & 0xffffu), 65535.0f);
      v[2 * b + 1] = (double)__fdiv_rn((float)(w[b] >> 16), 65535.0f);
    }
  }
};
template <>
struct Cell<VDI_VOXEL_F32> {
  static __device__ __forceinline__ void get(const void* cells, long long i, const double*,
                                             double v[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(cells) + 2 * i);
    const float4 b = __ldg(reinterpret_cast<const float4*>(cells) + 2 * i + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};

// Brick bi of brick_max classifies as always transparent (its maximum <=
// ess_max). u8: the raw byte against c.ess_u8, the largest v with v / 255
// (the f32 quotient of volume.py:48-50, widened) <= ess_max -- the same test,
// since the quotient grows with v -- without the table load and f64 compare.
template <int VT, class C>
__device__ __forceinline__ bool brick_empty(const C& c, long long bi, const double* tab) {
  if constexpr ((VT & 15) == VDI_VOXEL_U8)
    return (int)__ldg(static_cast<const unsigned char*>(c.a.brick_max) + bi) <= c.ess_u8;
  else
    return Voxel<(VT & 15)>::get(c.a.brick_max, bi, tab) <= c.a.ess_max;
}

// Kernel-variant flag (not part of the C ABI): the volume in memory is only
// a resident box of the full grid (VdiGenArgs.sub_origin / sub_dims), e.g.
// one rank's slab of a volume bricked across GPUs. Sample positions and cell
// indices stay those of the full grid; only the addresses are rebased.
constexpr int kVoxelSub = 32;

// volume.py:180-205 _trilinear. VT is a VDI_VOXEL_* type, optionally with the
// VDI_VOXEL_CELLS flag (c.a.volume then holds corner records) and kVoxelSub
// (then c.sub_* describe the resident box).
template <int VT, class C>
__device__ __forceinline__ double trilinear(const C& c, const double* tab, double px,
                                            double py, double pz) {
  const int nx = c.a.nx, ny = c.a.ny, nz = c.a.nz;
  const double gx = px * (double)(nx - 1);
  const double gy = py * (double)(ny - 1);
  const double gz = pz * (double)(nz - 1);
  int ix = (int)gx, iy = (int)gy, iz = (int)gz;
  if (ix > nx - 2) ix = nx - 2;
  if (iy > ny - 2) iy = ny - 2;
  if (iz > nz - 2) iz = nz - 2;
  long long sx = nx, sy = ny, voff = 0, boff = 0;
  if constexpr ((VT & kVoxelSub) != 0) {
    sx = c.sub_sx;
    sy = c.sub_sy;
    voff = c.sub_voff;
    boff = c.sub_boff;
    // a cell outside the resident box means the box was planned too small:
    // flag it (the result is then invalid) and keep the address in bounds
    const int lx = ix - c.sub_ox, ly = iy - c.sub_oy, lz = iz - c.sub_oz;
    if ((unsigned)lx > (unsigned)(c.sub_nx - 2) || (unsigned)ly > (unsigned)(c.sub_ny - 2) ||
        (unsigned)lz > (unsigned)(c.sub_nz - 2)) {
      if (c.sub_oob) atomicOr(c.sub_oob, 1u);
      ix = c.sub_ox + min(max(lx, 0), c.sub_nx - 2);
      iy = c.sub_oy + min(max(ly, 0), c.sub_ny - 2);
      iz = c.sub_oz + min(max(lz, 0), c.sub_nz - 2);
    }
  }
  if (c.ess) {
    // Exact empty-space skip: every voxel this sample can read lies in the
    // brick (+1 halo), whose maximum classifies at or below the last row of
    // the LUT's leading alpha == 0 run with margin, and a trilinear mix never
    // exceeds its largest input by more than a few ulps. -1 classifies to LUT
    // row 0, whose alpha is 0: the sample is transparent, as in the reference.
    const int lb = c.a.brick_log2;
    // brick counts fit 32 bits (a 2^31-brick grid would be 2^40 voxels)
    const long long bi = (long long)(((iz >> lb) * c.bny + (iy >> lb)) * c.bnx + (ix >> lb)) - boff;
    if (brick_empty<VT>(c, bi, tab)) return -1.0;
  }
  const double fx = gx - ix, fy = gy - iy, fz = gz - iz;
  if (VT & VDI_VOXEL_CELLS) {
    double v[8];
    Cell<(VT & 15)>::get(c.a.volume, ((long long)iz * sy + iy) * sx + ix - voff, tab, v);
    const double c00 = v[0] * (1 - fx) + v[1] * fx;
    const double c10 = v[2] * (1 - fx) + v[3] * fx;
    const double c01 = v[4] * (1 - fx) + v[5] * fx;
    const double c11 = v[6] * (1 - fx) + v[7] * fx;
    const double c0 = c00 * (1 - fy) + c10 * fy;
    const double c1 = c01 * (1 - fy) + c11 * fy;
    return c0 * (1 - fz) + c1 * fz;
  }
  // four row pointers, then [ptr + 0/1] gathers (no per-voxel 64-bit math)
  using T = typename Voxel<(VT & 15)>::type;
  const T* r00 = static_cast<const T*>(c.a.volume) + (((long long)iz * sy + iy) * sx + ix - voff);
  const T* r01 = r00 + sx;
  const T* r10 = r00 + sx * sy;
  const T* r11 = r10 + sx;
  using V = Voxel<(VT & 15)>;
  const double v000 = V::get(r00, 0, tab), v001 = V::get(r00, 1, tab);
  const double v010 = V::get(r01, 0, tab), v011 = V::get(r01, 1, tab);
  const double v100 = V::get(r10, 0, tab), v101 = V::get(r10, 1, tab);
  const double v110 = V::get(r11, 0, tab), v111 = V::get(r11, 1, tab);
  const double c00 = v000 * (1 - fx) + v001 * fx;
  const double c10 = v010 * (1 - fx) + v011 * fx;
  const double c01 = v100 * (1 - fx) + v101 * fx;
  const double c11 = v110 * (1 - fx) + v111 * fx;
  const double c0 = c00 * (1 - fy) + c10 * fy;
  const double c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz;
}

// Empty-brick runs, an exact shortcut over per-sample empty-space skipping.
// When the sample at parameter tm lies in a brick whose maximum classifies
// to alpha 0, every later sample whose cell stays in that brick is
// transparent too. The cell coordinate g_a = q_a (n_a - 1) of sample k is
// affine in k (tm = t0 + (k + 0.5) step up to rounding), so the samples that
// stay inside the brick with a margin of 1e-6 cells -- far above the few-ulp
// rounding of the sampler's own evaluation of g -- need not be sampled.
// Returns how many samples from this one on (>= 1, <= max_run) are known to
// be transparent, or 0 when this sample's brick is not an empty one.
// inv_ext / ext_pow2 / c.a.aabb as in the sampler; only with c.ess.
#ifndef VDI_RUN_F32
#define VDI_RUN_F32 1
#endif
template <int VT, class C>
__device__ __forceinline__ int empty_run(const C& c, const double* tab, const double o[3],
                                         const double d[3], double tm, double step,
                                         int max_run) {
  const int n[3] = {c.a.nx, c.a.ny, c.a.nz};
  double g[3];
  int cell[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double num = o[a] + tm * d[a] - c.a.aabb[a];
    const double v = c.ext_pow2[a] ? num * c.inv_ext[a]
                                   : div_by(num, c.a.aabb[3 + a] - c.a.aabb[a], c.inv_ext[a]);
    if (!(v >= 0.0 && v <= 1.0)) return 0;  // clamped sample: no run
    g[a] = v * (double)(n[a] - 1);
    int ic = (int)g[a];
    if (ic > n[a] - 2) ic = n[a] - 2;
    cell[a] = ic;
  }
  const int lb = c.a.brick_log2;
  long long boff = 0;
  if constexpr ((VT & kVoxelSub) != 0) boff = c.sub_boff;
  const long long bi = ((long long)(cell[2] >> lb) * c.bny + (cell[1] >> lb)) * c.bnx +
                       (cell[0] >> lb) - boff;
  if (!brick_empty<VT>(c, bi, tab)) return 0;
  const int B = 1 << lb;
  long long m = max_run - 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int b0 = (cell[a] >> lb) << lb;
    // the brick's g interval; the clamps make the outer bricks open-ended
    const double lo = b0 == 0 ? -INFINITY : (double)b0;
    const double hi = b0 + B - 1 >= n[a] - 2 ? INFINITY : (double)(b0 + B);
    const double dg = d[a] * step * (double)(n[a] - 1) * c.inv_ext[a];
#if VDI_RUN_F32
    // the run only has to be a lower bound: an f32 quotient (relative error
    // < 1e-6 after the two conversions) scaled by 1 - 2^-16 never exceeds
    // the exact one, and a shorter run only re-enters this test
    float lim = INFINITY;
    if (dg > 0.0)
      lim = __fdividef((float)(hi - 1e-6 - g[a]), (float)dg) * (1.0f - 0x1p-16f);
    else if (dg < 0.0)
      lim = __fdividef((float)(g[a] - lo - 1e-6), (float)-dg) * (1.0f - 0x1p-16f);
    if (!(lim >= 0.0f)) return 1;  // within the margin of the brick's edge
    if ((double)lim < (double)m) m = (long long)lim;
#else
    double lim = INFINITY;
    if (dg > 0.0) lim = (hi - 1e-6 - g[a]) / dg;
    else if (dg < 0.0) lim = (g[a] - lo - 1e-6) / -dg;
    if (!(lim >= 0.0)) return 1;  // within the margin of the brick's edge
    if (lim < (double)m) m = (long long)lim;
#endif
  }
  return 1 + (int)m;
}

// volume.py:164-177 _lut_classify: f64 lerp rounded to f32.
__device__ __forceinline__ float4 narrow(const double4 v) {
  return make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
}
__device__ __forceinline__ float4 classify(const double4* lut, int n, double s) {
  const double x = s * (double)(n - 1);
  if (x <= 0.0) return narrow(lut[0]);
  if (x >= (double)(n - 1)) return narrow(lut[n - 1]);
  const int i = (int)x;
  const double f = x - i;
  const double4 l0 = lut[i], l1 = lut[i + 1];
  float4 o;
  o.x = (float)(l0.x * (1.0 - f) + l1.x * f);
  o.y = (float)(l0.y * (1.0 - f) + l1.y * f);
  o.z = (float)(l0.z * (1.0 - f) + l1.z * f);
  o.w = (float)(l0.w * (1.0 - f) + l1.w * f);
  return o;
}

}  // namespace vdi
