// vdi_dvr.cu -- ground-truth direct volume rendering on sm_100a.
//
// Semantics: the reference's _dvr_kernel (dvr.py:21-89): the generation ray
// and clip (dvr.py:28-50 == generate.py:282-306), the same midpoint sampler
// (volume.py:164-205) and opacity length normalisation, composited front to
// back with early termination at early_term. f64 in the reference's order;
// the library is built with -fmad=false.
//
// B200 structure: one lane per ray; a warp starts on an 8x4 pixel tile and
// its lanes refill from a warp-uniform ray pool (one atomic per 32 rays) as
// their rays terminate, so no lane idles on a long neighbour and
// neighbouring lanes sample neighbouring voxels. The sampler is the
// generation one (vdi_sample.cuh): u8 voxels normalised through a shared
// 256-entry table, optional corner records (one load per sample) and exact
// empty-space skipping on brick maxima.
#include <cstdio>

#include "vdi_common.cuh"
#include "vdi_internal.h"
#include "vdi_sample.cuh"

namespace vdi {

constexpr int kDvrThreads = 128;
#ifndef VDI_DVR_MINB
#define VDI_DVR_MINB 6
#endif

struct DvrConst {
  VdiDvrArgs a;
  double inv_ext[3];
  int ext_pow2[3];
  double inv_lref;
  int lref_pow2;
  int ess, bnx, bny;
  int ess_u8;      // u8 volumes: ess_max as a byte threshold (brick_empty)
  int tiles_x, local_h;
  long long n_slots;
  unsigned long long* fetch;
  // resident-box fields of the shared sampler (unused: DVR samples full volumes)
  long long sub_sx, sub_sy, sub_voff, sub_boff;
  int sub_ox, sub_oy, sub_oz, sub_nx, sub_ny, sub_nz;
  unsigned* sub_oob;
};

struct DvrRay {
  double d[3], t0, t1;
  double r, g, b, a;
  int k, nsteps, pix, samples;
};

// dvr.py:28-50: pixel ray, AABB + frustum clip. Returns false on a miss.
__device__ __forceinline__ bool dvr_setup(const DvrConst& c, DvrRay& s, int pix) {
  const int lx = pix % c.a.width, ly = pix / c.a.width;
  const int gy = band_global_row(ly, c.a.band_rows, c.a.band_stride, c.a.band_offset);
  s.pix = pix;
  s.r = s.g = s.b = s.a = 0.0;
  s.k = 0;
  s.samples = 0;
  pixel_ray(c.a.inv_pv, c.a.eye, lx, gy, c.a.width, c.a.height, s.d);
  double ta, tb, fa, fb;
  if (!(clip_aabb(c.a.eye, s.d, c.a.aabb, ta, tb) && clip_frustum(c.a.pv, c.a.eye, s.d, fa, fb)))
    return false;
  s.t0 = dmax(dmax(ta, fa), 0.0);
  s.t1 = dmin(tb, fb);
  if (!(s.t1 > s.t0)) return false;
  s.nsteps = (int)ceil((s.t1 - s.t0) / c.a.step);
  return s.nsteps > 0;
}

// dvr.py:84-89: background blend and store.
__device__ __forceinline__ void dvr_finish(const DvrConst& c, const DvrRay& s) {
  const double* bg = c.a.bg;
  const double w = 1.0 - s.a;
  double2* o = reinterpret_cast<double2*>(c.a.image + 4 * (long long)s.pix);
  o[0] = make_double2(s.r + w * bg[0] * bg[3], s.g + w * bg[1] * bg[3]);
  o[1] = make_double2(s.b + w * bg[2] * bg[3], s.a + w * bg[3]);
  if (c.a.samples) c.a.samples[s.pix] = s.samples;
}

template <int VT>
__global__ void __launch_bounds__(kDvrThreads, VDI_DVR_MINB) dvr_kernel(const DvrConst c) {
  extern __shared__ double4 s_lut[];
  __shared__ double s_u8[256];
  for (int i = threadIdx.x; i < c.a.lut_n; i += blockDim.x) {
    const float4 l = reinterpret_cast<const float4*>(c.a.lut)[i];
    s_lut[i] = make_double4(l.x, l.y, l.z, l.w);
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_u8[i] = (double)__fdiv_rn((float)i, 255.0f);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const double step = c.a.step;
  unsigned long long total = 0;
  long long base = 0;
  int used = 32;
  bool have = false, done = false;
  DvrRay s;

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      // warp-uniform pool: lanes in `need` take consecutive slots
      const int n = __popc(need);
      const int rank = __popc(need & ((1u << lane) - 1u));
      const int avail = 32 - used;
      long long fresh = 0;
      if (n > avail) {
        if (lane == 0) fresh = (long long)atomicAdd(c.fetch, 32ull);
        fresh = __shfl_sync(0xffffffffu, fresh, 0);
      }
      const long long slot = rank < avail ? base + used + rank : fresh + (rank - avail);
      if (n > avail) {
        base = fresh;
        used = n - avail;
      } else {
        used += n;
      }
      if ((need >> lane) & 1u) {
        if (slot >= c.n_slots) {
          done = true;
        } else {
          const long long tile = slot >> 5;
          const int w = (int)(slot & 31);
          const int lx = (int)(tile % c.tiles_x) * kTileW + (w & 7);
          const int ly = (int)(tile / c.tiles_x) * kTileH + (w >> 3);
          if (lx < c.a.width && ly < c.local_h) {
            have = dvr_setup(c, s, ly * c.a.width + lx);
            if (!have) dvr_finish(c, s);
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    // dvr.py:52-83, one sample per iteration
    const double sa = s.t0 + (double)s.k * step;
    double sb = sa + step;
    if (sb > s.t1) sb = s.t1;
    bool end = !(sb > sa);
    if (!end) {
      s.samples += 1;
      const double tm = 0.5 * (sa + sb);
      double q[3];
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double num = c.a.eye[ax] + tm * s.d[ax] - c.a.aabb[ax];
        double v = c.ext_pow2[ax] ? num * c.inv_ext[ax]
                                  : div_by(num, c.a.aabb[3 + ax] - c.a.aabb[ax], c.inv_ext[ax]);
        q[ax] = dmin(dmax(v, 0.0), 1.0);
      }
      const double val = trilinear<VT>(c, s_u8, q[0], q[1], q[2]);
      const float4 rgba = classify(s_lut, c.a.lut_n, val);
      if (val == -1.0 && c.ess) {  // the empty-brick sentinel (or a genuine -1 sample)
        // a run of samples in an empty brick: all transparent (dvr.py:64-65)
        int run = empty_run<VT>(c, s_u8, c.a.eye, s.d, tm, step, s.nsteps - 1 - s.k);
        if (run > 1) {
          s.samples += run - 1;
          s.k += run - 1;
        }
      }
      if (rgba.w > 0.0f) {
        const double a = (double)rgba.w;
        const double dt = sb - sa;
        const double e = c.lref_pow2 ? dt * c.inv_lref : div_by(dt, c.a.lref, c.inv_lref);
        const double om = 1.0 - a;
        const double a_adj = 1.0 - (e == 1.0 ? om : pow(om, e));
        const double w = 1.0 - s.a;
        s.r += w * (double)rgba.x * a_adj;
        s.g += w * (double)rgba.y * a_adj;
        s.b += w * (double)rgba.z * a_adj;
        s.a += w * a_adj;
        if (s.a >= c.a.early_term) end = true;
      }
      s.k += 1;
      if (s.k >= s.nsteps) end = true;
    }
    if (end) {
      total += (unsigned long long)s.samples;
      dvr_finish(c, s);
      have = false;
    }
  }
  if (c.a.stat_sums) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    if (lane == 0 && total) atomicAdd(c.a.stat_sums, total);
  }
}

int dvr_launch(const VdiDvrArgs* a, cudaStream_t stream) {
  DvrConst c;
  c.a = *a;
  for (int i = 0; i < 3; ++i) {
    const double ext = a->aabb[3 + i] - a->aabb[i];
    int e;
    c.ext_pow2[i] = (frexp(ext, &e) == 0.5);
    c.inv_ext[i] = 1.0 / ext;
  }
  {
    int e;
    c.lref_pow2 = (frexp(a->lref, &e) == 0.5);
    c.inv_lref = 1.0 / a->lref;
  }
  const int band_rows = a->band_rows > 0 ? a->band_rows : 16;
  c.a.band_rows = band_rows;
  if (c.a.band_stride <= 0) c.a.band_stride = 1;
  c.local_h = local_rows(a->height, band_rows, c.a.band_stride, c.a.band_offset);
  c.tiles_x = (a->width + kTileW - 1) / kTileW;
  const long long tiles_y = (c.local_h + kTileH - 1) / kTileH;
  c.n_slots = (long long)c.tiles_x * tiles_y * 32;
  c.ess = a->brick_max != nullptr && a->ess_max >= 0.0 && a->brick_log2 >= 1;
  c.ess_u8 = -1;  // the largest v with (double)((float)v / 255) <= ess_max
  for (int v = 0; v < 256; ++v)
    if ((double)((float)v / 255.0f) <= a->ess_max) c.ess_u8 = v;
  if (c.ess) {
    const int B = 1 << a->brick_log2;
    c.bnx = (a->nx + B - 1) / B;
    c.bny = (a->ny + B - 1) / B;
  } else {
    c.bnx = c.bny = 0;
  }
  if (c.local_h <= 0) return VDI_OK;
  c.fetch = reinterpret_cast<unsigned long long*>(a->workspace);
  cudaError_t err = cudaMemsetAsync(c.fetch, 0, sizeof(unsigned long long), stream);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "dvr memset: %s", cudaGetErrorString(err));

  void (*k)(const DvrConst) = nullptr;
  switch (a->voxel_type) {
    case VDI_VOXEL_U8: k = dvr_kernel<VDI_VOXEL_U8>; break;
    case VDI_VOXEL_U16: k = dvr_kernel<VDI_VOXEL_U16>; break;
    case VDI_VOXEL_F32: k = dvr_kernel<VDI_VOXEL_F32>; break;
    case VDI_VOXEL_U8 | VDI_VOXEL_CELLS: k = dvr_kernel<VDI_VOXEL_U8 | VDI_VOXEL_CELLS>; break;
    case VDI_VOXEL_U16 | VDI_VOXEL_CELLS: k = dvr_kernel<VDI_VOXEL_U16 | VDI_VOXEL_CELLS>; break;
    case VDI_VOXEL_F32 | VDI_VOXEL_CELLS: k = dvr_kernel<VDI_VOXEL_F32 | VDI_VOXEL_CELLS>; break;
    default: return set_error(VDI_EINVAL, "unknown voxel_type %d", a->voxel_type);
  }
  const size_t smem = sizeof(double4) * (size_t)a->lut_n;
  if (smem > 48 * 1024) {
    err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "dvr smem: %s", cudaGetErrorString(err));
  }
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kDvrThreads, smem);
  if (per_sm < 1) per_sm = 1;
  long long blocks = (long long)sms * per_sm;
  const long long need = (c.n_slots / 32 + (kDvrThreads / 32) - 1) / (kDvrThreads / 32);
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  k<<<(unsigned)blocks, kDvrThreads, smem, stream>>>(c);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "dvr launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
