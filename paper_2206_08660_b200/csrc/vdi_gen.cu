// vdi_gen.cu -- VDI generation on sm_100a.
//
// Semantics: the reference's _generate_kernel (generate.py:276-319), which runs
// per ray the gamma bisection _find_gamma_list (219-273) over front-to-back
// passes _gen_list_pass (89-216) with _emit (53-86), trilinear sampling
// (volume.py:180-205) and LUT classification (volume.py:164-177). Arithmetic is
// f64 in the reference's order (no FMA: built with -fmad=false), f32 rounding
// at the LUT output and at the segment store, exactly as numba does.
//
// B200 structure: the reference's two nested loops (passes x samples) are
// flattened into a per-lane state machine whose every iteration is ONE sample.
// A lane whose ray finishes refills from a warp-uniform pool of ray indices
// (one atomicAdd per 32 rays), so the warp stays converged on the hot sample
// body even though passes per ray are bimodal (1 vs 5-22).
// Ray indices map to 8x4 pixel tiles so a warp's rays start spatially
// coherent. Segments are written straight into the output list during every
// pass; the only case whose result is not the last pass's output (the
// epsilon exit returning the cached high-gamma segments after a later
// low-gamma pass) replays the high pass, which is deterministic.
#include <cstdio>

#include "vdi_common.cuh"
#include "vdi_internal.h"

namespace vdi {

constexpr int kGenThreads = 128;

enum PassMode : int { kCount = 0, kCapped = 1, kRedo = 2 };

struct GenConst {
  VdiGenArgs a;
  double inv_ext[3];  // 1/extent where the extent is a power of two
  int ext_pow2[3];
  double inv_lref;
  int lref_pow2;
  int tiles_x;
  int local_h;
  long long n_slots;  // tiles * 32
  unsigned long long* counter;
};

template <int VT>
struct Voxel;
template <>
struct Voxel<VDI_VOXEL_F32> {
  static __device__ __forceinline__ double get(const void* p, long long i, const float*) {
    return (double)__ldg(reinterpret_cast<const float*>(p) + i);
  }
};
template <>
struct Voxel<VDI_VOXEL_U8> {
  // volume.py:48-50 normalises with an f32 division by 255; the 256 exact
  // quotients live in shared memory.
  static __device__ __forceinline__ double get(const void* p, long long i, const float* tab) {
    return (double)tab[__ldg(reinterpret_cast<const unsigned char*>(p) + i)];
  }
};
template <>
struct Voxel<VDI_VOXEL_U16> {
  static __device__ __forceinline__ double get(const void* p, long long i, const float*) {
    return (double)__fdiv_rn((float)__ldg(reinterpret_cast<const unsigned short*>(p) + i),
                             65535.0f);
  }
};

// volume.py:180-205 _trilinear.
template <int VT>
__device__ __forceinline__ double trilinear(const GenConst& c, const float* tab, double px,
                                            double py, double pz) {
  const int nx = c.a.nx, ny = c.a.ny, nz = c.a.nz;
  const double gx = px * (double)(nx - 1);
  const double gy = py * (double)(ny - 1);
  const double gz = pz * (double)(nz - 1);
  int ix = (int)gx, iy = (int)gy, iz = (int)gz;
  if (ix > nx - 2) ix = nx - 2;
  if (iy > ny - 2) iy = ny - 2;
  if (iz > nz - 2) iz = nz - 2;
  const double fx = gx - ix, fy = gy - iy, fz = gz - iz;
  const long long sy = nx, sz = (long long)nx * ny;
  const long long b = iz * sz + iy * sy + ix;
  const void* v = c.a.volume;
  const double v000 = Voxel<VT>::get(v, b, tab), v001 = Voxel<VT>::get(v, b + 1, tab);
  const double v010 = Voxel<VT>::get(v, b + sy, tab), v011 = Voxel<VT>::get(v, b + sy + 1, tab);
  const double v100 = Voxel<VT>::get(v, b + sz, tab), v101 = Voxel<VT>::get(v, b + sz + 1, tab);
  const double v110 = Voxel<VT>::get(v, b + sz + sy, tab);
  const double v111 = Voxel<VT>::get(v, b + sz + sy + 1, tab);
  const double c00 = v000 * (1 - fx) + v001 * fx;
  const double c10 = v010 * (1 - fx) + v011 * fx;
  const double c01 = v100 * (1 - fx) + v101 * fx;
  const double c11 = v110 * (1 - fx) + v111 * fx;
  const double c0 = c00 * (1 - fy) + c10 * fy;
  const double c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz;
}

// volume.py:164-177 _lut_classify: f64 lerp rounded to f32.
__device__ __forceinline__ float4 classify(const float4* lut, int n, double s) {
  const double x = s * (double)(n - 1);
  if (x <= 0.0) return lut[0];
  if (x >= (double)(n - 1)) return lut[n - 1];
  const int i = (int)x;
  const double f = x - i;
  const float4 l0 = lut[i], l1 = lut[i + 1];
  float4 o;
  o.x = (float)((double)l0.x * (1.0 - f) + (double)l1.x * f);
  o.y = (float)((double)l0.y * (1.0 - f) + (double)l1.y * f);
  o.z = (float)((double)l0.z * (1.0 - f) + (double)l1.z * f);
  o.w = (float)((double)l0.w * (1.0 - f) + (double)l1.w * f);
  return o;
}

struct RayState {
  // ray geometry
  double o[3], d[3], t0, t1;
  int nsteps, k;
  float* seg;  // this list's n_sg*6 floats (list-SoA)
  long long list;
  // current pass (generate.py:97-106)
  double gamma, fr_t, bk_t, mr, mg, mb, acc_r, acc_g, acc_b, acc_a, last_fr_t;
  float prev_back;
  int count, nsamp, active, mode;
  // bisection (generate.py:230-236)
  double low, high, bis_gamma;
  int first, last_n, high_n, passes, buf_is_high, samples;
};

// generate.py:53-86 _emit into the list-SoA slot `count`.
__device__ __forceinline__ void emit(const GenConst& c, RayState& s) {
  const double* pv = c.a.pv;
  const double zf = xform_z(pv, s.o[0] + s.fr_t * s.d[0], s.o[1] + s.fr_t * s.d[1],
                            s.o[2] + s.fr_t * s.d[2]);
  const double zb = xform_z(pv, s.o[0] + s.bk_t * s.d[0], s.o[1] + s.bk_t * s.d[1],
                            s.o[2] + s.bk_t * s.d[2]);
  float f = (float)zf, b = (float)zb;
  if (f < -1.0f) f = -1.0f;
  if (s.count > 0 && f < s.prev_back) f = s.prev_back;
  if (b > 1.0f) b = 1.0f;
  if (b <= f) b = nextafterf(f, 2.0f);
  const float a32 = (float)s.acc_a;
  float r32 = (float)s.acc_r, g32 = (float)s.acc_g, b32 = (float)s.acc_b;
  if (r32 > a32) r32 = a32;
  if (g32 > a32) g32 = a32;
  if (b32 > a32) b32 = a32;
  const int n_sg = c.a.n_sg;
  s.seg[s.count] = f;
  s.seg[n_sg + s.count] = b;
  reinterpret_cast<float4*>(s.seg + 2 * n_sg)[s.count] = make_float4(r32, g32, b32, a32);
  s.prev_back = b;
  s.last_fr_t = s.fr_t;
  s.count += 1;
}

__device__ __forceinline__ void start_pass(RayState& s, double g, int mode) {
  s.gamma = g;
  s.mode = mode;
  s.k = 0;
  s.count = 0;
  s.active = 0;
  s.nsamp = 0;
  s.fr_t = s.bk_t = 0.0;
  s.mr = s.mg = s.mb = 0.0;
  s.acc_r = s.acc_g = s.acc_b = s.acc_a = 0.0;
}

// Zero-fill the unused tail and publish the per-ray outputs
// (generate.py:314-319).
__device__ void finish_ray(const GenConst& c, RayState& s, double g, int n) {
  const int n_sg = c.a.n_sg;
  for (int i = n; i < n_sg; ++i) {
    s.seg[i] = 0.0f;
    s.seg[n_sg + i] = 0.0f;
    reinterpret_cast<float4*>(s.seg + 2 * n_sg)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  c.a.counts[s.list] = n;
  if (c.a.gammas) c.a.gammas[s.list] = g;
  if (c.a.passes) c.a.passes[s.list] = s.passes;
  if (c.a.samples) c.a.samples[s.list] = s.samples;
}

// Top of the bisection loop (generate.py:237-257): either start the next
// measurement pass or leave through the epsilon test. Returns false when the
// ray is finished.
__device__ bool bisect_next(const GenConst& c, RayState& s) {
  if (fabs(s.high - s.low) < c.a.eps) {
    double g;
    if (s.last_n == 0) {
      g = s.low;
    } else {
      g = s.high;
      if (s.high_n >= 0) {
        if (s.buf_is_high) {
          finish_ray(c, s, g, s.high_n);
          return false;
        }
        start_pass(s, g, kRedo);  // regenerate the cached high segments
        return true;
      }
    }
    start_pass(s, g, kCapped);
    return true;
  }
  start_pass(s, s.bis_gamma, kCount);
  return true;
}

// End of a pass with result n (generate.py:248-273). Returns false when the
// ray is finished.
__device__ bool pass_done(const GenConst& c, RayState& s, int n) {
  if (s.mode == kRedo) {
    finish_ray(c, s, s.high, s.high_n);
    return false;
  }
  s.passes += 1;
  if (s.mode == kCapped) {
    finish_ray(c, s, s.gamma, n);
    return false;
  }
  const int n_sg = c.a.n_sg;
  s.last_n = n;
  if (s.first) {
    s.first = 0;
    if (n < n_sg) {
      finish_ray(c, s, s.bis_gamma, n);
      return false;
    }
  }
  if (n > n_sg) {
    s.low = s.bis_gamma;
    s.buf_is_high = 0;
  } else if (n < n_sg - c.a.delta) {
    s.high = s.bis_gamma;
    s.high_n = n;
    s.buf_is_high = 1;
  } else {
    finish_ray(c, s, s.bis_gamma, n);
    return false;
  }
  s.bis_gamma = 0.5 * (s.low + s.high);
  return bisect_next(c, s);
}

// Ray setup (generate.py:282-309). Returns false on a miss.
__device__ bool setup_ray(const GenConst& c, RayState& s, int lx, int gy) {
  pixel_ray(c.a.inv_pv, c.a.eye, lx, gy, c.a.width, c.a.height, s.d);
  s.o[0] = c.a.eye[0];
  s.o[1] = c.a.eye[1];
  s.o[2] = c.a.eye[2];
  double ta, tb, fa, fb;
  if (!clip_aabb(s.o, s.d, c.a.aabb, ta, tb)) return false;
  if (!clip_frustum(c.a.pv, s.o, s.d, fa, fb)) return false;
  const double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb);
  if (t1 <= t0) return false;
  s.t0 = t0;
  s.t1 = t1;
  s.nsteps = (int)ceil((t1 - t0) / c.a.step);
  s.low = 0.0;
  s.high = kSqrt3;
  s.bis_gamma = c.a.gamma_init;
  s.first = 1;
  s.last_n = 1;
  s.high_n = -1;
  s.passes = 0;
  s.buf_is_high = 0;
  s.samples = 0;
  start_pass(s, s.bis_gamma, kCount);
  return true;
}

template <int VT>
__global__ void __launch_bounds__(kGenThreads) gen_kernel(const GenConst c) {
  extern __shared__ float4 s_lut[];
  __shared__ float s_u8[256];
  const int lut_n = c.a.lut_n;
  for (int i = threadIdx.x; i < lut_n; i += blockDim.x)
    s_lut[i] = reinterpret_cast<const float4*>(c.a.lut)[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_u8[i] = __fdiv_rn((float)i, 255.0f);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int n_sg = c.a.n_sg;
  const double step = c.a.step;
  // Warp-uniform ray pool: `pool` is the first index of the current 32-ray
  // chunk, `used` how many of it were handed out.
  long long pool = 0;
  int used = 32;
  bool have = false, done = false;
  RayState s;

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const int n = __popc(need);
      const int rank = __popc(need & ((1u << lane) - 1u));
      const int avail = 32 - used;
      long long fresh = 0;
      if (n > avail) {
        if (lane == 0) fresh = (long long)atomicAdd(c.counter, 32ull);
        fresh = __shfl_sync(0xffffffffu, fresh, 0);
      }
      if ((need >> lane) & 1u) {
        const long long slot = rank < avail ? pool + used + rank : fresh + (rank - avail);
        if (slot >= c.n_slots) {
          done = true;
        } else {
          // 8x4 pixel tiles in row-major tile order
          const long long tile = slot >> 5;
          const int w = (int)(slot & 31);
          const int lx = (int)(tile % c.tiles_x) * kTileW + (w & 7);
          const int ly = (int)(tile / c.tiles_x) * kTileH + (w >> 3);
          if (lx < c.a.width && ly < c.local_h) {
            s.list = (long long)ly * c.a.width + lx;
            s.seg = c.a.segs + s.list * (long long)(n_sg * 6);
            const int gy = band_global_row(ly, c.a.band_rows, c.a.band_stride, c.a.band_offset);
            have = setup_ray(c, s, lx, gy);
            if (!have) {
              s.passes = 0;
              s.samples = 0;
              finish_ray(c, s, 0.0, 0);
            }
          }
        }
      }
      if (n > avail) {
        pool = fresh;
        used = n - avail;
      } else {
        used += n;
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    // ---------------------------------------------------- one sample step
    // (generate.py:111-212)
    int ended = -1;  // >= 0: pass result
    const double ta = s.t0 + (double)s.k * step;
    double tb = ta + step;
    if (tb > s.t1) tb = s.t1;
    if (tb <= ta) {
      ended = 0;
    } else {
      if (s.mode != kRedo) s.samples += 1;
      const double tm = 0.5 * (ta + tb);
      double q[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double num = s.o[a] + tm * s.d[a] - c.a.aabb[a];
        double v = c.ext_pow2[a] ? num * c.inv_ext[a] : num / (c.a.aabb[3 + a] - c.a.aabb[a]);
        if (v < 0.0) v = 0.0;
        else if (v > 1.0) v = 1.0;
        q[a] = v;
      }
      const float4 rgba = classify(s_lut, lut_n, trilinear<VT>(c, s_u8, q[0], q[1], q[2]));
      const double a = (double)rgba.w;
      if (a <= 0.0) {
        if (s.active) {
          emit(c, s);
          s.active = 0;
        }
      } else {
        const double dt = tb - ta;
        const double e = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
        const double om = 1.0 - a;
        const double a_adj = 1.0 - (e == 1.0 ? om : pow(om, e));
        const double sr = (double)rgba.x * a_adj;
        const double sg = (double)rgba.y * a_adj;
        const double sb = (double)rgba.z * a_adj;
        bool merge = false, fresh_seg = false;
        if (!s.active) {
          if (s.count >= n_sg) {
            if (s.mode != kCapped) {
              ended = n_sg + 1;
            } else {
              // reopen the last supersegment (generate.py:151-165)
              s.count -= 1;
              s.fr_t = s.last_fr_t;
              const float4 l = reinterpret_cast<const float4*>(s.seg + 2 * n_sg)[s.count];
              s.acc_r = l.x;
              s.acc_g = l.y;
              s.acc_b = l.z;
              s.acc_a = l.w;
              s.prev_back = s.count > 0 ? s.seg[n_sg + s.count - 1] : 0.0f;
              s.acc_r += (1.0 - s.acc_a) * sr;
              s.acc_g += (1.0 - s.acc_a) * sg;
              s.acc_b += (1.0 - s.acc_a) * sb;
              s.acc_a += (1.0 - s.acc_a) * a_adj;
              s.bk_t = tb;
              s.mr = sr;
              s.mg = sg;
              s.mb = sb;
              s.nsamp = 1;
              s.active = 1;
            }
          } else {
            s.active = 1;
            fresh_seg = true;
          }
        } else {
          const double dr = s.mr - sr, dg = s.mg - sg, db = s.mb - sb;
          const double dist = sqrt(dr * dr + dg * dg + db * db);
          if (dist >= s.gamma) {
            if (s.count + 1 >= n_sg) {
              if (s.mode != kCapped) ended = n_sg + 1;
              else merge = true;
            } else {
              emit(c, s);
              fresh_seg = true;
            }
          } else {
            merge = true;
          }
        }
        if (fresh_seg) {
          s.fr_t = ta;
          s.bk_t = tb;
          s.mr = sr;
          s.mg = sg;
          s.mb = sb;
          s.nsamp = 1;
          s.acc_r = sr;
          s.acc_g = sg;
          s.acc_b = sb;
          s.acc_a = a_adj;
        } else if (merge) {
          s.acc_r += (1.0 - s.acc_a) * sr;
          s.acc_g += (1.0 - s.acc_a) * sg;
          s.acc_b += (1.0 - s.acc_a) * sb;
          s.acc_a += (1.0 - s.acc_a) * a_adj;
          s.bk_t = tb;
          s.nsamp += 1;
          const double inv = 1.0 / (double)s.nsamp;
          s.mr += (sr - s.mr) * inv;
          s.mg += (sg - s.mg) * inv;
          s.mb += (sb - s.mb) * inv;
        }
      }
      if (ended < 0) {
        s.k += 1;
        if (s.k >= s.nsteps) ended = 0;
      }
    }
    if (ended >= 0) {
      int n = ended;
      if (n == 0) {  // natural end or tb <= ta break (generate.py:213-216)
        if (s.active) emit(c, s);
        n = s.count;
      }
      have = pass_done(c, s, n);
    }
  }
}

int gen_launch(const VdiGenArgs* a, cudaStream_t stream) {
  GenConst c;
  c.a = *a;
  for (int i = 0; i < 3; ++i) {
    const double ext = a->aabb[3 + i] - a->aabb[i];
    int e;
    const double m = frexp(ext, &e);
    c.ext_pow2[i] = (m == 0.5);
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
  c.counter = reinterpret_cast<unsigned long long*>(a->workspace);
  if (c.local_h <= 0) return VDI_OK;
  cudaError_t err = cudaMemsetAsync(c.counter, 0, sizeof(unsigned long long), stream);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen memset: %s", cudaGetErrorString(err));

  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(float4) * a->lut_n;
  int per_sm = 0;
  void (*kern)(const GenConst) = nullptr;
  switch (a->voxel_type) {
    case VDI_VOXEL_U8: kern = gen_kernel<VDI_VOXEL_U8>; break;
    case VDI_VOXEL_U16: kern = gen_kernel<VDI_VOXEL_U16>; break;
    case VDI_VOXEL_F32: kern = gen_kernel<VDI_VOXEL_F32>; break;
    default: return set_error(VDI_EINVAL, "bad voxel_type %d", a->voxel_type);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGenThreads, smem);
  if (per_sm < 1) per_sm = 1;
  // persistent grid: every resident slot, but no more warps than 32-ray chunks
  long long blocks = (long long)sms * per_sm;
  const long long need = (c.n_slots / 32 + (kGenThreads / 32) - 1) / (kGenThreads / 32);
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kGenThreads, smem, stream>>>(c);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
