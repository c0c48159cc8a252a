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
//
// Sample cache: every bisection pass walks the same samples with a different
// gamma, so each lane keeps the classified RGBA (f32, exactly what
// _lut_classify returned) of its ray in an HBM scratch row; passes 2..k replay
// it instead of re-sampling the volume (16 B per replayed sample instead of 8
// voxel gathers + ~100 f64 ops). Transparent runs are stored run-length coded
// (head entry holds the run length), so replay crosses empty space in O(1).
// Replay is bit-identical by construction: the same f32 values enter the same
// f64 expressions.
//
// Exact shortcuts (same bits as the reference, fewer instructions):
//   * dist >= gamma  <=>  d2 >= thr(gamma), with thr the smallest double whose
//     correctly rounded sqrt is >= gamma (sqrt_rn is monotone), computed once
//     per pass;
//   * 1.0 / nsamp is read from a table of host-identical IEEE quotients;
//   * x / extent is x * (1 / extent) when the extent is a power of two.
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
  const double* inv_tab;  // inv_tab[n] == 1.0 / n, bit-exact (host IEEE division)
  int inv_n;
  int max_steps;          // per-lane sample-cache capacity
  float4* cache;          // [lanes][max_steps] classified samples
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
  float* seg;  // this list's list-SoA block
  long long list;
  // current pass (generate.py:97-106)
  double gamma, thr, fr_t, bk_t, mr, mg, mb, acc_r, acc_g, acc_b, acc_a, last_fr_t;
  float prev_back;
  int count, nsamp, active, mode;
  // bisection (generate.py:230-236)
  double low, high, bis_gamma;
  int first, last_n, high_n, passes, buf_is_high, samples;
  // sample cache frontier and the open transparent run at the frontier
  int cached, run_head;
};

// Smallest double s >= 0 with sqrt_rn(s) >= g, so that sqrt_rn(d2) >= g <=>
// d2 >= s for every d2 >= 0 (sqrt_rn is monotone non-decreasing).
__device__ double split_threshold(double g) {
  if (!(g > 0.0)) return -INFINITY;
  double s = g * g;
  while (sqrt(s) < g) s = nextafter(s, INFINITY);
  while (true) {
    const double p = nextafter(s, 0.0);
    if (sqrt(p) >= g) s = p;
    else break;
  }
  return s;
}

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
  s.seg[front_off(n_sg) + s.count] = f;
  s.seg[back_off(n_sg) + s.count] = b;
  reinterpret_cast<float4*>(s.seg)[s.count] = make_float4(r32, g32, b32, a32);
  s.prev_back = b;
  s.last_fr_t = s.fr_t;
  s.count += 1;
}

__device__ __forceinline__ void start_pass(RayState& s, double g, int mode) {
  s.gamma = g;
  s.thr = split_threshold(g);
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
    s.seg[front_off(n_sg) + i] = 0.0f;
    s.seg[back_off(n_sg) + i] = 0.0f;
    reinterpret_cast<float4*>(s.seg)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
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
  s.cached = 0;
  s.run_head = -1;
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
  const int max_steps = c.max_steps;
  float4* const cache =
      c.cache + ((long long)blockIdx.x * blockDim.x + threadIdx.x) * (long long)max_steps;
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
            s.seg = c.a.segs + s.list * (long long)list_stride(n_sg);
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

    // ------------------------------------- one sample (generate.py:111-212)
    int ended = -1;  // >= 0: pass result
    const double ta = s.t0 + (double)s.k * step;
    double tb = ta + step;
    if (tb > s.t1) tb = s.t1;
    if (tb <= ta) {
      ended = 0;
    } else {
      float4 rgba;
      int run = 1;
      if (s.k < s.cached) {
        rgba = cache[s.k];  // replay
        if (rgba.w <= 0.0f) {
          run = __float_as_int(rgba.x);
          if (run < 1) run = 1;
          if (run > s.cached - s.k) run = s.cached - s.k;
        }
      } else {
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
        rgba = classify(s_lut, lut_n, trilinear<VT>(c, s_u8, q[0], q[1], q[2]));
        if (s.k < max_steps) {
          if (rgba.w <= 0.0f) {
            cache[s.k] = make_float4(__int_as_float(1), 0.f, 0.f, 0.f);
            if (s.run_head < 0) s.run_head = s.k;
          } else {
            cache[s.k] = rgba;
            if (s.run_head >= 0) {  // close the transparent run
              cache[s.run_head].x = __int_as_float(s.k - s.run_head);
              s.run_head = -1;
            }
          }
          s.cached = s.k + 1;
        }
      }
      if (s.mode != kRedo) s.samples += run;
      if (rgba.w <= 0.0f) {
        // fully transparent: closes the open supersegment (generate.py:135-142)
        if (s.active) {
          emit(c, s);
          s.active = 0;
        }
        s.k += run;
      } else {
        const double a = (double)rgba.w;
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
              const float4 l = reinterpret_cast<const float4*>(s.seg)[s.count];
              s.acc_r = l.x;
              s.acc_g = l.y;
              s.acc_b = l.z;
              s.acc_a = l.w;
              s.prev_back = s.count > 0 ? s.seg[back_off(n_sg) + s.count - 1] : 0.0f;
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
          if (dr * dr + dg * dg + db * db >= s.thr) {  // == sqrt(...) >= gamma
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
          const double inv =
              s.nsamp < c.inv_n ? __ldg(c.inv_tab + s.nsamp) : 1.0 / (double)s.nsamp;
          s.mr += (sr - s.mr) * inv;
          s.mg += (sg - s.mg) * inv;
          s.mb += (sb - s.mb) * inv;
        }
        if (ended < 0) s.k += 1;
      }
      if (ended < 0 && s.k >= s.nsteps) ended = 0;
    }
    if (ended >= 0) {
      int n = ended;
      if (n == 0) {  // natural end or tb <= ta break (generate.py:213-216)
        if (s.active) emit(c, s);
        n = s.count;
      }
      // publish the open run's current length before any replay
      if (s.run_head >= 0) cache[s.run_head].x = __int_as_float(s.cached - s.run_head);
      have = pass_done(c, s, n);
    }
  }
}

__global__ void fill_inv_kernel(double* tab, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tab[i] = i > 0 ? 1.0 / (double)i : 0.0;
}

struct GenPlan {
  void (*kern)(const GenConst);
  long long blocks;
  int max_steps, inv_n;
  size_t off_inv, off_cache, total;
  size_t smem;
};

static int plan_gen(const VdiGenArgs* a, GenPlan& p, long long n_slots) {
  switch (a->voxel_type) {
    case VDI_VOXEL_U8: p.kern = gen_kernel<VDI_VOXEL_U8>; break;
    case VDI_VOXEL_U16: p.kern = gen_kernel<VDI_VOXEL_U16>; break;
    case VDI_VOXEL_F32: p.kern = gen_kernel<VDI_VOXEL_F32>; break;
    default: return set_error(VDI_EINVAL, "bad voxel_type %d", a->voxel_type);
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p.smem = sizeof(float4) * a->lut_n;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.kern, kGenThreads, p.smem);
  if (per_sm < 1) per_sm = 1;
  // persistent grid: every resident slot, but no more warps than 32-ray chunks
  p.blocks = (long long)sms * per_sm;
  const long long need = (n_slots / 32 + (kGenThreads / 32) - 1) / (kGenThreads / 32);
  if (n_slots >= 0 && p.blocks > need) p.blocks = need;
  if (p.blocks < 1) p.blocks = 1;
  // no ray has more samples than the box diagonal allows
  const double ex = a->aabb[3] - a->aabb[0], ey = a->aabb[4] - a->aabb[1],
               ez = a->aabb[5] - a->aabb[2];
  const double diag = sqrt(ex * ex + ey * ey + ez * ez);
  const double ms = ceil(diag / a->step) + 4.0;
  p.max_steps = ms > 1e7 ? 10000000 : (int)ms;
  p.inv_n = p.max_steps + 2;
  p.off_inv = 256;
  p.off_cache = (p.off_inv + sizeof(double) * p.inv_n + 255) & ~(size_t)255;
  p.total = p.off_cache + sizeof(float4) * (size_t)p.max_steps * (size_t)p.blocks * kGenThreads;
  return VDI_OK;
}

size_t gen_workspace_bytes(const VdiGenArgs* a) {
  GenPlan p;
  if (plan_gen(a, p, -1) != VDI_OK) return 0;
  return p.total;
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
  if (c.local_h <= 0) return VDI_OK;
  GenPlan p;
  int rc = plan_gen(a, p, c.n_slots);
  if (rc != VDI_OK) return rc;
  if (a->workspace_bytes < p.total)
    return set_error(VDI_EINVAL, "workspace too small: %zu < %zu bytes", a->workspace_bytes,
                     p.total);
  char* ws = reinterpret_cast<char*>(a->workspace);
  c.counter = reinterpret_cast<unsigned long long*>(ws);
  c.inv_tab = reinterpret_cast<const double*>(ws + p.off_inv);
  c.inv_n = p.inv_n;
  c.max_steps = p.max_steps;
  c.cache = reinterpret_cast<float4*>(ws + p.off_cache);
  cudaError_t err = cudaMemsetAsync(c.counter, 0, sizeof(unsigned long long), stream);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen memset: %s", cudaGetErrorString(err));
  fill_inv_kernel<<<(p.inv_n + 255) / 256, 256, 0, stream>>>(
      reinterpret_cast<double*>(ws + p.off_inv), p.inv_n);
  p.kern<<<(unsigned)p.blocks, kGenThreads, p.smem, stream>>>(c);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
