/*
 * vdi_oracle.c -- TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * (vdikit 0.1.0, /root/reference/pkg/src/vdikit) VDI generation and VDI
 * raycasting kernels, used as the parity checker for the B200 path and as
 * the CPU baseline ("port") in bench.py. Nothing in the product path may
 * link or call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg do.
 *
 * Arithmetic contract: R is numba-compiled f64 scalar
 * code with no FMA contraction, glibc pow/sqrt, f32 inputs promoted to f64,
 * and f32 rounding exactly at the LUT output and at the VDI store. This file
 * is compiled with -O2 -ffp-contract=off -fno-fast-math and evaluates every
 * expression in R's order, so on x86-64 it reproduces R bit for bit.
 * Pinned against the golden vectors in tests/golden/ (made from R itself by
 * tests/golden/make_golden.py).
 *
 * Segment layout here is R's: segs[(ly*W + lx)*n_sg*6 + k*6 + c],
 * c = front, back, r, g, b, a (vdi.py:3-7, 23-24).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SQRT3 1.7320508075688772 /* math.sqrt(3.0), generate.py:25 */

/* ---------------------------------------------------------------- geometry */

/* _geom.py:12-19 ndc_of; world_of (22-25) is the same with the inverse. */
static inline void xform(const double* m, double x, double y, double z,
                         double* ox, double* oy, double* oz) {
  double hx = m[0] * x + m[1] * y + m[2] * z + m[3];
  double hy = m[4] * x + m[5] * y + m[6] * z + m[7];
  double hz = m[8] * x + m[9] * y + m[10] * z + m[11];
  double hw = m[12] * x + m[13] * y + m[14] * z + m[15];
  *ox = hx / hw;
  *oy = hy / hw;
  *oz = hz / hw;
}

/* _geom.py:28-54 clip_aabb */
static inline int clip_aabb(double ox, double oy, double oz, double dx,
                            double dy, double dz, const double* bb,
                            double* t0o, double* t1o) {
  double t0 = -INFINITY, t1 = INFINITY;
  const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
  for (int a = 0; a < 3; ++a) {
    double lo = bb[a], hi = bb[3 + a];
    if (fabs(d[a]) < 1e-300) {
      if (o[a] < lo || o[a] > hi) return 0;
    } else {
      double ta = (lo - o[a]) / d[a];
      double tb = (hi - o[a]) / d[a];
      if (ta > tb) { double s = ta; ta = tb; tb = s; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    }
  }
  if (t1 < t0) return 0;
  *t0o = t0;
  *t1o = t1;
  return 1;
}

/* _geom.py:57-104 clip_frustum: homogeneous 7 half-space clip. */
static inline int clip_frustum(const double* m, double ox, double oy, double oz,
                               double dx, double dy, double dz, double* t0o,
                               double* t1o) {
  double p0x = m[0] * ox + m[1] * oy + m[2] * oz + m[3];
  double p0y = m[4] * ox + m[5] * oy + m[6] * oz + m[7];
  double p0z = m[8] * ox + m[9] * oy + m[10] * oz + m[11];
  double p0w = m[12] * ox + m[13] * oy + m[14] * oz + m[15];
  double pdx = m[0] * dx + m[1] * dy + m[2] * dz;
  double pdy = m[4] * dx + m[5] * dy + m[6] * dz;
  double pdz = m[8] * dx + m[9] * dy + m[10] * dz;
  double pdw = m[12] * dx + m[13] * dy + m[14] * dz;
  double cs[7] = {p0w, p0w - p0x, p0w + p0x, p0w - p0y,
                  p0w + p0y, p0w - p0z, p0w + p0z};
  double ds[7] = {pdw, pdw - pdx, pdw + pdx, pdw - pdy,
                  pdw + pdy, pdw - pdz, pdw + pdz};
  double t0 = -INFINITY, t1 = INFINITY;
  for (int i = 0; i < 7; ++i) {
    double c = cs[i], d = ds[i];
    if (fabs(d) < 1e-300) {
      if (c < 0) return 0;
    } else {
      double t = -c / d;
      if (d > 0) {
        if (t > t0) t0 = t;
      } else {
        if (t < t1) t1 = t;
      }
    }
  }
  if (t1 < t0) return 0;
  *t0o = t0;
  *t1o = t1;
  return 1;
}

static inline double dmax(double a, double b) { return b > a ? b : a; }
static inline double dmin(double a, double b) { return b < a ? b : a; }

/* Per-pixel eye ray (generate.py:282-294 / raycast.py:286-297). */
static inline void pixel_ray(const double* inv_pv, const double* eye, int col,
                             int row, int w, int h, double* d) {
  double ndcx = 2.0 * (col + 0.5) / w - 1.0;
  double ndcy = 2.0 * (row + 0.5) / h - 1.0;
  double wx, wy, wz;
  xform(inv_pv, ndcx, ndcy, -1.0, &wx, &wy, &wz);
  double dx = wx - eye[0], dy = wy - eye[1], dz = wz - eye[2];
  double norm = sqrt(dx * dx + dy * dy + dz * dz);
  d[0] = dx / norm;
  d[1] = dy / norm;
  d[2] = dz / norm;
}

/* --------------------------------------------------------------- sampler */

/* The sampled volume: R's f32 `normalized` array, or raw u8 voxels that
 * are normalised exactly as volume.py:48-50 does (f32 v / 255) -- the same
 * values, without a 4 B/voxel host copy (large configs). */
typedef struct {
  const float* f32;
  const uint8_t* u8;
} vox_t;

static float g_u8tab[256];
static void init_u8tab(void) {
  for (int i = 0; i < 256; ++i) g_u8tab[i] = (float)i / 255.0f;
}

static inline double vox(vox_t v, int64_t i) {
  return v.u8 ? (double)g_u8tab[v.u8[i]] : (double)v.f32[i];
}

/* volume.py:180-205 _trilinear on the normalized volume. */
static inline double trilinear(vox_t vol, int nx, int ny, int nz,
                               double px, double py, double pz) {
  double gx = px * (double)(nx - 1);
  double gy = py * (double)(ny - 1);
  double gz = pz * (double)(nz - 1);
  int64_t ix = (int64_t)gx, iy = (int64_t)gy, iz = (int64_t)gz;
  if (ix > nx - 2) ix = nx - 2;
  if (iy > ny - 2) iy = ny - 2;
  if (iz > nz - 2) iz = nz - 2;
  double fx = gx - (double)ix, fy = gy - (double)iy, fz = gz - (double)iz;
  const int64_t sx = 1, sy = nx, sz = (int64_t)nx * ny;
  const int64_t b = iz * sz + iy * sy + ix;
  double c00 = vox(vol, b) * (1 - fx) + vox(vol, b + sx) * fx;
  double c10 = vox(vol, b + sy) * (1 - fx) + vox(vol, b + sy + sx) * fx;
  double c01 = vox(vol, b + sz) * (1 - fx) + vox(vol, b + sz + sx) * fx;
  double c11 = vox(vol, b + sz + sy) * (1 - fx) + vox(vol, b + sz + sy + sx) * fx;
  double c0 = c00 * (1 - fy) + c10 * fy;
  double c1 = c01 * (1 - fy) + c11 * fy;
  return c0 * (1 - fz) + c1 * fz;
}

/* volume.py:164-177 _lut_classify: lerp in f64, rounded to f32. */
static inline void lut_classify(const float* lut, int n, double s, float* out) {
  double x = s * (double)(n - 1);
  if (x <= 0.0) {
    memcpy(out, lut, 16);
    return;
  }
  if (x >= (double)(n - 1)) {
    memcpy(out, lut + 4 * (n - 1), 16);
    return;
  }
  int64_t i = (int64_t)x;
  double f = x - (double)i;
  for (int c = 0; c < 4; ++c)
    out[c] = (float)((double)lut[4 * i + c] * (1.0 - f) +
                     (double)lut[4 * (i + 1) + c] * f);
}

/* ------------------------------------------------------------- generation */

typedef struct {
  vox_t vol;
  int nx, ny, nz;
  const float* lut;
  int lut_n;
  const double* pv;
  double ox, oy, oz, dx, dy, dz;
  const double* bb;
  double t0, t1, step, lref;
  int n_sg;
  int64_t* samples; /* executed-sample counter (loop iterations) */
} ray_ctx;

/* generate.py:53-86 _emit */
static inline int emit(const ray_ctx* r, float* out_seg, double* tseg, int count,
                       double fr_t, double bk_t, double acc_r, double acc_g,
                       double acc_b, double acc_a) {
  double tmp, zf, zb;
  xform(r->pv, r->ox + fr_t * r->dx, r->oy + fr_t * r->dy, r->oz + fr_t * r->dz,
        &tmp, &tmp, &zf);
  xform(r->pv, r->ox + bk_t * r->dx, r->oy + bk_t * r->dy, r->oz + bk_t * r->dz,
        &tmp, &tmp, &zb);
  float f = (float)zf, b = (float)zb;
  if (f < -1.0f) f = -1.0f;
  if (count > 0 && f < out_seg[(count - 1) * 6 + 1]) f = out_seg[(count - 1) * 6 + 1];
  if (b > 1.0f) b = 1.0f;
  if (b <= f) b = nextafterf(f, 2.0f);
  float a32 = (float)acc_a, r32 = (float)acc_r, g32 = (float)acc_g,
        b32 = (float)acc_b;
  if (r32 > a32) r32 = a32;
  if (g32 > a32) g32 = a32;
  if (b32 > a32) b32 = a32;
  float* o = out_seg + count * 6;
  o[0] = f;
  o[1] = b;
  o[2] = r32;
  o[3] = g32;
  o[4] = b32;
  o[5] = a32;
  tseg[count * 2 + 0] = fr_t;
  tseg[count * 2 + 1] = bk_t;
  return count + 1;
}

/* generate.py:89-216 _gen_list_pass. Returns the count (n_sg+1 = exceeded). */
static int gen_list_pass(const ray_ctx* r, double gamma, int capped,
                         float* out_seg, double* tseg) {
  const int n_sg = r->n_sg;
  int count = 0, active = 0, nsamp = 0;
  double fr_t = 0.0, bk_t = 0.0, mr = 0.0, mg = 0.0, mb = 0.0;
  double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
  const double ex = r->bb[3] - r->bb[0], ey = r->bb[4] - r->bb[1],
               ez = r->bb[5] - r->bb[2];
  const int64_t nsteps = (int64_t)ceil((r->t1 - r->t0) / r->step);
  for (int64_t k = 0; k < nsteps; ++k) {
    double ta = r->t0 + (double)k * r->step;
    double tb = ta + r->step;
    if (tb > r->t1) tb = r->t1;
    if (tb <= ta) break;
    if (r->samples) ++*r->samples;
    double tm = 0.5 * (ta + tb);
    double qx = (r->ox + tm * r->dx - r->bb[0]) / ex;
    double qy = (r->oy + tm * r->dy - r->bb[1]) / ey;
    double qz = (r->oz + tm * r->dz - r->bb[2]) / ez;
    if (qx < 0.0) qx = 0.0; else if (qx > 1.0) qx = 1.0;
    if (qy < 0.0) qy = 0.0; else if (qy > 1.0) qy = 1.0;
    if (qz < 0.0) qz = 0.0; else if (qz > 1.0) qz = 1.0;
    float rgba[4];
    lut_classify(r->lut, r->lut_n, trilinear(r->vol, r->nx, r->ny, r->nz, qx, qy, qz), rgba);
    double a = (double)rgba[3];
    if (a <= 0.0) {
      if (active) {
        count = emit(r, out_seg, tseg, count, fr_t, bk_t, acc_r, acc_g, acc_b, acc_a);
        active = 0;
      }
      continue;
    }
    double a_adj = 1.0 - pow(1.0 - a, (tb - ta) / r->lref);
    double sr = (double)rgba[0] * a_adj;
    double sg = (double)rgba[1] * a_adj;
    double sb = (double)rgba[2] * a_adj;
    if (!active) {
      if (count >= n_sg) {
        if (!capped) return n_sg + 1;
        /* reopen the last supersegment and smear into it (151-165) */
        count -= 1;
        fr_t = tseg[count * 2];
        acc_r = out_seg[count * 6 + 2];
        acc_g = out_seg[count * 6 + 3];
        acc_b = out_seg[count * 6 + 4];
        acc_a = out_seg[count * 6 + 5];
        acc_r += (1.0 - acc_a) * sr;
        acc_g += (1.0 - acc_a) * sg;
        acc_b += (1.0 - acc_a) * sb;
        acc_a += (1.0 - acc_a) * a_adj;
        bk_t = tb;
        mr = sr; mg = sg; mb = sb;
        nsamp = 1;
        active = 1;
      } else {
        active = 1;
        fr_t = ta;
        bk_t = tb;
        mr = sr; mg = sg; mb = sb;
        nsamp = 1;
        acc_r = sr; acc_g = sg; acc_b = sb; acc_a = a_adj;
      }
    } else {
      double dr = mr - sr, dg = mg - sg, db = mb - sb;
      double dist = sqrt(dr * dr + dg * dg + db * db);
      if (dist >= gamma) {
        if (count + 1 >= n_sg) {
          if (!capped) return n_sg + 1;
          acc_r += (1.0 - acc_a) * sr;
          acc_g += (1.0 - acc_a) * sg;
          acc_b += (1.0 - acc_a) * sb;
          acc_a += (1.0 - acc_a) * a_adj;
          bk_t = tb;
          nsamp += 1;
          double inv = 1.0 / (double)nsamp;
          mr += (sr - mr) * inv;
          mg += (sg - mg) * inv;
          mb += (sb - mb) * inv;
        } else {
          count = emit(r, out_seg, tseg, count, fr_t, bk_t, acc_r, acc_g, acc_b, acc_a);
          fr_t = ta;
          bk_t = tb;
          mr = sr; mg = sg; mb = sb;
          nsamp = 1;
          acc_r = sr; acc_g = sg; acc_b = sb; acc_a = a_adj;
        }
      } else {
        acc_r += (1.0 - acc_a) * sr;
        acc_g += (1.0 - acc_a) * sg;
        acc_b += (1.0 - acc_a) * sb;
        acc_a += (1.0 - acc_a) * a_adj;
        bk_t = tb;
        nsamp += 1;
        double inv = 1.0 / (double)nsamp;
        mr += (sr - mr) * inv;
        mg += (sg - mg) * inv;
        mb += (sb - mb) * inv;
      }
    }
  }
  if (active)
    count = emit(r, out_seg, tseg, count, fr_t, bk_t, acc_r, acc_g, acc_b, acc_a);
  return count;
}

/* Analysis hook (tools/bisect_predict.py): when set, every counting pass of
 * ray oidx appends (gamma, n) at g_trace[oidx * 48 + 2 * pass]. */
static double* g_trace = NULL;
static _Thread_local int64_t g_trace_ray = -1;

static inline void trace_pass(int pass, double gamma, int n) {
  if (g_trace && g_trace_ray >= 0 && pass < 24) {
    g_trace[g_trace_ray * 48 + 2 * pass] = gamma;
    g_trace[g_trace_ray * 48 + 2 * pass + 1] = (double)n;
  }
}

/* generate.py:219-273 _find_gamma_list (Alg. 1 as R implements it). */
static void find_gamma_list(const ray_ctx* r, int delta, double eps,
                            double gamma_init, float* out_seg, double* tseg,
                            float* high_seg, double* g_out, int* n_out,
                            int* passes_out) {
  const int n_sg = r->n_sg;
  double low = 0.0, high = SQRT3, gamma = gamma_init;
  int first = 1, last_n = 1, high_n = -1, passes = 0;
  for (;;) {
    if (fabs(high - low) < eps) {
      double g;
      if (last_n == 0) {
        g = low;
      } else {
        g = high;
        if (high_n >= 0) {
          memcpy(out_seg, high_seg, sizeof(float) * 6 * high_n);
          *g_out = g; *n_out = high_n; *passes_out = passes;
          return;
        }
      }
      int n = gen_list_pass(r, g, 1, out_seg, tseg);
      passes += 1;
      *g_out = g; *n_out = n; *passes_out = passes;
      return;
    }
    int n = gen_list_pass(r, gamma, 0, out_seg, tseg);
    trace_pass(passes, gamma, n);
    passes += 1;
    last_n = n;
    if (first) {
      first = 0;
      if (n < n_sg) {
        *g_out = gamma; *n_out = n; *passes_out = passes;
        return;
      }
    }
    if (n > n_sg) {
      low = gamma;
    } else if (n < n_sg - delta) {
      high = gamma;
      high_n = n;
      memcpy(high_seg, out_seg, sizeof(float) * 6 * n);
    } else {
      *g_out = gamma; *n_out = n; *passes_out = passes;
      return;
    }
    gamma = 0.5 * (low + high);
  }
}

/* One ray of generate.py:281-319 (_generate_kernel body). */
static void generate_ray(vox_t vol, int nx, int ny, int nz,
                         const float* lut, int lut_n, const double* pv,
                         const double* inv_pv, const double* eye,
                         const double* bb, int width, int height, int n_sg,
                         int delta, double eps, double gamma_init, double step,
                         double lref, int64_t idx, int64_t oidx, int32_t* counts, float* segs,
                         double* gammas, int32_t* passes, int64_t* samples,
                         double* tseg, float* high_seg) {
  int ly = (int)(idx / width), lx = (int)(idx % width);
  double d[3];
  pixel_ray(inv_pv, eye, lx, ly, width, height, d);
  idx = oidx; /* outputs go to oidx (compact row sets) */
  g_trace_ray = oidx;
  float* out_seg = segs + idx * (int64_t)n_sg * 6;
  counts[idx] = 0;
  if (gammas) gammas[idx] = 0.0;
  if (passes) passes[idx] = 0;
  if (samples) samples[idx] = 0;
  double ta, tb, fa, fb;
  int ok = clip_aabb(eye[0], eye[1], eye[2], d[0], d[1], d[2], bb, &ta, &tb) &&
           clip_frustum(pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], &fa, &fb);
  int n = 0;
  if (ok) {
    double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb);
    if (t1 > t0) {
      int64_t nsamp = 0;
      ray_ctx r = {vol, nx, ny, nz, lut, lut_n, pv, eye[0], eye[1], eye[2],
                   d[0], d[1], d[2], bb, t0, t1, step, lref, n_sg, &nsamp};
      double g;
      int p;
      find_gamma_list(&r, delta, eps, gamma_init, out_seg, tseg, high_seg, &g, &n, &p);
      counts[idx] = n;
      if (gammas) gammas[idx] = g;
      if (passes) passes[idx] = p;
      if (samples) samples[idx] = nsamp;
    }
  }
  /* zero-fill the unused tail (generate.py:317-319); misses stay zero. */
  memset(out_seg + (int64_t)n * 6, 0, sizeof(float) * 6 * (n_sg - n));
}

/* _generate_kernel over all rays, or only over the listed rows (bounded CPU
 * baseline samples). Output arrays are full (H, W) sized either way. */
static int generate_all(vox_t vol, int nx, int ny, int nz, const float* lut,
                  int lut_n, const double* pv, const double* inv_pv,
                  const double* eye, const double* bb, int width, int height,
                  int n_sg, int delta, double eps, double gamma_init,
                  double step, double lref, const int32_t* rows, int n_rows,
                  int nthreads, int32_t* counts, float* segs, double* gammas,
                  int32_t* passes, int64_t* samples) {
  /* n_rows < 0: the -n_rows listed rows, outputs packed as (n_rows, W) */
  const int compact = n_rows < 0;
  if (compact) n_rows = -n_rows;
  int64_t total = rows ? (int64_t)n_rows * width : (int64_t)width * height;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel
  {
    double* tseg = (double*)malloc(sizeof(double) * 2 * n_sg);
    float* high_seg = (float*)malloc(sizeof(float) * 6 * n_sg);
#pragma omp for schedule(dynamic, 64)
    for (int64_t j = 0; j < total; ++j) {
      int64_t idx = rows ? (int64_t)rows[j / width] * width + j % width : j;
      generate_ray(vol, nx, ny, nz, lut, lut_n, pv, inv_pv, eye, bb, width,
                   height, n_sg, delta, eps, gamma_init, step, lref, idx,
                   compact ? j : idx, counts, segs, gammas, passes, samples, tseg, high_seg);
    }
    free(tseg);
    free(high_seg);
  }
  return 0;
}

int vdio_generate(const float* vol, int nx, int ny, int nz, const float* lut,
                  int lut_n, const double* pv, const double* inv_pv,
                  const double* eye, const double* bb, int width, int height,
                  int n_sg, int delta, double eps, double gamma_init,
                  double step, double lref, const int32_t* rows, int n_rows,
                  int nthreads, int32_t* counts, float* segs, double* gammas,
                  int32_t* passes, int64_t* samples) {
  vox_t v = {vol, NULL};
  return generate_all(v, nx, ny, nz, lut, lut_n, pv, inv_pv, eye, bb, width, height, n_sg,
                      delta, eps, gamma_init, step, lref, rows, n_rows, nthreads, counts, segs,
                      gammas, passes, samples);
}

/* Analysis hook: the no-split trajectory of one ray (a counting pass with
 * gamma = +inf): the number of visible runs V and max over samples of the
 * d^2 the split test compares, so that every gamma with sqrt(d2max) < gamma
 * has no split and n(gamma) = V (or the abort at run n_sg + 1). */
static void nosplit_ray(const ray_ctx* r, int64_t* v_out, double* d2_out) {
  int active = 0, nsamp = 0;
  int64_t runs = 0;
  double mr = 0, mg = 0, mb = 0, d2max = 0.0;
  const double ex = r->bb[3] - r->bb[0], ey = r->bb[4] - r->bb[1], ez = r->bb[5] - r->bb[2];
  const int64_t nsteps = (int64_t)ceil((r->t1 - r->t0) / r->step);
  for (int64_t k = 0; k < nsteps; ++k) {
    double ta = r->t0 + (double)k * r->step;
    double tb = ta + r->step;
    if (tb > r->t1) tb = r->t1;
    if (tb <= ta) break;
    double tm = 0.5 * (ta + tb);
    double qx = (r->ox + tm * r->dx - r->bb[0]) / ex;
    double qy = (r->oy + tm * r->dy - r->bb[1]) / ey;
    double qz = (r->oz + tm * r->dz - r->bb[2]) / ez;
    if (qx < 0.0) qx = 0.0; else if (qx > 1.0) qx = 1.0;
    if (qy < 0.0) qy = 0.0; else if (qy > 1.0) qy = 1.0;
    if (qz < 0.0) qz = 0.0; else if (qz > 1.0) qz = 1.0;
    float rgba[4];
    lut_classify(r->lut, r->lut_n, trilinear(r->vol, r->nx, r->ny, r->nz, qx, qy, qz), rgba);
    double a = (double)rgba[3];
    if (a <= 0.0) { active = 0; continue; }
    double a_adj = 1.0 - pow(1.0 - a, (tb - ta) / r->lref);
    double sr = (double)rgba[0] * a_adj, sg = (double)rgba[1] * a_adj, sb = (double)rgba[2] * a_adj;
    if (!active) { active = 1; runs += 1; mr = sr; mg = sg; mb = sb; nsamp = 1; continue; }
    double dr = mr - sr, dg = mg - sg, db = mb - sb;
    double d2 = dr * dr + dg * dg + db * db;
    if (d2 > d2max) d2max = d2;
    nsamp += 1;
    double inv = 1.0 / (double)nsamp;
    mr += (sr - mr) * inv; mg += (sg - mg) * inv; mb += (sb - mb) * inv;
  }
  *v_out = runs;
  *d2_out = d2max;
}

int vdio_nosplit(const float* vol, int nx, int ny, int nz, const float* lut, int lut_n,
                 const double* pv, const double* inv_pv, const double* eye, const double* bb,
                 int width, int height, double step, double lref, const int32_t* rows,
                 int n_rows, int64_t* v_out, double* d2_out) {
  int64_t total = (int64_t)n_rows * width;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < total; ++j) {
    int64_t idx = (int64_t)rows[j / width] * width + j % width;
    int ly = (int)(idx / width), lx = (int)(idx % width);
    double d[3];
    pixel_ray(inv_pv, eye, lx, ly, width, height, d);
    v_out[j] = -1; d2_out[j] = -1.0;
    double ta, tb, fa, fb;
    if (!(clip_aabb(eye[0], eye[1], eye[2], d[0], d[1], d[2], bb, &ta, &tb) &&
          clip_frustum(pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], &fa, &fb))) continue;
    double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb);
    if (!(t1 > t0)) continue;
    vox_t v = {vol, NULL};
    ray_ctx r = {v, nx, ny, nz, lut, lut_n, pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], bb,
                 t0, t1, step, lref, 0, NULL};
    nosplit_ray(&r, v_out + j, d2_out + j);
  }
  return 0;
}

/* vdio_generate with the (gamma, n) trace of every counting pass recorded
 * into trace[(ray) * 48 + 2 * pass] (analysis only, not thread-safe across
 * concurrent calls). */
int vdio_generate_trace(const float* vol, int nx, int ny, int nz, const float* lut,
                        int lut_n, const double* pv, const double* inv_pv,
                        const double* eye, const double* bb, int width, int height,
                        int n_sg, int delta, double eps, double gamma_init,
                        double step, double lref, const int32_t* rows, int n_rows,
                        int nthreads, int32_t* counts, float* segs, double* gammas,
                        int32_t* passes, int64_t* samples, double* trace) {
  g_trace = trace;
  vox_t v = {vol, NULL};
  const int rc = generate_all(v, nx, ny, nz, lut, lut_n, pv, inv_pv, eye, bb, width, height,
                              n_sg, delta, eps, gamma_init, step, lref, rows, n_rows, nthreads,
                              counts, segs, gammas, passes, samples);
  g_trace = NULL;
  return rc;
}

/* The same over raw u8 voxels (normalised on the fly, volume.py:48-50). */
int vdio_generate_u8(const uint8_t* vol, int nx, int ny, int nz, const float* lut,
                     int lut_n, const double* pv, const double* inv_pv,
                     const double* eye, const double* bb, int width, int height,
                     int n_sg, int delta, double eps, double gamma_init,
                     double step, double lref, const int32_t* rows, int n_rows,
                     int nthreads, int32_t* counts, float* segs, double* gammas,
                     int32_t* passes, int64_t* samples) {
  init_u8tab();
  vox_t v = {NULL, vol};
  return generate_all(v, nx, ny, nz, lut, lut_n, pv, inv_pv, eye, bb, width, height, n_sg,
                      delta, eps, gamma_init, step, lref, rows, n_rows, nthreads, counts, segs,
                      gammas, passes, samples);
}

/* generate.py:322-346 _accumulate_grid (serial, as in R). */
int vdio_accumulate_grid(const int32_t* counts, const float* segs, int width,
                         int height, int n_sg, int gx, int gy, int gz,
                         double near, double far, double proj_a, double proj_b,
                         uint32_t* gcounts) {
  for (int64_t ly = 0; ly < height; ++ly) {
    int64_t cy0 = (ly * gy) / height;
    int64_t cy1 = ((ly + 1) * gy - 1) / height;
    for (int64_t lx = 0; lx < width; ++lx) {
      int n = counts[ly * width + lx];
      if (n == 0) continue;
      int64_t cx0 = (lx * gx) / width;
      int64_t cx1 = ((lx + 1) * gx - 1) / width;
      const float* s = segs + (ly * width + lx) * (int64_t)n_sg * 6;
      for (int k = 0; k < n; ++k) {
        double zf = s[k * 6], zb = s[k * 6 + 1];
        double d0 = proj_b / (proj_a - zf);
        double d1 = proj_b / (proj_a - zb);
        int64_t k0 = (int64_t)floor((d0 - near) / (far - near) * gz);
        int64_t k1 = (int64_t)floor((d1 - near) / (far - near) * gz);
        if (k0 < 0) k0 = 0;
        if (k0 > gz - 1) k0 = gz - 1;
        if (k1 < 0) k1 = 0;
        if (k1 > gz - 1) k1 = gz - 1;
        for (int64_t cz = k0; cz <= k1; ++cz)
          for (int64_t cy = cy0; cy <= cy1; ++cy)
            for (int64_t cx = cx0; cx <= cx1; ++cx)
              gcounts[(cz * gy + cy) * gx + cx] += 1;
      }
    }
  }
  return 0;
}

/* -------------------------------------------------------------- rendering */

/* raycast.py:51-62 _bins: smallest j in [start, stop] with backs[j] >= d. */
static inline int64_t bins(const float* backs, int stride, double d,
                           int64_t start, int64_t stop) {
  int64_t lo = start, hi = stop;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if ((double)backs[mid * stride] >= d) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

/* raycast.py:65-76 _bins_front: largest j in [start, stop] with fronts[j] <= d. */
static inline int64_t bins_front(const float* fronts, int stride, double d,
                                 int64_t start, int64_t stop) {
  int64_t lo = start, hi = stop;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if ((double)fronts[mid * stride] <= d) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

#define FR(i) ((double)fronts[(i) * (int64_t)stride])
#define BK(i) ((double)backs[(i) * (int64_t)stride])

/* raycast.py:79-141 _find_first (Alg. 2 + R's guards + reverse branch).
 * Returns the index or -1; *seed receives the reusable seed. */
static int64_t find_first(const float* fronts, const float* backs, int stride,
                          int64_t count, double d_entry, double d_exit,
                          int64_t p, int64_t* seed) {
  if (count == 0) {
    *seed = p;
    return -1;
  }
  int64_t index;
  if (d_entry <= d_exit) {
    index = -1;
    int64_t bs_start = -1, bs_end = -1;
    if (p < 0) {
      bs_start = 0;
      bs_end = count - 1;
    } else {
      double b1 = p < count ? BK(p) : INFINITY;
      double b0 = (0 <= p - 1 && p - 1 < count) ? BK(p - 1) : -INFINITY;
      int interval = (b1 >= d_entry ? 1 : 0) + (b0 >= d_entry ? 1 : 0);
      if (interval == 0) {
        bs_start = p + 1;
        bs_end = count - 1;
      } else if (interval == 2) {
        bs_start = 0;
        bs_end = p - 1;
      } else {
        if (p < count) {
          index = p;
        } else {
          bs_start = 0;
          bs_end = count - 1;
        }
      }
    }
    if (bs_end != -1) {
      if (bs_start > bs_end) {
        index = bs_start < 0 ? 0 : bs_start;
        if (index > count - 1) index = count - 1;
      } else {
        index = bins(backs, stride, d_entry, bs_start,
                     bs_end < count - 1 ? bs_end : count - 1);
      }
    }
    /* index == -1 here only if p >= 0 took the interval==1 path with
     * p < count, so it is always valid; numba would wrap a -1 index. */
    *seed = index;
    if (BK(index) < d_entry) return -1;
    if (FR(index) > d_exit) return -1;
    return index;
  }
  if (p < 0) {
    index = bins_front(fronts, stride, d_entry, 0, count - 1);
  } else {
    double f1 = p < count ? FR(p) : INFINITY;
    double f0 = (0 <= p + 1 && p + 1 < count) ? FR(p + 1) : INFINITY;
    if (p < count && f1 <= d_entry && f0 > d_entry) {
      index = p;
    } else if (f1 > d_entry) {
      index = bins_front(fronts, stride, d_entry, 0, p - 1 > 0 ? p - 1 : 0);
    } else {
      index = bins_front(fronts, stride, d_entry,
                         p + 1 < count - 1 ? p + 1 : count - 1, count - 1);
    }
  }
  if (index > count - 1) index = count - 1;
  *seed = index;
  if (FR(index) > d_entry) return -1;
  if (BK(index) < d_exit) return -1;
  return index;
}
#undef FR
#undef BK

int64_t vdio_find_first(const float* fronts, const float* backs, int64_t count,
                        double d_entry, double d_exit, int64_t p,
                        int64_t* seed) {
  return find_first(fronts, backs, 1, count, d_entry, d_exit, p, seed);
}

static inline int64_t floor_i(double x) { return (int64_t)floor(x); }
static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

/* One pixel of raycast.py:283-456. */
static void render_pixel(const float* segs, const int32_t* counts, int vdi_w,
                         int vdi_h, int n_sg, const double* gen_pv,
                         const double* gen_inv_pv, const double* bb,
                         const double* new_inv_pv, const double* eye, int out_w,
                         int out_h, int use_ess, const uint32_t* gcounts,
                         int gx, int gy, int gz, double near, double far,
                         double proj_a, double proj_b, double early_term,
                         const double* bg, int64_t idx, double* img,
                         int64_t* lists_vis, int64_t* segs_int,
                         int64_t* lists_searched) {
  int row = (int)(idx / out_w), col = (int)(idx % out_w);
  double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
  int64_t nvis = 0, nint = 0, nsearch = 0;
  double d[3];
  pixel_ray(new_inv_pv, eye, col, row, out_w, out_h, d);
  const double npx = eye[0], npy = eye[1], npz = eye[2];
  double ta, tb, fa, fb, t0 = 0.0, t1 = 0.0;
  int ok = 0;
  if (clip_aabb(npx, npy, npz, d[0], d[1], d[2], bb, &ta, &tb)) {
    if (clip_frustum(gen_pv, npx, npy, npz, d[0], d[1], d[2], &fa, &fb)) {
      t0 = dmax(dmax(ta, fa), 0.0);
      t1 = dmin(tb, fb);
      if (t1 > t0) ok = 1;
    }
  }
  if (ok) {
    double a0x, a0y, a0z, a1x, a1y, a1z;
    xform(gen_pv, npx + t0 * d[0], npy + t0 * d[1], npz + t0 * d[2], &a0x, &a0y, &a0z);
    xform(gen_pv, npx + t1 * d[0], npy + t1 * d[1], npz + t1 * d[2], &a1x, &a1y, &a1z);
    double cdx = a1x - a0x, cdy = a1y - a0y, cdz = a1z - a0z;
    int64_t cx = clampi(floor_i((a0x + 1.0) * vdi_w / 2.0), 0, vdi_w - 1);
    int64_t cy = clampi(floor_i((a0y + 1.0) * vdi_h / 2.0), 0, vdi_h - 1);
    int step_x = cdx > 0 ? 1 : (cdx < 0 ? -1 : 0);
    int step_y = cdy > 0 ? 1 : (cdy < 0 ? -1 : 0);
    double t_max_x, t_delta_x, t_max_y, t_delta_y;
    if (step_x != 0) {
      double bx = -1.0 + 2.0 * (double)(cx + (step_x > 0 ? 1 : 0)) / vdi_w;
      t_max_x = (bx - a0x) / cdx;
      t_delta_x = (2.0 / vdi_w) / fabs(cdx);
    } else {
      t_max_x = INFINITY;
      t_delta_x = INFINITY;
    }
    if (step_y != 0) {
      double by = -1.0 + 2.0 * (double)(cy + (step_y > 0 ? 1 : 0)) / vdi_h;
      t_max_y = (by - a0y) / cdy;
      t_delta_y = (2.0 / vdi_h) / fabs(cdy);
    } else {
      t_max_y = INFINITY;
      t_delta_y = INFINITY;
    }
    int64_t p = -1;
    double s_cur = 0.0;
    int done = 0;
    const int64_t max_iter = (int64_t)vdi_w + vdi_h + 4;
    for (int64_t it = 0; it < max_iter; ++it) {
      double s_exit = dmin(dmin(t_max_x, t_max_y), 1.0);
      if (s_exit < s_cur) s_exit = s_cur;
      double d_entry = a0z + s_cur * cdz;
      double d_exit = a0z + s_exit * cdz;
      nvis += 1;
      const int64_t lidx = cy * vdi_w + cx;
      int64_t count = counts[lidx];
      int search = count > 0;
      if (search && use_ess) {
        /* raycast.py:353-372 + _grid_cell_range 258-272 */
        double x_a = a0x + s_cur * cdx, y_a = a0y + s_cur * cdy;
        double x_b = a0x + s_exit * cdx, y_b = a0y + s_exit * cdy;
        double dep_a = proj_b / (proj_a - d_entry);
        double dep_b = proj_b / (proj_a - d_exit);
        int64_t cgx0 = clampi(floor_i((dmin(x_a, x_b) + 1.0) * gx / 2.0), 0, gx - 1);
        int64_t cgx1 = clampi(floor_i((dmax(x_a, x_b) + 1.0) * gx / 2.0), 0, gx - 1);
        int64_t cgy0 = clampi(floor_i((dmin(y_a, y_b) + 1.0) * gy / 2.0), 0, gy - 1);
        int64_t cgy1 = clampi(floor_i((dmax(y_a, y_b) + 1.0) * gy / 2.0), 0, gy - 1);
        int64_t cz0 = clampi(floor_i((dmin(dep_a, dep_b) - near) / (far - near) * gz), 0, gz - 1);
        int64_t cz1 = clampi(floor_i((dmax(dep_a, dep_b) - near) / (far - near) * gz), 0, gz - 1);
        int empty = 1;
        for (int64_t cz = cz0; cz <= cz1 && empty; ++cz)
          for (int64_t cgy = cgy0; cgy <= cgy1; ++cgy)
            for (int64_t cgx = cgx0; cgx <= cgx1; ++cgx)
              if (gcounts[(cz * gy + cgy) * gx + cgx] > 0) empty = 0;
        if (empty) search = 0;
      }
      if (search) {
        nsearch += 1;
        const float* ls = segs + lidx * (int64_t)n_sg * 6;
        const float* fronts = ls;
        const float* backs = ls + 1;
        int64_t seed;
        int64_t j = find_first(fronts, backs, 6, count, d_entry, d_exit, p, &seed);
        p = seed;
        if (j >= 0) {
          int fwd = d_entry <= d_exit;
          double zlo = dmin(d_entry, d_exit), zhi = dmax(d_entry, d_exit);
          double xc = -1.0 + 2.0 * (cx + 0.5) / vdi_w;
          double yc = -1.0 + 2.0 * (cy + 0.5) / vdi_h;
          int64_t k = j;
          while (0 <= k && k < count) {
            double fk = ls[k * 6], bk = ls[k * 6 + 1];
            double ilo = dmax(fk, zlo), ihi = dmin(bk, zhi);
            if (ilo > ihi) break;
            double s_a, s_b;
            if (fabs(cdz) < 1e-12) {
              s_a = s_cur;
              s_b = s_exit;
            } else {
              s_a = (ilo - a0z) / cdz;
              s_b = (ihi - a0z) / cdz;
              if (s_a > s_b) { double t = s_a; s_a = s_b; s_b = t; }
              if (s_a < s_cur) s_a = s_cur;
              if (s_b > s_exit) s_b = s_exit;
            }
            double w0x, w0y, w0z, w1x, w1y, w1z;
            xform(gen_inv_pv, a0x + s_a * cdx, a0y + s_a * cdy, a0z + s_a * cdz, &w0x, &w0y, &w0z);
            xform(gen_inv_pv, a0x + s_b * cdx, a0y + s_b * cdy, a0z + s_b * cdz, &w1x, &w1y, &w1z);
            double ddx = w1x - w0x, ddy = w1y - w0y, ddz = w1z - w0z;
            double l = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
            double wfx, wfy, wfz, wbx, wby, wbz;
            xform(gen_inv_pv, xc, yc, fk, &wfx, &wfy, &wfz);
            xform(gen_inv_pv, xc, yc, bk, &wbx, &wby, &wbz);
            double tx = wbx - wfx, ty = wby - wfy, tz = wbz - wfz;
            double thick = sqrt(tx * tx + ty * ty + tz * tz);
            double alpha = ls[k * 6 + 5];
            if (alpha > 0.0 && thick > 0.0) {
              double a_t = 1.0 - pow(1.0 - alpha, l / thick);
              double scale = a_t / alpha;
              double w = 1.0 - acc_a;
              acc_r += w * (double)ls[k * 6 + 2] * scale;
              acc_g += w * (double)ls[k * 6 + 3] * scale;
              acc_b += w * (double)ls[k * 6 + 4] * scale;
              acc_a += w * a_t;
            }
            nint += 1;
            p = k;
            if (acc_a >= early_term) {
              done = 1;
              break;
            }
            k += fwd ? 1 : -1;
          }
        }
      }
      if (done || acc_a >= early_term) break;
      if (s_exit >= 1.0) break;
      if (t_max_x <= t_max_y) {
        cx += step_x;
        s_cur = t_max_x;
        t_max_x += t_delta_x;
      } else {
        cy += step_y;
        s_cur = t_max_y;
        t_max_y += t_delta_y;
      }
      if (cx < 0 || cx >= vdi_w || cy < 0 || cy >= vdi_h) break;
    }
  }
  double w = 1.0 - acc_a;
  double* o = img + idx * 4;
  o[0] = acc_r + w * bg[0] * bg[3];
  o[1] = acc_g + w * bg[1] * bg[3];
  o[2] = acc_b + w * bg[2] * bg[3];
  o[3] = acc_a + w * bg[3];
  if (lists_vis) lists_vis[idx] = nvis;
  if (segs_int) segs_int[idx] = nint;
  if (lists_searched) lists_searched[idx] = nsearch;
}

int vdio_render(const float* segs, const int32_t* counts, int vdi_w, int vdi_h,
                int n_sg, const double* gen_pv, const double* gen_inv_pv,
                const double* bb, const double* new_inv_pv, const double* eye,
                int out_w, int out_h, int use_ess, const uint32_t* gcounts,
                int gx, int gy, int gz, double near, double far, double proj_a,
                double proj_b, double early_term, const double* bg,
                const int32_t* rows, int n_rows, int nthreads, double* img,
                int64_t* lists_vis, int64_t* segs_int,
                int64_t* lists_searched) {
  int64_t total = rows ? (int64_t)n_rows * out_w : (int64_t)out_w * out_h;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < total; ++j) {
    int64_t idx = rows ? (int64_t)rows[j / out_w] * out_w + j % out_w : j;
    render_pixel(segs, counts, vdi_w, vdi_h, n_sg, gen_pv, gen_inv_pv, bb,
                 new_inv_pv, eye, out_w, out_h, use_ess, gcounts, gx, gy, gz,
                 near, far, proj_a, proj_b, early_term, bg, idx, img,
                 lists_vis, segs_int, lists_searched);
  }
  return 0;
}

/* ------------------------------------------------------------------- DVR */

/* One pixel of dvr.py:21-89 _dvr_kernel: the generation ray and sampler
 * (same clip, midpoint sample, opacity length normalisation), composited
 * front to back with early termination. */
static void dvr_pixel(vox_t vol, int nx, int ny, int nz, const float* lut,
                      int lut_n, const double* pv, const double* inv_pv,
                      const double* eye, const double* bb, int width, int height,
                      double step, double lref, double early_term, const double* bg,
                      int64_t idx, double* img, int64_t* samples) {
  const int row = (int)(idx / width), col = (int)(idx % width);
  const double ex = bb[3] - bb[0], ey = bb[4] - bb[1], ez = bb[5] - bb[2];
  double d[3];
  pixel_ray(inv_pv, eye, col, row, width, height, d); /* dvr.py:28-40 */
  double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
  int64_t nexec = 0;
  double ta, tb, fa, fb;
  if (clip_aabb(eye[0], eye[1], eye[2], d[0], d[1], d[2], bb, &ta, &tb) &&
      clip_frustum(pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], &fa, &fb)) {
    const double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb); /* 47-48 */
    if (t1 > t0) {
      const int64_t nsteps = (int64_t)ceil((t1 - t0) / step);
      for (int64_t k = 0; k < nsteps; ++k) { /* dvr.py:51-83 */
        const double sa = t0 + (double)k * step;
        double sb = sa + step;
        if (sb > t1) sb = t1;
        if (sb <= sa) break;
        ++nexec;
        const double tm = 0.5 * (sa + sb);
        double qx = (eye[0] + tm * d[0] - bb[0]) / ex;
        double qy = (eye[1] + tm * d[1] - bb[1]) / ey;
        double qz = (eye[2] + tm * d[2] - bb[2]) / ez;
        qx = dmin(dmax(qx, 0.0), 1.0);
        qy = dmin(dmax(qy, 0.0), 1.0);
        qz = dmin(dmax(qz, 0.0), 1.0);
        float rgba[4];
        lut_classify(lut, lut_n, trilinear(vol, nx, ny, nz, qx, qy, qz), rgba);
        const double a = (double)rgba[3];
        if (a <= 0.0) continue;
        const double a_adj = 1.0 - pow(1.0 - a, (sb - sa) / lref);
        const double w = 1.0 - acc_a;
        acc_r += w * (double)rgba[0] * a_adj;
        acc_g += w * (double)rgba[1] * a_adj;
        acc_b += w * (double)rgba[2] * a_adj;
        acc_a += w * a_adj;
        if (acc_a >= early_term) break;
      }
    }
  }
  const double w = 1.0 - acc_a; /* dvr.py:84-89 */
  double* o = img + idx * 4;
  o[0] = acc_r + w * bg[0] * bg[3];
  o[1] = acc_g + w * bg[1] * bg[3];
  o[2] = acc_b + w * bg[2] * bg[3];
  o[3] = acc_a + w * bg[3];
  if (samples) samples[idx] = nexec;
}

/* dvr.py:21-89 over all pixels, or only over the listed rows. */
int vdio_dvr(const float* vol, int nx, int ny, int nz, const float* lut, int lut_n,
             const double* pv, const double* inv_pv, const double* eye,
             const double* bb, int width, int height, double step, double lref,
             double early_term, const double* bg, const int32_t* rows, int n_rows,
             int nthreads, double* img, int64_t* samples) {
  vox_t v = {vol, NULL};
  int64_t total = rows ? (int64_t)n_rows * width : (int64_t)width * height;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < total; ++j) {
    int64_t idx = rows ? (int64_t)rows[j / width] * width + j % width : j;
    dvr_pixel(v, nx, ny, nz, lut, lut_n, pv, inv_pv, eye, bb, width, height, step,
              lref, early_term, bg, idx, img, samples);
  }
  return 0;
}

/* --------------------------------------------------------------- preview */

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

static inline double sq(double x) { return x * x; } /* numba x ** 2 == x * x */

/* One pixel of preview.py:49-213 _preview_kernel: chord breakpoints at grid
 * cell boundaries (sorted, as np.sort), round(d_r * len * count) point
 * samples per non-empty cell, each taking the colour of the supersegment
 * containing it (R's _find_first with d_entry == d_exit) with opacity from
 * the distance to the previous sample. `brks` is caller scratch of
 * gx + gy + gz + 2 doubles. Returns the samples planned for this pixel. */
static int64_t preview_pixel(const float* segs, const int32_t* counts, int vdi_w,
                             int vdi_h, int n_sg, const double* gen_pv,
                             const double* gen_inv_pv, const double* bb,
                             const double* new_inv_pv, const double* eye, int out_w,
                             int out_h, const uint32_t* gcounts, int gx, int gy, int gz,
                             double near, double far, double proj_a, double proj_b,
                             double d_r, double early_term, const double* bg,
                             int64_t idx, double* img, int64_t* cell_samples,
                             double* brks) {
  const int row = (int)(idx / out_w), col = (int)(idx % out_w);
  double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
  int64_t total = 0;
  double d[3];
  pixel_ray(new_inv_pv, eye, col, row, out_w, out_h, d); /* 60-69 */
  double ta, tb, fa, fb, t0 = 0.0, t1 = 0.0;
  int ok = 0;
  if (clip_aabb(eye[0], eye[1], eye[2], d[0], d[1], d[2], bb, &ta, &tb) &&
      clip_frustum(gen_pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], &fa, &fb)) {
    t0 = dmax(dmax(ta, fa), 0.0);
    t1 = dmin(tb, fb);
    ok = t1 > t0;
  }
  if (ok) {
    double a0x, a0y, a0z, a1x, a1y, a1z;
    xform(gen_pv, eye[0] + t0 * d[0], eye[1] + t0 * d[1], eye[2] + t0 * d[2], &a0x, &a0y, &a0z);
    xform(gen_pv, eye[0] + t1 * d[0], eye[1] + t1 * d[1], eye[2] + t1 * d[2], &a1x, &a1y, &a1z);
    const double cdx = a1x - a0x, cdy = a1y - a0y, cdz = a1z - a0z;
    int nb = 0; /* 94-121 */
    brks[nb++] = 0.0;
    brks[nb++] = 1.0;
    if (fabs(cdx) > 1e-14)
      for (int i = 1; i < gx; ++i) {
        const double s = (-1.0 + 2.0 * i / gx - a0x) / cdx;
        if (0.0 < s && s < 1.0) brks[nb++] = s;
      }
    if (fabs(cdy) > 1e-14)
      for (int i = 1; i < gy; ++i) {
        const double s = (-1.0 + 2.0 * i / gy - a0y) / cdy;
        if (0.0 < s && s < 1.0) brks[nb++] = s;
      }
    if (fabs(cdz) > 1e-14)
      for (int i = 1; i < gz; ++i) {
        const double dep = near + (far - near) * i / gz;
        const double zb = proj_a - proj_b / dep;
        const double s = (zb - a0z) / cdz;
        if (0.0 < s && s < 1.0) brks[nb++] = s;
      }
    qsort(brks, (size_t)nb, sizeof(double), cmp_double); /* 122 */
    double prev_x, prev_y, prev_z;
    xform(gen_inv_pv, a0x, a0y, a0z, &prev_x, &prev_y, &prev_z); /* 125 */
    int64_t p = -1;
    int done = 0;
    for (int bi = 0; bi < nb - 1 && !done; ++bi) { /* 128-210 */
      const double s_a = brks[bi], s_b = brks[bi + 1];
      if (s_b - s_a < 1e-15) continue;
      const double sm = 0.5 * (s_a + s_b);
      const double mx = a0x + sm * cdx, my = a0y + sm * cdy, mz = a0z + sm * cdz;
      const int64_t cgx = clampi(floor_i((mx + 1.0) * gx / 2.0), 0, gx - 1);
      const int64_t cgy = clampi(floor_i((my + 1.0) * gy / 2.0), 0, gy - 1);
      const double mdep = proj_b / (proj_a - mz);
      const int64_t cgz = clampi(floor_i((mdep - near) / (far - near) * gz), 0, gz - 1);
      const int64_t cell = (cgz * gy + cgy) * gx + cgx;
      const uint32_t cnt = gcounts[cell];
      if (cnt == 0) continue;
      double w0x, w0y, w0z, w1x, w1y, w1z;
      xform(gen_inv_pv, a0x + s_a * cdx, a0y + s_a * cdy, a0z + s_a * cdz, &w0x, &w0y, &w0z);
      xform(gen_inv_pv, a0x + s_b * cdx, a0y + s_b * cdy, a0z + s_b * cdz, &w1x, &w1y, &w1z);
      const double seg_len = sqrt(sq(w1x - w0x) + sq(w1y - w0y) + sq(w1z - w0z));
      const int64_t n = (int64_t)floor(d_r * seg_len * (double)cnt + 0.5);
      if (n <= 0) continue;
      if (cell_samples) {
#pragma omp atomic
        cell_samples[cell] += n;
      }
      total += n;
      for (int64_t i = 0; i < n; ++i) {
        const double sf = s_a + ((double)i + 0.5) / (double)n * (s_b - s_a);
        const double sx = a0x + sf * cdx, sy = a0y + sf * cdy, sz = a0z + sf * cdz;
        double swx, swy, swz;
        xform(gen_inv_pv, sx, sy, sz, &swx, &swy, &swz);
        const double dist = sqrt(sq(swx - prev_x) + sq(swy - prev_y) + sq(swz - prev_z));
        prev_x = swx;
        prev_y = swy;
        prev_z = swz;
        const int64_t lx = clampi(floor_i((sx + 1.0) * vdi_w / 2.0), 0, vdi_w - 1);
        const int64_t ly = clampi(floor_i((sy + 1.0) * vdi_h / 2.0), 0, vdi_h - 1);
        const int64_t lc = counts[ly * vdi_w + lx];
        if (lc == 0) continue;
        const float* ls = segs + (ly * vdi_w + lx) * (int64_t)n_sg * 6;
        int64_t seed;
        const int64_t j = find_first(ls, ls + 1, 6, lc, sz, sz, p, &seed);
        p = seed;
        if (j < 0) continue;
        const float alpha = ls[j * 6 + 5];
        if (alpha <= 0.0f) continue;
        const double xc = -1.0 + 2.0 * (lx + 0.5) / vdi_w;
        const double yc = -1.0 + 2.0 * (ly + 0.5) / vdi_h;
        double wfx, wfy, wfz, wbx, wby, wbz;
        xform(gen_inv_pv, xc, yc, (double)ls[j * 6], &wfx, &wfy, &wfz);
        xform(gen_inv_pv, xc, yc, (double)ls[j * 6 + 1], &wbx, &wby, &wbz);
        const double thick = sqrt(sq(wbx - wfx) + sq(wby - wfy) + sq(wbz - wfz));
        if (thick <= 0.0) continue;
        const double a_t = 1.0 - pow(1.0 - (double)alpha, dist / thick);
        const double scale = a_t / (double)alpha;
        const double w = 1.0 - acc_a;
        acc_r += w * (double)ls[j * 6 + 2] * scale;
        acc_g += w * (double)ls[j * 6 + 3] * scale;
        acc_b += w * (double)ls[j * 6 + 4] * scale;
        acc_a += w * a_t;
        if (acc_a >= early_term) {
          done = 1;
          break;
        }
      }
    }
  }
  const double w = 1.0 - acc_a; /* 207-211 */
  double* o = img + idx * 4;
  o[0] = acc_r + w * bg[0] * bg[3];
  o[1] = acc_g + w * bg[1] * bg[3];
  o[2] = acc_b + w * bg[2] * bg[3];
  o[3] = acc_a + w * bg[3];
  return total;
}

/* preview.py:49-213 over all pixels (R runs it serially; pixels are
 * independent and cell_samples is an integer sum, so the order is free).
 * Returns the total planned samples. */
int64_t vdio_preview(const float* segs, const int32_t* counts, int vdi_w, int vdi_h,
                     int n_sg, const double* gen_pv, const double* gen_inv_pv,
                     const double* bb, const double* new_inv_pv, const double* eye,
                     int out_w, int out_h, const uint32_t* gcounts, int gx, int gy,
                     int gz, double near, double far, double proj_a, double proj_b,
                     double d_r, double early_term, const double* bg, int nthreads,
                     double* img, int64_t* cell_samples) {
  int64_t total = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel reduction(+ : total)
  {
    double* brks = (double*)malloc(sizeof(double) * (size_t)(gx + gy + gz + 2));
#pragma omp for schedule(dynamic, 16)
    for (int64_t j = 0; j < (int64_t)out_w * out_h; ++j)
      total += preview_pixel(segs, counts, vdi_w, vdi_h, n_sg, gen_pv, gen_inv_pv, bb,
                             new_inv_pv, eye, out_w, out_h, gcounts, gx, gy, gz, near, far,
                             proj_a, proj_b, d_r, early_term, bg, j, img, cell_samples, brks);
    free(brks);
  }
  return total;
}

/* ------------------------------------------------------------------- LZ4 */

/* lz4.py:13-17 */
#define LZ4_HASH_LOG 16
#define LZ4_MIN_MATCH 4
#define LZ4_LAST_LITERALS 5
#define LZ4_MFLIMIT 12

static inline uint32_t lz4_read32(const uint8_t* s, int64_t i) { /* lz4.py:34-38 */
  return (uint32_t)s[i] | ((uint32_t)s[i + 1] << 8) | ((uint32_t)s[i + 2] << 16) |
         ((uint32_t)s[i + 3] << 24);
}

static inline uint32_t lz4_hash32(uint32_t v) { /* lz4.py:28-31 */
  return ((v * 2654435761u) >> (32 - LZ4_HASH_LOG)) & ((1u << LZ4_HASH_LOG) - 1u);
}

static inline int64_t lz4_write_length(uint8_t* dst, int64_t o, int64_t len) { /* 41-48 */
  while (len >= 255) {
    dst[o++] = 255;
    len -= 255;
  }
  dst[o++] = (uint8_t)len;
  return o;
}

/* lz4.py:51-114 _compress_kernel: the reference's greedy single-probe
 * parse. dst must hold n + n / 255 + 16 bytes. Returns the block length. */
int64_t vdio_lz4_compress(const uint8_t* src, int64_t n, uint8_t* dst) {
  if (n == 0) return 0;
  int64_t* table = (int64_t*)malloc(sizeof(int64_t) << LZ4_HASH_LOG);
  for (int64_t k = 0; k < (1 << LZ4_HASH_LOG); ++k) table[k] = -1;
  int64_t o = 0, anchor = 0, i = 0;
  const int64_t limit = n - LZ4_MFLIMIT;
  while (i < limit) {
    const uint32_t h = lz4_hash32(lz4_read32(src, i));
    const int64_t cand = table[h];
    table[h] = i;
    if (cand >= 0 && i - cand <= 65535 && lz4_read32(src, cand) == lz4_read32(src, i)) {
      int64_t mlen = LZ4_MIN_MATCH;
      const int64_t mmax = n - LZ4_LAST_LITERALS - i;
      while (mlen < mmax && src[cand + mlen] == src[i + mlen]) ++mlen;
      const int64_t lit = i - anchor;
      const int64_t tok = o++;
      const int64_t lcode = lit >= 15 ? 15 : lit;
      if (lit >= 15) o = lz4_write_length(dst, o, lit - 15);
      memcpy(dst + o, src + anchor, (size_t)lit);
      o += lit;
      const int64_t off = i - cand;
      dst[o] = (uint8_t)(off & 0xFF);
      dst[o + 1] = (uint8_t)((off >> 8) & 0xFF);
      o += 2;
      const int64_t mcode = mlen - LZ4_MIN_MATCH;
      if (mcode >= 15) {
        dst[tok] = (uint8_t)((lcode << 4) | 15);
        o = lz4_write_length(dst, o, mcode - 15);
      } else {
        dst[tok] = (uint8_t)((lcode << 4) | mcode);
      }
      i += mlen;
      anchor = i;
      if (i < limit) table[lz4_hash32(lz4_read32(src, i - 2))] = i - 2;
    } else {
      ++i;
    }
  }
  const int64_t lit = n - anchor; /* final literal run (102-113) */
  const int64_t tok = o++;
  if (lit >= 15) {
    dst[tok] = 15 << 4;
    o = lz4_write_length(dst, o, lit - 15);
  } else {
    dst[tok] = (uint8_t)(lit << 4);
  }
  memcpy(dst + o, src + anchor, (size_t)lit);
  o += lit;
  free(table);
  return o;
}

/* lz4.py:117-168 _decompress_kernel: bytes written, or -1 on malformed input. */
int64_t vdio_lz4_decompress(const uint8_t* src, int64_t n, uint8_t* dst, int64_t out_n) {
  int64_t si = 0, di = 0;
  while (si < n) {
    const int token = src[si++];
    int64_t lit = token >> 4;
    if (lit == 15) {
      for (;;) {
        if (si >= n) return -1;
        const int b = src[si++];
        lit += b;
        if (b != 255) break;
      }
    }
    if (si + lit > n || di + lit > out_n) return -1;
    memcpy(dst + di, src + si, (size_t)lit);
    si += lit;
    di += lit;
    if (si >= n) break; /* last sequence has no match part */
    if (si + 2 > n) return -1;
    const int64_t off = (int64_t)src[si] | ((int64_t)src[si + 1] << 8);
    si += 2;
    if (off == 0 || off > di) return -1;
    int64_t mlen = token & 15;
    if (mlen == 15) {
      for (;;) {
        if (si >= n) return -1;
        const int b = src[si++];
        mlen += b;
        if (b != 255) break;
      }
    }
    mlen += LZ4_MIN_MATCH;
    if (di + mlen > out_n) return -1;
    const int64_t mp = di - off;
    for (int64_t k = 0; k < mlen; ++k) dst[di + k] = dst[mp + k]; /* overlapping copy */
    di += mlen;
  }
  return di;
}

int vdio_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
