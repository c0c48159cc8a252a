/* Offline study (not product, not the oracle): how many bisection passes of
 * R's _find_gamma_list could be answered from an earlier pass of the same ray
 * without re-walking the samples? A counting pass at gamma decides "split"
 * at each visible sample of an open segment iff d2 >= thr(gamma); two gammas
 * follow the same trajectory (same count, same abort position) iff no split
 * decision differs, i.e. iff thr(gamma') <= u2 (the smallest split d2) when
 * gamma' > gamma, or thr(gamma') > v2 (the largest non-split d2) when
 * gamma' < gamma. Built on the oracle's sampler (#include), run by
 * tools/study/bisect_intervals.py. */
#include "../../oracle/vdi_oracle.c"

static double thr_of(double g) { /* smallest s >= 0 with sqrt(s) >= g */
  if (!(g > 0.0)) return -INFINITY;
  double s = g * g;
  while (sqrt(s) < g) s = nextafter(s, INFINITY);
  for (;;) {
    double p = nextafter(s, 0.0);
    if (sqrt(p) >= g) s = p; else break;
  }
  return s;
}

/* a counting pass (gen_list_pass, capped = 0) that also reports u2 / v2 */
static int count_pass(const ray_ctx* r, double gamma, double* u2, double* v2) {
  const int n_sg = r->n_sg;
  const double thr = thr_of(gamma);
  int count = 0, active = 0, nsamp = 0;
  double mr = 0.0, mg = 0.0, mb = 0.0;
  *u2 = INFINITY;
  *v2 = -INFINITY;
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
    if (a <= 0.0) {
      if (active) { count++; active = 0; }
      continue;
    }
    double a_adj = 1.0 - pow(1.0 - a, (tb - ta) / r->lref);
    double sr = (double)rgba[0] * a_adj, sg = (double)rgba[1] * a_adj, sb = (double)rgba[2] * a_adj;
    if (!active) {
      if (count >= n_sg) return n_sg + 1;
      active = 1; mr = sr; mg = sg; mb = sb; nsamp = 1;
    } else {
      double dr = mr - sr, dg = mg - sg, db = mb - sb;
      double d2 = dr * dr + dg * dg + db * db;
      if (d2 >= thr) {
        if (d2 < *u2) *u2 = d2;
        if (count + 1 >= n_sg) return n_sg + 1;
        count++; mr = sr; mg = sg; mb = sb; nsamp = 1;
      } else {
        if (d2 > *v2) *v2 = d2;
        nsamp += 1;
        double inv = 1.0 / (double)nsamp;
        mr += (sr - mr) * inv; mg += (sg - mg) * inv; mb += (sb - mb) * inv;
      }
    }
  }
  if (active) count++;
  return count;
}

/* Per ray of rows[]: replays R's bisection with count_pass; a pass whose gamma
 * lies in the identical-trajectory interval of an earlier pass is "free".
 * out[0] passes (R semantics, counting passes only), out[1] free passes. */
void study_rows(const uint8_t* vol, int nx, int ny, int nz, const float* lut, int lut_n,
                const double* pv, const double* inv_pv, const double* eye, const double* bb,
                int width, int height, int n_sg, int delta, double eps, double gamma_init,
                double step, double lref, const int32_t* rows, int nrows, int64_t* out) {
  int64_t tot = 0, freep = 0, queued = 0;
  init_u8tab();
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : tot, freep, queued)
  for (int64_t q = 0; q < (int64_t)nrows * width; ++q) {
    int ly = rows[q / width], lx = (int)(q % width);
    double d[3];
    pixel_ray(inv_pv, eye, lx, ly, width, height, d);
    double ta, tb, fa, fb;
    if (!(clip_aabb(eye[0], eye[1], eye[2], d[0], d[1], d[2], bb, &ta, &tb) &&
          clip_frustum(pv, eye[0], eye[1], eye[2], d[0], d[1], d[2], &fa, &fb))) continue;
    double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb);
    if (!(t1 > t0)) continue;
    vox_t v = {NULL, vol};
    ray_ctx r = {v, nx, ny, nz, lut, lut_n, pv, eye[0], eye[1], eye[2],
                 d[0], d[1], d[2], bb, t0, t1, step, lref, n_sg, NULL};
    double low = 0.0, high = SQRT3, gamma = gamma_init;
    int first = 1, npass = 0;
    double G[64], U[64], V[64];
    int N[64];
    for (;;) {
      if (fabs(high - low) < eps) break;
      /* could this pass be answered by an earlier one? */
      const double th = thr_of(gamma);
      int hit = 0;
      for (int i = 0; i < npass && !hit; ++i) {
        if (gamma > G[i] ? U[i] >= th : (gamma < G[i] ? V[i] < th : 1)) hit = 1;
      }
      double u2, v2;
      int n = count_pass(&r, gamma, &u2, &v2);
      if (npass < 64) { G[npass] = gamma; U[npass] = u2; V[npass] = v2; N[npass] = n; }
      if (!first) { tot += 1; freep += hit; }
      npass++;
      if (first) {
        first = 0;
        if (n < n_sg) break;
        queued += 1;
      }
      if (n > n_sg) low = gamma;
      else if (n < n_sg - delta) high = gamma;
      else break;
      gamma = 0.5 * (low + high);
    }
    (void)N;
  }
  out[0] = tot;
  out[1] = freep;
  out[2] = queued;
}
