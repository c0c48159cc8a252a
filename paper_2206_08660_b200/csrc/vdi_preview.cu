// vdi_preview.cu -- preview rendering with dynamic subsampling on sm_100a.
//
// Semantics: the reference's _preview_kernel (preview.py:49-205), which R
// runs serially: per low-res pixel, the eye ray is clipped to the volume box
// and the generation frustum and projected to an NDC chord; the chord is
// split at AccelGrid cell boundaries; each non-empty cell gets
// round-half-up(d_r * world length * cell count) point samples at regular
// intervals; a sample takes the colour of the supersegment containing it
// (Alg. 2 search with d_entry == d_exit) with the opacity of the distance to
// the previous sample. Then bilinear_upsample (preview.py:208-223).
//
// B200 structure:
//  * one lane per pixel, 8x4 pixel tiles, lanes refill from a warp-uniform
//    pool (per-pixel sample counts range from 0 to thousands);
//  * the breakpoints are produced in sorted order by a 3-way merge of the
//    x, y and z boundary sequences instead of R's array + np.sort. Each
//    sequence is monotone in the boundary index (every step of its formula
//    is a correctly rounded monotone operation), so iterating it in the
//    chord's direction and merging yields exactly the sorted multiset --
//    no per-thread array, no sort; the first boundary inside (0, 1) is found
//    by binary search over the monotone sequence;
//  * lists are list-SoA; per-cell sample budgets go to cell_samples with
//    one 64-bit atomic per (pixel, non-empty cell).
#include "vdi_common.cuh"
#include "vdi_internal.h"
#include "vdi_search.cuh"

namespace vdi {

constexpr int kPreviewThreads = 128;

struct PreviewConst {
  VdiPreviewArgs a;
  int tiles_x;
  long long n_slots;
  unsigned long long* fetch;     // pixel pool
  unsigned int* unsorted;        // lists whose backs are not non-decreasing
};

// One axis' boundary sequence s(i) = (bound(i) - a0) / cd, i in [1, n-1],
// walked in the order that makes s non-decreasing.
struct BoundSeq {
  int m, count;    // position in walk order, number of boundaries (n - 1)
  int asc;         // i = asc ? 1 + m : n - 1 - m
  double next;     // s at m, or +inf when exhausted (s >= 1 or no more)
};

// preview.py:97-121: the three boundary formulas, in R's evaluation order.
template <int AX>
__device__ __forceinline__ double bound_s(const PreviewConst& c, int i, double a0, double cd) {
  const VdiPreviewArgs& a = c.a;
  if (AX == 0) return (-1.0 + 2.0 * i / a.gx - a0) / cd;
  if (AX == 1) return (-1.0 + 2.0 * i / a.gy - a0) / cd;
  const double dep = a.near + (a.far - a.near) * i / a.gz;
  const double zb = a.proj_a - a.proj_b / dep;
  return (zb - a0) / cd;
}

template <int AX>
__device__ __forceinline__ double seq_at(const PreviewConst& c, const BoundSeq& q, double a0,
                                         double cd, int n) {
  return bound_s<AX>(c, q.asc ? 1 + q.m : n - 1 - q.m, a0, cd);
}

// Position the walk on the first boundary with s > 0 (s is non-decreasing
// in m, so the boundaries inside (0, 1) are one contiguous run).
template <int AX>
__device__ __forceinline__ void seq_init(const PreviewConst& c, BoundSeq& q, double a0, double cd,
                                         int n) {
  q.count = n - 1;
  q.asc = cd > 0;
  q.next = INFINITY;
  if (!(fabs(cd) > 1e-14) || q.count <= 0) {
    q.m = q.count;
    return;
  }
  int lo = 0, hi = q.count;  // first m in [0, count) with s(m) > 0, or count
  while (lo < hi) {
    q.m = (lo + hi) >> 1;
    if (seq_at<AX>(c, q, a0, cd, n) > 0.0) hi = q.m;
    else lo = q.m + 1;
  }
  q.m = lo;
  if (q.m < q.count) {
    const double s = seq_at<AX>(c, q, a0, cd, n);
    if (s < 1.0) q.next = s;
  }
}

template <int AX>
__device__ __forceinline__ void seq_advance(const PreviewConst& c, BoundSeq& q, double a0,
                                            double cd, int n) {
  q.m += 1;
  q.next = INFINITY;
  if (q.m < q.count) {
    const double s = seq_at<AX>(c, q, a0, cd, n);
    if (s < 1.0) q.next = s;
  }
}

__device__ __forceinline__ double sq(double x) { return x * x; }  // numba x ** 2

// Serial-per-pixel form (one lane per pixel): the exact reference loop,
// including the seed chain of the Alg. 2 search. Used when some list's backs
// are not non-decreasing (possible only in hand-made VDIs that use the 1e-7
// overlap slack of validate_vdi); generated VDIs take preview_warp_kernel.
__global__ void __launch_bounds__(kPreviewThreads) preview_kernel(const PreviewConst c) {
  if (*c.unsorted == 0u) return;
  const VdiPreviewArgs& a = c.a;
  const int lane = threadIdx.x & 31;
  unsigned long long total = 0;
  long long base = 0;
  int used = 32;
  bool done_all = false;

  while (true) {
    // every lane that is free takes the next pixel of the pool
    long long slot = -1;
    {
      const unsigned need = __ballot_sync(0xffffffffu, !done_all);
      if (!need) break;
      const int n = __popc(need);
      const int rank = __popc(need & ((1u << lane) - 1u));
      const int avail = 32 - used;
      long long fresh = 0;
      if (n > avail) {
        if (lane == 0) fresh = (long long)atomicAdd(c.fetch, 32ull);
        fresh = __shfl_sync(0xffffffffu, fresh, 0);
      }
      slot = rank < avail ? base + used + rank : fresh + (rank - avail);
      if (n > avail) {
        base = fresh;
        used = n - avail;
      } else {
        used += n;
      }
      if (done_all) slot = -1;
    }
    if (slot < 0) continue;
    if (slot >= c.n_slots) {
      done_all = true;
      continue;
    }
    const long long tile = slot >> 5;
    const int tw = (int)(slot & 31);
    const int col = (int)(tile % c.tiles_x) * kTileW + (tw & 7);
    const int row = (int)(tile / c.tiles_x) * kTileH + (tw >> 3);
    if (col >= a.out_w || row >= a.out_h) continue;

    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
    double d[3];
    pixel_ray(a.new_inv_pv, a.eye, col, row, a.out_w, a.out_h, d);  // preview.py:60-69
    const double* eye = a.eye;
    double ta, tb, fa, fb, t0 = 0.0, t1 = 0.0;
    bool ok = false;
    if (clip_aabb(eye, d, a.aabb, ta, tb) && clip_frustum(a.gen_pv, eye, d, fa, fb)) {
      t0 = dmax(dmax(ta, fa), 0.0);
      t1 = dmin(tb, fb);
      ok = t1 > t0;
    }
    if (ok) {
      double a0x, a0y, a0z, a1x, a1y, a1z;
      xform(a.gen_pv, eye[0] + t0 * d[0], eye[1] + t0 * d[1], eye[2] + t0 * d[2], a0x, a0y, a0z);
      xform(a.gen_pv, eye[0] + t1 * d[0], eye[1] + t1 * d[1], eye[2] + t1 * d[2], a1x, a1y, a1z);
      const double cdx = a1x - a0x, cdy = a1y - a0y, cdz = a1z - a0z;
      BoundSeq qx, qy, qz;
      seq_init<0>(c, qx, a0x, cdx, a.gx);
      seq_init<1>(c, qy, a0y, cdy, a.gy);
      seq_init<2>(c, qz, a0z, cdz, a.gz);
      double px, py, pz;
      xform(a.gen_inv_pv, a0x, a0y, a0z, px, py, pz);  // preview.py:125
      int p = -1;
      bool done = false;
      double s_a = 0.0;  // sorted breakpoints: 0, merged boundaries, 1
      bool last = false;
      while (!done && !last) {
        double s_b;
        if (qx.next <= qy.next && qx.next <= qz.next && qx.next < INFINITY) {
          s_b = qx.next;
          seq_advance<0>(c, qx, a0x, cdx, a.gx);
        } else if (qy.next <= qz.next && qy.next < INFINITY) {
          s_b = qy.next;
          seq_advance<1>(c, qy, a0y, cdy, a.gy);
        } else if (qz.next < INFINITY) {
          s_b = qz.next;
          seq_advance<2>(c, qz, a0z, cdz, a.gz);
        } else {
          s_b = 1.0;
          last = true;
        }
        const double sa = s_a;
        s_a = s_b;
        if (s_b - sa < 1e-15) continue;  // preview.py:131-132
        const double sm = 0.5 * (sa + s_b);
        const double mx = a0x + sm * cdx, my = a0y + sm * cdy, mz = a0z + sm * cdz;
        const int cgx = clampi(floor_ll((mx + 1.0) * a.gx / 2.0), 0, a.gx - 1);
        const int cgy = clampi(floor_ll((my + 1.0) * a.gy / 2.0), 0, a.gy - 1);
        const double mdep = a.proj_b / (a.proj_a - mz);
        const int cgz = clampi(floor_ll((mdep - a.near) / (a.far - a.near) * a.gz), 0, a.gz - 1);
        const long long cell = ((long long)cgz * a.gy + cgy) * a.gx + cgx;
        const unsigned cnt = __ldg(a.grid + cell);
        if (cnt == 0u) continue;
        double w0x, w0y, w0z, w1x, w1y, w1z;
        xform(a.gen_inv_pv, a0x + sa * cdx, a0y + sa * cdy, a0z + sa * cdz, w0x, w0y, w0z);
        xform(a.gen_inv_pv, a0x + s_b * cdx, a0y + s_b * cdy, a0z + s_b * cdz, w1x, w1y, w1z);
        const double seg_len = sqrt(sq(w1x - w0x) + sq(w1y - w0y) + sq(w1z - w0z));
        const long long n = (long long)floor(a.d_r * seg_len * (double)cnt + 0.5);
        if (n <= 0) continue;
        if (a.cell_samples) atomicAdd(a.cell_samples + cell, (unsigned long long)n);
        total += (unsigned long long)n;
        const double dn = (double)n, span = s_b - sa;
        for (long long i = 0; i < n; ++i) {  // preview.py:160-205
          const double sf = sa + ((double)i + 0.5) / dn * span;
          const double sx = a0x + sf * cdx, sy = a0y + sf * cdy, sz = a0z + sf * cdz;
          double swx, swy, swz;
          xform(a.gen_inv_pv, sx, sy, sz, swx, swy, swz);
          const double dist = sqrt(sq(swx - px) + sq(swy - py) + sq(swz - pz));
          px = swx;
          py = swy;
          pz = swz;
          const int lx = clampi(floor_ll((sx + 1.0) * a.vdi_w / 2.0), 0, a.vdi_w - 1);
          const int ly = clampi(floor_ll((sy + 1.0) * a.vdi_h / 2.0), 0, a.vdi_h - 1);
          const long long lidx =
              (long long)vdi_storage_row(ly, a.vdi_band_rows, a.vdi_band_world,
                                         a.vdi_rows_per_rank) * a.vdi_w + lx;
          const int lc = __ldg(a.counts + lidx);
          if (lc == 0) continue;
          const float* ls = a.segs + lidx * (long long)list_stride(a.n_sg);
          const float* fronts = ls + front_off(a.n_sg);
          const float* backs = ls + back_off(a.n_sg);
          int seed;
          const int j = find_first(fronts, backs, lc, sz, sz, p, seed);
          p = seed;
          if (j < 0) continue;
          const float4 c4 = reinterpret_cast<const float4*>(ls)[j];
          if (c4.w <= 0.0f) continue;
          const double xc = -1.0 + 2.0 * (lx + 0.5) / a.vdi_w;
          const double yc = -1.0 + 2.0 * (ly + 0.5) / a.vdi_h;
          double wfx, wfy, wfz, wbx, wby, wbz;
          xform(a.gen_inv_pv, xc, yc, (double)fronts[j], wfx, wfy, wfz);
          xform(a.gen_inv_pv, xc, yc, (double)backs[j], wbx, wby, wbz);
          const double thick = sqrt(sq(wbx - wfx) + sq(wby - wfy) + sq(wbz - wfz));
          if (thick <= 0.0) continue;
          const double alpha = (double)c4.w;
          const double a_t = 1.0 - pow(1.0 - alpha, dist / thick);
          const double scale = a_t / alpha;
          const double w = 1.0 - acc_a;
          acc_r += w * (double)c4.x * scale;
          acc_g += w * (double)c4.y * scale;
          acc_b += w * (double)c4.z * scale;
          acc_a += w * a_t;
          if (acc_a >= a.early_term) {
            done = true;
            break;
          }
        }
      }
    }
    const double w = 1.0 - acc_a;  // preview.py:199-203
    double2* o = reinterpret_cast<double2*>(a.image + 4 * ((long long)row * a.out_w + col));
    o[0] = make_double2(acc_r + w * a.bg[0] * a.bg[3], acc_g + w * a.bg[1] * a.bg[3]);
    o[1] = make_double2(acc_b + w * a.bg[2] * a.bg[3], acc_a + w * a.bg[3]);
  }
  if (a.stat_sums) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
    if (lane == 0 && total) atomicAdd(a.stat_sums, total);
  }
}

// Counts lists whose backs are not non-decreasing. For non-decreasing backs
// the seeded search (raycast.py:79-121 with d_entry == d_exit == d) returns
// the global smallest j with back[j] >= d (or count - 1) for EVERY seed p:
// interval 0 puts every back[<= p] below d, interval 2 puts back[p - 1] at or
// above d, interval 1 makes p itself the smallest, and the clamped empty
// ranges land on count - 1 exactly as the full search does. So the samples
// of a pixel become independent and can be spread over a warp.
__global__ void unsorted_lists_kernel(const PreviewConst c) {
  const VdiPreviewArgs& a = c.a;
  const long long n = (long long)a.vdi_w * a.vdi_h;
  unsigned bad = 0;
  for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < n;
       l += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(l / a.vdi_w), x = (int)(l - (long long)r * a.vdi_w);
    const long long lidx =
        (long long)vdi_storage_row(r, a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank) *
            a.vdi_w + x;
    const int cnt = __ldg(a.counts + lidx);
    const float* backs = a.segs + lidx * (long long)list_stride(a.n_sg) + back_off(a.n_sg);
    for (int k = 0; k + 1 < cnt; ++k)
      if (!(__ldg(backs + k) <= __ldg(backs + k + 1))) {
        bad = 1;
        break;
      }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicAdd(c.unsorted, 1u);
}

constexpr int kPreviewWarpThreads = 128;

// Warp-per-pixel form for VDIs with sorted lists (*c.unsorted == 0). The
// warp walks the pixel's cell intervals together (warp-uniform values); the
// samples of an interval are spread over the lanes 32 at a time -- position,
// distance to the previous sample (shuffled from the neighbouring lane),
// list lookup, seed-free search, thickness and pow() -- and then composited
// in the reference's sample order by a lane-uniform serial loop over the
// contributing samples, so the accumulation and the early termination are
// exactly R's.
__global__ void __launch_bounds__(kPreviewWarpThreads) preview_warp_kernel(const PreviewConst c) {
  if (*c.unsorted != 0u) return;
  const VdiPreviewArgs& a = c.a;
  __shared__ double s_val[kPreviewWarpThreads / 32][5][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double(*sv)[32] = s_val[wib];
  unsigned long long total = 0;
  const long long npix = (long long)a.out_w * a.out_h;
  while (true) {
    long long pix = 0;
    if (lane == 0) pix = (long long)atomicAdd(c.fetch, 1ull);
    pix = __shfl_sync(0xffffffffu, pix, 0);
    if (pix >= npix) break;
    const int row = (int)(pix / a.out_w), col = (int)(pix - (long long)row * a.out_w);
    double acc_r = 0.0, acc_g = 0.0, acc_b = 0.0, acc_a = 0.0;
    double d[3];
    pixel_ray(a.new_inv_pv, a.eye, col, row, a.out_w, a.out_h, d);  // preview.py:60-69
    const double* eye = a.eye;
    double ta, tb, fa, fb, t0 = 0.0, t1 = 0.0;
    bool ok = false;
    if (clip_aabb(eye, d, a.aabb, ta, tb) && clip_frustum(a.gen_pv, eye, d, fa, fb)) {
      t0 = dmax(dmax(ta, fa), 0.0);
      t1 = dmin(tb, fb);
      ok = t1 > t0;
    }
    if (ok) {
      double a0x, a0y, a0z, a1x, a1y, a1z;
      xform(a.gen_pv, eye[0] + t0 * d[0], eye[1] + t0 * d[1], eye[2] + t0 * d[2], a0x, a0y, a0z);
      xform(a.gen_pv, eye[0] + t1 * d[0], eye[1] + t1 * d[1], eye[2] + t1 * d[2], a1x, a1y, a1z);
      const double cdx = a1x - a0x, cdy = a1y - a0y, cdz = a1z - a0z;
      BoundSeq qx, qy, qz;
      seq_init<0>(c, qx, a0x, cdx, a.gx);
      seq_init<1>(c, qy, a0y, cdy, a.gy);
      seq_init<2>(c, qz, a0z, cdz, a.gz);
      double px, py, pz;
      xform(a.gen_inv_pv, a0x, a0y, a0z, px, py, pz);  // preview.py:125
      bool done = false;
      double s_a = 0.0;
      bool last = false;
      while (!done && !last) {
        double s_b;
        if (qx.next <= qy.next && qx.next <= qz.next && qx.next < INFINITY) {
          s_b = qx.next;
          seq_advance<0>(c, qx, a0x, cdx, a.gx);
        } else if (qy.next <= qz.next && qy.next < INFINITY) {
          s_b = qy.next;
          seq_advance<1>(c, qy, a0y, cdy, a.gy);
        } else if (qz.next < INFINITY) {
          s_b = qz.next;
          seq_advance<2>(c, qz, a0z, cdz, a.gz);
        } else {
          s_b = 1.0;
          last = true;
        }
        const double sa = s_a;
        s_a = s_b;
        if (s_b - sa < 1e-15) continue;  // preview.py:131-132
        const double sm = 0.5 * (sa + s_b);
        const double mx = a0x + sm * cdx, my = a0y + sm * cdy, mz = a0z + sm * cdz;
        const int cgx = clampi(floor_ll((mx + 1.0) * a.gx / 2.0), 0, a.gx - 1);
        const int cgy = clampi(floor_ll((my + 1.0) * a.gy / 2.0), 0, a.gy - 1);
        const double mdep = a.proj_b / (a.proj_a - mz);
        const int cgz = clampi(floor_ll((mdep - a.near) / (a.far - a.near) * a.gz), 0, a.gz - 1);
        const long long cell = ((long long)cgz * a.gy + cgy) * a.gx + cgx;
        const unsigned cnt = __ldg(a.grid + cell);
        if (cnt == 0u) continue;
        double w0x, w0y, w0z, w1x, w1y, w1z;
        xform(a.gen_inv_pv, a0x + sa * cdx, a0y + sa * cdy, a0z + sa * cdz, w0x, w0y, w0z);
        xform(a.gen_inv_pv, a0x + s_b * cdx, a0y + s_b * cdy, a0z + s_b * cdz, w1x, w1y, w1z);
        const double seg_len = sqrt(sq(w1x - w0x) + sq(w1y - w0y) + sq(w1z - w0z));
        const long long n = (long long)floor(a.d_r * seg_len * (double)cnt + 0.5);
        if (n <= 0) continue;
        if (lane == 0) {
          if (a.cell_samples) atomicAdd(a.cell_samples + cell, (unsigned long long)n);
          total += (unsigned long long)n;
        }
        const double dn = (double)n, span = s_b - sa;
        for (long long base = 0; base < n && !done; base += 32) {  // preview.py:160-205
          const long long i = base + lane;
          const bool valid = i < n;
          const double sf = sa + ((double)i + 0.5) / dn * span;
          const double sx = a0x + sf * cdx, sy = a0y + sf * cdy, sz = a0z + sf * cdz;
          double swx, swy, swz;
          xform(a.gen_inv_pv, sx, sy, sz, swx, swy, swz);
          // previous sample: the neighbouring lane, or the carried one for lane 0
          double qx0 = __shfl_up_sync(0xffffffffu, swx, 1);
          double qy0 = __shfl_up_sync(0xffffffffu, swy, 1);
          double qz0 = __shfl_up_sync(0xffffffffu, swz, 1);
          if (lane == 0) {
            qx0 = px;
            qy0 = py;
            qz0 = pz;
          }
          const double dist = sqrt(sq(swx - qx0) + sq(swy - qy0) + sq(swz - qz0));
          const int lastl = (int)(n - base < 32 ? n - base - 1 : 31);
          px = __shfl_sync(0xffffffffu, swx, lastl);
          py = __shfl_sync(0xffffffffu, swy, lastl);
          pz = __shfl_sync(0xffffffffu, swz, lastl);
          bool con = false;
          double cr = 0.0, cg = 0.0, cb = 0.0, scale = 0.0, a_t = 0.0;
          if (valid) {
            const int lx = clampi(floor_ll((sx + 1.0) * a.vdi_w / 2.0), 0, a.vdi_w - 1);
            const int ly = clampi(floor_ll((sy + 1.0) * a.vdi_h / 2.0), 0, a.vdi_h - 1);
            const long long lidx =
                (long long)vdi_storage_row(ly, a.vdi_band_rows, a.vdi_band_world,
                                           a.vdi_rows_per_rank) * a.vdi_w + lx;
            const int lc = __ldg(a.counts + lidx);
            if (lc > 0) {
              const float* ls = a.segs + lidx * (long long)list_stride(a.n_sg);
              const float* fronts = ls + front_off(a.n_sg);
              const float* backs = ls + back_off(a.n_sg);
              int seed;
              const int j = find_first(fronts, backs, lc, sz, sz, -1, seed);
              if (j >= 0) {
                const float4 c4 = __ldg(reinterpret_cast<const float4*>(ls) + j);
                if (c4.w > 0.0f) {
                  const double xc = -1.0 + 2.0 * (lx + 0.5) / a.vdi_w;
                  const double yc = -1.0 + 2.0 * (ly + 0.5) / a.vdi_h;
                  double wfx, wfy, wfz, wbx, wby, wbz;
                  xform(a.gen_inv_pv, xc, yc, (double)fronts[j], wfx, wfy, wfz);
                  xform(a.gen_inv_pv, xc, yc, (double)backs[j], wbx, wby, wbz);
                  const double thick = sqrt(sq(wbx - wfx) + sq(wby - wfy) + sq(wbz - wfz));
                  if (thick > 0.0) {
                    const double alpha = (double)c4.w;
                    a_t = 1.0 - pow(1.0 - alpha, dist / thick);
                    scale = a_t / alpha;
                    cr = c4.x;
                    cg = c4.y;
                    cb = c4.z;
                    con = true;
                  }
                }
              }
            }
          }
          sv[0][lane] = cr;
          sv[1][lane] = cg;
          sv[2][lane] = cb;
          sv[3][lane] = scale;
          sv[4][lane] = a_t;
          unsigned m = __ballot_sync(0xffffffffu, con);
          __syncwarp();
          while (m) {  // R's order: front to back over the contributing samples
            const int k = __ffs(m) - 1;
            m &= m - 1;
            const double sc = sv[3][k];
            const double w = 1.0 - acc_a;
            acc_r += w * sv[0][k] * sc;
            acc_g += w * sv[1][k] * sc;
            acc_b += w * sv[2][k] * sc;
            acc_a += w * sv[4][k];
            if (acc_a >= a.early_term) {
              done = true;
              break;
            }
          }
          __syncwarp();
        }
      }
    }
    if (lane == 0) {
      const double w = 1.0 - acc_a;  // preview.py:199-203
      double2* o = reinterpret_cast<double2*>(a.image + 4 * pix);
      o[0] = make_double2(acc_r + w * a.bg[0] * a.bg[3], acc_g + w * a.bg[1] * a.bg[3]);
      o[1] = make_double2(acc_b + w * a.bg[2] * a.bg[3], acc_a + w * a.bg[3]);
    }
  }
  if (a.stat_sums && lane == 0 && total) atomicAdd(a.stat_sums, total);
}

int preview_launch(const VdiPreviewArgs* args, cudaStream_t stream) {
  PreviewConst c;
  c.a = *args;
  if (c.a.vdi_band_rows <= 0) c.a.vdi_band_rows = 16;
  if (c.a.vdi_band_world <= 0) c.a.vdi_band_world = 1;
  c.tiles_x = (args->out_w + kTileW - 1) / kTileW;
  const long long tiles_y = (args->out_h + kTileH - 1) / kTileH;
  c.n_slots = (long long)c.tiles_x * tiles_y * 32;
  c.fetch = reinterpret_cast<unsigned long long*>(args->workspace);
  c.unsorted = reinterpret_cast<unsigned int*>(c.fetch + 2);
  cudaError_t err = cudaMemsetAsync(c.fetch, 0, 4 * sizeof(unsigned long long), stream);
  if (err == cudaSuccess && args->cell_samples)
    err = cudaMemsetAsync(args->cell_samples, 0,
                          sizeof(unsigned long long) * (size_t)args->gx * args->gy * args->gz,
                          stream);
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "preview memset: %s", cudaGetErrorString(err));
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  {
    const long long lists = (long long)args->vdi_w * args->vdi_h;
    long long b = (lists + 255) / 256;
    if (b > (long long)sms * 8) b = (long long)sms * 8;
    unsorted_lists_kernel<<<(unsigned)(b < 1 ? 1 : b), 256, 0, stream>>>(c);
  }
  {
    // the warp form: one warp per pixel from a shared pixel counter
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, preview_warp_kernel,
                                                  kPreviewWarpThreads, 0);
    if (per < 1) per = 1;
    long long wb = (long long)sms * per;
    const long long npix = (long long)args->out_w * args->out_h;
    const long long need_w = (npix + kPreviewWarpThreads / 32 - 1) / (kPreviewWarpThreads / 32);
    if (wb > need_w) wb = need_w;
    preview_warp_kernel<<<(unsigned)(wb < 1 ? 1 : wb), kPreviewWarpThreads, 0, stream>>>(c);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, preview_kernel, kPreviewThreads, 0);
  if (per_sm < 1) per_sm = 1;
  long long blocks = (long long)sms * per_sm;
  const long long need = (c.n_slots + kPreviewThreads - 1) / kPreviewThreads;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  preview_kernel<<<(unsigned)blocks, kPreviewThreads, 0, stream>>>(c);
  err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "preview launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// preview.py:208-223 bilinear_upsample, same f64 expressions per element.
__global__ void upsample_kernel(const double* __restrict__ src, int w, int h,
                                double* __restrict__ dst, int out_w, int out_h, int ch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)out_w * out_h;
  if (i >= total) return;
  const int ox = (int)(i % out_w), oy = (int)(i / out_w);
  const double xs = ((double)ox + 0.5) * w / out_w - 0.5;
  const double ys = ((double)oy + 0.5) * h / out_h - 0.5;
  const long long fxl = (long long)floor(xs), fyl = (long long)floor(ys);
  const int x0 = (int)(fxl < 0 ? 0 : (fxl > w - 1 ? w - 1 : fxl));
  const int y0 = (int)(fyl < 0 ? 0 : (fyl > h - 1 ? h - 1 : fyl));
  const int x1 = x0 + 1 < w - 1 ? x0 + 1 : w - 1;
  const int y1 = y0 + 1 < h - 1 ? y0 + 1 : h - 1;
  const double fx = dmin(dmax(xs - x0, 0.0), 1.0);
  const double fy = dmin(dmax(ys - y0, 0.0), 1.0);
  const double* r0 = src + (long long)y0 * w * ch;
  const double* r1 = src + (long long)y1 * w * ch;
  for (int k = 0; k < ch; ++k) {
    const double top = r0[x0 * ch + k] * (1 - fx) + r0[x1 * ch + k] * fx;
    const double bot = r1[x0 * ch + k] * (1 - fx) + r1[x1 * ch + k] * fx;
    dst[i * ch + k] = top * (1 - fy) + bot * fy;
  }
}

int bilinear_upsample(const double* src, int w, int h, double* dst, int out_w, int out_h,
                      int channels, cudaStream_t stream) {
  const long long total = (long long)out_w * out_h;
  if (total == 0) return VDI_OK;
  upsample_kernel<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(src, w, h, dst, out_w,
                                                                       out_h, channels);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "upsample launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
