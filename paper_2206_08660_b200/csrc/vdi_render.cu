// vdi_render.cu -- novel-view VDI raycasting on sm_100a.
//
// Semantics: the reference's _render_kernel (raycast.py:275-456): per output
// pixel an eye ray is clipped to the volume box and the GENERATION frustum,
// projected to an NDC chord, and walked through the W x H list grid with the
// Amanatides-Woo DDA (x before y on ties); per list the ESS cell-range test
// (_grid_cell_range, 258-272) gates the Alg. 2 seeded search (_find_first,
// 79-141, with _bins 51-62 / _bins_front 65-76); intersected supersegments are
// composited front to back with the Eq. 2 length correction and early ray
// termination. f64 throughout, f32 depths promoted before every compare.
//
// Layout: lists are list-SoA (include/vdi_b200.h), so the search reads only
// the contiguous back[] run of a list and a supersegment's colour is one
// aligned float4. A warp owns an 8x4 pixel tile; neighbouring pixels walk
// neighbouring lists, which keeps the count/back/rgba loads L1-coherent.
#include <cstring>

#include "vdi_common.cuh"
#include "vdi_internal.h"
#include "vdi_search.cuh"

namespace vdi {

#ifndef VDI_RENDER_THREADS
#define VDI_RENDER_THREADS 128
#endif
constexpr int kRenderThreads = VDI_RENDER_THREADS;
#ifndef VDI_RANGE_AHEAD
#define VDI_RANGE_AHEAD 1  // 1: the walk loads the next list's depth range with its count
#endif
#ifndef VDI_RENDER_MINB
// blocks per SM: 20 warps, 96 registers, no spills (C3 0.93 ms; 24 warps: 1.03, 16: 1.00)
#define VDI_RENDER_MINB (640 / VDI_RENDER_THREADS)
#endif

// Storage row of VDI list row r: the explicit map when given
// (VdiRenderArgs.vdi_row_map), else the band map.
__device__ __forceinline__ int storage_row(const VdiRenderArgs& a, int r) {
  return a.vdi_row_map ? __ldg(a.vdi_row_map + r)
                       : vdi_storage_row(r, a.vdi_band_rows, a.vdi_band_world,
                                         a.vdi_rows_per_rank);
}

struct RenderConst {
  VdiRenderArgs a;
  int tiles_x;
  int local_h;
  long long n_slots;
  int lt_words;  // words of the list-tile bitmap staged in shared memory (0: none)
  int lt_wpr;    // its words per tile row
  double rfn;    // RN(1 / (far - near)): (x - near) / (far - near) via div_by
};

// List-tile occupancy (vdi_list_tiles): 8x8 lists per tile, one bitmap word
// per 32 horizontally adjacent tiles, rows padded to whole words.
constexpr int kListTile = 8;
__host__ __device__ inline int lt_words_per_row(int vdi_w) {
  return ((vdi_w + kListTile - 1) / kListTile + 31) / 32;
}

// Per-ray state that only the shading of a non-empty list reads and updates,
// kept in shared memory (one slot per thread, SoA: conflict-free): the
// empty-list walk then carries only its DDA state in registers, and the
// shading's f64 temporaries do not force the walk state to spill.
struct ShadeSmem {
  double a0x[kRenderThreads], a0y[kRenderThreads], a0z[kRenderThreads];
  double cdx[kRenderThreads], cdy[kRenderThreads], cdz[kRenderThreads];
  double acc_r[kRenderThreads], acc_g[kRenderThreads], acc_b[kRenderThreads];
  double acc_a[kRenderThreads];
  double dep_key[kRenderThreads], dep_val[kRenderThreads];  // last proj_b / (proj_a - d(s))
  int p[kRenderThreads];                                    // the Alg. 2 seed (raycast.py:344)
  int nint[kRenderThreads], nsearch[kRenderThreads];
  unsigned long long sum_vis[kRenderThreads], sum_int[kRenderThreads], sum_srch[kRenderThreads];
};

// _grid_cell_range (raycast.py:258-272) + the all-empty scan (359-370):
// true when every grid cell the chord piece [s_cur, s_exit] covers is empty.
// d = a0z + s cdz is a function of s alone, so the depth of a shared chord
// parameter (this list's entry = the previous list's exit) is reused.
template <bool kMask>
__device__ __forceinline__ bool ess_empty(const RenderConst& c, ShadeSmem& sm, int t, double a0x,
                                          double a0y, double cdx, double cdy, double s_cur,
                                          double s_exit, double d_entry, double d_exit) {
  const VdiRenderArgs& a = c.a;
  const double x_a = a0x + s_cur * cdx, y_a = a0y + s_cur * cdy;
  const double x_b = a0x + s_exit * cdx, y_b = a0y + s_exit * cdy;
  const double dep_a = s_cur == sm.dep_key[t] ? sm.dep_val[t] : a.proj_b / (a.proj_a - d_entry);
  const double dep_b = a.proj_b / (a.proj_a - d_exit);
  sm.dep_key[t] = s_exit;
  sm.dep_val[t] = dep_b;
  const int gx = a.gx, gy = a.gy, gz = a.gz;
  const int cgx0 = clampi(floor_ll((dmin(x_a, x_b) + 1.0) * gx / 2.0), 0, gx - 1);
  const int cgx1 = clampi(floor_ll((dmax(x_a, x_b) + 1.0) * gx / 2.0), 0, gx - 1);
  const int cgy0 = clampi(floor_ll((dmin(y_a, y_b) + 1.0) * gy / 2.0), 0, gy - 1);
  const int cgy1 = clampi(floor_ll((dmax(y_a, y_b) + 1.0) * gy / 2.0), 0, gy - 1);
  const double fn = a.far - a.near;
  const int cz0 = clampi(floor_ll(div_by(dmin(dep_a, dep_b) - a.near, fn, c.rfn) * gz), 0, gz - 1);
  const int cz1 = clampi(floor_ll(div_by(dmax(dep_a, dep_b) - a.near, fn, c.rfn) * gz), 0, gz - 1);
  if (kMask) {
    uint64_t m = 0;
    for (int cgy = cgy0; cgy <= cgy1; ++cgy)
      for (int cgx = cgx0; cgx <= cgx1; ++cgx) m |= __ldg(a.grid_zmask + cgy * gx + cgx);
    // bits cz0..cz1 (2 << 63 wraps to 0, which still yields bits cz0..63)
    const uint64_t want = (2ull << cz1) - (1ull << cz0);
    return (m & want) == 0;
  }
  for (int cz = cz0; cz <= cz1; ++cz)
    for (int cgy = cgy0; cgy <= cgy1; ++cgy)
      for (int cgx = cgx0; cgx <= cgx1; ++cgx)
        if (__ldg(a.grid + ((long long)cz * gy + cgy) * gx + cgx) > 0u) return false;
  return true;
}

// One non-empty list of the DDA (raycast.py:346-435 for count > 0): the ESS
// test, the seeded search and the Eq. 2 compositing. Returns true when the
// ray terminates (acc_a >= early_term).
//
// kFast (lists_sorted, a forward chord, lists_searched not counted): the
// search runs first and the ESS test only confirms a hit. This is the same
// result: with non-decreasing backs the forward search (raycast.py:88-121)
// returns the first back >= d_entry (or the last list entry) whatever the
// seed -- each seed interval either holds that index or prunes to a range
// that does -- so searching a list R would have skipped changes no later
// search; a miss composites nothing in either order; and a hit is
// composited iff the ESS test passes, as in R.
template <bool kMask>
__device__ __forceinline__ bool shade_list(const RenderConst& c, ShadeSmem& sm, int t, int cx,
                                           int cy, long long lidx, int count, double s_cur,
                                           double tmin, bool fast, bool range_test = true) {
  const VdiRenderArgs& a = c.a;
  const int vdi_w = a.vdi_w, vdi_h = a.vdi_h, n_sg = a.n_sg;
  const double a0x = sm.a0x[t], a0y = sm.a0y[t], a0z = sm.a0z[t];
  const double cdx = sm.cdx[t], cdy = sm.cdy[t], cdz = sm.cdz[t];
  double s_exit = dmin(tmin, 1.0);  // min(min(t_max_x, t_max_y), 1.0), raycast.py:345
  if (s_exit < s_cur) s_exit = s_cur;
  const double d_entry = a0z + s_cur * cdz;
  const double d_exit = a0z + s_exit * cdz;
  const float* ls = a.segs + lidx * (long long)list_stride(n_sg);
  const float* fronts = ls + front_off(n_sg);
  const float* backs = ls + back_off(n_sg);
  const float4* rgba = reinterpret_cast<const float4*>(ls);
  int seed, j;
  if (fast) {
    if (range_test && a.list_range) {
      // the chord piece misses the list's depth range: the search would miss
      // (no back >= d_entry, or every front > d_exit); the seed is not read
      // again on this ray (fast mode does not depend on it)
      const float2 r = __ldg(reinterpret_cast<const float2*>(a.list_range) + lidx);
      if (d_exit < (double)r.x || d_entry > (double)r.y) return false;
    }
    j = find_first(fronts, backs, count, d_entry, d_exit, sm.p[t], seed);
    if (j < 0) {
      sm.p[t] = seed;
      return false;
    }
    if (a.use_ess &&
        ess_empty<kMask>(c, sm, t, a0x, a0y, cdx, cdy, s_cur, s_exit, d_entry, d_exit))
      return false;
  } else {
    if (a.use_ess &&
        ess_empty<kMask>(c, sm, t, a0x, a0y, cdx, cdy, s_cur, s_exit, d_entry, d_exit))
      return false;
    sm.nsearch[t] += 1;
    j = find_first(fronts, backs, count, d_entry, d_exit, sm.p[t], seed);
  }
  sm.p[t] = seed;
  if (j < 0) return false;
  const bool fwd = d_entry <= d_exit;
  const double zlo = dmin(d_entry, d_exit), zhi = dmax(d_entry, d_exit);
  const double xc = -1.0 + 2.0 * (cx + 0.5) / vdi_w;
  const double yc = -1.0 + 2.0 * (cy + 0.5) / vdi_h;
  double acc_r = sm.acc_r[t], acc_g = sm.acc_g[t], acc_b = sm.acc_b[t], acc_a = sm.acc_a[t];
  int nint = sm.nint[t], p = seed;
  bool done = false;
  for (int k = j; 0 <= k && k < count; k += fwd ? 1 : -1) {
    const double fk = fronts[k], bk = backs[k];
    const double ilo = dmax(fk, zlo), ihi = dmin(bk, zhi);
    if (ilo > ihi) break;
    double s_a, s_b;
    if (fabs(cdz) < 1e-12) {
      s_a = s_cur;
      s_b = s_exit;
    } else {
      s_a = (ilo - a0z) / cdz;
      s_b = (ihi - a0z) / cdz;
      if (s_a > s_b) {
        const double tt = s_a;
        s_a = s_b;
        s_b = tt;
      }
      if (s_a < s_cur) s_a = s_cur;
      if (s_b > s_exit) s_b = s_exit;
    }
    double w0x, w0y, w0z, w1x, w1y, w1z;
    xform(a.gen_inv_pv, a0x + s_a * cdx, a0y + s_a * cdy, a0z + s_a * cdz, w0x, w0y, w0z);
    xform(a.gen_inv_pv, a0x + s_b * cdx, a0y + s_b * cdy, a0z + s_b * cdz, w1x, w1y, w1z);
    const double ex = w1x - w0x, ey = w1y - w0y, ez = w1z - w0z;
    const double l = sqrt(ex * ex + ey * ey + ez * ez);
    double wfx, wfy, wfz, wbx, wby, wbz;
    xform(a.gen_inv_pv, xc, yc, fk, wfx, wfy, wfz);
    xform(a.gen_inv_pv, xc, yc, bk, wbx, wby, wbz);
    const double tx = wbx - wfx, ty = wby - wfy, tz = wbz - wfz;
    const double thick = sqrt(tx * tx + ty * ty + tz * tz);
    const float4 c4 = rgba[k];
    const double alpha = c4.w;
    if (alpha > 0.0 && thick > 0.0) {
      const double a_t = 1.0 - pow(1.0 - alpha, l / thick);
      const double scale = a_t / alpha;
      const double wgt = 1.0 - acc_a;
      acc_r += wgt * (double)c4.x * scale;
      acc_g += wgt * (double)c4.y * scale;
      acc_b += wgt * (double)c4.z * scale;
      acc_a += wgt * a_t;
    }
    nint += 1;
    p = k;
    if (acc_a >= a.early_term) {
      done = true;
      break;
    }
  }
  sm.acc_r[t] = acc_r;
  sm.acc_g[t] = acc_g;
  sm.acc_b[t] = acc_b;
  sm.acc_a[t] = acc_a;
  sm.nint[t] = nint;
  sm.p[t] = p;
  return done;
}

// raycast.py:283-456, one thread per output pixel (a warp owns an 8x4 tile).
// The DDA loop is restated around one fact: the break test s_exit >= 1.0
// (raycast.py:430) is min(t_max_x, t_max_y) >= 1.0, because s_cur < 1.0 holds
// on every iteration the reference reaches, and the x-before-y tie rule
// (t_max_x <= t_max_y, 437) selects the same minimum. So an empty list costs
// one compare, one count load and the step; s_exit, the depths and the ESS
// test are evaluated only for lists with count > 0 (the reference evaluates
// d_entry / d_exit for every list but reads them only there). The early
// termination test (429) can only change after a shading. Same visits, same
// order, same arithmetic: the image and every counter are unchanged.
// One 8x4 tile of output pixels, lane w = pixel (w & 7, w >> 3) of the tile.
template <bool kTiles, bool kMask, bool kBands>
__device__ __forceinline__ void render_tile(const RenderConst& c, ShadeSmem& sm,
                                            const uint32_t* s_tiles, int tile) {
  const VdiRenderArgs& a = c.a;
  const int t = threadIdx.x;
  const int w = threadIdx.x & 31;
  const int col = (int)(tile % c.tiles_x) * kTileW + (w & 7);
  const int lrow = (int)(tile / c.tiles_x) * kTileH + (w >> 3);
  if (col < a.out_w && lrow < c.local_h) {
    const int row = band_global_row(lrow, a.band_rows, a.band_stride, a.band_offset);
    const int vdi_w = a.vdi_w, vdi_h = a.vdi_h;
    sm.acc_r[t] = sm.acc_g[t] = sm.acc_b[t] = sm.acc_a[t] = 0.0;
    sm.nint[t] = sm.nsearch[t] = 0;
    int nvis = 0;
    double d[3];
    pixel_ray(a.new_inv_pv, a.eye, col, row, a.out_w, a.out_h, d);
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
      sm.a0x[t] = a0x;
      sm.a0y[t] = a0y;
      sm.a0z[t] = a0z;
      sm.cdx[t] = cdx;
      sm.cdy[t] = cdy;
      sm.cdz[t] = cdz;
      int cx = clampi(floor_ll((a0x + 1.0) * vdi_w / 2.0), 0, vdi_w - 1);
      int cy = clampi(floor_ll((a0y + 1.0) * vdi_h / 2.0), 0, vdi_h - 1);
      const int step_x = cdx > 0 ? 1 : (cdx < 0 ? -1 : 0);
      const int step_y = cdy > 0 ? 1 : (cdy < 0 ? -1 : 0);
      double t_max_x = INFINITY, t_delta_x = INFINITY, t_max_y = INFINITY,
             t_delta_y = INFINITY;
      if (step_x != 0) {
        const double bx = -1.0 + 2.0 * (double)(cx + (step_x > 0 ? 1 : 0)) / vdi_w;
        t_max_x = (bx - a0x) / cdx;
        t_delta_x = (2.0 / vdi_w) / fabs(cdx);
      }
      if (step_y != 0) {
        const double by = -1.0 + 2.0 * (double)(cy + (step_y > 0 ? 1 : 0)) / vdi_h;
        t_max_y = (by - a0y) / cdy;
        t_delta_y = (2.0 / vdi_h) / fabs(cdy);
      }
      // search-first shading (shade_list kFast): sorted lists, a chord running
      // forward in depth (d_entry <= d_exit on every list), uncounted searches
      const bool fast = a.lists_sorted && !a.counters_exact && cdz >= 0.0;
      sm.p[t] = -1;
      sm.dep_key[t] = -1.0;  // chord parameters are >= 0
      sm.dep_val[t] = 0.0;
      double s_cur = 0.0;
      const int max_iter = vdi_w + vdi_h + 4;
      const int32_t* rowp =
          a.counts + (long long)storage_row(a, cy) * vdi_w;
      // a list of an empty tile has count 0: no load
      auto load_count = [&](const int32_t* rp, int x, int y) -> int {
        if (kTiles && !((s_tiles[(y >> 3) * c.lt_wpr + (x >> 8)] >> ((x >> 3) & 31)) & 1u))
          return 0;
        return __ldg(rp + x);
      };
      // The count of the next list is requested before the current list is
      // shaded (the DDA step does not depend on it), so its load latency
      // overlaps an iteration instead of stalling the next one.
      int cnt = load_count(rowp, cx, cy);
      const bool ranged = VDI_RANGE_AHEAD && fast && a.list_range != nullptr;
      const float2* rng_base = reinterpret_cast<const float2*>(a.list_range);
      float2 rng = make_float2(0.f, 0.f);
      if (ranged) rng = __ldg(rng_base + (rowp - a.counts) + cx);
      for (;;) {
        const bool xs = t_max_x <= t_max_y;
        const double tmin = xs ? t_max_x : t_max_y;
        nvis += 1;
        // the step, branch-free (a divergent x / y branch serialises the
        // warp on its few y-steppers); the crossed boundary is the next s_cur
        const double nx = t_max_x + t_delta_x, ny = t_max_y + t_delta_y;
        t_max_x = xs ? nx : t_max_x;
        t_max_y = xs ? t_max_y : ny;
        const int ncx = cx + (xs ? step_x : 0);
        const int ncy = cy + (xs ? 0 : step_y);
        const bool last = tmin >= 1.0 || nvis >= max_iter || (unsigned)ncx >= (unsigned)vdi_w ||
                          (unsigned)ncy >= (unsigned)vdi_h;
        const int32_t* nrowp = rowp;
        int ncnt = 0;
        if (!last) {
          if (!kBands) {
            nrowp = a.counts + (long long)ncy * vdi_w;
          } else if (!xs) {
            nrowp = a.counts + (long long)storage_row(a, ncy) * vdi_w;
          }
          ncnt = load_count(nrowp, ncx, ncy);
        }
        float2 nrng = rng;
        if (ranged && !last) nrng = __ldg(rng_base + (nrowp - a.counts) + ncx);
        if (cnt > 0) {
          bool go = true;
          if (ranged) {
            // the range test of shade_list, on the prefetched range
            double s_exit = dmin(tmin, 1.0);
            if (s_exit < s_cur) s_exit = s_cur;
            const double z0 = sm.a0z[t], dz = sm.cdz[t];
            go = !(z0 + s_exit * dz < (double)rng.x || z0 + s_cur * dz > (double)rng.y);
          }
          const long long lidx = (rowp - a.counts) + cx;
          if (go && shade_list<kMask>(c, sm, t, cx, cy, lidx, cnt, s_cur, tmin, fast, !ranged))
            break;
        }
        if (last) break;
        cx = ncx;
        cy = ncy;
        rowp = nrowp;
        s_cur = tmin;
        cnt = ncnt;
        rng = nrng;
      }
    }
    const double acc_a = sm.acc_a[t];
    const double wgt = 1.0 - acc_a;
    const long long pix = (long long)lrow * a.out_w + col;
    double2* o = reinterpret_cast<double2*>(a.image + pix * 4);
    o[0] = make_double2(sm.acc_r[t] + wgt * a.bg[0] * a.bg[3],
                        sm.acc_g[t] + wgt * a.bg[1] * a.bg[3]);
    o[1] = make_double2(sm.acc_b[t] + wgt * a.bg[2] * a.bg[3], acc_a + wgt * a.bg[3]);
    const int nint = sm.nint[t], nsearch = sm.nsearch[t];
    if (a.lists_visited) a.lists_visited[pix] = nvis;
    if (a.segs_intersected) a.segs_intersected[pix] = nint;
    if (a.lists_searched && a.counters_exact) a.lists_searched[pix] = nsearch;
    if (a.stat_sums) {
      sm.sum_vis[t] += nvis;
      sm.sum_int[t] += nint;
      sm.sum_srch[t] += a.counters_exact ? nsearch : 0;
    }
  }
}

template <bool kTiles, bool kMask, bool kBands, bool kDyn>
__global__ void __launch_bounds__(kRenderThreads, VDI_RENDER_MINB) render_kernel(const __grid_constant__ RenderConst c) {
  const VdiRenderArgs& a = c.a;
  extern __shared__ uint32_t s_tiles[];
  __shared__ ShadeSmem sm;
  if (kTiles) {
    for (int k = threadIdx.x; k < c.lt_words; k += blockDim.x) s_tiles[k] = __ldg(a.list_tiles + k);
    __syncthreads();
  }
  // per-thread counter sums across the thread's tiles
  sm.sum_vis[threadIdx.x] = sm.sum_int[threadIdx.x] = sm.sum_srch[threadIdx.x] = 0ull;
  const int n_tiles = (int)(c.n_slots >> 5);
  if (kDyn) {
    // resident grid; each warp takes the next tile from a.tile_counter, so
    // the tiles in flight stay a compact front of the image (as the block
    // scheduler keeps them) while no block waits on its slowest warp
    const int lane = threadIdx.x & 31;
    for (;;) {
      unsigned tile = 0;
      if (lane == 0) tile = atomicAdd(a.tile_counter, 1u);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile >= (unsigned)n_tiles) break;
      render_tile<kTiles, kMask, kBands>(c, sm, s_tiles, (int)tile);
    }
    // the last warp out resets the counter for the next launch
    if (lane == 0) {
      __threadfence();
      const unsigned total = gridDim.x * (blockDim.x >> 5);
      if (atomicAdd(a.tile_counter + 1, 1u) == total - 1) {
        a.tile_counter[0] = 0u;
        a.tile_counter[1] = 0u;
        __threadfence();
      }
    }
  } else {
    const int tile = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (tile < n_tiles)
      render_tile<kTiles, kMask, kBands>(c, sm, s_tiles, tile);
  }
  if (a.stat_sums) {
    unsigned long long sv = sm.sum_vis[threadIdx.x], si = sm.sum_int[threadIdx.x],
                       ss = sm.sum_srch[threadIdx.x];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, off);
      si += __shfl_xor_sync(0xffffffffu, si, off);
      ss += __shfl_xor_sync(0xffffffffu, ss, off);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(a.stat_sums + 0, sv);
      atomicAdd(a.stat_sums + 1, si);
      atomicAdd(a.stat_sums + 2, ss);
    }
  }
}

int render_launch(const VdiRenderArgs* args, cudaStream_t stream) {
  RenderConst c;
  c.a = *args;
  if (c.a.band_rows <= 0) c.a.band_rows = 16;
  if (c.a.band_stride <= 0) c.a.band_stride = 1;
  if (c.a.vdi_band_rows <= 0) c.a.vdi_band_rows = 16;
  if (c.a.vdi_band_world <= 0) c.a.vdi_band_world = 1;
  c.local_h = local_rows(args->out_h, c.a.band_rows, c.a.band_stride, c.a.band_offset);
  c.tiles_x = (args->out_w + kTileW - 1) / kTileW;
  c.rfn = 1.0 / (c.a.far - c.a.near);
  const long long tiles_y = (c.local_h + kTileH - 1) / kTileH;
  c.n_slots = (long long)c.tiles_x * tiles_y * 32;
  if (c.n_slots == 0) return VDI_OK;
  const long long blocks = (c.n_slots + kRenderThreads - 1) / kRenderThreads;
  c.lt_wpr = lt_words_per_row(c.a.vdi_w);
  const long long ltw = (long long)c.lt_wpr * ((c.a.vdi_h + kListTile - 1) / kListTile);
  // staged when it fits next to the resident blocks' registers (<= 32 KiB)
  c.lt_words = c.a.list_tiles && ltw <= 8192 ? (int)ltw : 0;
  const bool mask = c.a.grid_zmask != nullptr && c.a.gz <= 64;
  const size_t smem = sizeof(uint32_t) * (size_t)c.lt_words;
  // kBands: the VDI is an all-gathered band-sharded one (storage-row map)
  void (*fn)(RenderConst);
  const bool bands = c.a.vdi_band_world > 1 || c.a.vdi_row_map;
  const bool dyn = c.a.tile_counter != nullptr;
#define VDI_RK(T, M, B) \
  (dyn ? render_kernel<T, M, B, true> : render_kernel<T, M, B, false>)
  if (bands)
    fn = c.lt_words ? (mask ? VDI_RK(true, true, true) : VDI_RK(true, false, true))
                    : (mask ? VDI_RK(false, true, true) : VDI_RK(false, false, true));
  else
    fn = c.lt_words ? (mask ? VDI_RK(true, true, false) : VDI_RK(true, false, false))
                    : (mask ? VDI_RK(false, true, false) : VDI_RK(false, false, false));
#undef VDI_RK
  if (smem > 0) {
    const cudaError_t e =
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(VDI_ELAUNCH, "render smem: %s", cudaGetErrorString(e));
  }
  long long grid = blocks;
  if (dyn) {
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kRenderThreads, smem) !=
            cudaSuccess)
      return set_error(VDI_ELAUNCH, "render occupancy query: %s",
                       cudaGetErrorString(cudaGetLastError()));
    const long long resident = (long long)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > resident) grid = resident;
  }
  fn<<<(unsigned)grid, kRenderThreads, smem, stream>>>(c);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "render launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// vdi_grid_zmask: one thread per grid column; bit cz of its word is
// grid[cz][cgy][cgx] > 0 (consecutive threads read consecutive cells).
__global__ void grid_zmask_kernel(const uint32_t* __restrict__ grid, int gx, int gy, int gz,
                                  uint64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = gx * gy;
  if (i >= n) return;
  uint64_t m = 0;
  for (int cz = 0; cz < gz; ++cz)
    if (__ldg(grid + (long long)cz * n + i) > 0u) m |= 1ull << cz;
  out[i] = m;
}

int grid_zmask(const uint32_t* grid, int gx, int gy, int gz, uint64_t* out, cudaStream_t stream) {
  const int n = gx * gy;
  grid_zmask_kernel<<<(n + 255) / 256, 256, 0, stream>>>(grid, gx, gy, gz, out);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "grid_zmask launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// vdi_list_ranges: one thread per list; min front / max back over its
// entries (fronts and backs are contiguous runs of the list-SoA slot).
__global__ void list_ranges_kernel(const float* __restrict__ segs,
                                   const int32_t* __restrict__ counts, long long n_lists, int n_sg,
                                   float2* __restrict__ out) {
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n_lists) return;
  int n = __ldg(counts + l);
  n = n < 0 ? 0 : (n > n_sg ? n_sg : n);
  const float* ls = segs + l * (long long)list_stride(n_sg);
  const float* fronts = ls + front_off(n_sg);
  const float* backs = ls + back_off(n_sg);
  float lo = INFINITY, hi = -INFINITY;
  bool nan = false;
  for (int k = 0; k < n; ++k) {
    const float f = __ldg(fronts + k), b = __ldg(backs + k);
    nan |= f != f || b != b;
    lo = fminf(lo, f);
    hi = fmaxf(hi, b);
  }
  out[l] = nan ? make_float2(-INFINITY, INFINITY) : make_float2(lo, hi);
}

int list_ranges(const float* segs, const int32_t* counts, long long n_lists, int n_sg, float* out,
                cudaStream_t stream) {
  list_ranges_kernel<<<(unsigned)((n_lists + 255) / 256), 256, 0, stream>>>(
      segs, counts, n_lists, n_sg, reinterpret_cast<float2*>(out));
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "list_ranges launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// vdi_list_tiles: lane j of a warp owns tile (ty, 32 w + j) and scans its
// 8x8 counts (eight 32-byte row pieces per lane, contiguous across the warp);
// the warp's ballot is one bitmap word.
__global__ void list_tiles_kernel(const VdiRenderArgs a, uint32_t* __restrict__ tiles, int wpr,
                                  int n_words) {
  const int lane = threadIdx.x & 31;
  const int word = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (word >= n_words) return;  // warp-uniform
  const int ty = word / wpr, txi = (word - ty * wpr) * 32 + lane;
  const int x0 = txi * kListTile;
  bool any = false;
  if (x0 < a.vdi_w) {
    const int x1 = min(x0 + kListTile, a.vdi_w);
    const int y1 = min((ty + 1) * kListTile, a.vdi_h);
    for (int y = ty * kListTile; y < y1 && !any; ++y) {
      const int32_t* row = a.counts + (long long)vdi_storage_row(y, a.vdi_band_rows,
                                                                   a.vdi_band_world,
                                                                   a.vdi_rows_per_rank) *
                                          a.vdi_w;
      for (int x = x0; x < x1; ++x) any |= __ldg(row + x) > 0;
    }
  }
  const unsigned b = __ballot_sync(0xffffffffu, any);
  if (lane == 0) tiles[word] = b;
}

size_t list_tiles_words(int vdi_w, int vdi_h) {
  if (vdi_w < 1 || vdi_h < 1) return 0;
  return (size_t)lt_words_per_row(vdi_w) * (size_t)((vdi_h + kListTile - 1) / kListTile);
}

int list_tiles(const VdiRenderArgs* args, uint32_t* tiles, cudaStream_t stream) {
  VdiRenderArgs a = *args;
  if (a.vdi_band_rows <= 0) a.vdi_band_rows = 16;
  if (a.vdi_band_world <= 0) a.vdi_band_world = 1;
  const long long words = (long long)list_tiles_words(a.vdi_w, a.vdi_h);
  if (words == 0) return VDI_OK;
  const long long blocks = (words * 32 + 127) / 128;
  list_tiles_kernel<<<(unsigned)blocks, 128, 0, stream>>>(a, tiles, lt_words_per_row(a.vdi_w),
                                                         (int)words);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "list_tiles launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// raycast.py:494-518 composite_lists: the identity-view oracle, per list a
// front-to-back composite of its stored supersegments (no traversal, no
// search, no length correction). One thread per list (natural row order).
__global__ void composite_lists_kernel(const float* __restrict__ segs,
                                       const int32_t* __restrict__ counts, int w, int h,
                                       int n_sg, double early_term, double bg0, double bg1,
                                       double bg2, double bg3, double* __restrict__ img) {
  const long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= (long long)w * h) return;
  const float* ls = segs + l * (long long)list_stride(n_sg);
  const float4* c4 = reinterpret_cast<const float4*>(ls);
  double r = 0.0, g = 0.0, b = 0.0, a = 0.0;
  const int n = counts[l];
  for (int k = 0; k < n; ++k) {
    const float4 s = c4[k];
    const double wt = 1.0 - a;
    r += wt * (double)s.x;
    g += wt * (double)s.y;
    b += wt * (double)s.z;
    a += wt * (double)s.w;
    if (a >= early_term) break;
  }
  const double wt = 1.0 - a;
  double2* o = reinterpret_cast<double2*>(img + 4 * l);
  o[0] = make_double2(r + wt * bg0 * bg3, g + wt * bg1 * bg3);
  o[1] = make_double2(b + wt * bg2 * bg3, a + wt * bg3);
}

int composite_lists(const float* segs, const int32_t* counts, int w, int h, int n_sg,
                    double early_term, const double* bg, double* img, cudaStream_t stream) {
  const long long n = (long long)w * h;
  if (n <= 0) return VDI_OK;
  composite_lists_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
      segs, counts, w, h, n_sg, early_term, bg[0], bg[1], bg[2], bg[3], img);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "composite launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// raycast.py:159-222 _dda_cells for a batch of NDC chords (a0, a1: 6 f64 per
// query): the visited cells (cx, cy) and (z_entry, z_exit, s_entry, s_exit),
// at most w + h + 4 per query; n_out[q] = cells visited. One thread per chord
// (the same DDA arithmetic as render_kernel).
__global__ void dda_kernel(const double* __restrict__ chords, long long nq, int w, int h,
                           int cap, int32_t* __restrict__ cells, double* __restrict__ zs,
                           int32_t* __restrict__ n_out) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double x0 = chords[6 * q], y0 = chords[6 * q + 1], z0 = chords[6 * q + 2];
  const double dx = chords[6 * q + 3] - x0, dy = chords[6 * q + 4] - y0,
               dz = chords[6 * q + 5] - z0;
  int cx = clampi(floor_ll((x0 + 1.0) * w / 2.0), 0, w - 1);
  int cy = clampi(floor_ll((y0 + 1.0) * h / 2.0), 0, h - 1);
  const int step_x = dx > 0 ? 1 : (dx < 0 ? -1 : 0);
  const int step_y = dy > 0 ? 1 : (dy < 0 ? -1 : 0);
  double t_max_x = INFINITY, t_delta_x = INFINITY, t_max_y = INFINITY, t_delta_y = INFINITY;
  if (step_x != 0) {
    const double bx = -1.0 + 2.0 * (double)(cx + (step_x > 0 ? 1 : 0)) / w;
    t_max_x = (bx - x0) / dx;
    t_delta_x = (2.0 / w) / fabs(dx);
  }
  if (step_y != 0) {
    const double by = -1.0 + 2.0 * (double)(cy + (step_y > 0 ? 1 : 0)) / h;
    t_max_y = (by - y0) / dy;
    t_delta_y = (2.0 / h) / fabs(dy);
  }
  int n = 0;
  double s_cur = 0.0;
  for (int it = 0; it < w + h + 4 && n < cap; ++it) {
    double s_exit = dmin(dmin(t_max_x, t_max_y), 1.0);
    if (s_exit < s_cur) s_exit = s_cur;
    const long long o = q * (long long)cap + n;
    cells[2 * o] = cx;
    cells[2 * o + 1] = cy;
    zs[4 * o] = z0 + s_cur * dz;
    zs[4 * o + 1] = z0 + s_exit * dz;
    zs[4 * o + 2] = s_cur;
    zs[4 * o + 3] = s_exit;
    n += 1;
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
    if (cx < 0 || cx >= w || cy < 0 || cy >= h) break;
  }
  n_out[q] = n;
}

int dda_cells(const double* chords, long long nq, int w, int h, int cap, int32_t* cells,
              double* zs, int32_t* n_out, cudaStream_t stream) {
  if (nq <= 0) return VDI_OK;
  dda_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, stream>>>(chords, nq, w, h, cap, cells, zs,
                                                               n_out);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "dda launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// raycast.py:237-255 project_ray_to_ndc for a batch of world rays (origin,
// dir: 6 f64): clip to the volume box and the generation frustum; out (a0,
// a1: 6 f64) and hit flags.
__global__ void project_kernel(const double* __restrict__ rays, long long n, const RenderConst c,
                               double* __restrict__ out, int32_t* __restrict__ hit_out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double o[3] = {rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]};
  const double d[3] = {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]};
  double ta, tb, fa, fb;
  int hit = 0;
  if (clip_aabb(o, d, c.a.aabb, ta, tb) && clip_frustum(c.a.gen_pv, o, d, fa, fb)) {
    const double t0 = dmax(dmax(ta, fa), 0.0), t1 = dmin(tb, fb);
    if (t1 > t0) {
      hit = 1;
      xform(c.a.gen_pv, o[0] + t0 * d[0], o[1] + t0 * d[1], o[2] + t0 * d[2], out[6 * i],
            out[6 * i + 1], out[6 * i + 2]);
      xform(c.a.gen_pv, o[0] + t1 * d[0], o[1] + t1 * d[1], o[2] + t1 * d[2], out[6 * i + 3],
            out[6 * i + 4], out[6 * i + 5]);
    }
  }
  hit_out[i] = hit;
}

int project_rays(const double* rays, long long n, const double* gen_pv, const double* aabb,
                 double* out, int32_t* hit, cudaStream_t stream) {
  if (n <= 0) return VDI_OK;
  RenderConst c;
  memset(&c, 0, sizeof(c));
  for (int k = 0; k < 16; ++k) c.a.gen_pv[k] = gen_pv[k];
  for (int k = 0; k < 6; ++k) c.a.aabb[k] = aabb[k];
  project_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(rays, n, c, out, hit);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "project launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// Batch form of find_first_supersegment (raycast.py:144-156) for the A1 fuzz.
__global__ void find_first_batch_kernel(const float* fronts, const float* backs,
                                        const int32_t* counts, int n_max, const double* d_entry,
                                        const double* d_exit, const int32_t* seeds,
                                        int32_t* out_index, int32_t* out_seed, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int seed;
  out_index[i] = find_first(fronts + i * n_max, backs + i * n_max, counts[i], d_entry[i],
                            d_exit[i], seeds[i], seed);
  out_seed[i] = seed;
}

int find_first_batch(const float* fronts, const float* backs, const int32_t* counts,
                     int32_t n_max, const double* d_entry, const double* d_exit,
                     const int32_t* seeds, int32_t* out_index, int32_t* out_seed,
                     int64_t n, cudaStream_t stream) {
  if (n <= 0) return VDI_OK;
  find_first_batch_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
      fronts, backs, counts, n_max, d_entry, d_exit, seeds, out_index, out_seed, n);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "find_first launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
