// vdi_search.cuh -- the Alg. 2 supersegment search (raycast.py:51-141) and
// the small integer helpers shared by the novel-view renderer (vdi_render.cu)
// and the preview renderer (vdi_preview.cu). f32 depths are promoted to f64
// before every compare, as in the reference.
#pragma once

#include "vdi_common.cuh"

namespace vdi {

// raycast.py:51-62: smallest j in [start, stop] with backs[j] >= d.
__device__ __forceinline__ int bins(const float* backs, double d, int start, int stop) {
  int lo = start, hi = stop;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((double)backs[mid] >= d) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// raycast.py:65-76: largest j in [start, stop] with fronts[j] <= d.
__device__ __forceinline__ int bins_front(const float* fronts, double d, int start, int stop) {
  int lo = start, hi = stop;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((double)fronts[mid] <= d) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// raycast.py:79-141 _find_first. Returns index or -1; `seed` gets the seed.
__device__ __forceinline__ int find_first(const float* fronts, const float* backs, int count,
                                          double d_entry, double d_exit, int p, int& seed) {
  if (count == 0) {
    seed = p;
    return -1;
  }
  int index;
  if (d_entry <= d_exit) {
    index = -1;
    int bs_start = -1, bs_end = -1;
    if (p < 0) {
      bs_start = 0;
      bs_end = count - 1;
    } else {
      const double b1 = p < count ? (double)backs[p] : INFINITY;
      const double b0 = (p - 1 >= 0 && p - 1 < count) ? (double)backs[p - 1] : -INFINITY;
      const int interval = (b1 >= d_entry ? 1 : 0) + (b0 >= d_entry ? 1 : 0);
      if (interval == 0) {
        bs_start = p + 1;
        bs_end = count - 1;
      } else if (interval == 2) {
        bs_start = 0;
        bs_end = p - 1;
      } else if (p < count) {
        index = p;
      } else {
        bs_start = 0;
        bs_end = count - 1;
      }
    }
    if (bs_end != -1) {
      if (bs_start > bs_end) {
        index = bs_start < 0 ? 0 : bs_start;
        if (index > count - 1) index = count - 1;
      } else {
        index = bins(backs, d_entry, bs_start, bs_end < count - 1 ? bs_end : count - 1);
      }
    }
    seed = index;
    if ((double)backs[index] < d_entry) return -1;
    if ((double)fronts[index] > d_exit) return -1;
    return index;
  }
  if (p < 0) {
    index = bins_front(fronts, d_entry, 0, count - 1);
  } else {
    const double f1 = p < count ? (double)fronts[p] : INFINITY;
    const double f0 = (p + 1 >= 0 && p + 1 < count) ? (double)fronts[p + 1] : INFINITY;
    if (p < count && f1 <= d_entry && f0 > d_entry) {
      index = p;
    } else if (f1 > d_entry) {
      index = bins_front(fronts, d_entry, 0, p - 1 > 0 ? p - 1 : 0);
    } else {
      index = bins_front(fronts, d_entry, p + 1 < count - 1 ? p + 1 : count - 1, count - 1);
    }
  }
  if (index > count - 1) index = count - 1;
  seed = index;
  if ((double)fronts[index] > d_entry) return -1;
  if ((double)backs[index] < d_exit) return -1;
  return index;
}

__device__ __forceinline__ long long floor_ll(double x) { return (long long)floor(x); }
__device__ __forceinline__ int clampi(long long v, int lo, int hi) {
  return (int)(v < lo ? lo : (v > hi ? hi : v));
}

}  // namespace vdi
