// vdi_grid.cu -- AccelGrid accumulation and segment-layout conversion.
//
// grid_kernel reproduces _accumulate_grid (generate.py:322-346): every
// supersegment of list (lx, ly) increments the (cz, cy, cx) cells covering the
// list's NDC footprint (integer floor divisions; 1080 / 16 is not integral, so
// a list can straddle two rows of cells) and the view-depth slabs its
// [front, back] spans (depth = b / (a - z), generate.py:349-354). Counts are
// integers, so accumulating them with atomics in any order is bit-exact.
#include "vdi_common.cuh"
#include "vdi_internal.h"

namespace vdi {

struct GridConst {
  VdiGridArgs a;
  int local_h;
};

__global__ void grid_kernel(const GridConst c) {
  const VdiGridArgs& a = c.a;
  const long long list = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (list >= (long long)c.local_h * a.width) return;
  const int n = a.counts[list];
  if (n == 0) return;
  const int lrow = (int)(list / a.width), lx = (int)(list % a.width);
  const long long ly =
      image_row(lrow, a.band_rows, a.band_stride, a.band_offset, a.row_base, a.row_count);
  const int cy0 = (int)((ly * a.gy) / a.height);
  const int cy1 = (int)(((ly + 1) * a.gy - 1) / a.height);
  const int cx0 = (int)(((long long)lx * a.gx) / a.width);
  const int cx1 = (int)((((long long)lx + 1) * a.gx - 1) / a.width);
  const float* ls = a.segs + list * (long long)list_stride(a.n_sg);
  const float* fronts = ls + front_off(a.n_sg);
  const float* backs = ls + back_off(a.n_sg);
  const double fn = a.far - a.near;
  for (int k = 0; k < n; ++k) {
    const double zf = fronts[k], zb = backs[k];
    const double d0 = a.proj_b / (a.proj_a - zf);
    const double d1 = a.proj_b / (a.proj_a - zb);
    long long k0 = (long long)floor((d0 - a.near) / fn * a.gz);
    long long k1 = (long long)floor((d1 - a.near) / fn * a.gz);
    k0 = k0 < 0 ? 0 : (k0 > a.gz - 1 ? a.gz - 1 : k0);
    k1 = k1 < 0 ? 0 : (k1 > a.gz - 1 ? a.gz - 1 : k1);
    for (long long cz = k0; cz <= k1; ++cz)
      for (int cy = cy0; cy <= cy1; ++cy)
        for (int cx = cx0; cx <= cx1; ++cx)
          atomicAdd(a.grid + (cz * a.gy + cy) * a.gx + cx, 1u);
  }
}

int grid_launch(const VdiGridArgs* args, cudaStream_t stream) {
  GridConst c;
  c.a = *args;
  if (c.a.band_rows <= 0) c.a.band_rows = 16;
  if (c.a.band_stride <= 0) c.a.band_stride = 1;
  c.local_h = launch_rows(args->height, c.a.band_rows, c.a.band_stride, c.a.band_offset,
                          c.a.row_count);
  cudaError_t err;
  if (args->clear) {
    err = cudaMemsetAsync(args->grid, 0,
                          sizeof(uint32_t) * (size_t)args->gx * args->gy * args->gz, stream);
    if (err != cudaSuccess)
      return set_error(VDI_ELAUNCH, "grid memset: %s", cudaGetErrorString(err));
  }
  const long long n = (long long)c.local_h * args->width;
  if (n == 0) return VDI_OK;
  grid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(c);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "grid launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// list-SoA <-> the reference's (.., n_sg, 6) AoS; one thread per supersegment.
__global__ void soa_to_aos_kernel(const float* __restrict__ soa, float* __restrict__ aos,
                                  long long n, int n_sg) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long list = i / n_sg;
  const int k = (int)(i - list * n_sg);
  const float* s = soa + list * list_stride(n_sg);
  const float4 c = reinterpret_cast<const float4*>(s)[k];
  float* o = aos + i * 6;
  o[0] = s[front_off(n_sg) + k];
  o[1] = s[back_off(n_sg) + k];
  o[2] = c.x;
  o[3] = c.y;
  o[4] = c.z;
  o[5] = c.w;
}

__global__ void aos_to_soa_kernel(const float* __restrict__ aos, float* __restrict__ soa,
                                  long long n, int n_sg) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long list = i / n_sg;
  const int k = (int)(i - list * n_sg);
  const float* in = aos + i * 6;
  float* s = soa + list * list_stride(n_sg);
  s[front_off(n_sg) + k] = in[0];
  s[back_off(n_sg) + k] = in[1];
  reinterpret_cast<float4*>(s)[k] = make_float4(in[2], in[3], in[4], in[5]);
  if (k == 0)  // zero the alignment pad so the buffer is fully defined
    for (int p = 6 * n_sg; p < list_stride(n_sg); ++p) s[p] = 0.0f;
}

int segs_convert(const float* src, float* dst, int64_t n_lists, int32_t n_sg, bool to_aos,
                 cudaStream_t stream) {
  const long long n = (long long)n_lists * n_sg;
  if (n == 0) return VDI_OK;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (to_aos) soa_to_aos_kernel<<<blocks, 256, 0, stream>>>(src, dst, n, n_sg);
  else aos_to_soa_kernel<<<blocks, 256, 0, stream>>>(src, dst, n, n_sg);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "layout launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
