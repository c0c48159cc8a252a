// vdi_volume.cu -- per-volume acceleration data for generation.
//
// Brick maxima for exact empty-space skipping: brick (bx, by, bz) of edge
// B = 2^log2 stores the maximum raw voxel over voxels [B*b, min(B*b + B, n-1)]
// on every axis, i.e. the brick's cells plus the +1 trilinear halo
// (volume.py:190-205 reads voxels i and i+1 with i = floor(q (n-1)) clamped to
// n-2). A sample whose cell lies in a brick whose maximum classifies below the
// first non-zero-alpha LUT row is exactly transparent (see sample_at in
// vdi_gen.cu). The reduction is integer/float max, so it is exact.
#include "vdi_common.cuh"
#include "vdi_internal.h"

namespace vdi {

template <typename T>
__global__ void brick_max_kernel(const T* __restrict__ vol, T* __restrict__ out, int nx, int ny,
                                 int nz, int log2b, int bx_n, int by_n, long long n_bricks) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_bricks) return;
  const int bx = (int)(b % bx_n);
  const int by = (int)((b / bx_n) % by_n);
  const int bz = (int)(b / ((long long)bx_n * by_n));
  const int B = 1 << log2b;
  const int x0 = bx * B, y0 = by * B, z0 = bz * B;
  const int x1 = min(x0 + B, nx - 1), y1 = min(y0 + B, ny - 1), z1 = min(z0 + B, nz - 1);
  T m = vol[((long long)z0 * ny + y0) * nx + x0];
  for (int z = z0; z <= z1; ++z)
    for (int y = y0; y <= y1; ++y) {
      const T* row = vol + ((long long)z * ny + y) * nx;
      for (int x = x0; x <= x1; ++x) {
        const T v = __ldg(row + x);
        m = v > m ? v : m;
      }
    }
  out[b] = m;
}

int brick_max(const void* volume, int voxel_type, int nx, int ny, int nz, int log2b, void* out,
              cudaStream_t stream) {
  const int B = 1 << log2b;
  const int bx = (nx + B - 1) / B, by = (ny + B - 1) / B, bz = (nz + B - 1) / B;
  const long long n = (long long)bx * by * bz;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  switch (voxel_type) {
    case VDI_VOXEL_U8:
      brick_max_kernel<<<blocks, 128, 0, stream>>>(static_cast<const uint8_t*>(volume),
                                                   static_cast<uint8_t*>(out), nx, ny, nz, log2b,
                                                   bx, by, n);
      break;
    case VDI_VOXEL_U16:
      brick_max_kernel<<<blocks, 128, 0, stream>>>(static_cast<const uint16_t*>(volume),
                                                   static_cast<uint16_t*>(out), nx, ny, nz,
                                                   log2b, bx, by, n);
      break;
    case VDI_VOXEL_F32:
      brick_max_kernel<<<blocks, 128, 0, stream>>>(static_cast<const float*>(volume),
                                                   static_cast<float*>(out), nx, ny, nz, log2b,
                                                   bx, by, n);
      break;
    default:
      return set_error(VDI_EINVAL, "bad voxel_type %d", voxel_type);
  }
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "brick_max launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
