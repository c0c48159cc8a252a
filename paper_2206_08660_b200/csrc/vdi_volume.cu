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
#include <algorithm>
#include <type_traits>

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

// u8 bricks of 8 (nx % 8 == 0, 8-byte aligned volume): each row of a brick
// (9 voxels with the +1 overlap) is one aligned 8-byte load plus one byte,
// reduced with SIMD byte maxima.
__global__ void brick_max_u8x8_kernel(const uint8_t* __restrict__ vol, uint8_t* __restrict__ out,
                                      int nx, int ny, int nz, int bx_n, int by_n,
                                      long long n_bricks) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_bricks) return;
  const int bx = (int)(b % bx_n);
  const int by = (int)((b / bx_n) % by_n);
  const int bz = (int)(b / ((long long)bx_n * by_n));
  const int x0 = bx * 8, y0 = by * 8, z0 = bz * 8;
  const int y1 = min(y0 + 8, ny - 1), z1 = min(z0 + 8, nz - 1);
  const bool has_next = x0 + 8 <= nx - 1;  // the overlap voxel x0 + 8 exists
  unsigned m4 = 0u, me = 0u;
  for (int z = z0; z <= z1; ++z)
    for (int y = y0; y <= y1; ++y) {
      const uint8_t* row = vol + ((long long)z * ny + y) * nx + x0;
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(row));
      m4 = __vmaxu4(m4, __vmaxu4(w.x, w.y));
      if (has_next) me = max(me, (unsigned)__ldg(row + 8));
    }
  const unsigned a = max(m4 & 0xffu, (m4 >> 8) & 0xffu);
  const unsigned c = max((m4 >> 16) & 0xffu, m4 >> 24);
  out[b] = (uint8_t)max(max(a, c), me);
}

int brick_max(const void* volume, int voxel_type, int nx, int ny, int nz, int log2b, void* out,
              cudaStream_t stream) {
  const int B = 1 << log2b;
  const int bx = (nx + B - 1) / B, by = (ny + B - 1) / B, bz = (nz + B - 1) / B;
  const long long n = (long long)bx * by * bz;
  const unsigned blocks = (unsigned)((n + 127) / 128);
  switch (voxel_type) {
    case VDI_VOXEL_U8:
      if (log2b == 3 && nx % 8 == 0 && (reinterpret_cast<uintptr_t>(volume) & 7) == 0) {
        brick_max_u8x8_kernel<<<blocks, 128, 0, stream>>>(static_cast<const uint8_t*>(volume),
                                                          static_cast<uint8_t*>(out), nx, ny, nz,
                                                          bx, by, n);
        break;
      }
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

// Corner records (include/vdi_b200.h vdi_volume_cells): one thread per cell,
// x fastest, so the 8 corner reads coalesce across a warp (rows x and x+1 of
// four (y, z) rows) and the record stores are contiguous.
template <typename T>
struct CellRecord;
template <>
struct CellRecord<uint8_t> {
  static __device__ __forceinline__ void store(void* out, long long i, const uint8_t v[8]) {
    uint2 r;
    r.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((unsigned)v[3] << 24);
    r.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((unsigned)v[7] << 24);
    reinterpret_cast<uint2*>(out)[i] = r;
  }
};
template <>
struct CellRecord<uint16_t> {
  static __device__ __forceinline__ void store(void* out, long long i, const uint16_t v[8]) {
    uint4 r;
    r.x = v[0] | ((unsigned)v[1] << 16);
    r.y = v[2] | ((unsigned)v[3] << 16);
    r.z = v[4] | ((unsigned)v[5] << 16);
    r.w = v[6] | ((unsigned)v[7] << 16);
    reinterpret_cast<uint4*>(out)[i] = r;
  }
};
template <>
struct CellRecord<float> {
  static __device__ __forceinline__ void store(void* out, long long i, const float v[8]) {
    float4* o = reinterpret_cast<float4*>(out) + 2 * i;
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

// Brick mask for the corner records: a brick whose maximum classifies to
// alpha 0 (the generation / DVR empty-space test, vdi_sample.cuh) is never
// sampled, so its cells need no record. bmax == nullptr: write every cell.
template <typename T>
struct CellMask {
  const T* bmax;
  int lb, bnx, bny;
  double ess_max;
  __device__ __forceinline__ bool skip(int x, int y, int z) const {
    if (!bmax) return false;
    const T v = __ldg(bmax + ((long long)(z >> lb) * bny + (y >> lb)) * bnx + (x >> lb));
    double d;
    if (sizeof(T) == 1) d = (double)__fdiv_rn((float)v, 255.0f);
    else if (sizeof(T) == 2) d = (double)__fdiv_rn((float)v, 65535.0f);
    else d = (double)v;
    return d <= ess_max;
  }
};

template <typename T>
__global__ void cells_kernel(const T* __restrict__ vol, void* __restrict__ out, int nx, int ny,
                             int nz, const CellMask<T> mask) {
  const long long n = (long long)nx * ny * nz;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % nx);
    const long long yz = i / nx;
    const int y = (int)(yz % ny), z = (int)(yz / ny);
    if (mask.skip(x, y, z)) continue;
    const int dx = x + 1 < nx ? 1 : 0;
    const long long dy = y + 1 < ny ? nx : 0;
    const long long dz = z + 1 < nz ? (long long)nx * ny : 0;
    const T* p = vol + i;
    T v[8];
    v[0] = __ldg(p);
    v[1] = __ldg(p + dx);
    v[2] = __ldg(p + dy);
    v[3] = __ldg(p + dy + dx);
    v[4] = __ldg(p + dz);
    v[5] = __ldg(p + dz + dx);
    v[6] = __ldg(p + dz + dy);
    v[7] = __ldg(p + dz + dy + dx);
    CellRecord<T>::store(out, i, v);
  }
}

// u8 fast path (nx % 4 == 0): a thread builds the records of 4 cells along x
// from one aligned 32-bit word plus the next byte of each of the 4 (y, z)
// rows, and stores them as two 16-byte writes.
__global__ void cells_u8x4_kernel(const uint8_t* __restrict__ vol, uint4* __restrict__ out,
                                  int nx, int ny, int nz, const uint8_t* __restrict__ bmax,
                                  int lb, int bnx, int bny, int skip_max) {
  // one (y, z) row per block iteration: 32-bit row arithmetic, no division
  // per thread. A 4-cell group is skipped when its brick's maximum is <=
  // skip_max (the u8 form of CellMask: the largest v with v / 255 <= ess_max;
  // -1 = no mask).
  const int qx = nx >> 2;
  const int rows = ny * nz;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
    const int y = row % ny, z = row / ny;
    const long long dy = y + 1 < ny ? nx : 0;
    const long long dz = z + 1 < nz ? (long long)nx * ny : 0;
    const long long off[4] = {0, dy, dz, dy + dz};
    const long long rbase = (long long)row * nx;
    const uint8_t* brow = bmax ? bmax + ((long long)(z >> lb) * bny + (y >> lb)) * bnx : nullptr;
    for (int q = threadIdx.x; q < qx; q += blockDim.x) {
      const int x = q * 4;
      // the 4 cells share a brick (x % 4 == 0, edge >= 4)
      if (brow && (int)__ldg(brow + (x >> lb)) <= skip_max) continue;
      const long long base = rbase + x;
      const bool last = x + 4 >= nx;
      unsigned w[4], e[4];  // rows (y,z), (y+1,z), (y,z+1), (y+1,z+1)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        w[r] = __ldg(reinterpret_cast<const unsigned*>(vol + base + off[r]));
        // voxel x+4 (clamped to x+3 at the row end: the last cell repeats it)
        e[r] = last ? (w[r] >> 24) : (unsigned)__ldg(vol + base + off[r] + 4);
      }
      // cell j: rec[2j] = (v000 v001 v010 v011) = bytes j, j+1 of rows 0 and 1,
      // rec[2j+1] the same of rows 2 and 3; byte 4 of a row is e[r]
      unsigned n[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) n[r] = __funnelshift_r(w[r], e[r], 8);  // bytes 1..4
      const uint4 o0 = make_uint4(__byte_perm(w[0], w[1], 0x5410), __byte_perm(w[2], w[3], 0x5410),
                                  __byte_perm(w[0], w[1], 0x6521), __byte_perm(w[2], w[3], 0x6521));
      const uint4 o1 = make_uint4(__byte_perm(w[0], w[1], 0x7632), __byte_perm(w[2], w[3], 0x7632),
                                  __byte_perm(n[0], n[1], 0x7632), __byte_perm(n[2], n[3], 0x7632));
      uint4* o = out + 2 * (base >> 2);
      o[0] = o0;
      o[1] = o1;
    }
  }
}

// The same records, a thread walking its 4-cell group down z: rows (y, z+1)
// and (y+1, z+1) of one step are rows (y, z) and (y+1, z) of the next, so a
// step loads two row words (+ their next bytes) instead of four, and the row
// index math is paid once per z run. An empty brick's z range is skipped
// without loads (the window is reloaded at the next non-empty brick).
// Item = (y, chunk of kCellsZ slices); threads over the x groups.
constexpr int kCellsZ = 32;
constexpr int kCellsBatch = 4;
__global__ void cells_u8x4z_kernel(const uint8_t* __restrict__ vol, uint4* __restrict__ out,
                                   int nx, int ny, int nz, const uint8_t* __restrict__ bmax,
                                   int lb, int bnx, int bny, int skip_max) {
  const int qx = nx >> 2;
  const int nzc = (nz + kCellsZ - 1) / kCellsZ;
  const long long plane = (long long)nx * ny;
  for (int item = blockIdx.x; item < ny * nzc; item += gridDim.x) {
    const int y = item % ny, zb = (item / ny) * kCellsZ;
    const int ze = min(zb + kCellsZ, nz);
    const long long dy = y + 1 < ny ? nx : 0;
    for (int q = threadIdx.x; q < qx; q += blockDim.x) {
      const int x = q * 4;
      const bool last = x + 4 >= nx;
      const uint8_t* col = vol + (long long)y * nx + x;  // (x, y, z = 0)
      // voxels x .. x+3 (one word) and x + 4 (clamped to x + 3 at the row end)
      auto word = [&](const uint8_t* p, unsigned& w, unsigned& e) {
        w = __ldg(reinterpret_cast<const unsigned*>(p));
        e = last ? (w >> 24) : (unsigned)__ldg(p + 4);
      };
      unsigned w0 = 0, w1 = 0, e0 = 0, e1 = 0;  // rows (y, z), (y + 1, z)
      bool have = false;
      int z = zb;
      while (z < ze) {
        const int zend = min(((z >> lb) + 1) << lb, ze);  // this brick's slices
        if (bmax && (int)__ldg(bmax + ((long long)(z >> lb) * bny + (y >> lb)) * bnx +
                               (x >> lb)) <= skip_max) {
          z = zend;
          have = false;
          continue;
        }
        if (!have) {
          word(col + (long long)z * plane, w0, e0);
          word(col + (long long)z * plane + dy, w1, e1);
          have = true;
        }
        // kCellsBatch slices per batch: their row words are all requested
        // before the first record is built (memory-level parallelism)
        while (z < zend) {
          const int nb = zend - z < kCellsBatch ? zend - z : kCellsBatch;
          unsigned wa[kCellsBatch], ea[kCellsBatch], wb[kCellsBatch], eb[kCellsBatch];
#pragma unroll
          for (int j = 0; j < kCellsBatch; ++j) {
            if (j < nb) {
              const int zz = z + j;
              const long long dz = zz + 1 < nz ? plane : 0;
              const uint8_t* r0 = col + (long long)zz * plane + dz;  // rows (y, zz + 1)
              word(r0, wa[j], ea[j]);
              word(r0 + dy, wb[j], eb[j]);                            // and (y + 1, zz + 1)
            }
          }
#pragma unroll
          for (int j = 0; j < kCellsBatch; ++j) {
            if (j < nb) {
              const unsigned w2 = wa[j], e2 = ea[j], w3 = wb[j], e3 = eb[j];
              const unsigned n0 = __funnelshift_r(w0, e0, 8), n1 = __funnelshift_r(w1, e1, 8);
              const unsigned n2 = __funnelshift_r(w2, e2, 8), n3 = __funnelshift_r(w3, e3, 8);
              const uint4 o0 =
                  make_uint4(__byte_perm(w0, w1, 0x5410), __byte_perm(w2, w3, 0x5410),
                             __byte_perm(w0, w1, 0x6521), __byte_perm(w2, w3, 0x6521));
              const uint4 o1 =
                  make_uint4(__byte_perm(w0, w1, 0x7632), __byte_perm(w2, w3, 0x7632),
                             __byte_perm(n0, n1, 0x7632), __byte_perm(n2, n3, 0x7632));
              uint4* o = out + 2 * ((long long)(((z + j) * ny + y)) * (nx >> 2) + q);
              o[0] = o0;
              o[1] = o1;
              w0 = w2;
              w1 = w3;
              e0 = e2;
              e1 = e3;
            }
          }
          z += nb;
        }
      }
    }
  }
}

int volume_cells(const void* volume, int voxel_type, int nx, int ny, int nz, void* out,
                 cudaStream_t stream, const void* brick_max, int brick_log2, double ess_max) {
  const bool masked = brick_max != nullptr && ess_max >= 0.0 && brick_log2 >= 2;
  const int B = 1 << (brick_log2 > 0 ? brick_log2 : 3);
  const int bnx = (nx + B - 1) / B, bny = (ny + B - 1) / B;
  auto mk = [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    return CellMask<T>{masked ? static_cast<const T*>(brick_max) : nullptr, brick_log2, bnx, bny,
                       ess_max};
  };
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long n = (long long)nx * ny * nz;
  long long blocks = (n + 255) / 256;
  if (blocks > (long long)sms * 64) blocks = (long long)sms * 64;
  switch (voxel_type) {
    case VDI_VOXEL_U8:
      if (nx % 4 == 0) {
        // the largest u8 value the samplers classify as always transparent
        int skip_max = -1;
        if (masked)
          for (int v = 0; v < 256; ++v)
            if ((double)((float)v / 255.0f) <= ess_max) skip_max = v;
#ifndef VDI_CELLS_Z
#define VDI_CELLS_Z 1  // 1: cells_u8x4z_kernel (z walks), 0: one (y, z) row per block pass
#endif
        if (VDI_CELLS_Z) {
          const long long items = (long long)ny * ((nz + kCellsZ - 1) / kCellsZ);
          cells_u8x4z_kernel<<<(unsigned)std::min<long long>(items, (long long)sms * 16), 256, 0,
                               stream>>>(
              static_cast<const uint8_t*>(volume), static_cast<uint4*>(out), nx, ny, nz,
              masked ? static_cast<const uint8_t*>(brick_max) : nullptr,
              brick_log2 > 0 ? brick_log2 : 3, bnx, bny, skip_max);
        } else {
          cells_u8x4_kernel<<<(unsigned)std::min<long long>((long long)ny * nz,
                                                            (long long)sms * 32),
                              256, 0, stream>>>(
              static_cast<const uint8_t*>(volume), static_cast<uint4*>(out), nx, ny, nz,
              masked ? static_cast<const uint8_t*>(brick_max) : nullptr, brick_log2, bnx, bny,
              skip_max);
        }
      }
      else
        cells_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const uint8_t*>(volume),
                                                           out, nx, ny, nz, mk((uint8_t*)nullptr));
      break;
    case VDI_VOXEL_U16:
      cells_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const uint16_t*>(volume),
                                                         out, nx, ny, nz, mk((uint16_t*)nullptr));
      break;
    case VDI_VOXEL_F32:
      cells_kernel<<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const float*>(volume), out,
                                                         nx, ny, nz, mk((float*)nullptr));
      break;
    default:
      return set_error(VDI_EINVAL, "bad voxel_type %d", voxel_type);
  }
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess)
    return set_error(VDI_ELAUNCH, "volume_cells launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi

// ------------------------------------------------------------- synthetic
// Richtmyer-Meshkov-shaped u8 volume for config C5, built
// on the device because the 2048 x 2048 x 1920 brick (7.5 GiB) would take
// minutes to synthesise on the host. A mixing band |z - h(x, y)| < w around
// a perturbed interface h = 0.5 + sum_m A_m sin(2 pi k_m . (x, y) + phi_m);
// inside it a 4-octave value-noise fbm mapped to 60..255, outside 0. Integer
// hashing and f32 arithmetic: the same bytes on every run and every B200.
namespace vdi {

__device__ __forceinline__ uint32_t hash3(uint32_t x, uint32_t y, uint32_t z, uint32_t s) {
  uint32_t h = s ^ 0x9e3779b9u;
  h ^= x * 0x85ebca6bu;
  h = (h << 13) | (h >> 19);
  h ^= y * 0xc2b2ae35u;
  h = (h << 11) | (h >> 21);
  h ^= z * 0x27d4eb2fu;
  h ^= h >> 16;
  h *= 0x7feb352du;
  h ^= h >> 15;
  h *= 0x846ca68bu;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ float lattice(int x, int y, int z, uint32_t s) {
  return (float)(hash3((uint32_t)x, (uint32_t)y, (uint32_t)z, s) >> 8) * (1.0f / 16777216.0f);
}

__device__ __forceinline__ float smooth(float t) { return t * t * (3.0f - 2.0f * t); }

__device__ float value_noise(float px, float py, float pz, uint32_t s) {
  const float fx = floorf(px), fy = floorf(py), fz = floorf(pz);
  const int ix = (int)fx, iy = (int)fy, iz = (int)fz;
  const float tx = smooth(px - fx), ty = smooth(py - fy), tz = smooth(pz - fz);
  float c[2][2];
  for (int b = 0; b < 2; ++b)
    for (int a = 0; a < 2; ++a) {
      const float v0 = lattice(ix, iy + a, iz + b, s), v1 = lattice(ix + 1, iy + a, iz + b, s);
      c[b][a] = v0 + (v1 - v0) * tx;
    }
  const float c0 = c[0][0] + (c[0][1] - c[0][0]) * ty;
  const float c1 = c[1][0] + (c[1][1] - c[1][0]) * ty;
  return c0 + (c1 - c0) * tz;
}

struct RmModes {
  float kx[12], ky[12], amp[12], phase[12];
  float band;
  uint32_t seed;
};

// Writes the box [o, o + s) of the nx x ny x nz volume, stored (sz, sy, sx).
__global__ void synth_rm_kernel(uint8_t* __restrict__ out, int nx, int ny, int nz, int ox,
                                int oy, int oz, int bx, int by, int bz, const RmModes m) {
  const long long cols = (long long)bx * by;
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
       c += (long long)gridDim.x * blockDim.x) {
    const int ix = ox + (int)(c % bx), iy = oy + (int)(c / bx);
    const float x = (ix + 0.5f) / nx, y = (iy + 0.5f) / ny;
    float h = 0.5f;
    for (int k = 0; k < 12; ++k)
      h += m.amp[k] * sinf(6.28318530718f * (m.kx[k] * x + m.ky[k] * y) + m.phase[k]);
    for (int jz = 0; jz < bz; ++jz) {
      const int iz = oz + jz;
      const float z = (iz + 0.5f) / nz;
      uint8_t v = 0;
      if (fabsf(z - h) < m.band) {
        float f = 0.0f, a = 1.0f, norm = 0.0f, fr = 8.0f;
        for (int o = 0; o < 4; ++o) {
          f += a * value_noise(x * fr, y * fr, z * fr, m.seed + 977u * o);
          norm += a;
          a *= 0.5f;
          fr *= 2.0f;
        }
        f /= norm;
        v = (uint8_t)(60.0f + 195.0f * fminf(fmaxf(f, 0.0f), 1.0f) + 0.5f);
      }
      out[(long long)jz * cols + c] = v;
    }
  }
}

int synth_rm_u8(uint8_t* out, int nx, int ny, int nz, const int32_t* box, const float* modes,
                float band, uint32_t seed, cudaStream_t stream) {
  const int ox = box ? box[0] : 0, oy = box ? box[1] : 0, oz = box ? box[2] : 0;
  const int bx = box ? box[3] : nx, by = box ? box[4] : ny, bz = box ? box[5] : nz;
  if (ox < 0 || oy < 0 || oz < 0 || bx < 1 || by < 1 || bz < 1 || ox + bx > nx ||
      oy + by > ny || oz + bz > nz)
    return set_error(VDI_EINVAL, "synth box outside the volume");
  RmModes m;
  for (int k = 0; k < 12; ++k) {
    m.kx[k] = modes[4 * k];
    m.ky[k] = modes[4 * k + 1];
    m.amp[k] = modes[4 * k + 2];
    m.phase[k] = modes[4 * k + 3];
  }
  m.band = band;
  m.seed = seed;
  const long long cols = (long long)bx * by;
  long long blocks = (cols + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  synth_rm_kernel<<<(unsigned)blocks, 256, 0, stream>>>(out, nx, ny, nz, ox, oy, oz, bx, by, bz,
                                                        m);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "synth launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
