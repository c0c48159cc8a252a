// vdi_internal.h -- host-side glue shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include "../../include/vdi_b200.h"

namespace vdi {

int set_error(int code, const char* fmt, ...);

// Number of image rows r in [0, h) with ((r / band_rows) % stride) == offset.
inline int local_rows(int h, int band_rows, int stride, int offset) {
  if (stride <= 1) return h;
  int n = 0;
  for (int b = offset; b * band_rows < h; b += stride) {
    const int rem = h - b * band_rows;
    n += rem < band_rows ? rem : band_rows;
  }
  return n;
}

// Rows of a launch: the contiguous range when row_count > 0, else the band map.
inline int launch_rows(int h, int band_rows, int stride, int offset, int row_count) {
  return row_count > 0 ? row_count : local_rows(h, band_rows, stride, offset);
}

int gen_launch(const VdiGenArgs* a, cudaStream_t stream);
size_t gen_workspace_bytes(const VdiGenArgs* a, int recommended);
int grid_launch(const VdiGridArgs* a, cudaStream_t stream);
int render_launch(const VdiRenderArgs* a, cudaStream_t stream);
size_t list_tiles_words(int vdi_w, int vdi_h);
int list_tiles(const VdiRenderArgs* args, uint32_t* tiles, cudaStream_t stream);
int grid_zmask(const uint32_t* grid, int gx, int gy, int gz, uint64_t* out, cudaStream_t stream);
int list_ranges(const float* segs, const int32_t* counts, long long n_lists, int n_sg, float* out,
                cudaStream_t stream);
int dvr_launch(const VdiDvrArgs* a, cudaStream_t stream);
int gen_rays(const VdiGenArgs* a, const double* rays, const double* gammas_in, long long n,
             int mode, cudaStream_t stream);
int composite_lists(const float* segs, const int32_t* counts, int w, int h, int n_sg,
                    double early_term, const double* bg, double* img, cudaStream_t stream);
int dda_cells(const double* chords, long long nq, int w, int h, int cap, int32_t* cells,
              double* zs, int32_t* n_out, cudaStream_t stream);
int project_rays(const double* rays, long long n, const double* gen_pv, const double* aabb,
                 double* out, int32_t* hit, cudaStream_t stream);
size_t encode_workspace_bytes(int width, int height);
int encode_vdi1(const VdiEncodeArgs* a, cudaStream_t stream);
int decode_vdi1_lists(const uint8_t* src, int width, int rows, int n_sg, int32_t* counts,
                      float* segs, void* workspace, size_t ws_bytes, cudaStream_t stream);
size_t lz4_workspace_bytes(size_t n_max);
int lz4_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev, uint8_t* dst,
                 unsigned long long* out_len, void* workspace, size_t ws_bytes,
                 cudaStream_t stream);
size_t lzx_workspace_bytes(size_t n_max);
int lzx_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev, uint8_t* dst,
                 unsigned long long* out_len, void* workspace, size_t ws_bytes,
                 cudaStream_t stream);
int validate_vdi(const VdiValidateArgs* a, cudaStream_t stream);
int synth_rm_u8(uint8_t* out, int nx, int ny, int nz, const int32_t* box, const float* modes,
                float band, uint32_t seed, cudaStream_t stream);
int preview_launch(const VdiPreviewArgs* a, cudaStream_t stream);
int bilinear_upsample(const double* src, int w, int h, double* dst, int out_w, int out_h,
                      int channels, cudaStream_t stream);
int find_first_batch(const float* fronts, const float* backs, const int32_t* counts,
                     int32_t n_max, const double* d_entry, const double* d_exit,
                     const int32_t* seeds, int32_t* out_index, int32_t* out_seed,
                     int64_t n, cudaStream_t stream);
int brick_max(const void* volume, int voxel_type, int nx, int ny, int nz, int log2b, void* out,
              cudaStream_t stream);
int volume_cells(const void* volume, int voxel_type, int nx, int ny, int nz, void* out,
                 cudaStream_t stream, const void* brick_max = nullptr, int brick_log2 = 0,
                 double ess_max = -1.0);
int selftest_arith(long long n, unsigned long long seed, unsigned long long* bad,
                   cudaStream_t stream);
int segs_convert(const float* src, float* dst, int64_t n_lists, int32_t n_sg, bool to_aos,
                 cudaStream_t stream);

}  // namespace vdi
