// vdi_capi.cu -- the extern "C" entry points of include/vdi_b200.h:
// argument validation (mirroring the reference's ValueErrors where the Python
// layer has not already raised them), thread-local error text, dispatch.
#include <cstdarg>
#include <cstdio>

#include "vdi_internal.h"

namespace vdi {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace vdi

using vdi::set_error;

extern "C" {

const char* vdi_last_error(void) { return vdi::g_err; }

int vdi_abi_version(void) { return VDI_ABI_VERSION; }

size_t vdi_gen_workspace_bytes(const VdiGenArgs* a) {
  if (!a || !(a->step > 0)) return 0;
  return vdi::gen_workspace_bytes(a, 1);
}

size_t vdi_gen_workspace_min_bytes(const VdiGenArgs* a) {
  if (!a || !(a->step > 0)) return 0;
  return vdi::gen_workspace_bytes(a, 0);
}

int vdi_gen_launch(const VdiGenArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->volume || !a->lut || !a->counts || !a->segs || !a->workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  if (a->nx < 2 || a->ny < 2 || a->nz < 2)
    return set_error(VDI_EINVAL, "dims components must be >= 2 for trilinear sampling");
  if (a->lut_n < 2 || a->lut_n > 4096) return set_error(VDI_EINVAL, "lut_n out of range");
  if (a->width < 1 || a->height < 1) return set_error(VDI_EINVAL, "empty viewport");
  if (a->n_sg < 1) return set_error(VDI_EINVAL, "n_sg must be >= 1");
  if (!(a->eps > 0 && a->eps < 1)) return set_error(VDI_EINVAL, "epsilon must be in (0, 1)");
  if (!(a->step > 0) || !(a->lref > 0)) return set_error(VDI_EINVAL, "step must be > 0");
  if (a->band_stride > 1 && (a->band_offset < 0 || a->band_offset >= a->band_stride))
    return set_error(VDI_EINVAL, "band_offset out of range");
  if (reinterpret_cast<uintptr_t>(a->segs) % 16 != 0)
    return set_error(VDI_EINVAL, "segs must be 16-byte aligned");
  return vdi::gen_launch(a, static_cast<cudaStream_t>(stream));
}

int vdi_grid_launch(const VdiGridArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->segs || !a->counts || !a->grid) return set_error(VDI_EINVAL, "null device pointer");
  if (a->gx < 1 || a->gy < 1 || a->gz < 1) return set_error(VDI_EINVAL, "bad grid dims");
  return vdi::grid_launch(a, static_cast<cudaStream_t>(stream));
}

int vdi_render_launch(const VdiRenderArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->segs || !a->counts || !a->grid || !a->image)
    return set_error(VDI_EINVAL, "null device pointer");
  if (!(a->early_term > 0.0 && a->early_term <= 1.0))
    return set_error(VDI_EINVAL, "early_term_alpha must be in (0, 1]");
  if (a->vdi_w < 1 || a->vdi_h < 1 || a->n_sg < 1 || a->out_w < 1 || a->out_h < 1)
    return set_error(VDI_EINVAL, "bad sizes");
  if (a->gx < 1 || a->gy < 1 || a->gz < 1) return set_error(VDI_EINVAL, "bad grid dims");
  if (reinterpret_cast<uintptr_t>(a->segs) % 16 != 0)
    return set_error(VDI_EINVAL, "segs must be 16-byte aligned");
  return vdi::render_launch(a, static_cast<cudaStream_t>(stream));
}

size_t vdi_list_tiles_words(int32_t vdi_w, int32_t vdi_h) {
  return vdi::list_tiles_words(vdi_w, vdi_h);
}

int vdi_list_tiles(const VdiRenderArgs* a, uint32_t* tiles, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->counts || !tiles) return set_error(VDI_EINVAL, "null device pointer");
  if (a->vdi_w < 1 || a->vdi_h < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::list_tiles(a, tiles, static_cast<cudaStream_t>(stream));
}

int vdi_grid_zmask(const uint32_t* grid, int32_t gx, int32_t gy, int32_t gz, uint64_t* out,
                   vdi_stream_t stream) {
  if (!grid || !out) return set_error(VDI_EINVAL, "null device pointer");
  if (gx < 1 || gy < 1 || gz < 1 || gz > 64) return set_error(VDI_EINVAL, "bad grid dims");
  return vdi::grid_zmask(grid, gx, gy, gz, out, static_cast<cudaStream_t>(stream));
}

int vdi_list_ranges(const float* segs, const int32_t* counts, int64_t n_lists, int32_t n_sg,
                    float* out, vdi_stream_t stream) {
  if (n_lists < 0 || n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  if (n_lists == 0) return VDI_OK;
  if (!segs || !counts || !out) return set_error(VDI_EINVAL, "null device pointer");
  return vdi::list_ranges(segs, counts, n_lists, n_sg, out, static_cast<cudaStream_t>(stream));
}

int vdi_dvr_launch(const VdiDvrArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->volume || !a->lut || !a->image || !a->workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  if (a->nx < 2 || a->ny < 2 || a->nz < 2)
    return set_error(VDI_EINVAL, "dims components must be >= 2 for trilinear sampling");
  if (a->lut_n < 2 || a->lut_n > 4096) return set_error(VDI_EINVAL, "lut_n out of range");
  if (a->width < 1 || a->height < 1) return set_error(VDI_EINVAL, "empty viewport");
  if (!(a->step > 0) || !(a->lref > 0)) return set_error(VDI_EINVAL, "step must be > 0");
  if (a->band_stride > 1 && (a->band_offset < 0 || a->band_offset >= a->band_stride))
    return set_error(VDI_EINVAL, "band_offset out of range");
  if (reinterpret_cast<uintptr_t>(a->image) % 16 != 0)
    return set_error(VDI_EINVAL, "image must be 16-byte aligned");
  return vdi::dvr_launch(a, static_cast<cudaStream_t>(stream));
}

int vdi_preview_launch(const VdiPreviewArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->segs || !a->counts || !a->grid || !a->image || !a->workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  if (!(a->d_r > 0.0 && a->d_r <= 1.0)) return set_error(VDI_EINVAL, "d_r must be in (0, 1]");
  if (!(a->early_term > 0.0 && a->early_term <= 1.0))
    return set_error(VDI_EINVAL, "early_term must be in (0, 1]");
  if (a->vdi_w < 1 || a->vdi_h < 1 || a->n_sg < 1 || a->out_w < 1 || a->out_h < 1)
    return set_error(VDI_EINVAL, "bad sizes");
  if (a->gx < 1 || a->gy < 1 || a->gz < 1) return set_error(VDI_EINVAL, "bad grid dims");
  if (reinterpret_cast<uintptr_t>(a->segs) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(a->image) % 16 != 0)
    return set_error(VDI_EINVAL, "segs and image must be 16-byte aligned");
  return vdi::preview_launch(a, static_cast<cudaStream_t>(stream));
}

int vdi_bilinear_upsample(const double* src, int32_t w, int32_t h, double* dst, int32_t out_w,
                          int32_t out_h, int32_t channels, vdi_stream_t stream) {
  if (!src || !dst) return set_error(VDI_EINVAL, "null device pointer");
  if (w < 1 || h < 1 || out_w < 1 || out_h < 1 || channels < 1)
    return set_error(VDI_EINVAL, "bad sizes");
  return vdi::bilinear_upsample(src, w, h, dst, out_w, out_h, channels,
                                static_cast<cudaStream_t>(stream));
}

size_t vdi_vdi1_max_bytes(int32_t width, int32_t height, int32_t n_sg, int32_t gx, int32_t gy,
                          int32_t gz) {
  if (width < 0 || height < 0 || n_sg < 0 || gx < 0 || gy < 0 || gz < 0) return 0;
  const size_t n = (size_t)width * (size_t)height;
  return VDI_VDI1_HEADER_BYTES + 2 * n + 24 * n * (size_t)n_sg +
         4 * (size_t)gx * (size_t)gy * (size_t)gz;
}

size_t vdi_encode_workspace_bytes(int32_t width, int32_t height) {
  if (width < 0 || height < 0) return 0;
  return vdi::encode_workspace_bytes(width, height);
}

int vdi_encode_vdi1(const VdiEncodeArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->segs || !a->counts || !a->grid || !a->out || !a->workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  if (a->width < 1 || a->height < 1 || a->n_sg < 1 || a->gx < 1 || a->gy < 1 || a->gz < 1)
    return set_error(VDI_EINVAL, "bad sizes");
  if ((long long)a->width * a->height * (long long)a->n_sg > (1ll << 40))
    return set_error(VDI_EINVAL, "VDI too large");
  return vdi::encode_vdi1(a, static_cast<cudaStream_t>(stream));
}

int vdi_decode_vdi1_lists(const uint8_t* src, int32_t width, int32_t rows, int32_t n_sg,
                          int32_t* counts, float* segs, void* workspace, size_t workspace_bytes,
                          vdi_stream_t stream) {
  if (!src || !counts || !segs || !workspace) return set_error(VDI_EINVAL, "null device pointer");
  if (width < 1 || rows < 0 || n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  if (reinterpret_cast<uintptr_t>(segs) % 16 != 0)
    return set_error(VDI_EINVAL, "segs must be 16-byte aligned");
  return vdi::decode_vdi1_lists(src, width, rows, n_sg, counts, segs, workspace, workspace_bytes,
                                static_cast<cudaStream_t>(stream));
}

size_t vdi_lz4_max_bytes(size_t n) { return n + n / 255 + 16; }

size_t vdi_lz4_workspace_bytes(size_t n_max) { return vdi::lz4_workspace_bytes(n_max); }

int vdi_lz4_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev,
                     uint8_t* dst, unsigned long long* out_len, void* workspace,
                     size_t workspace_bytes, vdi_stream_t stream) {
  if ((!src && n_max) || !dst || !out_len || !workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  return vdi::lz4_compress(src, n_max, n_dev, dst, out_len, workspace, workspace_bytes,
                           static_cast<cudaStream_t>(stream));
}

size_t vdi_lz4_exact_workspace_bytes(size_t n_max) { return vdi::lzx_workspace_bytes(n_max); }

int vdi_lz4_compress_exact(const uint8_t* src, size_t n_max, const unsigned long long* n_dev,
                           uint8_t* dst, unsigned long long* out_len, void* workspace,
                           size_t workspace_bytes, vdi_stream_t stream) {
  if ((!src && n_max) || !dst || !out_len || !workspace)
    return set_error(VDI_EINVAL, "null device pointer");
  return vdi::lzx_compress(src, n_max, n_dev, dst, out_len, workspace, workspace_bytes,
                           static_cast<cudaStream_t>(stream));
}

int vdi_validate(const VdiValidateArgs* a, vdi_stream_t stream) {
  if (!a) return set_error(VDI_EINVAL, "null args");
  if (!a->segs || !a->counts || !a->result) return set_error(VDI_EINVAL, "null device pointer");
  if (a->width < 1 || a->height < 1 || a->n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::validate_vdi(a, static_cast<cudaStream_t>(stream));
}

int vdi_synth_rm_u8(uint8_t* out, int32_t nx, int32_t ny, int32_t nz, const int32_t* box_host,
                    const float* modes_host, float band, uint32_t seed, vdi_stream_t stream) {
  if (!out || !modes_host) return set_error(VDI_EINVAL, "null pointer");
  if (nx < 2 || ny < 2 || nz < 2) return set_error(VDI_EINVAL, "bad dims");
  return vdi::synth_rm_u8(out, nx, ny, nz, box_host, modes_host, band, seed,
                          static_cast<cudaStream_t>(stream));
}

int vdi_gen_rays(const VdiGenArgs* a, const double* rays, const double* gammas_in,
                 int64_t n_rays, int32_t mode, vdi_stream_t stream) {
  if (!a || (!rays && n_rays > 0)) return set_error(VDI_EINVAL, "null pointer");
  if (!a->volume || !a->lut || !a->counts || !a->segs)
    return set_error(VDI_EINVAL, "null device pointer");
  if (a->nx < 2 || a->ny < 2 || a->nz < 2) return set_error(VDI_EINVAL, "bad dims");
  if (a->n_sg < 1) return set_error(VDI_EINVAL, "n_sg must be >= 1");
  if (!(a->eps > 0 && a->eps < 1)) return set_error(VDI_EINVAL, "epsilon must be in (0, 1)");
  if (!(a->step > 0) || !(a->lref > 0)) return set_error(VDI_EINVAL, "step must be > 0");
  if (mode < 0 || mode > 2) return set_error(VDI_EINVAL, "bad mode");
  if ((a->voxel_type & ~15) != 0) return set_error(VDI_EINVAL, "plain voxel grids only");
  return vdi::gen_rays(a, rays, gammas_in, n_rays, mode, static_cast<cudaStream_t>(stream));
}

int vdi_composite_lists(const float* segs, const int32_t* counts, int32_t w, int32_t h,
                        int32_t n_sg, double early_term, const double* bg_host, double* image,
                        vdi_stream_t stream) {
  if (!segs || !counts || !bg_host || !image) return set_error(VDI_EINVAL, "null pointer");
  if (w < 1 || h < 1 || n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  if (!(early_term > 0.0 && early_term <= 1.0))
    return set_error(VDI_EINVAL, "early_term_alpha must be in (0, 1]");
  return vdi::composite_lists(segs, counts, w, h, n_sg, early_term, bg_host, image,
                              static_cast<cudaStream_t>(stream));
}

int vdi_dda_cells(const double* chords, int64_t n, int32_t w, int32_t h, int32_t cap,
                  int32_t* cells, double* zs, int32_t* counts, vdi_stream_t stream) {
  if ((!chords || !cells || !zs || !counts) && n > 0) return set_error(VDI_EINVAL, "null pointer");
  if (w < 1 || h < 1 || cap < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::dda_cells(chords, n, w, h, cap, cells, zs, counts, static_cast<cudaStream_t>(stream));
}

int vdi_project_rays(const double* rays, int64_t n, const double* gen_pv_host,
                     const double* aabb_host, double* out, int32_t* hit, vdi_stream_t stream) {
  if ((!rays || !out || !hit) && n > 0) return set_error(VDI_EINVAL, "null pointer");
  if (!gen_pv_host || !aabb_host) return set_error(VDI_EINVAL, "null host pointer");
  return vdi::project_rays(rays, n, gen_pv_host, aabb_host, out, hit,
                           static_cast<cudaStream_t>(stream));
}

int vdi_find_first_batch(const float* fronts, const float* backs, const int32_t* counts,
                         int32_t n_max, const double* d_entry, const double* d_exit,
                         const int32_t* seeds, int32_t* out_index, int32_t* out_seed,
                         int64_t n_queries, vdi_stream_t stream) {
  if (n_queries < 0 || n_max < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::find_first_batch(fronts, backs, counts, n_max, d_entry, d_exit, seeds, out_index,
                               out_seed, n_queries, static_cast<cudaStream_t>(stream));
}

int vdi_volume_brick_max(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny,
                         int32_t nz, int32_t brick_log2, void* out, vdi_stream_t stream) {
  if (!volume || !out) return set_error(VDI_EINVAL, "null device pointer");
  if (nx < 2 || ny < 2 || nz < 2 || brick_log2 < 1 || brick_log2 > 8)
    return set_error(VDI_EINVAL, "bad sizes");
  return vdi::brick_max(volume, voxel_type, nx, ny, nz, brick_log2, out,
                        static_cast<cudaStream_t>(stream));
}

size_t vdi_volume_cells_bytes(int32_t voxel_type, int32_t nx, int32_t ny, int32_t nz) {
  const size_t e = voxel_type == VDI_VOXEL_U8 ? 1 : voxel_type == VDI_VOXEL_U16 ? 2
                   : voxel_type == VDI_VOXEL_F32 ? 4 : 0;
  if (nx < 1 || ny < 1 || nz < 1) return 0;
  return 8 * e * (size_t)nx * (size_t)ny * (size_t)nz;
}

int vdi_volume_cells(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny, int32_t nz,
                     void* out, vdi_stream_t stream) {
  if (!volume || !out) return set_error(VDI_EINVAL, "null device pointer");
  if (nx < 2 || ny < 2 || nz < 2) return set_error(VDI_EINVAL, "bad sizes");
  if (reinterpret_cast<uintptr_t>(out) & 31) return set_error(VDI_EINVAL, "cells not 32-byte aligned");
  return vdi::volume_cells(volume, voxel_type, nx, ny, nz, out, static_cast<cudaStream_t>(stream));
}

int vdi_volume_cells_masked(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny,
                            int32_t nz, const void* brick_max, int32_t brick_log2, double ess_max,
                            void* out, vdi_stream_t stream) {
  if (!volume || !out || !brick_max) return set_error(VDI_EINVAL, "null device pointer");
  if (nx < 2 || ny < 2 || nz < 2) return set_error(VDI_EINVAL, "bad sizes");
  if (brick_log2 < 2 || brick_log2 > 10) return set_error(VDI_EINVAL, "bad brick_log2");
  if (reinterpret_cast<uintptr_t>(out) & 31) return set_error(VDI_EINVAL, "cells not 32-byte aligned");
  return vdi::volume_cells(volume, voxel_type, nx, ny, nz, out, static_cast<cudaStream_t>(stream),
                           brick_max, brick_log2, ess_max);
}

int vdi_selftest_arith(int64_t n, uint64_t seed, unsigned long long* bad,
                       vdi_stream_t stream) {
  if (!bad || n < 0) return set_error(VDI_EINVAL, "bad arguments");
  return vdi::selftest_arith(n, seed, bad, static_cast<cudaStream_t>(stream));
}

int vdi_segs_to_aos(const float* soa, float* aos, int64_t n_lists, int32_t n_sg,
                    vdi_stream_t stream) {
  if (n_lists < 0 || n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::segs_convert(soa, aos, n_lists, n_sg, true, static_cast<cudaStream_t>(stream));
}

int vdi_segs_from_aos(const float* aos, float* soa, int64_t n_lists, int32_t n_sg,
                      vdi_stream_t stream) {
  if (n_lists < 0 || n_sg < 1) return set_error(VDI_EINVAL, "bad sizes");
  return vdi::segs_convert(aos, soa, n_lists, n_sg, false, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
