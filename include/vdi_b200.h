/*
 * vdi_b200.h -- C ABI of the B200-native VDI generation / VDI raycasting path.
 *
 * The reference (vdikit 0.1.0, /root/reference/pkg) has no FFI: its hot path
 * is two numba kernels behind the Python functions `generate_vdi` and
 * `render_vdi`. The entry points below are the flat, C-like cut of those
 * kernels; the Python package paper_2206_08660_b200 binds
 * them with ctypes and keeps the reference's Python signatures on top.
 *
 *   vdi_gen_launch     replaces generate.py:276-319  _generate_kernel
 *                      (with _find_gamma_list generate.py:219-273,
 *                       _gen_list_pass generate.py:89-216, _emit generate.py:53-86)
 *   vdi_grid_launch    replaces generate.py:322-346  _accumulate_grid
 *   vdi_render_launch  replaces raycast.py:275-456   _render_kernel
 *                      (with _find_first raycast.py:79-141, _bins raycast.py:51-62)
 *   vdi_find_first_batch  batch form of raycast.py:144-156 find_first_supersegment
 *   vdi_dvr_launch     replaces dvr.py:21-89      _dvr_kernel (render_dvr's
 *                      ground-truth emission-absorption raycast)
 *   vdi_preview_launch replaces preview.py:49-205  _preview_kernel (point-sampled
 *                      preview through the AccelGrid)
 *   vdi_bilinear_upsample  replaces preview.py:208-223 bilinear_upsample
 *   vdi_encode_vdi1    replaces vdi.py:141-159    encode_vdi (VDI1 bytes, on device)
 *   vdi_lz4_compress_exact replaces lz4.py:51-114 _compress_kernel (byte-identical)
 *   vdi_lz4_compress   a chunk-parallel LZ4 block of the same format (decodable
 *                      by lz4.py:117-168, not byte-identical; faster)
 *   vdi_validate       replaces vdi.py:116-134    validate_vdi
 *   vdi_gen_rays       replaces generate.py:371-407 generate_list / find_gamma
 *                      (single-ray passes / bisections, batched)
 *   vdi_composite_lists replaces raycast.py:494-518 composite_lists
 *   vdi_dda_cells      replaces raycast.py:159-234 _dda_cells / dda_traverse (batched)
 *   vdi_project_rays   replaces raycast.py:237-255 project_ray_to_ndc (batched)
 *   vdi_segs_to_aos / vdi_segs_from_aos  device layout <-> the reference's
 *                      (H, W, n_sg, 6) f32 array (vdi.py:3-7, 23-24)
 *
 * Conventions
 *   - every pointer is a DEVICE pointer unless its name ends in _host;
 *   - matrices are row-major f64[16] holding the host's exact bits
 *     (Camera.proj_view / inv_proj_view, camera.py:108-112);
 *   - no entry point allocates or synchronises; all work is enqueued on
 *     `stream` (a cudaStream_t; NULL = legacy default stream);
 *   - return 0 on success, < 0 on bad arguments (VDI_EINVAL) or a launch
 *     error (VDI_ELAUNCH); vdi_last_error() gives a thread-local message.
 *
 * Device segment layout (VDI_LAYOUT_LIST_SOA): each list owns
 * vdi_list_stride(n_sg) = round_up(6*n_sg, 4) floats
 *   [rgba[0..n_sg) as float4 | front[0..n_sg) | back[0..n_sg) | pad]
 * so the Alg. 2 search touches only the contiguous `back` run and each
 * supersegment's colour is one aligned 16-byte load. VDI_LAYOUT_AOS is the
 * reference's [front, back, r, g, b, a] per supersegment.
 *
 * Row sharding: a "band map" (band_rows, band_stride, band_offset) selects
 * the image rows r with ((r / band_rows) % band_stride) == band_offset and
 * packs them densely, in order, into the output arrays ("local rows").
 * (band_rows, 1, 0) is the whole image in natural order.
 */
#ifndef VDI_B200_H
#define VDI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VDI_ABI_VERSION 8

#define VDI_OK 0
#define VDI_EINVAL (-1)
#define VDI_ELAUNCH (-2)

#define VDI_VOXEL_U8 0
#define VDI_VOXEL_U16 1
#define VDI_VOXEL_F32 2
/* Flag on VdiGenArgs.voxel_type: `volume` holds vdi_volume_cells() corner
 * records of the base type instead of the plain voxel grid. */
#define VDI_VOXEL_CELLS 16

#define VDI_LAYOUT_LIST_SOA 0
#define VDI_LAYOUT_AOS 1

typedef void* vdi_stream_t; /* cudaStream_t */

/* Floats per list in VDI_LAYOUT_LIST_SOA (16-byte aligned lists). */
static inline int32_t vdi_list_stride(int32_t n_sg) { return (6 * n_sg + 3) & ~3; }

/* Generation: one ray per viewport pixel, per-ray gamma bisection (Alg. 1 as
 * implemented in generate.py:219-273), supersegments written in
 * VDI_LAYOUT_LIST_SOA. Outputs are indexed by local row (band map). */
typedef struct VdiGenArgs {
  const void* volume;   /* (nz, ny, nx) x-fastest, voxel_type elements; with
                           VDI_VOXEL_CELLS, vdi_volume_cells() records */
  const float* lut;     /* (lut_n, 4) f32, TransferFunction.lut */
  const void* brick_max;/* vdi_volume_brick_max() of `volume`, or NULL (no skipping) */
  int32_t* counts;      /* OUT (local_h, width) */
  float* segs;          /* OUT (local_h, width, vdi_list_stride(n_sg)) list-SoA */
  double* gammas;       /* OUT (local_h, width), may be NULL */
  int32_t* passes;      /* OUT (local_h, width), may be NULL */
  int32_t* samples;     /* OUT executed samples per ray (R's loop semantics), may be NULL */
  void* workspace;      /* scratch, any content: queues, 1/n table, sample
                           cache. vdi_gen_workspace_bytes() is the recommended
                           size; less still works (rays that do not fit the
                           cache take more rounds / the fused fallback) down
                           to a minimum the launch checks (VDI_EINVAL). */
  size_t workspace_bytes;
  double pv[16];        /* generation proj*view */
  double inv_pv[16];
  double eye[3];
  double aabb[6];       /* lo xyz, hi xyz (volume.py:57-60) */
  double eps;           /* GenParams.epsilon */
  double gamma_init;
  double step;          /* resolved step (generate.py:38-50) */
  double lref;
  double ess_max;       /* normalised brick maximum at or below which every sample
                           classifies to alpha 0 exactly; < 0 disables skipping */
  int32_t voxel_type;
  int32_t nx, ny, nz;
  int32_t lut_n;
  int32_t width, height;
  int32_t n_sg, delta;
  int32_t band_rows, band_stride, band_offset;
  int32_t brick_log2;   /* brick edge 2^brick_log2 voxels */
  /* Resident box (volume bricked across GPUs): when sub_dims[0] > 0,
   * `volume` (and brick_max / corner records) hold only the voxels
   * [sub_origin, sub_origin + sub_dims) of the nx x ny x nz grid, stored
   * (sub_dims[2], sub_dims[1], sub_dims[0]) x-fastest; sub_origin must be a
   * multiple of the brick edge. Sample positions are unchanged, so results
   * equal the full-volume run when the box holds every cell the rays touch;
   * a touched cell outside it sets *sub_oob (device, may be NULL). */
  int32_t sub_origin[3];
  int32_t sub_dims[3];
  uint32_t* sub_oob;
  /* Contiguous row range (a load-balanced band of a bricked placement):
   * when row_count > 0, this launch's rays are image rows [row_base,
   * row_base + row_count) and band_rows / band_stride / band_offset are
   * ignored; local row j is image row row_base + j. */
  int32_t row_base, row_count;
} VdiGenArgs;

/* AccelGrid: per-cell supersegment counts (generate.py:322-346). `grid` is
 * (gz, gy, gx) u32 and is accumulated into (zero it first, or pass
 * clear=1). */
typedef struct VdiGridArgs {
  const float* segs;      /* list-SoA, local rows */
  const int32_t* counts;  /* local rows */
  uint32_t* grid;
  double near, far, proj_a, proj_b;
  int32_t width, height, n_sg;
  int32_t gx, gy, gz;
  int32_t band_rows, band_stride, band_offset;
  int32_t clear;
  int32_t row_base, row_count;  /* as VdiGenArgs */
} VdiGridArgs;

/* Novel-view rendering (raycast.py:275-456). The VDI is read through a band
 * map too (vdi_band_rows, vdi_band_world): list row r lives at storage row
 * ((r/b) / W)*b + (r%b) + ((r/b) % W) * rows_per_rank -- i.e. the layout an
 * all-gather of band-sharded generation leaves behind. (b, 1) = natural. */
typedef struct VdiRenderArgs {
  const float* segs;            /* list-SoA */
  const int32_t* counts;
  const uint32_t* grid;         /* (gz, gy, gx) */
  double* image;                /* OUT (local_out_h, out_w, 4) f64 premultiplied */
  int32_t* lists_visited;       /* OUT per pixel, may be NULL */
  int32_t* segs_intersected;    /* OUT per pixel, may be NULL */
  int32_t* lists_searched;      /* OUT per pixel, may be NULL */
  unsigned long long* stat_sums;/* OUT [3] += (visited, intersected, searched), may be NULL */
  double gen_pv[16];
  double gen_inv_pv[16];
  double new_inv_pv[16];
  double eye[3];                /* new camera position */
  double aabb[6];               /* Vdi.volume_aabb */
  double bg[4];                 /* straight RGBA background */
  double near, far, proj_a, proj_b;
  double early_term;
  int32_t vdi_w, vdi_h, n_sg;
  int32_t gx, gy, gz;
  int32_t out_w, out_h;
  int32_t use_ess;
  int32_t vdi_band_rows, vdi_band_world, vdi_rows_per_rank;
  int32_t band_rows, band_stride, band_offset;  /* output-row sharding */
  /* optional (may be NULL): occupancy bitmap of 8x8-list tiles
   * (vdi_list_tiles). A step of the DDA into a list of an empty tile is
   * counted as a visit without reading the list's count (it is 0), so the
   * image and every counter are unchanged. */
  const uint32_t* list_tiles;
  /* optional (may be NULL; ignored when gz > 64): vdi_grid_zmask() of
   * `grid`, one 64-bit word per grid column (cgy, cgx) whose bit cz is set
   * iff grid[cz][cgy][cgx] > 0. The ESS test (raycast.py:352-372) then ORs
   * the words of its column range and tests its slab range in one compare
   * instead of reading every cell; the result is the same. */
  const uint64_t* grid_zmask;
  /* 1: every list's fronts and backs are non-decreasing (true of generated
   * VDIs: _emit clamps, generate.py:58-62). Then, for rays whose chord runs
   * forward in depth, the Alg. 2 search result does not depend on its seed,
   * and the kernel may search a list first and evaluate the ESS test only to
   * confirm a hit (a miss composites nothing either way): same image, same
   * lists_visited / segs_intersected, fewer ESS tests. lists_searched is then
   * not counted (per-pixel array and stat_sums[2] are left unchanged) unless
   * counters_exact is 1. 0: the reference's order (ESS, then search). */
  int32_t lists_sorted;
  int32_t counters_exact;
  /* optional (may be NULL): storage row of every list row of the VDI
   * (vdi_h entries), overriding the vdi_band_* map -- the gathered VDI of
   * contiguous bands of unequal height (VdiGenArgs.row_count). */
  const int32_t* vdi_row_map;
  /* optional (may be NULL): vdi_list_ranges() of the VDI, two floats per
   * storage list: (min front, max back), (+inf, -inf) for an empty list and
   * (-inf, +inf) for a list holding a NaN depth. Used with lists_sorted on
   * forward chords when counters_exact is 0: a list whose range the chord
   * piece [d_entry, d_exit] misses (d_exit < min front or d_entry > max back)
   * has no supersegment with back >= d_entry and front <= d_exit, so the
   * search would miss; it is skipped without reading the list. Same image
   * and counters. */
  const float* list_range;
  /* optional (may be NULL): two zeroed u32 owned by the caller. Then the
   * render runs one resident grid whose warps take 8x4 pixel tiles from
   * tile_counter[0] in image order; the last warp resets both words to 0, so
   * the pair can be reused by the next launch on the same stream (not by a
   * concurrent one). NULL: one tile per warp. Same image and counters. */
  unsigned int* tile_counter;
} VdiRenderArgs;

/* Ground-truth direct volume rendering (dvr.py:21-89): the generation ray,
 * clip and sampler, composited front to back with early termination.
 * Outputs are indexed by local row (band map). */
typedef struct VdiDvrArgs {
  const void* volume;           /* as VdiGenArgs.volume (VDI_VOXEL_CELLS allowed) */
  const float* lut;             /* (lut_n, 4) f32 */
  const void* brick_max;        /* vdi_volume_brick_max() of the volume, or NULL */
  double* image;                /* OUT (local_h, width, 4) f64 premultiplied, 16 B aligned */
  int32_t* samples;             /* OUT executed samples per pixel, may be NULL */
  unsigned long long* stat_sums;/* OUT [1] += executed samples, may be NULL */
  void* workspace;              /* >= VDI_DVR_WORKSPACE_BYTES device bytes, any content */
  double pv[16];
  double inv_pv[16];
  double eye[3];
  double aabb[6];
  double bg[4];                 /* straight RGBA background */
  double step, lref;            /* render_dvr step / ref_step (resolved) */
  double early_term;            /* early_term_alpha */
  double ess_max;               /* as VdiGenArgs.ess_max */
  int32_t voxel_type;
  int32_t nx, ny, nz;
  int32_t lut_n;
  int32_t width, height;
  int32_t band_rows, band_stride, band_offset;
  int32_t brick_log2;
} VdiDvrArgs;

#define VDI_DVR_WORKSPACE_BYTES 256

/* Preview rendering with dynamic subsampling (preview.py:49-205) at the
 * low-res viewport out_w x out_h; upsample with vdi_bilinear_upsample. */
typedef struct VdiPreviewArgs {
  const float* segs;            /* list-SoA */
  const int32_t* counts;
  const uint32_t* grid;         /* (gz, gy, gx) */
  double* image;                /* OUT (out_h, out_w, 4) f64 premultiplied, 16 B aligned */
  unsigned long long* cell_samples; /* OUT (gz, gy, gx) planned samples, zeroed by the
                                   launch; may be NULL */
  unsigned long long* stat_sums;/* OUT [1] += total samples, may be NULL */
  void* workspace;              /* >= VDI_PREVIEW_WORKSPACE_BYTES device bytes */
  double gen_pv[16];
  double gen_inv_pv[16];
  double new_inv_pv[16];        /* low-res camera */
  double eye[3];
  double aabb[6];               /* Vdi.volume_aabb */
  double bg[4];
  double near, far, proj_a, proj_b;  /* grid near/far, generation depth constants */
  double d_r, early_term;
  int32_t vdi_w, vdi_h, n_sg;
  int32_t gx, gy, gz;
  int32_t out_w, out_h;
  int32_t vdi_band_rows, vdi_band_world, vdi_rows_per_rank;  /* as VdiRenderArgs */
} VdiPreviewArgs;

#define VDI_PREVIEW_WORKSPACE_BYTES 256

/* VDI1 serialisation (vdi.py:136-159): header | counts u16 | valid
 * supersegments f32 AoS in list order | grid u32, little endian. */
#define VDI_VDI1_HEADER_BYTES 160
typedef struct VdiEncodeArgs {
  const float* segs;            /* list-SoA */
  const int32_t* counts;
  const uint32_t* grid;         /* (gz, gy, gx) */
  uint8_t* out;                 /* OUT >= vdi_vdi1_max_bytes() device bytes */
  unsigned long long* out_len;  /* OUT (device) bytes written, may be NULL */
  void* workspace;              /* >= vdi_encode_workspace_bytes() */
  size_t workspace_bytes;
  uint8_t header[VDI_VDI1_HEADER_BYTES]; /* vdi.py:146-149: magic .. grid dims */
  int32_t width, height, n_sg;
  int32_t gx, gy, gz;
  int32_t vdi_band_rows, vdi_band_world, vdi_rows_per_rank;  /* as VdiRenderArgs */
} VdiEncodeArgs;

/* On-device validate_vdi (vdi.py:116-134). result[0] = min over failing
 * lists of (row-major list index << 3 | code), code 1 front >= back, 2
 * overlapping, 3 depth outside [-1, 1], 4 not premultiplied (the first
 * failing check of that list, in the reference's order), or ~0 if none;
 * result[1] = lists whose count is outside [0, n_sg]. */
typedef struct VdiValidateArgs {
  const float* segs;
  const int32_t* counts;
  unsigned long long* result;   /* OUT (device) [2] */
  int32_t width, height, n_sg;
  int32_t vdi_band_rows, vdi_band_world, vdi_rows_per_rank;
} VdiValidateArgs;

const char* vdi_last_error(void);
int vdi_abi_version(void);

/* Recommended / minimum workspace bytes for `args` on the current device. */
size_t vdi_gen_workspace_bytes(const VdiGenArgs* args);
size_t vdi_gen_workspace_min_bytes(const VdiGenArgs* args);
int vdi_gen_launch(const VdiGenArgs* args, vdi_stream_t stream);
int vdi_grid_launch(const VdiGridArgs* args, vdi_stream_t stream);
int vdi_render_launch(const VdiRenderArgs* args, vdi_stream_t stream);

/* Occupancy of 8x8-list tiles of a (band-sharded) VDI: bit t of the bitmap
 * (tiles row-major, ceil(vdi_w/8) per row) is set iff a list of tile t has
 * count > 0. Reads args->counts, vdi_w, vdi_h and the vdi_band_* fields;
 * writes vdi_list_tiles_words(vdi_w, vdi_h) words to tiles. An accelerator
 * for vdi_render_launch (VdiRenderArgs.list_tiles), SURVEY 8(f) rank 4. */
size_t vdi_list_tiles_words(int32_t vdi_w, int32_t vdi_h);
int vdi_list_tiles(const VdiRenderArgs* args, uint32_t* tiles, vdi_stream_t stream);
/* Per-column slab occupancy of an AccelGrid (gz, gy, gx) u32, gz <= 64:
 * out[cgy * gx + cgx] bit cz = grid[cz][cgy][cgx] > 0 (gx * gy words). An
 * accelerator for vdi_render_launch (VdiRenderArgs.grid_zmask). */
int vdi_grid_zmask(const uint32_t* grid, int32_t gx, int32_t gy, int32_t gz, uint64_t* out,
                   vdi_stream_t stream);
/* Depth range of every list of a list-SoA VDI (n_lists storage lists):
 * out[2 l] = min front, out[2 l + 1] = max back over its counts[l] entries;
 * (+inf, -inf) when empty, (-inf, +inf) when a depth is NaN. An accelerator
 * for vdi_render_launch (VdiRenderArgs.list_range). */
int vdi_list_ranges(const float* segs, const int32_t* counts, int64_t n_lists, int32_t n_sg,
                    float* out, vdi_stream_t stream);
int vdi_dvr_launch(const VdiDvrArgs* args, vdi_stream_t stream);
int vdi_preview_launch(const VdiPreviewArgs* args, vdi_stream_t stream);
/* (h, w, channels) f64 -> (out_h, out_w, channels), preview.py:208-223
 * (the caller handles the identity case, where R returns its input). */
int vdi_bilinear_upsample(const double* src, int32_t w, int32_t h, double* dst,
                          int32_t out_w, int32_t out_h, int32_t channels,
                          vdi_stream_t stream);

size_t vdi_vdi1_max_bytes(int32_t width, int32_t height, int32_t n_sg, int32_t gx, int32_t gy,
                          int32_t gz);
size_t vdi_encode_workspace_bytes(int32_t width, int32_t height);
int vdi_encode_vdi1(const VdiEncodeArgs* args, vdi_stream_t stream);

/* The lists of a VDI1 stream (counts u16 at byte 160, then the valid
 * supersegments) -> counts i32 (rows, width) + list-SoA segs with zeroed
 * tails (decode_vdi's arrays, vdi.py:162-210, on the device). workspace:
 * vdi_encode_workspace_bytes(width, rows). Used by the multi-GPU exchange,
 * which all-gathers packed VDI1 shards instead of the padded list-SoA. */
int vdi_decode_vdi1_lists(const uint8_t* src, int32_t width, int32_t rows, int32_t n_sg,
                          int32_t* counts, float* segs, void* workspace, size_t workspace_bytes,
                          vdi_stream_t stream);

/* LZ4 block compression of src[0, n) with n = min(*n_dev, n_max) when n_dev
 * is not NULL (a device length, e.g. VdiEncodeArgs.out_len), else n = n_max. dst holds
 * vdi_lz4_max_bytes(n_max); *out_len (device) receives the block length. */
size_t vdi_lz4_max_bytes(size_t n);
size_t vdi_lz4_workspace_bytes(size_t n_max);
int vdi_lz4_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev,
                     uint8_t* dst, unsigned long long* out_len, void* workspace,
                     size_t workspace_bytes, vdi_stream_t stream);
/* The same contract, but the block is the reference's own: one serial greedy
 * parse with lz4.py's 64 Ki-entry table, byte-identical to lz4.compress(src)
 * (lz4.py:51-114). Slower than vdi_lz4_compress (one warp parses). */
size_t vdi_lz4_exact_workspace_bytes(size_t n_max);
int vdi_lz4_compress_exact(const uint8_t* src, size_t n_max, const unsigned long long* n_dev,
                           uint8_t* dst, unsigned long long* out_len, void* workspace,
                           size_t workspace_bytes, vdi_stream_t stream);

int vdi_validate(const VdiValidateArgs* args, vdi_stream_t stream);

/* Single-ray generation for n arbitrary rays (rays: (n, 6) f64 origin xyz,
 * direction xyz), with the volume / LUT / camera / params of `args` (its
 * width, height, band map, workspace and brick fields are ignored; outputs
 * are indexed by ray): mode 0 = the full gamma bisection (find_gamma,
 * generate.py:390-407: counts, segs, gammas, passes, samples); mode 1 / 2 =
 * one counting / capped pass at gammas_in[i] (generate_list,
 * generate.py:371-387: counts[i] = n, n_sg + 1 when exceeded). */
#define VDI_RAYS_BISECT 0
#define VDI_RAYS_COUNT 1
#define VDI_RAYS_CAPPED 2
int vdi_gen_rays(const VdiGenArgs* args, const double* rays, const double* gammas_in,
                 int64_t n_rays, int32_t mode, vdi_stream_t stream);

/* composite_lists (raycast.py:494-518) of a (h, w) list-SoA VDI into an
 * (h, w, 4) f64 image; bg: HOST straight RGBA. */
int vdi_composite_lists(const float* segs, const int32_t* counts, int32_t w, int32_t h,
                        int32_t n_sg, double early_term, const double* bg_host, double* image,
                        vdi_stream_t stream);

/* _dda_cells (raycast.py:159-222) for n chords (6 f64: a0 xyz, a1 xyz):
 * cells (n, cap, 2) i32, zs (n, cap, 4) f64 (z_entry, z_exit, s_entry,
 * s_exit), counts (n,) i32; cap >= w + h + 4 holds every visit. */
int vdi_dda_cells(const double* chords, int64_t n, int32_t w, int32_t h, int32_t cap,
                  int32_t* cells, double* zs, int32_t* counts, vdi_stream_t stream);

/* project_ray_to_ndc (raycast.py:237-255) for n world rays (6 f64): out (n, 6)
 * NDC chord (a0, a1), hit (n,) 0/1; gen_pv, aabb: HOST f64[16], f64[6]. */
int vdi_project_rays(const double* rays, int64_t n, const double* gen_pv_host,
                     const double* aabb_host, double* out, int32_t* hit, vdi_stream_t stream);

/* Alg. 2 search over a batch of independent queries (raycast.py:79-156).
 * fronts/backs: (n_queries, n_max) f32, counts: (n_queries,), d_entry /
 * d_exit: f64, seeds: p. out_index = -1 for a miss. */
int vdi_find_first_batch(const float* fronts, const float* backs,
                         const int32_t* counts, int32_t n_max,
                         const double* d_entry, const double* d_exit,
                         const int32_t* seeds, int32_t* out_index,
                         int32_t* out_seed, int64_t n_queries,
                         vdi_stream_t stream);

/* Per-brick maximum of the raw voxels (edge 2^brick_log2, +1 trilinear halo):
 * out is (ceil(nz/B), ceil(ny/B), ceil(nx/B)) of the volume's voxel type.
 * Used for exact empty-space skipping in vdi_gen_launch. */
int vdi_volume_brick_max(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny,
                         int32_t nz, int32_t brick_log2, void* out, vdi_stream_t stream);

/* Corner records for generation: cell (x, y, z) of the (nz, ny, nx) grid
 * becomes the 8 voxels of its trilinear cube, [v(x,y,z), v(x+1,y,z),
 * v(x,y+1,z), v(x+1,y+1,z), v(x,y,z+1), v(x+1,y,z+1), v(x,y+1,z+1),
 * v(x+1,y+1,z+1)] (indices clamped to the grid), stored contiguously: one
 * aligned 8 x sizeof(voxel) load per sample instead of 8 gathers. The same
 * voxel values, so generation results are unchanged. `out` must hold
 * vdi_volume_cells_bytes() bytes, 32-byte aligned. Replaces nothing in the
 * reference: it is this library's HBM layout of Volume.normalized
 * (volume.py:48-50, read by _trilinear, volume.py:180-205). */
size_t vdi_volume_cells_bytes(int32_t voxel_type, int32_t nx, int32_t ny, int32_t nz);
int vdi_volume_cells(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny, int32_t nz,
                     void* out, vdi_stream_t stream);
/* The same, skipping the cells of bricks whose vdi_volume_brick_max()
 * value normalises to <= ess_max: the samplers' empty-space test skips those
 * samples before any corner-record load, so their records are never read
 * (and are left with any content). */
int vdi_volume_cells_masked(const void* volume, int32_t voxel_type, int32_t nx, int32_t ny,
                            int32_t nz, const void* brick_max, int32_t brick_log2, double ess_max,
                            void* out, vdi_stream_t stream);

/* Synthetic input for config C5 (not a reference function): a
 * Richtmyer-Meshkov-shaped u8 volume (nz, ny, nx) written on the device.
 * modes: 12 x (kx, ky, amplitude, phase) of the interface; band: half-width
 * of the mixing band in unit coordinates. box_host (or NULL = everything):
 * [ox, oy, oz, sx, sy, sz], write only that box, stored (sz, sy, sx). */
int vdi_synth_rm_u8(uint8_t* out, int32_t nx, int32_t ny, int32_t nz, const int32_t* box_host,
                    const float* modes_host, float band, uint32_t seed, vdi_stream_t stream);

/* Device self-check of the exact arithmetic shortcuts the kernels use, on n
 * random inputs: bad[0..3] (device, 4 x u64) receive the mismatch counts of
 * Markstein division, __drcp_rn reciprocals, the sqrt-free split threshold
 * and the shared-reciprocal world/NDC transform (all must be 0). */
int vdi_selftest_arith(int64_t n, uint64_t seed, unsigned long long* bad, vdi_stream_t stream);

/* Layout conversion for n_lists lists of n_sg supersegments. */
int vdi_segs_to_aos(const float* soa, float* aos, int64_t n_lists,
                    int32_t n_sg, vdi_stream_t stream);
int vdi_segs_from_aos(const float* aos, float* soa, int64_t n_lists,
                      int32_t n_sg, vdi_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VDI_B200_H */
