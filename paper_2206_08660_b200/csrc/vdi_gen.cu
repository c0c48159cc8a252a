// vdi_gen.cu -- VDI generation on sm_100a.
//
// Semantics: the reference's _generate_kernel (generate.py:276-319), which runs
// per ray the gamma bisection _find_gamma_list (219-273) over front-to-back
// passes _gen_list_pass (89-216) with _emit (53-86), trilinear sampling
// (volume.py:180-205) and LUT classification (volume.py:164-177). Arithmetic is
// f64 in the reference's order (no FMA: built with -fmad=false), f32 rounding
// at the LUT output and at the segment store, exactly as numba does.
//
// B200 structure. Every bisection pass walks the same samples with a new
// gamma, so the work splits into (a) sampling the volume once per sample and
// (b) replaying the per-sample segment logic per pass. Mixing both in one warp
// serialises them (profiles/r01_gen_v1_fused_cache.md: 16.7 of 32 lanes
// active), so generation runs in mode-coherent phases:
//
//   sample phase   one lane per ray (8x4 pixel tiles, lanes refill from a
//                  warp-uniform ray pool): sample + classify every step and run
//                  pass 1 (gamma_init) on the fly. Most rays finish here
//                  (pass 1 not exceeding n_sg ends the bisection). A ray whose
//                  pass 1 overflows gets an exact-size slot from a bump
//                  allocator and re-walks its samples in fill mode, storing
//                  the classified f32 RGBA (16 B) per sample; transparent runs
//                  are stored run-length coded. It is then queued.
//   bisect phase   replay-only lanes pull queued rays and run passes 2.. of the
//                  bisection on the stored samples: 16 B per sample and ~35 f64
//                  ops instead of 8 voxel gathers and ~120 f64 ops; transparent
//                  runs cost O(1).
//
// The cache capacity is whatever workspace the caller provides; rays that do
// not fit are deferred to the next round (up to kRounds), and anything left
// after that runs in the fused fallback kernel (sampling and replay in one
// lane, per-lane cache slot) -- same results, just slower.
//
// Replay is bit-identical by construction: the same f32 values enter the same
// f64 expressions. Exact shortcuts (same bits, fewer instructions):
//   * dist >= gamma  <=>  d2 >= thr(gamma), thr the smallest double whose
//     correctly rounded sqrt is >= gamma (sqrt_rn is monotone); per pass;
//   * 1.0 / nsamp comes from a table of host-identical IEEE quotients;
//   * x / extent is x * (1 / extent) when the extent is a power of two.
// Segments are written straight into the output list during every pass; the
// only result that is not the last pass's output (the epsilon exit returning
// the cached high-gamma segments after a later low-gamma pass) replays the
// high pass, which is deterministic.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "vdi_common.cuh"
#include "vdi_internal.h"
#include "vdi_sample.cuh"

namespace vdi {

constexpr int kGenThreads = 128;
#ifndef VDI_SAMPLE_MINB
#define VDI_SAMPLE_MINB 5  // 96 registers: 5 blocks/SM (measured: 9.59 -> 9.14 ms at C3)
#endif
#ifndef VDI_FILL_MINB
#define VDI_FILL_MINB 0  // no minimum (64 registers): 10 blocks/SM gave C3 -0.2 ms but C4 / C5 +4 ms
#endif
#if VDI_FILL_MINB > 0
#define VDI_FILL_BOUNDS __launch_bounds__(kGenThreads, VDI_FILL_MINB)
#else
#define VDI_FILL_BOUNDS __launch_bounds__(kGenThreads)
#endif
#ifndef VDI_BISECT_PF
#define VDI_BISECT_PF 1     // cache-row prefetch of the replays: 1 L1, 2 L2, 3 L1 + bulk L2
#endif
#ifndef VDI_BISECT_MODE
// cache stream: 2 A/B register slots + L1 prefetch, 3 cp.async ring in shared
// memory (measured C3 / C4 gen: 26.8 / 68.2 ms -> 23.1 / 61.6 ms with a ring
// of 4 at 4 blocks/SM; ring 8: 23.2 / 61.9)
#define VDI_BISECT_MODE 3
#endif
#ifndef VDI_BISECT_RING
#define VDI_BISECT_RING 4   // kMode 3: ring entries per lane (power of two)
#endif
#ifndef VDI_BISECT_AHEAD
#define VDI_BISECT_AHEAD 16  // entries ahead of the L1 prefetch
#endif
#ifndef VDI_EMIT_PF
#define VDI_EMIT_PF 1
#endif
#ifndef VDI_EMIT_MINB
#define VDI_EMIT_MINB 5  // 96 registers (A/B stream: 6 blocks best, 6.16 -> 5.64 ms; ring: 5)
#endif
constexpr int kRounds = 3;
constexpr long long kWideRays = 700000;  // launches below this many rays use the wide hand-off

enum PassMode : int { kCount = 0, kCapped = 1, kRedo = 2 };

// A ray whose pass 1 overflowed, handed from the sample phase to the bisect
// phase, and from there (with the deciding gamma) to the emit phase.
struct RayRec {
  double d[3];
  double t0, t1;
  double g_final;   // gamma of the pass whose segments are the result
  long long slot;   // first float4 of its cache run
  int list;         // local list index (row * width + col)
  int nsteps;       // samples stored
  int samples;      // samples executed so far (R semantics)
  int passes;       // passes so far (R semantics)
  int mode_final;   // kCount (window hit / cached high) or kCapped
  int first_vis;    // the first non-transparent sample (pass 1 of the sample phase)
  // bisection state handed from a narrow replay lane to the wide phase
  double low, high;
  int last_n, high_n;
};

// Where a queued ray's cache run is allocated: 0 = bump-allocated in the
// sample phase when the ray overflows (overflow order), 1 = after the queue
// compaction, by a prefix sum of row lengths in image order (rays past the
// capacity are then a suffix of the queue, deferred to the next round).
#ifndef VDI_ALLOC_IMAGE
#define VDI_ALLOC_IMAGE 1
#endif
// The order the bisect / emit phases take the queue in: 0 = overflow order
// (torder), 1 = image order (qidx). The two must agree: replay lanes run side
// by side on neighbouring queue entries, and their cache rows have to be
// neighbours in memory too. Measured C3 / C4 generation (ms): overflow /
// overflow 30.6 / 78.6, image / overflow 35.0 / 87.3, overflow / image 35.0 /
// 86.4, image / image 30.5 / 77.0 (a longest-row-first order: 40.0 / 88.4).
#ifndef VDI_REPLAY_ORDER
#define VDI_REPLAY_ORDER 1
#endif

// Cache entry of a non-transparent sample: the classified f32 RGBA, with the
// sign bit of r (r >= 0 always) set when the step's opacity exponent
// (tb - ta) / lref is not exactly 1, i.e. when the replay needs pow().
__device__ __forceinline__ bool entry_needs_pow(float4 e) { return signbit(e.x); }

// Per-round queues/counters (all zeroed at launch).
struct RoundCtl {
  unsigned long long fetch;     // sample-phase ray pool
  unsigned long long bump;      // cache allocator (float4 units)
  unsigned long long nrec;      // rays queued for the bisect phase
  unsigned long long rfetch;    // bisect-phase pool
  unsigned long long ndefer;    // rays deferred to the next round
  unsigned long long efetch;    // emit-phase pool
  unsigned long long ffetch;    // fill-phase pool (one ray per warp)
  unsigned long long nwide;     // rays handed to the wide bisect phase
  unsigned long long wfetch;    // wide-phase pool (one ray per warp)
  unsigned long long ntorder;   // rays appended in overflow order
  // VDI_BISECT_STATS builds only: narrow-replay steps on visible entries, on
  // transparent runs, the entries the runs covered, replays started
  unsigned long long st_vis, st_run, st_run_entries, st_replays;
  // VDI_FILL_STATS builds only: fill chunks, chunks whose valid samples all
  // lie in empty bricks, chunks whose valid samples are all transparent
  unsigned long long st_chunks, st_chunks_empty, st_chunks_transp;
  // bisection decisions seen so far in this round, per level: [0] up, [1] down
  // (the bisect replays' learned speculation direction)
  unsigned dir[2][32];
};

struct GenConst {
  VdiGenArgs a;
  double inv_ext[3];  // RN(1/extent): exact scale (power of two) or Markstein reciprocal
  int ext_pow2[3];
  double inv_lref;
  int lref_pow2;
  int tiles_x;
  int local_h;
  long long n_slots;  // tiles * 32
  const double* inv_tab;  // inv_tab[n] == 1.0 / n, bit-exact (host IEEE division)
  int inv_n;
  int inv_smem;       // leading inv_tab entries the bisect phase stages in shared memory
  int max_steps;
  float4* cache;
  unsigned long long cache_cap;  // float4 entries
  RayRec* recs;
  int* defer_in;   // ray source of rounds >= 1 (local list indices)
  int* defer_out;
  RoundCtl* ctl;   // this round
  RoundCtl* prev;  // previous round (its ndefer sizes defer_in)
  int round;
  int ess;         // empty-space skipping enabled
  int ess_u8;      // u8 volumes: ess_max as a byte threshold (brick_empty)
  int bnx, bny;    // brick grid x / y extent (of the resident box in kVoxelSub variants)
  // resident box (kVoxelSub variants): row strides, index rebases, origin, extent
  long long sub_sx, sub_sy, sub_voff, sub_boff;
  int sub_ox, sub_oy, sub_oz, sub_nx, sub_ny, sub_nz;
  unsigned* sub_oob;
  int* wide;         // rays handed to the wide bisect phase (record indices)
  // the round's queue: recs is indexed by local list; qbits marks the queued
  // lists and qidx (built from it) lists them in image order
  unsigned* qbits;
  int* qidx;
  unsigned* hitbits;  // round 0: bit s = tile slot s hits the volume (VDI_SETUP_PASS)
  int* torder;       // the same rays in the order they overflowed (bisect / emit)
  unsigned long long* qsum;  // per compaction block
  int wide_after;    // replays a narrow lane runs on one ray before handing it off
  int wide_tail;     // also hand off every ray once the narrow queue is drained
  int n_qblocks;     // queue compaction blocks (qsum holds 2 x (n_qblocks + 1))
  int chain_levels;  // bisect replays starting below this level use the down-chain shape
  int learn;         // learned chain directions at the later levels 
};

struct RayState {
  // ray geometry
  double o[3], d[3], t0, t1;
  int nsteps, k;
  float* seg;  // this list's list-SoA block
  int list;
  // current pass (generate.py:97-106)
  double gamma, thr, fr_t, bk_t, mr, mg, mb, acc_r, acc_g, acc_b, acc_a, last_fr_t;
  float prev_back;
  int count, nsamp, active, mode;
  // bisection (generate.py:230-236)
  double low, high, bis_gamma;
  int first, last_n, high_n, passes, buf_is_high, samples;
  int first_vis;  // sample phase: the first non-transparent sample of pass 1 (-1: none yet)
};

// Smallest double s >= 0 with sqrt_rn(s) >= g, so that sqrt_rn(d2) >= g <=>
// d2 >= s for every d2 >= 0 (sqrt_rn is monotone non-decreasing).
__device__ double split_threshold(double g) {
  if (!(g > 0.0)) return -INFINITY;
  double s = g * g;
  while (sqrt(s) < g) s = nextafter(s, INFINITY);
  while (true) {
    const double p = nextafter(s, 0.0);
    if (sqrt(p) >= g) s = p;
    else break;
  }
  return s;
}

// Sample position -> classified RGBA (generate.py:118-134 + volume.py).
template <int VT>
__device__ __forceinline__ float4 sample_at(const GenConst& c, const double4* lut,
                                            const double* tab, const RayState& s, double ta,
                                            double tb, bool* ess_hit = nullptr) {
  const double tm = 0.5 * (ta + tb);
  double q[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double num = s.o[a] + tm * s.d[a] - c.a.aabb[a];
    double v = c.ext_pow2[a] ? num * c.inv_ext[a]
                             : div_by(num, c.a.aabb[3 + a] - c.a.aabb[a], c.inv_ext[a]);
    if (v < 0.0) v = 0.0;
    else if (v > 1.0) v = 1.0;
    q[a] = v;
  }
  const double v = trilinear<VT>(c, tab, q[0], q[1], q[2]);
  if (ess_hit) *ess_hit = v == -1.0;  // the empty-brick sentinel (or a genuine -1 sample)
  return classify(lut, c.a.lut_n, v);
}

// generate.py:53-86 _emit into the list-SoA slot `count`.
__device__ __forceinline__ void emit(const GenConst& c, RayState& s) {
  const double* pv = c.a.pv;
  const double zf = xform_z(pv, s.o[0] + s.fr_t * s.d[0], s.o[1] + s.fr_t * s.d[1],
                            s.o[2] + s.fr_t * s.d[2]);
  const double zb = xform_z(pv, s.o[0] + s.bk_t * s.d[0], s.o[1] + s.bk_t * s.d[1],
                            s.o[2] + s.bk_t * s.d[2]);
  float f = (float)zf, b = (float)zb;
  if (f < -1.0f) f = -1.0f;
  if (s.count > 0 && f < s.prev_back) f = s.prev_back;
  if (b > 1.0f) b = 1.0f;
  if (b <= f) b = nextafterf(f, 2.0f);
  const float a32 = (float)s.acc_a;
  float r32 = (float)s.acc_r, g32 = (float)s.acc_g, b32 = (float)s.acc_b;
  if (r32 > a32) r32 = a32;
  if (g32 > a32) g32 = a32;
  if (b32 > a32) b32 = a32;
  const int n_sg = c.a.n_sg;
  s.seg[front_off(n_sg) + s.count] = f;
  s.seg[back_off(n_sg) + s.count] = b;
  reinterpret_cast<float4*>(s.seg)[s.count] = make_float4(r32, g32, b32, a32);
  s.prev_back = b;
  s.last_fr_t = s.fr_t;
  s.count += 1;
}

__device__ __forceinline__ void start_pass(RayState& s, double g, int mode) {
  s.gamma = g;
  s.thr = split_threshold(g);
  s.mode = mode;
  s.k = 0;
  s.count = 0;
  s.active = 0;
  s.nsamp = 0;
  s.fr_t = s.bk_t = 0.0;
  s.mr = s.mg = s.mb = 0.0;
  s.acc_r = s.acc_g = s.acc_b = s.acc_a = 0.0;
}

// One sample of _gen_list_pass after classification (generate.py:135-212).
// `run` >= 1 transparent samples are consumed at once (they only close the
// open segment). Returns -1 to continue, else the pass result (0 = reached
// the end: close with close_pass; n_sg + 1 = aborted counting pass);
// advances s.k.
__device__ __forceinline__ int segment_step(const GenConst& c, RayState& s, float4 rgba,
                                            double ta, double tb, int run) {
  const int n_sg = c.a.n_sg;
  if (s.mode != kRedo) s.samples += run;
  if (rgba.w <= 0.0f) {
    // fully transparent: closes the open supersegment (generate.py:135-142)
    if (s.active) {
      emit(c, s);
      s.active = 0;
    }
    s.k += run;
    return s.k >= s.nsteps ? 0 : -1;
  }
  const double a = (double)rgba.w;
  const double dt = tb - ta;
  const double e = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
  const double om = 1.0 - a;
  const double a_adj = 1.0 - (e == 1.0 ? om : pow(om, e));
  const double sr = (double)rgba.x * a_adj;
  const double sg = (double)rgba.y * a_adj;
  const double sb = (double)rgba.z * a_adj;
  bool merge = false, fresh = false;
  if (!s.active) {
    if (s.count >= n_sg) {
      if (s.mode != kCapped) return n_sg + 1;
      // reopen the last supersegment (generate.py:151-165)
      s.count -= 1;
      s.fr_t = s.last_fr_t;
      const float4 l = reinterpret_cast<const float4*>(s.seg)[s.count];
      s.acc_r = l.x;
      s.acc_g = l.y;
      s.acc_b = l.z;
      s.acc_a = l.w;
      s.prev_back = s.count > 0 ? s.seg[back_off(n_sg) + s.count - 1] : 0.0f;
      s.acc_r += (1.0 - s.acc_a) * sr;
      s.acc_g += (1.0 - s.acc_a) * sg;
      s.acc_b += (1.0 - s.acc_a) * sb;
      s.acc_a += (1.0 - s.acc_a) * a_adj;
      s.bk_t = tb;
      s.mr = sr;
      s.mg = sg;
      s.mb = sb;
      s.nsamp = 1;
      s.active = 1;
    } else {
      s.active = 1;
      fresh = true;
    }
  } else {
    const double dr = s.mr - sr, dg = s.mg - sg, db = s.mb - sb;
    if (dr * dr + dg * dg + db * db >= s.thr) {  // == sqrt(...) >= gamma
      if (s.count + 1 >= n_sg) {
        if (s.mode != kCapped) return n_sg + 1;
        merge = true;
      } else {
        emit(c, s);
        fresh = true;
      }
    } else {
      merge = true;
    }
  }
  if (fresh) {
    s.fr_t = ta;
    s.bk_t = tb;
    s.mr = sr;
    s.mg = sg;
    s.mb = sb;
    s.nsamp = 1;
    s.acc_r = sr;
    s.acc_g = sg;
    s.acc_b = sb;
    s.acc_a = a_adj;
  } else if (merge) {
    s.acc_r += (1.0 - s.acc_a) * sr;
    s.acc_g += (1.0 - s.acc_a) * sg;
    s.acc_b += (1.0 - s.acc_a) * sb;
    s.acc_a += (1.0 - s.acc_a) * a_adj;
    s.bk_t = tb;
    s.nsamp += 1;
    const double inv = s.nsamp < c.inv_n ? __ldg(c.inv_tab + s.nsamp) : 1.0 / (double)s.nsamp;
    s.mr += (sr - s.mr) * inv;
    s.mg += (sg - s.mg) * inv;
    s.mb += (sb - s.mb) * inv;
  }
  s.k += 1;
  return s.k >= s.nsteps ? 0 : -1;
}

// Natural end (or the tb <= ta break, generate.py:113-117, 213-216).
__device__ __forceinline__ int close_pass(const GenConst& c, RayState& s) {
  if (s.active) emit(c, s);
  return s.count;
}

// Zero-fill the unused tail and publish the per-ray outputs
// (generate.py:314-319).
__device__ void finish_ray(const GenConst& c, RayState& s, double g, int n) {
  const int n_sg = c.a.n_sg;
  for (int i = n; i < n_sg; ++i) {
    s.seg[front_off(n_sg) + i] = 0.0f;
    s.seg[back_off(n_sg) + i] = 0.0f;
    reinterpret_cast<float4*>(s.seg)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  c.a.counts[s.list] = n;
  if (c.a.gammas) c.a.gammas[s.list] = g;
  if (c.a.passes) c.a.passes[s.list] = s.passes;
  if (c.a.samples) c.a.samples[s.list] = s.samples;
}

// Top of the bisection loop (generate.py:237-257): either start the next
// measurement pass or leave through the epsilon test. Returns false when the
// ray is finished.
__device__ bool bisect_next(const GenConst& c, RayState& s) {
  if (fabs(s.high - s.low) < c.a.eps) {
    double g;
    if (s.last_n == 0) {
      g = s.low;
    } else {
      g = s.high;
      if (s.high_n >= 0) {
        if (s.buf_is_high) {
          finish_ray(c, s, g, s.high_n);
          return false;
        }
        start_pass(s, g, kRedo);  // regenerate the cached high segments
        return true;
      }
    }
    start_pass(s, g, kCapped);
    return true;
  }
  start_pass(s, s.bis_gamma, kCount);
  return true;
}

// End of a pass with result n (generate.py:248-273). Returns false when the
// ray is finished.
__device__ bool pass_done(const GenConst& c, RayState& s, int n) {
  if (s.mode == kRedo) {
    finish_ray(c, s, s.high, s.high_n);
    return false;
  }
  s.passes += 1;
  if (s.mode == kCapped) {
    finish_ray(c, s, s.gamma, n);
    return false;
  }
  const int n_sg = c.a.n_sg;
  s.last_n = n;
  if (s.first) {
    s.first = 0;
    if (n < n_sg) {
      finish_ray(c, s, s.bis_gamma, n);
      return false;
    }
  }
  if (n > n_sg) {
    s.low = s.bis_gamma;
    s.buf_is_high = 0;
  } else if (n < n_sg - c.a.delta) {
    s.high = s.bis_gamma;
    s.high_n = n;
    s.buf_is_high = 1;
  } else {
    finish_ray(c, s, s.bis_gamma, n);
    return false;
  }
  s.bis_gamma = 0.5 * (s.low + s.high);
  return bisect_next(c, s);
}

__device__ __forceinline__ void init_bisection(const GenConst& c, RayState& s) {
  s.low = 0.0;
  s.high = kSqrt3;
  s.bis_gamma = c.a.gamma_init;
  s.first = 1;
  s.last_n = 1;
  s.high_n = -1;
  s.passes = 0;
  s.buf_is_high = 0;
  s.samples = 0;
}

// Ray setup (generate.py:282-309) for local list `list`. Returns false on a
// miss (the list is then published empty, unless kPublishMiss is false).
template <bool kPublishMiss = true>
__device__ bool setup_ray(const GenConst& c, RayState& s, int list) {
  const int lx = list % c.a.width, ly = list / c.a.width;
  const int gy = image_row(ly, c.a.band_rows, c.a.band_stride, c.a.band_offset, c.a.row_base,
                           c.a.row_count);
  s.list = list;
  s.seg = c.a.segs + (long long)list * list_stride(c.a.n_sg);
  pixel_ray(c.a.inv_pv, c.a.eye, lx, gy, c.a.width, c.a.height, s.d);
  s.o[0] = c.a.eye[0];
  s.o[1] = c.a.eye[1];
  s.o[2] = c.a.eye[2];
  double ta, tb, fa, fb;
  bool hit = clip_aabb(s.o, s.d, c.a.aabb, ta, tb) && clip_frustum(c.a.pv, s.o, s.d, fa, fb);
  double t0 = 0.0, t1 = 0.0;
  if (hit) {
    t0 = dmax(dmax(ta, fa), 0.0);
    t1 = dmin(tb, fb);
    hit = t1 > t0;
  }
  init_bisection(c, s);
  if (!hit) {
    if (kPublishMiss) finish_ray(c, s, 0.0, 0);
    return false;
  }
  s.t0 = t0;
  s.t1 = t1;
  s.nsteps = (int)ceil((t1 - t0) / c.a.step);
  start_pass(s, s.bis_gamma, kCount);
  s.first_vis = -1;
  return true;
}

// Warp-uniform pool of work indices: one atomicAdd per 32 items. Lanes in
// `need` receive consecutive indices. Must be called warp-converged.
struct WarpPool {
  long long base = 0;
  int used = 32;
  __device__ __forceinline__ long long take(unsigned need, int lane,
                                            unsigned long long* counter) {
    const int n = __popc(need);
    const int rank = __popc(need & ((1u << lane) - 1u));
    const int avail = 32 - used;
    long long fresh = 0;
    if (n > avail) {
      if (lane == 0) fresh = (long long)atomicAdd(counter, 32ull);
      fresh = __shfl_sync(0xffffffffu, fresh, 0);
    }
    const long long idx = rank < avail ? base + used + rank : fresh + (rank - avail);
    if (n > avail) {
      base = fresh;
      used = n - avail;
    } else {
      used += n;
    }
    return idx;
  }
};

// Ray setup in a pre-pass (round 0): the clip / frustum / pixel-ray code and
// the rays that miss the volume leave the sample loop, whose code then fits
// the instruction caches better (its warps stalled 37 % on instruction
// fetch). The sample phase loads a hit ray's chord from its record.
#ifndef VDI_SETUP_PASS
#define VDI_SETUP_PASS 1
#endif

// Round 0 enumerates 8x4 pixel tiles; later rounds the deferred list.
// Returns a local list index, -1 for an empty slot, -2 when exhausted.
__device__ __forceinline__ int source_list(const GenConst& c, long long slot) {
  if (c.round == 0) {
    if (slot >= c.n_slots) return -2;
    const long long tile = slot >> 5;
    const int w = (int)(slot & 31);
    const int lx = (int)(tile % c.tiles_x) * kTileW + (w & 7);
    const int ly = (int)(tile / c.tiles_x) * kTileH + (w >> 3);
    return (lx < c.a.width && ly < c.local_h) ? ly * c.a.width + lx : -1;
  }
  if (slot >= (long long)c.prev->ndefer) return -2;
  return c.defer_in[slot];
}

// The sample phase's queue: round 0 the tile slots, a miss (setup pre-pass
// hit bit clear) as an empty slot; later rounds the deferred list. The
// tiles keep their order, so neighbouring warps sample neighbouring rays (a
// compacted queue of hits, appended warp by warp, measured C4 73 -> 87 ms:
// the f32 gathers lost their L2 locality).
__device__ __forceinline__ int sample_source(const GenConst& c, long long slot) {
  if (VDI_SETUP_PASS && c.round == 0 && slot < c.n_slots &&
      !((c.hitbits[slot >> 5] >> (slot & 31)) & 1u))
    return -1;
  return source_list(c, slot);
}

// A hit ray's state from its record (written by the setup pre-pass, or by
// the sample phase of an earlier round for a deferred ray): setup_ray's
// result without recomputing it.
__device__ __forceinline__ bool load_ray(const GenConst& c, RayState& s, int list) {
  const RayRec* r = c.recs + list;
  s.list = list;
  s.seg = c.a.segs + (long long)list * list_stride(c.a.n_sg);
  s.o[0] = c.a.eye[0];
  s.o[1] = c.a.eye[1];
  s.o[2] = c.a.eye[2];
  s.d[0] = r->d[0];
  s.d[1] = r->d[1];
  s.d[2] = r->d[2];
  s.t0 = r->t0;
  s.t1 = r->t1;
  s.nsteps = r->nsteps;
  init_bisection(c, s);
  start_pass(s, s.bis_gamma, kCount);
  s.first_vis = -1;
  return true;
}

// Round 0 setup pre-pass: one thread per tile slot; a miss publishes its
// empty list here, a hit writes its chord to its record and sets its hit bit
// (warp-aggregated, so the queue keeps the tile order).
__global__ void __launch_bounds__(kGenThreads) gen_setup_kernel(const GenConst c) {
  const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int list = slot < c.n_slots ? source_list(c, slot) : -1;
  bool hit = false;
  if (list >= 0) {
    RayState s;
    hit = setup_ray<false>(c, s, list);
    if (!hit) {  // finish_ray's per-list outputs; the slot is zeroed below
      c.a.counts[list] = 0;
      if (c.a.gammas) c.a.gammas[list] = 0.0;
      if (c.a.passes) c.a.passes[list] = 0;
      if (c.a.samples) c.a.samples[list] = 0;
    } else {
      RayRec* r = c.recs + list;
      r->d[0] = s.d[0];
      r->d[1] = s.d[1];
      r->d[2] = s.d[2];
      r->t0 = s.t0;
      r->t1 = s.t1;
      r->nsteps = s.nsteps;
      r->list = list;
    }
  }
  // the misses' list slots zeroed by the whole warp, one coalesced slot at a
  // time (finish_ray's zero-fill of all n_sg entries; the slot's padding too)
  const int stride = list_stride(c.a.n_sg);
  for (unsigned mm = __ballot_sync(0xffffffffu, list >= 0 && !hit); mm; mm &= mm - 1) {
    const int l = __shfl_sync(0xffffffffu, list, __ffs(mm) - 1);
    float4* slot4 = reinterpret_cast<float4*>(c.a.segs + (long long)l * stride);
    for (int i = lane; i < stride / 4; i += 32) slot4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // a warp is one tile: slots [32 w, 32 w + 32), one word of hit bits
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  if (lane == 0 && slot < c.n_slots) c.hitbits[slot >> 5] = m;
}

__device__ __forceinline__ void load_lut(const GenConst& c, double4* s_lut, double* s_u8) {
  for (int i = threadIdx.x; i < c.a.lut_n; i += blockDim.x) {
    const float4 l = reinterpret_cast<const float4*>(c.a.lut)[i];
    s_lut[i] = make_double4(l.x, l.y, l.z, l.w);
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    s_u8[i] = (double)__fdiv_rn((float)i, 255.0f);
  __syncthreads();
}

// ------------------------------------------------------------ sample phase
template <int VT>
__global__ void __launch_bounds__(kGenThreads, VDI_SAMPLE_MINB) gen_sample_kernel(const GenConst c) {
  extern __shared__ double4 s_lut[];
  __shared__ double s_u8[256];
  load_lut(c, s_lut, s_u8);
  const int lane = threadIdx.x & 31;
  const double step = c.a.step;
  WarpPool pool;
  bool have = false, done = false;
  RayState s;

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const long long idx = pool.take(need, lane, &c.ctl->fetch);
      if ((need >> lane) & 1u) {
        const int list = VDI_SETUP_PASS ? sample_source(c, idx) : source_list(c, idx);
        if (list == -2) {
          done = true;
        } else if (list >= 0) {
          have = VDI_SETUP_PASS ? load_ray(c, s, list) : setup_ray(c, s, list);
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    const double ta = s.t0 + (double)s.k * step;
    double tb = ta + step;
    if (tb > s.t1) tb = s.t1;
    {
      // pass 1 on the fly (gamma_init, counting mode)
      int ended = 0;
      if (tb > ta) {
        bool ess_hit = false;
        const float4 rgba = sample_at<VT>(c, s_lut, s_u8, s, ta, tb, &ess_hit);
        if (s.first_vis < 0 && rgba.w > 0.0f) s.first_vis = s.k;
        int run = 1;
        if (ess_hit) {
          // a run of samples in an empty brick: transparent, counted, not
          // sampled (never the last sample, whose tb is clipped to t1)
          run = empty_run<VT>(c, s_u8, s.o, s.d, 0.5 * (ta + tb), step, s.nsteps - 1 - s.k);
          if (run < 1) run = 1;
        }
        ended = segment_step(c, s, rgba, ta, tb, run);
      }
      if (ended < 0) continue;
      if (ended == 0) ended = close_pass(c, s);
      if (ended <= c.a.n_sg) {  // pass 1 fits: the bisection ends here
        s.passes = 1;
        finish_ray(c, s, s.bis_gamma, ended);
        have = false;
        continue;
      }
      // overflow: needs the bisection -> reserve its cache run
      const unsigned long long at =
          VDI_ALLOC_IMAGE ? 0ull : atomicAdd(&c.ctl->bump, (unsigned long long)s.nsteps);
      if (!VDI_ALLOC_IMAGE && at + (unsigned long long)s.nsteps > c.cache_cap) {
        const unsigned long long j = atomicAdd(&c.ctl->ndefer, 1ull);
        c.defer_out[j] = s.list;
        have = false;
        continue;
      }
      // queue it (its record at its list index; the queue is compacted in
      // image order after this phase); gen_fill_kernel stores its samples
      // one warp per ray
      RayRec r;
      r.d[0] = s.d[0];
      r.d[1] = s.d[1];
      r.d[2] = s.d[2];
      r.t0 = s.t0;
      r.t1 = s.t1;
      r.slot = (long long)at;
      r.list = s.list;
      r.nsteps = s.nsteps;
      r.samples = s.samples;
      r.passes = 1;
      r.g_final = 0.0;
      r.mode_final = kCount;
      r.first_vis = s.first_vis;
      c.recs[s.list] = r;
      atomicOr(c.qbits + (s.list >> 5), 1u << (s.list & 31));
      // overflow order (VDI_REPLAY_ORDER 0 only)
      if (!VDI_REPLAY_ORDER) c.torder[atomicAdd(&c.ctl->ntorder, 1ull)] = s.list;
      have = false;
    }
  }
}

// The bisect / emit queue: its length and its idx-th ray (see VDI_REPLAY_ORDER;
// with image-order allocation the overflow order also lists the deferred
// rays, whose slot is -1).
__device__ __forceinline__ long long replay_queue_len(const GenConst& c) {
  return (long long)(VDI_REPLAY_ORDER ? c.ctl->nrec
                                      : (VDI_ALLOC_IMAGE ? c.ctl->ntorder : c.ctl->nrec));
}
__device__ __forceinline__ int replay_queue_at(const GenConst& c, long long idx) {
  return VDI_REPLAY_ORDER ? c.qidx[idx] : c.torder[idx];
}

// Fill: VDI_FILL_FROM_VISIBLE starts at the chunk of pass 1's first visible
// sample; VDI_FILL_SPARSE writes only the head entry of a transparent run (the
// replays jump over runs, so the other entries are never read).
#ifndef VDI_FILL_FROM_VISIBLE
#define VDI_FILL_FROM_VISIBLE 1
#endif
#ifndef VDI_FILL_SPARSE
#define VDI_FILL_SPARSE 1
#endif

// -------------------------------------------------------------- fill phase
// One warp per queued ray: lane j classifies sample kb + j of 32-sample chunks
// and stores it in the ray's cache run (coalesced 512 B per chunk, coherent
// gathers, no lane idles on another ray). Transparent runs are run-length
// coded with ballot masks: a run's head entry holds the distance to the next
// visible sample (or to the end of the row); the open run of a chunk is
// carried to the next. The non-transparent entries carry the pow flag (sign
// of r) exactly as the lane-per-ray fill did. Sets rec->nsteps to the number
// of samples stored (the tb <= ta break, generate.py:113-117, stops earlier).
template <int VT>
__global__ void VDI_FILL_BOUNDS gen_fill_kernel(const GenConst c) {
  extern __shared__ double4 s_lut[];
  __shared__ double s_u8[256];
  load_lut(c, s_lut, s_u8);
  const int lane = threadIdx.x & 31;
  const long long nrec = (long long)c.ctl->nrec;
  const double step = c.a.step;
  RayState s;
  s.o[0] = c.a.eye[0];
  s.o[1] = c.a.eye[1];
  s.o[2] = c.a.eye[2];
  while (true) {
    long long idx = 0;
    if (lane == 0) idx = (long long)atomicAdd(&c.ctl->ffetch, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= nrec) break;
    RayRec* rec = c.recs + c.qidx[idx];
    s.d[0] = rec->d[0];
    s.d[1] = rec->d[1];
    s.d[2] = rec->d[2];
    s.t0 = rec->t0;
    s.t1 = rec->t1;
    const int nsteps = rec->nsteps;
    float4* cache = c.cache + rec->slot;
    int open_head = -1;  // warp-uniform
    int stored = nsteps;
    // pass 1 (the sample phase) found samples 0 .. first_vis - 1 transparent
    // (the same classification): one run from 0, so the fill starts at the
    // chunk of the first visible sample and patches the run's head there
    int kb0 = 0;
    const int fv = VDI_FILL_FROM_VISIBLE ? rec->first_vis : -1;
    if (fv >= 32 && fv < stored) {
      if (lane == 0) cache[0] = make_float4(__int_as_float(1), 0.f, 0.f, 0.f);
      open_head = 0;
      kb0 = fv & ~31;
    }
    for (int kb = kb0; kb < stored; kb += 32) {
      const int k = kb + lane;
      bool valid = k < stored;
      double ta = 0.0, tb = 0.0;
      if (valid) {
        ta = s.t0 + (double)k * step;
        tb = ta + step;
        if (tb > s.t1) tb = s.t1;
        valid = tb > ta;
      }
      // the reference loop breaks at the first k with tb <= ta
      const unsigned broke = __ballot_sync(0xffffffffu, k < stored && !valid);
      if (broke) stored = kb + __ffs(broke) - 1;
      valid = k < stored;
      float4 rgba = make_float4(0.f, 0.f, 0.f, 0.f);
      bool in_empty = false;
      if (valid) rgba = sample_at<VT>(c, s_lut, s_u8, s, ta, tb, &in_empty);
#ifdef VDI_FILL_STATS
      {
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        const unsigned emask = __ballot_sync(0xffffffffu, valid && in_empty);
        const unsigned tmask = __ballot_sync(0xffffffffu, valid && rgba.w <= 0.0f);
        if (lane == 0 && vmask) {
          atomicAdd(&c.ctl->st_chunks, 1ull);
          if (emask == vmask) atomicAdd(&c.ctl->st_chunks_empty, 1ull);
          if (tmask == vmask) atomicAdd(&c.ctl->st_chunks_transp, 1ull);
        }
      }
#endif
      const bool transp = valid && rgba.w <= 0.0f;
      const unsigned tm = __ballot_sync(0xffffffffu, transp);
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      const unsigned nt = vm & ~tm;  // visible samples of the chunk
      // a transparent lane 0 continues the run carried from the previous chunk
      const unsigned prev_t = (tm << 1) | (open_head >= 0 ? 1u : 0u);
      const unsigned heads = tm & ~prev_t;
      // close the carried run at the chunk's first visible sample
      if (open_head >= 0 && nt) {
        if (lane == 0)
          cache[open_head].x = __int_as_float(kb + __ffs(nt) - 1 - open_head);
        open_head = -1;
      }
      // a run's non-head entries are never read (VDI_FILL_SPARSE: not written)
      if (valid && (!VDI_FILL_SPARSE || !transp || ((heads >> lane) & 1u))) {
        float4 st;
        if (transp) {
          int len = 1;
          if ((heads >> lane) & 1u) {
            const unsigned after = nt & ~((2u << lane) - 1u);
            len = after ? __ffs(after) - 1 - lane : 1;  // open runs are patched later
          }
          st = make_float4(__int_as_float(len), 0.f, 0.f, 0.f);
        } else {
          const double dt = tb - ta;
          const double e = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
          st = rgba;
          if (e != 1.0) st.x = __int_as_float(__float_as_int(st.x) | 0x80000000);
        }
        cache[k] = st;
      }
      // the last head without a visible sample after it stays open
      if (heads) {
        const int last = 31 - __clz(heads);
        const unsigned after = nt & ~((2u << last) - 1u);
        if (!after) open_head = kb + last;
      }
      __syncwarp();
    }
    if (open_head >= 0 && lane == 0) cache[open_head].x = __int_as_float(stored - open_head);
    if (lane == 0) rec->nsteps = stored;
    __syncwarp();
  }
}

// ------------------------------------------------------------ bisect phase
// Passes 2.. of the bisection (generate.py:237-273) for the queued rays, as
// COUNT-ONLY replays: a counting pass's decisions (split, abort, transparent
// close) depend only on the running mean of premultiplied samples, never on
// the accumulated colour or the stored segments, so n(gamma) needs a few
// registers and no writes. The deciding (gamma, mode) is handed to the emit
// phase, which re-runs that one pass with full logic.
//
// Speculation: one replay evaluates the next kLevels levels of the bisection
// tree at once -- G = 2^kLevels - 1 gammas in heap order, node i's children
// being (gamma_i, high_i) [n > n_sg] at 2i+1 and (low_i, gamma_i) [n < n_sg -
// delta] at 2i+2, each gamma = 0.5 * (low + high) exactly as the reference
// forms it. The G count states are independent (ILP against FP64 latency) and
// share each loaded sample; R's control flow (epsilon tests included) is then
// replayed over the counts, so results and the reported passes/samples are
// exactly the reference's.

// Cache rows are read sequentially by one lane; a 128 B line holds 8 entries.
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}
// TMA bulk prefetch of `bytes` (multiple of 16, 16-B aligned) into L2
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
constexpr int kBulkEntries = 32;  // 512 B of cache row per bulk prefetch

// A lane's stream of cache entries: b[i] holds entry k + i (loads in flight),
// plus a cache-level prefetch kAhead entries ahead at line crossings
// (PF: 0 none, 1 into L1, 2 into L2, 3 = 1 plus a bulk L2 prefetch of the next
// kBulkEntries-entry chunk whenever the lane enters a chunk).
template <int D, int PF, int kAhead = 16>
struct EntryPipe {
  float4 b[D];
  __device__ __forceinline__ float4 cur() const { return b[0]; }
  __device__ __forceinline__ void prefetch(const float4* row, int at, int stored) {
    if (at < stored) {
      if (PF == 1 || PF == 3) prefetch_l1(row + at);
      if (PF == 2) prefetch_l2(row + at);
    }
  }
  __device__ __forceinline__ void bulk(const float4* row, int chunk, int stored) {
    const int at = chunk * kBulkEntries;
    if (at < stored) {
      const int n = stored - at < kBulkEntries ? stored - at : kBulkEntries;
      prefetch_l2_bulk(row + at, 16u * (unsigned)n);
    }
  }
  __device__ __forceinline__ void start(const float4* row, int k, int stored) {
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (k + i < stored) b[i] = row[k + i];
    if (PF) {
      prefetch(row, (k & ~7) + 8, stored);
      if (kAhead > 8) prefetch(row, (k & ~7) + kAhead, stored);
    }
    if (PF == 3) {
      bulk(row, k / kBulkEntries, stored);
      bulk(row, k / kBulkEntries + 1, stored);
    }
  }
  __device__ __forceinline__ void advance(const float4* row, int kold, int k, int stored) {
    if (k == kold + 1) {
#pragma unroll
      for (int i = 0; i + 1 < D; ++i) b[i] = b[i + 1];
      if (k + D - 1 < stored) b[D - 1] = row[k + D - 1];
    } else {
#pragma unroll
      for (int i = 0; i < D; ++i)
        if (k + i < stored) b[i] = row[k + i];
    }
    if (PF && (((kold + kAhead) ^ (k + kAhead)) & ~7) != 0)
      prefetch(row, k + kAhead, stored);
    if (PF == 3 && kold / kBulkEntries != k / kBulkEntries)
      bulk(row, k / kBulkEntries + 1, stored);
  }
};

// Two-slot ring with a parity bit: the entry after the current one is loaded
// straight into the slot just consumed, so no register shuffle follows the
// load (EntryPipe's b[0] = b[1] shift made ptxas load into a temporary and
// move it into place right after the LDG -- a stall on every sample).
// predicated 16-B load into the registers of `v` itself (left unchanged when
// !pred): written in PTX so the compiler cannot load into a temporary and
// select afterwards
// Asynchronous 16-B copies global -> shared (LDGSTS), for the kMode 3 rings:
// a lane keeps its next cache entries in flight in shared memory instead of
// registers. src-size 0 copies nothing (zero-fills), so the issue needs no
// branch past the end of a row.
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ float4 lds128(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ void ld_pred(float4& v, const float4* p, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " @q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n}\n"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
      : "l"(p), "r"((int)pred));
}

template <int PF, int kAhead = 16>
struct EntryRing {
  float4 b0, b1;
  bool par;  // current entry in b1
  __device__ __forceinline__ float4 cur() const {
    float4 e;
    e.x = par ? b1.x : b0.x;
    e.y = par ? b1.y : b0.y;
    e.z = par ? b1.z : b0.z;
    e.w = par ? b1.w : b0.w;
    return e;
  }
  __device__ __forceinline__ void prefetch(const float4* row, int at, int stored) {
    if (PF == 1 && at < stored) prefetch_l1(row + at);
  }
  __device__ __forceinline__ void start(const float4* row, int k, int stored) {
    par = false;
    if (k < stored) b0 = row[k];
    if (k + 1 < stored) b1 = row[k + 1];
    if (PF) {
      prefetch(row, (k & ~7) + 8, stored);
      if (kAhead > 8) prefetch(row, (k & ~7) + kAhead, stored);
    }
  }
  __device__ __forceinline__ void advance(const float4* row, int kold, int k, int stored) {
    if (k == kold + 1) {
      const bool more = k + 1 < stored;
      ld_pred(b1, row + k + 1, more && par);
      ld_pred(b0, row + k + 1, more && !par);
      par = !par;
    } else {
      start(row, k, stored);
      return;
    }
    if (PF && (((kold + kAhead) ^ (k + kAhead)) & ~7) != 0)
      prefetch(row, k + kAhead, stored);
  }
};

// The leading c.inv_smem entries of the 1/n table live in dynamic shared
// memory (larger n read the global table). The table is read through a 32-bit
// shared address computed once per thread (ld.shared): plain C++ accesses made
// the compiler rebuild the CTA's shared window base (S2R SR_CgaCtaId + LEA) at
// every read in the hot loop.
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// opened = the segments opened so far = R's count + (a segment is open): a
// transparent sample only closes (opened unchanged), a visible one that does
// not merge opens one (a split closes one and opens one), and R aborts a
// counting pass exactly when a visible sample would open segment n_sg + 1
// (generate.py:146-150, 176-180), i.e. !merge && opened >= n_sg. At the
// natural end R's n = count + active = opened.
// kend == 0 while the state is live; an abort sets kend = k + 1 (n stays
// n_sg + 1), the natural end sets kend = stored and n = opened.
struct CountState {
  double mr, mg, mb, thr;
  int opened, nsamp, kend, n;
  bool active;
};

__device__ __forceinline__ void count_reset(CountState& q, double gamma, int n_sg) {
  q.thr = split_threshold(gamma);
  q.mr = q.mg = q.mb = 0.0;
  q.opened = 0;
  q.nsamp = 0;
  q.kend = 0;
  q.n = n_sg + 1;
  q.active = false;
}

// One non-transparent sample for one count state (generate.py:166-212 minus
// the colour accumulation), branch-free: both outcomes are computed and
// selected so the G states of a lane run as straight-line FP64 code.
//  * t = s - m is exactly -(m - s), so t*t reproduces R's dr*dr bit for bit and
//    m + t*inv is R's `m += (s - m) * inv`;
//  * 1/n comes from the table of host-identical IEEE quotients;
//  * a resolved state (n >= 0) keeps stepping -- only its n and kend are
//    frozen, and nothing else of it is read again -- so the update needs no
//    guard (a guarded update compiled to a divergent branch per state).
// kSmemOnly: every 1/n the ray can need is in the shared table.
template <bool kTrack = false, bool kSmemOnly = false>
__device__ __forceinline__ void count_sample(CountState& q, double sr, double sg, double sb,
                                             int k, int n_sg, int inv_n, const double* g_inv,
                                             unsigned s_inv, double* d2max = nullptr,
                                             bool* split_seen = nullptr) {
  const double tr = sr - q.mr, tg = sg - q.mg, tb = sb - q.mb;
  const double d2 = tr * tr + tg * tg + tb * tb;
  const bool far = d2 >= q.thr;
  const bool live = q.kend == 0;
  const bool merge = q.active && !far;
  if (kTrack) {
    // the split test's d^2 along this state's trajectory (see gen_bisect_kernel;
    // read only when the state ran to the natural end, i.e. was live on
    // every step, so the steps after an abort need no guard)
    if (q.active && d2 > *d2max) *d2max = d2;
    if (q.active && far) *split_seen = true;
  }
  const bool abort = !merge && q.opened >= n_sg;
  const int ns = q.nsamp + 1;
  // nsamp <= max_steps, which the global table always covers; the shared copy
  // holds the first inv_n entries (selecting between two loads, never a
  // reciprocal sequence)
  const double inv = kSmemOnly ? lds_f64(s_inv + 8u * (unsigned)ns)
                               : (ns < inv_n ? lds_f64(s_inv + 8u * (unsigned)ns)
                                             : __ldg(g_inv + ns));
  const double nr = q.mr + tr * inv, ng = q.mg + tg * inv, nb = q.mb + tb * inv;
  q.kend = live && abort ? k + 1 : q.kend;
  q.opened += merge ? 0 : 1;
  q.mr = merge ? nr : sr;
  q.mg = merge ? ng : sg;
  q.mb = merge ? nb : sb;
  q.nsamp = merge ? ns : 1;
  q.active = true;
}

// kMode: how a lane streams its cache row -- 0 EntryPipe (register shift),
// 1 EntryRing (two slots, parity select), 2 A/B: the sample loop unrolled by
// two with static slot roles (step A reads only b0, step B only b1), so the
// load of an entry has a full A+B iteration to land and no instruction reads
// a slot whose load is in flight (scoreboards are per warp: EntryRing's
// select reads both slots and waits for both).
template <int kLevels, int kDepth, int kPF, int kMinB = 1, int kThreads = kGenThreads,
          int kAhead = 16, int kMode = 0, bool kSmemOnly = false>
__global__ void __launch_bounds__(kThreads, kMinB) gen_bisect_kernel(const GenConst c) {
  constexpr int kG = (1 << kLevels) - 1;
  extern __shared__ double g_s_inv[];
  // 1/n for the running means: host-identical IEEE quotients in shared memory
  const int inv_n = c.inv_n < c.inv_smem ? c.inv_n : c.inv_smem;
  for (int i = threadIdx.x; i < inv_n; i += blockDim.x) g_s_inv[i] = c.inv_tab[i];
  // opaque copy: keeps the address in a register instead of letting ptxas
  // rematerialise it from SR_CgaCtaId at every use
  unsigned s_inv;
  asm volatile("mov.u32 %0, %1;\n" : "=r"(s_inv) : "r"((unsigned)__cvta_generic_to_shared(g_s_inv)));
  // kMode 3: this lane's ring of kDepth cache entries, slot-major (slot j of
  // thread t at (j * kThreads + t) * 16: conflict-free across the warp)
  __shared__ float4 s_ring[kMode == 3 ? kDepth * kThreads : 1];
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(s_ring) + 16u * threadIdx.x;
  auto ring_at = [&](int k) -> unsigned {
    return ring0 + 16u * (unsigned)kThreads * (unsigned)(k & (kDepth - 1));
  };
  // entries k .. k + kDepth - 2 in flight, one commit group each
  auto ring_fill = [&](const float4* row, int k, int stored) {
    cp_async_wait<0>();  // a stale copy must not land over a new one
#pragma unroll
    for (int j = 0; j < kDepth - 1; ++j) {
      cp_async16(ring_at(k + j), row + (k + j < stored ? k + j : 0), k + j < stored);
      cp_async_commit();
    }
  };
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nrec = replay_queue_len(c);
  const int n_sg = c.a.n_sg;
  WarpPool pool;
  bool have = false, done = false, top = false;
  const float4* cache = nullptr;
  RayRec* rec = nullptr;
  int stored = 0, k = 0;
  typename std::conditional<kMode == 1, EntryRing<kPF, kAhead>,
                            EntryPipe<kDepth, kPF, kAhead>>::type pipe;
  float4 b0, b1;  // kMode 2: entries k and k+1 at the top of the unrolled loop
  // bisection state (generate.py:230-236)
  double low = 0.0, high = 0.0;
  int last_n = 0, high_n = 0, passes = 0, samples = 0;
  bool chain = false;  // this replay's speculation shape (see the top of the loop)
  int reps = 0;        // replays run on the current ray
  int cdir = 0;        // chain directions (bit i set: step i goes up)
  // No-split certificate: state 0 (this replay's largest gamma) records the
  // largest d^2 its split test saw and whether it split. With no split, its
  // trajectory is the gamma = inf one, so every gamma' with sqrt(d2max0) <
  // gamma' has no split either and the same count -- such levels need no
  // replay (their pass runs to the natural end: samples += stored).
  double d2max0 = 0.0;
  bool split0 = false;
  CountState q[kG];
#ifdef VDI_BISECT_STATS
  unsigned long long st_vis = 0, st_run = 0, st_run_entries = 0, st_replays = 0;
#endif

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const long long idx = pool.take(need, lane, &c.ctl->rfetch);
      if ((need >> lane) & 1u) {
        if (idx >= nrec) {
          done = true;
        } else if (c.recs[replay_queue_at(c, idx)].slot >= 0) {  // (deferred: slot -1)
          rec = c.recs + replay_queue_at(c, idx);
          cache = c.cache + rec->slot;
          stored = rec->nsteps;
          // state after the overflowing pass 1 (generate.py:253-273)
          low = c.a.gamma_init;
          high = kSqrt3;
          last_n = n_sg + 1;
          high_n = -1;
          passes = rec->passes;
          samples = rec->samples;
          have = true;
          top = true;
          reps = 0;
          if (c.wide_after == 0 && c.wide != nullptr) {  // straight to the wide phase
            rec->low = low;
            rec->high = high;
            rec->last_n = last_n;
            rec->high_n = high_n;
            c.wide[atomicAdd(&c.ctl->nwide, 1ull)] = (int)(rec - c.recs);
            have = false;
          }
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    if (top) {
      // top of the bisection loop: epsilon exit, or a replay of the next
      // kLevels levels
      top = false;
      if (fabs(high - low) < c.a.eps) {
        if (last_n == 0) {
          rec->g_final = low;
          rec->mode_final = kCapped;
          passes += 1;
        } else if (high_n >= 0) {
          rec->g_final = high;  // the cached high-gamma segments
          rec->mode_final = kCount;
        } else {
          rec->g_final = high;
          rec->mode_final = kCapped;
          passes += 1;
        }
        rec->passes = passes;
        rec->samples = samples;
        have = false;
        continue;
      }
      // speculation shape: the tree (node, both children) or, while the
      // bisection is in its first levels, where it goes down almost always
      // (tools/bisect_paths.py), the chain node -> down -> down, which covers
      // kG levels instead of kLevels when the prediction holds
      // Beyond those levels, a level whose decisions so far (this round, all
      // rays: ctl->dir) lean strongly one way gets a chain in that direction
      // when the next level leans too; otherwise the tree. The shape only
      // changes how many levels a replay covers, never a result.
      const int lvl0 = passes - 1;
      chain = kLevels == 2 && lvl0 < c.chain_levels;
      cdir = 0;  // bit i: the chain's step i goes up
      if (kLevels == 2 && !chain && lvl0 + 1 < 32 && c.learn) {
        int dirs = 0;
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const unsigned u = *((volatile unsigned*)&c.ctl->dir[0][lvl0 + j]);
          const unsigned dn = *((volatile unsigned*)&c.ctl->dir[1][lvl0 + j]);
          const unsigned tot = u + dn;
          if (tot < 256u) ok = false;
          else if (4u * u >= 3u * tot) dirs |= 1 << j;
          else if (!(4u * dn >= 3u * tot)) ok = false;
        }
        if (ok) {
          chain = true;
          cdir = dirs;
        }
      }
      double lo[kG], hi[kG], gam[kG];
      lo[0] = low;
      hi[0] = high;
#pragma unroll
      for (int i = 0; i < kG; ++i) {
        gam[i] = 0.5 * (lo[i] + hi[i]);
        if (chain) {
          if (i + 1 < kG) {
            const bool up = (cdir >> i) & 1;
            lo[i + 1] = up ? gam[i] : lo[i];
            hi[i + 1] = up ? hi[i] : gam[i];
          }
        } else if (2 * i + 2 < kG) {
          lo[2 * i + 1] = gam[i];
          hi[2 * i + 1] = hi[i];
          lo[2 * i + 2] = lo[i];
          hi[2 * i + 2] = gam[i];
        }
        count_reset(q[i], gam[i], n_sg);
      }
      d2max0 = 0.0;
      split0 = false;
#ifdef VDI_BISECT_STATS
      st_replays += 1;
#endif
      k = 0;
      if (kMode == 3) {
        // samples before pass 1's first visible one are one transparent run
        // from 0 (the fill's head entry): a replay may start past it with the
        // same (reset) count states
        const int k0 = rec->first_vis;
        if (k0 > 0 && k0 < stored) k = k0;
        ring_fill(cache, k, stored);
      } else if (kMode == 2) {
        ld_pred(b0, cache, 0 < stored);
        ld_pred(b1, cache + 1, 1 < stored);
        if (kPF) prefetch_l1(cache + 8);
      } else {
        pipe.start(cache, 0, stored);
      }
    }

    bool resolved = false;
    // one sample (or a transparent run) for all kG count states; returns the
    // entries consumed
    auto consume = [&](const float4 e) -> int {
      int run = 1;
      if (e.w <= 0.0f) {
        run = __float_as_int(e.x);
        if (run < 1) run = 1;
        if (run > stored - k) run = stored - k;
#ifdef VDI_BISECT_STATS
        st_run += 1;
        st_run_entries += run;
#endif
#pragma unroll
        for (int i = 0; i < kG; ++i) {
          // the transparent sample closes the segment (resolved states may
          // keep stepping, see count_sample)
          q[i].active = false;
        }
      } else {
        const double a = (double)e.w;
        double a_adj;
        if (entry_needs_pow(e)) {
          const double ta = rec->t0 + (double)k * c.a.step;
          double tb = ta + c.a.step;
          if (tb > rec->t1) tb = rec->t1;
          const double dt = tb - ta;
          const double ex = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
          a_adj = 1.0 - pow(1.0 - a, ex);
        } else {
          a_adj = 1.0 - (1.0 - a);
        }
        const double sr = (double)fabsf(e.x) * a_adj;
        const double sg = (double)e.y * a_adj;
        const double sb = (double)e.z * a_adj;
        count_sample<true, kSmemOnly>(q[0], sr, sg, sb, k, n_sg, inv_n, c.inv_tab, s_inv,
                                      &d2max0, &split0);
#pragma unroll
        for (int i = 1; i < kG; ++i)
          count_sample<false, kSmemOnly>(q[i], sr, sg, sb, k, n_sg, inv_n, c.inv_tab, s_inv);
#ifdef VDI_BISECT_STATS
        st_vis += 1;
#endif
      }
      return run;
    };
    auto all_resolved = [&]() {
      bool r = true;
#pragma unroll
      for (int i = 0; i < kG; ++i) r = r && q[i].kend != 0;
      return r;
    };
    auto natural_end = [&]() {
      // natural end (or the tb <= ta break)
#pragma unroll
      for (int i = 0; i < kG; ++i)
        if (q[i].kend == 0) {
          q[i].n = q[i].opened;
          q[i].kend = stored;
        }
    };
    if (kMode == 3) {
      for (int it = 0; it < 16; ++it) {
        if (k >= stored) {
          natural_end();
          resolved = true;
          break;
        }
        cp_async_wait<kDepth - 2>();  // entry k's group has landed
        const float4 e = lds128(ring_at(k));
        const int kold = k;
        k += consume(e);
        if (k != kold + 1) {  // skipped a transparent run: restart the ring at k
          ring_fill(cache, k, stored);
          continue;
        }
        // entry k + kDepth - 2 into the slot entry k - 2 vacated
        const int kn = k + kDepth - 2;
        cp_async16(ring_at(kn), cache + (kn < stored ? kn : 0), kn < stored);
        cp_async_commit();
        if ((it & 1) && all_resolved()) {  // tested every other step (see kMode 2)
          resolved = true;
          break;
        }
      }
    }
    if (kMode == 2) {
      for (int it = 0; it < 8; ++it) {
        if (k >= stored) {
          natural_end();
          resolved = true;
          break;
        }
        // step A: b0 = entry k, b1 = entry k + 1 (resolution is tested after
        // step B only: a resolved state's n and kend are frozen, so one more
        // step costs a step, not a result)
        int kold = k;
        k += consume(b0);
        if (k != kold + 1) {  // skipped a transparent run: refill both slots
          ld_pred(b0, cache + k, k < stored);
          ld_pred(b1, cache + k + 1, k + 1 < stored);
          if (kPF) prefetch_l1(cache + (k & ~7) + 8);
          continue;
        }
        ld_pred(b0, cache + k + 1, k + 1 < stored);
        if (kPF && (((kold + kAhead) ^ (k + kAhead)) & ~7) != 0 && k + kAhead < stored)
          prefetch_l1(cache + k + kAhead);
        if (k >= stored) continue;
        // step B: b1 = entry k, b0 = entry k + 1
        kold = k;
        k += consume(b1);
        if (all_resolved()) {
          resolved = true;
          break;
        }
        if (k != kold + 1) {
          ld_pred(b0, cache + k, k < stored);
          ld_pred(b1, cache + k + 1, k + 1 < stored);
          if (kPF) prefetch_l1(cache + (k & ~7) + 8);
          continue;
        }
        ld_pred(b1, cache + k + 1, k + 1 < stored);
        if (kPF && (((kold + kAhead) ^ (k + kAhead)) & ~7) != 0 && k + kAhead < stored)
          prefetch_l1(cache + k + kAhead);
      }
    }
    for (int it = 0; kMode < 2 && it < 16 && !resolved; ++it) {
     if (k >= stored) {
      // natural end (or the tb <= ta break)
#pragma unroll
      for (int i = 0; i < kG; ++i)
        if (q[i].kend == 0) {
          q[i].n = q[i].opened;
          q[i].kend = stored;
        }
      resolved = true;
     } else {
      const float4 e = pipe.cur();
      int run = 1;
      if (e.w <= 0.0f) {
        run = __float_as_int(e.x);
        if (run < 1) run = 1;
        if (run > stored - k) run = stored - k;
#pragma unroll
        for (int i = 0; i < kG; ++i)
          q[i].active = false;  // the transparent sample closes the segment
      } else {
        const double a = (double)e.w;
        double a_adj;
        if (entry_needs_pow(e)) {
          const double ta = rec->t0 + (double)k * c.a.step;
          double tb = ta + c.a.step;
          if (tb > rec->t1) tb = rec->t1;
          const double dt = tb - ta;
          const double ex = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
          a_adj = 1.0 - pow(1.0 - a, ex);
        } else {
          a_adj = 1.0 - (1.0 - a);
        }
        const double sr = (double)fabsf(e.x) * a_adj;
        const double sg = (double)e.y * a_adj;
        const double sb = (double)e.z * a_adj;
        count_sample<true, kSmemOnly>(q[0], sr, sg, sb, k, n_sg, inv_n, c.inv_tab, s_inv,
                                      &d2max0, &split0);
#pragma unroll
        for (int i = 1; i < kG; ++i)
          count_sample<false, kSmemOnly>(q[i], sr, sg, sb, k, n_sg, inv_n, c.inv_tab, s_inv);
      }
      const int kold = k;
      k += run;
      pipe.advance(cache, kold, k, stored);
      resolved = true;
#pragma unroll
      for (int i = 0; i < kG; ++i) resolved = resolved && q[i].kend != 0;
     }
    }
    if (!resolved) continue;

    // replay R's control flow over the speculated counts (generate.py:237-273)
    int node = 0;
    bool fin = false;
    for (int lvl = 0; lvl < kG && node >= 0; ++lvl) {
      if (lvl > 0 && fabs(high - low) < c.a.eps) break;  // handled at the top
      // static selection keeps q[] in registers. The node's gamma is the
      // midpoint of the current bracket: every speculated state was formed
      // that way from the bracket its ancestors' decisions leave, so it need
      // not stay live through the replay
      int n = 0, kend = 0;
      const double g = 0.5 * (low + high);
#pragma unroll
      for (int i = 0; i < kG; ++i)
        if (i == node) {
          n = q[i].n;
          kend = q[i].kend;
        }
      passes += 1;
      samples += kend;
      last_n = n;
      const int plvl = passes - 2;  // this pass's bisection level
      if (n > n_sg) {
        low = g;
        if (c.learn && plvl < 32) atomicAdd(&c.ctl->dir[0][plvl], 1u);
        node = chain ? (((cdir >> node) & 1) && node + 1 < kG ? node + 1 : -1)
                     : (2 * node + 1 < kG ? 2 * node + 1 : -1);
      } else if (n < n_sg - c.a.delta) {
        high = g;
        high_n = n;
        if (c.learn && plvl < 32) atomicAdd(&c.ctl->dir[1][plvl], 1u);
        node = chain ? (!((cdir >> node) & 1) && node + 1 < kG ? node + 1 : -1)
                     : (2 * node + 2 < kG ? 2 * node + 2 : -1);
      } else {
        rec->g_final = g;  // window hit: this pass's segments
        rec->mode_final = kCount;
        rec->passes = passes;
        rec->samples = samples;
        fin = true;
        break;
      }
    }
    if (!fin && !split0 && q[0].n <= n_sg && q[0].kend == stored) {
      // levels whose gamma is above the certified no-split bound: n = q[0].n,
      // a full pass each (generate.py:237-273 with the known count)
      const double dstar = sqrt(d2max0);
      const int nv = q[0].n;
      while (fabs(high - low) >= c.a.eps) {
        const double g = 0.5 * (low + high);
        if (!(dstar < g)) break;
        passes += 1;
        samples += stored;
        last_n = nv;
        if (nv > n_sg) {  // (not reached: nv <= n_sg)
          low = g;
        } else if (nv < n_sg - c.a.delta) {
          high = g;
          high_n = nv;
        } else {
          rec->g_final = g;
          rec->mode_final = kCount;
          rec->passes = passes;
          rec->samples = samples;
          fin = true;
          break;
        }
      }
    }
    if (fin) {
      have = false;
      continue;
    }
    ++reps;
    if (c.wide != nullptr &&
        (reps >= c.wide_after ||
         (c.wide_tail &&
          *reinterpret_cast<volatile unsigned long long*>(&c.ctl->rfetch) >=
              (unsigned long long)nrec))) {
      // a long bisection: hand the ray to the wide phase, where a warp
      // replays 5 levels at once (one gamma per lane) -- it would otherwise
      // be this lane's serial tail
      rec->low = low;
      rec->high = high;
      rec->last_n = last_n;
      rec->high_n = high_n;
      rec->passes = passes;
      rec->samples = samples;
      c.wide[atomicAdd(&c.ctl->nwide, 1ull)] = (int)(rec - c.recs);
      have = false;
      continue;
    }
    top = true;
  }
  if (kMode == 3) cp_async_wait<0>();
#ifdef VDI_BISECT_STATS
  atomicAdd(&c.ctl->st_vis, st_vis);
  atomicAdd(&c.ctl->st_run, st_run);
  atomicAdd(&c.ctl->st_run_entries, st_run_entries);
  atomicAdd(&c.ctl->st_replays, st_replays);
#endif
}

// ---------------------------------------------------------- wide bisect
// The bisections the narrow lanes handed off (gen_bisect_kernel): a group of
// kLanes lanes per ray, lane i < kLanes - 1 the count state of node i of the
// next log2(kLanes) levels of the bisection tree (heap order; node i's
// children 2i + 1 for n > n_sg (low = gamma) and 2i + 2 for n < n_sg - delta
// (high = gamma), every gamma = 0.5 * (low + high) formed exactly as the
// reference forms it). The group's lanes walk the cache row in step --
// kLanes entries per coalesced load, broadcast by shuffles -- and R's control
// flow (generate.py:237-273, epsilon exits included) is replayed over the
// counts, so passes, samples and the deciding pass are the reference's.
// A narrow lane runs ~200 dependent instructions per sample for its 3
// states; here each lane runs one state, so a ray's replay latency drops
// ~3x (kLanes 8: the tail of a launch) and a replay covers 3 or 5 levels.
template <int kLanes, bool kSmemOnly>
__global__ void __launch_bounds__(kGenThreads) gen_bisect_wide_kernel(const GenConst c) {
  constexpr int kG = kLanes - 1;
  constexpr int kLevels = kLanes == 32 ? 5 : (kLanes == 16 ? 4 : (kLanes == 8 ? 3 : 2));
  extern __shared__ double g_s_inv[];
  const int inv_n = c.inv_n < c.inv_smem ? c.inv_n : c.inv_smem;
  for (int i = threadIdx.x; i < inv_n; i += blockDim.x) g_s_inv[i] = c.inv_tab[i];
  unsigned s_inv;
  asm volatile("mov.u32 %0, %1;\n" : "=r"(s_inv) : "r"((unsigned)__cvta_generic_to_shared(g_s_inv)));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int sl = lane & (kLanes - 1);                    // lane within the group
  const int g0 = lane & ~(kLanes - 1);                   // the group's first lane
  const unsigned gm = kLanes == 32 ? 0xffffffffu : (((1u << kLanes) - 1u) << g0);
  const long long nwide = (long long)c.ctl->nwide;
  const int n_sg = c.a.n_sg;
  while (true) {
    long long wi = 0;
    if (sl == 0) wi = (long long)atomicAdd(&c.ctl->wfetch, 1ull);
    wi = __shfl_sync(gm, wi, g0);
    if (wi >= nwide) break;
    RayRec* rec = c.recs + c.wide[wi];
    const float4* cache = c.cache + rec->slot;
    const int stored = rec->nsteps;
    double low = rec->low, high = rec->high;
    int last_n = rec->last_n, high_n = rec->high_n;
    int passes = rec->passes, samples = rec->samples;
    bool fin = false;
    while (!fin) {
      if (fabs(high - low) < c.a.eps) {  // generate.py:238-252 (as the narrow top)
        if (sl == 0) {
          if (last_n == 0) {
            rec->g_final = low;
            rec->mode_final = kCapped;
          } else if (high_n >= 0) {
            rec->g_final = high;
            rec->mode_final = kCount;
          } else {
            rec->g_final = high;
            rec->mode_final = kCapped;
          }
        }
        if (last_n == 0 || high_n < 0) passes += 1;
        break;
      }
      // this lane's node: its gamma from the bracket along the heap path
      CountState q;
      {
        const unsigned x = (unsigned)(sl < kG ? sl : 0) + 1u;
        const int d = 31 - __clz(x);
        double lo = low, hi = high;
        for (int b = d - 1; b >= 0; --b) {
          const double g = 0.5 * (lo + hi);
          if ((x >> b) & 1u) hi = g;
          else lo = g;
        }
        count_reset(q, 0.5 * (lo + hi), n_sg);
      }
      if (sl >= kG) q.kend = 1;  // the spare lane is resolved from the start
      // walk the row: lane sl holds entry base + sl of the current chunk of
      // kLanes entries and base + kLanes + sl of the next (loaded ahead)
      int k = 0;
      int base = -2 * kLanes;
      float4 ent = make_float4(0.f, 0.f, 0.f, 0.f), nxt = ent;
      while (true) {
        if (k >= stored) {
          if (q.kend == 0) {
            q.n = q.opened;
            q.kend = stored;
          }
          break;
        }
        if (k - base >= kLanes) {
          if (k - base < 2 * kLanes) {
            ent = nxt;
            base += kLanes;
          } else {  // start, or a transparent run past the next chunk
            base = k;
            if (base + sl < stored) ent = __ldg(cache + base + sl);
          }
          if (base + kLanes + sl < stored) nxt = __ldg(cache + base + kLanes + sl);
        }
        const int src = g0 + (k - base);
        float4 e;
        e.x = __shfl_sync(gm, ent.x, src);
        e.y = __shfl_sync(gm, ent.y, src);
        e.z = __shfl_sync(gm, ent.z, src);
        e.w = __shfl_sync(gm, ent.w, src);
        int run = 1;
        if (e.w <= 0.0f) {
          run = __float_as_int(e.x);
          if (run < 1) run = 1;
          if (run > stored - k) run = stored - k;
          // the transparent sample closes the segment (opened unchanged)
          q.active = false;
        } else {
          const double a = (double)e.w;
          double a_adj;
          if (entry_needs_pow(e)) {
            const double ta = rec->t0 + (double)k * c.a.step;
            double tb = ta + c.a.step;
            if (tb > rec->t1) tb = rec->t1;
            const double dt = tb - ta;
            const double ex = c.lref_pow2 ? dt * c.inv_lref : dt / c.a.lref;
            a_adj = 1.0 - pow(1.0 - a, ex);
          } else {
            a_adj = 1.0 - (1.0 - a);
          }
          const double sr = (double)fabsf(e.x) * a_adj;
          const double sg = (double)e.y * a_adj;
          const double sb = (double)e.z * a_adj;
          count_sample<false, kSmemOnly>(q, sr, sg, sb, k, n_sg, inv_n, c.inv_tab, s_inv);
        }
        k += run;
        if (__all_sync(gm, q.kend != 0)) break;
      }
      // replay R's control flow over the counts (generate.py:237-273)
      int node = 0;
      for (int lvl = 0; lvl < kLevels && node >= 0; ++lvl) {
        if (lvl > 0 && fabs(high - low) < c.a.eps) break;  // handled at the top
        const int n = __shfl_sync(gm, q.n, g0 + node);
        const int kend = __shfl_sync(gm, q.kend, g0 + node);
        const double g = 0.5 * (low + high);
        passes += 1;
        samples += kend;
        last_n = n;
        if (n > n_sg) {
          low = g;
          node = 2 * node + 1 < kG ? 2 * node + 1 : -1;
        } else if (n < n_sg - c.a.delta) {
          high = g;
          high_n = n;
          node = 2 * node + 2 < kG ? 2 * node + 2 : -1;
        } else {
          if (sl == 0) {
            rec->g_final = g;  // window hit: this pass's segments
            rec->mode_final = kCount;
          }
          fin = true;
          break;
        }
      }
    }
    if (sl == 0) {
      rec->passes = passes;
      rec->samples = samples;
    }
    __syncwarp(gm);
  }
}

// -------------------------------------------------------------- emit phase
// The deciding pass of every queued ray, replayed with the full
// _gen_list_pass logic: segments, counts, gammas, passes, samples.
// kRing: entries k, k + 1 in two register slots read by an A/B-unrolled loop
// (see gen_bisect_kernel kMode 2); otherwise one load per sample.
// kStream 2: a per-lane cp.async ring of kEmitRing entries in shared memory
// (as the bisect replays' kMode 3).
#ifndef VDI_EMIT_RING
#define VDI_EMIT_RING 4
#endif
constexpr int kEmitRing = VDI_EMIT_RING;
template <int kStream>
__global__ void __launch_bounds__(kGenThreads, VDI_EMIT_MINB) gen_emit_kernel(const GenConst c) {
  constexpr bool kRing = kStream == 1;
  __shared__ float4 s_ring[kStream == 2 ? kEmitRing * kGenThreads : 1];
  const unsigned ring0 = (unsigned)__cvta_generic_to_shared(s_ring) + 16u * threadIdx.x;
  auto ring_at = [&](int k) -> unsigned {
    return ring0 + 16u * (unsigned)kGenThreads * (unsigned)(k & (kEmitRing - 1));
  };
  auto ring_fill = [&](const float4* row, int k, int stored) {
    cp_async_wait<0>();
#pragma unroll
    for (int j = 0; j < kEmitRing - 1; ++j) {
      cp_async16(ring_at(k + j), row + (k + j < stored ? k + j : 0), k + j < stored);
      cp_async_commit();
    }
  };
  const int lane = threadIdx.x & 31;
  const double step = c.a.step;
  const long long nrec = replay_queue_len(c);
  WarpPool pool;
  bool have = false, done = false;
  const float4* cache = nullptr;
  int stored = 0;
  double g = 0.0;
  RayState s;
  float4 b0, b1;

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const long long idx = pool.take(need, lane, &c.ctl->efetch);
      if ((need >> lane) & 1u) {
        if (idx >= nrec) {
          done = true;
        } else if (c.recs[replay_queue_at(c, idx)].slot >= 0) {  // (deferred: slot -1)
          const RayRec r = c.recs[replay_queue_at(c, idx)];
          s.list = r.list;
          s.seg = c.a.segs + (long long)r.list * list_stride(c.a.n_sg);
          s.o[0] = c.a.eye[0];
          s.o[1] = c.a.eye[1];
          s.o[2] = c.a.eye[2];
          s.d[0] = r.d[0];
          s.d[1] = r.d[1];
          s.d[2] = r.d[2];
          s.t0 = r.t0;
          s.t1 = r.t1;
          s.nsteps = r.nsteps;
          stored = r.nsteps;
          cache = c.cache + r.slot;
          init_bisection(c, s);
          s.passes = r.passes;
          s.samples = r.samples;
          g = r.g_final;
          // window hit / cached high: a counting pass that R does not count
          // again (kRedo); capped: R's final capped pass (counted)
          start_pass(s, g, r.mode_final == kCapped ? kCapped : kRedo);
          if (kStream == 2) {
            // past pass 1's first visible sample: the run before it only
            // counts its samples (a closed segment stays closed)
            const int k0 = r.first_vis;
            if (k0 > 0 && k0 < stored) {
              s.k = k0;
              if (s.mode != kRedo) s.samples += k0;
            }
            ring_fill(cache, s.k, stored);
          }
          if (kRing) {
            ld_pred(b0, cache, 0 < stored);
            ld_pred(b1, cache + 1, 1 < stored);
          }
          have = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    // one cache entry through segment_step: >= 0 when the pass ended
    auto entry_step = [&](float4 rgba) -> int {
      const double ta = s.t0 + (double)s.k * step;
      double tb = ta + step;
      if (tb > s.t1) tb = s.t1;
      int run = 1;
      if (rgba.w <= 0.0f) {
        run = __float_as_int(rgba.x);
        if (run < 1) run = 1;
        if (run > stored - s.k) run = stored - s.k;
      } else {
        rgba.x = fabsf(rgba.x);  // drop the pow flag
      }
      return segment_step(c, s, rgba, ta, tb, run);
    };
    int ended = -1;
    if (kStream == 2) {
      for (int it = 0; it < 8; ++it) {
        if (s.k >= stored) {
          ended = 0;
          break;
        }
        cp_async_wait<kEmitRing - 2>();  // entry k's group has landed
        const int kold = s.k;
        ended = entry_step(lds128(ring_at(s.k)));
        if (ended >= 0) break;
        if (s.k != kold + 1) {  // a transparent run: restart the ring at k
          ring_fill(cache, s.k, stored);
          continue;
        }
        const int kn = s.k + kEmitRing - 2;
        cp_async16(ring_at(kn), cache + (kn < stored ? kn : 0), kn < stored);
        cp_async_commit();
      }
    } else if (!kRing) {
      ended = s.k >= stored ? 0 : entry_step(cache[s.k]);
    } else {
      // (VDI_EMIT_PF: an L1 prefetch of the line kEmitAhead entries ahead
      // whenever that point crosses a line, as in the bisect replays -- the
      // last rays of a launch run alone and wait out every miss)
      constexpr int kEmitAhead = 16;
      for (int it = 0; it < 4; ++it) {
        if (s.k >= stored) {
          ended = 0;
          break;
        }
        // step A: b0 = entry k, b1 = entry k + 1
        int kold = s.k;
        ended = entry_step(b0);
        if (ended >= 0) break;
        if (s.k != kold + 1) {
          ld_pred(b0, cache + s.k, s.k < stored);
          ld_pred(b1, cache + s.k + 1, s.k + 1 < stored);
          if (VDI_EMIT_PF) prefetch_l1(cache + (s.k & ~7) + 8);
          continue;
        }
        ld_pred(b0, cache + s.k + 1, s.k + 1 < stored);
        if (VDI_EMIT_PF && (((kold + kEmitAhead) ^ (s.k + kEmitAhead)) & ~7) != 0 &&
            s.k + kEmitAhead < stored)
          prefetch_l1(cache + s.k + kEmitAhead);
        // step B: b1 = entry k, b0 = entry k + 1 (s.k < stored: the pass goes on)
        kold = s.k;
        ended = entry_step(b1);
        if (ended >= 0) break;
        if (s.k != kold + 1) {
          ld_pred(b0, cache + s.k, s.k < stored);
          ld_pred(b1, cache + s.k + 1, s.k + 1 < stored);
          if (VDI_EMIT_PF) prefetch_l1(cache + (s.k & ~7) + 8);
          continue;
        }
        ld_pred(b1, cache + s.k + 1, s.k + 1 < stored);
        if (VDI_EMIT_PF && (((kold + kEmitAhead) ^ (s.k + kEmitAhead)) & ~7) != 0 &&
            s.k + kEmitAhead < stored)
          prefetch_l1(cache + s.k + kEmitAhead);
      }
    }
    if (ended >= 0) {
      const int n = ended == 0 ? close_pass(c, s) : ended;
      finish_ray(c, s, g, n);
      have = false;
    }
  }
  if (kStream == 2) cp_async_wait<0>();
}

// ---------------------------------------------------------- fused fallback
// Rays left over after kRounds (cache exhausted): sampling and replay in one
// lane with a private cache slot of max_steps entries.
template <int VT>
__global__ void __launch_bounds__(kGenThreads) gen_fused_kernel(const GenConst c) {
  extern __shared__ double4 s_lut[];
  __shared__ double s_u8[256];
  load_lut(c, s_lut, s_u8);
  const int lane = threadIdx.x & 31;
  const double step = c.a.step;
  const int max_steps = c.max_steps;
  float4* const cache =
      c.cache + ((long long)blockIdx.x * blockDim.x + threadIdx.x) * (long long)max_steps;
  WarpPool pool;
  bool have = false, done = false;
  int cached = 0, run_head = -1;
  RayState s;

  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, !have && !done);
    if (need) {
      const long long idx = pool.take(need, lane, &c.ctl->fetch);
      if ((need >> lane) & 1u) {
        const int list = source_list(c, idx);
        if (list == -2) {
          done = true;
        } else if (list >= 0) {
          have = setup_ray(c, s, list);
          cached = 0;
          run_head = -1;
        }
      }
    }
    if (__all_sync(0xffffffffu, done)) break;
    if (!have) continue;

    int ended;
    const double ta = s.t0 + (double)s.k * step;
    double tb = ta + step;
    if (tb > s.t1) tb = s.t1;
    if (tb <= ta) {
      ended = 0;
    } else {
      float4 rgba;
      int run = 1;
      if (s.k < cached) {
        rgba = cache[s.k];
        if (rgba.w <= 0.0f) {
          run = __float_as_int(rgba.x);
          if (run < 1) run = 1;
          if (run > cached - s.k) run = cached - s.k;
        }
      } else {
        rgba = sample_at<VT>(c, s_lut, s_u8, s, ta, tb);
        if (s.k < max_steps) {
          if (rgba.w <= 0.0f) {
            cache[s.k] = make_float4(__int_as_float(1), 0.f, 0.f, 0.f);
            if (run_head < 0) run_head = s.k;
          } else {
            cache[s.k] = rgba;
            if (run_head >= 0) {
              cache[run_head].x = __int_as_float(s.k - run_head);
              run_head = -1;
            }
          }
          cached = s.k + 1;
        }
      }
      ended = segment_step(c, s, rgba, ta, tb, run);
    }
    if (ended >= 0) {
      if (ended == 0) ended = close_pass(c, s);
      if (run_head >= 0) cache[run_head].x = __int_as_float(cached - run_head);
      have = pass_done(c, s, ended);
    }
  }
}

// The round's queue in image order: qbits (bit l = local list l queued) ->
// qidx[0, nrec). Neighbouring queue entries are then neighbouring rays, so
// the fill warps running side by side sample the same record sectors (L2
// reuse) and the replay warps hold rays of similar control flow.
constexpr int kQBlock = 256;  // bit words per compaction block
// bits of word w's queued lists and (VDI_ALLOC_IMAGE) the sum of their rows
__device__ __forceinline__ unsigned long long word_steps(const GenConst& c, int w,
                                                         unsigned bits) {
  unsigned long long t = 0;
  for (unsigned b = bits; b; b &= b - 1) t += (unsigned)c.recs[w * 32 + (__ffs(b) - 1)].nsteps;
  return t;
}

__global__ void queue_count_kernel(const GenConst c, int n_words) {
  const int w = blockIdx.x * kQBlock + threadIdx.x;
  const unsigned bits = w < n_words ? c.qbits[w] : 0u;
  int v = __popc(bits);
  unsigned long long st = VDI_ALLOC_IMAGE ? word_steps(c, w, bits) : 0ull;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, off);
    if (VDI_ALLOC_IMAGE) st += __shfl_xor_sync(0xffffffffu, st, off);
  }
  __shared__ int s_w[kQBlock / 32];
  __shared__ unsigned long long s_st[kQBlock / 32];
  if ((threadIdx.x & 31) == 0) {
    s_w[threadIdx.x >> 5] = v;
    s_st[threadIdx.x >> 5] = st;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    unsigned long long ts = 0;
    for (int k = 0; k < kQBlock / 32; ++k) {
      t += s_w[k];
      ts += s_st[k];
    }
    c.qsum[blockIdx.x] = (unsigned long long)t;
    if (VDI_ALLOC_IMAGE) c.qsum[c.n_qblocks + 1 + blockIdx.x] = ts;
  }
}

// Exclusive scans of the per-block counts (and row-length sums) in place: one
// block of kScanThreads threads, kScanThreads block entries per chunk.
constexpr int kScanThreads = 1024;
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* s_w,
                                                              unsigned long long& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
  }
  if (lane == 31) s_w[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < kScanThreads / 32 ? s_w[lane] : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += u;
    }
    if (lane < kScanThreads / 32) s_w[lane] = w;  // inclusive per-warp totals
  }
  __syncthreads();
  total = s_w[kScanThreads / 32 - 1];
  const unsigned long long before = wid > 0 ? s_w[wid - 1] : 0ull;
  __syncthreads();  // s_w is reused by the next call
  return before + incl - v;
}

__global__ void __launch_bounds__(kScanThreads) queue_scan_kernel(const GenConst c, int nb) {
  __shared__ unsigned long long s_w[kScanThreads / 32];
  unsigned long long run = 0, srun = 0;
  for (int b0 = 0; b0 < nb; b0 += kScanThreads) {
    const int b = b0 + threadIdx.x;
    unsigned long long tot = 0;
    const unsigned long long v = b < nb ? c.qsum[b] : 0ull;
    const unsigned long long ex = block_excl_scan(v, s_w, tot);
    if (b < nb) c.qsum[b] = run + ex;
    run += tot;
    if (VDI_ALLOC_IMAGE) {
      const unsigned long long u = b < nb ? c.qsum[c.n_qblocks + 1 + b] : 0ull;
      const unsigned long long sx = block_excl_scan(u, s_w, tot);
      if (b < nb) c.qsum[c.n_qblocks + 1 + b] = srun + sx;
      srun += tot;
    }
  }
  if (threadIdx.x == 0) {
    c.ctl->nrec = run;  // VDI_ALLOC_IMAGE: lowered to the rays that fit by queue_write
    if (VDI_ALLOC_IMAGE) c.ctl->bump = srun < c.cache_cap ? srun : c.cache_cap;
  }
}

__global__ void queue_write_kernel(const GenConst c, int n_words) {
  __shared__ int s_w[kQBlock / 32];
  __shared__ unsigned long long s_st[kQBlock / 32];
  const int w = blockIdx.x * kQBlock + threadIdx.x;
  const unsigned bits = w < n_words ? c.qbits[w] : 0u;
  const int cnt = __popc(bits);
  const unsigned long long st = VDI_ALLOC_IMAGE ? word_steps(c, w, bits) : 0ull;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
  unsigned long long sincl = st;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
    if (VDI_ALLOC_IMAGE) {
      const unsigned long long su = __shfl_up_sync(0xffffffffu, sincl, off);
      if (lane >= off) sincl += su;
    }
  }
  if (lane == 31) {
    s_w[wid] = incl;
    s_st[wid] = sincl;
  }
  __syncthreads();
  int before = 0;
  unsigned long long sbefore = 0;
  for (int k = 0; k < wid; ++k) {
    before += s_w[k];
    sbefore += s_st[k];
  }
  long long at = (long long)c.qsum[blockIdx.x] + before + incl - cnt;
  if (!VDI_ALLOC_IMAGE) {
    for (unsigned b = bits; b; b &= b - 1) c.qidx[at++] = w * 32 + (__ffs(b) - 1);
    return;
  }
  unsigned long long slot = c.qsum[c.n_qblocks + 1 + blockIdx.x] + sbefore + sincl - st;
  for (unsigned b = bits; b; b &= b - 1) {
    const int list = w * 32 + (__ffs(b) - 1);
    RayRec* r = c.recs + list;
    const unsigned long long n = (unsigned)r->nsteps;
    if (slot + n <= c.cache_cap) {
      r->slot = (long long)slot;
      c.qidx[at] = list;
    } else {  // past the capacity: this and every later ray of the queue
      r->slot = -1;
      c.defer_out[atomicAdd(&c.ctl->ndefer, 1ull)] = list;
      atomicMin(&c.ctl->nrec, (unsigned long long)at);
    }
    ++at;
    slot += n;
  }
}

__global__ void fill_inv_kernel(double* tab, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tab[i] = i > 0 ? 1.0 / (double)i : 0.0;
}

// ------------------------------------------------------------------- host

struct GenPlan {
  void (*sample)(const GenConst);
  void (*fused)(const GenConst);
  void (*fill)(const GenConst);
  void (*bisect)(const GenConst);
  void (*wide)(const GenConst);
  void (*emit)(const GenConst);
  int sms, per_sm_sample, per_sm_fill, per_sm_bisect, per_sm_emit, per_sm_fused, per_sm_wide;
  int bisect_threads, inv_smem;
  int max_steps, inv_n;
  long long n_rays;
  size_t off_ctl, off_inv, off_recs, off_defer0, off_defer1, off_wide, off_qbits, off_qidx,
      off_torder, off_hitbits, off_qsum, off_cache;
  int n_qwords, n_qblocks;
  size_t smem, smem_inv;
};

static int plan_gen(const VdiGenArgs* a, GenPlan& p) {
#define VDI_GEN_KERNELS(VT)               \
  p.sample = gen_sample_kernel<VT>;       \
  p.fill = gen_fill_kernel<VT>;           \
  p.fused = gen_fused_kernel<VT>;
  const bool sub = a->sub_dims[0] > 0;
  switch (a->voxel_type | (sub ? kVoxelSub : 0)) {
    case VDI_VOXEL_U8 | VDI_VOXEL_CELLS:
      VDI_GEN_KERNELS(VDI_VOXEL_U8 | VDI_VOXEL_CELLS)
      break;
    case VDI_VOXEL_U16 | VDI_VOXEL_CELLS:
      VDI_GEN_KERNELS(VDI_VOXEL_U16 | VDI_VOXEL_CELLS)
      break;
    case VDI_VOXEL_F32 | VDI_VOXEL_CELLS:
      VDI_GEN_KERNELS(VDI_VOXEL_F32 | VDI_VOXEL_CELLS)
      break;
    case VDI_VOXEL_U8:
      VDI_GEN_KERNELS(VDI_VOXEL_U8)
      break;
    case VDI_VOXEL_U16:
      VDI_GEN_KERNELS(VDI_VOXEL_U16)
      break;
    case VDI_VOXEL_F32:
      VDI_GEN_KERNELS(VDI_VOXEL_F32)
      break;
    case VDI_VOXEL_U8 | VDI_VOXEL_CELLS | kVoxelSub:
      VDI_GEN_KERNELS(VDI_VOXEL_U8 | VDI_VOXEL_CELLS | kVoxelSub)
      break;
    case VDI_VOXEL_U8 | kVoxelSub:
      VDI_GEN_KERNELS(VDI_VOXEL_U8 | kVoxelSub)
      break;
    case VDI_VOXEL_U16 | kVoxelSub:
      VDI_GEN_KERNELS(VDI_VOXEL_U16 | kVoxelSub)
      break;
    case VDI_VOXEL_F32 | kVoxelSub:
      VDI_GEN_KERNELS(VDI_VOXEL_F32 | kVoxelSub)
      break;
    default:
      return set_error(VDI_EINVAL, "bad voxel_type %d", a->voxel_type);
  }
  // no ray has more samples than the box diagonal allows
  const double ex = a->aabb[3] - a->aabb[0], ey = a->aabb[4] - a->aabb[1],
               ez = a->aabb[5] - a->aabb[2];
  const double diag = sqrt(ex * ex + ey * ey + ez * ez);
  const double ms = ceil(diag / a->step) + 4.0;
  p.max_steps = ms > 1e7 ? 10000000 : (int)ms;
  p.inv_n = p.max_steps + 2;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, dev);
  p.smem = sizeof(double4) * a->lut_n;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_sample, p.sample, kGenThreads, p.smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_fill, p.fill, kGenThreads, p.smem);
  if (p.per_sm_fill < 1) p.per_sm_fill = 1;
  // count-only replays: 2 speculated levels, the A/B-unrolled entry loop, L1
  // line prefetch 16 entries ahead, 5 blocks of 128 per SM (<= 102
  // registers), 4096 shared 1/n entries (the variants measured in round 1 are
  // in profiles/r01_gen_v1_fused_cache.md)
  p.bisect_threads = kGenThreads;
  p.inv_smem = 4096;
#ifndef VDI_BISECT_MINB
// blocks per SM: 4 (128 registers) with the cp.async ring; the register
// stream (kMode 2) was best at 5 (96 registers)
#define VDI_BISECT_MINB 4
#endif
  p.bisect = p.inv_n <= p.inv_smem
                 ? gen_bisect_kernel<2, VDI_BISECT_RING, VDI_BISECT_PF, VDI_BISECT_MINB, 128,
                                     VDI_BISECT_AHEAD, VDI_BISECT_MODE, true>
                 : gen_bisect_kernel<2, VDI_BISECT_RING, VDI_BISECT_PF, VDI_BISECT_MINB, 128,
                                     VDI_BISECT_AHEAD, VDI_BISECT_MODE, false>;
#ifndef VDI_WIDE_LANES
#define VDI_WIDE_LANES 32
#endif
  p.wide = p.inv_n <= p.inv_smem ? gen_bisect_wide_kernel<VDI_WIDE_LANES, true>
                                 : gen_bisect_wide_kernel<VDI_WIDE_LANES, false>;
  // the A/B emit kernel uses no shared memory: give the unified L1 everything
#ifndef VDI_EMIT_STREAM
#define VDI_EMIT_STREAM 2  // 1: A/B register slots + L1 prefetch, 2: cp.async ring
#endif
  p.emit = gen_emit_kernel<VDI_EMIT_STREAM>;
  if (VDI_EMIT_STREAM != 2)
    cudaFuncSetAttribute(p.emit, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  p.smem_inv = sizeof(double) * (size_t)(p.inv_smem < p.inv_n ? p.inv_smem : p.inv_n);
  if (p.smem_inv > 48 * 1024)
    cudaFuncSetAttribute(p.bisect, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_inv);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_bisect, p.bisect, p.bisect_threads,
                                                p.smem_inv);
  if (p.smem_inv > 48 * 1024)
    cudaFuncSetAttribute(p.wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_inv);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_wide, p.wide, kGenThreads, p.smem_inv);
  if (p.per_sm_wide < 1) p.per_sm_wide = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_fused, p.fused, kGenThreads, p.smem);
  if (p.per_sm_sample < 1) p.per_sm_sample = 1;
  if (p.per_sm_bisect < 1) p.per_sm_bisect = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p.per_sm_emit, p.emit, kGenThreads, 0);
  if (p.per_sm_emit < 1) p.per_sm_emit = 1;
  if (p.per_sm_fused < 1) p.per_sm_fused = 1;
  const int bands = a->band_rows > 0 ? a->band_rows : 16;
  p.n_rays = (long long)a->width *
             launch_rows(a->height, bands, a->band_stride > 0 ? a->band_stride : 1,
                         a->band_offset, a->row_count);
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  p.off_ctl = 0;
  p.off_inv = up(sizeof(RoundCtl) * (kRounds + 1));
  p.off_recs = up(p.off_inv + sizeof(double) * p.inv_n);
  p.off_defer0 = up(p.off_recs + sizeof(RayRec) * (size_t)p.n_rays);
  p.off_defer1 = up(p.off_defer0 + sizeof(int) * (size_t)p.n_rays);
  p.off_wide = up(p.off_defer1 + sizeof(int) * (size_t)p.n_rays);
  p.n_qwords = (int)((p.n_rays + 31) / 32);
  p.n_qblocks = (p.n_qwords + kQBlock - 1) / kQBlock;
  p.off_qbits = up(p.off_wide + sizeof(int) * (size_t)p.n_rays);
  p.off_qidx = up(p.off_qbits + sizeof(unsigned) * (size_t)p.n_qwords);
  p.off_torder = up(p.off_qidx + sizeof(int) * (size_t)p.n_rays);
  {
    // one word per 8x4 tile of the launch's rows
    const long long tiles = (long long)((a->width + kTileW - 1) / kTileW) *
                            ((p.n_rays / (a->width > 0 ? a->width : 1) + kTileH - 1) / kTileH);
    p.off_hitbits = up(p.off_torder + sizeof(int) * (size_t)p.n_rays);
    p.off_qsum = up(p.off_hitbits + sizeof(unsigned) * (size_t)(tiles + 1));
  }
  p.off_cache = up(p.off_qsum + sizeof(unsigned long long) * (size_t)(2 * (p.n_qblocks + 1)));
  return VDI_OK;
}

// Minimum: room for one fused-fallback block of per-lane slots. Recommended:
// enough cache that one round holds every overflowing ray of typical scenes
// (~30% of rays x the longest chord), capped at half the free device memory.
size_t gen_workspace_bytes(const VdiGenArgs* a, int recommended) {
  GenPlan p;
  if (plan_gen(a, p) != VDI_OK) return 0;
  const size_t min_cache = sizeof(float4) * (size_t)kGenThreads * (size_t)p.max_steps;
  size_t rec = (size_t)(0.30 * (double)p.n_rays * (double)p.max_steps) * sizeof(float4);
  const size_t fused_all = sizeof(float4) * (size_t)p.sms * p.per_sm_fused * kGenThreads *
                           (size_t)p.max_steps;
  if (rec < fused_all) rec = fused_all;
  // cache cap: half of the device memory free now (never more than is free;
  // the caller keeps the other half). Rays that do not fit are deferred to
  // another round and re-sampled, which is what makes a small cap expensive
  // (C5: 24 GiB -> 989 ms, 64 GiB -> 426 ms, 120 GiB -> 372 ms of
  // generation), but the launch is correct at any size >= the minimum.
  if (!recommended) return p.off_cache + min_cache;  // (no device query on the launch path)
  size_t cap = min_cache;
  {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b / 2 > cap) cap = free_b / 2;
  }
  if (rec > cap) rec = cap;
  if (rec < min_cache) rec = min_cache;
  return p.off_cache + rec;
}

// ------------------------------------------------------- single rays (G14)
// generate_list / find_gamma (generate.py:371-407) for a batch of arbitrary
// rays: one thread per ray, the reference's sequential loop (each pass
// re-samples, as R does), on the same device helpers as the phased kernels.
// mode 0: the full bisection (_find_gamma_list); 1: one counting pass at
// gammas_in[i]; 2: one capped pass at gammas_in[i] (_gen_list_pass).
template <int VT>
__global__ void __launch_bounds__(kGenThreads) gen_rays_kernel(const GenConst c,
                                                              const double* __restrict__ rays,
                                                              const double* __restrict__ gin,
                                                              long long n, int mode) {
  extern __shared__ double4 s_lut[];
  __shared__ double s_u8[256];
  load_lut(c, s_lut, s_u8);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double step = c.a.step;
  RayState s;
  s.list = (int)i;
  s.seg = c.a.segs + i * (long long)list_stride(c.a.n_sg);
  s.o[0] = rays[6 * i];
  s.o[1] = rays[6 * i + 1];
  s.o[2] = rays[6 * i + 2];
  s.d[0] = rays[6 * i + 3];
  s.d[1] = rays[6 * i + 4];
  s.d[2] = rays[6 * i + 5];
  init_bisection(c, s);
  // generate.py:414-425 _clip_for_generation
  double ta, tb, fa, fb;
  bool hit = clip_aabb(s.o, s.d, c.a.aabb, ta, tb) && clip_frustum(c.a.pv, s.o, s.d, fa, fb);
  if (hit) {
    s.t0 = dmax(dmax(ta, fa), 0.0);
    s.t1 = dmin(tb, fb);
    hit = s.t1 > s.t0;
  }
  if (!hit) {
    // find_gamma returns (gamma_init, 0, zeros, 0); generate_list (0, zeros, False)
    finish_ray(c, s, mode == 0 ? c.a.gamma_init : gin[i], 0);
    return;
  }
  s.nsteps = (int)ceil((s.t1 - s.t0) / step);
  if (mode == 0) {
    start_pass(s, s.bis_gamma, kCount);
  } else {
    start_pass(s, gin[i], mode == 1 ? kCount : kCapped);
  }
  while (true) {
    const double sa = s.t0 + (double)s.k * step;
    double sb = sa + step;
    if (sb > s.t1) sb = s.t1;
    int ended;
    if (sb <= sa) {
      ended = 0;
    } else {
      const float4 rgba = sample_at<VT>(c, s_lut, s_u8, s, sa, sb);
      ended = segment_step(c, s, rgba, sa, sb, 1);
    }
    if (ended < 0) continue;
    if (ended == 0) ended = close_pass(c, s);
    if (mode != 0) {  // one pass: count (n_sg + 1 = exceeded) and the segments it wrote
      s.passes = 1;
      c.a.counts[i] = ended;
      if (c.a.samples) c.a.samples[i] = s.samples;
      return;
    }
    if (!pass_done(c, s, ended)) return;
  }
}

int gen_rays(const VdiGenArgs* a, const double* rays, const double* gammas_in, long long n,
             int mode, cudaStream_t stream) {
  if (n <= 0) return VDI_OK;
  if (mode != 0 && !gammas_in) return set_error(VDI_EINVAL, "mode 1/2 needs gammas_in");
  GenConst c;
  memset(&c, 0, sizeof(c));
  c.a = *a;
  for (int i = 0; i < 3; ++i) {
    const double ext = a->aabb[3 + i] - a->aabb[i];
    int e;
    c.ext_pow2[i] = (frexp(ext, &e) == 0.5);
    c.inv_ext[i] = 1.0 / ext;
  }
  {
    int e;
    c.lref_pow2 = (frexp(a->lref, &e) == 0.5);
    c.inv_lref = 1.0 / a->lref;
  }
  c.ess = 0;  // plain per-sample sampling (no brick maxima needed)
  c.inv_tab = nullptr;
  c.inv_n = 0;  // 1/n by IEEE division (no table)
  void (*k)(const GenConst, const double*, const double*, long long, int) = nullptr;
  switch (a->voxel_type) {
    case VDI_VOXEL_U8: k = gen_rays_kernel<VDI_VOXEL_U8>; break;
    case VDI_VOXEL_U16: k = gen_rays_kernel<VDI_VOXEL_U16>; break;
    case VDI_VOXEL_F32: k = gen_rays_kernel<VDI_VOXEL_F32>; break;
    default: return set_error(VDI_EINVAL, "bad voxel_type %d", a->voxel_type);
  }
  const size_t smem = sizeof(double4) * a->lut_n;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)smem);
    if (e != cudaSuccess) return set_error(VDI_ELAUNCH, "rays smem: %s", cudaGetErrorString(e));
  }
  k<<<(unsigned)((n + kGenThreads - 1) / kGenThreads), kGenThreads, smem, stream>>>(c, rays,
                                                                                   gammas_in, n,
                                                                                   mode);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "rays launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

int gen_launch(const VdiGenArgs* a, cudaStream_t stream) {
  GenConst c;
  c.a = *a;
  for (int i = 0; i < 3; ++i) {
    const double ext = a->aabb[3 + i] - a->aabb[i];
    int e;
    const double m = frexp(ext, &e);
    c.ext_pow2[i] = (m == 0.5);
    c.inv_ext[i] = 1.0 / ext;
  }
  {
    int e;
    c.lref_pow2 = (frexp(a->lref, &e) == 0.5);
    c.inv_lref = 1.0 / a->lref;
  }
  const int band_rows = a->band_rows > 0 ? a->band_rows : 16;
  c.a.band_rows = band_rows;
  if (c.a.band_stride <= 0) c.a.band_stride = 1;
  c.local_h =
      launch_rows(a->height, band_rows, c.a.band_stride, c.a.band_offset, c.a.row_count);
  c.tiles_x = (a->width + kTileW - 1) / kTileW;
  const long long tiles_y = (c.local_h + kTileH - 1) / kTileH;
  c.n_slots = (long long)c.tiles_x * tiles_y * 32;
  c.ess = a->brick_max != nullptr && a->ess_max >= 0.0 && a->brick_log2 >= 1;
  c.ess_u8 = -1;  // the largest v with (double)((float)v / 255) <= ess_max
  for (int v = 0; v < 256; ++v)
    if ((double)((float)v / 255.0f) <= a->ess_max) c.ess_u8 = v;
  const bool sub = a->sub_dims[0] > 0;
  const int rx = sub ? a->sub_dims[0] : a->nx, ry = sub ? a->sub_dims[1] : a->ny;
  if (c.ess) {
    const int B = 1 << a->brick_log2;
    c.bnx = (rx + B - 1) / B;
    c.bny = (ry + B - 1) / B;
  } else {
    c.bnx = c.bny = 0;
  }
  c.sub_ox = a->sub_origin[0];
  c.sub_oy = a->sub_origin[1];
  c.sub_oz = a->sub_origin[2];
  c.sub_nx = sub ? a->sub_dims[0] : a->nx;
  c.sub_ny = sub ? a->sub_dims[1] : a->ny;
  c.sub_nz = sub ? a->sub_dims[2] : a->nz;
  c.sub_sx = c.sub_nx;
  c.sub_sy = c.sub_ny;
  c.sub_voff = sub ? ((long long)c.sub_oz * c.sub_sy + c.sub_oy) * c.sub_sx + c.sub_ox : 0;
  c.sub_boff = 0;
  c.sub_oob = a->sub_oob;
  // replays that start below level 6 speculate the down-chain: on the queued
  // rays levels 0-2 go down > 98 % of the time at C3 and levels 0-5 always at
  // C4 / C5 (tools/bisect_paths.py). Measured gen: C3 40.2 -> 37.8 ms, C4 82.4
  // -> 73.9, C5 391 -> 359 (chain_levels = 0 restores the tree everywhere)
  c.chain_levels = 6;
  // narrow replays per ray before the hand-off to the wide phase. The wide
  // phase costs ~4x the instructions per bisection level, so it pays only
  // when a launch has too few rays to hide its longest rays' serial replays
  // (a band-sharded rank): C3 as 1 rank 31.5 ms without / 36.5 with; as one
  // of 8 ranks 12.0 / 8.9 ms (profiles/r02_wide_ab.log). With the cp.async
  // replays, one of 8 C3 ranks: after 2 / 3 / 4 / 6 / never: 7.25 / 6.93 /
  // 6.58 / 7.14 / 8.0 ms.
#ifndef VDI_WIDE_AFTER
#define VDI_WIDE_AFTER 4
#endif
  // learned chain directions beyond those levels (measured: C3 gen 33.6 ->
  // 32.8 ms; C4 / C5 within noise). learn = 0 disables.
  c.learn = 1;
  if (sub) {
    const int lb = a->brick_log2 >= 1 ? a->brick_log2 : 3;
    if (c.ess && ((c.sub_ox | c.sub_oy | c.sub_oz) & ((1 << lb) - 1)))
      return set_error(VDI_EINVAL, "sub_origin must be a multiple of the brick edge");
    c.sub_boff = ((long long)(c.sub_oz >> lb) * c.bny + (c.sub_oy >> lb)) * c.bnx +
                 (c.sub_ox >> lb);
  }
  if (c.local_h <= 0) return VDI_OK;
  GenPlan p;
  int rc = plan_gen(&c.a, p);
  c.wide_after = p.n_rays < kWideRays ? VDI_WIDE_AFTER : (1 << 30);
#ifndef VDI_WIDE_TAIL
#define VDI_WIDE_TAIL 0
#endif
  c.wide_tail = p.n_rays < kWideRays ? VDI_WIDE_TAIL : 0;
  if (rc != VDI_OK) return rc;
  const size_t need = gen_workspace_bytes(&c.a, 0);
  if (a->workspace_bytes < need)
    return set_error(VDI_EINVAL, "workspace too small: %zu < %zu bytes", a->workspace_bytes,
                     need);
  char* ws = reinterpret_cast<char*>(a->workspace);
  RoundCtl* ctl = reinterpret_cast<RoundCtl*>(ws + p.off_ctl);
  c.inv_tab = reinterpret_cast<const double*>(ws + p.off_inv);
  c.inv_n = p.inv_n;
  c.inv_smem = (int)(p.smem_inv / sizeof(double));
  c.max_steps = p.max_steps;
  c.recs = reinterpret_cast<RayRec*>(ws + p.off_recs);
  c.wide = reinterpret_cast<int*>(ws + p.off_wide);
  c.qbits = reinterpret_cast<unsigned*>(ws + p.off_qbits);
  c.qidx = reinterpret_cast<int*>(ws + p.off_qidx);
  c.torder = reinterpret_cast<int*>(ws + p.off_torder);
  c.hitbits = reinterpret_cast<unsigned*>(ws + p.off_hitbits);
  c.qsum = reinterpret_cast<unsigned long long*>(ws + p.off_qsum);
  c.n_qblocks = p.n_qblocks;
  c.cache = reinterpret_cast<float4*>(ws + p.off_cache);
  c.cache_cap = (a->workspace_bytes - p.off_cache) / sizeof(float4);
  int* defer[2] = {reinterpret_cast<int*>(ws + p.off_defer0),
                   reinterpret_cast<int*>(ws + p.off_defer1)};

  cudaError_t err = cudaMemsetAsync(ctl, 0, sizeof(RoundCtl) * (kRounds + 1), stream);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen memset: %s", cudaGetErrorString(err));
  fill_inv_kernel<<<(p.inv_n + 255) / 256, 256, 0, stream>>>(
      reinterpret_cast<double*>(ws + p.off_inv), p.inv_n);

  const long long chunks = c.n_slots / 32;
  auto grid_for = [&](int per_sm, long long items) {
    long long b = (long long)p.sms * per_sm;
    const long long need_b = (items + (kGenThreads / 32) - 1) / (kGenThreads / 32);
    if (items >= 0 && b > need_b) b = need_b;
    return (unsigned)(b < 1 ? 1 : b);
  };
  for (int r = 0; r < kRounds; ++r) {
    c.round = r;
    c.ctl = ctl + r;
    c.prev = r > 0 ? ctl + r - 1 : ctl;
    c.defer_in = defer[(r + 1) & 1];
    c.defer_out = defer[r & 1];
    cudaMemsetAsync(c.qbits, 0, sizeof(unsigned) * (size_t)p.n_qwords, stream);
    if (VDI_SETUP_PASS && r == 0)
      gen_setup_kernel<<<(unsigned)((c.n_slots + kGenThreads - 1) / kGenThreads), kGenThreads, 0,
                         stream>>>(c);
    p.sample<<<grid_for(p.per_sm_sample, r == 0 ? chunks : -1), kGenThreads, p.smem, stream>>>(c);
    queue_count_kernel<<<p.n_qblocks, kQBlock, 0, stream>>>(c, p.n_qwords);
    queue_scan_kernel<<<1, kScanThreads, 0, stream>>>(c, p.n_qblocks);
    queue_write_kernel<<<p.n_qblocks, kQBlock, 0, stream>>>(c, p.n_qwords);
    p.fill<<<grid_for(p.per_sm_fill, -1), kGenThreads, p.smem, stream>>>(c);
    p.bisect<<<grid_for(p.per_sm_bisect, -1), p.bisect_threads, p.smem_inv, stream>>>(c);
    p.wide<<<grid_for(p.per_sm_wide, -1), kGenThreads, p.smem_inv, stream>>>(c);
    p.emit<<<grid_for(p.per_sm_emit, -1), kGenThreads, 0, stream>>>(c);
  }
  // leftovers: the fused kernel over the last round's deferred rays
  c.round = kRounds;
  c.ctl = ctl + kRounds;
  c.prev = ctl + kRounds - 1;
  c.defer_in = defer[(kRounds - 1) & 1];
  c.defer_out = defer[kRounds & 1];
  {
    long long blocks = (long long)(c.cache_cap / (unsigned long long)p.max_steps) / kGenThreads;
    const long long full = (long long)p.sms * p.per_sm_fused;
    if (blocks > full) blocks = full;
    if (blocks < 1) return set_error(VDI_EINVAL, "workspace cannot hold one fallback block");
    p.fused<<<(unsigned)blocks, kGenThreads, p.smem, stream>>>(c);
  }
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "gen launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi

// ----------------------------------------------------------- self checks
// Device-side checks of the exact arithmetic shortcuts the kernels rely on
// (vdi_selftest_arith). counters: [0] Markstein quotient != IEEE quotient,
// [1] __drcp_rn(n) != 1.0 / n, [2] (d2 >= thr(g)) != (sqrt(d2) >= g),
// [3] shared-reciprocal xform != per-component division.
namespace vdi {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

__device__ __forceinline__ double rand_double(unsigned long long& s, int emin, int emax) {
  s = mix64(s + 0x9e3779b97f4a7c15ull);
  const unsigned long long mant = s >> 12;
  s = mix64(s + 0x9e3779b97f4a7c15ull);
  const int e = emin + (int)(s % (unsigned long long)(emax - emin + 1));
  const unsigned long long bits = ((unsigned long long)(1023 + e) << 52) | mant;
  double v = __longlong_as_double((long long)bits);
  if ((s >> 40) & 1) v = -v;
  return v;
}

__global__ void selftest_kernel(long long n, unsigned long long seed, unsigned long long* bad) {
  unsigned long long local[4] = {0, 0, 0, 0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long s = mix64(seed ^ (unsigned long long)i);
    const double x = rand_double(s, -40, 40), d = rand_double(s, -40, 40);
    if (div_by(x, d, 1.0 / d) != x / d) local[0] += 1;
    const double nn = (double)(1 + (i % (1 << 22)));
    if (__drcp_rn(nn) != 1.0 / nn) local[1] += 1;
    const double g = fabs(rand_double(s, -20, 1));
    const double t = split_threshold(g);
    const double d2a = fabs(rand_double(s, -40, 2));
    const double d2b = t * (1.0 + (double)((long long)(s % 9) - 4) * 1e-16);  // near thr
    if ((d2a >= t) != (sqrt(d2a) >= g)) local[2] += 1;
    if ((d2b >= t) != (sqrt(d2b) >= g)) local[2] += 1;
    double m[16];
    for (int j = 0; j < 16; ++j) m[j] = rand_double(s, -3, 3);
    const double px = rand_double(s, -2, 3), py = rand_double(s, -2, 3), pz = rand_double(s, -2, 3);
    double ox, oy, oz;
    xform(m, px, py, pz, ox, oy, oz);
    const double hx = m[0] * px + m[1] * py + m[2] * pz + m[3];
    const double hy = m[4] * px + m[5] * py + m[6] * pz + m[7];
    const double hz = m[8] * px + m[9] * py + m[10] * pz + m[11];
    const double hw = m[12] * px + m[13] * py + m[14] * pz + m[15];
    if (ox != hx / hw || oy != hy / hw || oz != hz / hw) local[3] += 1;
  }
  for (int j = 0; j < 4; ++j)
    if (local[j]) atomicAdd(bad + j, local[j]);
}

int selftest_arith(long long n, unsigned long long seed, unsigned long long* bad,
                   cudaStream_t stream) {
  cudaError_t err = cudaMemsetAsync(bad, 0, 4 * sizeof(unsigned long long), stream);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "selftest memset: %s", cudaGetErrorString(err));
  selftest_kernel<<<148 * 8, 256, 0, stream>>>(n, seed, bad);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "selftest launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
