// vdi_codec.cu -- the VDI wire path on sm_100a: VDI1 packing (vdi.py:141-159
// encode_vdi) and an LZ4 block compressor (lz4.py block format, decodable by
// lz4.py:117-168) that run on the device-resident VDI, so the server's
// generate_fn -> compress_fn path (proto.py:283-287, 328-334) never stages
// the (up to GiB-sized) raw VDI on the host.
//
// VDI1 packing. The byte stream is header (160 B, built on the host from the
// camera and AABB) | counts as u16 | valid supersegments as AoS f32 in list
// order | grid as u32. The packed-segment offsets are an exclusive scan of
// the counts: a per-block scan (1024 lists) + a one-block scan of the block
// totals; the scatter then fills each block's contiguous output range, one
// thread per supersegment (24 contiguous bytes), locating the source list by
// binary search in the block's shared prefix array.
//
// LZ4. The reference's compressor is one serial greedy parse with a 64 Ki
// hash table. Here the input is cut into 32 KiB chunks, one warp each; a warp
// runs the same greedy single-probe parse over its chunk (4 Ki-entry table
// in shared memory) 32 positions at a time: lane j hashes position i + j,
// takes its candidate from the nearest lower lane with the same hash
// (__match_any_sync) or else the table, and the lowest lane with a verified
// 4-byte match wins -- exactly the serial parse's decision, because every
// position before the winner would have been inserted and missed. Match
// extension compares 32 bytes per step. The chunks' trailing literals are
// carried into the next chunk's first sequence (a literal-only sequence may
// only end the block), so a one-block scan composes the carries and sizes,
// and a final pass writes each chunk's sequences at its offset. The output is
// a valid LZ4 block (matches start >= 12 bytes before the end and end >= 5
// bytes before it); its bytes differ from the reference's serial parse, but
// it decodes to the same input -- the property the transport relies on
// (test_acceptance.py A6: decompress(compress(raw)) == raw).
#include <cstdint>
#include <cstdlib>

#include "vdi_common.cuh"
#include "vdi_internal.h"

namespace vdi {

// p[0] = min(*src, v0) (or v0 when src is null), p[1] = v1 unless v1 == ~0.
__global__ void set_u64_kernel(unsigned long long* p, const unsigned long long* src,
                               unsigned long long v0, unsigned long long v1) {
  p[0] = src && *src < v0 ? *src : v0;
  if (v1 != ~0ull) p[1] = v1;
}

// ------------------------------------------------------------ VDI1 packing

constexpr int kEncBlock = 1024;
constexpr int kVdi1Header = 160;  // vdi.py:136-139: 20 + 80 + 48 + 12

static size_t enc_blocks(long long n_lists) { return (size_t)((n_lists + kEncBlock - 1) / kEncBlock); }

// Block b: counts -> u16 stream, and the block's count total.
__global__ void enc_counts_kernel(const VdiEncodeArgs a, unsigned long long* block_sums) {
  __shared__ unsigned long long s_sum[kEncBlock / 32];
  const long long n = (long long)a.width * a.height;
  const long long l = (long long)blockIdx.x * kEncBlock + threadIdx.x;
  int cnt = 0;
  if (l < n) {
    const int r = (int)(l / a.width), x = (int)(l - (long long)r * a.width);
    const long long li =
        (long long)vdi_storage_row(r, a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank) *
            a.width + x;
    cnt = a.counts[li];
    const unsigned short v = (unsigned short)cnt;  // vdi.py:148 astype("<u2")
    a.out[kVdi1Header + 2 * l] = (uint8_t)(v & 0xff);
    a.out[kVdi1Header + 2 * l + 1] = (uint8_t)(v >> 8);
  }
  unsigned long long s = (unsigned long long)cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long t = s_sum[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = t;
  }
}

// One block: exclusive scan of the block totals (in place), the total, the
// header bytes and out_len.
__global__ void enc_scan_kernel(const VdiEncodeArgs a, unsigned long long* block_sums, int nb,
                                unsigned long long* total_out) {
  __shared__ unsigned long long s_part[1024];
  const int t = threadIdx.x;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = b0 + per < nb ? b0 + per : nb;
  unsigned long long sum = 0;
  for (int b = b0; b < b1; ++b) sum += block_sums[b];
  s_part[t] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele
    const unsigned long long v = t >= off ? s_part[t - off] : 0ull;
    __syncthreads();
    s_part[t] += v;
    __syncthreads();
  }
  unsigned long long run = t > 0 ? s_part[t - 1] : 0ull;
  for (int b = b0; b < b1; ++b) {
    const unsigned long long v = block_sums[b];
    block_sums[b] = run;
    run += v;
  }
  if (t == 1023) {
    const unsigned long long total = s_part[1023];
    *total_out = total;
    const unsigned long long n = (unsigned long long)a.width * a.height;
    if (a.out_len)
      *a.out_len = kVdi1Header + 2ull * n + 24ull * total +
                   4ull * (unsigned long long)a.gx * a.gy * a.gz;
  }
  for (int i = t; i < kVdi1Header; i += blockDim.x) a.out[i] = a.header[i];
}

__device__ __forceinline__ void store_word(uint8_t* p, uint32_t w, bool aligned) {
  if (aligned) {
    *reinterpret_cast<uint32_t*>(p) = w;
  } else {
    p[0] = (uint8_t)w;
    p[1] = (uint8_t)(w >> 8);
    p[2] = (uint8_t)(w >> 16);
    p[3] = (uint8_t)(w >> 24);
  }
}

// Block b: its lists' valid supersegments, [front, back, r, g, b, a] each,
// into the contiguous range starting at its scanned offset.
__global__ void enc_segs_kernel(const VdiEncodeArgs a, const unsigned long long* block_off) {
  __shared__ int s_pre[kEncBlock + 1];
  __shared__ long long s_src[kEncBlock];
  __shared__ int s_tmp[kEncBlock / 32];
  const long long n = (long long)a.width * a.height;
  const long long l = (long long)blockIdx.x * kEncBlock + threadIdx.x;
  int cnt = 0;
  long long li = 0;
  if (l < n) {
    const int r = (int)(l / a.width), x = (int)(l - (long long)r * a.width);
    li = (long long)vdi_storage_row(r, a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank) *
             a.width + x;
    cnt = a.counts[li];
  }
  s_src[threadIdx.x] = li;
  // block exclusive scan of cnt
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) s_tmp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int w = s_tmp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    s_tmp[lane] = w;
  }
  __syncthreads();
  const int incl = v + (wid > 0 ? s_tmp[wid - 1] : 0);
  s_pre[threadIdx.x + 1] = incl;
  if (threadIdx.x == 0) s_pre[0] = 0;
  __syncthreads();
  const int bt = s_pre[kEncBlock];
  const unsigned long long base_byte =
      kVdi1Header + 2ull * (unsigned long long)n + 24ull * block_off[blockIdx.x];
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.out) + base_byte) & 3u) == 0;
  uint8_t* dst = a.out + base_byte;
  const int stride = list_stride(a.n_sg);
  // one thread per supersegment: locate its list once, write its 6 words
  for (int sidx = threadIdx.x; sidx < bt; sidx += blockDim.x) {
    int lo = 0, hi = kEncBlock - 1;  // list j with s_pre[j] <= sidx < s_pre[j + 1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= sidx) lo = mid;
      else hi = mid - 1;
    }
    const int j = sidx - s_pre[lo];
    const float* ls = a.segs + s_src[lo] * (long long)stride;
    const float4 c4 = reinterpret_cast<const float4*>(ls)[j];
    uint8_t* o = dst + 24ll * sidx;
    store_word(o, __float_as_uint(ls[front_off(a.n_sg) + j]), aligned);
    store_word(o + 4, __float_as_uint(ls[back_off(a.n_sg) + j]), aligned);
    store_word(o + 8, __float_as_uint(c4.x), aligned);
    store_word(o + 12, __float_as_uint(c4.y), aligned);
    store_word(o + 16, __float_as_uint(c4.z), aligned);
    store_word(o + 20, __float_as_uint(c4.w), aligned);
  }
}

__global__ void enc_grid_kernel(const VdiEncodeArgs a, const unsigned long long* total) {
  const unsigned long long n = (unsigned long long)a.width * a.height;
  const unsigned long long base = kVdi1Header + 2ull * n + 24ull * (*total);
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.out) + base) & 3u) == 0;
  const long long g = (long long)a.gx * a.gy * a.gz;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < g;
       k += (long long)gridDim.x * blockDim.x)
    store_word(a.out + base + 4 * k, a.grid[k], aligned);
}

size_t encode_workspace_bytes(int width, int height) {
  return 256 + sizeof(unsigned long long) * enc_blocks((long long)width * height);
}

int encode_vdi1(const VdiEncodeArgs* args, cudaStream_t stream) {
  const VdiEncodeArgs& a = *args;
  const long long n = (long long)a.width * a.height;
  const int nb = (int)enc_blocks(n);
  if (a.workspace_bytes < encode_workspace_bytes(a.width, a.height))
    return set_error(VDI_EINVAL, "encode workspace too small");
  unsigned long long* total = reinterpret_cast<unsigned long long*>(a.workspace);
  unsigned long long* bsum = total + 32;
  VdiEncodeArgs c = a;
  if (c.vdi_band_rows <= 0) c.vdi_band_rows = 16;
  if (c.vdi_band_world <= 0) c.vdi_band_world = 1;
  enc_counts_kernel<<<nb, kEncBlock, 0, stream>>>(c, bsum);
  enc_scan_kernel<<<1, 1024, 0, stream>>>(c, bsum, nb, total);
  enc_segs_kernel<<<nb, kEncBlock, 0, stream>>>(c, bsum);
  const long long g = (long long)a.gx * a.gy * a.gz;
  long long gb = (g + 255) / 256;
  if (gb > 4096) gb = 4096;
  enc_grid_kernel<<<(unsigned)(gb < 1 ? 1 : gb), 256, 0, stream>>>(c, total);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "encode launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// VDI1 lists -> list-SoA (the receiving side of the multi-GPU exchange, and
// decode_vdi's counts / segs on the device): counts u16 at byte 160, the
// valid supersegments AoS after them. One thread per list copies its
// supersegments into its list-SoA slot and zero-fills the tail (the
// reference's (H, W, n_sg, 6) array is zero past each count).
__global__ void dec_counts_kernel(const uint8_t* __restrict__ src, long long n,
                                  int32_t* __restrict__ counts, unsigned long long* block_sums) {
  __shared__ unsigned long long s_sum[kEncBlock / 32];
  const long long l = (long long)blockIdx.x * kEncBlock + threadIdx.x;
  int cnt = 0;
  if (l < n) {
    cnt = (int)src[kVdi1Header + 2 * l] | ((int)src[kVdi1Header + 2 * l + 1] << 8);
    counts[l] = cnt;
  }
  unsigned long long sm = (unsigned long long)cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = sm;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long t = s_sum[threadIdx.x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = t;
  }
}

__global__ void scan_blocks_kernel(unsigned long long* block_sums, int nb) {
  __shared__ unsigned long long s_part[1024];
  const int t = threadIdx.x;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = b0 + per < nb ? b0 + per : nb;
  unsigned long long sum = 0;
  for (int b = b0; b < b1; ++b) sum += block_sums[b];
  s_part[t] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const unsigned long long v = t >= off ? s_part[t - off] : 0ull;
    __syncthreads();
    s_part[t] += v;
    __syncthreads();
  }
  unsigned long long run = t > 0 ? s_part[t - 1] : 0ull;
  for (int b = b0; b < b1; ++b) {
    const unsigned long long v = block_sums[b];
    block_sums[b] = run;
    run += v;
  }
}

__global__ void dec_segs_kernel(const uint8_t* __restrict__ src, long long n, int n_sg,
                                const int32_t* __restrict__ counts,
                                const unsigned long long* __restrict__ block_off,
                                float* __restrict__ segs) {
  __shared__ int s_tmp[kEncBlock / 32];
  const long long l = (long long)blockIdx.x * kEncBlock + threadIdx.x;
  const int cnt = l < n ? counts[l] : 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) s_tmp[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int w = s_tmp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    s_tmp[lane] = w;
  }
  __syncthreads();
  // one warp per list of the block: the list's list-SoA slot (stride
  // floats, zero tail) written coalesced, its packed records read coalesced
  __shared__ long long s_excl[kEncBlock];
  __shared__ int s_cnt[kEncBlock];
  s_excl[threadIdx.x] = (long long)block_off[blockIdx.x] + (v - cnt) + (wid > 0 ? s_tmp[wid - 1] : 0);
  s_cnt[threadIdx.x] = cnt;
  __syncthreads();
  const int stride = list_stride(n_sg);
  const long long l0 = (long long)blockIdx.x * kEncBlock;
  // the records are 4-byte aligned when the stream is and 2 n is
  const bool al4 = ((reinterpret_cast<uintptr_t>(src) + kVdi1Header + 2 * n) & 3) == 0;
  for (int j = wid; j < kEncBlock && l0 + j < n; j += kEncBlock / 32) {
    const int c = s_cnt[j];
    const uint8_t* rec = src + kVdi1Header + 2 * n + 24 * s_excl[j];
    // four floats per lane and store: the rgba float4 of one record, or four
    // consecutive fronts / backs (pad zeros)
    float4* ls4 = reinterpret_cast<float4*>(segs + (l0 + j) * (long long)stride);
    auto field = [&](int k, int f) -> float {
      if (k >= c) return 0.f;
      const uint8_t* r = rec + 24 * k + 4 * f;
      return al4 ? __ldg(reinterpret_cast<const float*>(r))
                 : __uint_as_float((unsigned)r[0] | ((unsigned)r[1] << 8) |
                                   ((unsigned)r[2] << 16) | ((unsigned)r[3] << 24));
    };
    for (int q4 = lane; q4 < (stride >> 2); q4 += 32) {
      float4 v;
      if (q4 < n_sg) {
        v = make_float4(field(q4, 2), field(q4, 3), field(q4, 4), field(q4, 5));
      } else {
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int q = 4 * q4 + e;
          // fronts [4 n_sg, 5 n_sg), backs [5 n_sg, 6 n_sg), then the pad
          t[e] = q < 5 * n_sg ? field(q - 4 * n_sg, 0) : field(q - 5 * n_sg, 1);
        }
        v = make_float4(t[0], t[1], t[2], t[3]);
      }
      ls4[q4] = v;
    }
  }
}

int decode_vdi1_lists(const uint8_t* src, int width, int rows, int n_sg, int32_t* counts,
                      float* segs, void* workspace, size_t ws_bytes, cudaStream_t stream) {
  const long long n = (long long)width * rows;
  if (n <= 0) return VDI_OK;
  if (ws_bytes < encode_workspace_bytes(width, rows))
    return set_error(VDI_EINVAL, "decode workspace too small");
  const int nb = (int)enc_blocks(n);
  unsigned long long* bsum = reinterpret_cast<unsigned long long*>(workspace) + 32;
  dec_counts_kernel<<<nb, kEncBlock, 0, stream>>>(src, n, counts, bsum);
  scan_blocks_kernel<<<1, 1024, 0, stream>>>(bsum, nb);
  dec_segs_kernel<<<nb, kEncBlock, 0, stream>>>(src, n, n_sg, counts, bsum, segs);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "decode launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// -------------------------------------------------------------------- LZ4

constexpr int kLz4Chunk = 32768;
constexpr int kLz4HashLog = 12;  // default table: 4 Ki entries per warp
constexpr int kLz4MaxSeq = kLz4Chunk / 4 + 1;
constexpr int kLz4Warps = 4;
constexpr int kLz4Warm = 8192;   // bytes of the previous chunk hashed into a chunk's table
constexpr unsigned short kNoPos = 0xffffu;

struct ChunkSum {
  unsigned int nseq;   // sequences with a match
  unsigned int lead;   // literals before the first match (own bytes only)
  unsigned int trail;  // literals after the last match (carried forward)
  unsigned int len;    // chunk bytes
  unsigned long long rest;  // encoded bytes except the first sequence's literal field + literals
};

struct ChunkPlan {
  unsigned long long off;  // output offset of the chunk's first byte
  unsigned int cin;        // literals carried in from earlier chunks
  unsigned int pad;
};

struct Lz4Ws {
  unsigned long long* n_dev;  // input length actually used
  ChunkSum* sums;
  ChunkPlan* plans;
  uint2* seqs;                // per chunk kLz4MaxSeq x (lit | off << 16, mlen)
  unsigned long long* final_;  // [0] offset of the final sequence, [1] its literal count
};

__device__ __forceinline__ unsigned ext_len(unsigned long long L) {  // bytes after the nibble
  if (L < 15) return 0u;
  // 32-bit division whenever it suffices (the 64-bit one is a long subroutine)
  return L - 15 <= 0xffffffffull ? (unsigned)(L - 15) / 255u + 1u
                                 : (unsigned)((L - 15) / 255 + 1);
}

// 4 bytes at s + p, little endian, from the aligned words holding them (a
// word that holds a byte of the buffer is mapped: allocations are aligned).
__device__ __forceinline__ uint32_t rd32(const uint8_t* s, long long p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(s + p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  const uint32_t sh = (uint32_t)(a & 3) * 8;
  const uint32_t lo = __ldg(w);
  return sh ? __funnelshift_r(lo, __ldg(w + 1), sh) : lo;
}

// rd32 without the alignment branch, for p with p + 7 < n (both words mapped).
__device__ __forceinline__ uint32_t rd32_inner(const uint8_t* s, long long p) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(s + p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  return __funnelshift_r(__ldg(w), __ldg(w + 1), (uint32_t)(a & 3) * 8);
}

// The 4-byte values at positions i + lane (lane 0..31) of one warp, in two
// steps so the load can be issued an iteration early: each lane loads one
// aligned word of the 36-byte window (one coalesced load), and the unaligned
// values are assembled with two shuffles.
__device__ __forceinline__ uint32_t window_load(const uint8_t* s, long long n, long long i,
                                                int lane) {
  const uint32_t* wb =
      reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(s + i) & ~(uintptr_t)3);
  return reinterpret_cast<const uint8_t*>(wb + lane) < s + n ? __ldg(wb + lane) : 0u;
}
__device__ __forceinline__ uint32_t window_value(uint32_t wl, int o, int lane) {
  const int k = (o + lane) >> 2;
  const uint32_t lo = __shfl_sync(0xffffffffu, wl, k);
  const uint32_t hi = __shfl_sync(0xffffffffu, wl, k + 1);
  return __funnelshift_r(lo, hi, (uint32_t)((o + lane) & 3) * 8);
}

template <int HL>
__device__ __forceinline__ uint32_t lz4_hash(uint32_t v) {
  return (v * 2654435761u) >> (32 - HL);
}

// One warp per chunk: greedy parse -> sequences + chunk summary.
template <int HL>
__global__ void __launch_bounds__(kLz4Warps * 32) lz4_parse_kernel(const uint8_t* __restrict__ src,
                                                                 Lz4Ws ws, long long n_chunks) {
  extern __shared__ unsigned short s_tab[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned short* tab = s_tab + (size_t)wib * (1 << HL);
  const long long n = (long long)*ws.n_dev;
  const long long mlimit_g = n - 12;  // lz4.py:17 MFLIMIT
  const int o = (int)(reinterpret_cast<uintptr_t>(src) & 3);  // alignment of src + (4k)
  for (long long ch = (long long)blockIdx.x * kLz4Warps + wib; ch < n_chunks;
       ch += (long long)gridDim.x * kLz4Warps) {
    const long long cs = ch * kLz4Chunk;
    if (cs >= n) {
      if (lane == 0) ws.sums[ch] = ChunkSum{0u, 0u, 0u, 0u, 0ull};
      continue;
    }
    const long long ce = cs + kLz4Chunk < n ? cs + kLz4Chunk : n;
    const long long mend = ce < n - 5 ? ce : n - 5;  // matches end <= mend (LAST_LITERALS)
    // match starts < mlimit: room for a 4-byte match inside the chunk
    const long long mlimit = mend - 3 < mlimit_g ? mend - 3 : mlimit_g;
    // Positions are stored relative to tb = cs - chunk, so the table also
    // holds the previous chunk and matches may reach back into it (offsets
    // stay < 65536; the decoder has those bytes). The table is warmed with
    // every position of the previous chunk's last kLz4Warm bytes (the last
    // writer of a hash wins, as in a serial pass): with 4 Ki slots, a slot
    // whose last writer lies further back survives 8 Ki later positions with
    // probability e^-2, and such old candidates rarely match (C3: +0.01 %).
    const long long tb = cs - kLz4Chunk;
    {
      for (int k = lane; k < (1 << HL); k += 32) tab[k] = kNoPos;
      __syncwarp();
      if (cs > 0) {
        // two batches of 32 positions per step (independent until their
        // stores, which stay in position order)
        const long long w0 = cs - kLz4Warm;
        uint32_t wl0 = window_load(src, n, w0, lane), wl1 = window_load(src, n, w0 + 32, lane);
        for (long long q0 = w0; q0 < cs; q0 += 64) {
          const uint32_t wn0 = window_load(src, n, q0 + 64, lane);
          const uint32_t wn1 = window_load(src, n, q0 + 96, lane);
          const long long qa = q0 + lane, qb = qa + 32;
          const bool oka = qa + 3 < n, okb = qb + 3 < n;
          const uint32_t ha = lz4_hash<HL>(window_value(wl0, o, lane));
          const uint32_t hb = lz4_hash<HL>(window_value(wl1, o, lane));
          wl0 = wn0;
          wl1 = wn1;
          const unsigned pa = __match_any_sync(0xffffffffu, oka ? ha : (0x10000u + lane));
          const unsigned pb = __match_any_sync(0xffffffffu, okb ? hb : (0x10000u + lane));
          if (oka && !(pa >> lane >> 1)) tab[ha] = (unsigned short)(qa - tb);
          __syncwarp();
          if (okb && !(pb >> lane >> 1)) tab[hb] = (unsigned short)(qb - tb);
          __syncwarp();
        }
      }
    }
    // the parse runs in 32-bit offsets from base (the table's origin)
    const long long base = cs > 0 ? tb : cs;
    const uint8_t* sb = src + base;
    const long long nrl = n - base < 3ll * kLz4Chunk ? n - base : 3ll * kLz4Chunk;
    const int nr = (int)nrl;  // readable bytes from sb (clamped)
    const int mlim = (int)(mlimit - base), mendr = (int)(mend - base);
    uint2* seq = ws.seqs + ch * kLz4MaxSeq;
    unsigned nseq = 0, lead = 0;
    unsigned long long rest = 0;
    int i = (int)(cs - base), anchor = i;
    // windows of the batch and of its no-match successor are loaded ahead
    uint32_t wl = window_load(sb, nr, i, lane), w1 = window_load(sb, nr, i + 32, lane);
    while (i < mlim) {
      const uint32_t w2 = window_load(sb, nr, i + 64, lane);
      const int p = i + lane;
      const bool valid = p < mlim;
      const uint32_t v = window_value(wl, (o + (i & 3)) & 3, lane);
      const uint32_t h = lz4_hash<HL>(v);
      // the table candidate and its bytes are fetched while the warp finds
      // same-hash lanes; a lower lane's candidate is its own value
      const unsigned short t = valid ? tab[h] : kNoPos;
      const int tc = t != kNoPos ? (int)t : -1;
      // (candidates lie >= 12 bytes before the end: both words are mapped)
      const uint32_t tv0 = rd32_inner(sb, tc >= 0 ? tc : 0);
      const uint32_t tv = tc >= 0 ? tv0 : ~v;
      const unsigned key = valid ? h : (0x10000u + lane);
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const unsigned lt = (1u << lane) - 1u;
      const unsigned lower = peers & lt;
      const int pl = lower ? 31 - __clz(lower) : lane;
      const uint32_t pv = __shfl_sync(0xffffffffu, v, pl);
      const int cand = lower ? i + pl : tc;
      const bool match = valid && (lower ? pv == v : tv == v);
      const unsigned mm = __ballot_sync(0xffffffffu, match);
      const int w = mm ? __ffs(mm) - 1 : 31;
      const unsigned upto = w == 31 ? 0xffffffffu : ((2u << w) - 1u);
      // every position up to the winner (all, without one) was inserted
      // (lz4.py:62); the last writer of a hash wins
      __syncwarp();
      if (valid && ((1u << lane) & upto) && !(peers & upto & ~lt & ~(1u << lane)))
        tab[h] = (unsigned short)p;
      __syncwarp();
      if (!mm) {
        i += 32;
        wl = w1;
        w1 = w2;
        continue;
      }
      const int pw = i + w;
      const int cw = __shfl_sync(0xffffffffu, cand, w);
      // extend (lz4.py:66-69), 32 bytes per step
      int mlen = 4;
      const int mmax = mendr - pw;
      while (true) {
        const int k = mlen + lane;
        const bool stop = k >= mmax || sb[cw + k] != sb[pw + k];
        const unsigned sbits = __ballot_sync(0xffffffffu, stop);
        if (sbits) {
          mlen += __ffs(sbits) - 1;
          break;
        }
        mlen += 32;
      }
      const unsigned lit = (unsigned)(pw - anchor);
      if (lane == 0) {
        seq[nseq] = make_uint2(lit | ((unsigned)(pw - cw) << 16), (unsigned)mlen);
        rest += 3ull + ext_len((unsigned long long)(mlen - 4));
        if (nseq == 0) lead = lit;
        else rest += ext_len(lit) + (unsigned long long)lit;
      }
      nseq += 1;
      i = pw + mlen;
      anchor = i;
      if (i < mlim && lane == 0) tab[lz4_hash<HL>(rd32(sb, i - 2))] = (unsigned short)(i - 2);
      wl = window_load(sb, nr, i, lane);
      w1 = window_load(sb, nr, i + 32, lane);
      __syncwarp();
    }
    if (lane == 0)
      ws.sums[ch] = ChunkSum{nseq, lead, (unsigned)(ce - base - anchor), (unsigned)(ce - cs), rest};
  }
}

// The effect of a run of chunks on (carried literals cin, output offset
// off): without a match the run only carries its bytes forward; with one,
// its first sequence absorbs cin and the run leaves its trailing literals.
// Composition (then) keeps that form, so runs combine in a warp scan.
struct Lz4Carry {
  int any;                        // the run holds a sequence with a match
  unsigned long long pre;         // bytes before its first match chunk
  unsigned long long lead;        // that chunk's own leading literals
  unsigned long long after;       // encoded bytes besides the first literal field
  unsigned long long cout;        // literals carried out (when any)
  unsigned long long lenall;      // all bytes of the run
  __device__ static Lz4Carry identity() { return Lz4Carry{0, 0ull, 0ull, 0ull, 0ull, 0ull}; }
  __device__ void apply(unsigned long long& cin, unsigned long long& off) const {
    if (any) {
      const unsigned long long L = cin + pre + lead;
      off += after + ext_len(L) + L;
      cin = cout;
    } else {
      cin += lenall;
    }
  }
  __device__ Lz4Carry then(const Lz4Carry& g) const {  // this run, then g
    Lz4Carry r;
    r.lenall = lenall + g.lenall;
    if (!any) {
      r.any = g.any;
      r.pre = lenall + g.pre;
      r.lead = g.lead;
      r.after = g.after;
      r.cout = g.cout;
    } else if (!g.any) {
      r.any = 1;
      r.pre = pre;
      r.lead = lead;
      r.after = after;
      r.cout = cout + g.lenall;
    } else {
      const unsigned long long L = cout + g.pre + g.lead;
      r.any = 1;
      r.pre = pre;
      r.lead = lead;
      r.after = after + g.after + ext_len(L) + L;
      r.cout = g.cout;
    }
    return r;
  }
  __device__ Lz4Carry shfl_up(int d) const {
    Lz4Carry r;
    r.any = __shfl_up_sync(0xffffffffu, any, d);
    r.pre = __shfl_up_sync(0xffffffffu, pre, d);
    r.lead = __shfl_up_sync(0xffffffffu, lead, d);
    r.after = __shfl_up_sync(0xffffffffu, after, d);
    r.cout = __shfl_up_sync(0xffffffffu, cout, d);
    r.lenall = __shfl_up_sync(0xffffffffu, lenall, d);
    return r;
  }
};

// One block: compose the chunks' carry/size functions, assign offsets.
// Chunk with matches: size(cin) = rest + ext(cin + lead) + cin + lead,
// cout = trail. Chunk without: size 0, cout = cin + len.
__global__ void lz4_scan_kernel(Lz4Ws ws, long long n_chunks, unsigned long long* out_len) {
  __shared__ int s_any[1024];
  __shared__ unsigned long long s_pre[1024], s_lead[1024], s_after[1024], s_cout[1024],
      s_lenall[1024];
  const int t = threadIdx.x;
  const long long per = (n_chunks + 1023) / 1024;
  const long long c0 = t * per, c1 = c0 + per < n_chunks ? c0 + per : n_chunks;
  // range summary
  int any = 0;
  unsigned long long pre = 0, lead = 0, after = 0, cout = 0, lenall = 0;
  for (long long c = c0; c < c1; ++c) {
    const ChunkSum s = ws.sums[c];
    lenall += s.len;
    if (s.nseq == 0) {
      if (!any) pre += s.len;
      else cout += s.len;
      continue;
    }
    if (!any) {
      any = 1;
      lead = s.lead;
      after = s.rest;  // first chunk's literal part is added when cin is known
    } else {
      const unsigned long long L = cout + s.lead;
      after += s.rest + ext_len(L) + L;
    }
    cout = s.trail;
  }
  s_any[t] = any;
  s_pre[t] = pre;
  s_lead[t] = lead;
  s_after[t] = after;
  s_cout[t] = cout;
  s_lenall[t] = lenall;
  __syncthreads();
  unsigned long long* s_cin = s_pre;   // reused: thread k's carry-in ...
  unsigned long long* s_off = s_lead;  // ... and output offset
  if (t < 32) {
    // warp 0: lane l composes the summaries of threads [32 l, 32 l + 32),
    // a warp scan composes the lanes, and each lane then walks its 32 again
    // assigning carry-ins and offsets (64 serial steps instead of 1024)
    Lz4Carry acc = Lz4Carry::identity();
    for (int j = 0; j < 32; ++j) {
      const int k = 32 * t + j;
      acc = acc.then(Lz4Carry{s_any[k], s_pre[k], s_lead[k], s_after[k], s_cout[k], s_lenall[k]});
    }
    Lz4Carry inc = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const Lz4Carry up = inc.shfl_up(d);
      if (t >= d) inc = up.then(inc);
    }
    const Lz4Carry exc = inc.shfl_up(1);
    unsigned long long cin = 0, off = 0;
    if (t > 0) exc.apply(cin, off);
    for (int j = 0; j < 32; ++j) {
      const int k = 32 * t + j;
      const Lz4Carry f{s_any[k], s_pre[k], s_lead[k], s_after[k], s_cout[k], s_lenall[k]};
      s_cin[k] = cin;
      s_off[k] = off;
      f.apply(cin, off);
    }
    if (t == 31) {
      const unsigned long long n = *ws.n_dev;
      ws.final_[0] = off;
      ws.final_[1] = cin;
      *out_len = n == 0 ? 0ull : off + 1ull + ext_len(cin) + cin;
    }
  }
  __syncthreads();
  unsigned long long cin = s_cin[t], off = s_off[t];
  for (long long c = c0; c < c1; ++c) {
    const ChunkSum s = ws.sums[c];
    ws.plans[c] = ChunkPlan{off, (unsigned)cin, 0u};
    if (s.nseq == 0) {
      cin += s.len;
    } else {
      const unsigned long long L = cin + s.lead;
      off += s.rest + ext_len(L) + L;
      cin = s.trail;
    }
  }
}

// Warp-parallel sequence writer: token, literal-length extension, literals
// [lsrc, lsrc + L), then (unless final) offset + match-length extension.
__device__ __forceinline__ unsigned long long put_seq(uint8_t* __restrict__ dst,
                                                      unsigned long long o,
                                                      const uint8_t* __restrict__ src,
                                                      long long lsrc, unsigned long long L,
                                                      bool final_, unsigned off, long long mlen,
                                                      int lane) {
  const unsigned long long lcode = L >= 15 ? 15 : L;
  const long long mc = mlen - 4;
  const unsigned long long mcode = final_ ? 0 : (mc >= 15 ? 15 : (unsigned long long)mc);
  if (lane == 0) dst[o] = (uint8_t)((lcode << 4) | mcode);
  o += 1;
  const unsigned el = ext_len(L);
  for (unsigned k = lane; k < el; k += 32)
    dst[o + k] = k + 1 < el ? 255 : (uint8_t)((L - 15) - 255ull * (el - 1));
  o += el;
  for (unsigned long long k = lane; k < L; k += 32) dst[o + k] = src[lsrc + k];
  o += L;
  if (final_) return o;
  if (lane == 0) {
    dst[o] = (uint8_t)(off & 0xff);
    dst[o + 1] = (uint8_t)(off >> 8);
  }
  o += 2;
  const unsigned em = ext_len((unsigned long long)mc);
  for (unsigned k = lane; k < em; k += 32)
    dst[o + k] = k + 1 < em ? 255 : (uint8_t)((mc - 15) - 255ll * (em - 1));
  return o + em;
}

__global__ void __launch_bounds__(kLz4Warps * 32) lz4_emit_kernel(const uint8_t* __restrict__ src,
                                                                uint8_t* __restrict__ dst,
                                                                Lz4Ws ws, long long n_chunks) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long n = (long long)*ws.n_dev;
  for (long long ch = (long long)blockIdx.x * kLz4Warps + wib; ch <= n_chunks;
       ch += (long long)gridDim.x * kLz4Warps) {
    if (ch == n_chunks) {  // the literal-only final sequence (lz4.py:102-113)
      if (n > 0) {
        const unsigned long long L = ws.final_[1];
        put_seq(dst, ws.final_[0], src, n - (long long)L, L, true, 0, 0, lane);
      }
      continue;
    }
    const ChunkSum s = ws.sums[ch];
    if (s.nseq == 0) continue;
    const ChunkPlan pl = ws.plans[ch];
    const long long cs = ch * kLz4Chunk;
    const uint2* seq = ws.seqs + ch * kLz4MaxSeq;
    unsigned long long o = pl.off;           // output offset of the batch
    long long pos = cs - (long long)pl.cin;  // literal source of the batch
    // 32 sequences per step: one coalesced load of their records, warp scans
    // of their encoded sizes and source spans, headers written by the owning
    // lane, literals copied by the owning lane (short) or the warp (long)
    for (unsigned kb = 0; kb < s.nseq; kb += 32) {
      const unsigned k = kb + lane;
      const bool v = k < s.nseq;
      const uint2 q = v ? seq[k] : make_uint2(0u, 4u);
      const unsigned off = q.x >> 16;
      const unsigned long long L = (q.x & 0xffffu) + (k == 0 ? (unsigned long long)pl.cin : 0ull);
      const unsigned mlen = q.y;
      const unsigned el = ext_len(L), em = ext_len((unsigned long long)(mlen - 4));
      const unsigned long long size = v ? 3ull + el + L + em : 0ull;
      const unsigned long long span = v ? L + mlen : 0ull;
      unsigned long long so = size, sp = span;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long a = __shfl_up_sync(0xffffffffu, so, d);
        const unsigned long long b = __shfl_up_sync(0xffffffffu, sp, d);
        if (lane >= d) {
          so += a;
          sp += b;
        }
      }
      const unsigned long long mo = o + so - size;            // this sequence's token
      const long long ms = pos + (long long)(sp - span);      // its literals' source
      const unsigned long long lo = mo + 1 + el;              // its literals' destination
      if (v) {
        const unsigned mc = mlen - 4;
        dst[mo] = (uint8_t)(((L >= 15 ? 15u : (unsigned)L) << 4) | (mc >= 15 ? 15u : mc));
        if (el <= 32)
          for (unsigned j = 0; j < el; ++j)
            dst[mo + 1 + j] = j + 1 < el ? 255 : (uint8_t)((L - 15) - 255ull * (el - 1));
        const unsigned long long om = lo + L;
        dst[om] = (uint8_t)(off & 0xff);
        dst[om + 1] = (uint8_t)(off >> 8);
        for (unsigned j = 0; j < em; ++j)
          dst[om + 2 + j] = j + 1 < em ? 255 : (uint8_t)((mc - 15) - 255u * (em - 1));
        if (L < 32)
          for (unsigned j = 0; j < (unsigned)L; ++j) dst[lo + j] = src[ms + j];
      }
      // long literal-length extensions (carried literals) and long literal runs
      unsigned big = __ballot_sync(0xffffffffu, v && (el > 32 || L >= 32));
      while (big) {
        const int j = __ffs(big) - 1;
        big &= big - 1;
        const unsigned long long jL = __shfl_sync(0xffffffffu, L, j);
        const unsigned long long jlo = __shfl_sync(0xffffffffu, lo, j);
        const long long jms = __shfl_sync(0xffffffffu, ms, j);
        const unsigned jel = __shfl_sync(0xffffffffu, el, j);
        if (jel > 32)
          for (unsigned x = lane; x < jel; x += 32)
            dst[jlo - jel + x] = x + 1 < jel ? 255 : (uint8_t)((jL - 15) - 255ull * (jel - 1));
        if (jL >= 32)
          for (unsigned long long x = lane; x < jL; x += 32) dst[jlo + x] = src[jms + x];
      }
      o += __shfl_sync(0xffffffffu, so, 31);
      pos += (long long)__shfl_sync(0xffffffffu, sp, 31);
    }
  }
}

static long long lz4_chunks(size_t n) { return (long long)((n + kLz4Chunk - 1) / kLz4Chunk); }

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t lz4_workspace_bytes(size_t n_max) {
  const long long nc = lz4_chunks(n_max);
  return 256 + align256(sizeof(ChunkSum) * (size_t)(nc + 1)) +
         align256(sizeof(ChunkPlan) * (size_t)(nc + 1)) +
         sizeof(uint2) * (size_t)kLz4MaxSeq * (size_t)(nc + 1);
}

int lz4_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev, uint8_t* dst,
                 unsigned long long* out_len, void* workspace, size_t ws_bytes,
                 cudaStream_t stream) {
  if (ws_bytes < lz4_workspace_bytes(n_max)) return set_error(VDI_EINVAL, "lz4 workspace too small");
  char* w = static_cast<char*>(workspace);
  Lz4Ws ws;
  ws.n_dev = reinterpret_cast<unsigned long long*>(w);
  ws.final_ = ws.n_dev + 2;
  size_t off = 256;
  const long long nc = lz4_chunks(n_max);
  ws.sums = reinterpret_cast<ChunkSum*>(w + off);
  off += align256(sizeof(ChunkSum) * (size_t)(nc + 1));
  ws.plans = reinterpret_cast<ChunkPlan*>(w + off);
  off += align256(sizeof(ChunkPlan) * (size_t)(nc + 1));
  ws.seqs = reinterpret_cast<uint2*>(w + off);
  set_u64_kernel<<<1, 1, 0, stream>>>(ws.n_dev, n_dev, n_max, ~0ull);
  cudaError_t err;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long nch = nc > 0 ? nc : 0;
  if (nch > 0) {
    long long b = (nch + kLz4Warps - 1) / kLz4Warps;
    if (b > (long long)sms * 16) b = (long long)sms * 16;
    // 4 K-entry tables, 24 warps/SM (2 K: faster, larger blocks; 8 K: the
    // reverse; measured in profiles/r01_bench_codec.jsonl)
    const size_t smem = sizeof(unsigned short) * kLz4Warps * ((size_t)1 << kLz4HashLog);
    err = cudaFuncSetAttribute(lz4_parse_kernel<kLz4HashLog>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "lz4 smem: %s", cudaGetErrorString(err));
    lz4_parse_kernel<kLz4HashLog><<<(unsigned)b, kLz4Warps * 32, smem, stream>>>(src, ws, nch);
  }
  lz4_scan_kernel<<<1, 1024, 0, stream>>>(ws, nch, out_len);
  {
    long long b = (nch + 1 + kLz4Warps - 1) / kLz4Warps;
    if (b > (long long)sms * 16) b = (long long)sms * 16;
    lz4_emit_kernel<<<(unsigned)b, kLz4Warps * 32, 0, stream>>>(src, dst, ws, nch);
  }
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "lz4 launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// ------------------------------------------------- LZ4, exact (serial) parse
// lz4.py:51-114 reproduced byte for byte: ONE greedy parse over the whole
// input with the reference's 64 Ki-entry table (_HASH_LOG 16), so the block
// equals lz4.compress(data) exactly. The parse is inherently serial (each
// decision depends on the table the previous ones left), so one warp runs it,
// 32 positions per step with the same exact batch rule as the chunked parse:
// lane j hashes position i + j, takes its candidate from the nearest lower
// lane with the same hash (a later table write the serial loop would have
// seen) or from the table, and the lowest lane with a verified match is the
// serial decision; the table then receives the positions up to it, the last
// writer of a hash winning.
//
// A serial parse is bound by the latency of its dependent reads, so all of
// them are shared-memory reads (224 KiB):
//  * the table: 17-bit positions (a u16 array and a bit array; a stored s
//    decodes at position p to age (p - s) mod 2^17, and ages 1..65535 are
//    the reference's in-window candidates) plus a valid bit per entry. A
//    sweep every 32 Ki positions (and after a longer jump, with the jump
//    added) drops entries 64 Ki or more behind -- out of the window, so the
//    reference could not use them either -- so every valid age stays below
//    2^17 and decodes exactly;
//  * the input: a ring of 4 KiB segments holding the 64 KiB window behind
//    the current segment, the segment and the next (candidates and the bytes
//    a match extends over; beyond it -- long matches -- the bytes come from
//    global memory).
// Same-hash lanes of a batch are found with __match_any_sync only when a
// cheap test says there may be some: each lane stores its lane id at a
// 13-bit hash of its hash in a scratch table and reads it back; with no
// other lane there, no lane shares its hash. (MATCH.ANY on 32 distinct keys
// costs hundreds of cycles; two of the 32 16-bit hashes coincide in < 1 % of
// batches, two 13-bit ones in ~6 %.)
// The sequences go to a list; a prefix sum of their encoded sizes places
// them, and one warp per sequence writes them.
constexpr int kLzxHash = 16;
constexpr int kLzxSegLog = 12;
constexpr int kLzxSeg = 1 << kLzxSegLog;  // ring segment bytes
constexpr int kLzxSegs = 18;              // 64 KiB of window + the segment + the next
constexpr int kLzxScratch = 8192;         // lane-collision scratch entries (u8)
constexpr long long kLzxSweep = 32768;
constexpr unsigned kLzxKeep = 65536;  // a sweep keeps entries younger than this (the window)

struct LzxSeq {
  unsigned long long pos;     // match start (the final literal-only sequence: n)
  unsigned long long anchor;  // first literal
  unsigned off, mlen;         // mlen 0: the final sequence
};

struct LzxWs {
  unsigned long long* n_dev;  // [0] input length, [1] sequences (incl. the final one)
  LzxSeq* seqs;
  unsigned long long* bsum;   // per emit block
};

constexpr int kLzxBlocks = 1184;  // emit blocks (8 per SM)

__device__ __forceinline__ uint32_t lzx_hash(uint32_t v) { return (v * 2654435761u) >> 16; }

struct LzxSmem {
  unsigned short* tab;  // [65536] position bits 0..15
  uint32_t* hbits;      // [2048] position bit 16
  uint32_t* vbits;      // [2048] valid
  uint32_t* ring;       // [kLzxSeg * kLzxSegs / 4]
  uint8_t* scratch;     // [kLzxScratch]
};

__device__ __forceinline__ uint32_t ring_word(const uint32_t* ring, long long q) {
  const unsigned seg = (unsigned)(q >> kLzxSegLog);
  return ring[(seg % kLzxSegs) * (kLzxSeg / 4) + (((unsigned)q & (kLzxSeg - 1)) >> 2)];
}
__device__ __forceinline__ uint32_t ring_rd32(const uint32_t* ring, long long p) {
  const long long q = p & ~3ll;
  return __funnelshift_r(ring_word(ring, q), ring_word(ring, q + 4), (unsigned)(p & 3) * 8);
}

// word q (4-aligned position) of the source, from the aligned words holding
// it; words at or past the end read as 0 (a word holding a byte of the
// buffer is mapped: allocations are aligned)
__device__ __forceinline__ uint32_t src_word(const uint8_t* src, long long n, long long q) {
  const uint8_t* a = src + q;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(a) & ~(uintptr_t)3);
  const unsigned sh = (unsigned)(reinterpret_cast<uintptr_t>(a) & 3) * 8;
  const uint8_t* end = src + n;
  const uint32_t lo = reinterpret_cast<const uint8_t*>(w) < end ? __ldg(w) : 0u;
  if (!sh) return lo;
  const uint32_t hi = reinterpret_cast<const uint8_t*>(w + 1) < end ? __ldg(w + 1) : 0u;
  return __funnelshift_r(lo, hi, sh);
}

// Keep segments [seg(i) - 16, seg(i) + 2) in the ring (loaded: [seg_lo, seg_hi)).
__device__ __forceinline__ void lzx_ensure(const LzxSmem& sm, const uint8_t* src, long long n,
                                           long long i, long long& seg_lo, long long& seg_hi,
                                           int lane) {
  constexpr long long kBack = kLzxSegs - 2;
  const long long cur = i >> kLzxSegLog;
  const long long t_lo = cur - kBack > 0 ? cur - kBack : 0, t_hi = cur + 2;
  if (seg_hi >= t_hi) return;
  long long s0 = seg_hi > t_lo ? seg_hi : t_lo;
  for (long long s = s0; s < t_hi; ++s) {
    uint32_t* dst = sm.ring + (unsigned)(s % kLzxSegs) * (kLzxSeg / 4);
    const long long base = s * kLzxSeg;
#pragma unroll 8
    for (int k = lane; k < kLzxSeg / 4; k += 32) dst[k] = src_word(src, n, base + 4ll * k);
  }
  seg_lo = t_lo;
  seg_hi = t_hi;
  __syncwarp();
}

// Drop entries whose age (relative to ref, plus extra) is >= kLzxKeep.
__device__ __forceinline__ void lzx_sweep(const LzxSmem& sm, long long ref, long long extra,
                                          int lane) {
  const unsigned r17 = (unsigned)(ref & 0x1ffff);
  for (int wd = lane; wd < (1 << kLzxHash) / 32; wd += 32) {
    uint32_t bits = sm.vbits[wd];
    const uint32_t hb = sm.hbits[wd];
    uint32_t keep = bits;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const unsigned s17 = sm.tab[wd * 32 + b] | (((hb >> b) & 1u) << 16);
      const unsigned age = (r17 - s17) & 0x1ffffu;
      if ((long long)age + extra >= (long long)kLzxKeep) keep &= ~(1u << b);
    }
    sm.vbits[wd] = keep;
  }
  __syncwarp();
}

__device__ __forceinline__ void lzx_insert(const LzxSmem& sm, uint32_t h, long long p) {
  sm.tab[h] = (unsigned short)(p & 0xffff);
  const uint32_t bit = 1u << (h & 31);
  if ((p >> 16) & 1) atomicOr(sm.hbits + (h >> 5), bit);
  else atomicAnd(sm.hbits + (h >> 5), ~bit);
  atomicOr(sm.vbits + (h >> 5), bit);
}

__global__ void __launch_bounds__(32) lzx_parse_kernel(const uint8_t* __restrict__ src, LzxWs ws) {
  extern __shared__ uint32_t x_smem[];
  LzxSmem sm;
  sm.tab = reinterpret_cast<unsigned short*>(x_smem);
  sm.hbits = x_smem + (1 << kLzxHash) / 2;
  sm.vbits = sm.hbits + (1 << kLzxHash) / 32;
  sm.ring = sm.vbits + (1 << kLzxHash) / 32;
  sm.scratch = reinterpret_cast<uint8_t*>(sm.ring + kLzxSeg * kLzxSegs / 4);
  const int lane = threadIdx.x;
  const long long n = (long long)ws.n_dev[0];
  for (int k = lane; k < (1 << kLzxHash) / 32; k += 32) sm.vbits[k] = sm.hbits[k] = 0u;
  long long seg_lo = 0, seg_hi = 0;
  lzx_ensure(sm, src, n, 0, seg_lo, seg_hi, lane);
  const long long limit = n - 12;  // lz4.py:62 (MFLIMIT)
  long long i = 0, anchor = 0, next_sweep = kLzxSweep;
  unsigned long long nseq = 0;
  while (i < limit) {
    if (i >= next_sweep) {
      lzx_sweep(sm, i, 0, lane);
      next_sweep = i + kLzxSweep;
    }
    lzx_ensure(sm, src, n, i, seg_lo, seg_hi, lane);
    const long long p = i + lane;
    const bool valid = p < limit;
    const uint32_t v = ring_rd32(sm.ring, p);
    const uint32_t h = lzx_hash(v);
    const unsigned st = sm.tab[h] | (((sm.hbits[h >> 5] >> (h & 31)) & 1u) << 16);
    const bool vb = valid && ((sm.vbits[h >> 5] >> (h & 31)) & 1u);
    const unsigned age = ((unsigned)(p & 0x1ffff) - st) & 0x1ffffu;
    const long long tc = vb && age != 0u && age <= 65535u ? p - (long long)age : -1;
    const uint32_t tv = tc >= 0 ? ring_rd32(sm.ring, tc) : ~v;
    const unsigned key = valid ? h : (0x10000u + lane);
    const unsigned sk = key & (kLzxScratch - 1);
    sm.scratch[sk] = (uint8_t)lane;
    __syncwarp();
    const bool alone = sm.scratch[sk] == (uint8_t)lane;
    const unsigned peers =
        __all_sync(0xffffffffu, alone) ? (1u << lane) : __match_any_sync(0xffffffffu, key);
    const unsigned lt = (1u << lane) - 1u;
    const unsigned lower = peers & lt;
    const int pl = lower ? 31 - __clz(lower) : lane;
    const uint32_t pv = __shfl_sync(0xffffffffu, v, pl);
    const long long cand = lower ? i + pl : tc;
    const bool match = valid && (lower ? pv == v : tv == v);
    const unsigned mm = __ballot_sync(0xffffffffu, match);
    const int w = mm ? __ffs(mm) - 1 : 31;
    const unsigned upto = w == 31 ? 0xffffffffu : ((2u << w) - 1u);
    __syncwarp();
    if (valid && ((1u << lane) & upto) && !(peers & upto & ~lt & ~(1u << lane)))
      lzx_insert(sm, h, p);
    __syncwarp();
    if (!mm) {
      i += 32;
      continue;
    }
    const long long pw = i + w;
    const long long cw = __shfl_sync(0xffffffffu, cand, w);
    // extend (lz4.py:66-69), 32 bytes per step; bytes past the ring's
    // lookahead (long matches) come from global memory
    long long mlen = 4;
    const long long mmax = n - 5 - pw;
    const long long hi_b = seg_hi * kLzxSeg;
    while (true) {
      const long long k = mlen + lane;
      bool stop = k >= mmax;
      if (!stop) {
        const long long xa = cw + k, xb = pw + k;
        const unsigned ba = xa < hi_b ? (ring_word(sm.ring, xa & ~3ll) >> ((xa & 3) * 8)) & 0xffu
                                      : (unsigned)src[xa];
        const unsigned bb = xb < hi_b ? (ring_word(sm.ring, xb & ~3ll) >> ((xb & 3) * 8)) & 0xffu
                                      : (unsigned)src[xb];
        stop = ba != bb;
      }
      const unsigned sbits = __ballot_sync(0xffffffffu, stop);
      if (sbits) {
        mlen += __ffs(sbits) - 1;
        break;
      }
      mlen += 32;
    }
    if (lane == 0)
      ws.seqs[nseq] = LzxSeq{(unsigned long long)pw, (unsigned long long)anchor,
                             (unsigned)(pw - cw), (unsigned)mlen};
    nseq += 1;
    i = pw + mlen;
    anchor = i;
    if (i >= next_sweep) {  // ages are exact relative to pw (the last insert)
      lzx_sweep(sm, pw, i - pw, lane);
      next_sweep = i + kLzxSweep;
    }
    if (i < limit) {
      lzx_ensure(sm, src, n, i, seg_lo, seg_hi, lane);
      if (lane == 0) lzx_insert(sm, lzx_hash(ring_rd32(sm.ring, i - 2)), i - 2);
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (n > 0) {
      ws.seqs[nseq] = LzxSeq{(unsigned long long)n, (unsigned long long)anchor, 0u, 0u};
      nseq += 1;
    }
    ws.n_dev[1] = nseq;
  }
}

__device__ __forceinline__ unsigned long long lzx_size(const LzxSeq& q) {
  const unsigned long long lit = q.pos - q.anchor;
  unsigned long long sz = 1 + ext_len(lit) + lit;
  if (q.mlen) sz += 2 + ext_len((unsigned long long)q.mlen - 4);
  return sz;
}

__device__ __forceinline__ void lzx_range(const LzxWs& ws, long long& b0, long long& b1) {
  const long long m = (long long)ws.n_dev[1];
  const long long per = (m + kLzxBlocks - 1) / kLzxBlocks;
  b0 = blockIdx.x * per;
  b1 = b0 + per < m ? b0 + per : m;
}

__global__ void __launch_bounds__(1024) lzx_size_kernel(LzxWs ws) {
  __shared__ unsigned long long s_w[32];
  long long b0, b1;
  lzx_range(ws, b0, b1);
  unsigned long long sum = 0;
  for (long long k = b0 + threadIdx.x; k < b1; k += blockDim.x) sum += lzx_size(ws.seqs[k]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long v = s_w[threadIdx.x];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) ws.bsum[blockIdx.x] = v;
  }
}

__device__ __forceinline__ unsigned long long lzx_put_len(uint8_t* dst, unsigned long long d,
                                                          unsigned long long len) {
  while (len >= 255) {  // lz4.py:43-49 _write_length
    dst[d++] = 255;
    len -= 255;
  }
  dst[d++] = (uint8_t)len;
  return d;
}

// Block b writes its sequence range: sizes -> block scan (1024 at a time) ->
// one warp per sequence (the header and extension bytes by lane 0, the
// literals 32 bytes per step by the warp).
__global__ void __launch_bounds__(1024) lzx_emit_kernel(const uint8_t* __restrict__ src,
                                                        uint8_t* __restrict__ dst, LzxWs ws,
                                                        unsigned long long* out_len) {
  __shared__ unsigned long long s_off[1024];
  __shared__ unsigned long long s_w[32];
  long long b0, b1;
  lzx_range(ws, b0, b1);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  unsigned long long run = ws.bsum[blockIdx.x];
  for (long long c0 = b0; c0 < b1; c0 += 1024) {
    const long long k = c0 + t;
    const unsigned long long sz = k < b1 ? lzx_size(ws.seqs[k]) : 0ull;
    unsigned long long v = sz;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += u;
    }
    if (lane == 31) s_w[wid] = v;
    __syncthreads();
    if (wid == 0) {
      unsigned long long x = s_w[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += u;
      }
      s_w[lane] = x;
    }
    __syncthreads();
    s_off[t] = run + (wid > 0 ? s_w[wid - 1] : 0ull) + v - sz;
    const unsigned long long total = s_w[31];
    __syncthreads();
    const long long cn = b1 - c0 < 1024 ? b1 - c0 : 1024;
    for (long long j = wid; j < cn; j += 32) {
      const LzxSeq q = ws.seqs[c0 + j];
      unsigned long long d = s_off[j];
      const unsigned long long lit = q.pos - q.anchor;
      const unsigned lcode = lit >= 15 ? 15u : (unsigned)lit;
      const unsigned mcode = q.mlen ? (q.mlen - 4 >= 15 ? 15u : q.mlen - 4) : 0u;
      unsigned long long dl = d + 1;  // literals start
      if (lane == 0) {
        dst[d] = (uint8_t)((lcode << 4) | mcode);
        if (lit >= 15) dl = lzx_put_len(dst, d + 1, lit - 15);
      }
      dl = __shfl_sync(0xffffffffu, dl, 0);
      for (unsigned long long x = lane; x < lit; x += 32) dst[dl + x] = src[q.anchor + x];
      if (q.mlen && lane == 0) {
        unsigned long long e = dl + lit;
        dst[e] = (uint8_t)(q.off & 0xff);
        dst[e + 1] = (uint8_t)((q.off >> 8) & 0xff);
        if (q.mlen - 4 >= 15) lzx_put_len(dst, e + 2, (unsigned long long)q.mlen - 4 - 15);
      }
    }
    run += total;
    __syncthreads();
  }
  if (blockIdx.x == kLzxBlocks - 1 && t == 0) *out_len = run;
}

size_t lzx_workspace_bytes(size_t n_max) {
  return 256 + align256(sizeof(LzxSeq) * (n_max / 4 + 2)) +
         align256(sizeof(unsigned long long) * kLzxBlocks);
}

int lzx_compress(const uint8_t* src, size_t n_max, const unsigned long long* n_dev, uint8_t* dst,
                 unsigned long long* out_len, void* workspace, size_t ws_bytes,
                 cudaStream_t stream) {
  if (ws_bytes < lzx_workspace_bytes(n_max))
    return set_error(VDI_EINVAL, "lz4 exact workspace too small");
  char* w = static_cast<char*>(workspace);
  LzxWs ws;
  ws.n_dev = reinterpret_cast<unsigned long long*>(w);
  size_t off = 256;
  ws.seqs = reinterpret_cast<LzxSeq*>(w + off);
  off += align256(sizeof(LzxSeq) * (n_max / 4 + 2));
  ws.bsum = reinterpret_cast<unsigned long long*>(w + off);
  set_u64_kernel<<<1, 1, 0, stream>>>(ws.n_dev, n_dev, n_max, 0ull);
  const size_t smem = sizeof(unsigned short) * ((size_t)1 << kLzxHash) +
                      2 * sizeof(uint32_t) * ((size_t)1 << kLzxHash) / 32 +
                      (size_t)kLzxSeg * kLzxSegs + kLzxScratch;
  cudaError_t err =
      cudaFuncSetAttribute(lzx_parse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "lz4x smem: %s", cudaGetErrorString(err));
  lzx_parse_kernel<<<1, 32, smem, stream>>>(src, ws);
  lzx_size_kernel<<<kLzxBlocks, 1024, 0, stream>>>(ws);
  scan_blocks_kernel<<<1, 1024, 0, stream>>>(ws.bsum, kLzxBlocks);
  lzx_emit_kernel<<<kLzxBlocks, 1024, 0, stream>>>(src, dst, ws, out_len);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "lz4x launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

// ------------------------------------------------------- validate_vdi

// vdi.py:116-134 on the device. codes: 1 front >= back, 2 overlapping,
// 3 depth outside [-1, 1], 4 colour not premultiplied (first failing check
// of a list, in the reference's order); result[0] = min over failing lists
// of (list << 3 | code), result[1] = count-range violations.
__global__ void validate_kernel(const VdiValidateArgs a, unsigned long long* result) {
  const long long n = (long long)a.width * a.height;
  const float lo_f = (float)(-1.0 - 1e-6), hi_f = (float)(1.0 + 1e-6);
  unsigned long long best = ~0ull;
  unsigned long long range_bad = 0;
  for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < n;
       l += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(l / a.width), x = (int)(l - (long long)r * a.width);
    const long long li =
        (long long)vdi_storage_row(r, a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank) *
            a.width + x;
    const int cnt = a.counts[li];
    if (cnt < 0 || cnt > a.n_sg) {
      range_bad += 1;
      continue;
    }
    if (cnt == 0) continue;
    const float* ls = a.segs + li * (long long)list_stride(a.n_sg);
    const float* fr = ls + front_off(a.n_sg);
    const float* bk = ls + back_off(a.n_sg);
    const float4* c4 = reinterpret_cast<const float4*>(ls);
    int code = 0;
    for (int k = 0; k < cnt && !code; ++k)
      if (!(fr[k] < bk[k])) code = 1;
    for (int k = 0; k + 1 < cnt && !code; ++k)
      if (!(bk[k] <= __fadd_rn(fr[k + 1], 1e-7f))) code = 2;
    if (!code) {
      float fmn = fr[0], bmx = bk[0];
      for (int k = 1; k < cnt; ++k) {
        fmn = fminf(fmn, fr[k]);
        bmx = fmaxf(bmx, bk[k]);
      }
      if (fmn < lo_f || bmx > hi_f) code = 3;
    }
    for (int k = 0; k < cnt && !code; ++k) {
      const float4 c = c4[k];
      const float m = fmaxf(fmaxf(c.x, c.y), c.z);
      if (m > __fadd_rn(c.w, 1e-6f)) code = 4;
    }
    if (code) {
      const unsigned long long key = ((unsigned long long)l << 3) | (unsigned long long)code;
      if (key < best) best = key;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
    best = ob < best ? ob : best;
    range_bad += __shfl_xor_sync(0xffffffffu, range_bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (best != ~0ull) atomicMin(result, best);
    if (range_bad) atomicAdd(result + 1, range_bad);
  }
}

int validate_vdi(const VdiValidateArgs* args, cudaStream_t stream) {
  VdiValidateArgs c = *args;
  if (c.vdi_band_rows <= 0) c.vdi_band_rows = 16;
  if (c.vdi_band_world <= 0) c.vdi_band_world = 1;
  set_u64_kernel<<<1, 1, 0, stream>>>(c.result, nullptr, ~0ull, 0ull);
  cudaError_t err;
  const long long n = (long long)c.width * c.height;
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  validate_kernel<<<(unsigned)(b < 1 ? 1 : b), 256, 0, stream>>>(c, c.result);
  err = cudaGetLastError();
  if (err != cudaSuccess) return set_error(VDI_ELAUNCH, "validate launch: %s", cudaGetErrorString(err));
  return VDI_OK;
}

}  // namespace vdi
