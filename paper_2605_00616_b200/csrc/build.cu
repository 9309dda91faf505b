// build.cu -- offline profile-table build on the GPU (emu_tables_build).
//
// Replaces build_pack (profile.py:230-267), PhaseTable.from_buckets
// (profile.py:122-129) and, in canonical mode, save_pack's ascending sample
// order (profile.py:281-282):
//   1. k_validate   : StepTraceRecord.validate per record (profile.py:61-79);
//                     smallest failing index wins (build_pack reports the first).
//   2. k_make_keys  : hi = phase << (top bit) | (tt-1) << cbits | (conc-1),
//                     lo = lat_bits (positive doubles order like their IEEE
//                     bit patterns); the phase rides in hi's top bit, which
//                     no digit pass reads, so it costs no sort pass.  The
//                     digit histograms of every pass come out of the same
//                     read of the records.
//   3. LSD radix sort, 8-bit digits, stable: per 4096-record tile, warp
//      match_any ranking into shared memory in digit order, then coalesced
//      digit runs out (k_radix_scatter); scratch from a stream-ordered pool:
//        canonical -> digits of lo then hi   (bucket key, then latency value)
//        capture   -> digits of hi only      (stable = build_pack's dict appends)
//      digit positions whose histogram is a single bin are skipped.
//   4. the sorted run IS the combined table; a stable partition on the phase
//      bit gives the decode and mixed runs in the same order (no second sort);
//   5. segment each run: head flags -> exclusive scan -> bucket SoA, offsets,
//      row index (distinct tt) and key ranges.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <string>
#include <vector>

#include "emu_internal.cuh"
#include "prof.h"
#include "scan.cuh"
#include "tables.h"

namespace emu {

constexpr int kRThreads = 256;
constexpr int kRWarps = kRThreads / 32;
constexpr int kRRounds = 16;
constexpr int kRTile = kRThreads * kRRounds;

struct RecIn {
  const int32_t* tt;
  const int32_t* conc;
  const uint8_t* ph;
  const double* lat;
  const int64_t* step;
  int64_t n;
};

// Four records per thread per iteration (their loads issue together: the
// check is a pure stream, latency-bound at one record per thread).
__device__ __forceinline__ int record_check(const RecIn& r, int64_t i, int32_t t, int32_t c, double l) {
  if (r.step && r.step[i] < 0) return 1;
  if (t < 1) return 2;
  if (c < 1) return 3;
  if (r.ph[i] == 0 && t < c) return 4;
  if (!(l > 0.0)) return 5;
  return 0;
}
__global__ void __launch_bounds__(256, 6) k_validate(RecIn r, unsigned long long* first_bad, int* maxv) {
  int mt = 0, mc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i0 < r.n; i0 += stride) {
    int32_t t[4], c[4];
    double l[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int64_t i = i0 + (int64_t)q * gridDim.x * blockDim.x;
      t[q] = 1;
      c[q] = 1;
      l[q] = 1.0;
      if (i < r.n) {
        t[q] = r.tt[i];
        c[q] = r.conc[i];
        l[q] = r.lat[i];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int64_t i = i0 + (int64_t)q * gridDim.x * blockDim.x;
      if (i >= r.n) continue;
      const int code = record_check(r, i, t[q], c[q], l[q]);
      if (code) atomicMin(first_bad, ((unsigned long long)i << 3) | (unsigned long long)code);
      mt = max(mt, t[q]);
      mc = max(mc, c[q]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mt = max(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&maxv[0], mt);
    atomicMax(&maxv[1], mc);
  }
}

// The phase bit of a key word (decode 0, mixed 1) and the bucket key under it.
template <typename H>
__device__ __forceinline__ unsigned key_phase(H h) {
  return (unsigned)(h >> (8 * sizeof(H) - 1));
}
template <typename H>
__device__ __forceinline__ H key_bucket(H h) {
  return h & (H)(~((H)1 << (8 * sizeof(H) - 1)));
}

struct PassSet {
  int n;
  int word[17];  // 0 = lo, 1 = hi (entry n is a sentinel)
  int shift[17];
};

// One digit's histogram into a CTA's shared counters: a warp whose valid
// digits all agree (the exponent digits of the latencies) adds once instead
// of 32 same-address shared atomics.
__device__ __forceinline__ void hist_add(unsigned int* sh, unsigned d, bool v) {
  const unsigned vm = __ballot_sync(0xffffffffu, v);
  if (!vm) return;
  const int leader = __ffs(vm) - 1;
  const unsigned d0 = __shfl_sync(0xffffffffu, d, leader);
  if (__all_sync(0xffffffffu, !v || d == d0)) {
    if ((int)(threadIdx.x & 31) == leader) atomicAdd(&sh[d0], (unsigned)__popc(vm));
  } else if (v) {
    atomicAdd(&sh[d], 1u);
  }
}

// Keys of every record, the bits in which any record differs from record 0
// (diff[0] latency word, diff[1] bucket key: a digit position whose 8 bits
// never differ is the same for all records and its pass is skipped), and the
// histogram of the first pass's digit (hword/hshift: the lowest latency digit
// in canonical mode, else the lowest key digit).  Each later pass's histogram
// is counted by the pass before it (k_onesweep), so the records are read once
// here instead of once per pass.
template <typename H>
__global__ void __launch_bounds__(256) k_make_keys(RecIn r, int cbits, int lsb, H* __restrict__ hi,
                                                   uint64_t* __restrict__ lo, int hword, int hshift, unsigned int* hist,
                                                   unsigned long long* diff) {
  __shared__ unsigned int sh[256];
  sh[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t k0 = (((uint64_t)(uint32_t)(r.tt[0] - 1) << cbits) | (uint64_t)(uint32_t)(r.conc[0] - 1))
                      << lsb | (lsb && r.ph[0] ? 1ULL : 0ULL);
  const uint64_t l0 = (uint64_t)__double_as_longlong(r.lat[0]);
  uint64_t dk = 0, dl = 0;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < r.n; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;  // warp-uniform trip count (votes in hist_add)
    const bool v = i < r.n;
    uint64_t h = 0, l = 0;
    if (v) {
      h = ((uint64_t)(uint32_t)(r.tt[i] - 1) << cbits) | (uint64_t)(uint32_t)(r.conc[i] - 1);
      l = (uint64_t)__double_as_longlong(r.lat[i]);
      if (lsb) {  // canonical dense builds: the phase sorts just below the bucket key
        h = h << 1 | (r.ph[i] ? 1ULL : 0ULL);
        hi[i] = (H)h;
      } else {
        hi[i] = (H)h | (r.ph[i] ? (H)1 << (8 * sizeof(H) - 1) : (H)0);
      }
      lo[i] = l;
      dk |= h ^ k0;
      dl |= l ^ l0;
    }
    hist_add(sh, (unsigned)(((hword ? h : l) >> hshift) & 255u), v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dk |= __shfl_xor_sync(0xffffffffu, dk, o);
    dl |= __shfl_xor_sync(0xffffffffu, dl, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (dl) atomicOr(&diff[0], (unsigned long long)dl);
    if (dk) atomicOr(&diff[1], (unsigned long long)dk);
  }
  __syncthreads();
  if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

// One digit's histogram over the key arrays (only when make_keys guessed the
// first pass wrong: its lowest digit turned out to be the same everywhere).
template <typename H>
__global__ void __launch_bounds__(256) k_digit_hist1(const H* __restrict__ hi, const uint64_t* __restrict__ lo,
                                                     int64_t n, int word, int shift, unsigned int* hist) {
  __shared__ unsigned int sh[256];
  sh[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    const bool v = i < n;
    const uint64_t w = v ? (word ? (uint64_t)key_bucket(hi[i]) : lo[i]) : 0;
    hist_add(sh, (unsigned)((w >> shift) & 255u), v);
  }
  __syncthreads();
  if (sh[threadIdx.x]) atomicAdd(&hist[threadIdx.x], sh[threadIdx.x]);
}

// Record count of every (phase, bucket key) over the dense key domain
// [0, 2^kb) per phase, from the SORTED records: a warp's 32 consecutive
// records share one or two keys, so one atomic per distinct key per warp is
// cheap (counting before the sort hammers the hot decode keys).  The tables'
// buckets and offsets then come from scans over the domain (segment_dense)
// instead of scans over the records.
template <typename H>
__global__ void k_dense_count(const H* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n, int kb, int lsb,
                              unsigned int* __restrict__ dcnt) {
  const int lane = threadIdx.x & 31;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;  // warp-uniform trip count (match_any below)
    const bool v = i < n;
    const unsigned key = !v    ? 0xffffffffu - (unsigned)lane
                         : lsb ? ((unsigned)(hi[i] & 1u) << kb) | (unsigned)(hi[i] >> 1)
                               : (key_phase(hi[i]) << kb) | (unsigned)key_bucket(hi[i]);
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (v && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&dcnt[key], (unsigned)__popc(peers));
  }
}

__global__ void __launch_bounds__(kRThreads) k_radix_up(const uint64_t* __restrict__ key, uint64_t kmask, int shift,
                                                       int64_t n, int64_t nblk, unsigned int* counts) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRTile;
#pragma unroll 4
  for (int k = 0; k < kRRounds; k++) {
    const int64_t i = base + (int64_t)k * kRThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[((key[i] & kmask) >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * nblk + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of (hi, lo) pairs by one digit of `key` (== hi or lo).  The
// tile is first ranked into shared memory in digit order (warp match_any per
// round of 256, stable), then written out with consecutive threads on
// consecutive output positions: every digit's run of the tile is a coalesced
// segment instead of 256 interleaved 8-byte streams.
constexpr int kRSmem = kRTile * 16;
__global__ void __launch_bounds__(kRThreads) k_radix_scatter(const uint64_t* __restrict__ key, int shift, int key_is_hi,
                                                            const uint64_t* __restrict__ a_hi,
                                                            const uint64_t* __restrict__ a_lo, uint64_t* __restrict__ b_hi,
                                                            uint64_t* __restrict__ b_lo, int64_t n, int64_t nblk,
                                                            const unsigned int* __restrict__ offs) {
  extern __shared__ uint64_t tile[];  // [kRTile] hi, then [kRTile] lo
  uint64_t* s_hi = tile;
  uint64_t* s_lo = tile + kRTile;
  __shared__ unsigned int gofs[256];
  __shared__ unsigned int tstart[256];
  __shared__ unsigned int run[256];
  __shared__ unsigned short wh[kRWarps][256];
  __shared__ unsigned int wsum[kRWarps];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t blk = blockIdx.x;
  const int64_t base = blk * kRTile;
  const int cnt_tile = (int)min((int64_t)kRTile, n - base);
  // this tile's digit counts from the scanned (digit-major) offsets
  const int64_t flat = (int64_t)t * nblk + blk;
  const unsigned int o0 = offs[flat];
  const unsigned int o1 = (t == 255 && blk == nblk - 1) ? (unsigned int)n : offs[flat + 1];
  gofs[t] = o0;
  const unsigned int c = o1 - o0;
  // exclusive scan of the 256 counts -> tile-local digit starts
  unsigned int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  run[t] = 0;
  __syncthreads();
  unsigned int wb = 0;
  for (int q = 0; q < w; q++) wb += wsum[q];
  tstart[t] = wb + x - c;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int k = 0; k < kRRounds; k++) {
    const int li = k * kRThreads + t;
    const int64_t i = base + li;
    const bool valid = li < cnt_tile;
#pragma unroll
    for (int q = 0; q < kRWarps; q++) wh[q][t] = 0;
    __syncthreads();
    uint64_t h = 0, l = 0;
    if (valid) {
      h = a_hi[i];
      l = a_lo[i];
    }
    const unsigned d = valid ? (unsigned)(((key_is_hi ? key_bucket(h) : l) >> shift) & 255u) : 256u + (unsigned)lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wh[w][d] = (unsigned short)__popc(peers);
    __syncthreads();
    {
      unsigned r = run[t];
#pragma unroll
      for (int q = 0; q < kRWarps; q++) {
        unsigned cc = wh[q][t];
        wh[q][t] = (unsigned short)r;
        r += cc;
      }
      run[t] = r;
    }
    __syncthreads();
    if (valid) {
      const unsigned lp = tstart[d] + wh[w][d] + rank;
      s_hi[lp] = h;
      s_lo[lp] = l;
    }
    __syncthreads();  // wh is rewritten by the next round
  }
  for (int j = t; j < cnt_tile; j += kRThreads) {
    const uint64_t h = s_hi[j], l = s_lo[j];
    const unsigned d = (unsigned)(((key_is_hi ? key_bucket(h) : l) >> shift) & 255u);
    const unsigned pos = gofs[d] + (unsigned)j - tstart[d];
    b_hi[pos] = h;
    b_lo[pos] = l;
  }
}

// One LSD pass without an up-sweep ("onesweep"): every pass's global digit
// starts come from the single all-digits histogram (k_make_keys); a tile's
// offset inside each digit bucket comes from a decoupled look-back over the
// tiles before it.  Tiles take their index from an atomic counter in launch
// order, so a tile only ever waits on tiles that are already running.
// Per record and pass: the (hi, lo) pair is read once and written once
// (12 B each way with 32-bit bucket keys) -- no separate counting pass.
// look[t * 256 + d] = flag << 30 | value: flag 1 = tile t's own count of digit
// d, flag 2 = inclusive prefix over tiles <= t (values < 2^30: n < 2^30).
#ifndef EMU_LOOKBACK
#define EMU_LOOKBACK 16
#endif
constexpr unsigned kLookAgg = 1u << 30, kLookPre = 2u << 30, kLookVal = (1u << 30) - 1u;
#ifndef EMU_OS_ITEMS
#define EMU_OS_ITEMS 12
#endif
constexpr int kOsItems = EMU_OS_ITEMS;          // records per thread of a onesweep tile
constexpr int kOsTile = kRThreads * kOsItems;
#ifndef EMU_OS_MINB
#define EMU_OS_MINB 4
#endif
template <typename H>
__global__ void __launch_bounds__(kRThreads, EMU_OS_MINB) k_onesweep(const H* __restrict__ a_hi, const uint64_t* __restrict__ a_lo,
                                                       H* __restrict__ b_hi, uint64_t* __restrict__ b_lo, int64_t n,
                                                       int shift, int key_is_hi, const unsigned int* __restrict__ hcur,
                                                       unsigned int* look, unsigned int* tile_ctr,
                                                       unsigned int* __restrict__ hnext, int nshift, int nword) {
  constexpr int kWarpItems = kOsTile / kRWarps;  // consecutive records per warp
  extern __shared__ __align__(16) unsigned char osm[];
  uint64_t* s_lo = reinterpret_cast<uint64_t*>(osm);
  H* s_hi = reinterpret_cast<H*>(osm + (size_t)kOsTile * 8);
  __shared__ unsigned short wcnt[kRWarps][256];  // per-warp digit counts, then each warp's offset in the digit
  __shared__ unsigned int tstart[256];
  __shared__ unsigned int gofs[256];  // the digit's global start + this tile's exclusive prefix
  __shared__ unsigned int wsum[kRWarps];
  __shared__ unsigned int gsum[kRWarps];
  __shared__ unsigned int nh[256];  // the next pass's digit counts of this tile
  __shared__ unsigned int s_tile;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_tile = atomicAdd(tile_ctr, 1u);
  const unsigned hc = hcur[t];  // this pass's global count of digit t (counted by the pass before)
#pragma unroll
  for (int q = 0; q < kRWarps; q++) wcnt[q][t] = 0;
  nh[t] = 0;
  __syncthreads();
  const unsigned tile = s_tile;
  const int64_t base = (int64_t)tile * kOsTile;
  const int cnt_tile = (int)min((int64_t)kOsTile, n - base);
  const unsigned lt_mask = (1u << lane) - 1u;
  // ---- load: warp w owns records [w*512, (w+1)*512) of the tile, 32 per round (coalesced)
  H h[kOsItems];
  uint64_t l[kOsItems];
  unsigned rk[kOsItems / 2];  // warp-local ranks (< 512), two per register
#pragma unroll
  for (int k = 0; k < kOsItems; k++) {
    const int li = w * kWarpItems + k * 32 + lane;
    h[k] = 0;
    l[k] = 0;
    if (li < cnt_tile) {
      h[k] = a_hi[base + li];
      l[k] = a_lo[base + li];
    }
  }
  // ---- warp-private ranking (no block barriers): rank = the warp's running
  // count of the digit + this round's rank among equal digits.  The lowest
  // lane of each digit group adds the group to the warp's counter (two 16-bit
  // counters per word) and broadcasts the old count; a warp's shared atomics
  // execute in issue order, so rounds need no __syncwarp.  12 records per
  // thread keep the pass in 64 registers without spills (16 spilled; measured
  // 7.9 vs 8.3 ms for the 10 C4 passes).
  unsigned* wc32 = reinterpret_cast<unsigned*>(&wcnt[w][0]);
#pragma unroll
  for (int k = 0; k < kOsItems; k++) {
    const bool valid = w * kWarpItems + k * 32 + lane < cnt_tile;
    const unsigned d = valid ? (unsigned)(((key_is_hi ? (uint64_t)key_bucket(h[k]) : l[k]) >> shift) & 255u) : 256u + (unsigned)lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned r = __popc(peers & lt_mask);
    unsigned old = 0;
    if (valid && r == 0) old = atomicAdd(&wc32[d >> 1], (unsigned)__popc(peers) << ((d & 1) * 16));
    old = __shfl_sync(0xffffffffu, old, __ffs(peers) - 1);
    const unsigned before = (old >> ((d & 1) * 16)) & 0xffffu;
    if (k & 1)
      rk[k >> 1] |= (before + r) << 16;
    else
      rk[k >> 1] = before + r;
  }
  __syncthreads();
  // ---- per digit: the tile's count and each warp's offset inside the digit
  unsigned c = 0;
#pragma unroll
  for (int q = 0; q < kRWarps; q++) {
    const unsigned cq = wcnt[q][t];
    wcnt[q][t] = (unsigned short)c;
    c += cq;
  }
  if (tile == 0)
    atomicExch(&look[t], kLookPre | c);
  else
    atomicExch(&look[(size_t)tile * 256 + t], kLookAgg | c);
  unsigned x = c, g = hc;  // exclusive scans of the tile's and the global digit counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    const unsigned z = __shfl_up_sync(0xffffffffu, g, o);
    if (lane >= o) {
      x += y;
      g += z;
    }
  }
  if (lane == 31) {
    wsum[w] = x;
    gsum[w] = g;
  }
  __syncthreads();
  unsigned wb = 0, gb = 0;
  for (int q = 0; q < w; q++) {
    wb += wsum[q];
    gb += gsum[q];
  }
  tstart[t] = wb + x - c;
  const unsigned gstart = gb + g - hc;
  __syncthreads();
  // ---- stage the tile in digit order
#pragma unroll
  for (int k = 0; k < kOsItems; k++) {
    if (w * kWarpItems + k * 32 + lane < cnt_tile) {
      const unsigned d = (unsigned)(((key_is_hi ? (uint64_t)key_bucket(h[k]) : l[k]) >> shift) & 255u);
      const unsigned lp = tstart[d] + wcnt[w][d] + ((rk[k >> 1] >> ((k & 1) * 16)) & 0xffffu);
      s_hi[lp] = h[k];
      s_lo[lp] = l[k];
    }
  }
  // ---- look back for the tile's exclusive prefix in every digit bucket:
  // 16 predecessors per step are read at once (independent loads), so the
  // dependent chain is ~1/16 of the distance to the nearest inclusive prefix
  unsigned excl = 0;
  if (tile > 0) {
    constexpr int kLB = EMU_LOOKBACK;
    bool done = false;
    for (int64_t q0 = (int64_t)tile - 1; !done; q0 -= kLB) {
      unsigned v[kLB];
#pragma unroll
      for (int i = 0; i < kLB; i++)
        v[i] = q0 - i >= 0 ? *(volatile unsigned int*)&look[(size_t)(q0 - i) * 256 + t] : (2u << 30);  // before tile 0: prefix 0
#pragma unroll
      for (int i = 0; i < kLB; i++) {
        if (done) break;
        while ((v[i] & ~kLookVal) == 0) v[i] = *(volatile unsigned int*)&look[(size_t)(q0 - i) * 256 + t];
        excl += v[i] & kLookVal;
        done = (v[i] & ~kLookVal) == kLookPre;
      }
    }
    atomicExch(&look[(size_t)tile * 256 + t], kLookPre | (excl + c));
  }
  gofs[t] = gstart + excl;
  __syncthreads();
  // ---- write every digit's run of the tile out contiguously
  for (int j = t; j < cnt_tile; j += kRThreads) {
    const H hv = s_hi[j];
    const uint64_t lv = s_lo[j];
    const unsigned d = (unsigned)(((key_is_hi ? (uint64_t)key_bucket(hv) : lv) >> shift) & 255u);
    const unsigned pos = gofs[d] + (unsigned)j - tstart[d];
    b_hi[pos] = hv;
    b_lo[pos] = lv;
    if (hnext) atomicAdd(&nh[((nword ? (uint64_t)key_bucket(hv) : lv) >> nshift) & 255u], 1u);
  }
  if (hnext) {  // the next pass's histogram, counted on the way out
    __syncthreads();
    if (nh[t]) atomicAdd(&hnext[t], nh[t]);
  }
}

// Stable partition by the phase bit (hi's top bit): decode (0) records first.
template <typename H>
struct PhaseIn {
  const H* hi;
  __device__ uint32_t operator()(int64_t i) const { return key_phase(hi[i]) ? 0u : 1u; }
};
template <typename H>
struct PhaseOut {
  const H* hi;
  const uint64_t* lo;
  H* d_hi;
  uint64_t* d_lo;
  H* m_hi;
  uint64_t* m_lo;
  __device__ void operator()(int64_t i, uint32_t ex) const {
    if (key_phase(hi[i])) {
      const int64_t j = i - (int64_t)ex;
      m_hi[j] = hi[i];
      m_lo[j] = lo[i];
    } else {
      d_hi[ex] = hi[i];
      d_lo[ex] = lo[i];
    }
  }
};

// Segmenting a sorted run into buckets.
template <typename H>
struct HeadIn {
  const H* hi;
  __device__ uint32_t operator()(int64_t i) const {
    return (i == 0 || key_bucket(hi[i]) != key_bucket(hi[i - 1])) ? 1u : 0u;
  }
};
template <typename H>
struct HeadOut {
  const H* hi;
  const uint64_t* lo;
  int cbits;
  int32_t* bkt_tt;
  int32_t* bkt_conc;
  int64_t* bkt_off;
  double* samples;
  __device__ void operator()(int64_t i, uint32_t ex) const {
    const uint64_t h = (uint64_t)key_bucket(hi[i]);
    if (i == 0 || h != (uint64_t)key_bucket(hi[i - 1])) {
      bkt_tt[ex] = (int32_t)(h >> cbits) + 1;
      bkt_conc[ex] = (int32_t)(h & ((1ULL << cbits) - 1ULL)) + 1;
      bkt_off[ex] = i;
    }
    samples[i] = __longlong_as_double((long long)lo[i]);
  }
};

struct RowIn {
  const int32_t* tt;
  __device__ uint32_t operator()(int64_t b) const { return (b == 0 || tt[b] != tt[b - 1]) ? 1u : 0u; }
};
struct RowOut {
  const int32_t* tt;
  int32_t* row_tt;
  int64_t* row_start;
  __device__ void operator()(int64_t b, uint32_t ex) const {
    if (b == 0 || tt[b] != tt[b - 1]) {
      row_tt[ex] = tt[b];
      row_start[ex] = b;
    }
  }
};

__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

// Dense-domain segmentation: table j (0 decode, 1 mixed, 2 combined) over the
// key domain; a scan element packs (1 bucket << 32 | records) for a key with
// records, so one 64-bit exclusive scan gives each bucket's index and offset.
struct DenseIn {
  const unsigned int* c0;  // decode counts per key
  const unsigned int* c1;  // mixed counts per key
  int j;
  __device__ unsigned int cnt(int64_t k) const { return j == 0 ? c0[k] : j == 1 ? c1[k] : c0[k] + c1[k]; }
  __device__ uint64_t operator()(int64_t k) const {
    const unsigned int c = cnt(k);
    return c ? ((1ULL << 32) | c) : 0ULL;
  }
};
struct DenseOut {
  DenseIn in;
  int cbits;
  int32_t* bkt_tt;
  int32_t* bkt_conc;
  int64_t* bkt_off;
  unsigned int* koff;  // the key's first sample in this table (lsb builds), else null
  __device__ void operator()(int64_t k, uint64_t ex) const {
    if (!in.cnt(k)) return;
    if (koff) koff[k] = (unsigned int)(ex & 0xffffffffULL);
    const int64_t b = (int64_t)(ex >> 32);
    bkt_tt[b] = (int32_t)(k >> cbits) + 1;
    bkt_conc[b] = (int32_t)(k & ((1LL << cbits) - 1)) + 1;
    bkt_off[b] = (int64_t)(ex & 0xffffffffULL);
  }
};
// The samples of all three tables in one pass over the sorted records: the
// combined table is the sorted run, the phase tables its stable partition.
template <typename H>
struct SampleOut {
  const H* hi;
  const uint64_t* lo;
  double* comb;
  double* dec;
  double* mix;
  __device__ void operator()(int64_t i, uint32_t ex) const {
    const double v = __longlong_as_double((long long)lo[i]);
    comb[i] = v;
    if (key_phase(hi[i]))
      mix[i - (int64_t)ex] = v;
    else
      dec[ex] = v;
  }
};

// Samples of all three tables from a run sorted by (bucket key, phase,
// latency) -- canonical dense builds: a key's decode records then its mixed
// records, each ascending.  The phase tables take their sub-runs as they are;
// the combined bucket is the merge of the two (a record's place = its rank in
// its own sub-run + the count of the other sub-run's values below it, ties
// going to decode first -- equal values, so the order among them is moot).
__device__ __forceinline__ int64_t count_below(const uint64_t* __restrict__ a, int64_t m, uint64_t v, bool inclusive) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const uint64_t x = a[mid];
    if (x < v || (inclusive && x == v))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
template <typename H>
__global__ void __launch_bounds__(256) k_samples(const H* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n,
                                                 int kb, const unsigned int* __restrict__ dcnt,
                                                 const unsigned int* __restrict__ koff, double* __restrict__ dec,
                                                 double* __restrict__ mix, double* __restrict__ comb) {
  const int64_t K = 1LL << kb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = (uint64_t)hi[i], bits = lo[i];
    const int64_t k = (int64_t)(h >> 1);
    const int64_t s0 = koff[2 * K + k];  // the key's combined bucket = its run in the sorted records
    const int64_t na = dcnt[k], nb = dcnt[K + k];
    const double v = __longlong_as_double((long long)bits);
    int64_t pos;
    if (!(h & 1u)) {
      const int64_t r = i - s0;
      dec[koff[k] + r] = v;
      pos = s0 + r + (nb ? count_below(lo + s0 + na, nb, bits, false) : 0);
    } else {
      const int64_t r = i - s0 - na;
      mix[koff[K + k] + r] = v;
      pos = s0 + r + (na ? count_below(lo + s0, na, bits, true) : 0);
    }
    comb[pos] = v;
  }
}

// ---- key-first canonical builds (the default; EMU_BUILD_KF=0 turns it off):
// the records are sorted by (bucket key, phase) only (3 passes instead of 10);
// each (key, phase) sub-run is then sorted by latency on its own.  Runs of
// <= 256 records: one warp, bitonic sort held in registers; <= 4096: one CTA,
// value bins of ~32 records in shared memory, each sorted by a warp the same
// way; larger (the hot decode keys): split into bins of ~256 records (at most
// 4096 bins) by the value's place between the sub-run's min and max
// (monotone, so bins are ordered), scattered into place by two
// shared-memory-histogram passes, and each bin sorted like a run.  A bin over
// 4096 records (heavy ties, clustered values) sets a flag and the build falls
// back to the full passes.  C4: 9.6 ms against 10.7 for the full passes
// (128-record bins: 10.05 ms; 512 and 1024 overflow and fall back).
struct SegItem {
  int64_t start;  // first record of the run in the sorted-by-key order
  int32_t count;
  int32_t src1;   // 1: the run already sits in the output array (a bin), 0: read it from the key-sorted array
};
#ifndef EMU_SEG_BIN
#define EMU_SEG_BIN 256
#endif
#ifndef EMU_SEG_MAXBINS
#define EMU_SEG_MAXBINS 4096
#endif
constexpr int kSegSmall = 256, kSegMedium = 4096, kSegBin = EMU_SEG_BIN, kSegSmemBins = EMU_SEG_MAXBINS;
// bins of a large sub-run: ~kSegBin records each, at most kSegSmemBins (shared-memory counters)
__host__ __device__ __forceinline__ int64_t seg_nbins(int64_t c) {
  const int64_t nb = (c + kSegBin - 1) / kSegBin;
  return nb < kSegSmemBins ? nb : kSegSmemBins;
}
struct SegCtl {
  int n_small, n_medium, n_large, oversize;
  int next_small, next_medium;
  int pad[2];
};

__global__ void k_seg_classify(const unsigned int* __restrict__ dcnt, const unsigned int* __restrict__ comb_off,
                               int64_t K, const uint64_t* __restrict__ lo_in, uint64_t* __restrict__ lo_out,
                               SegItem* small, SegItem* medium, SegItem* large, SegCtl* ctl) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < 2 * K; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned c = dcnt[j];
    if (!c) continue;
    const int64_t k = j < K ? j : j - K;
    const int64_t st = (int64_t)comb_off[k] + (j < K ? 0 : (int64_t)dcnt[k]);
    if (c == 1) {
      lo_out[st] = lo_in[st];
      continue;
    }
    const SegItem it{st, (int32_t)c, 0};
    if (c <= (unsigned)kSegSmall)
      small[atomicAdd(&ctl->n_small, 1)] = it;
    else if (c <= (unsigned)kSegMedium)
      medium[atomicAdd(&ctl->n_medium, 1)] = it;
    else
      large[atomicAdd(&ctl->n_large, 1)] = it;
  }
}

// Per large sub-run: min and max of the latency bits (positive doubles order
// like their bit patterns); blockIdx.y = sub-run, blockIdx.x = chunk of it.
__global__ void __launch_bounds__(256) k_seg_minmax(const SegItem* __restrict__ large, const SegCtl* __restrict__ ctl,
                                                    const uint64_t* __restrict__ lo, unsigned long long* mn,
                                                    unsigned long long* mx) {
  for (int it = blockIdx.y; it < ctl->n_large; it += gridDim.y) {
    const SegItem g = large[it];
    unsigned long long a = ~0ULL, b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.count; i += (int64_t)gridDim.x * blockDim.x) {
      const unsigned long long v = lo[g.start + i];
      a = v < a ? v : a;
      b = v > b ? v : b;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o), y = __shfl_xor_sync(0xffffffffu, b, o);
      a = x < a ? x : a;
      b = y > b ? y : b;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&mn[it], a);
      atomicMax(&mx[it], b);
    }
  }
}

// Bin bases of the large sub-runs (one CTA: a handful of items).
__global__ void k_seg_binbase(const SegItem* __restrict__ large, const SegCtl* __restrict__ ctl,
                              int64_t* __restrict__ bbase, int64_t* total) {
  if (threadIdx.x != 0) return;
  int64_t acc = 0;
  for (int it = 0; it < ctl->n_large; it++) {
    bbase[it] = acc;
    acc += seg_nbins(large[it].count);
  }
  *total = acc;
}

// Value bins of a run with minimum a and maximum b (latency bits): bin =
// floor((v - a) * nb / (b - a)), the scale computed once per run.  Every step
// is a correctly rounded IEEE op of a non-decreasing argument, so the bin is
// monotone non-decreasing in v (bins are ordered).
struct SegScale {
  double a, k;  // min as a double, nb / (max - min)
  int64_t nb;
  bool flat;    // max == min (or an infinite max): everything in bin 0 / the last bin
  uint64_t b;
};
__device__ __forceinline__ SegScale seg_scale(uint64_t a, uint64_t b, int64_t nb) {
  SegScale s;
  s.a = __longlong_as_double((long long)a);
  const double r = __longlong_as_double((long long)b) - s.a;
  s.k = (double)nb / r;
  s.nb = nb;
  s.b = b;
  s.flat = !(r > 0.0) || !(s.k < 1e308);
  return s;
}
__device__ __forceinline__ int64_t seg_bin_of(uint64_t v, const SegScale& s) {
  if (s.flat) return v == s.b && s.b != (uint64_t)__double_as_longlong(s.a) ? s.nb - 1 : 0;
  const double x = (__longlong_as_double((long long)v) - s.a) * s.k;
  if (!(x >= 0.0)) return v == s.b ? s.nb - 1 : 0;  // an infinite maximum: inf - inf
  return x < (double)s.nb ? (int64_t)x : s.nb - 1;
}

// pass 0: count records per bin; pass 1: scatter them into place (bin order).
// blockIdx.y = sub-run, blockIdx.x = a contiguous chunk of it.  Sub-runs of
// count in shared memory and touch the global counters once per (CTA, bin);
// the chunk is read twice in pass 1 (count, then place: the second read hits L2).
template <int PASS>
__global__ void __launch_bounds__(256) k_seg_bins(const SegItem* __restrict__ large, const SegCtl* __restrict__ ctl,
                                                  const unsigned long long* __restrict__ mn,
                                                  const unsigned long long* __restrict__ mx,
                                                  const int64_t* __restrict__ bbase, const uint64_t* __restrict__ lo,
                                                  unsigned int* bcnt, const unsigned int* __restrict__ boff,
                                                  uint64_t* __restrict__ out) {
  extern __shared__ unsigned int sh[];  // [kSegSmemBins] counts, then [kSegSmemBins] bases
  for (int it = blockIdx.y; it < ctl->n_large; it += gridDim.y) {
    const SegItem g = large[it];
    const int64_t nb = seg_nbins(g.count), base = bbase[it];
    const SegScale sc = seg_scale(mn[it], mx[it], nb);
    const int64_t per = (g.count + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = min((int64_t)g.count, (int64_t)blockIdx.x * per), c1 = min((int64_t)g.count, c0 + per);
    unsigned int* cnt = sh;
    unsigned int* bas = sh + kSegSmemBins;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) cnt[q] = 0;
    __syncthreads();
    // four independent loads per thread in flight (the loop is latency-bound otherwise)
    for (int64_t i0 = c0 + threadIdx.x; i0 < c1; i0 += 4 * (int64_t)blockDim.x) {
      uint64_t v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t i = i0 + u * (int64_t)blockDim.x;
        v[u] = i < c1 ? lo[g.start + i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (i0 + u * (int64_t)blockDim.x < c1) atomicAdd(&cnt[seg_bin_of(v[u], sc)], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < nb; q += blockDim.x) {
      const unsigned c = cnt[q];
      if (PASS == 0) {
        if (c) atomicAdd(&bcnt[base + q], c);
      } else {
        bas[q] = c ? atomicAdd(&bcnt[base + q], c) + (boff[base + q] - boff[base]) : 0u;
        cnt[q] = 0;
      }
    }
    __syncthreads();
    if (PASS == 1) {
      for (int64_t i0 = c0 + threadIdx.x; i0 < c1; i0 += 4 * (int64_t)blockDim.x) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int64_t i = i0 + u * (int64_t)blockDim.x;
          v[u] = i < c1 ? lo[g.start + i] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (i0 + u * (int64_t)blockDim.x < c1) {
            const int q = (int)seg_bin_of(v[u], sc);
            out[g.start + (int64_t)bas[q] + atomicAdd(&cnt[q], 1u)] = v[u];
          }
      }
      __syncthreads();
    }
  }
}

// The bins of every large sub-run as sort items (their records already sit in
// the output array, in place).
__global__ void k_seg_binitems(const SegItem* __restrict__ large, const SegCtl* __restrict__ ctl_in,
                               const int64_t* __restrict__ bbase, const unsigned int* __restrict__ bcnt,
                               const unsigned int* __restrict__ boff, SegItem* small, SegItem* medium, SegCtl* ctl) {
  for (int it = blockIdx.y; it < ctl_in->n_large; it += gridDim.y) {
    const SegItem g = large[it];
    const int64_t nb = seg_nbins(g.count), base = bbase[it];
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nb; q += (int64_t)gridDim.x * blockDim.x) {
      const unsigned c = bcnt[base + q];
      if (c <= 1) continue;
      const SegItem b{g.start + (int64_t)(boff[base + q] - boff[base]), (int32_t)c, 1};
      if (c <= (unsigned)kSegSmall)
        small[atomicAdd(&ctl->n_small, 1)] = b;
      else if (c <= (unsigned)kSegMedium)
        medium[atomicAdd(&ctl->n_medium, 1)] = b;
      else
        atomicExch(&ctl->oversize, 1);
    }
  }
}

// One warp per run of <= kSegSmall records: bitonic sort held in registers
// (E consecutive elements per lane; partners in other lanes via shuffles,
// inside a lane via register swaps -- no shared memory, no syncs).
template <int E>
__device__ __forceinline__ void warp_bitonic_run(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst,
                                                 int64_t start, int n, int lane) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = lane * E + e;
    v[e] = i < n ? src[start + i] : ~0ULL;
  }
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lm = j / E;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; e++) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], lm);
          const bool up = ((lane * E + e) & k) == 0;
          const bool keep_min = lower == up;
          v[e] = keep_min ? (o < v[e] ? o : v[e]) : (o > v[e] ? o : v[e]);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; e++) {
          const int q = e ^ j;
          if (q > e) {
            const bool up = ((lane * E + e) & k) == 0;
            const uint64_t a = v[e], b = v[q];
            const bool sw = (a > b) == up;
            v[e] = sw ? b : a;
            v[q] = sw ? a : b;
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; e++) {
    const int i = lane * E + e;
    if (i < n) dst[start + i] = v[e];
  }
}

constexpr int kSegSmallWarps = 4;
__global__ void __launch_bounds__(32 * kSegSmallWarps) k_seg_sort_small(const SegItem* __restrict__ items, SegCtl* ctl,
                                                                       const uint64_t* __restrict__ lo_in,
                                                                       uint64_t* lo_out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n_items = ctl->n_small;
  for (int it = blockIdx.x * kSegSmallWarps + w; it < n_items; it += gridDim.x * kSegSmallWarps) {
    const SegItem g = items[it];
    const uint64_t* src = g.src1 ? lo_out : lo_in;
    // in place (src == dst) is safe: every lane holds its elements before any store
    if (g.count <= 32)
      warp_bitonic_run<1>(src, lo_out, g.start, g.count, lane);
    else if (g.count <= 64)
      warp_bitonic_run<2>(src, lo_out, g.start, g.count, lane);
    else if (g.count <= 128)
      warp_bitonic_run<4>(src, lo_out, g.start, g.count, lane);
    else
      warp_bitonic_run<8>(src, lo_out, g.start, g.count, lane);
  }
}

// One CTA per run of 257-4096 records: a bucket sort inside shared memory --
// split the run into ~24-record value bins (min/max-normalised, monotone), then
// each bin sorted by one warp with the register bitonic; a bin over 256
// records (ties, clustered values) sends the whole run to a shared-memory
// bitonic sort instead.  (Holding the run in registers instead of a second
// shared buffer, for 4 CTAs/SM instead of 3, measured slower: 3.1 vs 2.6 ms.)
#ifndef EMU_SEG_SUBT
#define EMU_SEG_SUBT 24
#endif
constexpr int kSegSub = 256;  // value bins per run at most (~EMU_SEG_SUBT records each)
__global__ void __launch_bounds__(256) k_seg_sort_medium(const SegItem* __restrict__ items, SegCtl* ctl,
                                                         const uint64_t* __restrict__ lo_in, uint64_t* lo_out) {
  extern __shared__ uint64_t sv[];  // [kSegMedium] the run, then [kSegMedium] the run in bin order
  uint64_t* sb = sv + kSegMedium;
  __shared__ unsigned int hist[kSegSub], cur[kSegSub], wtot[8];
  __shared__ unsigned long long rmn[8], rmx[8];
  __shared__ int big;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int n_items = ctl->n_medium;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const SegItem g = items[it];
    const uint64_t* src = g.src1 ? lo_out : lo_in;
    const int n = g.count;
    unsigned long long a = ~0ULL, b = 0;
    for (int i0 = t; i0 < n; i0 += 4 * blockDim.x) {
      uint64_t v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = i0 + u * (int)blockDim.x < n ? src[g.start + i0 + u * blockDim.x] : 0;
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (i0 + u * (int)blockDim.x < n) {
          sv[i0 + u * blockDim.x] = v[u];
          a = v[u] < a ? v[u] : a;
          b = v[u] > b ? v[u] : b;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, a, o), y = __shfl_xor_sync(0xffffffffu, b, o);
      a = x < a ? x : a;
      b = y > b ? y : b;
    }
    if (lane == 0) {
      rmn[w] = a;
      rmx[w] = b;
    }
    hist[t] = 0;
    if (t == 0) big = 0;
    __syncthreads();
    a = rmn[0];
    b = rmx[0];
#pragma unroll
    for (int q = 1; q < 8; q++) {
      a = rmn[q] < a ? rmn[q] : a;
      b = rmx[q] > b ? rmx[q] : b;
    }
    const int nsub = min(kSegSub, (n + EMU_SEG_SUBT - 1) / EMU_SEG_SUBT);
    const SegScale sc = seg_scale(a, b, nsub);
    for (int i = t; i < n; i += blockDim.x) atomicAdd(&hist[seg_bin_of(sv[i], sc)], 1u);
    __syncthreads();
    // exclusive scan of the bin counts (one per thread)
    const unsigned c = hist[t];
    unsigned x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    unsigned wb = 0;
    for (int q = 0; q < w; q++) wb += wtot[q];
    cur[t] = wb + x - c;
    if (c > 256) big = 1;
    __syncthreads();
    if (!big) {
      for (int i = t; i < n; i += blockDim.x) {
        const uint64_t v = sv[i];
        sb[atomicAdd(&cur[seg_bin_of(v, sc)], 1u)] = v;
      }
      __syncthreads();
      for (int q = w; q < nsub; q += 8) {  // cur[q] is now the end of bin q
        const int cq = (int)hist[q], s0 = (int)cur[q] - cq;
        if (cq <= 1) continue;
        if (cq <= 32)
          warp_bitonic_run<1>(sb, sb, s0, cq, lane);
        else if (cq <= 64)
          warp_bitonic_run<2>(sb, sb, s0, cq, lane);
        else if (cq <= 128)
          warp_bitonic_run<4>(sb, sb, s0, cq, lane);
        else
          warp_bitonic_run<8>(sb, sb, s0, cq, lane);
      }
      __syncthreads();
      for (int i = t; i < n; i += blockDim.x) lo_out[g.start + i] = sb[i];
    } else {  // a bin too big for one warp: bitonic sort of the whole run
      int P = 1;
      while (P < n) P <<= 1;
      for (int i = n + t; i < P; i += blockDim.x) sv[i] = ~0ULL;
      __syncthreads();
      for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = t; i < P; i += blockDim.x) {
            const int l = i ^ j;
            if (l > i) {
              const uint64_t p = sv[i], q = sv[l];
              if ((p > q) == ((i & k) == 0)) {
                sv[i] = q;
                sv[l] = p;
              }
            }
          }
          __syncthreads();
        }
      for (int i = t; i < n; i += blockDim.x) lo_out[g.start + i] = sv[i];
    }
    __syncthreads();
  }
}

__global__ void k_conc_range(const int32_t* c, int64_t n, int* mm) {
  int lo = 0x7fffffff, hi = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo = min(lo, c[i]);
    hi = max(hi, c[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}


static cudaError_t pool_alloc(void** p, size_t bytes, cudaStream_t s) { return table_alloc(p, bytes, s); }

// Build scratch (key arrays, sort buffers, look-back flags, staged host
// inputs) is bump-allocated from one persistent device buffer: no allocator
// calls inside a build, so its time does not depend on what the pool did
// last.  A build that needs more takes the excess from the pool and the
// buffer is regrown to the peak for the next one.  Builds hold g_build_mu
// (one at a time per process); emu_build_scratch_release frees the buffer.
struct BuildScratch {
  char* base = nullptr;
  size_t cap = 0, used = 0, peak = 0;
};
static BuildScratch g_scratch;
static std::mutex g_build_mu;

static cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s, std::vector<void*>* spill) {
  const size_t sz = ((bytes > 0 ? bytes : 1) + 255) & ~(size_t)255;
  g_scratch.peak = std::max(g_scratch.peak, g_scratch.used + sz);
  if (g_scratch.used + sz <= g_scratch.cap) {
    *p = g_scratch.base + g_scratch.used;
    g_scratch.used += sz;
    return cudaSuccess;
  }
  g_scratch.used += sz;
  const cudaError_t e = pool_alloc(p, sz, s);
  if (e == cudaSuccess) spill->push_back(*p);
  return e;
}

// After a build (stream synchronized): grow the buffer to the peak it needed.
static void scratch_settle() {
  if (g_scratch.peak > g_scratch.cap) {
    cudaFree(g_scratch.base);
    g_scratch.base = nullptr;
    g_scratch.cap = 0;
    const size_t want = g_scratch.peak + (g_scratch.peak >> 4);
    if (cudaMalloc((void**)&g_scratch.base, want) == cudaSuccess)
      g_scratch.cap = want;
    else
      cudaGetLastError();
  }
  g_scratch.used = 0;
  g_scratch.peak = 0;
}

// Table outputs (TableBuf::release returns them to the pool).
template <typename T>
static int palloc(cudaStream_t s, T** p, int64_t n) {
  *p = nullptr;
  EMU_CUDA(pool_alloc((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1), s));
  return EMU_OK;
}

static int grid_of(int64_t n, int threads, int cap) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

static int bits_for(int64_t maxval_minus1) {
  int b = 1;
  while (b < 62 && (maxval_minus1 >> b) != 0) b++;
  return b;
}

// Segment one sorted run of m records into a TableBuf.
static int segment_finish(TableBuf& tb, int64_t nb, int64_t m, unsigned int* partial, unsigned int* total_dev,
                          int* mm_dev, cudaStream_t s);

template <typename H>
static int segment(const H* hi, const uint64_t* lo, int64_t m, int cbits, unsigned int* partial,
                   unsigned int* total_dev, int* mm_dev, cudaStream_t s, TableBuf& tb) {
  tb = TableBuf();
  int rc;
  if (m == 0) {
    if ((rc = palloc(s, &tb.bkt_tt, 0)) || (rc = palloc(s, &tb.bkt_conc, 0)) || (rc = palloc(s, &tb.bkt_off, 1)) ||
        (rc = palloc(s, &tb.samples, 0)) || (rc = palloc(s, &tb.row_tt, 0)) || (rc = palloc(s, &tb.row_start, 1)))
      return rc;
    EMU_CUDA(cudaMemsetAsync(tb.bkt_off, 0, 8, s));
    EMU_CUDA(cudaMemsetAsync(tb.row_start, 0, 8, s));
    return EMU_OK;
  }
  // pass 1: count buckets
  EMU_CUDA(device_excl_scan<unsigned int>(HeadIn<H>{hi}, [] __device__(int64_t, unsigned int) {}, m, partial, total_dev, s));
  unsigned int nb_u = 0;
  EMU_CUDA(cudaMemcpyAsync(&nb_u, total_dev, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  const int64_t nb = nb_u;
  if ((rc = palloc(s, &tb.bkt_tt, nb)) || (rc = palloc(s, &tb.bkt_conc, nb)) || (rc = palloc(s, &tb.bkt_off, nb + 1)) ||
      (rc = palloc(s, &tb.samples, m)))
    return rc;
  HeadOut<H> ho{hi, lo, cbits, tb.bkt_tt, tb.bkt_conc, tb.bkt_off, tb.samples};
  EMU_CUDA(device_excl_scan<unsigned int>(HeadIn<H>{hi}, ho, m, partial, total_dev, s));
  EMU_CUDA(cudaMemcpyAsync(tb.bkt_off + nb, &m, 8, cudaMemcpyHostToDevice, s));
  return segment_finish(tb, nb, m, partial, total_dev, mm_dev, s);
}

// Rows (distinct tt), key ranges and the search index of a table whose bucket
// arrays and samples are written.
static int segment_finish(TableBuf& tb, int64_t nb, int64_t m, unsigned int* partial, unsigned int* total_dev,
                          int* mm_dev, cudaStream_t s) {
  int rc;
  // rows
  EMU_CUDA(device_excl_scan<unsigned int>(RowIn{tb.bkt_tt}, [] __device__(int64_t, unsigned int) {}, nb, partial,
                                          total_dev, s));
  unsigned int nr_u = 0;
  EMU_CUDA(cudaMemcpyAsync(&nr_u, total_dev, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  const int64_t nr = nr_u;
  if ((rc = palloc(s, &tb.row_tt, nr)) || (rc = palloc(s, &tb.row_start, nr + 1))) return rc;
  EMU_CUDA(device_excl_scan<unsigned int>(RowIn{tb.bkt_tt}, RowOut{tb.bkt_tt, tb.row_tt, tb.row_start}, nb, partial,
                                          total_dev, s));
  EMU_CUDA(cudaMemcpyAsync(tb.row_start + nr, &nb, 8, cudaMemcpyHostToDevice, s));
  // ranges
  int mm_init[2] = {0x7fffffff, 0};
  EMU_CUDA(cudaMemcpyAsync(mm_dev, mm_init, 8, cudaMemcpyHostToDevice, s));
  EMU_LAUNCH("conc_range", s, k_conc_range<<<grid_of(nb, 256, 1024), 256, 0, s>>>(tb.bkt_conc, nb, mm_dev));
  EMU_CUDA(cudaGetLastError());
  int mm[2];
  int32_t t0 = 0, t1 = 0;
  EMU_CUDA(cudaMemcpyAsync(mm, mm_dev, 8, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaMemcpyAsync(&t0, tb.bkt_tt, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaMemcpyAsync(&t1, tb.bkt_tt + nb - 1, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  tb.nb = nb;
  tb.ns = m;
  tb.nrows = nr;
  tb.tt_lo = t0;
  tb.tt_hi = t1;
  tb.c_lo = mm[0];
  tb.c_hi = mm[1];
  if (!index_on_host()) return build_search_index_dev(tb, s);
  std::vector<int32_t> htt((size_t)nb), hcc((size_t)nb);
  std::vector<int64_t> hoff((size_t)nb + 1);
  EMU_CUDA(cudaMemcpyAsync(htt.data(), tb.bkt_tt, 4 * nb, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaMemcpyAsync(hcc.data(), tb.bkt_conc, 4 * nb, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaMemcpyAsync(hoff.data(), tb.bkt_off, 8 * (nb + 1), cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  return build_search_index(tb, htt.data(), hcc.data(), hoff.data(), s);
}

// Scratch of the key-first latency sort (all null: the run is fully sorted).
struct SegScratch {
  uint64_t* lo_out = nullptr;  // the sorted latencies (k_samples reads them)
  SegItem *small = nullptr, *medium = nullptr, *large = nullptr;
  SegCtl* ctl = nullptr;
  uint64_t *mn = nullptr, *mx = nullptr;
  int64_t* bbase = nullptr;  // [cap_large + 1]: the last entry is the bin total
  unsigned int *bcnt = nullptr, *boff = nullptr;
  int64_t nbins_cap = 0;
};
constexpr int kSegFallback = 1000;  // a latency bin too big to sort in shared memory: redo with the full passes

// The three tables from the dense per-(phase, key) counts and the sorted
// records: one packed scan over the key domain per table (buckets, offsets),
// then every sample placed directly (canonical) or one scan over the records
// (capture order), then rows / ranges / index.

template <typename H>
static int segment_dense(const H* hi, const uint64_t* lo, int64_t n, int cbits, int kb, const unsigned int* dcnt,
                         uint64_t* part64, uint64_t* tot64, unsigned int* partial, unsigned int* total_dev,
                         int* mm_dev, cudaStream_t s, TableBuf* tab, unsigned int* koff, const SegScratch& sg) {
  const int64_t D = 1LL << kb;
  const int64_t np = (D + kScanTile - 1) / kScanTile + 1;
  int rc;
  for (int j = 0; j < 3; j++)
    EMU_CUDA(device_excl_scan<uint64_t>(DenseIn{dcnt, dcnt + D, j}, [] __device__(int64_t, uint64_t) {}, D,
                                        part64 + j * np, tot64 + j, s));
  uint64_t tot[3];
  EMU_CUDA(cudaMemcpyAsync(tot, tot64, sizeof(tot), cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  for (int j = 0; j < 3; j++) {
    TableBuf& tb = tab[j];
    tb = TableBuf();
    const int64_t nb = (int64_t)(tot[j] >> 32), m = (int64_t)(tot[j] & 0xffffffffULL);
    if ((rc = palloc(s, &tb.bkt_tt, nb)) || (rc = palloc(s, &tb.bkt_conc, nb)) ||
        (rc = palloc(s, &tb.bkt_off, nb + 1)) || (rc = palloc(s, &tb.samples, m)))
      return rc;
    EMU_CUDA(device_excl_scan<uint64_t>(DenseIn{dcnt, dcnt + D, j},
                                        DenseOut{DenseIn{dcnt, dcnt + D, j}, cbits, tb.bkt_tt, tb.bkt_conc, tb.bkt_off,
                                                 koff ? koff + j * D : nullptr},
                                        D, part64 + j * np, tot64 + j, s));
    int64_t* off_end = tb.bkt_off + nb;
    EMU_LAUNCH("fill_end", s, k_set_i64<<<1, 1, 0, s>>>(off_end, m));
  }
  if (sg.lo_out) {  // key-first: sort every (key, phase) sub-run by latency into sg.lo_out
    EMU_CUDA(cudaMemsetAsync(sg.ctl, 0, sizeof(SegCtl), s));
    EMU_LAUNCH("seg_classify", s, k_seg_classify<<<grid_of(2 * D, 256, kNumSMs * 16), 256, 0, s>>>(
                                      dcnt, koff + 2 * D, D, lo, sg.lo_out, sg.small, sg.medium, sg.large, sg.ctl));
    SegCtl hc;
    EMU_CUDA(cudaMemcpyAsync(&hc, sg.ctl, sizeof(hc), cudaMemcpyDeviceToHost, s));
    EMU_CUDA(cudaStreamSynchronize(s));
    if (hc.n_large > 0) {
      const unsigned gy = (unsigned)std::min(hc.n_large, 65535);
      EMU_CUDA(cudaMemsetAsync(sg.mn, 0xff, sizeof(uint64_t) * hc.n_large, s));
      EMU_CUDA(cudaMemsetAsync(sg.mx, 0, sizeof(uint64_t) * hc.n_large, s));
      const unsigned gm = (unsigned)std::max<int64_t>(1, std::min<int64_t>(256, (int64_t)kNumSMs * 16 / gy + 1));
      EMU_LAUNCH("seg_minmax", s, k_seg_minmax<<<dim3(gm, gy), 256, 0, s>>>(
                                      sg.large, sg.ctl, lo, (unsigned long long*)sg.mn, (unsigned long long*)sg.mx));
      EMU_LAUNCH("seg_binbase", s, k_seg_binbase<<<1, 32, 0, s>>>(sg.large, sg.ctl, sg.bbase, sg.bbase + hc.n_large));
      EMU_CUDA(cudaMemsetAsync(sg.bcnt, 0, sizeof(unsigned int) * sg.nbins_cap, s));
      const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(256, (int64_t)kNumSMs * 24 / gy + 1));
      const size_t bsm = 2 * kSegSmemBins * sizeof(unsigned int);
      EMU_CUDA(cudaFuncSetAttribute(k_seg_bins<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      EMU_CUDA(cudaFuncSetAttribute(k_seg_bins<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      EMU_LAUNCH("seg_bins", s, k_seg_bins<0><<<dim3(gx, gy), 256, bsm, s>>>(sg.large, sg.ctl, (unsigned long long*)sg.mn,
                                                                            (unsigned long long*)sg.mx, sg.bbase,
                                                                            lo, sg.bcnt, sg.boff, sg.lo_out));
      const unsigned int* bc = sg.bcnt;
      unsigned int* bo = sg.boff;
      EMU_CUDA(device_excl_scan<unsigned int>([bc] __device__(int64_t i) { return bc[i]; },
                                              [bo] __device__(int64_t i, unsigned int ex) { bo[i] = ex; },
                                              sg.nbins_cap, partial, total_dev, s));
      EMU_CUDA(cudaMemsetAsync(sg.bcnt, 0, sizeof(unsigned int) * sg.nbins_cap, s));
      EMU_LAUNCH("seg_bins", s, k_seg_bins<1><<<dim3(gx, gy), 256, bsm, s>>>(sg.large, sg.ctl, (unsigned long long*)sg.mn,
                                                                            (unsigned long long*)sg.mx, sg.bbase,
                                                                            lo, sg.bcnt, sg.boff, sg.lo_out));
      EMU_LAUNCH("seg_binitems", s, k_seg_binitems<<<dim3(16, gy), 256, 0, s>>>(sg.large, sg.ctl, sg.bbase, sg.bcnt,
                                                                                 sg.boff, sg.small, sg.medium, sg.ctl));
    }
    EMU_LAUNCH("seg_sort_small", s, k_seg_sort_small<<<kNumSMs * 12, 32 * kSegSmallWarps, 0, s>>>(sg.small, sg.ctl, lo,
                                                                                           sg.lo_out));
    EMU_CUDA(cudaFuncSetAttribute(k_seg_sort_medium, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(2 * kSegMedium * sizeof(uint64_t))));
    EMU_LAUNCH("seg_sort_medium", s, k_seg_sort_medium<<<kNumSMs * 3, 256, 2 * kSegMedium * sizeof(uint64_t), s>>>(
                                         sg.medium, sg.ctl, lo, sg.lo_out));
    EMU_CUDA(cudaMemcpyAsync(&hc, sg.ctl, sizeof(hc), cudaMemcpyDeviceToHost, s));
    EMU_CUDA(cudaStreamSynchronize(s));
    if (hc.oversize) return kSegFallback;
    lo = sg.lo_out;
  }
  if (koff)  // run sorted by (key, phase, latency): direct placement, no scan over the records
    EMU_LAUNCH("samples", s, k_samples<H><<<grid_of(n, 256, kNumSMs * 16), 256, 0, s>>>(
                                 hi, lo, n, kb, dcnt, koff, tab[0].samples, tab[1].samples, tab[2].samples));
  else
    EMU_CUDA(device_excl_scan<unsigned int>(PhaseIn<H>{hi},
                                            SampleOut<H>{hi, lo, tab[2].samples, tab[0].samples, tab[1].samples}, n,
                                            partial, total_dev, s));
  for (int j = 0; j < 3; j++) {
    const int64_t nb = (int64_t)(tot[j] >> 32), m = (int64_t)(tot[j] & 0xffffffffULL);
    if (nb == 0) {  // empty table (e.g. no mixed records): the shapes segment() gives it
      if ((rc = palloc(s, &tab[j].row_tt, 0)) || (rc = palloc(s, &tab[j].row_start, 1))) return rc;
      EMU_CUDA(cudaMemsetAsync(tab[j].row_start, 0, 8, s));
      continue;
    }
    if ((rc = segment_finish(tab[j], nb, m, partial, total_dev, mm_dev, s))) return rc;
  }
  return EMU_OK;
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace emu

namespace emu {

// Steps 2-5 of emu_tables_build for bucket keys of type H (uint32_t when
// (tt-1) << cbits | (conc-1) fits, else uint64_t).  Scratch comes from salloc
// (freed by the caller); the three tables are written to tab[0..2].
template <typename H>
static int sort_and_segment(const RecIn& r, int64_t n, bool canonical, int cbits, int tbits, cudaStream_t s,
                            TableBuf* tab, const std::function<int(void**, size_t)>& alloc, unsigned int* total_dev,
                            int* small, const std::function<void(const char*)>& mark, bool allow_kf = true) {
  int rc;
  auto salloc = [&](auto** p, int64_t count) -> int {
    return alloc(reinterpret_cast<void**>(p), sizeof(**p) * (size_t)(count > 0 ? count : 1));
  };
  H *hi0, *hi1;
  uint64_t *lo0, *lo1;
  unsigned int *counts = nullptr, *hist = nullptr, *partial = nullptr, *look = nullptr,
               *tile_ctr = nullptr;
  const int64_t nblk = (n + kRTile - 1) / kRTile, nos = (n + kOsTile - 1) / kOsTile;
  // EMU_ONESWEEP=0 (64-bit keys only): the up-sweep + scan + scatter passes instead
  const char* os_env = getenv("EMU_ONESWEEP");
  const bool onesweep = n < (1LL << 30) && !(os_env && os_env[0] == '0' && sizeof(H) == 8);
  const int64_t ncount = onesweep ? 1 : 256 * nblk;
  const int64_t npart = std::max<int64_t>((ncount + kScanTile - 1) / kScanTile, (n + kScanTile - 1) / kScanTile) + 1;
  if ((rc = salloc(&hi0, n)) || (rc = salloc(&lo0, n)) || (rc = salloc(&hi1, n)) || (rc = salloc(&lo1, n)) ||
      (rc = salloc(&counts, ncount)) || (rc = salloc(&hist, 17 * 256 + 4)) || (rc = salloc(&partial, npart)) ||
      (rc = salloc(&look, onesweep ? 256 * nos : 1)) ||
      (rc = salloc(&tile_ctr, 16)))
    return rc;
  // key domains up to 2^24 per phase: dense counts -> segment_dense (no scans over the records)
  const int kb = tbits + cbits;
  const bool dense = kb <= 24 && getenv("EMU_DENSE_SEGMENT") == nullptr;
  const int64_t D = dense ? (1LL << kb) : 0;
  const int64_t np64 = (D + kScanTile - 1) / kScanTile + 1;
  unsigned int *dcnt = nullptr, *koff = nullptr;
  uint64_t *part64 = nullptr, *tot64 = nullptr;
  // canonical dense builds sort the phase as the lowest key bit (decode before
  // mixed inside a key) and place every sample directly (k_samples)
  const int lsb = canonical && dense && getenv("EMU_PHASE_SCAN") == nullptr ? 1 : 0;
  // key-first (canonical dense builds): sort by (key, phase) only, then each
  // sub-run by latency on chip (EMU_BUILD_KF=0: the full latency passes instead)
  static const bool kf_env = [] {
    const char* e = getenv("EMU_BUILD_KF");
    return !(e && e[0] == '0');
  }();
  const bool kf = lsb && allow_kf && kf_env;
  SegScratch sg;
  if (dense) {
    if ((rc = salloc(&dcnt, 2 * D)) || (rc = salloc(&part64, 3 * np64)) || (rc = salloc(&tot64, 4))) return rc;
    if (lsb && (rc = salloc(&koff, 3 * D))) return rc;
    EMU_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(unsigned int) * 2 * D, s));
  }
  if (kf) {
    const int64_t runs = std::min<int64_t>(2 * D, n), cap_large = n / kSegMedium + 1;
    sg.nbins_cap = n / kSegBin + cap_large + 1;
    if ((rc = salloc(&sg.lo_out, n)) || (rc = salloc(&sg.small, runs + sg.nbins_cap)) ||
        (rc = salloc(&sg.medium, runs + sg.nbins_cap)) || (rc = salloc(&sg.large, cap_large)) ||
        (rc = salloc(&sg.ctl, 1)) || (rc = salloc(&sg.mn, cap_large)) || (rc = salloc(&sg.mx, cap_large)) ||
        (rc = salloc(&sg.bbase, cap_large + 1)) || (rc = salloc(&sg.bcnt, sg.nbins_cap)) ||
        (rc = salloc(&sg.boff, sg.nbins_cap)))
      return rc;
  }
  // keys, the differing bits and the first digit's histogram; then the passes
  // are the digit positions in which some record differs from record 0
  const int hword0 = canonical && !kf ? 0 : 1;
  EMU_CUDA(cudaMemsetAsync(hist, 0, 4 * 17 * 256 + 16, s));  // hist[17][256], then diff[2]
  unsigned long long* diff = reinterpret_cast<unsigned long long*>(hist + 17 * 256);
  EMU_LAUNCH("make_keys", s,
             k_make_keys<H><<<grid_of(n, 256, kNumSMs * 8), 256, 0, s>>>(r, cbits, lsb, hi0, lo0, hword0, 0, hist, diff));
  unsigned long long dh[2];
  EMU_CUDA(cudaMemcpyAsync(dh, diff, 16, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  PassSet ps{};
  if (canonical && !kf)
    for (int sft = 0; sft < 64; sft += 8)
      if ((dh[0] >> sft) & 255u) {
        ps.word[ps.n] = 0;
        ps.shift[ps.n++] = sft;
      }
  for (int sft = 0; sft < tbits + cbits + lsb; sft += 8)
    if ((dh[1] >> sft) & 255u) {
      ps.word[ps.n] = 1;
      ps.shift[ps.n++] = sft;
    }
  if (ps.n > 0 && (ps.word[0] != hword0 || ps.shift[0] != 0)) {  // the guessed first digit never varies
    EMU_CUDA(cudaMemsetAsync(hist, 0, 4 * 256, s));
    EMU_LAUNCH("digit_hist1", s, k_digit_hist1<H><<<grid_of(n, 256, kNumSMs * 8), 256, 0, s>>>(
                                     hi0, lo0, n, ps.word[0], ps.shift[0], hist));
  }
  EMU_CUDA(cudaMemsetAsync(tile_ctr, 0, 4 * 16, s));
  mark("keys+hist");
  // LSD passes
  const size_t osmem = (size_t)kOsTile * (8 + sizeof(H));
  if (onesweep) {
    EMU_CUDA(cudaFuncSetAttribute(k_onesweep<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)osmem));
  } else {
    EMU_CUDA(cudaFuncSetAttribute(k_radix_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kRSmem));
  }
  for (int p = 0; p < ps.n; p++) {
    if (onesweep) {
      EMU_CUDA(cudaMemsetAsync(look, 0, sizeof(unsigned int) * 256 * nos, s));
      EMU_LAUNCH("onesweep", s, k_onesweep<H><<<(unsigned)nos, kRThreads, osmem, s>>>(
                                    hi0, lo0, hi1, lo1, n, ps.shift[p], ps.word[p], hist + p * 256, look, tile_ctr + p,
                                    p + 1 < ps.n ? hist + (p + 1) * 256 : nullptr, ps.shift[p + 1], ps.word[p + 1]));
    } else {
      if constexpr (std::is_same<H, uint64_t>::value) {
        const uint64_t* key = ps.word[p] ? hi0 : lo0;
        EMU_LAUNCH("radix_up", s, k_radix_up<<<(unsigned)nblk, kRThreads, 0, s>>>(key, ps.word[p] ? ~(1ULL << 63) : ~0ULL, ps.shift[p], n, nblk, counts));
        EMU_CUDA(device_excl_scan<unsigned int>(
            [counts] __device__(int64_t i) { return counts[i]; },
            [counts] __device__(int64_t i, unsigned int ex) { counts[i] = ex; }, ncount, partial, total_dev, s));
        EMU_LAUNCH("radix_scatter", s, k_radix_scatter<<<(unsigned)nblk, kRThreads, kRSmem, s>>>(
                                           key, ps.shift[p], ps.word[p], hi0, lo0, hi1, lo1, n, nblk, counts));
      } else {
        return fail(EMU_ERR_INVALID, "internal: 32-bit keys need the onesweep sort");
      }
    }
    std::swap(hi0, hi1);
    std::swap(lo0, lo1);
  }
  EMU_CUDA(cudaGetLastError());
  mark("radix sort");
  if (dense) {
    EMU_LAUNCH("dense_count", s, k_dense_count<H><<<grid_of(n, 256, kNumSMs * 16), 256, 0, s>>>(hi0, lo0, n, kb, lsb, dcnt));
    rc = segment_dense<H>(hi0, lo0, n, cbits, kb, dcnt, part64, tot64, partial, total_dev, small + 2, s, tab, koff,
                          sg);
    mark("segment (dense)");
    if (rc == kSegFallback) {  // a latency bin over 4096 records: the full LSD passes instead
      for (int j = 0; j < 3; j++) tab[j].release();
      return sort_and_segment<H>(r, n, canonical, cbits, tbits, s, tab, alloc, total_dev, small, mark, false);
    }
    return rc;
  }
  // combined table = sorted run; decode/mixed = stable partition by phase
  if ((rc = segment<H>(hi0, lo0, n, cbits, partial, total_dev, small + 2, s, tab[2]))) return rc;
  mark("segment combined");
  EMU_CUDA(device_excl_scan<unsigned int>(PhaseIn<H>{hi0}, [] __device__(int64_t, unsigned int) {}, n, partial,
                                          total_dev, s));
  unsigned int n_dec = 0;
  EMU_CUDA(cudaMemcpyAsync(&n_dec, total_dev, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  EMU_CUDA(device_excl_scan<unsigned int>(PhaseIn<H>{hi0}, PhaseOut<H>{hi0, lo0, hi1, lo1, hi1 + n_dec, lo1 + n_dec}, n,
                                          partial, total_dev, s));
  mark("phase partition");
  if ((rc = segment<H>(hi1, lo1, n_dec, cbits, partial, total_dev, small + 2, s, tab[0]))) return rc;
  mark("segment decode");
  return segment<H>(hi1 + n_dec, lo1 + n_dec, n - n_dec, cbits, partial, total_dev, small + 2, s, tab[1]);
}

}  // namespace emu

using namespace emu;

extern "C" int emu_tables_build(const int32_t* tt, const int32_t* conc, const uint8_t* phase, const double* lat,
                                const int64_t* step, int64_t n, int canonical, void* stream, emu_tables_t* out,
                                int64_t* bad_index, int32_t* bad_code) {
  if (!out) return fail(EMU_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (bad_index) *bad_index = -1;
  if (bad_code) *bad_code = 0;
  if (n < 0) return fail(EMU_ERR_INVALID, "negative record count");
  if (n >= (1LL << 31)) return fail(EMU_ERR_INVALID, "record count must be < 2^31 per build");
  cudaStream_t s = as_stream(stream);
  static const bool trace = getenv("EMU_BUILD_TRACE") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    fprintf(stderr, "[emu build] %-24s %8.3f ms\n", what, ms);
  };
  std::lock_guard<std::mutex> build_lock(g_build_mu);
  g_scratch.used = 0;
  g_scratch.peak = 0;
  // Stage host inputs on the device (device inputs are used in place).
  std::vector<void*> owned;  // scratch that did not fit the persistent buffer
  auto stage = [&](const void* src, size_t bytes, const void** dst) -> int {
    if (!src || bytes == 0 || is_device_ptr(src)) {
      *dst = src;
      return EMU_OK;
    }
    void* d = nullptr;
    EMU_CUDA(scratch_alloc(&d, bytes, s, &owned));
    EMU_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
    *dst = d;
    return EMU_OK;
  };
  auto free_owned = [&]() {
    for (void* p : owned) cudaFreeAsync(p, s);
    owned.clear();
    if (cudaStreamSynchronize(s) == cudaSuccess) scratch_settle();
  };
  auto salloc = [&](auto** p, int64_t count) -> int {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(p)>>;
    *p = nullptr;
    void* q = nullptr;
    EMU_CUDA(scratch_alloc(&q, sizeof(**p) * (size_t)(count > 0 ? count : 1), s, &owned));
    *p = (decltype(*p))q;
    (void)sizeof(T);
    return EMU_OK;
  };
  RecIn r{};
  r.n = n;
  int rc;
  if ((rc = stage(tt, 4 * n, (const void**)&r.tt)) || (rc = stage(conc, 4 * n, (const void**)&r.conc)) ||
      (rc = stage(phase, n, (const void**)&r.ph)) || (rc = stage(lat, 8 * n, (const void**)&r.lat)) ||
      (rc = stage(step, step ? 8 * n : 0, (const void**)&r.step))) {
    free_owned();
    return rc;
  }
  unsigned long long* first_bad = nullptr;
  int* small = nullptr;  // maxv[2], mm[2]
  unsigned int* total_dev = nullptr;
  if ((rc = salloc(&first_bad, 1)) || (rc = salloc(&small, 4)) || (rc = salloc(&total_dev, 2))) {
    free_owned();
    return rc;
  }
  auto* t = new emu_tables_s();
  auto bail = [&](int code) {
    for (int j = 0; j < 3; j++) t->tab[j].release();
    delete t;
    free_owned();
    return code;
  };
  if (n == 0) {
    for (int j = 0; j < 3; j++)
      if ((rc = segment<uint64_t>(nullptr, nullptr, 0, 1, nullptr, nullptr, nullptr, s, t->tab[j]))) return bail(rc);
    if (cudaStreamSynchronize(s) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "build sync"));
    free_owned();
    *out = t;
    return EMU_OK;
  }
  // 1. validate
  unsigned long long fb_init = ~0ULL;
  int mv_init[2] = {0, 0};
  if (cudaMemcpyAsync(first_bad, &fb_init, 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(small, mv_init, 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "build init"));
  EMU_LAUNCH("validate", s, k_validate<<<grid_of(n, 256, kNumSMs * 16), 256, 0, s>>>(r, first_bad, small));
  unsigned long long fb = 0;
  int mv[2];
  if (cudaMemcpyAsync(&fb, first_bad, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(mv, small, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "k_validate"));
  if (fb != ~0ULL) {
    if (bad_index) *bad_index = (int64_t)(fb >> 3);
    if (bad_code) *bad_code = (int32_t)(fb & 7);
    bail(0);
    return fail(EMU_ERR_INVALID, "trace record " + std::to_string(fb >> 3) + " failed validation check " +
                                     std::to_string(fb & 7));
  }
  mark("validate");
  const int cbits = bits_for((int64_t)mv[1] - 1);
  const int tbits = bits_for((int64_t)mv[0] - 1);
  // 2.-5. keys, sort, partition, segment: 32-bit bucket keys when they fit
  const std::function<int(void**, size_t)> alloc_fn = [&](void** p, size_t bytes) -> int {
    *p = nullptr;
    EMU_CUDA(scratch_alloc(p, bytes, s, &owned));
    return EMU_OK;
  };
  const std::function<void(const char*)> mark_fn = mark;
  if (tbits + cbits <= 31 && n < (1LL << 30))  // bit 31 carries the phase
    rc = sort_and_segment<uint32_t>(r, n, canonical != 0, cbits, tbits, s, t->tab, alloc_fn, total_dev, small, mark_fn);
  else
    rc = sort_and_segment<uint64_t>(r, n, canonical != 0, cbits, tbits, s, t->tab, alloc_fn, total_dev, small, mark_fn);
  if (rc) return bail(rc);
  if (cudaStreamSynchronize(s) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "build"));
  mark("segment mixed");
  free_owned();
  mark("free");
  *out = t;
  return EMU_OK;
}

extern "C" int emu_build_scratch_release(void) {
  std::lock_guard<std::mutex> lk(g_build_mu);
  EMU_CUDA(cudaFree(g_scratch.base));
  g_scratch = BuildScratch();
  return EMU_OK;
}
