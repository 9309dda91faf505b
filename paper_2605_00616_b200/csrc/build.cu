// build.cu -- offline profile-table build on the GPU (emu_tables_build).
//
// Replaces build_pack (profile.py:230-267), PhaseTable.from_buckets
// (profile.py:122-129) and, in canonical mode, save_pack's ascending sample
// order (profile.py:281-282):
//   1. k_validate   : StepTraceRecord.validate per record (profile.py:61-79);
//                     smallest failing index wins (build_pack reports the first).
//   2. k_make_keys  : hi = (tt-1) << cbits | (conc-1), lo = lat_bits << 1 | phase
//                     (positive doubles order like their IEEE bit patterns).
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

__global__ void k_validate(RecIn r, unsigned long long* first_bad, int* maxv) {
  int mt = 0, mc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = r.tt[i], c = r.conc[i];
    const double l = r.lat[i];
    int code = 0;
    if (r.step && r.step[i] < 0)
      code = 1;
    else if (t < 1)
      code = 2;
    else if (c < 1)
      code = 3;
    else if (r.ph[i] == 0 && t < c)
      code = 4;
    else if (!(l > 0.0))
      code = 5;
    if (code) atomicMin(first_bad, ((unsigned long long)i << 3) | (unsigned long long)code);
    mt = max(mt, t);
    mc = max(mc, c);
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

__global__ void k_make_keys(RecIn r, int cbits, uint64_t* __restrict__ hi, uint64_t* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r.n; i += (int64_t)gridDim.x * blockDim.x) {
    hi[i] = ((uint64_t)(uint32_t)(r.tt[i] - 1) << cbits) | (uint64_t)(uint32_t)(r.conc[i] - 1);
    lo[i] = ((uint64_t)__double_as_longlong(r.lat[i]) << 1) | (r.ph[i] ? 1ULL : 0ULL);
  }
}

struct PassSet {
  int n;
  int word[16];  // 0 = lo, 1 = hi
  int shift[16];
};

// Histograms of every candidate digit position in one read of the keys.
__global__ void k_digit_hist(const uint64_t* __restrict__ hi, const uint64_t* __restrict__ lo, int64_t n, PassSet ps,
                             unsigned int* hist) {
  extern __shared__ unsigned int sh[];
  for (int i = threadIdx.x; i < ps.n * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = hi[i], l = lo[i];
    for (int p = 0; p < ps.n; p++) {
      const uint64_t w = ps.word[p] ? h : l;
      atomicAdd(&sh[p * 256 + (int)((w >> ps.shift[p]) & 255u)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ps.n * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void __launch_bounds__(kRThreads) k_radix_up(const uint64_t* __restrict__ key, int shift, int64_t n,
                                                       int64_t nblk, unsigned int* counts) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRTile;
#pragma unroll 4
  for (int k = 0; k < kRRounds; k++) {
    const int64_t i = base + (int64_t)k * kRThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 255u], 1u);
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
    const unsigned d = valid ? (unsigned)(((key_is_hi ? h : l) >> shift) & 255u) : 256u + (unsigned)lane;
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
    const unsigned d = (unsigned)(((key_is_hi ? h : l) >> shift) & 255u);
    const unsigned pos = gofs[d] + (unsigned)j - tstart[d];
    b_hi[pos] = h;
    b_lo[pos] = l;
  }
}

// Stable partition by phase bit (lo & 1): decode (0) records first.
struct PhaseIn {
  const uint64_t* lo;
  __device__ uint32_t operator()(int64_t i) const { return (lo[i] & 1ULL) ? 0u : 1u; }
};
struct PhaseOut {
  const uint64_t* hi;
  const uint64_t* lo;
  uint64_t* d_hi;
  uint64_t* d_lo;
  uint64_t* m_hi;
  uint64_t* m_lo;
  __device__ void operator()(int64_t i, uint32_t ex) const {
    if (lo[i] & 1ULL) {
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
struct HeadIn {
  const uint64_t* hi;
  __device__ uint32_t operator()(int64_t i) const { return (i == 0 || hi[i] != hi[i - 1]) ? 1u : 0u; }
};
struct HeadOut {
  const uint64_t* hi;
  const uint64_t* lo;
  int cbits;
  int32_t* bkt_tt;
  int32_t* bkt_conc;
  int64_t* bkt_off;
  double* samples;
  __device__ void operator()(int64_t i, uint32_t ex) const {
    const uint64_t h = hi[i];
    if (i == 0 || h != hi[i - 1]) {
      bkt_tt[ex] = (int32_t)(h >> cbits) + 1;
      bkt_conc[ex] = (int32_t)(h & ((1ULL << cbits) - 1ULL)) + 1;
      bkt_off[ex] = i;
    }
    samples[i] = __longlong_as_double((long long)(lo[i] >> 1));
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


// Build scratch comes from the device's stream-ordered memory pool, kept
// reserved between builds (release threshold = max): repeated builds reuse it
// instead of mapping and unmapping GBs with cudaMalloc / cudaFree.
static cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static bool pool_set = false;
  if (!pool_set) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  return cudaMallocAsync(p, bytes > 0 ? bytes : 1, s);
}

// Table outputs from the same pool (TableBuf::release frees them with cudaFree).
template <typename T>
static int palloc(cudaStream_t s, T** p, int64_t n) {
  *p = nullptr;
  EMU_CUDA(scratch_alloc((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1), s));
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
static int segment(const uint64_t* hi, const uint64_t* lo, int64_t m, int cbits, unsigned int* partial,
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
  EMU_CUDA(device_excl_scan<unsigned int>(HeadIn{hi}, [] __device__(int64_t, unsigned int) {}, m, partial, total_dev, s));
  unsigned int nb_u = 0;
  EMU_CUDA(cudaMemcpyAsync(&nb_u, total_dev, 4, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  const int64_t nb = nb_u;
  if ((rc = palloc(s, &tb.bkt_tt, nb)) || (rc = palloc(s, &tb.bkt_conc, nb)) || (rc = palloc(s, &tb.bkt_off, nb + 1)) ||
      (rc = palloc(s, &tb.samples, m)))
    return rc;
  HeadOut ho{hi, lo, cbits, tb.bkt_tt, tb.bkt_conc, tb.bkt_off, tb.samples};
  EMU_CUDA(device_excl_scan<unsigned int>(HeadIn{hi}, ho, m, partial, total_dev, s));
  EMU_CUDA(cudaMemcpyAsync(tb.bkt_off + nb, &m, 8, cudaMemcpyHostToDevice, s));
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
  // Stage host inputs on the device (device inputs are used in place).
  std::vector<void*> owned;
  auto stage = [&](const void* src, size_t bytes, const void** dst) -> int {
    if (!src || bytes == 0 || is_device_ptr(src)) {
      *dst = src;
      return EMU_OK;
    }
    void* d = nullptr;
    EMU_CUDA(scratch_alloc(&d, bytes, s));
    owned.push_back(d);
    EMU_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
    *dst = d;
    return EMU_OK;
  };
  auto free_owned = [&]() {
    for (void* p : owned) cudaFreeAsync(p, s);
    owned.clear();
  };
  auto salloc = [&](auto** p, int64_t count) -> int {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(p)>>;
    *p = nullptr;
    void* q = nullptr;
    EMU_CUDA(scratch_alloc(&q, sizeof(**p) * (size_t)(count > 0 ? count : 1), s));
    *p = (decltype(*p))q;
    owned.push_back(q);
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
      if ((rc = segment(nullptr, nullptr, 0, 1, nullptr, nullptr, nullptr, s, t->tab[j]))) return bail(rc);
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
  // 2. keys (double buffered)
  uint64_t *hi0, *lo0, *hi1, *lo1;
  unsigned int *counts = nullptr, *hist = nullptr, *partial = nullptr;
  const int64_t nblk = (n + kRTile - 1) / kRTile;
  const int64_t ncount = 256 * nblk;
  const int64_t npart = std::max<int64_t>((ncount + kScanTile - 1) / kScanTile, (n + kScanTile - 1) / kScanTile) + 1;
  if ((rc = salloc(&hi0, n)) || (rc = salloc(&lo0, n)) || (rc = salloc(&hi1, n)) || (rc = salloc(&lo1, n)) ||
      (rc = salloc(&counts, ncount)) || (rc = salloc(&hist, 16 * 256)) || (rc = salloc(&partial, npart)))
    return bail(rc);
  EMU_LAUNCH("make_keys", s, k_make_keys<<<grid_of(n, 256, kNumSMs * 16), 256, 0, s>>>(r, cbits, hi0, lo0));
  // 3. which digit positions actually vary
  PassSet ps{};
  if (canonical)
    for (int sft = 0; sft < 64; sft += 8) {
      ps.word[ps.n] = 0;
      ps.shift[ps.n++] = sft;
    }
  for (int sft = 0; sft < tbits + cbits; sft += 8) {
    ps.word[ps.n] = 1;
    ps.shift[ps.n++] = sft;
  }
  if (cudaMemsetAsync(hist, 0, 4 * 16 * 256, s) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "memset"));
  EMU_LAUNCH("digit_hist", s, k_digit_hist<<<grid_of(n, 256, kNumSMs * 4), 256, ps.n * 256 * 4, s>>>(hi0, lo0, n, ps, hist));
  std::vector<unsigned int> hh(16 * 256);
  if (cudaMemcpyAsync(hh.data(), hist, 4 * 16 * 256, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "k_digit_hist"));
  mark("keys+hist");
  // 4. LSD passes
  if (cudaFuncSetAttribute(k_radix_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kRSmem) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "radix smem attribute"));
  for (int p = 0; p < ps.n; p++) {
    unsigned int mx = *std::max_element(hh.begin() + p * 256, hh.begin() + (p + 1) * 256);
    if ((int64_t)mx == n) continue;  // all records share this digit: pass is the identity
    const uint64_t* key = ps.word[p] ? hi0 : lo0;
    EMU_LAUNCH("radix_up", s, k_radix_up<<<(unsigned)nblk, kRThreads, 0, s>>>(key, ps.shift[p], n, nblk, counts));
    cudaError_t e = device_excl_scan<unsigned int>(
        [counts] __device__(int64_t i) { return counts[i]; },
        [counts] __device__(int64_t i, unsigned int ex) { counts[i] = ex; }, ncount, partial, total_dev, s);
    if (e != cudaSuccess) return bail(cuda_fail(e, "radix scan"));
    EMU_LAUNCH("radix_scatter", s, k_radix_scatter<<<(unsigned)nblk, kRThreads, kRSmem, s>>>(
                                       key, ps.shift[p], ps.word[p], hi0, lo0, hi1, lo1, n, nblk, counts));
    std::swap(hi0, hi1);
    std::swap(lo0, lo1);
  }
  if (cudaGetLastError() != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "radix sort"));
  mark("radix sort");
  // 5. combined table = sorted run; decode/mixed = stable partition by phase
  if ((rc = segment(hi0, lo0, n, cbits, partial, total_dev, small + 2, s, t->tab[2]))) return bail(rc);
  mark("segment combined");
  cudaError_t e = device_excl_scan<unsigned int>(PhaseIn{lo0}, [] __device__(int64_t, unsigned int) {}, n, partial,
                                                 total_dev, s);
  if (e != cudaSuccess) return bail(cuda_fail(e, "phase partition count"));
  unsigned int n_dec = 0;
  if (cudaMemcpyAsync(&n_dec, total_dev, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "phase partition"));
  e = device_excl_scan<unsigned int>(PhaseIn{lo0}, PhaseOut{hi0, lo0, hi1, lo1, hi1 + n_dec, lo1 + n_dec}, n, partial,
                                     total_dev, s);
  if (e != cudaSuccess) return bail(cuda_fail(e, "phase partition"));
  mark("phase partition");
  if ((rc = segment(hi1, lo1, n_dec, cbits, partial, total_dev, small + 2, s, t->tab[0]))) return bail(rc);
  mark("segment decode");
  if ((rc = segment(hi1 + n_dec, lo1 + n_dec, n - n_dec, cbits, partial, total_dev, small + 2, s, t->tab[1])))
    return bail(rc);
  if (cudaStreamSynchronize(s) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "build"));
  mark("segment mixed");
  free_owned();
  mark("free");
  *out = t;
  return EMU_OK;
}
