// emu_internal.cuh -- shared device code of libemu_b200 (sm_100a).
//
// Bit-exactness rules:
//  * every float64 op on the oracle path is an explicit IEEE round-to-nearest
//    intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn) and the library is
//    compiled with -fmad=false, so no FMA contraction can change a distance,
//    weight or CDF bit relative to numpy (oracle.py:92-97, :124-127, :133);
//  * reductions whose order numpy fixes (pairwise sum, sequential cumsum) are
//    executed in exactly numpy's order by one thread.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/emu_abi.h"

namespace emu {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define EMU_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::emu::cuda_fail(_e, #call); \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

// ------------------------------------------------------------------ tables
// Kernel-side view of one canonical table (buckets sorted by (tt, conc)).
struct DevTable {
  const int32_t* bkt_tt;
  const int32_t* bkt_conc;
  const int64_t* bkt_off;
  const double* samples;
  const int32_t* row_tt;     // distinct tt, ascending
  const int64_t* row_start;  // nrows + 1
  int64_t nb, ns, nrows;
  int32_t tt_lo, tt_hi, c_lo, c_hi;
  // Summed-area tables over the dense key grid (tt - tt_lo, conc - c_lo):
  // bsat/ssat[(i)*(gnc+1) + j] = buckets / samples with tt index < i and conc
  // index < j.  gnt = gnc = 0 when the grid would be too large (fallback search).
  const int32_t* bsat;
  const int32_t* ssat;
  int64_t gnt, gnc;
  // Occupancy bitmap of the same grid: row i, word k holds conc indices
  // 32k..32k+31 (bit set = bucket exists); wpre = set bits in earlier words of
  // the row; rowbase[i] = first bucket of tt index i.  wpr words per row.
  const uint32_t* bmap;
  const int32_t* wpre;
  const int32_t* rowbase;
  int32_t wpr;
  // Column index of the same grid: buckets ordered by (conc, tt).
  const int32_t* col_start;
  const int32_t* col_tt;
  const int32_t* col_b;
  // sq_t[k] = (k / span_t)^2 rounded exactly like norm_dist, k < lt (same for conc).
  const double* sq_t;
  const double* sq_c;
  int64_t lt, lc;
};

// normalized_distance (oracle.py:62-77): exact integer deltas, IEEE rn ops.
__device__ __forceinline__ double norm_dist(int64_t dtt, int64_t dc, int64_t span_t, int64_t span_c) {
  double dt = span_t ? __ddiv_rn((double)dtt, (double)span_t) : 0.0;
  double dd = span_c ? __ddiv_rn((double)dc, (double)span_c) : 0.0;
  return __dsqrt_rn(__dadd_rn(__dmul_rn(dt, dt), __dmul_rn(dd, dd)));
}

// x ** p with numpy's fast scalar-power paths (2 -> square, 0.5 -> sqrt, 1 -> x).
__device__ __forceinline__ double shepard_pow(double x, double p) {
  if (p == 2.0) return __dmul_rn(x, x);
  if (p == 1.0) return x;
  if (p == 0.5) return __dsqrt_rn(x);
  return pow(x, p);
}

// numpy pairwise_sum over a[0..n) (float64 add.reduce starting from +0.0):
// n < 8 sequential; n <= 128 eight interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then a sequential tail; larger n splits
// at n2 = n/2 - (n/2)%8 and adds the two halves.
__device__ __forceinline__ double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, a[i]);
  return res;
}

// Iterative post-order evaluation of numpy's recursion (no device-stack
// recursion: pools can hold every bucket of a table).
static __device__ __noinline__ double pairwise_sum(const double* a, int64_t n) {
  if (n <= 128) return pairwise_leaf(a, n);
  int64_t lo_[24], n_[24];
  double left_[24];
  int state_[24];
  int sp = 0;
  lo_[0] = 0;
  n_[0] = n;
  state_[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int64_t fl = lo_[sp], fn = n_[sp];
    if (fn <= 128) {
      ret = pairwise_leaf(a + fl, fn);
      sp--;
      continue;
    }
    int64_t n2 = fn / 2;
    n2 -= n2 % 8;
    if (state_[sp] == 0) {
      state_[sp] = 1;
      sp++;
      lo_[sp] = fl;
      n_[sp] = n2;
      state_[sp] = 0;
    } else if (state_[sp] == 1) {
      left_[sp] = ret;
      state_[sp] = 2;
      sp++;
      lo_[sp] = fl + n2;
      n_[sp] = fn - n2;
      state_[sp] = 0;
    } else {
      ret = __dadd_rn(left_[sp], ret);
      sp--;
    }
  }
  return ret;
}

// ------------------------------------------------------------------- RNGs
struct Pcg64 {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t has_u32, u32;
};

__device__ __forceinline__ uint64_t pcg64_next64(Pcg64& g) {
  // state = state * M + inc  (128-bit), M = 0x2360ED051FC65DA4_4385DF649FCCF645
  const uint64_t m_hi = 0x2360ED051FC65DA4ULL, m_lo = 0x4385DF649FCCF645ULL;
  uint64_t lo = g.s_lo * m_lo;
  uint64_t hi = __umul64hi(g.s_lo, m_lo) + g.s_lo * m_hi + g.s_hi * m_lo;
  uint64_t nlo = lo + g.i_lo;
  uint64_t nhi = hi + g.i_hi + (nlo < lo ? 1ULL : 0ULL);
  g.s_lo = nlo;
  g.s_hi = nhi;
  uint64_t x = nhi ^ nlo;
  unsigned rot = (unsigned)(nhi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg64_next32(Pcg64& g) {
  if (g.has_u32) {
    g.has_u32 = 0;
    return g.u32;
  }
  uint64_t v = pcg64_next64(g);
  g.has_u32 = 1;
  g.u32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

__device__ __forceinline__ double unit_double(uint64_t v) {
  return __dmul_rn((double)(v >> 11), 1.0 / 9007199254740992.0);
}

// EXPLICIT-mode continuation words (PCG-RXS-M-XS 32-bit hash of the previous word).
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  uint32_t s = x * 747796405u + 2891336453u;
  uint32_t w = ((s >> ((s >> 28u) + 4u)) ^ s) * 277803737u;
  return (w >> 22u) ^ w;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Generator.integers(n) via Lemire with rejection on a 32-bit word source.
template <typename NextWord>
__device__ __forceinline__ uint32_t lemire_index(uint32_t n, uint32_t first_word, NextWord next) {
  if (n <= 1u) return 0u;
  uint64_t m = (uint64_t)first_word * n;
  uint32_t left = (uint32_t)m;
  if (left < n) {
    uint32_t thr = (0u - n) % n;  // (2^32 - n) mod n == (UINT32_MAX - (n-1)) % n
    while (left < thr) {
      m = (uint64_t)next() * n;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// ---------------------------------------------------------------- pool slots
// The pool arena is allocated in 16-byte units; pools start on even units
// (32 B, one L2 sector).
struct __align__(16) Slot {
  double cdf;
  int32_t soff;
  int32_t n;
};

// A drawn bucket: its first sample and sample count.
struct PoolPick {
  int32_t soff;
  int32_t n;
};

// Pool layout in the arena (two-level inverse-CDF index), for K buckets in
// G = ceil(K/8) groups of 8:
//   [header: G-1 split cdfs (the last cdf of every group but the final one),
//    padded to an even unit count]
//   [cdf: K doubles -- each 8-bucket group is 64 B on a sector boundary]
//   [data: K x {int32 first sample, int32 count}]
// A draw reads the header (<= 3 splits for K <= 32: one 32-B sector), the
// chosen group's cdfs with <= 4 16-byte loads, then one 8-byte data word:
// 5-6 load instructions per query instead of one per cdf.  (A variant with
// 32-bit integer search keys per group -- one sector per group, integer
// compares -- measured 4-6 % slower in k_sample / k_sweep and in the pool
// build's finish: the draw is bound by its dependent L2 round trips, not by
// the compares, and the extra key array grows the arena.)
constexpr int kGroupSlots = 8;
__host__ __device__ __forceinline__ int64_t pool_groups(int64_t K) { return (K + kGroupSlots - 1) / kGroupSlots; }
__host__ __device__ __forceinline__ int64_t pool_header_slots(int64_t K) {
  const int64_t h = pool_groups(K) / 2;  // ceil((G - 1) / 2) units
  return (h + 1) & ~(int64_t)1;
}
__host__ __device__ __forceinline__ int64_t pool_cdf_units(int64_t K) { return (K + 1) / 2; }
__host__ __device__ __forceinline__ int64_t pool_total_slots(int64_t K) {
  return (pool_header_slots(K) + 2 * pool_cdf_units(K) + 1) & ~(int64_t)1;
}

// Arena pointers of a pool at unit `start`.
struct PoolPtrs {
  double* header;  // nullptr when G == 1
  double* cdf;
  int2* data;
  int32_t K;
};
__device__ __forceinline__ PoolPtrs pool_ptrs(Slot* arena, int64_t start, int64_t K) {
  const int64_t hs = pool_header_slots(K);
  PoolPtrs p;
  p.header = hs ? reinterpret_cast<double*>(arena + start) : nullptr;
  p.cdf = reinterpret_cast<double*>(arena + start + hs);
  p.data = reinterpret_cast<int2*>(arena + start + hs + pool_cdf_units(K));
  p.K = (int32_t)K;
  return p;
}
// Writer side: bucket j's cdf and data (and its group split in the header).
__device__ __forceinline__ void pool_put(const PoolPtrs& pp, int32_t j, double cdf, int2 dv) {
  pp.cdf[j] = cdf;
  pp.data[j] = dv;
  if (pp.header && (j % kGroupSlots) == kGroupSlots - 1 && j < pp.K - 1) pp.header[j / kGroupSlots] = cdf;
}

// Key-map entry: 0 empty, -1 claimed (being built); a built pool is either
//   (K << 32) | start                        K >= 2 buckets at arena unit start
//   kEntryDirect | soff << 31 | n            K == 1: the bucket itself, no arena
// (bit 62 tags a direct entry; K < 2^30, soff, n < 2^31).  Single-bucket pools
// (e.g. every decode key whose own bucket holds >= floor samples) then draw
// with map entry -> sample: two dependent loads instead of four.
constexpr long long kEntryEmpty = 0;
constexpr long long kEntryPending = -1;
constexpr unsigned long long kEntryDirect = 1ULL << 62;
__device__ __forceinline__ long long make_entry(int64_t K, int64_t start) {
  return (long long)(((uint64_t)K << 32) | (uint64_t)start);
}
__device__ __forceinline__ long long make_entry_direct(int64_t soff, int64_t n) {
  return (long long)(kEntryDirect | ((uint64_t)soff << 31) | (uint64_t)n);
}

constexpr unsigned long long kHashEmpty = 0x8000000080000000ULL;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Loads of the draw path; CG = true reads through L2 only (a long-running
// kernel must not see L1 lines older than the pools other kernels rebuilt).
template <bool CG, typename T>
__device__ __forceinline__ T ldp(const T* p) {
  if (CG) return __ldcg(p);
  return *p;
}

// numpy's random() draw: u = (next64 >> 11) * 2^-53; the pick works on k = next64 >> 11.
__device__ __forceinline__ uint64_t unit_k53(uint64_t next64) { return next64 >> 11; }

// searchsorted(cdf, u, 'right') over the pool at arena[start] (K buckets),
// u = k53 * 2^-53 (numpy's random()): returns the chosen bucket.
// cdf[K-1] == 1.0 > u, so a hit always exists.  32-bit offset arithmetic
// (K, start < 2^31 units).
// 32-byte loads (LDG.E.256 on sm_100): a draw reads a pool's header and one
// 8-cdf group with three instead of six 16-byte loads.  Pools start on 32-B
// boundaries and their parts on even 16-B units, so every such load is aligned;
// it may read up to 48 B past what the draw uses (still inside the pool, the
// next pool, or the arena's slack units).
template <bool CG>
__device__ __forceinline__ double4 ld256(const double* p) {
  double4 v;
  if (CG)
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  else
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}

template <bool CG>
__device__ __forceinline__ PoolPick pool_draw_slot(const Slot* __restrict__ arena, int64_t start64, int64_t K64,
                                                   uint64_t k53) {
  const double u = __dmul_rn((double)k53, 1.0 / 9007199254740992.0);
  const int32_t K = (int32_t)K64;
  const Slot* P = arena + start64;
  const int32_t G = (K + kGroupSlots - 1) >> 3;
  const int32_t hs = ((G >> 1) + 1) & ~1;
  int32_t g = 0;
  if (G > 1) {
    const double* sp = reinterpret_cast<const double*>(P);
    if (G <= 5) {  // <= 4 splits: one 32-byte load, count splits <= u
      const double4 a = ld256<CG>(sp);
      g = (a.x <= u) + (G > 2 && a.y <= u) + (G > 3 && a.z <= u) + (G > 4 && a.w <= u);
    } else {
      int32_t lo = 0, hi = G - 1;  // number of splits <= u
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (ldp<CG>(sp + mid) <= u)
          lo = mid + 1;
        else
          hi = mid;
      }
      g = lo;
    }
  }
  const double* C = reinterpret_cast<const double*>(P + hs) + g * kGroupSlots;
  const int32_t n = min(kGroupSlots, K - g * kGroupSlots);
  const double4 c0 = ld256<CG>(C);
  int32_t j = (c0.x <= u) + (n > 1 && c0.y <= u) + (n > 2 && c0.z <= u) + (n > 3 && c0.w <= u);
  if (n > 4) {
    const double4 c1 = ld256<CG>(C + 4);
    j += (c1.x <= u) + (n > 5 && c1.y <= u) + (n > 6 && c1.z <= u) + (n > 7 && c1.w <= u);
  }
  const int2 d = ldp<CG>(reinterpret_cast<const int2*>(P + hs + ((K + 1) >> 1)) + g * kGroupSlots + j);
  PoolPick pk;
  pk.soff = d.x;
  pk.n = d.y;
  return pk;
}

// The bucket a draw k53 selects from a built entry e (> 0).
template <bool CG = false>
__device__ __forceinline__ PoolPick pool_pick(const Slot* __restrict__ arena, long long e, uint64_t k53) {
  const unsigned long long v = (unsigned long long)e;
  if (v & kEntryDirect) {
    PoolPick pk;
    pk.soff = (int32_t)((v >> 31) & 0x7fffffffULL);
    pk.n = (int32_t)(v & 0x7fffffffULL);
    return pk;
  }
  return pool_draw_slot<CG>(arena, (int64_t)(v & 0xffffffffULL), (int64_t)(v >> 32), k53);
}

// Oracle-side device state passed by value to kernels.
struct MapView {
  long long* dense;  // 2 * dom_tt * dom_conc entries
  int32_t dom_tt, dom_conc;
  unsigned long long* hkeys;  // 2 planes * hcap
  long long* hvals;
  int64_t hcap;  // power of two, per plane
};

// Locate (and optionally insert) the entry of a key. Returns a global entry
// index: dense in [0, D), hash in [D, D + 2*hcap); -1 if the hash is full.
__device__ __forceinline__ int64_t map_dense_size(const MapView& m) {
  return 2LL * m.dom_tt * m.dom_conc;
}

__device__ __forceinline__ long long* map_entry_ptr(const MapView& m, int64_t idx) {
  int64_t D = map_dense_size(m);
  return idx < D ? &m.dense[idx] : &m.hvals[idx - D];
}

template <bool kInsert>
__device__ __forceinline__ int64_t map_find(const MapView& m, int plane, int32_t tt, int32_t conc) {
  if (tt >= 1 && tt <= m.dom_tt && conc >= 1 && conc <= m.dom_conc)  // dense map < 2^27 entries: 32-bit math
    return (int64_t)((plane * m.dom_tt + (tt - 1)) * m.dom_conc + (conc - 1));
  unsigned long long key = ((unsigned long long)(uint32_t)tt << 32) | (uint32_t)conc;
  uint64_t mask = (uint64_t)m.hcap - 1;
  uint64_t h = mix64(key) & mask;
  unsigned long long* keys = m.hkeys + (int64_t)plane * m.hcap;
  for (int64_t probe = 0; probe < m.hcap; probe++) {
    unsigned long long k = keys[h];
    if (k == key) return map_dense_size(m) + (int64_t)plane * m.hcap + (int64_t)h;
    if (k == kHashEmpty) {
      if (!kInsert) return -1;
      unsigned long long old = atomicCAS(&keys[h], kHashEmpty, key);
      if (old == kHashEmpty || old == key) return map_dense_size(m) + (int64_t)plane * m.hcap + (int64_t)h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}

}  // namespace emu
