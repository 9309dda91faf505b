// pool.cuh -- exact windowed neighbour expansion + Shepard CDF (sm_100a).
//
// Replaces the per-key O(B log B) lexsort of _pool_order (oracle.py:80-105)
// and _selection_probs + Generator.choice's cdf (oracle.py:124-127, :133) with
// a windowed search over the table's row index (rows = distinct tt):
//
//   * d(dt, dc) is monotone non-decreasing in |dt| and |dc| under IEEE rn,
//     so an integer window |t-tt| <= Wt, |c-conc| <= Wc holds every bucket with
//     d < d_edge = min(d(Wt+1, 0), d(0, Wc+1)) (an axis the window already
//     spans contributes +inf);
//   * candidates inside the window are sorted by (d, bucket index) -- bucket
//     index order is (tt, conc) order, i.e. lexsort((conc, tt, d));
//   * the prefix is accepted iff its last distance is strictly below d_edge
//     (then every bucket outside the window sorts after it), or the window
//     spans the whole table; otherwise the window grows and the search repeats.
//
// One "group" (a warp, NT = 32, or a whole CTA) owns one key; candidates live
// in a group workspace (shared memory, or a global scratch for huge windows).
#pragma once
#include "emu_internal.cuh"

namespace emu {

// Optional per-phase cycle accounting (build with -DEMU_STATS; see tools/pool_stats.py).
#ifdef EMU_STATS
__device__ unsigned long long g_stats[32];
#define EMU_PHASE_BEGIN() long long _emu_ph = clock64()
#define EMU_PHASE(i)                                                                   \
  do {                                                                                 \
    const long long _n = clock64();                                                    \
    if ((threadIdx.x & 31) == 0) atomicAdd(&::emu::g_stats[i], (unsigned long long)(_n - _emu_ph)); \
    _emu_ph = _n;                                                                      \
  } while (0)
#define EMU_STAT(i, v) \
  do { if ((threadIdx.x & 31) == 0) atomicAdd(&::emu::g_stats[i], (unsigned long long)(v)); } while (0)
#define EMU_LSTAT(i, v) atomicAdd(&::emu::g_stats[i], (unsigned long long)(v))
#else
#define EMU_PHASE_BEGIN() \
  do {                    \
  } while (0)
#define EMU_PHASE(i) \
  do {               \
  } while (0)
#define EMU_STAT(i, v) \
  do {                 \
  } while (0)
#define EMU_LSTAT(i, v) \
  do {                  \
  } while (0)
#endif

// Debug-build invariant checks (build with -DEMU_CHECK; `make check`): a failed
// check prints the key and bumps g_check_fail, read by emu_check_read().
#ifdef EMU_CHECK
__device__ unsigned long long g_check_fail;
#define EMU_DCHECK(cond, ...)                 \
  do {                                        \
    if (!(cond)) {                            \
      printf(__VA_ARGS__);                    \
      atomicAdd(&::emu::g_check_fail, 1ULL);  \
    }                                         \
  } while (0)
#else
#define EMU_DCHECK(cond, ...) \
  do {                        \
  } while (0)
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr int64_t kInfW = 1LL << 40;

// ----------------------------------------------------------- group primitives
template <int NT>
struct Grp {  // whole CTA of NT threads (NT multiple of 32, <= 1024)
  static constexpr int kWarps = NT / 32;
  __device__ static int rank() { return threadIdx.x; }
  __device__ static void sync() { __syncthreads(); }
  // exclusive scan; scr must hold >= kWarps + 1 long longs.
  __device__ static long long excl_scan(long long v, long long& total, long long* scr) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scr[w] = x;
    __syncthreads();
    if (w == 0) {
      long long s = lane < kWarps ? scr[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(kFull, s, o);
        if (lane >= o) s += y;
      }
      if (lane < kWarps) scr[lane] = s;  // inclusive warp prefix
    }
    __syncthreads();
    long long base = w ? scr[w - 1] : 0;
    total = scr[kWarps - 1];
    __syncthreads();
    return base + x - v;
  }
  __device__ static int count(bool p, long long* scr) {
    long long tot;
    excl_scan(p ? 1 : 0, tot, scr);
    return (int)tot;
  }
};

template <>
struct Grp<32> {
  __device__ static int rank() { return threadIdx.x & 31; }
  __device__ static void sync() { __syncwarp(); }
  __device__ static long long excl_scan(long long v, long long& total, long long*) {
    int lane = threadIdx.x & 31;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    total = __shfl_sync(kFull, x, 31);
    return x - v;
  }
  __device__ static int count(bool p, long long*) { return __popc(__ballot_sync(kFull, p)); }
};

// ----------------------------------------------------------- workspace
struct PoolWS {
  double* d;      // cap candidate distances
  int32_t* b;     // cap candidate bucket indices
  int64_t cap;    // power of two
  long long* scr; // >= 40 long longs (scan scratch + broadcasts)
  double* dsh;    // >= 10 doubles (broadcast + pairwise accumulators)
  int32_t* rows;  // 3 * NT ints: per-round row bucket start, prefix, |dt|
  int32_t* n;     // ncache: sample count of sorted candidate j (filled by prefix_k)
  int32_t* o;     // ncache: first sample of sorted candidate j
  int64_t ncache;
};

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi, int64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t upper_bound_i32(const int32_t* a, int64_t lo, int64_t hi, int64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool cand_less(double da, int32_t ba, double db, int32_t bb) {
  return da < db || (da == db && ba < bb);
}

// Debug builds: the sorted candidates ws[0..pos) are strictly increasing in
// (distance, bucket) and every bucket index is valid.
template <int NT>
__device__ __forceinline__ void check_sorted(const DevTable& T, const PoolWS& ws, int64_t pos, int64_t C, int32_t t,
                                             int32_t c, int tag) {
#ifdef EMU_CHECK
  EMU_DCHECK(pos >= 0 && pos <= C && pos <= ws.cap, "CHECK pos tag=%d NT=%d key=(%d,%d) pos=%lld C=%lld cap=%lld\n",
             tag, NT, t, c, (long long)pos, (long long)C, (long long)ws.cap);
  for (int64_t i = Grp<NT>::rank(); i < pos; i += NT) {
    const int32_t bb = ws.b[i];
    EMU_DCHECK(bb >= 0 && bb < T.nb, "CHECK bucket tag=%d NT=%d key=(%d,%d) i=%lld/%lld bb=%d nb=%lld\n", tag, NT, t,
               c, (long long)i, (long long)pos, bb, (long long)T.nb);
    if (i > 0)
      EMU_DCHECK(cand_less(ws.d[i - 1], ws.b[i - 1], ws.d[i], bb),
                 "CHECK order tag=%d NT=%d key=(%d,%d) i=%lld/%lld (%.17g,%d) !< (%.17g,%d)\n", tag, NT, t, c,
                 (long long)i, (long long)pos, ws.d[i - 1], ws.b[i - 1], ws.d[i], bb);
  }
  Grp<NT>::sync();
#endif
}


template <int NT>
__device__ void bitonic_sort(double* d, int32_t* b, int64_t P) {
  using G = Grp<NT>;
  for (int64_t k = 2; k <= P; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = G::rank(); i < P; i += NT) {
        int64_t ixj = i ^ j;
        if (ixj > i) {
          double da = d[i], db = d[ixj];
          int32_t ba = b[i], bb = b[ixj];
          bool up = (i & k) == 0;
          bool sw = up ? cand_less(db, bb, da, ba) : cand_less(da, ba, db, bb);
          if (sw) {
            d[i] = db;
            d[ixj] = da;
            b[i] = bb;
            b[ixj] = ba;
          }
        }
      }
      G::sync();
    }
  }
}

// Initial normalized window radius: the disc that would hold `floor` samples
// if the table's samples were spread uniformly over its normalized extent.
__device__ __forceinline__ double initial_radius(const DevTable& T, int64_t mfloor) {
  double n = (double)(T.ns > 0 ? T.ns : 1);
  double r = sqrt((double)mfloor / (3.141592653589793 * n));
  return r > 1e-12 ? r : 1e-12;
}

// Search one key.  On success returns K >= 1 with the sorted pool in
// ws.d[0..K) / ws.b[0..K); returns -1 if a window needs more than ws.cap
// candidates (caller escalates to a bigger workspace).  T must be nonempty.
template <int NT>
__device__ int64_t pool_search_grow(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const PoolWS& ws) {
  using G = Grp<NT>;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const double r0 = initial_radius(T, mfloor);
  double gt = 0.0, gc = 0.0;
  if (span_t) {
    int64_t g = max(max((int64_t)T.tt_lo - t, (int64_t)t - T.tt_hi), (int64_t)0);
    gt = (double)g / (double)span_t;
  }
  if (span_c) {
    int64_t g = max(max((int64_t)T.c_lo - c, (int64_t)c - T.c_hi), (int64_t)0);
    gc = (double)g / (double)span_c;
  }
  const double rb = fmax(gt, gc);
  int64_t prevWt = -1, prevWc = -1;
  for (int it = 0; it < 200; it++) {
    double r = rb + r0 * exp2((double)it);
    int64_t Wt = kInfW, Wc = kInfW;
    if (span_t) {
      double w = floor(r * (double)span_t);
      Wt = w >= (double)kInfW ? kInfW : (int64_t)w;
    }
    if (span_c) {
      double w = floor(r * (double)span_c);
      Wc = w >= (double)kInfW ? kInfW : (int64_t)w;
    }
    if (Wt == prevWt && Wc == prevWc) continue;
    prevWt = Wt;
    prevWc = Wc;
    G::sync();  // every thread has finished reading the previous window's workspace
    const bool cov_t = Wt >= kInfW || ((int64_t)t - Wt <= T.tt_lo && (int64_t)t + Wt >= T.tt_hi);
    const bool cov_c = Wc >= kInfW || ((int64_t)c - Wc <= T.c_lo && (int64_t)c + Wc >= T.c_hi);
    const int64_t rlo = lower_bound_i32(T.row_tt, 0, T.nrows, (int64_t)t - Wt);
    const int64_t rhi = upper_bound_i32(T.row_tt, rlo, T.nrows, (int64_t)t + Wt);
    // ---- enumerate window candidates (one row per thread per round)
    long long C = 0;
    bool ovf = false;
    for (int64_t base = rlo; base < rhi; base += NT) {
      int64_t r_ = base + G::rank();
      int64_t blo = 0, bhi = 0;
      int32_t rtt = 0;
      if (r_ < rhi) {
        rtt = T.row_tt[r_];
        int64_t rs = T.row_start[r_], re = T.row_start[r_ + 1];
        if (Wc >= kInfW) {
          blo = rs;
          bhi = re;
        } else {
          blo = lower_bound_i32(T.bkt_conc, rs, re, (int64_t)c - Wc);
          bhi = upper_bound_i32(T.bkt_conc, blo, re, (int64_t)c + Wc);
        }
      }
      long long len = bhi - blo, tot;
      long long ex = G::excl_scan(len, tot, ws.scr);
      if (C + tot > ws.cap) {
        ovf = true;
        break;
      }
      for (int64_t k = 0; k < len; k++) {
        int64_t bb = blo + k;
        ws.d[C + ex + k] = norm_dist((int64_t)t - rtt, (int64_t)c - T.bkt_conc[bb], span_t, span_c);
        ws.b[C + ex + k] = (int32_t)bb;
      }
      C += tot;
    }
    if (ovf) return -1;
    int64_t P = 1;
    while (P < C) P <<= 1;
    for (int64_t i = C + G::rank(); i < P; i += NT) {
      ws.d[i] = __longlong_as_double(0x7ff0000000000000LL);
      ws.b[i] = 0x7fffffff;
    }
    G::sync();
    if (P > 1) bitonic_sort<NT>(ws.d, ws.b, P);
    // ---- shortest prefix reaching the floor (K <= floor since counts >= 1)
    const int64_t lim = C < mfloor ? C : mfloor;
    long long carry = 0;
    int64_t K = -1;
    for (int64_t base = 0; base < lim; base += NT) {
      int64_t j = base + G::rank();
      long long cnt = 0;
      if (j < lim) {
        int32_t bb = ws.b[j];
        cnt = T.bkt_off[bb + 1] - T.bkt_off[bb];
      }
      long long tot;
      long long ex = G::excl_scan(cnt, tot, ws.scr);
      long long incl = carry + ex + cnt;
      int below = G::count(j < lim && incl < mfloor, ws.scr);
      if (carry + tot >= mfloor) {
        K = base + below + 1;
        break;
      }
      carry += tot;
    }
    check_sorted<NT>(T, ws, C, C, t, c, 3);
    if (K < 0) {
      EMU_DCHECK(!(cov_t && cov_c) || T.ns < mfloor, "CHECK exhaustive(grow) NT=%d key=(%d,%d) C=%lld ns=%lld\n", NT, t,
                 c, (long long)C, (long long)T.ns);
      if (cov_t && cov_c) return C;  // the table holds fewer than mfloor samples
      continue;
    }
    double et = cov_t ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(Wt + 1, 0, span_t, span_c);
    double ec = cov_c ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(0, Wc + 1, span_t, span_c);
    double d_edge = fmin(et, ec);
    // read d_K, then sync: a faster thread returning K starts pool_finish,
    // which overwrites ws.d with masses (WAR race -> non-uniform returns)
    const double dK = ws.d[K - 1];
    G::sync();
    if (dK < d_edge) return K;
  }
  return -1;  // unreachable for a finite table
}

// ---------------------------------------------------------------- SAT search
// Squared normalized delta |k| / span, bit-identical to norm_dist's terms.
__device__ __forceinline__ double sq_delta(int64_t k, int64_t span, const double* tab, int64_t len) {
  if (span == 0) return 0.0;
  if (k < 0) k = -k;
  if (k < len) return tab[k];
  const double q = __ddiv_rn((double)k, (double)span);
  return __dmul_rn(q, q);
}

__device__ __forceinline__ double dist_tab(const DevTable& T, int64_t dtt, int64_t dc, int64_t span_t, int64_t span_c) {
  return __dsqrt_rn(__dadd_rn(sq_delta(dtt, span_t, T.sq_t, T.lt), sq_delta(dc, span_c, T.sq_c, T.lc)));
}

// A query window in grid coordinates.  Grids hold < 2^27 cells, so grid
// indices and cell offsets fit in int32.
struct Win {
  int64_t Wt, Wc;
  int32_t i0, i1, j0, j1;  // clipped grid index ranges (empty if i0 > i1 or j0 > j1)
  bool cov_t, cov_c;
};

__device__ __forceinline__ int64_t radius_to_w(double r, int64_t span) {
  if (!span) return kInfW;
  const double w = floor(r * (double)span);
  return w >= (double)kInfW ? kInfW : (int64_t)w;
}

__device__ __forceinline__ Win make_win(const DevTable& T, int32_t t, int32_t c, int64_t Wt, int64_t Wc) {
  Win w;
  w.Wt = Wt;
  w.Wc = Wc;
  const int64_t lt = (int64_t)t - Wt, ht = (int64_t)t + Wt, lc = (int64_t)c - Wc, hc = (int64_t)c + Wc;
  w.cov_t = lt <= T.tt_lo && ht >= T.tt_hi;
  w.cov_c = lc <= T.c_lo && hc >= T.c_hi;
  w.i0 = (int32_t)min(max((int64_t)0, lt - T.tt_lo), T.gnt);
  w.i1 = (int32_t)max(min(T.gnt - 1, ht - T.tt_lo), (int64_t)-1);
  w.j0 = (int32_t)min(max((int64_t)0, lc - T.c_lo), T.gnc);
  w.j1 = (int32_t)max(min(T.gnc - 1, hc - T.c_lo), (int64_t)-1);
  return w;
}

__device__ __forceinline__ int sat_rect(const int32_t* __restrict__ S, int32_t st, const Win& w) {
  if (w.i0 > w.i1 || w.j0 > w.j1) return 0;
  const int32_t r0 = w.i0 * st, r1 = (w.i1 + 1) * st;
  return S[r1 + w.j1 + 1] - S[r0 + w.j1 + 1] - S[r1 + w.j0] + S[r0 + w.j0];
}

// Column j's slice [lo, lo + cnt) of the column index (buckets ordered by
// (conc, tt)) over grid rows [i0, i1], from the bucket SAT: four loads instead
// of two binary searches over the column (rows [0, i) hold S[i][j+1] - S[i][j]).
__device__ __forceinline__ void col_range(const DevTable& T, int32_t i0, int32_t i1, int32_t j, int32_t& lo,
                                          int32_t& cnt) {
  const int32_t st = (int32_t)T.gnc + 1;
  const int32_t a = i0 * st + j, b = (i1 + 1) * st + j;
  const int32_t before = T.bsat[a + 1] - T.bsat[a];
  lo = T.col_start[j] + before;
  cnt = T.bsat[b + 1] - T.bsat[b] - before;
}

// 2^((l - 8) / 4): the radius grid of the SAT probe.
__constant__ double kRadiusStep[32] = {
    0.25, 0.29730177875068026, 0.3535533905932738, 0.42044820762685725, 0.5, 0.5946035575013605,
    0.7071067811865476, 0.8408964152537145, 1.0, 1.189207115002721, 1.4142135623730951, 1.681792830507429,
    2.0, 2.378414230005442, 2.8284271247461903, 3.363585661014858, 4.0, 4.756828460010884, 5.656854249492381,
    6.727171322029716, 8.0, 9.513656920021768, 11.313708498984761, 13.454342644059432, 16.0, 19.027313840043536,
    22.627416997969522, 26.908685288118864, 32.0, 38.05462768008707, 45.254833995939045, 53.81737057623773};

// Bitonic sort of 32*E (d, bucket) keys held E per lane (element q*32 + lane).
template <int E>
__device__ __forceinline__ void warp_bitonic(double (&d)[E], int32_t (&b)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int q = 0; q < E; q++) {
          const int p = q ^ (j >> 5);
          if (p > q) {
            const bool asc = ((q * 32 + lane) & k) == 0;
            const bool sw = asc ? cand_less(d[p], b[p], d[q], b[q]) : cand_less(d[q], b[q], d[p], b[p]);
            if (sw) {
              const double td = d[q];
              const int32_t tb = b[q];
              d[q] = d[p];
              b[q] = b[p];
              d[p] = td;
              b[p] = tb;
            }
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < E; q++) {
          const double pd = __shfl_xor_sync(kFull, d[q], j);
          const int32_t pb = __shfl_xor_sync(kFull, b[q], j);
          const bool asc = ((q * 32 + lane) & k) == 0;
          const bool lower = (lane & j) == 0;
          const bool mine_less = cand_less(d[q], b[q], pd, pb);
          if (mine_less != (lower == asc)) {
            d[q] = pd;
            b[q] = pb;
          }
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void warp_sort_ws(const PoolWS& ws, int C) {
  const int lane = threadIdx.x & 31;
  double d[E];
  int32_t b[E];
#pragma unroll
  for (int q = 0; q < E; q++) {
    const int i = q * 32 + lane;
    d[q] = i < C ? ws.d[i] : __longlong_as_double(0x7ff0000000000000LL);
    b[q] = i < C ? ws.b[i] : 0x7fffffff;
  }
  warp_bitonic<E>(d, b);
  __syncwarp();
#pragma unroll
  for (int q = 0; q < E; q++) {
    const int i = q * 32 + lane;
    if (i < C) {
      ws.d[i] = d[q];
      ws.b[i] = b[q];
    }
  }
  __syncwarp();
}

// Multi-warp groups (NT > 32), up to 128 candidates per warp: each warp sorts
// its run of 128 in registers (warp_bitonic), then every element's final
// position is its index in its run plus, for each other run, the number of
// elements there that order before it (binary search in shared memory; the
// (distance, bucket) keys are distinct, so ranks are exact).  Two passes over
// shared memory instead of the log^2 stages of the shared-memory bitonic
// network.  Returns false (caller sorts otherwise) above 128 per warp.
template <int NT>
__device__ __forceinline__ bool grp_sort_runs(const PoolWS& ws, int64_t pos) {
  constexpr int W = NT / 32;
  if (NT <= 32 || pos > 128 * (int64_t)W) return false;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = w * 128;
  const int len = (int)max((int64_t)0, min((int64_t)128, pos - r0));
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  double d[4];
  int32_t b[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int i = q * 32 + lane;
    d[q] = i < len ? ws.d[r0 + i] : kInf;
    b[q] = i < len ? ws.b[r0 + i] : 0x7fffffff;
  }
  if (len > 0) warp_bitonic<4>(d, b);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int i = q * 32 + lane;
    if (i < len) {
      ws.d[r0 + i] = d[q];
      ws.b[r0 + i] = b[q];
    }
  }
  __syncthreads();
  int dst[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int i = q * 32 + lane;
    dst[q] = -1;
    if (i < len) {
      int p = i;
      for (int v = 0; v < W; v++) {
        const int lv = (int)max((int64_t)0, min((int64_t)128, pos - v * 128));
        if (v == w || lv == 0) continue;
        const double* rd = ws.d + v * 128;
        const int32_t* rb = ws.b + v * 128;
        int lo = 0, hi = lv;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (cand_less(rd[mid], rb[mid], d[q], b[q]))
            lo = mid + 1;
          else
            hi = mid;
        }
        p += lo;
      }
      dst[q] = p;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; q++)
    if (dst[q] >= 0) {
      ws.d[dst[q]] = d[q];
      ws.b[dst[q]] = b[q];
    }
  __syncthreads();
  return true;
}

// Multi-warp groups, up to 4 candidates per thread: bucket sort by d^2 (512
// bins over [0, max d^2]: monotone in d, so bins are in distance order), then
// each bin's few entries ordered by (d, bucket) in place.  Elements travel in
// registers, bin counts live in the ncache arrays (free until prefix_k).  Four
// barriers and O(pos) work instead of sorting networks; returns false (caller
// sorts otherwise) when it does not apply.
template <int NT>
__device__ __forceinline__ bool grp_bucket_sort(const PoolWS& ws, int64_t pos) {
  constexpr int E = 4, NB = 512;
  using G = Grp<NT>;
  if (NT <= 32 || pos > (int64_t)E * NT || 2 * ws.ncache < NB + NB / 32) return false;
  const int r = G::rank(), lane = r & 31;
  int* cnt = ws.n;  // NB + NB/32 ints, skewed (ws.o follows: 2 * ncache ints in all)
  auto at = [](int b) { return b + (b >> 5); };  // bin b's slot: conflict-free per-thread runs
  double d[E];
  int32_t b[E];
  double mx = 0.0;
#pragma unroll
  for (int q = 0; q < E; q++) {
    const int i = q * NT + r;
    d[q] = 0.0;
    b[q] = 0;
    if (i < pos) {
      d[q] = ws.d[i];
      b[q] = ws.b[i];
      mx = fmax(mx, d[q]);
    }
  }
  for (int i = r; i < NB + NB / 32; i += NT) cnt[i] = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 0) ws.dsh[r >> 5] = mx;
  G::sync();
  mx = ws.dsh[0];
#pragma unroll
  for (int q = 1; q < NT / 32; q++) mx = fmax(mx, ws.dsh[q]);
  const double sc = mx > 0.0 && mx < 1e300 ? (double)NB / __dmul_rn(mx, mx) : 0.0;
  int bin[E], rk[E];
#pragma unroll
  for (int q = 0; q < E; q++) {
    bin[q] = -1;
    if (q * NT + r < pos) {
      const double v = __dmul_rn(__dmul_rn(d[q], d[q]), sc);
      bin[q] = v < (double)(NB - 1) ? (int)v : NB - 1;
      rk[q] = atomicAdd(&cnt[at(bin[q])], 1);
    }
  }
  G::sync();
  // exclusive scan of the bin counts: NB / NT consecutive bins per thread
  constexpr int PER = NB / NT;
  int loc[PER];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < PER; k++) {
    loc[k] = sum;
    sum += cnt[at(r * PER + k)];
  }
  long long tot;
  const int ex = (int)G::excl_scan(sum, tot, ws.scr);
#pragma unroll
  for (int k = 0; k < PER; k++) cnt[at(r * PER + k)] = ex + loc[k];
  G::sync();
#pragma unroll
  for (int q = 0; q < E; q++)
    if (bin[q] >= 0) {
      const int p = cnt[at(bin[q])] + rk[q];
      ws.d[p] = d[q];
      ws.b[p] = b[q];
    }
  G::sync();
  // entries sharing a bin: insertion sort by (d, bucket)
  for (int bn = r; bn < NB; bn += NT) {
    const int s0 = cnt[at(bn)], s1 = bn + 1 < NB ? cnt[at(bn + 1)] : (int)pos;
    for (int x = s0 + 1; x < s1; x++) {
      const double dx = ws.d[x];
      const int32_t bx = ws.b[x];
      int y = x;
      while (y > s0 && cand_less(dx, bx, ws.d[y - 1], ws.b[y - 1])) {
        ws.d[y] = ws.d[y - 1];
        ws.b[y] = ws.b[y - 1];
        y--;
      }
      ws.d[y] = dx;
      ws.b[y] = bx;
    }
  }
  G::sync();
  return true;
}

// Shortest prefix of the sorted candidates (sd, sb)[0..C) reaching the floor,
// or -1 if the C candidates hold fewer than mfloor samples.  Caches each
// scanned candidate's sample count / first sample in ws.n / ws.o.
template <int NT>
__device__ int64_t prefix_k(const DevTable& T, const int32_t* sb, int64_t C, int64_t mfloor, const PoolWS& ws) {
  using G = Grp<NT>;
  const int64_t lim = C < mfloor ? C : mfloor;
  long long carry = 0;
  for (int64_t base = 0; base < lim; base += NT) {
    const int64_t j = base + G::rank();
    long long cnt = 0;
    if (j < lim) {
      const int32_t bb = sb[j];
      EMU_DCHECK(bb >= 0 && bb < T.nb, "CHECK prefix_k NT=%d j=%lld bb=%d nb=%lld C=%lld\n", NT, (long long)j, bb,
                 (long long)T.nb, (long long)C);
      const int64_t o0 = T.bkt_off[bb];
      cnt = T.bkt_off[bb + 1] - o0;
      if (j < ws.ncache) {
        ws.n[j] = (int32_t)cnt;
        ws.o[j] = (int32_t)o0;
      }
    }
    long long tot;
    const long long ex = G::excl_scan(cnt, tot, ws.scr);
    const int below = G::count(j < lim && carry + ex + cnt < mfloor, ws.scr);
    if (carry + tot >= mfloor) return base + below + 1;
    carry += tot;
  }
  return -1;
}

// Windowed search driven by the summed-area tables:
//   1. each of 32 lanes sizes a window for one radius r_l (geometric grid) and
//      counts its samples in O(1) from ssat; the first radius whose window
//      holds >= floor samples (or spans the table) wins, refined by a second
//      32-lane probe between the last miss and that hit -> r1;
//   2. every sample of the r1 window lies within sqrt(2)*r1, so the window for
//      r2 = sqrt(2)*r1 contains the whole pool and passes the exact d_edge
//      test (checked anyway; -2 asks the caller for the growth fallback);
//      candidates farther than r2 cannot be pooled and are dropped;
//   3. the r2 window's buckets are enumerated row by row (bsat gives each
//      row's conc sub-range in O(1)) or by scanning the tt slab, whichever is
//      fewer items; distances use the exact squared-delta tables;
//   4. candidates are sorted in registers (warp bitonic, <= 128) or shared
//      memory, then the prefix reaching the floor is taken.
// Returns K, -1 if the window exceeds ws.cap (escalate), -2 to fall back.
// Append a candidate to the workspace.  A warp compacts with a ballot (same
// order as a scan); multi-warp groups reserve slots with one shared-memory
// atomic per warp instead of a block-wide scan per round: the order of the
// candidates does not matter, the sort that follows imposes the total
// (distance, bucket) order.
template <int NT>
__device__ __forceinline__ void append_cand(bool in, double d, int32_t bb, const PoolWS& ws, int& pos, int* acnt) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(kFull, in);
  int base = pos;
  if (NT > 32) {
    base = 0;
    if (lane == 0 && m) base = atomicAdd(acnt, __popc(m));
    base = __shfl_sync(kFull, base, 0);
  } else {
    pos += __popc(m);
  }
  if (in) {
    const int o = base + __popc(m & ((1u << lane) - 1u));
    EMU_DCHECK(o >= 0 && o < ws.cap, "CHECK append_cand NT=%d o=%d cap=%lld\n", NT, o, (long long)ws.cap);
    ws.d[o] = d;
    ws.b[o] = bb;
  }
}

// Precomputed search window of one key (k_pool_prep, thread per key).
struct KeyWin {
  int64_t Wt, Wc;          // r2 window half-widths (kInfW = unbounded)
  double dmax;             // candidates farther than this cannot be pooled
  int32_t i0, i1, j0, j1;  // r2 window in grid coordinates
  int32_t off, cap;        // candidate scratch slice [off, off + cap)
  int32_t pos;             // candidates written (<= cap)
  int32_t flags;           // kWinReady | kWinCovT | kWinCovC
};
// kWinBig: the window was computed but holds more than a warp workspace (the
// group tier takes it as is, without its own radius search).
constexpr int32_t kWinReady = 1, kWinCovT = 2, kWinCovC = 4, kWinBig = 8;

template <int NT>
__device__ int64_t pool_search_sat(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const PoolWS& ws,
                                   int64_t& sorted_off, const KeyWin* kwin = nullptr) {
  using G = Grp<NT>;
  EMU_PHASE_BEGIN();
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const int32_t st = (int32_t)T.gnc + 1;
  Win w;
  double r1, dmax;
  int C;
  if (kwin) {  // the window k_pool_prep found (same rules: r1 search on the SAT, r2 = sqrt(2) r1)
    w.Wt = kwin->Wt;
    w.Wc = kwin->Wc;
    w.i0 = kwin->i0;
    w.i1 = kwin->i1;
    w.j0 = kwin->j0;
    w.j1 = kwin->j1;
    w.cov_t = kwin->flags & kWinCovT;
    w.cov_c = kwin->flags & kWinCovC;
    dmax = kwin->dmax;
    r1 = dmax < 1e300 ? dmax / (1.4142135623730951 * (1.0 + 1e-9) * (1.0 + 1e-9)) : dmax;
    C = kwin->cap;
  } else {
  double gtd = 0.0, gcd = 0.0;
  if (span_t) gtd = (double)max(max((int64_t)T.tt_lo - t, (int64_t)t - T.tt_hi), (int64_t)0) / (double)span_t;
  if (span_c) gcd = (double)max(max((int64_t)T.c_lo - c, (int64_t)c - T.c_hi), (int64_t)0) / (double)span_c;
  const double rb = fmax(gtd, gcd);
  const double r0 = initial_radius(T, mfloor);
  // ---- 1. radius search
  double rmiss = -1.0;
  r1 = -1.0;
  double scale = 1.0;
  for (int round = 0; round < 10 && r1 < 0.0; round++, scale *= 256.0) {
    bool ok = true;
    double rl = 0.0;
    if (G::rank() < 32) {
      const int l = G::rank();
      rl = (round == 0 && l == 0) ? rb : rb + r0 * scale * kRadiusStep[l];
      const Win w = make_win(T, t, c, radius_to_w(rl, span_t), radius_to_w(rl, span_c));
      ok = (w.cov_t && w.cov_c) || sat_rect(T.ssat, st, w) >= mfloor;
    }
    const int first = G::count(!ok, ws.scr);  // ok is monotone in the radius
    if (NT == 32) {
      const double hit = __shfl_sync(kFull, rl, first & 31);
      const double miss = __shfl_sync(kFull, rl, (first + 31) & 31);
      if (first < 32) {
        r1 = hit;
        if (first > 0) rmiss = miss;
      } else {
        rmiss = miss;
      }
    } else {
      if (G::rank() == (first == 0 ? 0 : first - 1)) ws.dsh[0] = rl;
      if (first < 32 && G::rank() == first) ws.dsh[1] = rl;
      G::sync();
      if (first < 32) {
        r1 = ws.dsh[1];
        if (first > 0) rmiss = ws.dsh[0];
      } else {
        rmiss = ws.dsh[0];
      }
      G::sync();
    }
  }
  EMU_PHASE(0);
  if (r1 < 0.0) return -2;
  if (rmiss >= 0.0 && r1 > rmiss) {  // refine inside (rmiss, r1]
    bool ok = true;
    double rl = r1;
    if (G::rank() < 32) {
      rl = (G::rank() == 31) ? r1 : rmiss + (r1 - rmiss) * (double)(G::rank() + 1) * (1.0 / 32.0);
      const Win w = make_win(T, t, c, radius_to_w(rl, span_t), radius_to_w(rl, span_c));
      ok = (w.cov_t && w.cov_c) || sat_rect(T.ssat, st, w) >= mfloor;
    }
    const int first = G::count(!ok, ws.scr);
    if (NT == 32) {
      r1 = __shfl_sync(kFull, rl, first & 31);
    } else {
      if (first < 32 && G::rank() == first) ws.dsh[1] = rl;
      G::sync();
      if (first < 32) r1 = ws.dsh[1];
      G::sync();
    }
  }
  EMU_PHASE(1);
  // ---- 2. the guaranteed window; pool members lie within dmax of the query
  const double r2 = r1 * 1.4142135623730951 * (1.0 + 1e-9);
  w = make_win(T, t, c, radius_to_w(r2, span_t), radius_to_w(r2, span_c));
  const Win w1 = make_win(T, t, c, radius_to_w(r1, span_t), radius_to_w(r1, span_c));
  const bool exhaust = w1.cov_t && w1.cov_c && sat_rect(T.ssat, st, w1) < mfloor;
  dmax = exhaust ? __longlong_as_double(0x7ff0000000000000LL) : r2 * (1.0 + 1e-9);
  C = sat_rect(T.bsat, st, w);
  }
  EMU_STAT(8, C);
  EMU_PHASE(2);
  if (C > ws.cap) return -1;
  // ---- 3. enumerate (candidates beyond dmax cannot be pooled and are dropped).
  // Group tiers also count, per thread, the samples within each of the 8 pivot
  // radii of step 3b while the candidate's bucket is at hand.
  const bool pivots = NT > 32 && dmax < 1e300;
  double pv[8];
  unsigned pacc[8];
#pragma unroll
  for (int l = 0; l < 8; l++) {
    pv[l] = r1 * (1.0 + 0.41421356237309515 * (double)(l + 1) * 0.125);
    pacc[l] = 0;
  }
  // (each candidate counts at most min(floor, 2^20) samples: the per-thread and
  // per-warp sums stay in 32 bits; a capped count can only make a pivot look
  // short of the floor, never the reverse)
  auto pivot_count = [&](bool in, double d, int32_t bb) {
    if (!pivots || !in) return;
    const unsigned cn = (unsigned)min(min((int64_t)(T.bkt_off[bb + 1] - T.bkt_off[bb]), mfloor), (int64_t)1 << 20);
#pragma unroll
    for (int l = 0; l < 8; l++) pacc[l] += d <= pv[l] ? cn : 0u;
  };
  int pos = 0;
  int* acnt = reinterpret_cast<int*>(ws.scr + 32);  // group tiers: append counter
  if (NT > 32) {
    if (G::rank() == 0) *acnt = 0;
    G::sync();
  }
  if (C > 0) {
    const int32_t nri = w.i1 - w.i0 + 1;
    const int32_t b0 = T.bsat[w.i0 * st + (st - 1)], b1 = T.bsat[(w.i1 + 1) * st + (st - 1)];
    const int32_t ncj = w.j1 - w.j0 + 1;
    if (ncj * 16 < nri && ncj <= NT) {  // tall, narrow window: column index (see warp_enumerate)
      const int32_t tlo = T.tt_lo + w.i0, thi = T.tt_lo + w.i1;
      const int r = G::rank();
      int32_t lo = 0, cnt = 0;
      if (r < ncj) {
        col_range(T, w.i0, w.i1, w.j0 + r, lo, cnt);
      }
      long long tot;
      const int ex = (int)G::excl_scan(cnt, tot, ws.scr);
      ws.rows[r] = lo;
      ws.rows[NT + r] = ex;
      G::sync();
      for (int kb = 0; kb < (int)tot; kb += NT) {
        const int k = kb + r;
        bool in = false;
        double d = 0.0;
        int32_t bb = 0;
        if (k < (int)tot) {
          int l0 = 0, h0 = ncj;  // last column whose prefix <= k
          while (h0 - l0 > 1) {
            const int mid = (l0 + h0) >> 1;
            if (ws.rows[NT + mid] <= k)
              l0 = mid;
            else
              h0 = mid;
          }
          const int32_t idx = ws.rows[l0] + (k - ws.rows[NT + l0]);
          bb = T.col_b[idx];
          d = dist_tab(T, (int64_t)t - T.col_tt[idx], (int64_t)c - (T.c_lo + w.j0 + l0), span_t, span_c);
          in = d <= dmax;
        }
        pivot_count(in, d, bb);
        append_cand<NT>(in, d, bb, ws, pos, acnt);
      }
      G::sync();
    } else if (b1 - b0 <= 2 * nri || C == b1 - b0) {  // scan the tt slab
      const int32_t clo = T.c_lo + w.j0, chi = T.c_lo + w.j1;
      for (int32_t base = b0; base < b1; base += NT) {
        const int32_t b = base + G::rank();
        bool in = false;
        double d = 0.0;
        if (b < b1) {
          const int32_t bc = T.bkt_conc[b];
          if (bc >= clo && bc <= chi) {
            d = dist_tab(T, (int64_t)t - T.bkt_tt[b], (int64_t)c - bc, span_t, span_c);
            in = d <= dmax;
          }
        }
        pivot_count(in, d, b);
        append_cand<NT>(in, d, b, ws, pos, acnt);
      }
    } else {  // row by row: bsat gives each row's conc sub-range
      for (int32_t base = w.i0; base <= w.i1; base += NT) {
        const int32_t i = base + G::rank();
        int len = 0;
        int32_t lo = 0;
        if (i <= w.i1) {
          const int32_t r0i = i * st, r1i = r0i + st;
          const int32_t rs = T.bsat[r0i + st - 1];
          lo = rs + T.bsat[r1i + w.j0] - T.bsat[r0i + w.j0];
          len = rs + T.bsat[r1i + w.j1 + 1] - T.bsat[r0i + w.j1 + 1] - lo;
        }
        long long tot;
        const int ex = (int)G::excl_scan(len, tot, ws.scr);
        ws.rows[G::rank()] = lo;
        ws.rows[NT + G::rank()] = ex;
        ws.rows[2 * NT + G::rank()] = (int32_t)((int64_t)t - (T.tt_lo + i));
        G::sync();
        const int nrow = min(NT, w.i1 - base + 1);
        for (int kb = 0; kb < (int)tot; kb += NT) {
          const int k = kb + G::rank();
          bool in = false;
          double d = 0.0;
          int32_t bb = 0;
          if (k < (int)tot) {
            int lo_r = 0, hi_r = nrow;  // last row with prefix <= k
            while (hi_r - lo_r > 1) {
              const int mid = (lo_r + hi_r) >> 1;
              if (ws.rows[NT + mid] <= k)
                lo_r = mid;
              else
                hi_r = mid;
            }
            bb = ws.rows[lo_r] + (k - ws.rows[NT + lo_r]);
            d = dist_tab(T, ws.rows[2 * NT + lo_r], (int64_t)c - T.bkt_conc[bb], span_t, span_c);
            in = d <= dmax;
          }
          pivot_count(in, d, bb);
          append_cand<NT>(in, d, bb, ws, pos, acnt);
        }
        G::sync();
      }
    }
  }
  G::sync();
  if (NT > 32) {
    pos = *acnt;
    G::sync();
  }
  // ---- 3b. (group / CTA tiers) drop candidates beyond the pool radius bound.
  // d_K lies in [~r1, sqrt(2) r1]: of 8 pivots r1 * (1 + (sqrt(2)-1)(l+1)/8) the
  // smallest whose disc already holds >= floor samples bounds d_K, and every
  // candidate beyond it sorts after the pool.  Typical M = 256 windows shrink
  // from ~1.8 K to ~1.1 K candidates, halving the shared-memory sort.
  if (pivots && pos > 64) {
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ws.scr) + 16;
    if (G::rank() < 8) cnt[G::rank()] = 0;
    G::sync();
#pragma unroll
    for (int l = 0; l < 8; l++) {
      const unsigned v = __reduce_add_sync(kFull, pacc[l]);
      if ((G::rank() & 31) == 0 && v) atomicAdd(&cnt[l], (unsigned long long)v);
    }
    G::sync();
    int l = 0;
    while (l < 7 && cnt[l] < (unsigned long long)mfloor) l++;
    const bool use = cnt[l] >= (unsigned long long)mfloor;
    const double piv = r1 * (1.0 + 0.41421356237309515 * (double)(l + 1) * 0.125);
    G::sync();
    if (use) {  // compact in place, appending with one shared atomic per warp (the sort imposes the order)
      int* ocnt = reinterpret_cast<int*>(ws.scr + 32);
      if (G::rank() == 0) *ocnt = 0;
      G::sync();
      const int lane = G::rank() & 31;
      for (int base = 0; base < pos; base += NT) {
        const int i = base + G::rank();
        double d = 0.0;
        int32_t bb = 0;
        bool keep = false;
        if (i < pos) {
          d = ws.d[i];
          bb = ws.b[i];
          keep = d <= piv;
        }
        G::sync();  // this round is read before any of it is overwritten (writes stay below base + NT)
        const unsigned m = __ballot_sync(kFull, keep);
        int o = 0;
        if (lane == 0 && m) o = atomicAdd(ocnt, __popc(m));
        o = __shfl_sync(kFull, o, 0);
        if (keep) {
          const int q = o + __popc(m & ((1u << lane) - 1u));
          ws.d[q] = d;
          ws.b[q] = bb;
        }
      }
      G::sync();
      pos = *ocnt;
      G::sync();
    }
  }
  EMU_PHASE(3);
  EMU_STAT(9, pos);
  // ---- 4. order
  sorted_off = 0;
  if (NT == 32 && pos <= 128) {
    if (pos <= 32)
      warp_sort_ws<1>(ws, pos);
    else if (pos <= 64)
      warp_sort_ws<2>(ws, pos);
    else
      warp_sort_ws<4>(ws, pos);
  } else if (!grp_bucket_sort<NT>(ws, pos) && !grp_sort_runs<NT>(ws, pos)) {
    int64_t P = 1;
    while (P < pos) P <<= 1;
    for (int64_t i = pos + G::rank(); i < P; i += NT) {
      ws.d[i] = __longlong_as_double(0x7ff0000000000000LL);
      ws.b[i] = 0x7fffffff;
    }
    G::sync();
    if (P > 1) bitonic_sort<NT>(ws.d, ws.b, P);
  }
  EMU_PHASE(4);
  check_sorted<NT>(T, ws, pos, C, t, c, 1);
  const int64_t K = prefix_k<NT>(T, ws.b, pos, mfloor, ws);
  EMU_PHASE(5);
  EMU_STAT(10, K);
  EMU_STAT(11, 1);
  if (K < 0) {
    EMU_DCHECK(!(w.cov_t && w.cov_c) || pos < mfloor || T.ns < mfloor,
               "CHECK exhaustive(sat) NT=%d key=(%d,%d) pos=%d C=%d nb=%lld ns=%lld dmax=%g\n", NT, t, c, pos, C,
               (long long)T.nb, (long long)T.ns, dmax);
    return (w.cov_t && w.cov_c) ? pos : -2;
  }
  const double et = w.cov_t ? __longlong_as_double(0x7ff0000000000000LL) : dist_tab(T, w.Wt + 1, 0, span_t, span_c);
  const double ec = w.cov_c ? __longlong_as_double(0x7ff0000000000000LL) : dist_tab(T, 0, w.Wc + 1, span_t, span_c);
  // every thread reads d_K before any returns: the caller's pool_finish
  // overwrites ws.d (a group whose warps raced here returned non-uniformly and
  // desynchronised its barriers -- the round-1 out-of-grid known issue)
  const double dK = ws.d[K - 1];
  G::sync();
  return dK < fmin(et, ec) ? K : -2;
}

// ------------------------------------------------- thread-per-key SAT passes
// The scalar parts of the SAT search run one key per THREAD (k_pool_win /
// k_pool_enum); the warp kernel then only sorts, takes the prefix and builds
// the CDF.  Same window rules as pool_search_sat (see its comment).


__device__ __forceinline__ bool win_ok(const DevTable& T, int32_t t, int32_t c, double r, int64_t span_t,
                                       int64_t span_c, int32_t st, int64_t mfloor) {
  const Win w = make_win(T, t, c, radius_to_w(r, span_t), radius_to_w(r, span_c));
  return (w.cov_t && w.cov_c) || sat_rect(T.ssat, st, w) >= mfloor;
}

// Radius search by doubling + bisection on the SAT (thread level).  Returns
// false if the table has no grid (the warp kernel then runs the full search).
__device__ bool key_window(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, KeyWin& kw) {
  kw.flags = 0;
  kw.pos = 0;
  if (T.gnt <= 0) return false;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const int32_t st = (int32_t)T.gnc + 1;
  double gtd = 0.0, gcd = 0.0;
  if (span_t) gtd = (double)max(max((int64_t)T.tt_lo - t, (int64_t)t - T.tt_hi), (int64_t)0) / (double)span_t;
  if (span_c) gcd = (double)max(max((int64_t)T.c_lo - c, (int64_t)c - T.c_hi), (int64_t)0) / (double)span_c;
  const double rb = fmax(gtd, gcd);
  double r1;
  if (win_ok(T, t, c, rb, span_t, span_c, st, mfloor)) {
    r1 = rb;
  } else {
    double lo = rb, step = initial_radius(T, mfloor), hi = rb + step;
    int guard = 0;
    while (!win_ok(T, t, c, hi, span_t, span_c, st, mfloor)) {
      lo = hi;
      step *= 2.0;
      hi = rb + step;
      if (++guard > 200) return false;
    }
    // Bisection until the windows of lo (too small) and hi (enough samples)
    // differ by one step of one axis: hi's window is then the minimal one, and
    // r1 = the smallest radius that still yields it (its breakpoint).
    for (int it = 0; it < 40; it++) {
      const int64_t dwt = radius_to_w(hi, span_t) - radius_to_w(lo, span_t);
      const int64_t dwc = radius_to_w(hi, span_c) - radius_to_w(lo, span_c);
      if ((span_t ? dwt : 0) + (span_c ? dwc : 0) <= 1) break;
      const double mid = 0.5 * (lo + hi);
      if (win_ok(T, t, c, mid, span_t, span_c, st, mfloor))
        hi = mid;
      else
        lo = mid;
    }
    r1 = hi;
    {
      const int64_t wt = radius_to_w(hi, span_t), wc = radius_to_w(hi, span_c);
      double rb2 = 0.0;
      if (span_t) rb2 = fmax(rb2, (double)wt / (double)span_t);
      if (span_c) rb2 = fmax(rb2, (double)wc / (double)span_c);
      for (int k = 0; k < 4 && rb2 < hi; k++, rb2 = nextafter(rb2, 1e300))
        if (radius_to_w(rb2, span_t) == wt && radius_to_w(rb2, span_c) == wc) {
          r1 = fmax(rb2, rb);
          break;
        }
    }
  }
  const double r2 = r1 * 1.4142135623730951 * (1.0 + 1e-9);
  const Win w = make_win(T, t, c, radius_to_w(r2, span_t), radius_to_w(r2, span_c));
  const Win w1 = make_win(T, t, c, radius_to_w(r1, span_t), radius_to_w(r1, span_c));
  const bool exhaust = w1.cov_t && w1.cov_c && sat_rect(T.ssat, st, w1) < mfloor;
  kw.Wt = w.Wt;
  kw.Wc = w.Wc;
  kw.i0 = w.i0;
  kw.i1 = w.i1;
  kw.j0 = w.j0;
  kw.j1 = w.j1;
  kw.dmax = exhaust ? __longlong_as_double(0x7ff0000000000000LL) : r2 * (1.0 + 1e-9);
  kw.cap = sat_rect(T.bsat, st, w);
  kw.flags = kWinReady | (w.cov_t ? kWinCovT : 0) | (w.cov_c ? kWinCovC : 0);
  return true;
}

// Warp: enumerate the window's candidates into ws[0..pos) from the occupancy
// bitmap (one row per lane per round: the row's 1-2 bitmap words give its
// buckets; bucket index = rowbase + wpre + popcount, conc = bit position), then
// drop those farther than dmax.  Returns pos, or -1 if they do not fit.
__device__ int warp_enumerate(const DevTable& T, int32_t t, int32_t c, const KeyWin& kw, const PoolWS& ws) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  if (kw.cap <= 0) return 0;
  if (kw.cap > ws.cap) return -1;
  const int32_t nrows = kw.i1 - kw.i0 + 1, ncols = kw.j1 - kw.j0 + 1;
  if (ncols * 16 < nrows) {
    // Tall, narrow windows (sparse long-context tables: windows thousands of
    // tt rows tall, a few conc columns wide): per column, binary-search the
    // window's tt range in the column index, then take the candidates
    // lane-parallel.  Candidate order is irrelevant: the sort breaks distance
    // ties on the bucket index.
    const int32_t tlo = T.tt_lo + kw.i0, thi = T.tt_lo + kw.i1;
    int pos = 0;
    for (int32_t cbase = kw.j0; cbase <= kw.j1; cbase += 32) {
      const int32_t j = cbase + lane;
      int32_t lo = 0, cnt = 0;
      if (j <= kw.j1) {
        col_range(T, kw.i0, kw.i1, j, lo, cnt);
      }
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
      }
      const int tot = __shfl_sync(kFull, x, 31);
      ws.rows[lane] = lo;
      ws.rows[32 + lane] = x - cnt;
      __syncwarp();
      const int ncol = min(32, kw.j1 - cbase + 1);
      for (int kb = 0; kb < tot; kb += 32) {
        const int k = kb + lane;
        bool in = false;
        double d = 0.0;
        int32_t b = 0;
        if (k < tot) {
          int l0 = 0, h0 = ncol;  // last column whose prefix <= k
          while (h0 - l0 > 1) {
            const int mid = (l0 + h0) >> 1;
            if (ws.rows[32 + mid] <= k)
              l0 = mid;
            else
              h0 = mid;
          }
          const int32_t idx = ws.rows[l0] + (k - ws.rows[32 + l0]);
          b = T.col_b[idx];
          d = __dsqrt_rn(__dadd_rn(sq_delta((int64_t)t - T.col_tt[idx], span_t, T.sq_t, T.lt),
                                   sq_delta((int64_t)c - (T.c_lo + cbase + l0), span_c, T.sq_c, T.lc)));
          in = d <= kw.dmax;
        }
        const unsigned m = __ballot_sync(kFull, in);
        if (in) {
          ws.d[pos + __popc(m & lt)] = d;
          ws.b[pos + __popc(m & lt)] = b;
        }
        pos += __popc(m);
      }
      __syncwarp();
    }
    return pos;
  }
  {
    // Sparse rows: scan the window's tt slab -- contiguous in bucket order --
    // when it holds fewer buckets than the window has rows.
    const int32_t b0 = T.rowbase[kw.i0], b1 = T.rowbase[kw.i1 + 1];
    if (b1 - b0 <= nrows) {
      const int32_t clo = T.c_lo + kw.j0, chi = T.c_lo + kw.j1;
      int pos = 0;
      for (int32_t base = b0; base < b1; base += 32) {
        const int32_t b = base + lane;
        bool in = false;
        double d = 0.0;
        if (b < b1) {
          const int32_t bc = T.bkt_conc[b];
          if (bc >= clo && bc <= chi) {
            d = dist_tab(T, (int64_t)t - T.bkt_tt[b], (int64_t)c - bc, span_t, span_c);
            in = d <= kw.dmax;
          }
        }
        const unsigned m = __ballot_sync(kFull, in);
        if (in) {
          ws.d[pos + __popc(m & lt)] = d;
          ws.b[pos + __popc(m & lt)] = b;
        }
        pos += __popc(m);
      }
      __syncwarp();
      return pos;
    }
  }
  const int32_t w0 = kw.j0 >> 5, w1 = kw.j1 >> 5;
  int pos = 0;
  for (int32_t rbase = kw.i0; rbase <= kw.i1; rbase += 32) {
    const int32_t i = rbase + lane;
    int cnt = 0;
    if (i <= kw.i1) {
      for (int32_t wd = w0; wd <= w1; wd++) {
        uint32_t m = T.bmap[(int64_t)i * T.wpr + wd];
        if (wd == w0) m &= 0xffffffffu << (kw.j0 & 31);
        if (wd == w1 && (kw.j1 & 31) != 31) m &= (2u << (kw.j1 & 31)) - 1u;
        cnt += __popc(m);
      }
    }
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (cnt) {
      int p = pos + x - cnt;
      const int32_t rb = T.rowbase[i];
      const double sqt = sq_delta((int64_t)t - (T.tt_lo + i), span_t, T.sq_t, T.lt);
      for (int32_t wd = w0; wd <= w1; wd++) {
        const int64_t wi = (int64_t)i * T.wpr + wd;
        const uint32_t word = T.bmap[wi];
        uint32_t m = word;
        if (wd == w0) m &= 0xffffffffu << (kw.j0 & 31);
        if (wd == w1 && (kw.j1 & 31) != 31) m &= (2u << (kw.j1 & 31)) - 1u;
        if (!m) continue;
        const int32_t pre = rb + T.wpre[wi];
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1u;
          const int32_t jj = wd * 32 + j;
          ws.d[p] = __dsqrt_rn(__dadd_rn(sqt, sq_delta((int64_t)c - (T.c_lo + jj), span_c, T.sq_c, T.lc)));
          ws.b[p] = pre + __popc(word & ((1u << j) - 1u));
          p++;
        }
      }
    }
    pos += __shfl_sync(kFull, x, 31);
  }
  __syncwarp();
  // in-place compaction: keep d <= dmax (write index never passes read index)
  int out = 0;
  for (int base = 0; base < pos; base += 32) {
    const int k = base + lane;
    double d = 0.0;
    int32_t b = 0;
    bool keep = false;
    if (k < pos) {
      d = ws.d[k];
      b = ws.b[k];
      keep = d <= kw.dmax;
    }
    const unsigned m = __ballot_sync(kFull, keep);
    __syncwarp();
    if (keep) {
      ws.d[out + __popc(m & lt)] = d;
      ws.b[out + __popc(m & lt)] = b;
    }
    out += __popc(m);
    __syncwarp();
  }
  return out;
}

// Warp fast path from a thread-computed window: enumerate, sort, take the
// prefix, verify.  Returns K (sorted pool in ws[0..K)), or -2 to fall back.
__device__ int64_t pool_from_window(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const KeyWin& kw,
                                    const PoolWS& ws) {
  EMU_PHASE_BEGIN();
  const int pos = warp_enumerate(T, t, c, kw, ws);
  EMU_PHASE(3);
  EMU_STAT(8, kw.cap);
  EMU_STAT(9, pos);
  if (pos < 0) return -2;
  if (pos <= 32)
    warp_sort_ws<1>(ws, pos);
  else if (pos <= 64)
    warp_sort_ws<2>(ws, pos);
  else if (pos <= 128)
    warp_sort_ws<4>(ws, pos);
  else {
    int64_t P = 1;
    while (P < pos) P <<= 1;
    if (P > ws.cap) return -2;
    for (int64_t i = pos + (threadIdx.x & 31); i < P; i += 32) {
      ws.d[i] = __longlong_as_double(0x7ff0000000000000LL);
      ws.b[i] = 0x7fffffff;
    }
    __syncwarp();
    bitonic_sort<32>(ws.d, ws.b, P);
  }
  EMU_PHASE(4);
  check_sorted<32>(T, ws, pos, kw.cap, t, c, 2);
  const int64_t K = prefix_k<32>(T, ws.b, pos, mfloor, ws);
  EMU_PHASE(5);
  EMU_STAT(10, K);
  EMU_STAT(11, 1);
  const bool cov_t = kw.flags & kWinCovT, cov_c = kw.flags & kWinCovC;
  if (K < 0) return (cov_t && cov_c) ? pos : -2;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const double et = cov_t ? kInf : dist_tab(T, kw.Wt + 1, 0, span_t, span_c);
  const double ec = cov_c ? kInf : dist_tab(T, 0, kw.Wc + 1, span_t, span_c);
  const double dK = ws.d[K - 1];
  __syncwarp();
  return dK < fmin(et, ec) ? K : -2;
}

// Dispatcher: SAT search when the table has a grid, else (or if the SAT
// window fails its exact check) the window-growth search.  The sorted pool
// is at ws.d/ws.b + sorted_off.
template <int NT>
__device__ int64_t pool_search(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const PoolWS& ws,
                               int64_t& sorted_off, bool& cached, const KeyWin* kwin = nullptr) {
  sorted_off = 0;
  cached = true;
  if (T.gnt > 0) {
    const int64_t K = pool_search_sat<NT>(T, t, c, mfloor, ws, sorted_off, kwin);
    if (K != -2) return K;
    Grp<NT>::sync();
    sorted_off = 0;
  }
  cached = false;
  return pool_search_grow<NT>(T, t, c, mfloor, ws);
}

// Shepard weights -> probabilities -> cdf for the pool in ws[0..K), numpy order.
// Writes (optionally) bucket/dist/prob/cdf arrays and/or cache slots.
template <int NT>
__device__ void pool_finish(const DevTable& T, int64_t K, double p, double eps, const PoolWS& ws_in,
                            int64_t sorted_off, bool cached, const PoolPtrs* slots,
                            int32_t* o_bkt, double* o_dist, double* o_prob, double* o_cdf) {
  using G = Grp<NT>;
  PoolWS ws = ws_in;
  ws.d += sorted_off;
  ws.b += sorted_off;
  EMU_DCHECK(K >= 1, "CHECK pool_finish NT=%d K=%lld\n", NT, (long long)K);
  const bool use_cache = cached && K <= ws.ncache;
  for (int64_t j = G::rank(); j < K; j += NT) {
    int32_t bb = ws.b[j];
    double d = ws.d[j];
    const int64_t n = use_cache ? (int64_t)ws.n[j] : T.bkt_off[bb + 1] - T.bkt_off[bb];
    if (o_bkt) o_bkt[j] = bb;
    if (o_dist) o_dist[j] = d;
    double x = d > eps ? d : eps;  // np.maximum(d, eps)
    double w = __ddiv_rn(1.0, shepard_pow(x, p));
    ws.d[j] = __dmul_rn(w, (double)n);  // mass
  }
  G::sync();
  if (K <= 128) {  // numpy's 8-accumulator leaf: lanes 0..7 own one accumulator each
    double r = 0.0;
    const int64_t body = K < 8 ? 0 : K - (K % 8);
    if (G::rank() < 8 && K >= 8) {
      r = ws.d[G::rank()];
      for (int64_t i = 8 + G::rank(); i < body; i += 8) r = __dadd_rn(r, ws.d[i]);
      ws.dsh[2 + G::rank()] = r;
    }
    G::sync();
    if (G::rank() == 0) {
      double res;
      if (K < 8) {
        res = 0.0;
        for (int64_t i = 0; i < K; i++) res = __dadd_rn(res, ws.d[i]);
      } else {
        const double* q = ws.dsh + 2;
        res = __dadd_rn(__dadd_rn(__dadd_rn(q[0], q[1]), __dadd_rn(q[2], q[3])),
                        __dadd_rn(__dadd_rn(q[4], q[5]), __dadd_rn(q[6], q[7])));
        for (int64_t i = body; i < K; i++) res = __dadd_rn(res, ws.d[i]);
      }
      ws.dsh[0] = res;
    }
  } else if (NT >= 128 && K <= 256) {
    // numpy's recursion for 128 < K <= 256: A = [0, n2), n2 = K/2 - (K/2)%8, and
    // B = [n2, K), itself split the same way when longer than 128.  Each leaf
    // (<= 128) is one warp's 8-accumulator block; S = A + B (or A + (B1 + B2)).
    double* part = reinterpret_cast<double*>(ws.scr);  // 3 leaves x 8 partial accumulators
    const int64_t n2 = (K / 2) - (K / 2) % 8, m = K - n2;
    const int64_t m2 = m > 128 ? (m / 2) - (m / 2) % 8 : m;
    const int64_t lb3[3] = {0, n2, n2 + m2}, ln3[3] = {n2, m2, m - m2};
    const int nleaf = m > 128 ? 3 : 2;
    const int g = G::rank() >> 5, q = G::rank() & 31;
    if (g < nleaf && q < 8) {
      const int64_t lb = lb3[g], ln = ln3[g];
      const int64_t body = ln - (ln % 8);
      double r = ws.d[lb + q];
      for (int64_t i = 8 + q; i < body; i += 8) r = __dadd_rn(r, ws.d[lb + i]);
      part[g * 8 + q] = r;
    }
    G::sync();
    if (G::rank() == 0) {
      double leaf[3];
      for (int h = 0; h < nleaf; h++) {
        const double* r = part + h * 8;
        const int64_t lb = lb3[h], ln = ln3[h];
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (int64_t i = ln - (ln % 8); i < ln; i++) res = __dadd_rn(res, ws.d[lb + i]);
        leaf[h] = res;
      }
      ws.dsh[0] = __dadd_rn(leaf[0], nleaf == 3 ? __dadd_rn(leaf[1], leaf[2]) : leaf[1]);
    }
  } else if (G::rank() == 0) {
    ws.dsh[0] = pairwise_sum(ws.d, K);
  }
  G::sync();
  const double S = ws.dsh[0];
  for (int64_t j = G::rank(); j < K; j += NT) {
    double pr = __ddiv_rn(ws.d[j], S);
    ws.d[j] = pr;
    if (o_prob) o_prob[j] = pr;
  }
  G::sync();
  if (G::rank() == 0) {  // np.cumsum: strictly sequential (loads hoisted 8 at a time)
    double acc = ws.d[0];
    int64_t j = 1;
    for (; j + 8 <= K; j += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; q++) v[q] = ws.d[j + q];
#pragma unroll
      for (int q = 0; q < 8; q++) {
        acc = __dadd_rn(acc, v[q]);
        ws.d[j + q] = acc;
      }
    }
    for (; j < K; j++) {
      acc = __dadd_rn(acc, ws.d[j]);
      ws.d[j] = acc;
    }
  }
  G::sync();
  const double last = ws.d[K - 1];
  for (int64_t j = G::rank(); j < K; j += NT) {
    double cdf = __ddiv_rn(ws.d[j], last);
    if (o_cdf) o_cdf[j] = cdf;
    if (slots) {
      int2 dv;
      if (use_cache) {
        dv.x = ws.o[j];
        dv.y = ws.n[j];
      } else {
        const int32_t bb = ws.b[j];
        const int64_t o0 = T.bkt_off[bb];
        dv.x = (int32_t)o0;
        dv.y = (int32_t)(T.bkt_off[bb + 1] - o0);
      }
      pool_put(*slots, (int32_t)j, cdf, dv);
    }
  }
  G::sync();
}

}  // namespace emu
