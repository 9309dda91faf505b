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
    if (K < 0) {
      if (cov_t && cov_c) return C;  // the table holds fewer than mfloor samples
      continue;
    }
    double et = cov_t ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(Wt + 1, 0, span_t, span_c);
    double ec = cov_c ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(0, Wc + 1, span_t, span_c);
    double d_edge = fmin(et, ec);
    if (ws.d[K - 1] < d_edge) return K;
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

struct Win {
  int64_t Wt, Wc;
  int64_t i0, i1, j0, j1;  // clipped grid index ranges (empty if i0 > i1 or j0 > j1)
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
  w.cov_t = Wt >= kInfW || ((int64_t)t - Wt <= T.tt_lo && (int64_t)t + Wt >= T.tt_hi);
  w.cov_c = Wc >= kInfW || ((int64_t)c - Wc <= T.c_lo && (int64_t)c + Wc >= T.c_hi);
  const int64_t gt = T.gnt - 1, gc = T.gnc - 1;
  w.i0 = Wt >= kInfW ? 0 : max((int64_t)0, (int64_t)t - Wt - T.tt_lo);
  w.i1 = Wt >= kInfW ? gt : min(gt, (int64_t)t + Wt - T.tt_lo);
  w.j0 = Wc >= kInfW ? 0 : max((int64_t)0, (int64_t)c - Wc - T.c_lo);
  w.j1 = Wc >= kInfW ? gc : min(gc, (int64_t)c + Wc - T.c_lo);
  return w;
}

__device__ __forceinline__ long long sat_rect(const int32_t* S, int64_t st, const Win& w) {
  if (w.i0 > w.i1 || w.j0 > w.j1) return 0;
  return (long long)S[(w.i1 + 1) * st + w.j1 + 1] - S[w.i0 * st + w.j1 + 1] - S[(w.i1 + 1) * st + w.j0] +
         S[w.i0 * st + w.j0];
}

// Rank-sort C <= cap/2 candidates of ws[0..C) into ws[cap/2 ..) (stable by
// construction: keys (d, bucket) are unique).
template <int NT>
__device__ void rank_sort(const PoolWS& ws, int64_t C) {
  using G = Grp<NT>;
  double* sd = ws.d + ws.cap / 2;
  int32_t* sb = ws.b + ws.cap / 2;
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  if (NT == 32 && C <= 32) {
    const int lane = G::rank();
    const double dm = lane < C ? ws.d[lane] : kInf;
    const int32_t bm = lane < C ? ws.b[lane] : 0x7fffffff;
    int r = 0;
    for (int k = 0; k < C; k++) {
      const double dk = __shfl_sync(kFull, dm, k);
      const int32_t bk = __shfl_sync(kFull, bm, k);
      r += cand_less(dk, bk, dm, bm) ? 1 : 0;
    }
    if (lane < C) {
      sd[r] = dm;
      sb[r] = bm;
    }
  } else {
    // each thread ranks up to 4 own candidates held in registers against a
    // single broadcast pass over all C candidates
    constexpr int kOwn = 4;
    for (int64_t base = 0; base < C; base += (int64_t)NT * kOwn) {
      double od[kOwn];
      int32_t ob[kOwn];
      int orank[kOwn];
#pragma unroll
      for (int q = 0; q < kOwn; q++) {
        const int64_t i = base + G::rank() + (int64_t)q * NT;
        od[q] = i < C ? ws.d[i] : kInf;
        ob[q] = i < C ? ws.b[i] : 0x7fffffff;
        orank[q] = 0;
      }
      for (int64_t k = 0; k < C; k++) {
        const double dk = ws.d[k];
        const int32_t bk = ws.b[k];
#pragma unroll
        for (int q = 0; q < kOwn; q++) orank[q] += cand_less(dk, bk, od[q], ob[q]) ? 1 : 0;
      }
#pragma unroll
      for (int q = 0; q < kOwn; q++) {
        const int64_t i = base + G::rank() + (int64_t)q * NT;
        if (i < C) {
          sd[orank[q]] = od[q];
          sb[orank[q]] = ob[q];
        }
      }
    }
  }
  G::sync();
}

// Shortest prefix of the sorted candidates (sd, sb)[0..C) reaching the floor,
// or -1 if the C candidates hold fewer than mfloor samples.
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
      cnt = T.bkt_off[bb + 1] - T.bkt_off[bb];
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
//      counts its samples in O(1) from ssat; the first radius r1 whose window
//      holds >= floor samples (or spans the table) wins;
//   2. every sample of that window lies within sqrt(2)*r1, so the window for
//      r2 = sqrt(2)*r1 contains the whole pool and passes the exact d_edge
//      test (checked anyway; -2 asks the caller for the growth fallback);
//   3. the r2 window's buckets are enumerated row by row (bsat gives each
//      row's conc sub-range in O(1)) or by scanning the tt slab, whichever is
//      fewer items; distances use the exact squared-delta tables;
//   4. candidates are rank-sorted (small C) or bitonic-sorted.
// Returns K, -1 if the window exceeds ws.cap (escalate), -2 to fall back.
template <int NT>
__device__ int64_t pool_search_sat(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const PoolWS& ws,
                                   int64_t& sorted_off) {
  using G = Grp<NT>;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const int64_t st = T.gnc + 1;
  double gtd = 0.0, gcd = 0.0;
  if (span_t) gtd = (double)max(max((int64_t)T.tt_lo - t, (int64_t)t - T.tt_hi), (int64_t)0) / (double)span_t;
  if (span_c) gcd = (double)max(max((int64_t)T.c_lo - c, (int64_t)c - T.c_hi), (int64_t)0) / (double)span_c;
  const double rb = fmax(gtd, gcd);
  const double r0 = initial_radius(T, mfloor);
  // ---- 1. radius search (32 radii per round, then 32 between the last miss and the first hit)
  double r1 = -1.0, rmiss = -1.0;
  for (int round = 0; round < 10 && r1 < 0.0; round++) {
    bool ok = true;
    double rl = 0.0;
    if (G::rank() < 32) {
      const int l = G::rank() + 32 * round;
      rl = (l == 0) ? rb : rb + r0 * exp2((double)(l - 8) * 0.25);
      const Win w = make_win(T, t, c, radius_to_w(rl, span_t), radius_to_w(rl, span_c));
      ok = (w.cov_t && w.cov_c) || sat_rect(T.ssat, st, w) >= mfloor;
    }
    const int first = G::count(!ok, ws.scr);  // ok is monotone in the radius
    if (G::rank() == (first == 0 ? 0 : first - 1)) ws.dsh[0] = rl;
    if (first < 32 && G::rank() == first) ws.dsh[1] = rl;
    G::sync();
    if (first < 32) {
      r1 = ws.dsh[1];
      if (first > 0 || round > 0) rmiss = (first > 0) ? ws.dsh[0] : rmiss;
    } else {
      rmiss = ws.dsh[0];
    }
    G::sync();
  }
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
    if (first < 32 && G::rank() == first) ws.dsh[1] = rl;
    G::sync();
    if (first < 32) r1 = ws.dsh[1];
    G::sync();
  }
  // ---- 2. the guaranteed window; pool members lie within dmax of the query
  const double r2 = r1 * 1.4142135623730951 * (1.0 + 1e-9);
  const Win w = make_win(T, t, c, radius_to_w(r2, span_t), radius_to_w(r2, span_c));
  const Win w1 = make_win(T, t, c, radius_to_w(r1, span_t), radius_to_w(r1, span_c));
  const bool exhaust = w1.cov_t && w1.cov_c && sat_rect(T.ssat, st, w1) < mfloor;
  const double dmax = exhaust ? __longlong_as_double(0x7ff0000000000000LL) : r2 * (1.0 + 1e-9);
  const long long C = sat_rect(T.bsat, st, w);
  if (C > ws.cap) return -1;
  // ---- 3. enumerate (candidates beyond dmax cannot be pooled and are dropped)
  long long pos = 0;
  if (C > 0) {
    const int64_t nri = w.i1 - w.i0 + 1;
    const int64_t b0 = T.bsat[w.i0 * st + T.gnc], b1 = T.bsat[(w.i1 + 1) * st + T.gnc];
    if (b1 - b0 <= 2 * nri || C == b1 - b0) {  // scan the tt slab
      const int64_t clo = (int64_t)T.c_lo + w.j0, chi = (int64_t)T.c_lo + w.j1;
      for (int64_t base = b0; base < b1; base += NT) {
        const int64_t b = base + G::rank();
        bool in = false;
        double d = 0.0;
        if (b < b1) {
          const int32_t bc = T.bkt_conc[b];
          if (bc >= clo && bc <= chi) {
            d = dist_tab(T, (int64_t)t - T.bkt_tt[b], (int64_t)c - bc, span_t, span_c);
            in = d <= dmax;
          }
        }
        long long tot;
        const long long ex = G::excl_scan(in ? 1 : 0, tot, ws.scr);
        if (in) {
          ws.d[pos + ex] = d;
          ws.b[pos + ex] = (int32_t)b;
        }
        pos += tot;
      }
    } else {  // row by row: bsat gives each row's conc sub-range
      for (int64_t base = w.i0; base <= w.i1; base += NT) {
        const int64_t i = base + G::rank();
        long long len = 0;
        int32_t lo = 0;
        if (i <= w.i1) {
          const int64_t rs = T.bsat[i * st + T.gnc];
          lo = (int32_t)(rs + T.bsat[(i + 1) * st + w.j0] - T.bsat[i * st + w.j0]);
          const int64_t hi = rs + T.bsat[(i + 1) * st + w.j1 + 1] - T.bsat[i * st + w.j1 + 1];
          len = hi - lo;
        }
        long long tot;
        const long long ex = G::excl_scan(len, tot, ws.scr);
        ws.rows[G::rank()] = lo;
        ws.rows[NT + G::rank()] = (int32_t)ex;
        ws.rows[2 * NT + G::rank()] = (int32_t)((int64_t)t - (T.tt_lo + i));
        G::sync();
        const int nrow = (int)min((int64_t)NT, w.i1 - base + 1);
        for (long long kb = 0; kb < tot; kb += NT) {
          const long long k = kb + G::rank();
          bool in = false;
          double d = 0.0;
          int32_t bb = 0;
          if (k < tot) {
            int lo_r = 0, hi_r = nrow;  // last row with prefix <= k
            while (hi_r - lo_r > 1) {
              const int mid = (lo_r + hi_r) >> 1;
              if (ws.rows[NT + mid] <= k)
                lo_r = mid;
              else
                hi_r = mid;
            }
            bb = ws.rows[lo_r] + (int32_t)(k - ws.rows[NT + lo_r]);
            d = dist_tab(T, ws.rows[2 * NT + lo_r], (int64_t)c - T.bkt_conc[bb], span_t, span_c);
            in = d <= dmax;
          }
          long long kt;
          const long long ex2 = G::excl_scan(in ? 1 : 0, kt, ws.scr);
          if (in) {
            ws.d[pos + ex2] = d;
            ws.b[pos + ex2] = bb;
          }
          pos += kt;
        }
        G::sync();
      }
    }
  }
  G::sync();
  // ---- 4. order
  if (2 * pos <= ws.cap && pos <= (NT == 32 ? 128 : NT)) {
    rank_sort<NT>(ws, pos);
    sorted_off = ws.cap / 2;
  } else {
    int64_t P = 1;
    while (P < pos) P <<= 1;
    for (int64_t i = pos + G::rank(); i < P; i += NT) {
      ws.d[i] = __longlong_as_double(0x7ff0000000000000LL);
      ws.b[i] = 0x7fffffff;
    }
    G::sync();
    if (P > 1) bitonic_sort<NT>(ws.d, ws.b, P);
    sorted_off = 0;
  }
  const double* sd = ws.d + sorted_off;
  const int32_t* sb = ws.b + sorted_off;
  const int64_t K = prefix_k<NT>(T, sb, pos, mfloor, ws);
  if (K < 0) return (w.cov_t && w.cov_c) ? pos : -2;
  const double et = w.cov_t ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(w.Wt + 1, 0, span_t, span_c);
  const double ec = w.cov_c ? __longlong_as_double(0x7ff0000000000000LL) : norm_dist(0, w.Wc + 1, span_t, span_c);
  return sd[K - 1] < fmin(et, ec) ? K : -2;
}

// Dispatcher: SAT search when the table has a grid, else (or if the SAT
// window fails its exact check) the window-growth search.  The sorted pool
// is at ws.d/ws.b + sorted_off.
template <int NT>
__device__ int64_t pool_search(const DevTable& T, int32_t t, int32_t c, int64_t mfloor, const PoolWS& ws,
                               int64_t& sorted_off) {
  sorted_off = 0;
  if (T.gnt > 0) {
    const int64_t K = pool_search_sat<NT>(T, t, c, mfloor, ws, sorted_off);
    if (K != -2) return K;
    Grp<NT>::sync();
    sorted_off = 0;
  }
  return pool_search_grow<NT>(T, t, c, mfloor, ws);
}

// Shepard weights -> probabilities -> cdf for the pool in ws[0..K), numpy order.
// Writes (optionally) bucket/dist/prob/cdf arrays and/or cache slots.
template <int NT>
__device__ void pool_finish(const DevTable& T, int64_t K, double p, double eps, const PoolWS& ws_in,
                            int64_t sorted_off, Slot* slots,
                            int32_t* o_bkt, double* o_dist, double* o_prob, double* o_cdf) {
  using G = Grp<NT>;
  PoolWS ws = ws_in;
  ws.d += sorted_off;
  ws.b += sorted_off;
  for (int64_t j = G::rank(); j < K; j += NT) {
    int32_t bb = ws.b[j];
    double d = ws.d[j];
    int64_t n = T.bkt_off[bb + 1] - T.bkt_off[bb];
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
  if (G::rank() == 0) {  // np.cumsum: strictly sequential
    double acc = ws.d[0];
    for (int64_t j = 1; j < K; j++) {
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
      int32_t bb = ws.b[j];
      int64_t o0 = T.bkt_off[bb];
      Slot s;
      s.cdf = cdf;
      s.soff = (int32_t)o0;
      s.n = (int32_t)(T.bkt_off[bb + 1] - o0);
      slots[j] = s;
    }
  }
  G::sync();
}

}  // namespace emu
