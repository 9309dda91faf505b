// pool_tile.cuh -- tile tier of the pool build: one warp per tile of 32
// neighbouring keys, one LANE per key (sm_100a).
//
// Why: the warp-per-key tier (pool.cuh, k_pool_warp) spends ~2.2k warp
// instructions per key on a problem of ~40 candidates: register bitonic
// networks, lane-0 serial cumsums and warp scans dominate.  At the bench
// configs the cold sweep's new keys cover a dense part of the key grid, so
// 32 keys that are neighbours in (phase, conc, tt) share most of their
// windows.  Here the warp enumerates the UNION of the 32 keys' r2 windows
// once into shared memory (column index: buckets by (conc, tt)), and every
// lane then runs the whole search for its own key over that list:
//
//   1. (uniform loop over the union) own-window test + a float squared
//      distance: a membership bitmask (d <= dmax) and a conservative
//      8-pivot histogram of sample counts;
//   2. the smallest pivot whose disc already holds >= floor samples bounds
//      d_K (the pool radius); only members within it get an EXACT distance
//      (norm_dist's IEEE rn ops via the squared-delta tables) and go to the
//      lane's list;
//   3. selection sort of that list by (d, bucket) until the prefix reaches
//      the floor -- lexsort((conc, tt, d)) order, oracle.py:98-103;
//   4. the same exact d_edge test as pool_from_window; then Shepard weights,
//      numpy's pairwise sum, probabilities, sequential cumsum and cdf in
//      exactly pool_finish's operation order (oracle.py:124-127, :133).
//
// The candidate set per key is the one pool_from_window enumerates (own r2
// window, d <= dmax), so pools are identical; every key that does not fit
// (window out of the grid, union > kTileU candidates, list > kTileL entries,
// failed d_edge test) is handed to the warp tier unchanged.
#pragma once
#include "pool.cuh"

namespace emu {

constexpr int kTileU = 256;       // union candidates per tile
#ifndef EMU_TILE_L
#define EMU_TILE_L 36
#endif
constexpr int kTileL = EMU_TILE_L;  // exact candidates per key (after the pivot)
constexpr int kTileWarps = 2;
constexpr int kTileThreads = 32 * kTileWarps;
constexpr int kTileRowShift = 4;  // ordering bins: 16 grid rows of one conc column
constexpr int kTileMaxFloor = 32;
constexpr int kTileRowPath = 512; // union boxes up to this many grid rows enumerate by rows
#ifndef EMU_TILE_MINB
#define EMU_TILE_MINB 6
#endif

struct TileWarp {
  int4 u[kTileU];             // union candidates in BUCKET order: (tt, conc, count, bucket)
  double d[kTileL * 32];      // per-lane list, entry e of lane l at [e * 32 + l] (staging for the union sort)
  uint8_t j[kTileL * 32];     // union index of that entry (= bucket order: ties in d break on it)
  uint8_t perm[kTileL * 32];  // sorted order: the e-th smallest entry of lane l is perm[e * 32 + l]
  uint8_t h[32 * 32];         // per lane: distance-bin counts (32 bins, <= kTileL each), then bin starts
};
static_assert(kTileL * 32 * 8 >= kTileU * 16, "the union staging area lives in TileWarp::d");
constexpr int kTileBytes = (int)sizeof(TileWarp) * kTileWarps;

// Ordering bins of the tile tier (per plane: gnc columns x ceil(gnt / 16) row blocks).
struct TileIdx {
  int64_t base[2];  // first bin of each plane
  int64_t nbt[2];   // row blocks per column (0: plane not tiled)
  int64_t nb;       // total bins
};

__device__ __forceinline__ int64_t tile_bin(const DevTable& T, const TileIdx& ti, int ph, int32_t t, int32_t c,
                                            const KeyWin& k, int64_t floor) {
  if (floor > kTileMaxFloor || !(k.flags & kWinReady) || ti.nbt[ph] == 0 || k.cap > kTileU) return -1;
  if (t < T.tt_lo || t > T.tt_hi || c < T.c_lo || c > T.c_hi) return -1;
  const int64_t i = (int64_t)t - T.tt_lo, j = (int64_t)c - T.c_lo;
  return ti.base[ph] + j * ti.nbt[ph] + (i >> kTileRowShift);
}

__device__ __forceinline__ void warp_push(int* list, int* count, bool p, int v) {
  const unsigned m = __ballot_sync(kFull, p);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (p) list[base + __popc(m & ((1u << lane) - 1u))] = v;
}

// Per key: its bin (counting-sort rank) or the warp tier's list.
// kbin: >= 0 bin, -1 warp tier, -2 skipped (arena overflow in prep: the host retries).
template <int MODE>
__global__ void __launch_bounds__(256) k_tile_bin(DevTable P0, DevTable P1, Keys keys, Cfg cfg, TileIdx ti,
                                                  const KeyWin* __restrict__ kw, const long long* __restrict__ resv,
                                                  int* cnt, int* kbin, int* krank, int* fb_list, int* fb_n) {
  const int64_t n = keys.count_dev ? (int64_t)*keys.count_dev : keys.count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {  // warp-uniform trips
    const int64_t w = base + threadIdx.x;
    int64_t bin = -3;
    if (w < n) {
      const int ph = keys.ph[w] ? 1 : 0;
      const KeyWin k = kw[w];
      bin = (MODE == 0 && resv[w] == -2) ? -2 : tile_bin(ph ? P1 : P0, ti, ph, keys.tt[w], keys.conc[w], k, cfg.floor);
      if (bin >= 0) krank[w] = atomicAdd(&cnt[bin], 1);
      kbin[w] = (int)bin;
      if (k.flags & kWinBig) bin = -4;  // already on the group tier's list (k_pool_prep)
    }
    warp_push(fb_list, fb_n, bin == -1, (int)w);
  }
}

template <int MODE>
__global__ void k_tile_scatter(Keys keys, TileIdx ti, const int* __restrict__ kbin, const int* __restrict__ krank,
                               const int* __restrict__ off, const int* __restrict__ total, int* order) {
  const int64_t n = keys.count_dev ? (int64_t)*keys.count_dev : keys.count;
  const int n0 = ti.base[1] < ti.nb ? off[ti.base[1]] : *total;  // plane-0 keys
  const int pad = ((n0 + 31) & ~31) - n0;                         // plane 1 starts on a tile boundary
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n; w += (int64_t)gridDim.x * blockDim.x) {
    const int b = kbin[w];
    if (b < 0) continue;
    order[off[b] + krank[w] + (b >= ti.base[1] ? pad : 0)] = (int)w;
  }
}

// numpy pairwise-sum leaf over a lane-strided array (same operation order as pairwise_leaf).
__device__ __forceinline__ double pairwise_leaf_lane(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i * 32]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; q++) r[q] = a[q * 32];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; q++) r[q] = __dadd_rn(r[q], a[(i + q) * 32]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; i++) res = __dadd_rn(res, a[i * 32]);
  return res;
}

// Enumerate every bucket of the grid box rows [i0, i1] x cols [j0, j1] into
// tw.u in bucket ((tt, conc)) order.  Short boxes walk the occupancy bitmap row
// by row (already in bucket order); tall ones (sparse long-context tables) use
// the column index -- per column two binary searches give the tt range -- and
// merge the columns: an entry's place is its index in its column plus, for
// every other column, how many of that column's buckets precede it.  Returns
// the count, or -1 if the box has more than 32 columns on the column path.
__device__ __forceinline__ int tile_enum_union(const DevTable& T, int32_t i0, int32_t i1, int32_t j0, int32_t j1,
                                               TileWarp& tw) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int pos = 0;
  if (i1 - i0 < kTileRowPath) {
    const int32_t w0 = j0 >> 5, w1 = j1 >> 5;
    for (int32_t rbase = i0; rbase <= i1; rbase += 32) {
      const int32_t i = rbase + lane;
      int cnt = 0;
      if (i <= i1) {
        for (int32_t wd = w0; wd <= w1; wd++) {
          uint32_t m = T.bmap[(int64_t)i * T.wpr + wd];
          if (wd == w0) m &= 0xffffffffu << (j0 & 31);
          if (wd == w1 && (j1 & 31) != 31) m &= (2u << (j1 & 31)) - 1u;
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
        for (int32_t wd = w0; wd <= w1; wd++) {
          const int64_t wi = (int64_t)i * T.wpr + wd;
          const uint32_t word = T.bmap[wi];
          uint32_t m = word;
          if (wd == w0) m &= 0xffffffffu << (j0 & 31);
          if (wd == w1 && (j1 & 31) != 31) m &= (2u << (j1 & 31)) - 1u;
          const int32_t pre = rb + T.wpre[wi];
          while (m) {
            const int jb = __ffs(m) - 1;
            m &= m - 1u;
            const int32_t b = pre + __popc(word & ((1u << jb) - 1u));
            const int64_t o0 = T.bkt_off[b];
            tw.u[p++] = make_int4(T.tt_lo + i, T.c_lo + wd * 32 + jb, (int32_t)(T.bkt_off[b + 1] - o0), b);
          }
        }
      }
      pos += __shfl_sync(kFull, x, 31);
    }
    __syncwarp();
    return pos;
  }
  // column path: at most 32 columns (one per lane)
  if (j1 - j0 >= 32) return -1;
  int4* stg = reinterpret_cast<int4*>(tw.d);
  const int32_t tlo = T.tt_lo + i0, thi = T.tt_lo + i1;
  const int32_t j = j0 + lane;
  int32_t lo = 0, cnt = 0;
  if (j <= j1) {
    col_range(T, i0, i1, j, lo, cnt);
  }
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  const int ex = x - cnt, tot = __shfl_sync(kFull, x, 31);
  if (tot > kTileU) return kTileU + 1;
  const int ncol = j1 - j0 + 1;
  for (int kb = 0; kb < tot; kb += 32) {
    const int k = kb + lane;
    int l0 = 0;  // last column whose exclusive prefix <= k (uniform trip count: every shuffle has all lanes)
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = l0 + step;
      const int exc = __shfl_sync(kFull, ex, cand & 31);
      if (cand < ncol && exc <= k) l0 = cand;
    }
    const int exl = __shfl_sync(kFull, ex, l0), lol = __shfl_sync(kFull, lo, l0);
    if (k < tot) {
      const int32_t idx = lol + (k - exl);
      const int32_t b = T.col_b[idx];
      const int64_t o0 = T.bkt_off[b];
      stg[k] = make_int4(T.col_tt[idx], T.c_lo + j0 + l0, (int32_t)(T.bkt_off[b + 1] - o0), b);
    }
  }
  __syncwarp();
  int maxlen = __reduce_max_sync(kFull, cnt);
  int top = 1;
  while (top <= maxlen) top <<= 1;
  for (int kb = 0; kb < tot; kb += 32) {
    const int k = kb + lane;
    const bool ok = k < tot;
    const int4 v = ok ? stg[k] : make_int4(0, 0, 0, 0x7fffffff);
    int q = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int cand = q + step;
      const int exc = __shfl_sync(kFull, ex, cand & 31);
      if (cand < ncol && exc <= k) q = cand;
    }
    int rank = k - __shfl_sync(kFull, ex, q);
    for (int c2 = 0; c2 < ncol; c2++) {
      const int s0 = __shfl_sync(kFull, ex, c2), len = __shfl_sync(kFull, cnt, c2);
      int base = 0;  // buckets of column c2 that precede v (branch-free search, uniform trips)
      for (int step = top >> 1; step > 0; step >>= 1)
        if (base + step <= len && stg[s0 + base + step - 1].w < v.w) base += step;
      rank += (c2 == q) ? 0 : base;
    }
    __syncwarp();
    if (ok) tw.u[rank] = v;
  }
  __syncwarp();
  (void)lt;
  return tot;
}

// Lane l of a warp handles key w (or none: w < 0).  Returns K >= 1 with the
// lane's pool: sorted entry e (< K) is list slot tw.perm[e * 32 + lane]; or a
// negative reason for the warp tier (-2 list overflow, -3 prefix, -4 window test).
__device__ __forceinline__ int tile_search(const DevTable& T, int32_t t, int32_t c, const KeyWin& k, int64_t mfloor,
                                           int Cu, TileWarp& tw) {
  const int lane = threadIdx.x & 31;
  const int64_t span_t = (int64_t)T.tt_hi - T.tt_lo, span_c = (int64_t)T.c_hi - T.c_lo;
  const float inv_t = span_t ? 1.0f / (float)span_t : 0.0f, inv_c = span_c ? 1.0f / (float)span_c : 0.0f;
  const int32_t Wt = (int32_t)min(k.Wt, (int64_t)0x3fffffff), Wc = (int32_t)min(k.Wc, (int64_t)0x3fffffff);
  const bool exhaust = !(k.dmax < 1e300);
  const float dmax2 = exhaust ? 3.0e38f : (float)(k.dmax * k.dmax) * (1.0f + 4e-5f);
  uint8_t* h = tw.h + lane;  // lane-strided
  // ---- 1. membership bitmask: own window and float distance <= dmax (uniform loop over the union)
  uint32_t mask[kTileU / 32];
#pragma unroll
  for (int wd = 0; wd < kTileU / 32; wd++) {
    uint32_t mw = 0;
    if (wd * 32 < Cu) {
      const int lim = min(32, Cu - wd * 32);
      for (int b0 = 0; b0 < lim; b0 += 4) {
#pragma unroll
        for (int x = 0; x < 4; x++) {
          const int bi = b0 + x;
          const int4 q = tw.u[wd * 32 + bi];  // entries past Cu hold stale data; masked below
          const int32_t dt = t - q.x, dc = c - q.y;
          const float ft = (float)dt * inv_t, fc = (float)dc * inv_c;
          const bool in = bi < lim && abs(dt) <= Wt && abs(dc) <= Wc && ft * ft + fc * fc <= dmax2;
          mw |= (in ? 1u : 0u) << bi;
        }
      }
    }
    mask[wd] = mw;
  }
  // ---- 2. pool radius bound: 16 pivots in squared distance, r1^2 (1 + (l + 1) / 16);
  // the smallest whose disc certainly holds >= floor samples bounds d_K.  The
  // counts use a float squared distance inflated past any rounding (never an
  // overcount); 16-bit counters packed two per register.
  double piv = k.dmax;
  if (!exhaust) {
    const double r1 = k.dmax / (1.4142135623730951 * (1.0 + 1e-9) * (1.0 + 1e-9));  // r2 / sqrt(2) / (1 + 1e-9)
    const float inv_r1sq = (float)(1.0 / (r1 * r1)) * (1.0f + 4e-5f);
    const uint32_t cap = (uint32_t)min(mfloor, (int64_t)1024);
    uint32_t hc[8];
#pragma unroll
    for (int r = 0; r < 8; r++) hc[r] = 0;
#pragma unroll
    for (int wd = 0; wd < kTileU / 32; wd++) {
      uint32_t mw = mask[wd];
      while (mw) {
        const int bi = __ffs(mw) - 1;
        mw &= mw - 1u;
        const int4 q = tw.u[wd * 32 + bi];
        const float ft = (float)(t - q.x) * inv_t, fc = (float)(c - q.y) * inv_c;
        const float v = (ft * ft + fc * fc) * inv_r1sq;  // >= (exact d / r1)^2
        const int lb = v <= 1.0f ? 0 : (int)fminf(ceilf((v - 1.0f) * 16.0f) - 1.0f, 16.0f);
        const uint32_t z = min((uint32_t)q.z, cap) << ((lb & 1) * 16);
#pragma unroll
        for (int r = 0; r < 8; r++) hc[r] += (lb >> 1) == r ? z : 0u;
      }
    }
    uint32_t cum = 0;
    int lp = -1;
#pragma unroll
    for (int l = 0; l < 16; l++) {
      cum += (hc[l >> 1] >> ((l & 1) * 16)) & 0xffffu;
      if (lp < 0 && cum >= (uint32_t)mfloor) lp = l;
    }
    if (lp >= 0) piv = fmin(k.dmax, r1 * sqrt(1.0 + (double)(lp + 1) * 0.0625) * (1.0 + 1e-12));
  }
  // ---- 3. members within the bound (float filter), then their exact distances
  // (norm_dist's IEEE ops via the squared-delta tables), two at a time, counted
  // into 32 distance bins
  const float piv2 = exhaust ? 3.0e38f : (float)(piv * piv) * (1.0f + 4e-5f);
  const double scale = (piv > 0.0 && piv < 1e300) ? 32.0 / piv : 0.0;  // bin(d) = floor(d * scale): monotone in d
  int m = 0;
  bool ovf = false;
#pragma unroll
  for (int wd = 0; wd < kTileU / 32; wd++) {
    uint32_t mw = mask[wd];
    while (mw) {
      const int bi = __ffs(mw) - 1;
      mw &= mw - 1u;
      const int jj = wd * 32 + bi;
      const int4 q = tw.u[jj];
      const float ft = (float)(t - q.x) * inv_t, fc = (float)(c - q.y) * inv_c;
      if (ft * ft + fc * fc > piv2) continue;
      if (m == kTileL) {
        ovf = true;
        break;
      }
      tw.j[m * 32 + lane] = (uint8_t)jj;
      m++;
    }
  }
#pragma unroll
  for (int l = 0; l < 32; l++) h[l * 32] = 0;
  int m2 = 0;  // entries kept after the exact test (compacted in place)
  for (int e = 0; e < m; e += 2) {
    const bool two = e + 1 < m;
    const int ja = tw.j[e * 32 + lane], jb = two ? tw.j[(e + 1) * 32 + lane] : ja;
    const int4 qa = tw.u[ja], qb = tw.u[jb];
    const double da = dist_tab(T, t - qa.x, c - qa.y, span_t, span_c);
    const double db = dist_tab(T, t - qb.x, c - qb.y, span_t, span_c);
    if (da <= piv) {
      tw.d[m2 * 32 + lane] = da;
      tw.j[m2 * 32 + lane] = (uint8_t)ja;
      h[min(31, (int)(da * scale)) * 32] += 1;
      m2++;
    }
    if (two && db <= piv) {
      tw.d[m2 * 32 + lane] = db;
      tw.j[m2 * 32 + lane] = (uint8_t)jb;
      h[min(31, (int)(db * scale)) * 32] += 1;
      m2++;
    }
  }
  m = m2;
  EMU_LSTAT(23, m);
  if (ovf) return -2;
  // ---- 4. bucket sort by (d, bucket): bins in order, then an insertion pass
  // that only moves entries within a bin (an earlier bin's d is strictly
  // smaller); the union is in bucket order, so the union index breaks ties
  {
    int st = 0;
#pragma unroll
    for (int l = 0; l < 32; l++) {
      const int cnt = h[l * 32];
      h[l * 32] = (uint8_t)st;
      st += cnt;
    }
  }
  for (int e = 0; e < m; e++) {
    const int bn = min(31, (int)(tw.d[e * 32 + lane] * scale));
    const int p = h[bn * 32];
    h[bn * 32] = (uint8_t)(p + 1);
    tw.perm[p * 32 + lane] = (uint8_t)e;
  }
  for (int p = 1; p < m; p++) {
    const int x = tw.perm[p * 32 + lane];
    const double dx = tw.d[x * 32 + lane];
    int q = p;
    while (q > 0) {
      const int y = tw.perm[(q - 1) * 32 + lane];
      const double dy = tw.d[y * 32 + lane];
      if (!(dx < dy || (dx == dy && tw.j[x * 32 + lane] < tw.j[y * 32 + lane]))) break;
      tw.perm[q * 32 + lane] = (uint8_t)y;
      q--;
    }
    tw.perm[q * 32 + lane] = (uint8_t)x;
  }
  // ---- 5. the shortest prefix holding >= floor samples
  int64_t cum = 0;
  int K = -1;
  for (int e = 0; e < m; e++) {
    cum += tw.u[tw.j[tw.perm[e * 32 + lane] * 32 + lane]].z;
    if (cum >= mfloor) {
      K = e + 1;
      break;
    }
  }
  const bool cov_t = k.flags & kWinCovT, cov_c = k.flags & kWinCovC;
  if (K < 0) {
    if (!(cov_t && cov_c) || !exhaust || m == 0) return -3;
    K = m;  // the table holds fewer than floor samples: every bucket (sorted above)
  }
  // ---- 6. the exact window test (as pool_from_window)
  const double kInf = __longlong_as_double(0x7ff0000000000000LL);
  const double et = cov_t ? kInf : dist_tab(T, k.Wt + 1, 0, span_t, span_c);
  const double ec = cov_c ? kInf : dist_tab(T, 0, k.Wc + 1, span_t, span_c);
  return tw.d[tw.perm[(K - 1) * 32 + lane] * 32 + lane] < fmin(et, ec) ? K : -4;
}

// Shepard weights -> probabilities -> cdf of the lane's pool, pool_finish's
// operation order; writes cache slots (MODE 0) or explicit outputs (MODE 1).
template <int MODE>
__device__ __forceinline__ void tile_finish(const DevTable& T, int K, const Cfg& cfg, TileWarp& tw, const PoolPtrs* pp,
                                            int32_t* o_bkt, double* o_dist, double* o_prob, double* o_cdf) {
  const int lane = threadIdx.x & 31;
  double* a = tw.d + lane;              // slot s of this lane at a[s * 32]
  const uint8_t* pm = tw.perm + lane;   // e-th smallest -> slot pm[e * 32]
  for (int e = 0; e < K; e++) {
    const int sl = pm[e * 32];
    const double d = a[sl * 32];
    const int4 q = tw.u[tw.j[sl * 32 + lane]];
    if (MODE == 1) {
      o_bkt[e] = q.w;
      o_dist[e] = d;
    }
    const double x = d > cfg.eps ? d : cfg.eps;
    a[sl * 32] = __dmul_rn(__ddiv_rn(1.0, shepard_pow(x, cfg.p)), (double)q.z);  // mass
  }
  // numpy's pairwise sum (K <= floor <= 32: the 8-accumulator leaf), in sorted order
  double S;
  if (K < 8) {
    S = 0.0;
    for (int e = 0; e < K; e++) S = __dadd_rn(S, a[pm[e * 32] * 32]);
  } else {
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; q++) r[q] = a[pm[q * 32] * 32];
    int i = 8;
    for (; i < K - (K % 8); i += 8) {
#pragma unroll
      for (int q = 0; q < 8; q++) r[q] = __dadd_rn(r[q], a[pm[(i + q) * 32] * 32]);
    }
    S = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                  __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < K; i++) S = __dadd_rn(S, a[pm[i * 32] * 32]);
  }
  double acc = 0.0;
  for (int e = 0; e < K; e++) {
    const int sl = pm[e * 32];
    const double pr = __ddiv_rn(a[sl * 32], S);
    if (MODE == 1) o_prob[e] = pr;
    acc = e == 0 ? pr : __dadd_rn(acc, pr);  // np.cumsum: sequential
    a[sl * 32] = acc;
  }
  const double last = acc;
  for (int e = 0; e < K; e++) {
    const int sl = pm[e * 32];
    const double cdf = __ddiv_rn(a[sl * 32], last);
    if (MODE == 1) {
      o_cdf[e] = cdf;
    } else {
      const int4 q = tw.u[tw.j[sl * 32 + lane]];
      pool_put(*pp, e, cdf, make_int2((int32_t)T.bkt_off[q.w], q.z));
    }
  }
}

}  // namespace emu
