// oracle.cu -- the B200 latency oracle: lazy pool cache + batched sampling.
//
// Mirrors LatencyOracle (oracle.py:181-228).  A batch of Q queries runs as
//   k_mark      : each query claims its (phase, tt, conc) map entry; the first
//                 claimer appends the key to the batch's new-key list
//                 (the cache-miss branch of _pooled, oracle.py:200-204);
//   k_pool_warp : one warp per new key: windowed neighbour search + Shepard CDF
//                 (pool.cuh), pool written to the slot arena, entry published;
//   k_pool_cta  : keys whose window overflowed a warp workspace, one CTA each
//                 (shared memory, else a global scratch that always fits);
//   k_sample    : one thread per query: map -> pool -> searchsorted(cdf, u,
//                 'right') -> Lemire index -> literal sample (_draw, :130-135).
// All four are stream-ordered with no host round trip; the host reads one
// flag word per batch to detect arena/hash exhaustion and retry.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <string>
#include <vector>

#include "emu_internal.cuh"
#include "prof.h"
#include "pool.cuh"
#include "scan.cuh"
#include "tables.h"

namespace emu {

enum : int { FLAG_ARENA = 1, FLAG_HASH = 2, FLAG_MISSING = 4, FLAG_BADPOOL = 8 };

constexpr int kWarpCap = 256;  // candidates per warp workspace
constexpr int kWarpsPerCta = 4;
constexpr int kWarpThreads = 32 * kWarpsPerCta;
constexpr int kWarpBytes = kWarpCap * 12 + 40 * 8 + 10 * 8 + 3 * 32 * 4 + kWarpCap * 4;  // d,b,scr,dsh,rows,n,o
#ifndef EMU_WARP_MINB
#define EMU_WARP_MINB 8  // 64 registers: 8 CTAs x 4 warps per SM (smem 4.9 KB per warp)
#endif
constexpr int kWarpGrid = kNumSMs * EMU_WARP_MINB;
constexpr int kCtaThreads = 256;
constexpr int kCtaCap = 8192;  // candidates in shared memory per CTA
constexpr int kCtaSmem = kCtaCap * 12;
constexpr int kCtaCache = 1024;  // cached counts/offsets per CTA workspace
constexpr int kGrpThreads = 128;  // middle tier: one 4-warp group per key
#ifndef EMU_GRP_CAP
#define EMU_GRP_CAP 1024
#endif
#ifndef EMU_GRP_CACHE
#define EMU_GRP_CACHE 512
#endif
// Group workspace: 1024 candidates (12 KB) + 512 cached counts/offsets keep a
// group CTA at ~18 KB of shared memory, so the 64-register limit (8 groups per
// SM) binds instead of shared memory (6 per SM at 2048 / 1024: C3 M=256 45.4 ->
// 37.9 ms); the rare larger windows go to the CTA tier.
constexpr int kGrpCap = EMU_GRP_CAP;      // candidates per group workspace (bigger windows: CTA tier)
constexpr int kGrpCache = EMU_GRP_CACHE;  // cached counts/offsets per group
constexpr int kGrpSmem = kGrpCap * 12;
#ifndef EMU_GRP_MINB
#define EMU_GRP_MINB 8  // 4-warp groups per SM in the grid (C3 M=256: 84 vs 96 ms at 4)
#endif
constexpr int kGrpGrid = kNumSMs * EMU_GRP_MINB;
constexpr int kCtaGrid = kNumSMs;
constexpr int kSampleThreads = 256;
constexpr int kQPT = 4;  // queries per thread, interleaved for memory-level parallelism
constexpr int64_t kArenaSlack = 4;  // units past arena_cap: a draw's 32-B loads may read up to 48 B past a pool
constexpr int64_t kHostChunk = 1 << 21;  // queries per pipelined chunk of emu_oracle_sample_host (2M: 5.04 ms e2e at C2 vs 5.73 at 1M, 6.93 at 512k)

struct BatchCtl {
  int flags;
  int bad_key[4];  // first key whose pool failed validation: claimed flag, phase, tt, conc
  int ctl_pad[3];
  // per-pass counters from here on (reset_counters): a chunk's passes keep the flags
  unsigned long long cand_used;  // candidate scratch bump pointer
  int new_count;
  int miss_count;  // k_sweep: queries left for k_sample_list (read with new_count in one copy)
  int work;
  int esc_count;
  int esc_work;
  int esc2_count;  // keys too big for the 128-thread group tier -> CTA tier
  int esc2_work;
  int tile_work;   // tile tier: chunk counter
  int tile_total;  // tile tier: keys binned
  int fb_n;        // keys handed from the tile tier to the warp tier
  int fb_work;
  int dense_n;     // cold path: keys from the bitmap, in (phase, conc, tt) order
  int dense_n0;    // ... of which phase 0
  int hash_n;      // cold path: keys outside the dense map (side list)
};

struct Keys {
  const int32_t* tt;
  const int32_t* conc;
  const uint8_t* ph;
  const int64_t* entry;
  const int* count_dev;  // number of keys (device), or nullptr -> count
  int64_t count;
};

struct Sink {
  MapView map;
  Slot* arena;
  int64_t arena_cap;
  unsigned long long* arena_used;
  int32_t* x_bkt;
  double* x_dist;
  double* x_prob;
  double* x_cdf;
  int64_t* x_K;
  int64_t kmax;
  int* flags;
  int* bad_key;  // BatchCtl::bad_key
};

struct Cfg {
  int64_t floor;
  double p, eps;
};
}  // namespace emu

#include "pool_tile.cuh"

namespace emu {

// Result of one engine step, written by k_step straight into mapped pinned
// host memory; the host spins on `seq` (no memcpy, no stream sync).
struct StepOut {
  double lat;
  int32_t sidx;
  int32_t flags;
  uint32_t seq;
  uint32_t pad;
};

__device__ __forceinline__ void publish_step(StepOut* out, double lat, int32_t sidx, int32_t flags, uint32_t seq) {
  volatile StepOut* v = out;
  v->lat = lat;
  v->sidx = sidx;
  v->flags = flags;
  __threadfence_system();
  v->seq = seq;
}

// --------------------------------------------------------------- kernels
// Write a found pool (K entries sorted in ws at soff) to the sink.  MODE 0:
// cache arena slots at `reserved` (or freshly allocated when reserved == -1;
// reserved == -2 means the arena overflowed in prep: leave the key pending)
// and publish its map entry.  MODE 1: explicit fixed-stride outputs.
// A pool can never hold more than min(floor, B) buckets (every bucket has >= 1
// sample, oracle.py:99-103): a larger K is an internal error.  MODE 0 then
// leaves the key's entry pending and flags the batch, naming the key; the host
// call fails instead of drawing from it.
__device__ __forceinline__ void report_bad_pool(const Sink& sk, int ph, int32_t t, int32_t c) {
  atomicOr(sk.flags, FLAG_BADPOOL);
  if (sk.bad_key && atomicCAS(&sk.bad_key[0], 0, 1) == 0) {
    sk.bad_key[1] = ph;
    sk.bad_key[2] = t;
    sk.bad_key[3] = c;
  }
}

template <int NT, int MODE>
__device__ void emit_pool(const DevTable& T, int64_t w, int64_t K, int64_t entry_idx, int64_t soff, bool cached,
                          long long reserved, const Cfg& cfg, const PoolWS& ws, const Sink& sk, int ph, int32_t t,
                          int32_t c) {
  using G = Grp<NT>;
  if (MODE == 0) {
    if (K > cfg.floor || K > T.nb) {
      if (G::rank() == 0) report_bad_pool(sk, ph, t, c);
      G::sync();
      return;
    }
    if (K == 1 && reserved != -2) {  // direct entry: the bucket itself (cdf == [1.0]), no arena slots
      if (G::rank() == 0) {
        const int32_t bb = ws.b[soff];
        const int64_t o0 = T.bkt_off[bb];
        *map_entry_ptr(sk.map, entry_idx) = make_entry_direct(o0, T.bkt_off[bb + 1] - o0);
      }
      G::sync();
      return;
    }
    long long start = reserved;
    if (start == -1) {
      if (G::rank() == 0) {
        const unsigned long long tot = (unsigned long long)pool_total_slots(K);
        unsigned long long st = atomicAdd(sk.arena_used, tot);
        long long s = (st + tot <= (unsigned long long)sk.arena_cap) ? (long long)st : -2LL;
        if (s < 0) atomicOr(sk.flags, FLAG_ARENA);
        ws.scr[36] = s;
      }
      G::sync();
      start = ws.scr[36];
      G::sync();
    }
    if (start < 0) return;
    EMU_PHASE_BEGIN();
    const PoolPtrs pp = pool_ptrs(sk.arena, start, K);
    pool_finish<NT>(T, K, cfg.p, cfg.eps, ws, soff, cached, &pp, nullptr, nullptr, nullptr, nullptr);
    // entries are consumed by a later kernel: stream order publishes them
    if (G::rank() == 0) *map_entry_ptr(sk.map, entry_idx) = make_entry(K, start);
    EMU_PHASE(6);
  } else {
    if (K > sk.kmax) {  // cannot fit the key's output stride (see the known issue in DESIGN.md): report, don't write
      if (G::rank() == 0) sk.x_K[w] = K + (int64_t)NT * 1000000;  // the error message names the tier (32/128/256)
      G::sync();
      return;
    }
    const int64_t base = w * sk.kmax;
    pool_finish<NT>(T, K, cfg.p, cfg.eps, ws, soff, cached, nullptr, sk.x_bkt + base, sk.x_dist + base,
                    sk.x_prob + base, sk.x_cdf + base);
    if (G::rank() == 0) sk.x_K[w] = K;
  }
}

// Full in-group search (no precomputed candidates).  false = window too big
// for this workspace.
template <int NT, int MODE>
__device__ bool process_key(const DevTable& T, int64_t w, int ph, int32_t t, int32_t c, int64_t entry_idx,
                            const Cfg& cfg, const PoolWS& ws, const Sink& sk, const KeyWin* kwin = nullptr) {
  int64_t soff = 0;
  bool cached = false;
  const int64_t K = pool_search<NT>(T, t, c, cfg.floor, ws, soff, cached, kwin);
  if (K < 0) return false;
  emit_pool<NT, MODE>(T, w, K, entry_idx, soff, cached, -1, cfg, ws, sk, ph, t, c);
  return true;
}

// Warp-aggregated bump allocation: each lane asks for `need`, one atomic per warp.
__device__ __forceinline__ long long warp_alloc(unsigned long long* counter, long long need) {
  const int lane = threadIdx.x & 31;
  long long x = need;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  const long long total = __shfl_sync(kFull, x, 31);
  unsigned long long base = 0;
  if (lane == 31 && total > 0) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(kFull, base, 31);
  return (long long)base + x - need;
}

// Thread per new key: SAT radius search -> window (KeyWin) and (MODE 0) the
// pool's arena reservation min(floor, window buckets), one atomic per warp.
template <int MODE>
__global__ void __launch_bounds__(256) k_pool_prep(DevTable P0, DevTable P1, Keys keys, Cfg cfg, Sink sk, KeyWin* kw,
                                                   long long* resv, int* esc_list, int* esc_count, int* wl,
                                                   int* wl_n, int all_to_grp) {
  const int64_t n = keys.count_dev ? (int64_t)*keys.count_dev : keys.count;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t w = base + threadIdx.x;
    const bool valid = w < n;
    KeyWin k;
    k.flags = 0;
    k.cap = 0;
    bool ready = false;
    bool win = false;
    if (valid) {
      const DevTable& T = keys.ph[w] ? P1 : P0;
      win = key_window(T, keys.tt[w], keys.conc[w], cfg.floor, k);
      ready = win && k.cap <= kWarpCap;
    }
    // too big for a warp: keep the window for the group tier (kWinBig), no reservation
    if (!ready) k.flags = win ? ((k.flags & ~kWinReady) | kWinBig) : 0;
    long long r = -1;
    if (MODE == 0) {
      const long long need = ready && !all_to_grp ? pool_total_slots(k.cap < cfg.floor ? k.cap : cfg.floor) : 0;
      const long long st = warp_alloc(sk.arena_used, need);
      if (ready && !all_to_grp) {
        r = (st + need <= sk.arena_cap) ? st : -2;
        if (r == -2) atomicOr(sk.flags, FLAG_ARENA);
      }
    }
    if (valid) {
      kw[w] = k;
      resv[w] = r;
    }
    // windows too big for a warp go straight onto the group tier's list; without
    // the tile tier the others form the warp tier's list (wl)
    const bool big = valid && (k.flags & kWinBig);
    warp_push(esc_list, esc_count, all_to_grp ? valid : big, (int)w);
    if (wl && !all_to_grp) warp_push(wl, wl_n, valid && !big, (int)w);
  }
}

template <int QPT>
__global__ void k_mark(MapView m, const int32_t* __restrict__ qt, const int32_t* __restrict__ qc,
                       const uint8_t* __restrict__ qp, int64_t Q, int32_t* nk_tt, int32_t* nk_c, uint8_t* nk_p,
                       int64_t* nk_e, BatchCtl* ctl) {
  __shared__ int s_cnt, s_base;
  const int64_t tile = (int64_t)blockDim.x * QPT;
  for (int64_t b0 = (int64_t)blockIdx.x * tile; b0 < Q; b0 += (int64_t)gridDim.x * tile) {  // warp-uniform trip count
    const int64_t base = b0 + threadIdx.x;
    int32_t t[QPT], c[QPT];
    int ph[QPT];
    int64_t idx[QPT];
    long long cur[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      const int64_t i = base + (int64_t)j * blockDim.x;
      idx[j] = -2;
      if (i < Q) {
        ph[j] = qp[i] ? 1 : 0;  // kept in L2: k_sample re-reads the keys next
        t[j] = qt[i];
        c[j] = qc[i];
        idx[j] = map_find<true>(m, ph[j], t[j], c[j]);
      }
      // a hint only (the CAS decides): an L2 load, not a volatile (system-scope) one
      cur[j] = idx[j] >= 0 ? __ldcg(map_entry_ptr(m, idx[j])) : -1;
    }
#pragma unroll
    for (int j = 0; j < QPT; j++)
      if (idx[j] == -1) atomicOr(&ctl->flags, FLAG_HASH);
    // claim empty entries; winners append their key.  The append counter is a
    // single address every CTA hits in the first wave, so it takes one atomic
    // per CTA per tile (warp offsets come from a shared-memory counter).
    bool won[QPT];
    unsigned bal[QPT];
    int wcnt = 0;
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      won[j] = false;
      const bool cand = idx[j] >= 0 && cur[j] == kEntryEmpty;
      if (__any_sync(kFull, cand)) {
        // one CAS per distinct key per warp (the cold sweep's first wave hits
        // a few hot entries from every warp at once)
        const unsigned peers = __match_any_sync(kFull, cand ? (unsigned long long)idx[j]
                                                            : (0xffffffff00000000ULL | (threadIdx.x & 31)));
        if (cand && (__ffs(peers) - 1) == (int)(threadIdx.x & 31))
          won[j] = atomicCAS((unsigned long long*)map_entry_ptr(m, idx[j]), 0ULL,
                             (unsigned long long)kEntryPending) == 0ULL;
      }
      bal[j] = __ballot_sync(kFull, won[j]);
      wcnt += __popc(bal[j]);
    }
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_cnt = 0;
    if (!__syncthreads_or(wcnt)) continue;  // warm tile: nothing claimed in this CTA
    int woff = 0;
    if (lane == 0 && wcnt) woff = atomicAdd(&s_cnt, wcnt);
    __syncthreads();
    if (threadIdx.x == 0) s_base = atomicAdd(&ctl->new_count, s_cnt);
    __syncthreads();
    if (!wcnt) continue;
    woff = __shfl_sync(kFull, woff, 0) + s_base;
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      if (won[j]) {
        const int pos = woff + __popc(bal[j] & ((1u << lane) - 1u));
        nk_tt[pos] = t[j];
        nk_c[pos] = c[j];
        nk_p[pos] = (uint8_t)ph[j];
        nk_e[pos] = idx[j];
      }
      woff += __popc(bal[j]);
    }
  }
}

// Cold batches (an empty cache): dedupe by a bitmap over the dense key domain
// instead of claiming map entries.  Bit (phase, conc, tt) of every query is set
// with a fire-and-forget atomic (one per distinct key per warp); a scan of the
// bitmap then lists the batch's keys in (phase, conc, tt) order -- the tile
// tier's neighbour order, so no binning pass is needed -- and clears it.  Keys
// outside the dense map take k_mark's claim path into a side list.
__device__ __forceinline__ int64_t bit_plane_stride(const MapView& m) {
  return (((int64_t)m.dom_tt * m.dom_conc) + 31) & ~(int64_t)31;
}
__global__ void k_mark_bits(MapView m, const int32_t* __restrict__ qt, const int32_t* __restrict__ qc,
                            const uint8_t* __restrict__ qp, int64_t Q, unsigned int* bits, int32_t* hk_tt,
                            int32_t* hk_c, uint8_t* hk_p, int64_t* hk_e, BatchCtl* ctl) {
  // k_mark's claim (an L2 hint load skips claimed entries; one CAS per distinct
  // key per warp), but a winner only sets its key's bit: no append counter, no
  // block barrier; the key list comes from the bitmap scan, in tile order
  const int lane = threadIdx.x & 31;
  const int64_t ps = bit_plane_stride(m);
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < Q; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;  // warp-uniform trip count (match_any below)
    const bool v = i < Q;
    int ph = 0;
    int32_t t = 0, c = 0;
    if (v) {
      ph = qp[i] ? 1 : 0;  // kept in L2: k_sample re-reads the keys next
      t = qt[i];
      c = qc[i];
    }
    const int64_t idx = v ? map_find<true>(m, ph, t, c) : -2;
    const long long cur = idx >= 0 ? __ldcg(map_entry_ptr(m, idx)) : -1;  // a hint only (the CAS decides)
    if (idx == -1) atomicOr(&ctl->flags, FLAG_HASH);
    const bool cand = idx >= 0 && cur == kEntryEmpty;
    if (!__any_sync(kFull, cand)) continue;
    const unsigned peers =
        __match_any_sync(kFull, cand ? (unsigned long long)idx : (0xffffffff00000000ULL | (unsigned)lane));
    if (!cand || (__ffs(peers) - 1) != lane) continue;
    if (atomicCAS((unsigned long long*)map_entry_ptr(m, idx), 0ULL, (unsigned long long)kEntryPending) != 0ULL)
      continue;
    if (idx < map_dense_size(m)) {
      const uint64_t bit = (uint64_t)ph * ps + (uint64_t)(c - 1) * m.dom_tt + (uint64_t)(t - 1);
      atomicOr(&bits[bit >> 5], 1u << (bit & 31));
    } else {  // rare: keys outside the dense map
      const int pos = atomicAdd(&ctl->hash_n, 1);
      hk_tt[pos] = t;
      hk_c[pos] = c;
      hk_p[pos] = (uint8_t)ph;
      hk_e[pos] = idx;
    }
  }
}

// Bitmap -> key list in bit order: per-block popcount totals, a scan of those,
// then one word per thread emits its set bits (block scan for its offset) and
// clears the word for the next batch.
constexpr int kBitThreads = 256;
__global__ void __launch_bounds__(kBitThreads) k_bits_count(const unsigned int* __restrict__ w, int64_t nwords,
                                                           unsigned int* blk_tot) {
  __shared__ unsigned int sm[33];
  const int64_t i = (int64_t)blockIdx.x * kBitThreads + threadIdx.x;
  unsigned int tot;
  block_excl_scan<unsigned int>(i < nwords ? (unsigned)__popc(w[i]) : 0u, tot, sm);
  if (threadIdx.x == 0) blk_tot[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(kBitThreads) k_bits_emit(unsigned int* __restrict__ w, int64_t nwords,
                                                          int64_t plane_words, const unsigned int* __restrict__ blk_off,
                                                          MapView m, int32_t* nk_tt, int32_t* nk_c, uint8_t* nk_p,
                                                          int64_t* nk_e, int* n0) {
  __shared__ unsigned int sm[33];
  const int64_t i = (int64_t)blockIdx.x * kBitThreads + threadIdx.x;
  unsigned int word = i < nwords ? w[i] : 0u;
  unsigned int tot;
  unsigned int ex = blk_off[blockIdx.x] + block_excl_scan<unsigned int>((unsigned)__popc(word), tot, sm);
  if (i == plane_words) *n0 = (int)ex;
  if (!word) return;
  w[i] = 0u;
  const int64_t ps = plane_words * 32;
  while (word) {
    const int b = __ffs(word) - 1;
    word &= word - 1u;
    const int64_t bit = i * 32 + b;
    const int ph = bit >= ps ? 1 : 0;
    const uint32_t r = (uint32_t)(bit - (int64_t)ph * ps);  // < dom_tt * dom_conc < 2^27: 32-bit division
    const uint32_t c0 = r / (uint32_t)m.dom_tt, t0 = r - c0 * (uint32_t)m.dom_tt;
    nk_tt[ex] = t0 + 1;
    nk_c[ex] = c0 + 1;
    nk_p[ex] = (uint8_t)ph;
    nk_e[ex] = ((int64_t)ph * m.dom_tt + t0) * m.dom_conc + c0;  // map_find's dense index
    ex++;
  }
}

// After the bitmap scan: the side-list keys follow the dense ones (straight to
// the warp tier; they are outside every tile) and new_count covers both.
__global__ void k_append_hash(const int32_t* hk_tt, const int32_t* hk_c, const uint8_t* hk_p, const int64_t* hk_e,
                              int32_t* nk_tt, int32_t* nk_c, uint8_t* nk_p, int64_t* nk_e, BatchCtl* ctl,
                              int* fb_list) {
  const int n = ctl->dense_n, nh = ctl->hash_n;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nh; k += gridDim.x * blockDim.x) {
    nk_tt[n + k] = hk_tt[k];
    nk_c[n + k] = hk_c[k];
    nk_p[n + k] = hk_p[k];
    nk_e[n + k] = hk_e[k];
    fb_list[k] = n + k;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->new_count = n + nh;
    ctl->fb_n = nh;
  }
}

// Warp per new key: precomputed candidates -> register sort -> prefix ->
// Shepard CDF; keys without a fast-path window run the full in-warp search,
// and windows too large for a warp are escalated to k_pool_cta.
template <int MODE>
__global__ void __launch_bounds__(kWarpThreads, EMU_WARP_MINB) k_pool_warp(DevTable P0, DevTable P1, Keys keys, Cfg cfg, Sink sk,
                                                            const KeyWin* kw, const long long* resv, int* work,
                                                            int* esc_list, int* esc_count, const int* list,
                                                            const int* list_n) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem + warp * kWarpBytes;
  PoolWS ws;
  ws.d = (double*)base;
  ws.b = (int32_t*)(base + kWarpCap * 8);
  ws.scr = (long long*)(base + kWarpCap * 12);
  ws.dsh = (double*)(base + kWarpCap * 12 + 40 * 8);
  ws.rows = (int32_t*)(base + kWarpCap * 12 + 40 * 8 + 10 * 8);
  ws.n = (int32_t*)(base + kWarpCap * 12 + 40 * 8 + 10 * 8 + 3 * 32 * 4);
  ws.o = ws.n + kWarpCap / 2;
  ws.ncache = kWarpCap / 2;
  ws.cap = kWarpCap;
  // all new keys, or (after the tile tier) the keys it handed over
  const int64_t n = list ? (int64_t)*list_n : keys.count_dev ? (int64_t)*keys.count_dev : keys.count;
  int64_t w_end = 0, w = 0;
  for (;;) {
    if (w >= w_end) {  // grab keys two at a time (dynamic balance, half the atomics)
      int g = 0;
      if (lane == 0) g = atomicAdd(work, 2);
      w = __shfl_sync(kFull, g, 0);
      w_end = w + 2;
    }
    if (w >= n) break;
    const int64_t wk = list ? (int64_t)list[w++] : w++;
    const bool mixed = keys.ph[wk] != 0;
    const DevTable& T = mixed ? P1 : P0;
    const int64_t ent = keys.entry ? keys.entry[wk] : 0;
    const KeyWin k = kw[wk];
    if (k.flags & kWinReady) {
      const long long r = MODE == 0 ? resv[wk] : -1;
      if (r == -2) continue;  // arena overflow: the host flushes and retries
      const int64_t K = pool_from_window(T, keys.tt[wk], keys.conc[wk], cfg.floor, k, ws);
      if (K >= 0) {
        emit_pool<32, MODE>(T, wk, K, ent, 0, true, r, cfg, ws, sk, mixed ? 1 : 0, keys.tt[wk], keys.conc[wk]);
        continue;
      }
      __syncwarp();
    }
    if (k.flags & kWinBig) continue;  // k_pool_prep put it on the group tier's list
    const bool ok = process_key<32, MODE>(T, wk, mixed ? 1 : 0, keys.tt[wk], keys.conc[wk], ent, cfg, ws, sk);
    if (!ok && lane == 0) {
      int e = atomicAdd(esc_count, 1);
      esc_list[e] = (int)wk;
    }
  }
}

// Tile tier (pool_tile.cuh): a warp per 32 consecutive keys of the
// (phase, conc, tt)-ordered new-key list, a lane per key; keys that do not fit
// go to fb_list for the warp tier.
template <int MODE>
__global__ void __launch_bounds__(kTileThreads, EMU_TILE_MINB)
    k_pool_tile(DevTable P0, DevTable P1, Keys keys, Cfg cfg, Sink sk, TileIdx ti, const KeyWin* __restrict__ kw,
                const long long* __restrict__ resv, const int* __restrict__ order, const int* __restrict__ off,
                const int* __restrict__ total, const int* __restrict__ dense_n0, int* work, int* fb_list,
                int* fb_n) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  TileWarp& tw = reinterpret_cast<TileWarp*>(smem)[threadIdx.x >> 5];
  // binned (order != nullptr): keys counting-sorted into tile bins by k_tile_bin;
  // dense: the first *total keys come straight from the cold path's bitmap scan,
  // already in (phase, conc, tt) order, not yet checked for tile eligibility
  const bool dense = order == nullptr;
  const int n0 = dense ? *dense_n0 : ti.base[1] < ti.nb ? off[ti.base[1]] : *total;
  const int p1 = (n0 + 31) & ~31;
  const int nslots = p1 + (*total - n0);
  const int nch = (nslots + 31) >> 5;
  for (;;) {
    int ch = 0;
    if (lane == 0) ch = atomicAdd(work, 1);
    ch = __shfl_sync(kFull, ch, 0);
    if (ch >= nch) break;
    const int pos = ch * 32 + lane;
    const int ph = ch * 32 >= p1 ? 1 : 0;  // a tile never straddles the planes
    const DevTable& T = ph ? P1 : P0;
    int w = -1;
    if (pos < nslots && (pos < n0 || pos >= p1)) w = dense ? (pos < n0 ? pos : n0 + (pos - p1)) : order[pos];
    EMU_DCHECK(w < (keys.count_dev ? *keys.count_dev : keys.count), "CHECK tile w=%d pos=%d n0=%d p1=%d nslots=%d\n", w,
               pos, n0, p1, nslots);
    KeyWin k;
    k.flags = 0;
    int32_t t = 0, c = 0;
    if (w >= 0) {
      k = kw[w];
      t = keys.tt[w];
      c = keys.conc[w];
    }
    if (dense) {  // k_tile_bin's test: ineligible keys leave the tile -- to the warp tier, except big
                  // windows (already on the group tier's list) and keys whose arena reservation failed
                  // in prep (left pending for the host's flush-and-retry)
      bool out = false, fb = false;
      if (w >= 0) {
        const bool pend = MODE == 0 && resv[w] == -2;
        out = pend || tile_bin(T, ti, ph, t, c, k, cfg.floor) < 0;
        fb = out && !pend && !(k.flags & kWinBig);
      }
      warp_push(fb_list, fb_n, fb, w);
      if (out) w = -1;
    }
    const bool has = w >= 0 && k.i0 <= k.i1 && k.j0 <= k.j1;
    const int i0 = __reduce_min_sync(kFull, has ? k.i0 : 0x7fffffff), i1 = __reduce_max_sync(kFull, has ? k.i1 : -1);
    const int j0 = __reduce_min_sync(kFull, has ? k.j0 : 0x7fffffff), j1 = __reduce_max_sync(kFull, has ? k.j1 : -1);
    int Cu = 0;
    if (i0 <= i1 && j0 <= j1) {
      Win u;
      u.i0 = i0;
      u.i1 = i1;
      u.j0 = j0;
      u.j1 = j1;
      Cu = sat_rect(T.bsat, (int32_t)T.gnc + 1, u);
    }
    EMU_STAT(16, 1);
    EMU_STAT(17, Cu);
    if (Cu <= kTileU && Cu > 0) Cu = tile_enum_union(T, i0, i1, j0, j1, tw);
    if (Cu < 0 || Cu > kTileU) {  // union too wide for the tile: every key goes to the warp tier
      if (w >= 0) EMU_LSTAT(18, 1);
      warp_push(fb_list, fb_n, w >= 0, w);
      continue;
    }
    int K = -2;
    if (w >= 0) {
      K = tile_search(T, t, c, k, cfg.floor, Cu, tw);
      EMU_LSTAT(K == -2 ? 19 : K == -3 ? 20 : K == -4 ? 21 : 22, 1);
    }
    EMU_DCHECK(K != 0 && K <= 64, "CHECK tile K=%d w=%d Cu=%d\n", K, w, Cu);
    warp_push(fb_list, fb_n, w >= 0 && K < 0, w);
    if (w >= 0 && K > 0) {
      if (MODE == 0) {
        const long long r = resv[w];
        long long* ep = map_entry_ptr(sk.map, keys.entry[w]);
        if (K > cfg.floor || K > T.nb) {
          report_bad_pool(sk, ph, t, c);
        } else if (K == 1) {  // direct entry: the bucket itself
          const int4 q = tw.u[tw.j[tw.perm[lane] * 32 + lane]];
          *ep = make_entry_direct(T.bkt_off[q.w], q.z);
        } else {
          long long start = r;
          if (start == -1) {
            const unsigned long long tot = (unsigned long long)pool_total_slots(K);
            const unsigned long long st = atomicAdd(sk.arena_used, tot);
            start = (st + tot <= (unsigned long long)sk.arena_cap) ? (long long)st : -2LL;
            if (start < 0) atomicOr(sk.flags, FLAG_ARENA);
          }
          if (start >= 0) {
            const PoolPtrs pp = pool_ptrs(sk.arena, start, K);
            tile_finish<0>(T, K, cfg, tw, &pp, nullptr, nullptr, nullptr, nullptr);
            *ep = make_entry(K, start);
          }
        }
      } else {
        const int64_t base = (int64_t)w * sk.kmax;
        if (K > sk.kmax) {
          sk.x_K[w] = K + (int64_t)1000000;
        } else {
          tile_finish<1>(T, K, cfg, tw, nullptr, sk.x_bkt + base, sk.x_dist + base, sk.x_prob + base, sk.x_cdf + base);
          sk.x_K[w] = K;
        }
      }
    }
    __syncwarp();  // the next tile overwrites the union list
  }
}

// Middle tier: one 128-thread group (CTA) per key escalated by the warp tier
// (windows of 257..2048 candidates, e.g. M = 256 on sparse tables); keys that
// still overflow go on to the CTA tier.
template <int MODE>
__global__ void __launch_bounds__(kGrpThreads, EMU_GRP_MINB) k_pool_grp(DevTable P0, DevTable P1, Keys keys, Cfg cfg, Sink sk,
                                                          const KeyWin* __restrict__ kw, int* work,
                                                          const int* esc_list, const int* esc_count,
                                                          int* esc2_list, int* esc2_count) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long scr[40];
  __shared__ double dsh[10];
  __shared__ int s_w;
  __shared__ int32_t rows[3 * kGrpThreads];
  __shared__ int32_t ncache[2 * kGrpCache];
  PoolWS ws{(double*)smem, (int32_t*)(smem + kGrpCap * 8), kGrpCap, scr, dsh, rows, ncache, ncache + kGrpCache,
            kGrpCache};
  // esc_list == nullptr: every new key, in order (small batches, no k_pool_prep:
  // the group's own 32-lane radius probe finds the window in two rounds)
  const int n = esc_list ? *esc_count : (keys.count_dev ? *keys.count_dev : (int)keys.count);
  for (;;) {
    if (threadIdx.x == 0) s_w = atomicAdd(work, 1);
    __syncthreads();
    const int i = s_w;
    __syncthreads();
    if (i >= n) break;
    const int w = esc_list ? esc_list[i] : i;
    const DevTable& T = keys.ph[w] ? P1 : P0;
    const int64_t ent = keys.entry ? keys.entry[w] : 0;
    KeyWin k;
    k.flags = 0;
    if (kw) k = kw[w];
    const bool ok = process_key<kGrpThreads, MODE>(T, w, keys.ph[w] ? 1 : 0, keys.tt[w], keys.conc[w], ent, cfg, ws,
                                                   sk, (k.flags & (kWinBig | kWinReady)) ? &k : nullptr);
    if (!ok && threadIdx.x == 0) esc2_list[atomicAdd(esc2_count, 1)] = w;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kCtaThreads) k_pool_cta(DevTable P0, DevTable P1, Keys keys, Cfg cfg, Sink sk,
                                                          int* esc_work, const int* esc_list, const int* esc_count,
                                                          double* gd, int32_t* gb, int64_t gcap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long scr[40];
  __shared__ double dsh[10];
  __shared__ int s_w;
  __shared__ int32_t rows[3 * kCtaThreads];
  __shared__ int32_t ncache[2 * kCtaCache];
  PoolWS ws{(double*)smem, (int32_t*)(smem + kCtaCap * 8), kCtaCap, scr, dsh, rows, ncache, ncache + kCtaCache,
            kCtaCache};
  PoolWS wg{gd + (int64_t)blockIdx.x * gcap, gb + (int64_t)blockIdx.x * gcap, gcap, scr, dsh, rows, ncache,
            ncache + kCtaCache, kCtaCache};
  const int n = *esc_count;
  for (;;) {
    if (threadIdx.x == 0) s_w = atomicAdd(esc_work, 1);
    __syncthreads();
    const int i = s_w;
    __syncthreads();
    if (i >= n) break;
    const int w = esc_list[i];
    const bool mixed = keys.ph[w] != 0;
    const DevTable& T = mixed ? P1 : P0;
    const int64_t ent = keys.entry ? keys.entry[w] : 0;
    bool ok = process_key<kCtaThreads, MODE>(T, w, mixed ? 1 : 0, keys.tt[w], keys.conc[w], ent, cfg, ws, sk);
    if (!ok && gd != nullptr) ok = process_key<kCtaThreads, MODE>(T, w, mixed ? 1 : 0, keys.tt[w], keys.conc[w], ent, cfg, wg, sk);
    if (!ok && threadIdx.x == 0) atomicOr(sk.flags, FLAG_MISSING);
  }
}


// Lemire index for query qid after the first word w0 (EXPLICIT: hash32 chain;
// PHILOX: the block-0 spare word, then blocks 1, 2, ... of Philox(qid)).
template <int RNG>
__device__ __forceinline__ uint32_t draw_index(uint32_t n, uint32_t w0, uint4 px, uint64_t qid, uint2 key) {
  if (RNG == EMU_RNG_EXPLICIT) {
    uint32_t st = w0;
    return lemire_index(n, w0, [&]() {
      st = hash32(st);
      return st;
    });
  }
  int pos = 3;
  uint32_t blk = 0;
  uint4 buf = px;
  return lemire_index(n, w0, [&]() {
    if (pos == 4) {
      blk++;
      buf = philox4x32_10(make_uint4((uint32_t)qid, (uint32_t)(qid >> 32), blk, 0u), key);
      pos = 0;
    }
    const uint32_t v = pos == 0 ? buf.x : pos == 1 ? buf.y : pos == 2 ? buf.z : buf.w;
    pos++;
    return v;
  });
}


// One thread handles kQPT queries (block-strided so every load stays
// coalesced) and advances their dependent chains -- map entry, CDF binary
// search, slot, sample -- in lockstep, so 4 independent loads are in flight
// per step.  Per-query inputs/outputs are streamed with evict-first hints so
// the key map, pool arena and samples stay L2-resident.
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p, bool hint) {
  return hint ? __ldcs(p) : *p;
}
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v, bool hint) {
  if (hint)
    __stcs(p, v);
  else
    *p = v;
}

template <int RNG, int QPT, bool HINT>
__global__ void __launch_bounds__(kSampleThreads, (QPT <= 1 ? 8 : QPT == 2 ? 6 : 4)) k_sample(MapView m, const Slot* __restrict__ arena,
                                                           const double* __restrict__ s0, const double* __restrict__ s1,
                                                           const int32_t* __restrict__ qt, const int32_t* __restrict__ qc,
                                                           const uint8_t* __restrict__ qp, int64_t Q,
                                                           const uint64_t* __restrict__ usel,
                                                           const uint32_t* __restrict__ uidx, uint64_t seed,
                                                           uint64_t ctr_base, double* __restrict__ out_lat,
                                                           int32_t* __restrict__ out_sidx, int* flags) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t tile = (int64_t)blockDim.x * QPT;
  for (int64_t base = (int64_t)blockIdx.x * tile + threadIdx.x; base < Q; base += (int64_t)gridDim.x * tile) {
    int64_t i[QPT];
    bool v[QPT];
    int ph[QPT];
    long long e[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      i[j] = base + (int64_t)j * blockDim.x;
      v[j] = i[j] < Q;
      ph[j] = 0;
      int32_t t = 0, c = 0;
      if (v[j]) {
        ph[j] = ld_stream(qp + i[j], HINT) ? 1 : 0;
        t = ld_stream(qt + i[j], HINT);
        c = ld_stream(qc + i[j], HINT);
      }
      const int64_t idx = v[j] ? map_find<false>(m, ph[j], t, c) : -1;
      e[j] = idx >= 0 ? *map_entry_ptr(m, idx) : 0;
    }
    uint64_t us[QPT];
    uint32_t w0[QPT];
    uint4 px[QPT];
    uint64_t u[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      px[j] = make_uint4(0, 0, 0, 0);
      if (RNG == EMU_RNG_EXPLICIT) {
        us[j] = v[j] ? ld_stream(usel + i[j], HINT) : 0;
        w0[j] = v[j] ? ld_stream(uidx + i[j], HINT) : 0;
      } else {
        const uint64_t qid = ctr_base + (uint64_t)i[j];
        px[j] = philox4x32_10(make_uint4((uint32_t)qid, (uint32_t)(qid >> 32), 0u, 0u), key);
        us[j] = (uint64_t)px[j].x | ((uint64_t)px[j].y << 32);
        w0[j] = px[j].z;
      }
      u[j] = unit_k53(us[j]);
    }
    // two-level inverse-CDF lookup (header split, then one 8-slot group)
    PoolPick sl[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++)
      if (v[j] && e[j] > 0) sl[j] = pool_pick(arena, e[j], u[j]);
    double lat[QPT];
    int32_t sidx[QPT];
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      if (!v[j]) continue;
      if (e[j] <= 0) {
        sidx[j] = -1;
        continue;
      }
      const uint32_t k = draw_index<RNG>((uint32_t)sl[j].n, w0[j], px[j], ctr_base + (uint64_t)i[j], key);
      sidx[j] = sl[j].soff + (int32_t)k;
      lat[j] = (ph[j] ? s1 : s0)[sidx[j]];
    }
#pragma unroll
    for (int j = 0; j < QPT; j++) {
      if (!v[j]) continue;
      if (sidx[j] < 0) {
        st_stream(out_lat + i[j], __longlong_as_double(0x7ff8000000000000LL), HINT);
        st_stream(out_sidx + i[j], -1, HINT);
        atomicOr(flags, FLAG_MISSING);
      } else {
        st_stream(out_lat + i[j], lat[j], HINT);
        st_stream(out_sidx + i[j], sidx[j], HINT);
      }
    }
  }
}

// One query's draw from its (built) map entry e: the inverse-CDF pick and the
// Lemire index, exactly as k_sample; writes lat / sidx of query i.
template <int RNG, bool CG = false>
__device__ __forceinline__ void draw_query(const Slot* __restrict__ arena, const double* __restrict__ s0,
                                           const double* __restrict__ s1, long long e, int ph, int64_t i,
                                           const uint64_t* __restrict__ usel, const uint32_t* __restrict__ uidx,
                                           uint2 key, uint64_t ctr_base, double* __restrict__ out_lat,
                                           int32_t* __restrict__ out_sidx, bool hint) {
  uint64_t us;
  uint32_t w0;
  uint4 px = make_uint4(0, 0, 0, 0);
  if (RNG == EMU_RNG_EXPLICIT) {
    us = ld_stream(usel + i, hint);
    w0 = ld_stream(uidx + i, hint);
  } else {
    const uint64_t qid = ctr_base + (uint64_t)i;
    px = philox4x32_10(make_uint4((uint32_t)qid, (uint32_t)(qid >> 32), 0u, 0u), key);
    us = (uint64_t)px.x | ((uint64_t)px.y << 32);
    w0 = px.z;
  }
  const PoolPick sl = pool_pick<CG>(arena, e, unit_k53(us));
  const uint32_t k = draw_index<RNG>((uint32_t)sl.n, w0, px, ctr_base + (uint64_t)i, key);
  const int32_t sidx = sl.soff + (int32_t)k;
  st_stream(out_lat + i, ldp<CG>((ph ? s1 : s0) + sidx), hint);
  st_stream(out_sidx + i, sidx, hint);
}

// Streaming sweep for a cache that already holds most keys: ONE pass over the
// queries.  A query whose pool is built is drawn at once; any other query is
// appended to the miss list (and its key claimed and appended to the new-key
// list, as k_mark does).  After the pool tiers, k_sample_list draws the misses
// only, so each key / uniform is read from HBM once (41 B/query explicit).
template <int RNG, bool CG>
__global__ void __launch_bounds__(kSampleThreads, 8) k_sweep(MapView m, const Slot* __restrict__ arena,
                                                             const double* __restrict__ s0,
                                                             const double* __restrict__ s1,
                                                             const int32_t* __restrict__ qt,
                                                             const int32_t* __restrict__ qc,
                                                             const uint8_t* __restrict__ qp, int64_t Q,
                                                             const uint64_t* __restrict__ usel,
                                                             const uint32_t* __restrict__ uidx, uint64_t seed,
                                                             uint64_t ctr_base, double* __restrict__ out_lat,
                                                             int32_t* __restrict__ out_sidx, int32_t* nk_tt,
                                                             int32_t* nk_c, uint8_t* nk_p, int64_t* nk_e, int* miss,
                                                             BatchCtl* ctl) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < Q; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;  // warp-uniform trip count: every ballot has all lanes
    const bool v = i < Q;
    int ph = 0;
    int32_t t = 0, c = 0;
    if (v) {
      ph = __ldcs(qp + i) ? 1 : 0;
      t = __ldcs(qt + i);
      c = __ldcs(qc + i);
    }
    const int64_t idx = v ? map_find<true>(m, ph, t, c) : -2;
    const long long e = idx >= 0 ? ldp<CG>(map_entry_ptr(m, idx)) : -1;
    if (idx == -1) atomicOr(&ctl->flags, FLAG_HASH);
    const bool hit = e > 0;
    if (hit) draw_query<RNG, CG>(arena, s0, s1, e, ph, i, usel, uidx, key, ctr_base, out_lat, out_sidx, true);
    // claim empty entries: one CAS per distinct key per warp
    const bool cand = idx >= 0 && e == kEntryEmpty;
    bool won = false;
    if (__any_sync(kFull, cand)) {
      const unsigned peers =
          __match_any_sync(kFull, cand ? (unsigned long long)idx : (0xffffffff00000000ULL | (unsigned)lane));
      if (cand && (__ffs(peers) - 1) == lane)
        won = atomicCAS((unsigned long long*)map_entry_ptr(m, idx), 0ULL, (unsigned long long)kEntryPending) == 0ULL;
    }
    const unsigned mb = __ballot_sync(kFull, v && !hit);
    if (mb) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&ctl->miss_count, __popc(mb));
      base = __shfl_sync(kFull, base, 0);
      if (v && !hit) miss[base + __popc(mb & lt)] = (int)i;
    }
    const unsigned wb = __ballot_sync(kFull, won);
    if (wb) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&ctl->new_count, __popc(wb));
      base = __shfl_sync(kFull, base, 0);
      if (won) {
        const int pos = base + __popc(wb & lt);
        nk_tt[pos] = t;
        nk_c[pos] = c;
        nk_p[pos] = (uint8_t)ph;
        nk_e[pos] = idx;
      }
    }
  }
}

// The misses of k_sweep, after the pool tiers built their pools (gathered by
// query index; the list is a small fraction of the sweep on a warm cache).
template <int RNG>
__global__ void __launch_bounds__(kSampleThreads, 8) k_sample_list(MapView m, const Slot* __restrict__ arena,
                                                                   const double* __restrict__ s0,
                                                                   const double* __restrict__ s1,
                                                                   const int32_t* __restrict__ qt,
                                                                   const int32_t* __restrict__ qc,
                                                                   const uint8_t* __restrict__ qp,
                                                                   const int* __restrict__ list,
                                                                   const int* __restrict__ list_n,
                                                                   const uint64_t* __restrict__ usel,
                                                                   const uint32_t* __restrict__ uidx, uint64_t seed,
                                                                   uint64_t ctr_base, double* __restrict__ out_lat,
                                                                   int32_t* __restrict__ out_sidx, int* flags) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int n = *list_n;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int64_t i = list[j];
    const int ph = qp[i] ? 1 : 0;
    const int64_t idx = map_find<false>(m, ph, qt[i], qc[i]);
    const long long e = idx >= 0 ? *map_entry_ptr(m, idx) : 0;
    if (e > 0) {
      draw_query<RNG>(arena, s0, s1, e, ph, i, usel, uidx, key, ctr_base, out_lat, out_sidx, false);
    } else {
      out_lat[i] = __longlong_as_double(0x7ff8000000000000LL);
      out_sidx[i] = -1;
      atomicOr(flags, FLAG_MISSING);
    }
  }
}

// Compacting sampler: a warp takes 32*CQ queries (CQ per lane, coalesced),
// finishes the direct-entry ones (single-bucket pools: entry -> sample) at
// once and queues the rest in shared memory; the queue is then drained with
// every lane busy (header -> cdf group -> bucket data -> sample).  ~71 % of
// the config-2 queries are direct, so the pool path runs on dense warps
// instead of on every warp with a third of its lanes.
struct PendingDraw {
  long long e;
  uint64_t us;
  uint32_t w0, pw;
  int32_t rel;
  int32_t pad;
};

template <int RNG, int CQ>
__global__ void __launch_bounds__(256) k_sample_c(MapView m, const Slot* __restrict__ arena,
                                                  const double* __restrict__ s0, const double* __restrict__ s1,
                                                  const int32_t* __restrict__ qt, const int32_t* __restrict__ qc,
                                                  const uint8_t* __restrict__ qp, int64_t Q,
                                                  const uint64_t* __restrict__ usel, const uint32_t* __restrict__ uidx,
                                                  uint64_t seed, uint64_t ctr_base, double* __restrict__ out_lat,
                                                  int32_t* __restrict__ out_sidx, int* flags) {
  __shared__ PendingDraw qs[8][32 * CQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  PendingDraw* wq = qs[warp];
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t tb = ((int64_t)blockIdx.x * 8 + warp) * (32 * CQ); tb < Q; tb += nwarps * (32 * CQ)) {
    int np = 0;
#pragma unroll
    for (int j = 0; j < CQ; j++) {
      const int rel = j * 32 + lane;
      const int64_t i = tb + rel;
      const bool v = i < Q;
      int ph = 0;
      long long e = 0;
      uint64_t us = 0;
      uint32_t w0 = 0, pw = 0;
      if (v) {
        ph = __ldcs(qp + i) ? 1 : 0;
        const int64_t idx = map_find<false>(m, ph, __ldcs(qt + i), __ldcs(qc + i));
        e = idx >= 0 ? *map_entry_ptr(m, idx) : 0;
        if (RNG == EMU_RNG_EXPLICIT) {
          us = __ldcs(usel + i);
          w0 = __ldcs(uidx + i);
        } else {
          const uint64_t qid = ctr_base + (uint64_t)i;
          const uint4 px = philox4x32_10(make_uint4((uint32_t)qid, (uint32_t)(qid >> 32), 0u, 0u), key);
          us = (uint64_t)px.x | ((uint64_t)px.y << 32);
          w0 = px.z;
          pw = px.w;
        }
      }
      const bool direct = v && e > 0 && ((unsigned long long)e & kEntryDirect);
      const bool pend = v && e > 0 && !direct;
      if (direct) {
        const unsigned long long ev = (unsigned long long)e;
        const int32_t soff = (int32_t)((ev >> 31) & 0x7fffffffULL), n = (int32_t)(ev & 0x7fffffffULL);
        const uint32_t k = draw_index<RNG>((uint32_t)n, w0, make_uint4(0, 0, 0, pw), ctr_base + (uint64_t)i, key);
        const int32_t sidx = soff + (int32_t)k;
        __stcs(out_lat + i, (ph ? s1 : s0)[sidx]);
        __stcs(out_sidx + i, sidx);
      } else if (v && e <= 0) {
        __stcs(out_lat + i, __longlong_as_double(0x7ff8000000000000LL));
        __stcs(out_sidx + i, -1);
        atomicOr(flags, FLAG_MISSING);
      }
      const unsigned bal = __ballot_sync(kFull, pend);
      if (pend) {
        PendingDraw& P = wq[np + __popc(bal & lt)];
        P.e = e;
        P.us = us;
        P.w0 = w0;
        P.pw = pw;
        P.rel = rel | (ph << 30);
      }
      np += __popc(bal);
    }
    __syncwarp();
    for (int k = lane; k < np; k += 32) {
      const PendingDraw P = wq[k];
      const int64_t i = tb + (P.rel & 0x3fffffff);
      const int ph = P.rel >> 30;
      const PoolPick pk = pool_pick(arena, P.e, unit_k53(P.us));
      const uint32_t kk = draw_index<RNG>((uint32_t)pk.n, P.w0, make_uint4(0, 0, 0, P.pw), ctr_base + (uint64_t)i, key);
      const int32_t sidx = pk.soff + (int32_t)kk;
      __stcs(out_lat + i, (ph ? s1 : s0)[sidx]);
      __stcs(out_sidx + i, sidx);
    }
    __syncwarp();
  }
}

// One query per thread with the next grid-stride iteration's stream inputs
// (keys, uniforms) loaded before the current query's dependent L2 chain
// (entry -> pool -> bucket -> sample): the DRAM latency of the streams hides
// behind the chain instead of adding to it.
template <int RNG>
__global__ void __launch_bounds__(kSampleThreads, 8) k_sample_pf(MapView m, const Slot* __restrict__ arena,
                                                                 const double* __restrict__ s0,
                                                                 const double* __restrict__ s1,
                                                                 const int32_t* __restrict__ qt,
                                                                 const int32_t* __restrict__ qc,
                                                                 const uint8_t* __restrict__ qp, int64_t Q,
                                                                 const uint64_t* __restrict__ usel,
                                                                 const uint32_t* __restrict__ uidx, uint64_t seed,
                                                                 uint64_t ctr_base, double* __restrict__ out_lat,
                                                                 int32_t* __restrict__ out_sidx, int* flags) {
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t t = 0, c = 0;
  uint8_t p = 0;
  uint64_t us = 0;
  uint32_t w0 = 0;
  if (i < Q) {
    p = __ldcs(qp + i);
    t = __ldcs(qt + i);
    c = __ldcs(qc + i);
    if (RNG == EMU_RNG_EXPLICIT) {
      us = __ldcs(usel + i);
      w0 = __ldcs(uidx + i);
    }
  }
  for (; i < Q; i += stride) {
    const int64_t nx = i + stride;
    int32_t nt = 0, nc = 0;
    uint8_t np_ = 0;
    uint64_t nus = 0;
    uint32_t nw0 = 0;
    if (nx < Q) {
      np_ = __ldcs(qp + nx);
      nt = __ldcs(qt + nx);
      nc = __ldcs(qc + nx);
      if (RNG == EMU_RNG_EXPLICIT) {
        nus = __ldcs(usel + nx);
        nw0 = __ldcs(uidx + nx);
      }
    }
    const int ph = p ? 1 : 0;
    const int64_t idx = map_find<false>(m, ph, t, c);
    const long long e = idx >= 0 ? *map_entry_ptr(m, idx) : 0;
    uint4 px = make_uint4(0, 0, 0, 0);
    if (RNG != EMU_RNG_EXPLICIT) {
      const uint64_t qid = ctr_base + (uint64_t)i;
      px = philox4x32_10(make_uint4((uint32_t)qid, (uint32_t)(qid >> 32), 0u, 0u), key);
      us = (uint64_t)px.x | ((uint64_t)px.y << 32);
      w0 = px.z;
    }
    if (e > 0) {
      const PoolPick pk = pool_pick(arena, e, unit_k53(us));
      const uint32_t k = draw_index<RNG>((uint32_t)pk.n, w0, px, ctr_base + (uint64_t)i, key);
      const int32_t sidx = pk.soff + (int32_t)k;
      __stcs(out_lat + i, (ph ? s1 : s0)[sidx]);
      __stcs(out_sidx + i, sidx);
    } else {
      __stcs(out_lat + i, __longlong_as_double(0x7ff8000000000000LL));
      __stcs(out_sidx + i, -1);
      atomicOr(flags, FLAG_MISSING);
    }
    t = nt;
    c = nc;
    p = np_;
    us = nus;
    w0 = nw0;
  }
}

__device__ __forceinline__ Pcg64 load_pcg(const uint64_t* st6) {
  Pcg64 g;
  g.s_hi = st6[0];
  g.s_lo = st6[1];
  g.i_hi = st6[2];
  g.i_lo = st6[3];
  g.has_u32 = (uint32_t)st6[4];
  g.u32 = (uint32_t)st6[5];
  return g;
}

__device__ __forceinline__ void store_pcg(uint64_t* st6, const Pcg64& g) {
  st6[0] = g.s_hi;
  st6[1] = g.s_lo;
  st6[2] = g.i_hi;
  st6[3] = g.i_lo;
  st6[4] = g.has_u32;
  st6[5] = g.u32;
}

// One draw of LatencyOracle.sample on the PCG64 stream: choice() draws one
// double; integers(n) draws buffered u32 words only when n > 1.
__device__ __forceinline__ int32_t pcg_draw(Pcg64& g, const Slot* arena, long long e) {
  const PoolPick s = pool_pick(arena, e, unit_k53(pcg64_next64(g)));
  uint32_t j = 0;
  if (s.n > 1) {
    uint32_t w0 = pcg64_next32(g);
    j = lemire_index((uint32_t)s.n, w0, [&]() { return pcg64_next32(g); });
  }
  return s.soff + (int32_t)j;
}

__global__ void k_sample_pcg(MapView m, const Slot* __restrict__ arena, const double* __restrict__ s0,
                             const double* __restrict__ s1, const int32_t* __restrict__ qt,
                             const int32_t* __restrict__ qc, const uint8_t* __restrict__ qp, int64_t Q, uint64_t* st6,
                             double* __restrict__ out_lat, int32_t* __restrict__ out_sidx, int* flags) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Pcg64 g = load_pcg(st6);
  for (int64_t i = 0; i < Q; i++) {
    const int ph = qp[i] ? 1 : 0;
    const int64_t idx = map_find<false>(m, ph, qt[i], qc[i]);
    const long long e = idx >= 0 ? *map_entry_ptr(m, idx) : 0;
    if (e <= 0) {
      atomicOr(flags, FLAG_MISSING);
      return;  // stream state left untouched: the host retries the whole batch
    }
    const int32_t sidx = pcg_draw(g, arena, e);
    out_lat[i] = (ph ? s1 : s0)[sidx];
    out_sidx[i] = sidx;
  }
  store_pcg(st6, g);
}

// Single engine step: claim/build the key's pool if needed (one CTA), then
// one PCG64 draw.  The whole per-step backend call in one launch.
__global__ void __launch_bounds__(kCtaThreads) k_step(DevTable P0, DevTable P1, Cfg cfg, Sink sk, int32_t t, int32_t c,
                                                      int ph, uint64_t* st6, double* gd, int32_t* gb, int64_t gcap,
                                                      StepOut* out, uint32_t seq) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ long long scr[40];
  __shared__ double dsh[10];
  __shared__ long long s_idx, s_e;
  __shared__ int32_t rows[3 * kCtaThreads];
  __shared__ int32_t ncache[2 * kCtaCache];
  const DevTable& T = ph ? P1 : P0;
  if (threadIdx.x == 0) {
    *sk.flags = 0;
    int64_t idx = map_find<true>(sk.map, ph, t, c);
    long long e = -2;
    if (idx >= 0) {
      long long* ep = map_entry_ptr(sk.map, idx);
      e = *ep;
      if (e == kEntryEmpty) *ep = kEntryPending;
    }
    s_idx = idx;
    s_e = e;
  }
  __syncthreads();
  const long long idx = s_idx;
  if (idx < 0) {
    if (threadIdx.x == 0) publish_step(out, 0.0, -1, FLAG_HASH, seq);
    return;
  }
  if (s_e == kEntryEmpty) {
    PoolWS ws{(double*)smem, (int32_t*)(smem + kCtaCap * 8), kCtaCap, scr, dsh, rows, ncache,
              ncache + kCtaCache, kCtaCache};
    bool ok = process_key<kCtaThreads, 0>(T, 0, ph, t, c, idx, cfg, ws, sk);
    if (!ok && gd != nullptr) {
      PoolWS wg{gd, gb, gcap, scr, dsh, rows, ncache, ncache + kCtaCache, kCtaCache};
      ok = process_key<kCtaThreads, 0>(T, 0, ph, t, c, idx, cfg, wg, sk);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long e = *(volatile long long*)map_entry_ptr(sk.map, idx);
    if (e <= 0) {
      publish_step(out, 0.0, -1, *sk.flags & FLAG_ARENA ? FLAG_ARENA : *sk.flags & FLAG_BADPOOL ? FLAG_BADPOOL : FLAG_MISSING,
                   seq);
      return;
    }
    Pcg64 g = load_pcg(st6);
    const int32_t sidx = pcg_draw(g, sk.arena, e);
    store_pcg(st6, g);
    publish_step(out, T.samples[sidx], sidx, 0, seq);
  }
}

constexpr int32_t kStepMiss = 8;  // k_step_hit: key not cached yet, run k_step

// Cached-key fast path of an engine step: one thread, no shared memory.
__global__ void k_step_hit(MapView m, const Slot* __restrict__ arena, const double* __restrict__ s0,
                           const double* __restrict__ s1, int32_t t, int32_t c, int ph, uint64_t* st6, StepOut* out,
                           uint32_t seq) {
  if (threadIdx.x != 0) return;
  const int64_t idx = map_find<false>(m, ph, t, c);
  const long long e = idx >= 0 ? *(volatile long long*)map_entry_ptr(m, idx) : 0;
  if (e <= 0) {
    publish_step(out, 0.0, -1, kStepMiss, seq);
    return;
  }
  Pcg64 g = load_pcg(st6);
  const int32_t sidx = pcg_draw(g, arena, e);
  store_pcg(st6, g);
  publish_step(out, (ph ? s1 : s0)[sidx], sidx, 0, seq);
}

// ------------------------------------------------------------ step server
// The engine calls the oracle once per step, synchronously (engine.py:555-557),
// so a kernel launch per call dominates its latency.  The step server is a
// one-warp kernel that stays resident while steps keep coming: the host writes
// a request into mapped pinned memory, lane 0 sees it over PCIe, serves it
// exactly like k_step_hit (cached keys; misses go back to the host, which
// launches k_step) and writes the result back into mapped memory.  It exits
// after `idle_ns` without a request or after `max_ns`; the host relaunches it
// on demand.  The idle timeout (EMU_STEP_SERVER_IDLE_US, default 100 ms) is
// longer than the engine's step cadence (it sleeps the sampled latency between
// calls, engine.py:565: ms), so the server survives the gaps; whenever the
// library itself needs the server gone (reallocation, destroy) or the caller
// wants a prompt device-wide sync (emu_oracle_park), the host sets the park
// bit in the request's phase word and the server exits on its next poll.
// Requests carry a sequence number; a (re)started server first serves any
// request it has not served yet, so a request written while the server was
// exiting is never lost.
struct __align__(16) StepReq {
  uint32_t seq;
  int32_t tt, conc, phase;  // phase bit 31: park (exit now) when no request is pending
};
constexpr uint32_t kParkBit = 0x80000000u;

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_step_server(MapView m, const Slot* __restrict__ arena, const double* __restrict__ s0,
                              const double* __restrict__ s1, uint64_t* st6, const StepReq* req, StepOut* out,
                              uint32_t* served_dev, volatile int* alive, uint64_t idle_ns, uint64_t max_ns) {
  if (threadIdx.x != 0) return;
  uint32_t served = *(volatile uint32_t*)served_dev;
  const uint64_t t0 = global_ns();
  uint64_t t_last = t0;
  for (;;) {
    // one 16-byte read over PCIe: the host writes the fields before the
    // sequence number (x86 store order), so a snapshot with a new seq has them
    uint32_t sq, ut, uc, up;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(sq), "=r"(ut), "=r"(uc), "=r"(up)
                 : "l"(req));
    if (sq != served) {
      const int32_t t = (int32_t)ut, c = (int32_t)uc, ph = (up & ~kParkBit) ? 1 : 0;
      const int64_t idx = map_find<false>(m, ph, t, c);
      const long long e = idx >= 0 ? __ldcg(map_entry_ptr(m, idx)) : 0;
      if (e <= 0) {
        publish_step(out, 0.0, -1, 8 /* kStepMiss */, sq);
      } else {
        Pcg64 g;
        g.s_hi = __ldcg(st6 + 0);
        g.s_lo = __ldcg(st6 + 1);
        g.i_hi = __ldcg(st6 + 2);
        g.i_lo = __ldcg(st6 + 3);
        g.has_u32 = (uint32_t)__ldcg(st6 + 4);
        g.u32 = (uint32_t)__ldcg(st6 + 5);
        const PoolPick pk = pool_pick<true>(arena, e, unit_k53(pcg64_next64(g)));
        uint32_t j = 0;
        if (pk.n > 1) {
          const uint32_t w0 = pcg64_next32(g);
          j = lemire_index((uint32_t)pk.n, w0, [&]() { return pcg64_next32(g); });
        }
        const int32_t sidx = pk.soff + (int32_t)j;
        __stcg(st6 + 0, g.s_hi);
        __stcg(st6 + 1, g.s_lo);
        __stcg(st6 + 2, g.i_hi);
        __stcg(st6 + 3, g.i_lo);
        __stcg(st6 + 4, (uint64_t)g.has_u32);
        __stcg(st6 + 5, (uint64_t)g.u32);
        __threadfence();
        publish_step(out, __ldcg((ph ? s1 : s0) + sidx), sidx, 0, sq);
      }
      served = sq;
      *(volatile uint32_t*)served_dev = served;
      t_last = global_ns();
      continue;
    }
    const uint64_t now = global_ns();
    if ((up & kParkBit) || now - t_last > idle_ns || now - t0 > max_ns) break;
  }
  __threadfence();
  *alive = 0;
  __threadfence_system();
}

__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_gather_pools(const int64_t* __restrict__ x_K, const int64_t* __restrict__ off, int64_t n, int64_t kmax,
                               int64_t out_base, const int32_t* xb, const double* xd, const double* xp, const double* xc,
                               int32_t* ob, double* od, double* op, double* oc, int64_t cap) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nw) {
    const int64_t K = x_K[u], o = off[u] - out_base;
    for (int64_t j = lane; j < K; j += 32) {
      if (off[u] + j >= cap) break;
      ob[o + j] = xb[u * kmax + j];
      od[o + j] = xd[u * kmax + j];
      op[o + j] = xp[u * kmax + j];
      oc[o + j] = xc[u * kmax + j];
    }
  }
}

__global__ void k_table_of_key(const uint8_t* kp, int64_t U, int t0, int t1, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < U; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = kp[i] ? t1 : t0;
}

// ------------------------------------------------------------- host side
static int grid_for(int64_t n, int threads, int max_blocks) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

template <typename T>
static int dalloc(T** p, int64_t n) {
  *p = nullptr;
  EMU_CUDA(cudaMalloc((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1)));
  return EMU_OK;
}

static bool g_attrs_set = false;
static int set_kernel_attrs() {
  if (g_attrs_set) return EMU_OK;
  EMU_CUDA(cudaFuncSetAttribute(k_pool_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarpBytes * kWarpsPerCta));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarpBytes * kWarpsPerCta));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_tile<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_grp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGrpSmem));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_grp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGrpSmem));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_cta<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem));
  EMU_CUDA(cudaFuncSetAttribute(k_pool_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem));
  EMU_CUDA(cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSmem));
  g_attrs_set = true;
  return EMU_OK;
}

}  // namespace emu

using namespace emu;

struct emu_oracle_s {
  emu_tables_t T = nullptr;
  Cfg cfg{};
  int plane_tab[2] = {0, 1};
  DevTable plane[2];
  bool has_data = false;
  int64_t kmax = 1;  // max pool size: min(floor, max plane buckets)
  // key map
  MapView map{};
  // arena
  Slot* arena = nullptr;
  int64_t arena_cap = 0;
  unsigned long long* arena_used = nullptr;
  // batch scratch
  BatchCtl* ctl = nullptr;
  int32_t* nk_tt = nullptr;
  int32_t* nk_c = nullptr;
  uint8_t* nk_p = nullptr;
  int64_t* nk_e = nullptr;
  int* esc = nullptr;
  int* esc2 = nullptr;
  int64_t chunk_cap = 0;
  bool cold = true;          // cache flushed since the last batch: the head of the next batch takes the mark path
  bool sweep_ok = false;     // the last chunk met few new keys: warm chunks take the one-pass k_sweep
  bool last_swept = false;   // the last chunk went through k_sweep (its miss count is in ctl_host)
  int* miss = nullptr;       // k_sweep miss list (query indices)
  int64_t miss_cap = 0;
  int64_t arena_max = 0;  // growth limit for the pool arena (slots)
  int64_t nk_cap = 0;  // allocated new-key capacity (lazy)
  KeyWin* kw = nullptr;
  long long* resv = nullptr;
  // tile tier: ordering bins and per-key scratch (EMU_TILE=0 disables the tier)
  bool tile_on = true;
  TileIdx ti{};
  int* tile_cnt = nullptr;   // ti.nb + 1
  int* tile_off = nullptr;   // ti.nb + 1
  int* tile_part = nullptr;  // scan partials
  int* kbin = nullptr;
  int* krank = nullptr;
  int* order = nullptr;
  int* fb_list = nullptr;
  // cold-path dedupe bitmap over the dense key domain (self-clearing) and the
  // side list of keys outside it
  unsigned int* bits = nullptr;
  int64_t bits_words = 0;
  unsigned int* bits_part = nullptr;
  int32_t* hk_tt = nullptr;
  int32_t* hk_c = nullptr;
  uint8_t* hk_p = nullptr;
  int64_t* hk_e = nullptr;
  // CTA global scratch
  double* gd = nullptr;
  int32_t* gb = nullptr;
  int64_t gcap = 0;
  // rng / step
  uint64_t* pcg = nullptr;
  StepOut* step_dev = nullptr;   // device alias of step_host (mapped)
  // step server (k_step_server): mapped request mailbox + liveness flag
  StepReq* req_host = nullptr;
  StepReq* req_dev = nullptr;
  int* alive_host = nullptr;
  int* alive_dev = nullptr;
  uint32_t* served_dev = nullptr;
  cudaStream_t srv_stream = nullptr;
  cudaEvent_t async_done = nullptr;  // recorded after asynchronous calls (flush)
  cudaEvent_t srv_done = nullptr;    // recorded after each server launch: completed = not running
  bool async_pending = false;
  bool server = true;                // EMU_STEP_SERVER=0 disables
  StepOut* step_host = nullptr;  // pinned, mapped
  uint32_t step_seq = 0;
  int* flags_host = nullptr;
  BatchCtl* ctl_host = nullptr;  // pinned: the head of BatchCtl after a k_sweep
  // host staging for emu_oracle_sample_host (pipelined: copy-in stream,
  // compute on the caller's stream, copy-out stream; one event pair per chunk)
  void* stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_cmp;
  cudaEvent_t ev_start = nullptr;
  int* flag_log = nullptr;  // device: flags of each pipelined chunk
  int* flag_log_host = nullptr;
  int64_t flag_log_cap = 0;
};

static Sink make_sink(emu_oracle_t o) {
  Sink s{};
  s.map = o->map;
  s.arena = o->arena;
  s.arena_cap = o->arena_cap;
  s.arena_used = o->arena_used;
  s.flags = &o->ctl->flags;
  s.bad_key = o->ctl->bad_key;
  s.kmax = o->kmax;
  return s;
}

// FLAG_BADPOOL: fail the call naming the first offending key.
static int bad_pool_error(emu_oracle_t o, cudaStream_t s) {
  int bk[4] = {0, 0, 0, 0};
  EMU_CUDA(cudaMemcpyAsync(bk, o->ctl->bad_key, sizeof(bk), cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  return fail(EMU_ERR_CUDA, "internal error: invalid pool (K > min(floor, buckets)) for key phase=" +
                                std::to_string(bk[1]) + " tt=" + std::to_string(bk[2]) + " conc=" + std::to_string(bk[3]));
}

static int oracle_flush(emu_oracle_t o, cudaStream_t s) {
  o->cold = true;
  int64_t D = 2LL * o->map.dom_tt * o->map.dom_conc;
  EMU_CUDA(cudaMemsetAsync(o->map.dense, 0, sizeof(long long) * D, s));
  EMU_LAUNCH("flush", s, k_fill_u64<<<grid_for(2 * o->map.hcap, 256, 4096), 256, 0, s>>>(o->map.hkeys, 2 * o->map.hcap, kHashEmpty));
  EMU_CUDA(cudaGetLastError());
  EMU_CUDA(cudaMemsetAsync(o->map.hvals, 0, sizeof(long long) * 2 * o->map.hcap, s));
  EMU_CUDA(cudaMemsetAsync(o->arena_used, 0, sizeof(unsigned long long), s));
  return EMU_OK;
}

namespace emu {
int oracle_views(emu_oracle_t o, MapView* m, const Slot** arena, const double** s0, const double** s1) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  *m = o->map;
  *arena = o->arena;
  *s0 = o->plane[0].samples;
  *s1 = o->plane[1].samples;
  return EMU_OK;
}
}  // namespace emu

// Park the step server (it exits on its next poll) and wait for it, before the
// arrays it was launched with are reallocated or freed.
static void quiesce_server(emu_oracle_t o) {
  if (!o->srv_stream) return;
  if (o->req_host) {
    volatile StepReq* rq = o->req_host;
    rq->phase = (int32_t)kParkBit;  // seq unchanged: no request pending
    std::atomic_thread_fence(std::memory_order_seq_cst);
  }
  cudaStreamSynchronize(o->srv_stream);
}

static int alloc_hash(emu_oracle_t o, int64_t hcap) {
  quiesce_server(o);
  cudaFree(o->map.hkeys);
  cudaFree(o->map.hvals);
  o->map.hkeys = nullptr;
  o->map.hvals = nullptr;
  int rc;
  if ((rc = dalloc(&o->map.hkeys, 2 * hcap)) || (rc = dalloc(&o->map.hvals, 2 * hcap))) return rc;
  o->map.hcap = hcap;
  return EMU_OK;
}

static int64_t pow2_at_least(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

extern "C" {

int emu_oracle_create(emu_tables_t t, int32_t floor, double shepard_power, double epsilon, int32_t dom_tt,
                      int32_t dom_conc, int64_t arena_slots, int64_t hash_slots, void* stream, emu_oracle_t* out) {
  if (!out || !t) return fail(EMU_ERR_INVALID, "NULL tables/out");
  *out = nullptr;
  if (floor < 1) return fail(EMU_ERR_INVALID, "reliability_floor must be >= 1, got " + std::to_string(floor));
  if (!(shepard_power > 0)) return fail(EMU_ERR_INVALID, "shepard_power must be > 0");
  if (!(epsilon > 0)) return fail(EMU_ERR_INVALID, "epsilon_distance must be > 0");
  int rc = set_kernel_attrs();
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  auto* o = new emu_oracle_s();
  o->T = t;
  o->cfg.floor = floor;
  o->cfg.p = shepard_power;
  o->cfg.eps = epsilon;
  int64_t max_nb = 1;
  int32_t tt_hi = 1, c_hi = 1;
  for (int ph = 0; ph < 2; ph++) {
    o->plane_tab[ph] = t->tab[ph].nb > 0 ? ph : 2;
    o->plane[ph] = t->tab[o->plane_tab[ph]].view();
    max_nb = std::max(max_nb, t->tab[o->plane_tab[ph]].nb);
  }
  for (int i = 0; i < 3; i++) {
    if (t->tab[i].nb > 0) {
      tt_hi = std::max(tt_hi, t->tab[i].tt_hi);
      c_hi = std::max(c_hi, t->tab[i].c_hi);
    }
  }
  o->has_data = t->tab[2].nb > 0;
  o->kmax = std::min<int64_t>(floor, max_nb);
  int64_t dt = dom_tt > 0 ? dom_tt : tt_hi, dc = dom_conc > 0 ? dom_conc : c_hi;
  const int64_t kMaxDense = 1LL << 27;
  while (2 * dt * dc > kMaxDense && dt > 1) dt = (dt + 1) / 2;
  if (2 * dt * dc > kMaxDense) dc = std::max<int64_t>(1, kMaxDense / (2 * dt));
  o->map.dom_tt = (int32_t)dt;
  o->map.dom_conc = (int32_t)dc;
  o->arena_cap = arena_slots > 0 ? arena_slots : (1LL << 26);
  if (o->arena_cap > 0x7fffffffLL) o->arena_cap = 0x7fffffffLL;
  if (arena_slots > 0) {
    o->arena_max = o->arena_cap;  // caller-fixed size: chunk instead of growing
  } else {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    o->arena_max = std::max<int64_t>(o->arena_cap, std::min<int64_t>(0x7fffffffLL, (int64_t)(free_b / 4 / sizeof(Slot))));
  }
  int64_t hcap = pow2_at_least(hash_slots > 0 ? hash_slots : (1LL << 16));
  o->chunk_cap = 1LL << 24;
  o->gcap = pow2_at_least(max_nb);
  bool need_global = o->gcap > kCtaCap;
  if ((rc = dalloc(&o->map.dense, 2 * dt * dc)) || (rc = alloc_hash(o, hcap)) || (rc = dalloc(&o->arena, o->arena_cap + kArenaSlack)) ||
      (rc = dalloc(&o->arena_used, 1)) || (rc = dalloc(&o->ctl, 1)) || (rc = dalloc(&o->pcg, 6)) ||

      (need_global && ((rc = dalloc(&o->gd, kCtaGrid * o->gcap)) || (rc = dalloc(&o->gb, kCtaGrid * o->gcap))))) {
    emu_oracle_destroy(o);
    return rc;
  }
  // a draw's wide loads also read a pool's padding: keep the whole arena initialized
  if (cudaMemset(o->arena, 0, sizeof(Slot) * (o->arena_cap + kArenaSlack)) != cudaSuccess) {
    emu_oracle_destroy(o);
    return cuda_fail(cudaGetLastError(), "arena memset");
  }
  {
    const char* tv = getenv("EMU_TILE");
    o->tile_on = !(tv && tv[0] == '0');
    int64_t nb = 0;
    for (int ph = 0; ph < 2; ph++) {
      const DevTable& T = o->plane[ph];
      o->ti.base[ph] = nb;
      o->ti.nbt[ph] = T.gnt > 0 ? (T.gnt + (1 << kTileRowShift) - 1) >> kTileRowShift : 0;
      nb += o->ti.nbt[ph] * T.gnc;
    }
    o->ti.nb = nb;
    if (nb == 0 || nb > (1LL << 26)) o->tile_on = false;
    if (o->tile_on && ((rc = dalloc(&o->tile_cnt, nb + 1)) || (rc = dalloc(&o->tile_off, nb + 1)) ||
                       (rc = dalloc(&o->tile_part, (nb + kScanTile) / kScanTile + 1)))) {
      emu_oracle_destroy(o);
      return rc;
    }
  }
  if (cudaHostAlloc((void**)&o->step_host, sizeof(StepOut), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&o->step_dev, o->step_host, 0) != cudaSuccess ||
      cudaHostAlloc((void**)&o->flags_host, sizeof(int) * 4, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void**)&o->ctl_host, sizeof(BatchCtl), cudaHostAllocDefault) != cudaSuccess) {
    emu_oracle_destroy(o);
    return fail(EMU_ERR_CUDA, "cudaHostAlloc failed");
  }
  memset((void*)o->step_host, 0, sizeof(StepOut));
  {
    const char* sv = getenv("EMU_STEP_SERVER");
    o->server = !(sv && sv[0] == '0');
    if (cudaHostAlloc((void**)&o->req_host, sizeof(StepReq), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&o->req_dev, o->req_host, 0) != cudaSuccess ||
        cudaHostAlloc((void**)&o->alive_host, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&o->alive_dev, o->alive_host, 0) != cudaSuccess ||
        cudaMalloc((void**)&o->served_dev, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemset(o->served_dev, 0, sizeof(uint32_t)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&o->srv_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&o->srv_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&o->async_done, cudaEventDisableTiming) != cudaSuccess) {
      emu_oracle_destroy(o);
      return fail(EMU_ERR_CUDA, "step server setup failed");
    }
    memset((void*)o->req_host, 0, sizeof(StepReq));
    *o->alive_host = 0;
  }
  if ((rc = oracle_flush(o, s))) {
    emu_oracle_destroy(o);
    return rc;
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    emu_oracle_destroy(o);
    return cuda_fail(e, "emu_oracle_create");
  }
  *out = o;
  return EMU_OK;
}

void emu_oracle_destroy(emu_oracle_t o) {
  if (o) {
    cudaFree(o->miss);
    cudaFree(o->bits);
    cudaFree(o->bits_part);
    cudaFree(o->hk_tt);
    cudaFree(o->hk_c);
    cudaFree(o->hk_p);
    cudaFree(o->hk_e);
  }
  if (!o) return;
  cudaFree(o->map.dense);
  cudaFree(o->map.hkeys);
  cudaFree(o->map.hvals);
  cudaFree(o->arena);
  cudaFree(o->arena_used);
  cudaFree(o->ctl);
  cudaFree(o->nk_tt);
  cudaFree(o->nk_c);
  cudaFree(o->nk_p);
  cudaFree(o->nk_e);
  cudaFree(o->esc);
  cudaFree(o->esc2);
  cudaFree(o->kw);
  cudaFree(o->resv);
  cudaFree(o->tile_cnt);
  cudaFree(o->tile_off);
  cudaFree(o->tile_part);
  cudaFree(o->kbin);
  cudaFree(o->krank);
  cudaFree(o->order);
  cudaFree(o->fb_list);
  cudaFree(o->gd);
  cudaFree(o->gb);
  cudaFree(o->pcg);
  cudaFree(o->stage);
  for (cudaEvent_t e : o->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : o->ev_cmp) cudaEventDestroy(e);
  if (o->ev_start) cudaEventDestroy(o->ev_start);
  if (o->cp_in) cudaStreamDestroy(o->cp_in);
  if (o->cp_out) cudaStreamDestroy(o->cp_out);
  cudaFree(o->flag_log);
  if (o->flag_log_host) cudaFreeHost(o->flag_log_host);
  quiesce_server(o);
  if (o->srv_stream) cudaStreamDestroy(o->srv_stream);
  if (o->srv_done) cudaEventDestroy(o->srv_done);
  if (o->async_done) cudaEventDestroy(o->async_done);
  cudaFree(o->served_dev);
  if (o->req_host) cudaFreeHost(o->req_host);
  if (o->alive_host) cudaFreeHost(o->alive_host);
  if (o->step_host) cudaFreeHost(o->step_host);
  if (o->flags_host) cudaFreeHost(o->flags_host);
  if (o->ctl_host) cudaFreeHost(o->ctl_host);
  delete o;
}

int emu_oracle_flush(emu_oracle_t o, void* stream) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  const int rc = oracle_flush(o, as_stream(stream));
  if (rc) return rc;
  EMU_CUDA(cudaEventRecord(o->async_done, as_stream(stream)));  // the step server waits for it
  o->async_pending = true;
  return EMU_OK;
}

int emu_oracle_stats(emu_oracle_t o, int64_t* n_pools, int64_t* n_slots) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  unsigned long long used = 0;
  EMU_CUDA(cudaMemcpy(&used, o->arena_used, sizeof(used), cudaMemcpyDeviceToHost));
  if (n_slots) *n_slots = (int64_t)used;
  if (n_pools) *n_pools = -1;  // not tracked on device
  return EMU_OK;
}

}  // extern "C"

// Per-batch key scratch, sized lazily: a batch of n queries (or n explicit
// keys) has at most min(n, map entries) new keys.
static int ensure_key_capacity(emu_oracle_t o, int64_t n_keys) {
  int64_t need = std::max<int64_t>(4096, pow2_at_least(n_keys));
  if (need <= o->nk_cap) return EMU_OK;
  cudaFree(o->nk_tt);
  cudaFree(o->nk_c);
  cudaFree(o->nk_p);
  cudaFree(o->nk_e);
  cudaFree(o->esc);
  cudaFree(o->esc2);
  cudaFree(o->kw);
  cudaFree(o->resv);
  cudaFree(o->kbin);
  cudaFree(o->krank);
  cudaFree(o->order);
  cudaFree(o->fb_list);
  cudaFree(o->hk_tt);
  cudaFree(o->hk_c);
  cudaFree(o->hk_p);
  cudaFree(o->hk_e);
  o->hk_tt = nullptr;
  o->hk_c = nullptr;
  o->hk_p = nullptr;
  o->hk_e = nullptr;
  o->kbin = o->krank = o->order = o->fb_list = nullptr;
  o->nk_tt = nullptr;
  o->nk_c = nullptr;
  o->nk_p = nullptr;
  o->nk_e = nullptr;
  o->esc = nullptr;
  o->esc2 = nullptr;
  o->kw = nullptr;
  o->resv = nullptr;
  o->nk_cap = 0;
  int rc;
  if ((rc = dalloc(&o->nk_tt, need)) || (rc = dalloc(&o->nk_c, need)) || (rc = dalloc(&o->nk_p, need)) ||
      (rc = dalloc(&o->nk_e, need)) || (rc = dalloc(&o->esc, need)) || (rc = dalloc(&o->esc2, need)) ||
      (rc = dalloc(&o->kw, need)) || (rc = dalloc(&o->resv, need)) || (rc = dalloc(&o->kbin, need)) ||
      (rc = dalloc(&o->krank, need)) || (rc = dalloc(&o->order, need + 64)) || (rc = dalloc(&o->fb_list, need)) ||
      (rc = dalloc(&o->hk_tt, need)) || (rc = dalloc(&o->hk_c, need)) || (rc = dalloc(&o->hk_p, need)) ||
      (rc = dalloc(&o->hk_e, need)))
    return rc;
  o->nk_cap = need;
  return EMU_OK;
}

static int64_t map_entries(emu_oracle_t o) { return 2LL * o->map.dom_tt * o->map.dom_conc + 2 * o->map.hcap; }

static int grid_knob(int which, int dflt) {  // EMU_GRIDS=<prep>,<sample> CTAs per SM (tuning)
  static int g[2] = {-1, -1};
  if (g[0] < 0) {
    g[0] = 4;
    g[1] = 16;
    if (const char* v = getenv("EMU_GRIDS")) sscanf(v, "%d,%d", &g[0], &g[1]);
  }
  return g[which] > 0 ? g[which] : dflt;
}
#define kPrepGrid (kNumSMs * grid_knob(0, 4))

struct CntIn {
  const int* c;
  __device__ int operator()(int64_t i) const { return c[i]; }
};
struct OffOut {
  int* o;
  __device__ void operator()(int64_t i, int v) const { o[i] = v; }
};

// The pool tiers after k_mark / explicit keys: prep (thread per key: SAT window,
// arena reservation) -> tile tier (counting sort of the keys into (phase, conc,
// tt) bins, warp per 32 keys, lane per key) -> warp tier for the keys the tile
// tier handed over (or all keys) -> group tier -> CTA tier.
// known_new >= 0: the host knows the number of new keys; a small batch
// (<= kSmallBatch) skips k_pool_prep and the tile and warp tiers: every key goes
// to the group tier, whose 4 warps per key (32-lane radius probe, then the
// window) finish one key sooner than a thread + a warp do -- with few keys the
// tiers' latency, not their throughput, is the cost (config 5's scenario
// batches each bring a few hundred to a few thousand new keys).
constexpr int64_t kSmallBatch = 2048;
template <int MODE>
static int launch_pool_tiers(emu_oracle_t o, const Keys& keys, const Sink& sk, cudaStream_t s, bool sync_check,
                             bool dense_keys = false, int64_t known_new = -1) {
  const bool small = known_new >= 0 && known_new <= kSmallBatch && !getenv("EMU_NO_SMALL_BATCH");
  static const bool tile_debug = getenv("EMU_TILE_DEBUG") != nullptr;
  auto chk = [&](const char* what) -> int {
    EMU_CUDA(cudaGetLastError());
    if (sync_check || tile_debug) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_fail(e, what);
    }
    if (tile_debug) {
      BatchCtl c{};
      EMU_CUDA(cudaMemcpy(&c, o->ctl, sizeof(c), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[emu] after %s: new %d work %d tile_work %d tile_total %d fb_n %d fb_work %d esc %d flags %d\n",
              what, c.new_count, c.work, c.tile_work, c.tile_total, c.fb_n, c.fb_work, c.esc_count, c.flags);
    }
    return EMU_OK;
  };
  int rc;
  if (!small)
  EMU_LAUNCH("pool_prep", s, k_pool_prep<MODE><<<kPrepGrid, 256, 0, s>>>(
                                 o->plane[0], o->plane[1], keys, o->cfg, sk, o->kw, o->resv, o->esc,
                                 &o->ctl->esc_count, o->tile_on ? nullptr : o->fb_list, &o->ctl->fb_n, small ? 1 : 0));
  if ((rc = chk("pool_prep"))) return rc;
  const int* list = o->fb_list;  // the warp tier's keys: from prep, or handed over by the tile tier
  const int* list_n = &o->ctl->fb_n;
  int* warp_work = &o->ctl->fb_work;
  if (small) {
    // tile and warp tiers skipped: prep put every key on the group tier's list
  } else if (o->tile_on && dense_keys) {  // cold path: keys already in tile order (build_missing_cold)
    EMU_LAUNCH("pool_tile", s, k_pool_tile<MODE><<<kNumSMs * EMU_TILE_MINB, kTileThreads, kTileBytes, s>>>(
                                   o->plane[0], o->plane[1], keys, o->cfg, sk, o->ti, o->kw, o->resv, nullptr,
                                   nullptr, &o->ctl->dense_n, &o->ctl->dense_n0, &o->ctl->tile_work, o->fb_list,
                                   &o->ctl->fb_n));
    if ((rc = chk("pool_tile"))) return rc;
  } else if (o->tile_on) {
    EMU_CUDA(cudaMemsetAsync(o->tile_cnt, 0, sizeof(int) * o->ti.nb, s));
    EMU_LAUNCH("tile_bin", s, k_tile_bin<MODE><<<kPrepGrid, 256, 0, s>>>(o->plane[0], o->plane[1], keys, o->cfg, o->ti,
                                                                          o->kw, o->resv, o->tile_cnt, o->kbin, o->krank,
                                                                          o->fb_list, &o->ctl->fb_n));
    if ((rc = chk("tile_bin"))) return rc;
    EMU_CUDA(device_excl_scan<int>(CntIn{o->tile_cnt}, OffOut{o->tile_off}, o->ti.nb, o->tile_part,
                                   &o->ctl->tile_total, s));
    if ((rc = chk("tile_scan"))) return rc;
    EMU_LAUNCH("tile_scatter", s, k_tile_scatter<MODE><<<kPrepGrid, 256, 0, s>>>(keys, o->ti, o->kbin, o->krank,
                                                                                  o->tile_off, &o->ctl->tile_total,
                                                                                  o->order));
    if ((rc = chk("tile_scatter"))) return rc;
    if (getenv("EMU_TILE_DEBUG")) {
      BatchCtl c{};
      EMU_CUDA(cudaMemcpyAsync(&c, o->ctl, sizeof(c), cudaMemcpyDeviceToHost, s));
      EMU_CUDA(cudaStreamSynchronize(s));
      std::vector<int> off(o->ti.nb), ord(c.tile_total + 64);
      EMU_CUDA(cudaMemcpy(off.data(), o->tile_off, 4 * o->ti.nb, cudaMemcpyDeviceToHost));
      EMU_CUDA(cudaMemcpy(ord.data(), o->order, 4 * (c.tile_total + 64), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[emu] tile debug: n=%lld binned=%d fb=%d nb=%lld base1=%lld off[base1]=%d ord[0..4]=%d %d %d %d\n",
              (long long)keys.count, c.tile_total, c.fb_n, (long long)o->ti.nb, (long long)o->ti.base[1],
              o->ti.base[1] < o->ti.nb ? off[o->ti.base[1]] : -1, ord[0], ord[1], ord[2], ord[3]);
    }
    EMU_LAUNCH("pool_tile", s, k_pool_tile<MODE><<<kNumSMs * EMU_TILE_MINB, kTileThreads, kTileBytes, s>>>(
                                   o->plane[0], o->plane[1], keys, o->cfg, sk, o->ti, o->kw, o->resv, o->order,
                                   o->tile_off, &o->ctl->tile_total, nullptr, &o->ctl->tile_work, o->fb_list,
                                   &o->ctl->fb_n));
    if ((rc = chk("pool_tile"))) return rc;
  }
  if (!small)
  EMU_LAUNCH("pool_warp", s, k_pool_warp<MODE><<<kWarpGrid, kWarpThreads, kWarpBytes * kWarpsPerCta, s>>>(
                                 o->plane[0], o->plane[1], keys, o->cfg, sk, o->kw, o->resv, warp_work, o->esc,
                                 &o->ctl->esc_count, list, list_n));
  if ((rc = chk("pool_warp"))) return rc;
  EMU_LAUNCH("pool_grp", s, k_pool_grp<MODE><<<kGrpGrid, kGrpThreads, kGrpSmem, s>>>(
                                o->plane[0], o->plane[1], keys, o->cfg, sk, small ? nullptr : o->kw,
                                &o->ctl->esc_work, small ? nullptr : o->esc, &o->ctl->esc_count, o->esc2,
                                &o->ctl->esc2_count));
  if ((rc = chk("pool_grp"))) return rc;
  EMU_LAUNCH("pool_cta", s, k_pool_cta<MODE><<<kCtaGrid, kCtaThreads, kCtaSmem, s>>>(o->plane[0], o->plane[1], keys,
                                                                                     o->cfg, sk, &o->ctl->esc2_work,
                                                                                     o->esc2, &o->ctl->esc2_count, o->gd,
                                                                                     o->gb, o->gcap));
  return chk("pool_cta");
}

// Zero the per-pass counters of BatchCtl (the flags and bad key survive: one
// chunk's passes report together; callers zero the whole block per chunk).
static cudaError_t reset_counters(emu_oracle_t o, cudaStream_t s) {
  constexpr size_t off = offsetof(BatchCtl, cand_used);
  return cudaMemsetAsync(reinterpret_cast<char*>(o->ctl) + off, 0, sizeof(BatchCtl) - off, s);
}

// Build missing pools for a chunk of queries: mark -> the pool tiers.  No host round trip.
static int build_missing(emu_oracle_t o, const int32_t* qt, const int32_t* qc, const uint8_t* qp, int64_t Q,
                         cudaStream_t s) {
  int rc = ensure_key_capacity(o, std::min<int64_t>(Q, map_entries(o)));
  if (rc) return rc;
  o->cold = false;
  EMU_CUDA(reset_counters(o, s));
  {
    // EMU_MARK=<qpt>,<ctas per SM> (tuning knob).  Default 2 queries per
    // thread, up to 8 CTAs per SM: 0.124 ms per 10M-query cold sweep vs 0.153
    // for 4 x 16 and 0.183 for 8 x 16 (the first wave's CAS round trips sit on
    // each tile's critical path, so shorter tiles hide them better); 32 CTAs
    // per SM gain 3 us there but cost 18 % on warm 1M-query batches (config 5)
    static int mq = -1, mg = 8;
    if (mq < 0) {
      mq = 2;
      if (const char* v = getenv("EMU_MARK")) sscanf(v, "%d,%d", &mq, &mg);
    }
    const int cap = kNumSMs * mg;
    if (mq == 8)
      EMU_LAUNCH("mark", s, k_mark<8><<<grid_for((Q + 7) / 8, 256, cap), 256, 0, s>>>(o->map, qt, qc, qp, Q, o->nk_tt,
                                                                                    o->nk_c, o->nk_p, o->nk_e, o->ctl));
    else if (mq == 1)
      EMU_LAUNCH("mark", s, k_mark<1><<<grid_for(Q, 256, cap), 256, 0, s>>>(o->map, qt, qc, qp, Q, o->nk_tt, o->nk_c,
                                                                          o->nk_p, o->nk_e, o->ctl));
    else if (mq == 2)
      EMU_LAUNCH("mark", s, k_mark<2><<<grid_for((Q + 1) / 2, 256, cap), 256, 0, s>>>(o->map, qt, qc, qp, Q, o->nk_tt,
                                                                                    o->nk_c, o->nk_p, o->nk_e, o->ctl));
    else
      EMU_LAUNCH("mark", s, k_mark<4><<<grid_for((Q + 3) / 4, 256, cap), 256, 0, s>>>(o->map, qt, qc, qp, Q, o->nk_tt,
                                                                                    o->nk_c, o->nk_p, o->nk_e, o->ctl));
  }
  EMU_CUDA(cudaGetLastError());
  Keys keys{o->nk_tt, o->nk_c, o->nk_p, o->nk_e, &o->ctl->new_count, 0};
  // one round trip for the new-key count: nothing to build skips the tiers, a
  // few keys take the small-batch route
  EMU_CUDA(cudaMemcpyAsync(o->ctl_host, o->ctl, offsetof(BatchCtl, miss_count) + sizeof(int), cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  const int64_t known = o->ctl_host->new_count;
  rc = known == 0 ? EMU_OK : launch_pool_tiers<0>(o, keys, make_sink(o), s, false, false, known);
  static const bool tile_stats = [] {
    const char* v = getenv("EMU_TILE_STATS");
    return v && v[0] == '1';
  }();
  if (!rc && tile_stats) {  // tuning aid: how many new keys each tier took
    BatchCtl c{};
    EMU_CUDA(cudaMemcpyAsync(&c, o->ctl, sizeof(c), cudaMemcpyDeviceToHost, s));
    EMU_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "[emu] new keys %d  tile-binned %d  to warp tier %d  to group tier %d  to CTA tier %d\n",
            c.new_count, c.tile_total, o->tile_on ? c.fb_n : c.new_count, c.esc_count, c.esc2_count);
  }
  return rc;
}

// Cold batch (the cache was just flushed): k_mark_bits -> bitmap scan (keys in
// tile order) -> side-list keys appended -> the pool tiers with the tile tier
// reading the keys in place (no k_tile_bin / scan / scatter).  Falls back to
// build_missing without the tile tier.
static int build_missing_cold(emu_oracle_t o, const int32_t* qt, const int32_t* qc, const uint8_t* qp, int64_t Q,
                              cudaStream_t s) {
  static const bool off = [] {
    const char* v = getenv("EMU_COLD_BITMAP");
    return v && v[0] == '0';
  }();
  if (!o->tile_on || off) return build_missing(o, qt, qc, qp, Q, s);
  int rc = ensure_key_capacity(o, std::min<int64_t>(Q, map_entries(o)));
  if (rc) return rc;
  const int64_t ps = ((int64_t)o->map.dom_tt * o->map.dom_conc + 31) & ~(int64_t)31;
  const int64_t words = 2 * ps / 32;
  if (words != o->bits_words) {
    cudaFree(o->bits);
    cudaFree(o->bits_part);
    o->bits = nullptr;
    o->bits_part = nullptr;
    o->bits_words = 0;
    if ((rc = dalloc(&o->bits, words)) || (rc = dalloc(&o->bits_part, (words + kBitThreads - 1) / kBitThreads + 1)))
      return rc;
    EMU_CUDA(cudaMemsetAsync(o->bits, 0, 4 * words, s));
    o->bits_words = words;
  }
  o->cold = false;
  EMU_CUDA(reset_counters(o, s));
  EMU_LAUNCH("mark", s, k_mark_bits<<<grid_for(Q, 256, kNumSMs * 8), 256, 0, s>>>(o->map, qt, qc, qp, Q, o->bits,
                                                                                  o->hk_tt, o->hk_c, o->hk_p,
                                                                                  o->hk_e, o->ctl));
  const int64_t nblk = (words + kBitThreads - 1) / kBitThreads;
  EMU_LAUNCH("bits", s, k_bits_count<<<(unsigned)nblk, kBitThreads, 0, s>>>(o->bits, words, o->bits_part));
  EMU_LAUNCH("bits", s, k_scan_partials<unsigned int><<<1, 1024, 0, s>>>(
                            o->bits_part, nblk, reinterpret_cast<unsigned int*>(&o->ctl->dense_n)));
  EMU_LAUNCH("bits", s, k_bits_emit<<<(unsigned)nblk, kBitThreads, 0, s>>>(o->bits, words, ps / 32, o->bits_part,
                                                                           o->map, o->nk_tt, o->nk_c, o->nk_p,
                                                                           o->nk_e, &o->ctl->dense_n0));
  EMU_LAUNCH("append_hash", s, k_append_hash<<<1, 256, 0, s>>>(o->hk_tt, o->hk_c, o->hk_p, o->hk_e, o->nk_tt,
                                                                     o->nk_c, o->nk_p, o->nk_e, o->ctl, o->fb_list));
  EMU_CUDA(cudaGetLastError());
  Keys keys{o->nk_tt, o->nk_c, o->nk_p, o->nk_e, &o->ctl->new_count, 0};
  return launch_pool_tiers<0>(o, keys, make_sink(o), s, false, true);
}

// Flags of the chunk (and, in ctl_host, its new-key / miss counts).
static int read_flags(emu_oracle_t o, cudaStream_t s, int* flags) {
  EMU_CUDA(cudaMemcpyAsync(o->ctl_host, o->ctl, offsetof(BatchCtl, miss_count) + sizeof(int), cudaMemcpyDeviceToHost,
                           s));
  EMU_CUDA(cudaStreamSynchronize(s));
  *flags = o->ctl_host->flags;
  return EMU_OK;
}

// Which path the next warm chunk takes.  k_sweep draws hits in its single pass
// but sends every miss through a second, gathering pass (and a host round trip
// to size it); a chunk that still meets many new keys -- what-if scenarios
// exploring new batch shapes -- is cheaper as k_mark + tiers + k_sample.
// (C5, 512 scenarios x 1M steps: 222 ms with k_sweep on every chunk.)
static void update_path(emu_oracle_t o, bool swept, int64_t n) {
  static const int mode = [] {  // EMU_SWEEP=0: never k_sweep, 1: always (tuning knob)
    const char* v = getenv("EMU_SWEEP");
    return v ? atoi(v) : -1;
  }();
  if (mode >= 0) {
    o->sweep_ok = mode == 1;
    return;
  }
  if (n <= 0) return;
  const double frac = swept ? (double)o->ctl_host->miss_count / (double)n : (double)o->ctl_host->new_count / (double)n;
  o->sweep_ok = frac < (swept ? 0.02 : 0.002);
}

// Handle a failed chunk: grow the hash on overflow; always flush the cache.
// Returns the (possibly reduced) chunk size to retry with, or -1 if hopeless.
// started_cold: the failed chunk began on an empty cache.  A chunk that
// overflowed a cache filled by earlier chunks is retried whole after the flush;
// only one that overflowed on its own is halved (bounded below by what always fits).
static int64_t recover(emu_oracle_t o, int flags, int64_t chunk, cudaStream_t s, int* rc, bool started_cold) {
  *rc = EMU_OK;
  if (flags & FLAG_HASH) {
    if ((*rc = alloc_hash(o, o->map.hcap * 4))) return -1;
  }
  if ((flags & FLAG_ARENA) && o->arena_cap < o->arena_max) {  // grow the arena before resorting to chunking
    quiesce_server(o);
    cudaFree(o->arena);
    o->arena = nullptr;
    o->arena_cap = std::min(o->arena_max, o->arena_cap * 4);
    if ((*rc = dalloc(&o->arena, o->arena_cap + kArenaSlack))) return -1;
    if (cudaMemsetAsync(o->arena, 0, sizeof(Slot) * (o->arena_cap + kArenaSlack), s) != cudaSuccess) {
      *rc = cuda_fail(cudaGetLastError(), "arena memset");
      return -1;
    }
    if ((*rc = oracle_flush(o, s))) return -1;
    return chunk;
  }
  if ((*rc = oracle_flush(o, s))) return -1;
  if (flags & FLAG_ARENA) {
    int64_t fit = std::max<int64_t>(1, o->arena_cap / std::max<int64_t>(1, pool_total_slots(o->kmax)));
    if (!started_cold) return chunk;
    if (chunk <= 1 && fit <= 1) return -1;
    return std::min(chunk / 2 > 0 ? chunk / 2 : 1, fit);
  }
  return chunk;
}

// Sampler variant: queries per thread and streaming-cache hints; 0 = the
// compacting sampler (k_sample_c), 3 = one query per thread with the next
// query's streams prefetched (k_sample_pf).  Defaults (measured, config 2):
// EXPLICIT k_sample<1 query/thread, hints> 0.137 ms; PHILOX k_sample_pf
// 0.148 ms (k_sample 0.161, k_sample_c 0.151).
// EMU_SAMPLE_VARIANT="qpt,hint" overrides for tuning runs.
static void sample_variant(int rng_mode, int* qpt, int* hint) {
  static int q = -2, h = -1;
  if (q == -2) {
    q = -1;
    h = -1;
    const char* v = getenv("EMU_SAMPLE_VARIANT");
    if (v) sscanf(v, "%d,%d", &q, &h);
    if (q != -1 && q != 0 && q != 1 && q != 2 && q != 3 && q != 4 && q != 8) q = -1;
  }
  *qpt = q >= 0 ? q : (rng_mode == EMU_RNG_EXPLICIT ? 1 : 3);
  *hint = h < 0 ? (rng_mode == EMU_RNG_EXPLICIT ? 1 : 0) : (h ? 1 : 0);
}

template <int RNG, int QPT, bool HINT>
static void launch_sample_t(emu_oracle_t o, const int32_t* qt, const int32_t* qc, const uint8_t* qp, int64_t n,
                            const uint64_t* us, const uint32_t* ui, uint64_t seed, uint64_t ctr, double* lat,
                            int32_t* sidx, cudaStream_t s) {
  const int grid = grid_for((n + QPT - 1) / QPT, kSampleThreads, kNumSMs * grid_knob(1, 16));
  EMU_LAUNCH("sample", s, k_sample<RNG, QPT, HINT><<<grid, kSampleThreads, 0, s>>>(
                              o->map, o->arena, o->plane[0].samples, o->plane[1].samples, qt, qc, qp, n, us, ui, seed,
                              ctr, lat, sidx, &o->ctl->flags));
}

template <int RNG>
static void launch_sample_r(emu_oracle_t o, const int32_t* qt, const int32_t* qc, const uint8_t* qp, int64_t n,
                            const uint64_t* us, const uint32_t* ui, uint64_t seed, uint64_t ctr, double* lat,
                            int32_t* sidx, cudaStream_t s) {
  int q, h;
  sample_variant(RNG, &q, &h);
  if (q == 3) {
    const int grid = grid_for(n, kSampleThreads, kNumSMs * 8);
    EMU_LAUNCH("sample", s, k_sample_pf<RNG><<<grid, kSampleThreads, 0, s>>>(o->map, o->arena, o->plane[0].samples,
                                                                            o->plane[1].samples, qt, qc, qp, n, us, ui,
                                                                            seed, ctr, lat, sidx, &o->ctl->flags));
    return;
  }
  if (q == 0 || q == 8) {
    const int per = q == 0 ? 64 : 128;
    const int grid = grid_for((n + per - 1) / per, 8, kNumSMs * 64);
    if (q == 0)
      EMU_LAUNCH("sample", s, k_sample_c<RNG, 2><<<grid, 256, 0, s>>>(o->map, o->arena, o->plane[0].samples,
                                                                      o->plane[1].samples, qt, qc, qp, n, us, ui, seed,
                                                                      ctr, lat, sidx, &o->ctl->flags));
    else
      EMU_LAUNCH("sample", s, k_sample_c<RNG, 4><<<grid, 256, 0, s>>>(o->map, o->arena, o->plane[0].samples,
                                                                      o->plane[1].samples, qt, qc, qp, n, us, ui, seed,
                                                                      ctr, lat, sidx, &o->ctl->flags));
    return;
  }
  if (q == 1 && h) launch_sample_t<RNG, 1, true>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  if (q == 1 && !h) launch_sample_t<RNG, 1, false>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  if (q == 2 && h) launch_sample_t<RNG, 2, true>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  if (q == 2 && !h) launch_sample_t<RNG, 2, false>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  if (q == 4 && h) launch_sample_t<RNG, 4, true>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  if (q == 4 && !h) launch_sample_t<RNG, 4, false>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
}

static int launch_sample(emu_oracle_t o, int rng_mode, const int32_t* qt, const int32_t* qc, const uint8_t* qp,
                         int64_t n, const uint64_t* us, const uint32_t* ui, uint64_t seed, uint64_t ctr, double* lat,
                         int32_t* sidx, cudaStream_t s) {
  if (rng_mode == EMU_RNG_EXPLICIT)
    launch_sample_r<EMU_RNG_EXPLICIT>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  else
    launch_sample_r<EMU_RNG_PHILOX>(o, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

// Queries of a batch on a COLD cache that take the two-pass path (k_mark ->
// tiers -> k_sample) before the rest streams through k_sweep.  Default: all of
// them -- splitting a cold batch's distinct keys over two tier passes costs more
// than the second read of the key stream saves (C2 cold step 1.29 ms at a 25 %
// head vs 0.88 ms two-pass).  EMU_SWEEP_HEAD=<fraction, %> (0: sweep everything).
static int64_t cold_head(int64_t n) {
  static const int pct = [] {
    const char* v = getenv("EMU_SWEEP_HEAD");
    return v ? std::max(0, std::min(100, atoi(v))) : 100;
  }();
  return std::min<int64_t>(n, (n * pct + 99) / 100);
}

// One chunk of a batch, device-resident, no host round trip: pools for the
// keys not cached yet, then every query's draw.  Flags accumulate in ctl.
// may_sync: the caller allows one host round trip after k_sweep, so the pool
// tiers and k_sample_list are only launched when there are new keys / misses
// (a warm sweep then costs one kernel, not a dozen near-empty ones); the
// pipelined host path passes false to keep its copies overlapped.
// *flags_out (if given): the chunk's final flags when that round trip already
// read them (nothing launched after k_sweep), else -1.
static int draw_chunk(emu_oracle_t o, int rng_mode, const int32_t* qt, const int32_t* qc, const uint8_t* qp,
                      int64_t n, const uint64_t* us, const uint32_t* ui, uint64_t seed, uint64_t ctr, double* lat,
                      int32_t* sidx, cudaStream_t s, bool may_sync, int* flags_out = nullptr) {
  if (flags_out) *flags_out = -1;
  // cold: the bitmap path for the head (all of it by default); warm with few new
  // keys lately: k_sweep; otherwise the two-pass path (k_mark, tiers, k_sample)
  const bool two_pass = !o->cold && !o->sweep_ok;
  const int64_t head = o->cold ? cold_head(n) : 0;
  const int64_t m = n - head;
  o->cold = false;
  o->last_swept = false;
  if (two_pass) {
    int rc = build_missing(o, qt, qc, qp, n, s);
    if (!rc) rc = launch_sample(o, rng_mode, qt, qc, qp, n, us, ui, seed, ctr, lat, sidx, s);
    return rc;
  }
  int rc;
  // scratch first: reallocating after the head pass is enqueued would stall on it
  if ((rc = ensure_key_capacity(o, std::min<int64_t>(n, map_entries(o))))) return rc;
  if (m > o->miss_cap) {
    cudaFree(o->miss);
    o->miss = nullptr;
    o->miss_cap = 0;
    if ((rc = dalloc(&o->miss, pow2_at_least(m)))) return rc;
    o->miss_cap = pow2_at_least(m);
  }
  if (head > 0) {
    if ((rc = build_missing_cold(o, qt, qc, qp, head, s))) return rc;
    if ((rc = launch_sample(o, rng_mode, qt, qc, qp, head, us, ui, seed, ctr, lat, sidx, s))) return rc;
  }
  if (m <= 0) return EMU_OK;
  qt += head, qc += head, qp += head, lat += head, sidx += head, ctr += (uint64_t)head;
  if (us) us += head, ui += head;
  if (head > 0) EMU_CUDA(reset_counters(o, s));  // (callers zero the whole block before a chunk)
  o->last_swept = true;
  const int grid = grid_for(m, kSampleThreads, kNumSMs * 8);
  const uint64_t sd = seed;
  // EMU_SWEEP_CG=1: the sweep's gathers (entry, pool, sample) through L2 only (tuning knob)
  static const bool cg = [] {
    const char* v = getenv("EMU_SWEEP_CG");
    return v && v[0] == '1';
  }();
#define EMU_SWEEP_LAUNCH(R, C)                                                                                     \
  EMU_LAUNCH("sweep", s, (k_sweep<R, C><<<grid, kSampleThreads, 0, s>>>(                                          \
                             o->map, o->arena, o->plane[0].samples, o->plane[1].samples, qt, qc, qp, m, us, ui, sd, \
                             ctr, lat, sidx, o->nk_tt, o->nk_c, o->nk_p, o->nk_e, o->miss, o->ctl)))
  if (rng_mode == EMU_RNG_EXPLICIT) {
    if (cg)
      EMU_SWEEP_LAUNCH(EMU_RNG_EXPLICIT, true);
    else
      EMU_SWEEP_LAUNCH(EMU_RNG_EXPLICIT, false);
  } else {
    if (cg)
      EMU_SWEEP_LAUNCH(EMU_RNG_PHILOX, true);
    else
      EMU_SWEEP_LAUNCH(EMU_RNG_PHILOX, false);
  }
#undef EMU_SWEEP_LAUNCH
  EMU_CUDA(cudaGetLastError());
  int lgrid = kNumSMs * 4;
  if (may_sync) {  // flags .. miss_count in one copy
    EMU_CUDA(cudaMemcpyAsync(o->ctl_host, o->ctl, offsetof(BatchCtl, miss_count) + sizeof(int), cudaMemcpyDeviceToHost,
                             s));
    EMU_CUDA(cudaStreamSynchronize(s));
    if (o->ctl_host->miss_count == 0) {  // every query was drawn in the pass
      if (flags_out) *flags_out = o->ctl_host->flags;
      return EMU_OK;
    }
    lgrid = grid_for(o->ctl_host->miss_count, kSampleThreads, kNumSMs * 4);
  }
  Keys keys{o->nk_tt, o->nk_c, o->nk_p, o->nk_e, &o->ctl->new_count, 0};
  if ((!may_sync || o->ctl_host->new_count > 0) &&
      (rc = launch_pool_tiers<0>(o, keys, make_sink(o), s, false, false, may_sync ? o->ctl_host->new_count : -1)))
    return rc;
  if (rng_mode == EMU_RNG_EXPLICIT)
    EMU_LAUNCH("sample_list", s, k_sample_list<EMU_RNG_EXPLICIT><<<lgrid, kSampleThreads, 0, s>>>(
                                     o->map, o->arena, o->plane[0].samples, o->plane[1].samples, qt, qc, qp, o->miss,
                                     &o->ctl->miss_count, us, ui, sd, ctr, lat, sidx, &o->ctl->flags));
  else
    EMU_LAUNCH("sample_list", s, k_sample_list<EMU_RNG_PHILOX><<<lgrid, kSampleThreads, 0, s>>>(
                                     o->map, o->arena, o->plane[0].samples, o->plane[1].samples, qt, qc, qp, o->miss,
                                     &o->ctl->miss_count, us, ui, sd, ctr, lat, sidx, &o->ctl->flags));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

extern "C" {

int emu_oracle_sample(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc, const uint8_t* q_phase, int64_t Q,
                      int rng_mode, const uint64_t* u_sel, const uint32_t* u_idx, uint64_t seed, uint64_t ctr_base,
                      double* out_lat, int32_t* out_sidx, void* stream) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  if (Q < 0) return fail(EMU_ERR_INVALID, "negative query count");
  if (Q == 0) return EMU_OK;
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  if (rng_mode != EMU_RNG_EXPLICIT && rng_mode != EMU_RNG_PHILOX) return fail(EMU_ERR_INVALID, "unknown rng_mode");
  if (rng_mode == EMU_RNG_EXPLICIT && (!u_sel || !u_idx)) return fail(EMU_ERR_INVALID, "explicit mode needs u_sel/u_idx");
  cudaStream_t s = as_stream(stream);
  int64_t chunk = std::min(Q, o->chunk_cap);
  int64_t done = 0;
  int attempts = 0;
  while (done < Q) {
    const int64_t n = std::min(chunk, Q - done);
    const bool cold0 = o->cold;
    int fk = -1;
    EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    int rc = draw_chunk(o, rng_mode, q_tt + done, q_conc + done, q_phase + done, n, u_sel ? u_sel + done : nullptr,
                        u_idx ? u_idx + done : nullptr, seed, ctr_base + (uint64_t)done, out_lat + done,
                        out_sidx + done, s, true, &fk);
    if (rc) return rc;
    EMU_CUDA(cudaGetLastError());
    int flags = fk;
    if (fk < 0 && (rc = read_flags(o, s, &flags))) return rc;
    update_path(o, o->last_swept, n);
    if (flags) {
      if (++attempts > 16) return fail(EMU_ERR_CUDA, "oracle could not fit a chunk after 16 retries");
      if (flags & FLAG_BADPOOL) return bad_pool_error(o, s);
      if (!(flags & (FLAG_ARENA | FLAG_HASH)))
        return fail(EMU_ERR_CUDA, "internal error: pool missing after build (flags=" + std::to_string(flags) + ")");
      chunk = recover(o, flags, n, s, &rc, cold0);
      if (rc) return rc;
      if (chunk < 0) return fail(EMU_ERR_CAPACITY, "pool arena too small for a single query's pool");
      continue;
    }
    done += n;
    attempts = 0;
  }
  return EMU_OK;
}

int emu_oracle_sample_pcg64(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc, const uint8_t* q_phase,
                            int64_t Q, uint64_t* pcg_state, double* out_lat, int32_t* out_sidx, void* stream) {
  if (!o || !pcg_state) return fail(EMU_ERR_INVALID, "NULL oracle/state");
  if (Q < 0) return fail(EMU_ERR_INVALID, "negative query count");
  if (Q == 0) return EMU_OK;
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  cudaStream_t s = as_stream(stream);
  int64_t chunk = std::min(Q, o->chunk_cap);
  int64_t done = 0;
  int attempts = 0;
  while (done < Q) {
    const int64_t n = std::min(chunk, Q - done);
    const bool cold0 = o->cold;
    EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    int rc = build_missing(o, q_tt + done, q_conc + done, q_phase + done, n, s);
    if (rc) return rc;
    EMU_LAUNCH("sample_pcg", s, k_sample_pcg<<<1, 32, 0, s>>>(o->map, o->arena, o->plane[0].samples, o->plane[1].samples, q_tt + done,
                                  q_conc + done, q_phase + done, n, pcg_state, out_lat + done, out_sidx + done,
                                  &o->ctl->flags));
    EMU_CUDA(cudaGetLastError());
    int flags = 0;
    if ((rc = read_flags(o, s, &flags))) return rc;
    if (flags) {
      if (++attempts > 16) return fail(EMU_ERR_CUDA, "oracle could not fit a chunk after 16 retries");
      if (flags & FLAG_BADPOOL) return bad_pool_error(o, s);
      if (!(flags & (FLAG_ARENA | FLAG_HASH)))
        return fail(EMU_ERR_CUDA, "internal error: pool missing after build (flags=" + std::to_string(flags) + ")");
      chunk = recover(o, flags, n, s, &rc, cold0);
      if (rc) return rc;
      if (chunk < 0) return fail(EMU_ERR_CAPACITY, "pool arena too small for a single query's pool");
      continue;
    }
    done += n;
    attempts = 0;
  }
  return EMU_OK;
}

int emu_oracle_sample_host(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc, const uint8_t* q_phase, int64_t Q,
                           int rng_mode, const uint64_t* u_sel, const uint32_t* u_idx, uint64_t seed, uint64_t ctr_base,
                           double* out_lat, int32_t* out_sidx, void* stream) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  if (Q <= 0) return Q == 0 ? EMU_OK : fail(EMU_ERR_INVALID, "negative query count");
  if (!out_lat) return fail(EMU_ERR_INVALID, "NULL out_lat");
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  if (rng_mode != EMU_RNG_EXPLICIT && rng_mode != EMU_RNG_PHILOX) return fail(EMU_ERR_INVALID, "unknown rng_mode");
  const bool ex = rng_mode == EMU_RNG_EXPLICIT;
  if (ex && (!u_sel || !u_idx)) return fail(EMU_ERR_INVALID, "explicit mode needs u_sel/u_idx");
  cudaStream_t s = as_stream(stream);
  size_t per = 4 + 4 + 1 + (ex ? 12 : 0) + 8 + 4;
  size_t need = per * (size_t)Q + 256;
  if (need > o->stage_bytes) {
    cudaFree(o->stage);
    o->stage = nullptr;
    o->stage_bytes = 0;
    EMU_CUDA(cudaMalloc(&o->stage, need));
    o->stage_bytes = need;
  }
  char* p = (char*)o->stage;
  auto carve = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 15) & ~(size_t)15;
    return r;
  };
  uint64_t* d_us = ex ? (uint64_t*)carve(8 * Q) : nullptr;
  double* d_lat = (double*)carve(8 * Q);
  int32_t* d_qt = (int32_t*)carve(4 * Q);
  int32_t* d_qc = (int32_t*)carve(4 * Q);
  uint32_t* d_ui = ex ? (uint32_t*)carve(4 * Q) : nullptr;
  int32_t* d_si = (int32_t*)carve(4 * Q);
  uint8_t* d_qp = (uint8_t*)carve(Q);
  // Pipeline: chunk i's copy-in (cp_in) overlaps chunk i-1's pool build +
  // draws (s) and chunk i-2's copy-out (cp_out).  Draws are pure functions of
  // (query, uniforms / counter, pool), so chunking never changes a result.
  // Staging covers all Q queries: no buffer is reused within a call.
  static const int64_t host_chunk = [] {
    const char* v = getenv("EMU_HOST_CHUNK");
    return v ? std::max<int64_t>(1024, atoll(v)) : kHostChunk;
  }();
  const int64_t chunk = std::min<int64_t>(std::max<int64_t>(o->chunk_cap, 1), host_chunk);
  const int64_t nch = (Q + chunk - 1) / chunk;
  // EMU_HOST_TRACE=1: timing events, and a per-chunk timeline on stderr (tuning aid)
  static const bool trace = getenv("EMU_HOST_TRACE") != nullptr;
  const unsigned evf = trace ? cudaEventDefault : cudaEventDisableTiming;
  if (!o->cp_in) {
    EMU_CUDA(cudaStreamCreateWithFlags(&o->cp_in, cudaStreamNonBlocking));
    EMU_CUDA(cudaStreamCreateWithFlags(&o->cp_out, cudaStreamNonBlocking));
    EMU_CUDA(cudaEventCreateWithFlags(&o->ev_start, evf));
  }
  while ((int64_t)o->ev_in.size() < nch) {
    cudaEvent_t a, b;
    EMU_CUDA(cudaEventCreateWithFlags(&a, evf));
    EMU_CUDA(cudaEventCreateWithFlags(&b, evf));
    o->ev_in.push_back(a);
    o->ev_cmp.push_back(b);
  }
  if (nch > o->flag_log_cap) {
    cudaFree(o->flag_log);
    if (o->flag_log_host) cudaFreeHost(o->flag_log_host);
    o->flag_log = nullptr;
    o->flag_log_host = nullptr;
    o->flag_log_cap = 0;
    EMU_CUDA(cudaMalloc(&o->flag_log, sizeof(int) * nch));
    EMU_CUDA(cudaHostAlloc((void**)&o->flag_log_host, sizeof(int) * nch, cudaHostAllocDefault));
    o->flag_log_cap = nch;
  }
  EMU_CUDA(cudaEventRecord(o->ev_start, s));  // earlier work on s may still use the staging
  EMU_CUDA(cudaStreamWaitEvent(o->cp_in, o->ev_start, 0));
  for (int64_t i = 0; i < nch; i++) {
    const int64_t a = i * chunk, n = std::min(chunk, Q - a);
    EMU_CUDA(cudaMemcpyAsync(d_qt + a, q_tt + a, 4 * n, cudaMemcpyDefault, o->cp_in));
    EMU_CUDA(cudaMemcpyAsync(d_qc + a, q_conc + a, 4 * n, cudaMemcpyDefault, o->cp_in));
    EMU_CUDA(cudaMemcpyAsync(d_qp + a, q_phase + a, n, cudaMemcpyDefault, o->cp_in));
    if (ex) {
      EMU_CUDA(cudaMemcpyAsync(d_us + a, u_sel + a, 8 * n, cudaMemcpyDefault, o->cp_in));
      EMU_CUDA(cudaMemcpyAsync(d_ui + a, u_idx + a, 4 * n, cudaMemcpyDefault, o->cp_in));
    }
    EMU_CUDA(cudaEventRecord(o->ev_in[i], o->cp_in));
    EMU_CUDA(cudaStreamWaitEvent(s, o->ev_in[i], 0));
    EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    int rc = draw_chunk(o, rng_mode, d_qt + a, d_qc + a, d_qp + a, n, ex ? d_us + a : nullptr, ex ? d_ui + a : nullptr,
                        seed, ctr_base + (uint64_t)a, d_lat + a, d_si + a, s, false);
    if (rc) return rc;
    EMU_CUDA(cudaMemcpyAsync(o->flag_log + i, &o->ctl->flags, sizeof(int), cudaMemcpyDeviceToDevice, s));
    EMU_CUDA(cudaEventRecord(o->ev_cmp[i], s));
    EMU_CUDA(cudaStreamWaitEvent(o->cp_out, o->ev_cmp[i], 0));
    EMU_CUDA(cudaMemcpyAsync(out_lat + a, d_lat + a, 8 * n, cudaMemcpyDefault, o->cp_out));
    if (out_sidx) EMU_CUDA(cudaMemcpyAsync(out_sidx + a, d_si + a, 4 * n, cudaMemcpyDefault, o->cp_out));
  }
  EMU_CUDA(cudaMemcpyAsync(o->flag_log_host, o->flag_log, sizeof(int) * nch, cudaMemcpyDeviceToHost, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  EMU_CUDA(cudaStreamSynchronize(o->cp_out));
  if (trace) {
    for (int64_t i = 0; i < nch; i++) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, o->ev_start, o->ev_in[i]);
      cudaEventElapsedTime(&b, o->ev_start, o->ev_cmp[i]);
      fprintf(stderr, "[emu host] chunk %lld: copied in %.3f ms, computed %.3f ms\n", (long long)i, a, b);
    }
  }
  int64_t bad = -1;
  for (int64_t i = 0; i < nch && bad < 0; i++)
    if (o->flag_log_host[i]) bad = i;
  if (bad < 0) return EMU_OK;
  // A chunk overflowed the arena / hash: redo it and everything after it with
  // the serial path (flush + retry with smaller chunks); inputs are resident.
  const int64_t a = bad * chunk, n = Q - a;
  int rc = oracle_flush(o, s);  // drop entries left claimed by the failed chunk
  if (rc) return rc;
  rc = emu_oracle_sample(o, d_qt + a, d_qc + a, d_qp + a, n, rng_mode, ex ? d_us + a : nullptr,
                             ex ? d_ui + a : nullptr, seed, ctr_base + (uint64_t)a, d_lat + a, d_si + a, stream);
  if (rc) return rc;
  EMU_CUDA(cudaMemcpyAsync(out_lat + a, d_lat + a, 8 * n, cudaMemcpyDefault, s));
  if (out_sidx) EMU_CUDA(cudaMemcpyAsync(out_sidx + a, d_si + a, 4 * n, cudaMemcpyDefault, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  return EMU_OK;
}

// Build (without drawing) the pools of n keys [dev] that are not cached yet:
// the warm-up half of emu_oracle_sample, used by the closed-loop scheduler.
int emu_oracle_prefetch(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc, const uint8_t* q_phase, int64_t n,
                        void* stream) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  if (n < 0) return fail(EMU_ERR_INVALID, "negative key count");
  if (n == 0) return EMU_OK;
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  cudaStream_t s = as_stream(stream);
  for (int attempt = 0; attempt < 16; attempt++) {
    EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    int rc = build_missing(o, q_tt, q_conc, q_phase, n, s);
    if (rc) return rc;
    int flags = 0;
    if ((rc = read_flags(o, s, &flags))) return rc;
    if (flags & FLAG_BADPOOL) return bad_pool_error(o, s);
    if (!(flags & (FLAG_ARENA | FLAG_HASH))) return EMU_OK;
    recover(o, flags, n, s, &rc, true);
    if (rc) return rc;
  }
  return fail(EMU_ERR_CAPACITY, "oracle could not place the pools of the pending keys");
}

int emu_oracle_seed_pcg64(emu_oracle_t o, const uint64_t* st6) {
  if (!o || !st6) return fail(EMU_ERR_INVALID, "NULL oracle/state");
  EMU_CUDA(cudaMemcpy(o->pcg, st6, 6 * sizeof(uint64_t), cudaMemcpyDefault));
  // a pageable-source copy may return before its DMA lands; the step server
  // (another stream) must see the new state on its next request
  EMU_CUDA(cudaStreamSynchronize(0));
  return EMU_OK;
}

int emu_oracle_get_pcg64(emu_oracle_t o, uint64_t* st6) {
  if (!o || !st6) return fail(EMU_ERR_INVALID, "NULL oracle/state");
  EMU_CUDA(cudaMemcpy(st6, o->pcg, 6 * sizeof(uint64_t), cudaMemcpyDefault));
  return EMU_OK;
}

static constexpr uint64_t kServerMaxNs = 2000000000ULL;  // relaunched at least every 2 s
// exit after this long without a step (EMU_STEP_SERVER_IDLE_US, default 100 ms:
// longer than the engine's inter-step sleeps, so cadence calls find it resident)
static uint64_t server_idle_ns() {
  static const uint64_t v = [] {
    const char* e = getenv("EMU_STEP_SERVER_IDLE_US");
    const long long us = e ? atoll(e) : 100000;
    return (uint64_t)std::max<long long>(us, 1) * 1000ULL;
  }();
  return v;
}

int emu_oracle_park(emu_oracle_t o) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  quiesce_server(o);
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

static int launch_server(emu_oracle_t o) {
  *(volatile int*)o->alive_host = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  EMU_LAUNCH("step_server", o->srv_stream,
             k_step_server<<<1, 32, 0, o->srv_stream>>>(o->map, o->arena, o->plane[0].samples, o->plane[1].samples,
                                                        o->pcg, o->req_dev, o->step_dev, o->served_dev,
                                                        o->alive_dev, server_idle_ns(), kServerMaxNs));
  EMU_CUDA(cudaGetLastError());
  EMU_CUDA(cudaEventRecord(o->srv_done, o->srv_stream));
  return EMU_OK;
}

// One step through the resident server: returns the result flags (0 = done,
// kStepMiss = key not cached), or -1 with an error set.
static int step_via_server(emu_oracle_t o, int32_t tt, int32_t conc, int ph, double* out_lat) {
  if (o->async_pending) {  // stream order: pools the server reads must be settled
    if (cudaEventSynchronize(o->async_done) != cudaSuccess) return -1 + 0 * cuda_fail(cudaGetLastError(), "flush");
    o->async_pending = false;
  }
  volatile StepReq* rq = o->req_host;
  volatile StepOut* h = o->step_host;
  const uint32_t seq = ++o->step_seq;
  rq->tt = tt;
  rq->conc = conc;
  rq->phase = ph;  // clears the park bit
  std::atomic_thread_fence(std::memory_order_seq_cst);
  rq->seq = seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (!*(volatile int*)o->alive_host && cudaEventQuery(o->srv_done) != cudaErrorNotReady) {
    if (launch_server(o)) return -1;
  }
  for (uint64_t spin = 1; h->seq != seq; spin++) {
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaEventQuery(o->srv_done);
      if (e != cudaSuccess && e != cudaErrorNotReady) return -1 + 0 * cuda_fail(e, "k_step_server");
      std::atomic_thread_fence(std::memory_order_seq_cst);
      if (e == cudaSuccess && h->seq != seq && launch_server(o)) return -1;  // exited before our request
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  const int f = h->flags;
  if (f == 0) *out_lat = h->lat;
  return f;
}

int emu_oracle_step(emu_oracle_t o, int32_t tt, int32_t conc, int32_t phase, double* out_lat) {
  if (!o || !out_lat) return fail(EMU_ERR_INVALID, "NULL oracle/out");
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  const int ph = phase ? 1 : 0;
  cudaStream_t s = 0;
  volatile StepOut* h = o->step_host;
  bool full = false;  // first try the cached-key path (resident server, else k_step_hit)
  if (o->server) {
    const int f = step_via_server(o, tt, conc, ph, out_lat);
    if (f < 0) return EMU_ERR_CUDA;
    if (f == 0) return EMU_OK;
    full = true;  // kStepMiss: build the pool with k_step below
  }
  for (int attempt = 0; attempt < 5; attempt++) {
    const uint32_t seq = ++o->step_seq;
    if (!full) {
      EMU_LAUNCH("step_hit", s, k_step_hit<<<1, 32, 0, s>>>(o->map, o->arena, o->plane[0].samples, o->plane[1].samples,
                                                              tt, conc, ph, o->pcg, o->step_dev, seq));
    } else {
      Sink sk = make_sink(o);
      EMU_LAUNCH("step", s, k_step<<<1, kCtaThreads, kCtaSmem, s>>>(o->plane[0], o->plane[1], o->cfg, sk, tt, conc, ph,
                                                                   o->pcg, o->gd, o->gb, o->gcap, o->step_dev, seq));
    }
    EMU_CUDA(cudaGetLastError());
    // spin on the mapped result; poll the stream now and then so a failed
    // kernel surfaces as an error instead of a hang
    for (uint64_t spin = 1; h->seq != seq; spin++) {
      if ((spin & 4095) == 0) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_fail(e, "k_step");
        if (e == cudaSuccess && h->seq != seq) {
          std::atomic_thread_fence(std::memory_order_seq_cst);
          if (h->seq != seq) return fail(EMU_ERR_CUDA, "k_step finished without publishing its result");
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const int f = h->flags;
    if (f == 0) {
      *out_lat = h->lat;
      return EMU_OK;
    }
    if (f == kStepMiss) {
      full = true;
      continue;
    }
    EMU_CUDA(cudaStreamSynchronize(s));
    if (f & FLAG_BADPOOL) return bad_pool_error(o, s);
    int rc = EMU_OK;
    if (f & FLAG_HASH) rc = alloc_hash(o, o->map.hcap * 4);
    if (!rc) rc = oracle_flush(o, s);
    if (!rc) EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    if (rc) return rc;
  }
  return fail(EMU_ERR_CAPACITY, "oracle step could not place its pool");
}

int emu_oracle_pool(emu_oracle_t o, const int32_t* key_tt, const int32_t* key_conc, const uint8_t* key_phase, int64_t U,
                    int64_t* pool_off, int32_t* pool_bkt, double* pool_dist, double* pool_prob, double* pool_cdf,
                    int64_t cap, int32_t* table_of_key, void* stream) {
  if (!o) return fail(EMU_ERR_INVALID, "NULL oracle");
  if (U < 0) return fail(EMU_ERR_INVALID, "negative key count");
  cudaStream_t s = as_stream(stream);
  static const bool sync_check = [] {
    const char* v = getenv("EMU_SYNC_CHECK");
    return v && v[0] == '1';
  }();
  std::vector<int64_t> off((size_t)U + 1, 0);
  if (U == 0) {
    EMU_CUDA(cudaMemcpyAsync(pool_off, off.data(), sizeof(int64_t), cudaMemcpyHostToDevice, s));
    EMU_CUDA(cudaStreamSynchronize(s));
    return EMU_OK;
  }
  if (!o->has_data) return fail(EMU_ERR_NO_DATA, "profile pack has no samples in any table");
  const int64_t kmax = o->kmax;
  const int64_t budget = 256LL << 20;
  int64_t chunkU = std::max<int64_t>(1, std::min<int64_t>(U, budget / (kmax * 28)));
  int32_t* xb = nullptr;
  double *xd = nullptr, *xp = nullptr, *xc = nullptr;
  int64_t* xK = nullptr;
  int64_t* doff = nullptr;
  int rc;
  struct Scratch {  // freed on every return path
    int32_t*& xb;
    double *&xd, *&xp, *&xc;
    int64_t *&xK, *&doff;
    ~Scratch() {
      cudaFree(xb);
      cudaFree(xd);
      cudaFree(xp);
      cudaFree(xc);
      cudaFree(xK);
      cudaFree(doff);
    }
  } scratch{xb, xd, xp, xc, xK, doff};
  if ((rc = dalloc(&xb, chunkU * kmax)) || (rc = dalloc(&xd, chunkU * kmax)) || (rc = dalloc(&xp, chunkU * kmax)) ||
      (rc = dalloc(&xc, chunkU * kmax)) || (rc = dalloc(&xK, chunkU)) || (rc = dalloc(&doff, chunkU))) {
    return rc;
  }
  if ((rc = ensure_key_capacity(o, chunkU))) {
    return rc;
  }
  std::vector<int64_t> hK((size_t)chunkU);
  bool over = false;
  for (int64_t u0 = 0; u0 < U; u0 += chunkU) {
    const int64_t n = std::min(chunkU, U - u0);
    EMU_CUDA(cudaMemsetAsync(o->ctl, 0, sizeof(BatchCtl), s));
    EMU_CUDA(cudaMemsetAsync(xK, 0xff, 8 * n, s));  // -1: a key no tier emitted is caught below
    Keys keys{key_tt + u0, key_conc + u0, key_phase + u0, nullptr, nullptr, n};
    Sink sk = make_sink(o);
    sk.x_bkt = xb;
    sk.x_dist = xd;
    sk.x_prob = xp;
    sk.x_cdf = xc;
    sk.x_K = xK;
    if ((rc = launch_pool_tiers<1>(o, keys, sk, s, sync_check))) return rc;
    EMU_CUDA(cudaMemcpyAsync(hK.data(), xK, 8 * n, cudaMemcpyDeviceToHost, s));
    EMU_CUDA(cudaStreamSynchronize(s));
    for (int64_t u = 0; u < n; u++) {
      if (hK[u] < 0 || hK[u] > kmax) {
        return fail(EMU_ERR_CUDA, "emu_oracle_pool: key " + std::to_string(u0 + u) + " got no valid pool (K=" +
                                      std::to_string(hK[u]) + ")");
      }
      off[u0 + u + 1] = off[u0 + u] + hK[u];
    }
    if (off[u0 + n] > cap) over = true;
    if (!over) {
      EMU_CUDA(cudaMemcpyAsync(doff, off.data() + u0, 8 * n, cudaMemcpyHostToDevice, s));
      EMU_LAUNCH("gather", s, k_gather_pools<<<grid_for(n * 32, 256, 4096), 256, 0, s>>>(xK, doff, n, kmax, 0, xb, xd, xp, xc, pool_bkt,
                                                                 pool_dist, pool_prob, pool_cdf, cap));
      EMU_CUDA(cudaGetLastError());
      EMU_CUDA(cudaStreamSynchronize(s));
    }
  }
  EMU_CUDA(cudaMemcpyAsync(pool_off, off.data(), 8 * (U + 1), cudaMemcpyHostToDevice, s));
  if (table_of_key) {
    EMU_LAUNCH("table_of_key", s, k_table_of_key<<<grid_for(U, 256, 1024), 256, 0, s>>>(key_phase, U, o->plane_tab[0], o->plane_tab[1], table_of_key));
    EMU_CUDA(cudaGetLastError());
  }
  EMU_CUDA(cudaStreamSynchronize(s));
  if (over) return fail(EMU_ERR_CAPACITY, "pool output capacity exceeded; pool_off holds the sizes");
  return EMU_OK;
}

}  // extern "C"

#ifdef EMU_STATS
extern "C" int emu_stats_read(unsigned long long* out32) {
  EMU_CUDA(cudaMemcpyFromSymbol(out32, emu::g_stats, sizeof(unsigned long long) * 32));
  unsigned long long z[32] = {0};
  EMU_CUDA(cudaMemcpyToSymbol(emu::g_stats, z, sizeof(z)));
  return EMU_OK;
}
#endif

#ifdef EMU_CHECK
// Debug builds: number of failed device invariant checks since the last read.
extern "C" int emu_check_read(unsigned long long* n) {
  EMU_CUDA(cudaDeviceSynchronize());
  EMU_CUDA(cudaMemcpyFromSymbol(n, emu::g_check_fail, sizeof(unsigned long long)));
  unsigned long long z = 0;
  EMU_CUDA(cudaMemcpyToSymbol(emu::g_check_fail, &z, sizeof(z)));
  return EMU_OK;
}
#endif
