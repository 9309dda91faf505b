/*
 * emu_oracle.c -- CPU restatement of LLM-Emu's density-aware profile oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the "port" CPU baseline timed by bench.py.  Nothing in the product
 * package (paper_2605_00616_b200/) may import, link or execute it; only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs do.
 *
 * Parity pinning: tests/test_oracle_cpu.py checks every function here against
 * golden vectors produced by the unmodified reference (tests/golden/, made by
 * tests/golden/make_golden.py importing /root/reference/pkg/src/serve_emu) and
 * against the reference test-suite fixtures.
 *
 * The reference's arithmetic lives in numpy 2.3 (pinned floor numpy>=1.24,
 * pkg/pyproject.toml:11); the restated numpy semantics are:
 *   - ndarray.sum of float64: pairwise summation (8 accumulators, blocks of
 *     128, split n2 = n/2 - (n/2)%8), reduction starting from +0.0.
 *   - x ** 2.0 -> x*x, x ** 0.5 -> sqrt(x), x ** 1.0 -> x (numpy fast scalar
 *     power); other exponents -> pow() (numpy uses a SIMD pow that can differ
 *     by 1 ulp: the CDF tolerance 1e-6 applies there).
 *   - ndarray.cumsum: sequential.
 *   - Generator.choice(K, p): cdf = cumsum(p); cdf /= cdf[-1];
 *     idx = searchsorted(cdf, random(), 'right'); random() = (next64>>11)*2^-53.
 *   - Generator.integers(n): n == 1 -> 0 without drawing; else Lemire on
 *     PCG64's buffered next_uint32 with threshold (2^32 - n) % n.
 *   - PCG64: 128-bit LCG, multiplier 0x2360ED051FC65DA44385DF649FCCF645,
 *     XSL-RR output of the stepped state.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __uint128_t u128;

/* ------------------------------------------------------------------ tables */
typedef struct {
  int64_t nb, ns;
  const int32_t* tt;   /* sorted by (tt, conc) */
  const int32_t* conc;
  const int64_t* off;  /* nb + 1 */
  const double* samples;
  int32_t tt_lo, tt_hi, c_lo, c_hi;
} ora_table;

static void table_ranges(ora_table* t) {
  if (t->nb == 0) return;
  t->tt_lo = t->tt[0];
  t->tt_hi = t->tt[t->nb - 1];
  int32_t lo = t->conc[0], hi = t->conc[0];
  for (int64_t i = 1; i < t->nb; i++) {
    if (t->conc[i] < lo) lo = t->conc[i];
    if (t->conc[i] > hi) hi = t->conc[i];
  }
  t->c_lo = lo;
  t->c_hi = hi;
}

/* normalized_distance, oracle.py:62-77 (and the vectorised form :92-97).
 * (t - tt) is an exact integer in double; '/' and sqrt are IEEE rn. */
double ora_distance(int64_t t, int64_t c, int64_t tt, int64_t conc, int64_t tt_lo, int64_t tt_hi,
                    int64_t c_lo, int64_t c_hi) {
  volatile double dt = 0.0, dc = 0.0; /* volatile: forbid FMA contraction */
  if (tt_hi != tt_lo) dt = (double)(t - tt) / (double)(tt_hi - tt_lo);
  if (c_hi != c_lo) dc = (double)(c - conc) / (double)(c_hi - c_lo);
  volatile double a = dt * dt;
  volatile double b = dc * dc;
  volatile double s = a + b;
  return sqrt(s);
}

/* ------------------------------------------------------- pool (Alg. 1) ---- */
typedef struct {
  double d;
  int32_t b;
} cand;

static inline int cand_less(const cand* x, const cand* y) {
  /* np.lexsort((concs, tts, dists)): by distance, then tt, then conc.  Buckets
   * are sorted by (tt, conc), so the tie-break is ascending bucket index. */
  if (x->d != y->d) return x->d < y->d;
  return x->b < y->b;
}

static int cand_cmp(const void* a, const void* b) {
  const cand* x = (const cand*)a;
  const cand* y = (const cand*)b;
  if (cand_less(x, y)) return -1;
  if (cand_less(y, x)) return 1;
  return 0;
}

static void heap_sift_down(cand* h, int64_t n, int64_t i) {
  /* max-heap by cand order */
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && cand_less(&h[m], &h[l])) m = l;
    if (r < n && cand_less(&h[m], &h[r])) m = r;
    if (m == i) return;
    cand tmp = h[i];
    h[i] = h[m];
    h[m] = tmp;
    i = m;
  }
}

/* _pool_order (oracle.py:80-105): the shortest prefix of the (d, tt, conc)
 * order whose cumulative count reaches floor, or every bucket if the table
 * holds fewer than floor samples.  Because each bucket holds >= 1 sample the
 * prefix has at most floor entries, so the floor smallest candidates are
 * selected with a bounded heap and then sorted -- same result as lexsort.
 * scratch must hold nb cands.  Returns K. */
int64_t ora_pool(const ora_table* t, int64_t q_tt, int64_t q_c, int64_t floor, int32_t* out_bkt,
                 double* out_dist, cand* scratch) {
  int64_t nb = t->nb;
  if (nb == 0) return 0;
  int64_t cap = floor < nb ? floor : nb;
  int64_t n = 0;
  for (int64_t i = 0; i < nb; i++) {
    cand c;
    c.d = ora_distance(q_tt, q_c, t->tt[i], t->conc[i], t->tt_lo, t->tt_hi, t->c_lo, t->c_hi);
    c.b = (int32_t)i;
    if (n < cap) {
      scratch[n++] = c;
      if (n == cap)
        for (int64_t j = cap / 2 - 1; j >= 0; j--) heap_sift_down(scratch, cap, j);
    } else if (cand_less(&c, &scratch[0])) {
      scratch[0] = c;
      heap_sift_down(scratch, cap, 0);
    }
  }
  qsort(scratch, (size_t)n, sizeof(cand), cand_cmp);
  int64_t cum = 0, k = n;
  for (int64_t j = 0; j < n; j++) {
    int32_t b = scratch[j].b;
    cum += t->off[b + 1] - t->off[b];
    if (cum >= floor) {
      k = j + 1;
      break;
    }
  }
  for (int64_t j = 0; j < k; j++) {
    out_bkt[j] = scratch[j].b;
    out_dist[j] = scratch[j].d;
  }
  return k;
}

/* numpy pairwise_sum for float64 (add.reduce on a contiguous array). */
double ora_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return ora_pairwise_sum(a, n2) + ora_pairwise_sum(a + n2, n - n2);
  }
}

static double shepard_pow(double x, double p) {
  if (p == 2.0) return x * x;
  if (p == 1.0) return x;
  if (p == 0.5) return sqrt(x);
  return pow(x, p);
}

/* _selection_probs (oracle.py:124-127) followed by the cdf Generator.choice
 * builds (cumsum, then / cdf[-1]).  mass, probs, cdf: K entries each. */
void ora_probs(const double* dist, const int64_t* counts, int64_t K, double p, double eps,
               double* mass, double* probs, double* cdf) {
  for (int64_t j = 0; j < K; j++) {
    double x = dist[j] > eps ? dist[j] : eps; /* np.maximum(d, eps) */
    volatile double w = 1.0 / shepard_pow(x, p);
    mass[j] = w * (double)counts[j];
  }
  double s = ora_pairwise_sum(mass, K);
  for (int64_t j = 0; j < K; j++) probs[j] = mass[j] / s;
  double acc = 0.0;
  for (int64_t j = 0; j < K; j++) {
    acc = (j == 0) ? probs[0] : acc + probs[j];
    cdf[j] = acc;
  }
  double last = cdf[K - 1];
  for (int64_t j = 0; j < K; j++) cdf[j] = cdf[j] / last;
}

/* searchsorted(cdf, u, side='right'): number of entries <= u. */
int64_t ora_search_right(const double* cdf, int64_t K, double u) {
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* ------------------------------------------------------------------ RNGs -- */
typedef struct {
  u128 state, inc;
  int has_uint32;
  uint32_t uinteger;
} pcg64;

static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static inline uint64_t pcg64_next64(pcg64* g) {
  g->state = g->state * PCG_MULT + g->inc;
  uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(g->state >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

static inline uint32_t pcg64_next32(pcg64* g) {
  if (g->has_uint32) {
    g->has_uint32 = 0;
    return g->uinteger;
  }
  uint64_t v = pcg64_next64(g);
  g->has_uint32 = 1;
  g->uinteger = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

static inline double u64_to_unit(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }

/* PCG-RXS-M-XS 32-bit hash: the continuation word stream of EXPLICIT mode. */
static inline uint32_t hash32(uint32_t x) {
  uint32_t s = x * 747796405u + 2891336453u;
  uint32_t w = ((s >> ((s >> 28u) + 4u)) ^ s) * 277803737u;
  return (w >> 22u) ^ w;
}

/* Philox4x32-10 (Salmon et al., SC'11; Random123 philox4x32_R with R=10). */
void ora_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Word streams for the index draw. */
typedef struct {
  int mode; /* 0 explicit, 1 philox, 2 pcg64 */
  uint32_t cur;
  int first;
  /* philox */
  uint64_t qid, seed;
  uint32_t buf[4];
  int pos, block;
  pcg64* g;
} word_stream;

static uint32_t ws_next(word_stream* s) {
  if (s->mode == 2) return pcg64_next32(s->g);
  if (s->mode == 0) {
    if (s->first) {
      s->first = 0;
      return s->cur;
    }
    s->cur = hash32(s->cur);
    return s->cur;
  }
  if (s->pos == 4) {
    uint32_t ctr[4] = {(uint32_t)s->qid, (uint32_t)(s->qid >> 32), (uint32_t)s->block, 0};
    uint32_t key[2] = {(uint32_t)s->seed, (uint32_t)(s->seed >> 32)};
    ora_philox4x32_10(ctr, key, s->buf);
    s->block++;
    s->pos = 0;
  }
  return s->buf[s->pos++];
}

/* Generator.integers(n) for 1 <= n <= 2^32 (numpy random_bounded_uint64_fill
 * -> buffered_bounded_lemire_uint32). */
static uint32_t lemire_index(word_stream* s, uint64_t n) {
  if (n == 1) return 0;
  if (n == 4294967296ULL) return ws_next(s);
  uint32_t excl = (uint32_t)n;
  uint64_t m = (uint64_t)ws_next(s) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    uint32_t thr = (uint32_t)((0xFFFFFFFFu - (excl - 1)) % excl);
    while (left < thr) {
      m = (uint64_t)ws_next(s) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

/* ------------------------------------------------------- oracle instance -- */
typedef struct {
  int64_t key;    /* (plane<<62) | ((tt & 0x7fffffff)<<31) | (conc & 0x7fffffff); -1 empty */
  int64_t start;  /* offset into pool store */
  int64_t K;
} cache_ent;

typedef struct {
  cache_ent* ents;
  int64_t cap, used;
  /* pool store */
  double* cdf;
  int64_t* soff; /* sample offset of the bucket */
  int64_t* cnt;
  int64_t store_cap, store_used;
  /* scratch */
  cand* scratch;
  int32_t* bk;
  double* dist;
  int64_t* cnts;
  double* mass;
  double* probs;
} ora_cache;

typedef struct {
  ora_table tab[3];
  int plane_table[2]; /* effective table per phase (combined fallback) */
  int64_t floor;
  double p, eps;
} ora_oracle;

static uint64_t key_hash(int64_t k) {
  uint64_t x = (uint64_t)k;
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static void cache_init(ora_cache* c, int64_t max_nb) {
  memset(c, 0, sizeof(*c));
  c->cap = 1024;
  c->ents = (cache_ent*)malloc(sizeof(cache_ent) * c->cap);
  for (int64_t i = 0; i < c->cap; i++) c->ents[i].key = -1;
  c->store_cap = 4096;
  c->cdf = (double*)malloc(sizeof(double) * c->store_cap);
  c->soff = (int64_t*)malloc(sizeof(int64_t) * c->store_cap);
  c->cnt = (int64_t*)malloc(sizeof(int64_t) * c->store_cap);
  int64_t m = max_nb > 0 ? max_nb : 1;
  c->scratch = (cand*)malloc(sizeof(cand) * m);
  c->bk = (int32_t*)malloc(sizeof(int32_t) * m);
  c->dist = (double*)malloc(sizeof(double) * m);
  c->cnts = (int64_t*)malloc(sizeof(int64_t) * m);
  c->mass = (double*)malloc(sizeof(double) * m);
  c->probs = (double*)malloc(sizeof(double) * m);
}

static void cache_free(ora_cache* c) {
  free(c->ents);
  free(c->cdf);
  free(c->soff);
  free(c->cnt);
  free(c->scratch);
  free(c->bk);
  free(c->dist);
  free(c->cnts);
  free(c->mass);
  free(c->probs);
}

static cache_ent* cache_find(ora_cache* c, int64_t key, int* found) {
  uint64_t mask = (uint64_t)c->cap - 1;
  uint64_t h = key_hash(key) & mask;
  for (;;) {
    cache_ent* e = &c->ents[h];
    if (e->key == key) {
      *found = 1;
      return e;
    }
    if (e->key == -1) {
      *found = 0;
      return e;
    }
    h = (h + 1) & mask;
  }
}

static void cache_grow(ora_cache* c) {
  cache_ent* old = c->ents;
  int64_t oc = c->cap;
  c->cap *= 2;
  c->ents = (cache_ent*)malloc(sizeof(cache_ent) * c->cap);
  for (int64_t i = 0; i < c->cap; i++) c->ents[i].key = -1;
  for (int64_t i = 0; i < oc; i++)
    if (old[i].key != -1) {
      int f;
      cache_ent* e = cache_find(c, old[i].key, &f);
      *e = old[i];
    }
  free(old);
}

/* LatencyOracle._pooled (oracle.py:200-222): cached pool of (phase, tt, conc). */
static cache_ent* pooled(const ora_oracle* o, ora_cache* c, int phase, int64_t tt, int64_t conc) {
  int64_t key = ((int64_t)phase << 62) | ((tt & 0x7fffffffLL) << 31) | (conc & 0x7fffffffLL);
  int f;
  cache_ent* e = cache_find(c, key, &f);
  if (f) return e;
  const ora_table* t = &o->tab[o->plane_table[phase]];
  int64_t K = ora_pool(t, tt, conc, o->floor, c->bk, c->dist, c->scratch);
  for (int64_t j = 0; j < K; j++) c->cnts[j] = t->off[c->bk[j] + 1] - t->off[c->bk[j]];
  if (c->store_used + K > c->store_cap) {
    while (c->store_used + K > c->store_cap) c->store_cap *= 2;
    c->cdf = (double*)realloc(c->cdf, sizeof(double) * c->store_cap);
    c->soff = (int64_t*)realloc(c->soff, sizeof(int64_t) * c->store_cap);
    c->cnt = (int64_t*)realloc(c->cnt, sizeof(int64_t) * c->store_cap);
  }
  ora_probs(c->dist, c->cnts, K, o->p, o->eps, c->mass, c->probs, c->cdf + c->store_used);
  for (int64_t j = 0; j < K; j++) {
    c->soff[c->store_used + j] = t->off[c->bk[j]];
    c->cnt[c->store_used + j] = c->cnts[j];
  }
  e->key = key;
  e->start = c->store_used;
  e->K = K;
  c->store_used += K;
  c->used++;
  if (c->used * 2 > c->cap) {
    cache_grow(c);
    e = cache_find(c, key, &f);
  }
  return e;
}

/* _draw (oracle.py:130-135) given the pool entry and a word stream. */
static void draw(const ora_oracle* o, const ora_cache* c, const cache_ent* e, int phase,
                 uint64_t usel, word_stream* ws, double* lat, int32_t* sidx) {
  double u = u64_to_unit(usel);
  int64_t j = ora_search_right(c->cdf + e->start, e->K, u);
  int64_t n = c->cnt[e->start + j];
  int64_t s = c->soff[e->start + j] + lemire_index(ws, (uint64_t)n);
  const ora_table* t = &o->tab[o->plane_table[phase]];
  *lat = t->samples[s];
  *sidx = (int32_t)s;
}

static int64_t max_nb(const ora_oracle* o) {
  int64_t m = 0;
  for (int i = 0; i < 3; i++)
    if (o->tab[i].nb > m) m = o->tab[i].nb;
  return m;
}

/* Returns 0 ok, 1 no data. */
static int oracle_setup(ora_oracle* o, const int64_t nbs[3], const int64_t nss[3],
                        const int32_t* tts[3], const int32_t* concs[3], const int64_t* offs[3],
                        const double* samples[3], int64_t floor, double p, double eps) {
  for (int i = 0; i < 3; i++) {
    o->tab[i].nb = nbs[i];
    o->tab[i].ns = nss[i];
    o->tab[i].tt = tts[i];
    o->tab[i].conc = concs[i];
    o->tab[i].off = offs[i];
    o->tab[i].samples = samples[i];
    table_ranges(&o->tab[i]);
  }
  for (int ph = 0; ph < 2; ph++) o->plane_table[ph] = o->tab[ph].nb > 0 ? ph : 2;
  o->floor = floor;
  o->p = p;
  o->eps = eps;
  for (int ph = 0; ph < 2; ph++)
    if (o->tab[o->plane_table[ph]].nb == 0) return 1;
  return 0;
}

typedef struct {
  const ora_oracle* o;
  const int32_t *qt, *qc;
  const uint8_t* qp;
  int64_t lo, hi;
  int mode;
  const uint64_t* usel;
  const uint32_t* uidx;
  uint64_t seed, ctr_base;
  double* lat;
  int32_t* sidx;
} shard_arg;

static void* shard_run(void* arg) {
  shard_arg* a = (shard_arg*)arg;
  ora_cache c;
  cache_init(&c, max_nb(a->o));
  for (int64_t i = a->lo; i < a->hi; i++) {
    int ph = a->qp[i] ? 1 : 0;
    cache_ent* e = pooled(a->o, &c, ph, a->qt[i], a->qc[i]);
    word_stream ws;
    memset(&ws, 0, sizeof(ws));
    uint64_t usel;
    if (a->mode == 0) {
      ws.mode = 0;
      ws.cur = a->uidx[i];
      ws.first = 1;
      usel = a->usel[i];
    } else {
      ws.mode = 1;
      ws.qid = a->ctr_base + (uint64_t)i;
      ws.seed = a->seed;
      ws.pos = 4;
      ws.block = 0;
      uint32_t w0 = ws_next(&ws), w1 = ws_next(&ws);
      usel = (uint64_t)w0 | ((uint64_t)w1 << 32);
    }
    draw(a->o, &c, e, ph, usel, &ws, &a->lat[i], &a->sidx[i]);
  }
  cache_free(&c);
  return NULL;
}

/* Batched sampling, EXPLICIT (mode 0) or PHILOX (mode 1) uniforms, sharded
 * over `threads` POSIX threads (each with its own pool cache, like one
 * LatencyOracle per process).  Returns 0 ok, 1 no data. */
int ora_sample_batch(const int64_t nbs[3], const int64_t nss[3], const int32_t* tts[3],
                     const int32_t* concs[3], const int64_t* offs[3], const double* samples[3],
                     int64_t floor, double p, double eps, const int32_t* qt, const int32_t* qc,
                     const uint8_t* qp, int64_t Q, int mode, const uint64_t* usel,
                     const uint32_t* uidx, uint64_t seed, uint64_t ctr_base, double* lat,
                     int32_t* sidx, int threads) {
  ora_oracle o;
  if (oracle_setup(&o, nbs, nss, tts, concs, offs, samples, floor, p, eps)) return 1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  shard_arg args[256];
  int64_t per = (Q + threads - 1) / threads;
  int nt = 0;
  for (int k = 0; k < threads; k++) {
    int64_t lo = (int64_t)k * per, hi = lo + per < Q ? lo + per : Q;
    if (lo >= hi) break;
    args[k] = (shard_arg){&o, qt, qc, qp, lo, hi, mode, usel, uidx, seed, ctr_base, lat, sidx};
    nt++;
  }
  if (nt == 1) {
    shard_run(&args[0]);
  } else {
    for (int k = 0; k < nt; k++) pthread_create(&th[k], NULL, shard_run, &args[k]);
    for (int k = 0; k < nt; k++) pthread_join(th[k], NULL);
  }
  return 0;
}

/* Sequential PCG64-stream sampling: LatencyOracle.sample called Q times
 * (oracle.py:224-226).  state6 = {state_hi, state_lo, inc_hi, inc_lo,
 * has_uint32, uinteger}, advanced in place.  Returns 0 ok, 1 no data. */
int ora_sample_pcg64(const int64_t nbs[3], const int64_t nss[3], const int32_t* tts[3],
                     const int32_t* concs[3], const int64_t* offs[3], const double* samples[3],
                     int64_t floor, double p, double eps, const int32_t* qt, const int32_t* qc,
                     const uint8_t* qp, int64_t Q, uint64_t* state6, double* lat, int32_t* sidx) {
  ora_oracle o;
  if (oracle_setup(&o, nbs, nss, tts, concs, offs, samples, floor, p, eps)) return 1;
  pcg64 g;
  g.state = ((u128)state6[0] << 64) | state6[1];
  g.inc = ((u128)state6[2] << 64) | state6[3];
  g.has_uint32 = (int)state6[4];
  g.uinteger = (uint32_t)state6[5];
  ora_cache c;
  cache_init(&c, max_nb(&o));
  for (int64_t i = 0; i < Q; i++) {
    int ph = qp[i] ? 1 : 0;
    cache_ent* e = pooled(&o, &c, ph, qt[i], qc[i]);
    word_stream ws;
    memset(&ws, 0, sizeof(ws));
    ws.mode = 2;
    ws.g = &g;
    uint64_t usel = pcg64_next64(&g);
    draw(&o, &c, e, ph, usel, &ws, &lat[i], &sidx[i]);
  }
  cache_free(&c);
  state6[0] = (uint64_t)(g.state >> 64);
  state6[1] = (uint64_t)g.state;
  state6[2] = (uint64_t)(g.inc >> 64);
  state6[3] = (uint64_t)g.inc;
  state6[4] = (uint64_t)g.has_uint32;
  state6[5] = g.uinteger;
  return 0;
}

/* Explicit pools for U keys (pool_neighbors + _selection_probs + choice cdf).
 * pool_off[U+1]; outputs sized cap.  Returns 0 ok, 1 no data, 4 capacity. */
int ora_pool_batch(const int64_t nbs[3], const int64_t nss[3], const int32_t* tts[3],
                   const int32_t* concs[3], const int64_t* offs[3], const double* samples[3],
                   int64_t floor, double p, double eps, const int32_t* kt, const int32_t* kc,
                   const uint8_t* kp, int64_t U, int64_t* pool_off, int32_t* pool_bkt,
                   double* pool_dist, double* pool_prob, double* pool_cdf, int64_t cap,
                   int32_t* table_of_key) {
  ora_oracle o;
  if (oracle_setup(&o, nbs, nss, tts, concs, offs, samples, floor, p, eps)) return 1;
  int64_t m = max_nb(&o);
  cand* scratch = (cand*)malloc(sizeof(cand) * (m ? m : 1));
  int32_t* bk = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  double* dist = (double*)malloc(sizeof(double) * (m ? m : 1));
  int64_t* cnts = (int64_t*)malloc(sizeof(int64_t) * (m ? m : 1));
  double* mass = (double*)malloc(sizeof(double) * (m ? m : 1));
  double* probs = (double*)malloc(sizeof(double) * (m ? m : 1));
  double* cdf = (double*)malloc(sizeof(double) * (m ? m : 1));
  int rc = 0;
  pool_off[0] = 0;
  for (int64_t u = 0; u < U; u++) {
    int ph = kp[u] ? 1 : 0;
    int ti = o.plane_table[ph];
    const ora_table* t = &o.tab[ti];
    int64_t K = ora_pool(t, kt[u], kc[u], floor, bk, dist, scratch);
    for (int64_t j = 0; j < K; j++) cnts[j] = t->off[bk[j] + 1] - t->off[bk[j]];
    ora_probs(dist, cnts, K, p, eps, mass, probs, cdf);
    int64_t base = pool_off[u];
    pool_off[u + 1] = base + K;
    table_of_key[u] = ti;
    if (base + K > cap) {
      rc = 4;
      continue;
    }
    for (int64_t j = 0; j < K; j++) {
      pool_bkt[base + j] = bk[j];
      pool_dist[base + j] = dist[j];
      pool_prob[base + j] = probs[j];
      pool_cdf[base + j] = cdf[j];
    }
  }
  free(scratch);
  free(bk);
  free(dist);
  free(cnts);
  free(mass);
  free(probs);
  free(cdf);
  return rc;
}

/* --------------------------------------------------------- table build ---- */
typedef struct {
  int32_t tt, conc;
  uint64_t lat_bits;
  int64_t idx;
} rec_key;

static int canonical_flag;

static int rec_cmp(const void* a, const void* b) {
  const rec_key* x = (const rec_key*)a;
  const rec_key* y = (const rec_key*)b;
  if (x->tt != y->tt) return x->tt < y->tt ? -1 : 1;
  if (x->conc != y->conc) return x->conc < y->conc ? -1 : 1;
  if (canonical_flag && x->lat_bits != y->lat_bits) return x->lat_bits < y->lat_bits ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0); /* stable: capture order */
}

/* build_pack (profile.py:230-267) over record SoA.  For each table id
 * (0 decode, 1 mixed, 2 combined) writes bucket arrays (capacity n each) and
 * samples (capacity n each); nb_out[3], ns_out[3].  canonical != 0 orders
 * samples ascending inside each bucket (save_pack, profile.py:281-282).
 * Returns 0 ok, or 2 with *bad_index / *bad_code (first invalid record,
 * checks in StepTraceRecord.validate order, profile.py:61-79). */
int ora_build(const int32_t* tt, const int32_t* conc, const uint8_t* phase, const double* lat,
              const int64_t* step, int64_t n, int canonical, int32_t* bt[3], int32_t* bc[3],
              int64_t* boff[3], double* bs[3], int64_t nb_out[3], int64_t ns_out[3],
              int64_t* bad_index, int32_t* bad_code) {
  for (int64_t i = 0; i < n; i++) {
    int code = 0;
    if (step && step[i] < 0)
      code = 1;
    else if (tt[i] < 1)
      code = 2;
    else if (conc[i] < 1)
      code = 3;
    else if (phase[i] == 0 && tt[i] < conc[i])
      code = 4;
    else if (!(lat[i] > 0.0))
      code = 5;
    if (code) {
      *bad_index = i;
      *bad_code = code;
      return 2;
    }
  }
  rec_key* keys = (rec_key*)malloc(sizeof(rec_key) * (n ? n : 1));
  for (int64_t i = 0; i < n; i++) {
    keys[i].tt = tt[i];
    keys[i].conc = conc[i];
    memcpy(&keys[i].lat_bits, &lat[i], 8);
    keys[i].idx = i;
  }
  canonical_flag = canonical;
  qsort(keys, (size_t)n, sizeof(rec_key), rec_cmp);
  for (int t = 0; t < 3; t++) {
    int64_t nb = 0, ns = 0;
    int32_t ptt = 0, pc = 0;
    for (int64_t i = 0; i < n; i++) {
      int64_t r = keys[i].idx;
      if (t < 2 && (int)(phase[r] ? 1 : 0) != t) continue;
      if (ns == 0 || keys[i].tt != ptt || keys[i].conc != pc) {
        bt[t][nb] = keys[i].tt;
        bc[t][nb] = keys[i].conc;
        boff[t][nb] = ns;
        nb++;
        ptt = keys[i].tt;
        pc = keys[i].conc;
      }
      bs[t][ns++] = lat[r];
    }
    boff[t][nb] = ns;
    nb_out[t] = nb;
    ns_out[t] = ns;
  }
  free(keys);
  return 0;
}

/* ---------------------------------------------------------- token fill ---- */
/* Token part of EmulatorEngine._apply_outcome (engine.py:464-483). */
void ora_token_fill(const uint8_t* is_prefill, const int32_t* chunk, const int32_t* progress,
                    const int32_t* prompt_len, const int32_t* generated, const int32_t* target,
                    int64_t n, int32_t* out_ids, uint8_t* out_finished) {
  for (int64_t e = 0; e < n; e++) {
    int decoding = 0, emit = 0;
    int32_t gen = generated[e];
    if (is_prefill[e]) {
      if (progress[e] + chunk[e] == prompt_len[e]) {
        decoding = 1;
        emit = 1;
      }
    } else {
      decoding = 1;
      emit = 1;
    }
    out_ids[e] = emit ? gen : -1;
    int32_t after = gen + (emit ? 1 : 0);
    out_finished[e] = (uint8_t)(decoding && after >= target[e]);
  }
}

/* Raw PCG64 words for tests. */
void ora_pcg64_words(uint64_t* state6, int64_t n, uint64_t* out) {
  pcg64 g;
  g.state = ((u128)state6[0] << 64) | state6[1];
  g.inc = ((u128)state6[2] << 64) | state6[3];
  g.has_uint32 = (int)state6[4];
  g.uinteger = (uint32_t)state6[5];
  for (int64_t i = 0; i < n; i++) out[i] = pcg64_next64(&g);
  state6[0] = (uint64_t)(g.state >> 64);
  state6[1] = (uint64_t)g.state;
}

uint32_t ora_hash32(uint32_t x) { return hash32(x); }
