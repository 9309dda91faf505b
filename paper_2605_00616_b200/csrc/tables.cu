// tables.cu -- device-resident profile tables (emu_tables_* of emu_abi.h).
//
// HBM layout per table (SoA, 64-byte aligned cudaMalloc blocks):
//   bkt_tt   i32[B]   bucket keys, sorted by (tt, conc)        (PhaseTable.from_buckets,
//   bkt_conc i32[B]                                            profile.py:122-129)
//   bkt_off  i64[B+1] sample offsets (bucket b = samples[off[b]:off[b+1]])
//   samples  f64[N]   latencies, the pack's own order inside a bucket
//   row_tt   i32[R]   distinct tt values (row index for the neighbour window)
//   row_start i64[R+1] first bucket of each row
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "emu_internal.cuh"
#include "prof.h"
#include "tables.h"

namespace emu {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return EMU_ERR_CUDA;
}

// Every table array comes from the device's stream-ordered pool, kept
// reserved (release threshold = max): repeated builds and table handles reuse
// the memory instead of mapping and unmapping it (cudaMalloc / cudaFree made
// the 100M-record build's time swing by 3x with what the previous build left).
cudaError_t table_alloc(void** p, size_t bytes, cudaStream_t s) {
  static const bool pool_set = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return true;
  }();
  (void)pool_set;
  return cudaMallocAsync(p, bytes > 0 ? bytes : 1, s);
}

void TableBuf::release() {
  cudaDeviceSynchronize();  // kernels on any stream may still read the table
  for (void* p : {(void*)bkt_tt, (void*)bkt_conc, (void*)bkt_off, (void*)samples, (void*)row_tt, (void*)row_start,
                  (void*)bsat, (void*)ssat, (void*)bmap, (void*)wpre, (void*)rowbase, (void*)col_start, (void*)col_tt,
                  (void*)col_b, (void*)sq_t, (void*)sq_c})
    if (p) cudaFreeAsync(p, 0);
  cudaStreamSynchronize(0);
  *this = TableBuf();
}

DevTable TableBuf::view() const {
  DevTable t;
  t.bkt_tt = bkt_tt;
  t.bkt_conc = bkt_conc;
  t.bkt_off = bkt_off;
  t.samples = samples;
  t.row_tt = row_tt;
  t.row_start = row_start;
  t.nb = nb;
  t.ns = ns;
  t.nrows = nrows;
  t.tt_lo = tt_lo;
  t.tt_hi = tt_hi;
  t.c_lo = c_lo;
  t.c_hi = c_hi;
  t.bsat = bsat;
  t.ssat = ssat;
  t.gnt = gnt;
  t.gnc = gnc;
  t.bmap = bmap;
  t.wpre = wpre;
  t.rowbase = rowbase;
  t.wpr = wpr;
  t.col_start = col_start;
  t.col_tt = col_tt;
  t.col_b = col_b;
  t.sq_t = sq_t;
  t.sq_c = sq_c;
  t.lt = lt;
  t.lc = lc;
  return t;
}

__global__ void k_sq_table(double* out, int64_t n, int64_t span) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double q = span ? __ddiv_rn((double)k, (double)span) : 0.0;
    out[k] = __dmul_rn(q, q);
  }
}

constexpr int64_t kMaxGridCells = 1LL << 27;  // per summed-area table (512 MB of int32)
constexpr int64_t kMaxSqTable = 1LL << 22;

int build_search_index(TableBuf& tb, const int32_t* h_tt, const int32_t* h_cc, const int64_t* h_off, cudaStream_t s) {
  if (tb.nb == 0) return EMU_OK;
  const int64_t span_t = (int64_t)tb.tt_hi - tb.tt_lo, span_c = (int64_t)tb.c_hi - tb.c_lo;
  tb.lt = std::min<int64_t>(span_t + 1, kMaxSqTable);
  tb.lc = std::min<int64_t>(span_c + 1, kMaxSqTable);
  EMU_CUDA(table_alloc((void**)&tb.sq_t, 8 * tb.lt, s));
  EMU_CUDA(table_alloc((void**)&tb.sq_c, 8 * tb.lc, s));
  EMU_LAUNCH("index", s, k_sq_table<<<(unsigned)std::min<int64_t>(1024, (tb.lt + 255) / 256), 256, 0, s>>>(tb.sq_t, tb.lt, span_t));
  EMU_LAUNCH("index", s, k_sq_table<<<(unsigned)std::min<int64_t>(1024, (tb.lc + 255) / 256), 256, 0, s>>>(tb.sq_c, tb.lc, span_c));
  EMU_CUDA(cudaGetLastError());
  const int64_t gnt = span_t + 1, gnc = span_c + 1;
  if (gnt > kMaxGridCells || gnc > kMaxGridCells || (gnt + 1) * (gnc + 1) > kMaxGridCells) return EMU_OK;
  const int64_t st = gnc + 1, cells = (gnt + 1) * st;
  std::vector<int32_t> B((size_t)cells, 0), S((size_t)cells, 0);
  for (int64_t b = 0; b < tb.nb; b++) {
    const int64_t i = (int64_t)h_tt[b] - tb.tt_lo, j = (int64_t)h_cc[b] - tb.c_lo;
    B[(size_t)((i + 1) * st + (j + 1))] = 1;
    S[(size_t)((i + 1) * st + (j + 1))] = (int32_t)(h_off[b + 1] - h_off[b]);
  }
  for (int64_t i = 1; i <= gnt; i++) {
    int64_t rb = 0, rs = 0;
    const size_t row = (size_t)(i * st), prev = (size_t)((i - 1) * st);
    for (int64_t j = 1; j <= gnc; j++) {
      rb += B[row + j];
      rs += S[row + j];
      B[row + j] = (int32_t)(B[prev + j] + rb);
      S[row + j] = (int32_t)(S[prev + j] + rs);
    }
  }
  // occupancy bitmap + per-word prefix counts + row bases
  const int64_t wpr = (gnc + 31) / 32;
  std::vector<uint32_t> bm((size_t)(gnt * wpr), 0u);
  std::vector<int32_t> wp((size_t)(gnt * wpr), 0), rbase((size_t)gnt + 1, 0);
  for (int64_t b = 0; b < tb.nb; b++) {
    const int64_t i = (int64_t)h_tt[b] - tb.tt_lo, j = (int64_t)h_cc[b] - tb.c_lo;
    bm[(size_t)(i * wpr + j / 32)] |= 1u << (j % 32);
    rbase[(size_t)i + 1] += 1;
  }
  for (int64_t i = 0; i < gnt; i++) {
    rbase[(size_t)i + 1] += rbase[(size_t)i];
    int32_t acc = 0;
    for (int64_t k = 0; k < wpr; k++) {
      wp[(size_t)(i * wpr + k)] = acc;
      acc += __builtin_popcount(bm[(size_t)(i * wpr + k)]);
    }
  }
  // column index: buckets by (conc, tt) (counting sort on conc; tt ascending
  // within a column because buckets are already in (tt, conc) order)
  std::vector<int32_t> cstart((size_t)gnc + 1, 0), ctt((size_t)tb.nb), cb((size_t)tb.nb);
  for (int64_t b = 0; b < tb.nb; b++) cstart[(size_t)(h_cc[b] - tb.c_lo) + 1]++;
  for (int64_t j = 0; j < gnc; j++) cstart[(size_t)j + 1] += cstart[(size_t)j];
  {
    std::vector<int32_t> fill(cstart.begin(), cstart.end() - 1);
    for (int64_t b = 0; b < tb.nb; b++) {
      const int32_t k = fill[(size_t)(h_cc[b] - tb.c_lo)]++;
      ctt[(size_t)k] = h_tt[b];
      cb[(size_t)k] = (int32_t)b;
    }
  }
  EMU_CUDA(table_alloc((void**)&tb.col_start, 4 * (gnc + 1), s));
  EMU_CUDA(table_alloc((void**)&tb.col_tt, 4 * std::max<int64_t>(1, tb.nb), s));
  EMU_CUDA(table_alloc((void**)&tb.col_b, 4 * std::max<int64_t>(1, tb.nb), s));
  EMU_CUDA(cudaMemcpyAsync(tb.col_start, cstart.data(), 4 * (gnc + 1), cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.col_tt, ctt.data(), 4 * tb.nb, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.col_b, cb.data(), 4 * tb.nb, cudaMemcpyHostToDevice, s));
  EMU_CUDA(table_alloc((void**)&tb.bsat, 4 * cells, s));
  EMU_CUDA(table_alloc((void**)&tb.ssat, 4 * cells, s));
  EMU_CUDA(table_alloc((void**)&tb.bmap, 4 * gnt * wpr, s));
  EMU_CUDA(table_alloc((void**)&tb.wpre, 4 * gnt * wpr, s));
  EMU_CUDA(table_alloc((void**)&tb.rowbase, 4 * (gnt + 1), s));
  EMU_CUDA(cudaMemcpyAsync(tb.bsat, B.data(), 4 * cells, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.ssat, S.data(), 4 * cells, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.bmap, bm.data(), 4 * gnt * wpr, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.wpre, wp.data(), 4 * gnt * wpr, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.rowbase, rbase.data(), 4 * (gnt + 1), cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  tb.wpr = (int32_t)wpr;
  tb.gnt = gnt;
  tb.gnc = gnc;
  return EMU_OK;
}

// ---------------------------------------------------------------------------
// The same search index built on the device from the device bucket arrays
// (table build / create path; EMU_INDEX_HOST=1 selects the host version above,
// which the tests use as the cross-check).  Grids are (gnt+1) x (gnc+1) with a
// zero first row and column.
// ---------------------------------------------------------------------------

__global__ void k_idx_fill(const int32_t* __restrict__ btt, const int32_t* __restrict__ bcc,
                           const int64_t* __restrict__ boff, int64_t nb, int32_t tt_lo, int32_t c_lo, int64_t st,
                           int64_t wpr, int32_t* B, int32_t* S, uint32_t* bm) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)btt[b] - tt_lo, j = (int64_t)bcc[b] - c_lo;
    B[(i + 1) * st + (j + 1)] = 1;
    S[(i + 1) * st + (j + 1)] = (int32_t)(boff[b + 1] - boff[b]);
    atomicOr(&bm[i * wpr + j / 32], 1u << (j % 32));
  }
}

// inclusive prefix along each grid row (warp per row), both grids
__global__ void k_idx_rows(int32_t* B, int32_t* S, int64_t rows, int64_t st) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int32_t cb = 0, cs = 0;
    for (int64_t j0 = 1; j0 < st; j0 += 32) {
      const int64_t j = j0 + lane;
      int32_t vb = j < st ? B[r * st + j] : 0, vs = j < st ? S[r * st + j] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t yb = __shfl_up_sync(0xffffffffu, vb, o), ys = __shfl_up_sync(0xffffffffu, vs, o);
        if (lane >= o) {
          vb += yb;
          vs += ys;
        }
      }
      if (j < st) {
        B[r * st + j] = cb + vb;
        S[r * st + j] = cs + vs;
      }
      cb += __shfl_sync(0xffffffffu, vb, 31);
      cs += __shfl_sync(0xffffffffu, vs, 31);
    }
  }
}

// column prefix in three passes: chunk sums, scan of chunk sums, apply
__global__ void k_idx_col_sums(const int32_t* B, const int32_t* S, int64_t rows, int64_t st, int64_t chunk,
                               int32_t* PB, int32_t* PS) {
  const int64_t nch = (rows + chunk - 1) / chunk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nch * st; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ch = t / st, j = t % st;
    int32_t sb = 0, ss = 0;
#pragma unroll 8
    for (int64_t r = ch * chunk; r < rows && r < (ch + 1) * chunk; r++) {
      sb += B[r * st + j];
      ss += S[r * st + j];
    }
    PB[t] = sb;
    PS[t] = ss;
  }
}

__global__ void k_idx_col_scan(int32_t* PB, int32_t* PS, int64_t nch, int64_t st) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < st; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t ab = 0, as = 0;
#pragma unroll 8
    for (int64_t ch = 0; ch < nch; ch++) {  // exclusive
      const int32_t vb = PB[ch * st + j], vs = PS[ch * st + j];
      PB[ch * st + j] = ab;
      PS[ch * st + j] = as;
      ab += vb;
      as += vs;
    }
  }
}

__global__ void k_idx_col_apply(int32_t* B, int32_t* S, int64_t rows, int64_t st, int64_t chunk, const int32_t* PB,
                                const int32_t* PS) {
  const int64_t nch = (rows + chunk - 1) / chunk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nch * st; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ch = t / st, j = t % st;
    int32_t ab = PB[t], as = PS[t];
#pragma unroll 8
    for (int64_t r = ch * chunk; r < rows && r < (ch + 1) * chunk; r++) {
      ab += B[r * st + j];
      as += S[r * st + j];
      B[r * st + j] = ab;
      S[r * st + j] = as;
    }
  }
}

// per grid row: first bucket (lower bound of the row's tt in bucket order) and
// the exclusive popcount prefix of its bitmap words
__global__ void k_idx_bitrows(const int32_t* __restrict__ btt, int64_t nb, int32_t tt_lo, int64_t gnt,
                              const uint32_t* __restrict__ bm, int64_t wpr, int32_t* wp, int32_t* rbase) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= gnt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)tt_lo + i;
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)btt[mid] < v)
        lo = mid + 1;
      else
        hi = mid;
    }
    rbase[i] = (int32_t)lo;
    if (i < gnt) {
      int32_t acc = 0;
      for (int64_t k = 0; k < wpr; k++) {
        wp[i * wpr + k] = acc;
        acc += __popc(bm[i * wpr + k]);
      }
    }
  }
}

// column index: buckets ordered by (conc, tt).  col_start from the SAT's last
// row; a bucket's rank in its column = occupied cells above it in that column
__global__ void k_idx_colstart(const int32_t* B, int64_t gnt, int64_t st, int32_t* cstart) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int32_t* last = B + gnt * st;  // SAT row gnt: column j+1 holds the count of columns <= j
    cstart[0] = 0;
    for (int64_t j = 1; j < st; j++) cstart[j] = last[j];
  }
}

__global__ void k_idx_cols(const int32_t* __restrict__ btt, const int32_t* __restrict__ bcc, int64_t nb, int32_t tt_lo,
                           int32_t c_lo, int64_t st, const int32_t* B, const int32_t* cstart, int32_t* ctt, int32_t* cb) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)btt[b] - tt_lo, j = (int64_t)bcc[b] - c_lo;
    // rows 0..i-1 of column j: SAT(i, j+1) - SAT(i, j)
    const int64_t k = cstart[j] + (B[i * st + j + 1] - B[i * st + j]);
    ctt[k] = btt[b];
    cb[k] = (int32_t)b;
  }
}

int build_search_index_dev(TableBuf& tb, cudaStream_t s) {
  if (tb.nb == 0) return EMU_OK;
  const int64_t span_t = (int64_t)tb.tt_hi - tb.tt_lo, span_c = (int64_t)tb.c_hi - tb.c_lo;
  tb.lt = std::min<int64_t>(span_t + 1, kMaxSqTable);
  tb.lc = std::min<int64_t>(span_c + 1, kMaxSqTable);
  EMU_CUDA(table_alloc((void**)&tb.sq_t, 8 * tb.lt, s));
  EMU_CUDA(table_alloc((void**)&tb.sq_c, 8 * tb.lc, s));
  EMU_LAUNCH("index", s, k_sq_table<<<(unsigned)std::min<int64_t>(1024, (tb.lt + 255) / 256), 256, 0, s>>>(tb.sq_t, tb.lt, span_t));
  EMU_LAUNCH("index", s, k_sq_table<<<(unsigned)std::min<int64_t>(1024, (tb.lc + 255) / 256), 256, 0, s>>>(tb.sq_c, tb.lc, span_c));
  EMU_CUDA(cudaGetLastError());
  const int64_t gnt = span_t + 1, gnc = span_c + 1;
  if (gnt > kMaxGridCells || gnc > kMaxGridCells || (gnt + 1) * (gnc + 1) > kMaxGridCells) {
    EMU_CUDA(cudaStreamSynchronize(s));
    return EMU_OK;
  }
  const int64_t st = gnc + 1, rows = gnt + 1, cells = rows * st, wpr = (gnc + 31) / 32;
  // column scan in chunks of rows: short per-thread chains, at most 512 chunks
  const int64_t chunk = std::max<int64_t>(16, (rows + 511) / 512), nch = (rows + chunk - 1) / chunk;
  EMU_CUDA(table_alloc((void**)&tb.bsat, 4 * cells, s));
  EMU_CUDA(table_alloc((void**)&tb.ssat, 4 * cells, s));
  EMU_CUDA(table_alloc((void**)&tb.bmap, 4 * gnt * wpr, s));
  EMU_CUDA(table_alloc((void**)&tb.wpre, 4 * gnt * wpr, s));
  EMU_CUDA(table_alloc((void**)&tb.rowbase, 4 * (gnt + 1), s));
  EMU_CUDA(table_alloc((void**)&tb.col_start, 4 * (gnc + 1), s));
  EMU_CUDA(table_alloc((void**)&tb.col_tt, 4 * std::max<int64_t>(1, tb.nb), s));
  EMU_CUDA(table_alloc((void**)&tb.col_b, 4 * std::max<int64_t>(1, tb.nb), s));
  int32_t* part = nullptr;
  EMU_CUDA(cudaMallocAsync((void**)&part, 8 * (size_t)nch * st, s));
  EMU_CUDA(cudaMemsetAsync(tb.bsat, 0, 4 * cells, s));
  EMU_CUDA(cudaMemsetAsync(tb.ssat, 0, 4 * cells, s));
  EMU_CUDA(cudaMemsetAsync(tb.bmap, 0, 4 * gnt * wpr, s));
  const auto g = [](int64_t n, int t) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, kNumSMs * 8)); };
  EMU_LAUNCH("index", s, k_idx_fill<<<g(tb.nb, 256), 256, 0, s>>>(tb.bkt_tt, tb.bkt_conc, tb.bkt_off, tb.nb, tb.tt_lo,
                                                                   tb.c_lo, st, wpr, tb.bsat, tb.ssat, tb.bmap));
  EMU_LAUNCH("index", s, k_idx_rows<<<g(rows * 32, 256), 256, 0, s>>>(tb.bsat, tb.ssat, rows, st));
  EMU_LAUNCH("index", s, k_idx_col_sums<<<g(nch * st, 256), 256, 0, s>>>(tb.bsat, tb.ssat, rows, st, chunk, part,
                                                                          part + nch * st));
  EMU_LAUNCH("index", s, k_idx_col_scan<<<g(st, 128), 128, 0, s>>>(part, part + nch * st, nch, st));
  EMU_LAUNCH("index", s, k_idx_col_apply<<<g(nch * st, 256), 256, 0, s>>>(tb.bsat, tb.ssat, rows, st, chunk, part,
                                                                           part + nch * st));
  EMU_LAUNCH("index", s, k_idx_bitrows<<<g(gnt + 1, 256), 256, 0, s>>>(tb.bkt_tt, tb.nb, tb.tt_lo, gnt, tb.bmap, wpr,
                                                                       tb.wpre, tb.rowbase));
  EMU_LAUNCH("index", s, k_idx_colstart<<<1, 32, 0, s>>>(tb.bsat, gnt, st, tb.col_start));
  EMU_LAUNCH("index", s, k_idx_cols<<<g(tb.nb, 256), 256, 0, s>>>(tb.bkt_tt, tb.bkt_conc, tb.nb, tb.tt_lo, tb.c_lo, st,
                                                                   tb.bsat, tb.col_start, tb.col_tt, tb.col_b));
  EMU_CUDA(cudaGetLastError());
  EMU_CUDA(cudaFreeAsync(part, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  tb.wpr = (int32_t)wpr;
  tb.gnt = gnt;
  tb.gnc = gnc;
  return EMU_OK;
}

bool index_on_host() {
  const char* v = getenv("EMU_INDEX_HOST");
  return v && v[0] == '1';
}

template <typename T>
static int dev_alloc(T** p, int64_t n) {
  *p = nullptr;
  EMU_CUDA(table_alloc((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1), 0));
  return EMU_OK;
}

// Host-side copy of a (host or device) array.
template <typename T>
static int to_host(std::vector<T>& out, const T* src, int64_t n, cudaStream_t s) {
  out.resize((size_t)(n > 0 ? n : 0));
  if (n > 0) {
    EMU_CUDA(cudaMemcpyAsync(out.data(), src, sizeof(T) * (size_t)n, cudaMemcpyDefault, s));
    EMU_CUDA(cudaStreamSynchronize(s));
  }
  return EMU_OK;
}

// Upload one table and derive its row index + ranges.  Host-resident copies
// of keys/offsets are kept for validation (ProfilePack.validate,
// profile.py:178-194); this is construction, not the per-query path.
static int upload_table(const emu_table_view* v, const char* name, cudaStream_t s, TableBuf& tb) {
  tb = TableBuf();
  if (!v) return fail(EMU_ERR_INVALID, std::string(name) + " table view is NULL");
  int64_t nb = v->n_buckets, ns = v->n_samples;
  if (nb < 0 || ns < 0) return fail(EMU_ERR_INVALID, std::string(name) + " table has negative sizes");
  std::vector<int32_t> tt, cc;
  std::vector<int64_t> off;
  std::vector<double> smp;
  int rc;
  if ((rc = to_host(tt, v->bkt_tt, nb, s))) return rc;
  if ((rc = to_host(cc, v->bkt_conc, nb, s))) return rc;
  if ((rc = to_host(off, v->bkt_off, nb + 1, s))) return rc;
  if ((rc = to_host(smp, v->samples, ns, s))) return rc;
  if (nb == 0 && ns != 0) return fail(EMU_ERR_INVALID, std::string(name) + " table has samples but no buckets");
  if (off.empty() || off[0] != 0 || off[nb] != ns)
    return fail(EMU_ERR_INVALID, std::string(name) + " table offsets do not span its samples");
  if (ns >= (1LL << 31)) return fail(EMU_ERR_INVALID, std::string(name) + " table holds >= 2^31 samples");
  std::vector<int32_t> row_tt;
  std::vector<int64_t> row_start;
  for (int64_t i = 0; i < nb; i++) {
    if (tt[i] < 1 || cc[i] < 1)
      return fail(EMU_ERR_INVALID, std::string("bucket key (") + std::to_string(tt[i]) + ", " +
                                       std::to_string(cc[i]) + ") must be positive");
    if (off[i + 1] <= off[i])
      return fail(EMU_ERR_INVALID, std::string("bucket (") + std::to_string(tt[i]) + ", " +
                                       std::to_string(cc[i]) + ") has no samples");
    if (i > 0) {
      bool ordered = tt[i] > tt[i - 1] || (tt[i] == tt[i - 1] && cc[i] > cc[i - 1]);
      if (!ordered) {
        if (tt[i] == tt[i - 1] && cc[i] == cc[i - 1])
          return fail(EMU_ERR_INVALID, std::string(name) + " table has duplicate bucket (" +
                                           std::to_string(tt[i]) + ", " + std::to_string(cc[i]) + ")");
        return fail(EMU_ERR_INVALID, std::string(name) + " table buckets are not sorted by (tt, conc)");
      }
    }
    if (i == 0 || tt[i] != tt[i - 1]) {
      row_tt.push_back(tt[i]);
      row_start.push_back(i);
    }
  }
  row_start.push_back(nb);
  for (int64_t i = 0; i < ns; i++)
    if (!(smp[i] > 0.0)) return fail(EMU_ERR_INVALID, std::string(name) + " table has a nonpositive sample");
  tb.nb = nb;
  tb.ns = ns;
  tb.nrows = (int64_t)row_tt.size();
  if (nb > 0) {
    tb.tt_lo = tt[0];
    tb.tt_hi = tt[nb - 1];
    tb.c_lo = *std::min_element(cc.begin(), cc.end());
    tb.c_hi = *std::max_element(cc.begin(), cc.end());
  }
  if ((rc = dev_alloc(&tb.bkt_tt, nb)) || (rc = dev_alloc(&tb.bkt_conc, nb)) || (rc = dev_alloc(&tb.bkt_off, nb + 1)) ||
      (rc = dev_alloc(&tb.samples, ns)) || (rc = dev_alloc(&tb.row_tt, tb.nrows)) ||
      (rc = dev_alloc(&tb.row_start, tb.nrows + 1))) {
    tb.release();
    return rc;
  }
  EMU_CUDA(cudaMemcpyAsync(tb.bkt_tt, tt.data(), 4 * nb, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.bkt_conc, cc.data(), 4 * nb, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.bkt_off, off.data(), 8 * (nb + 1), cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.samples, smp.data(), 8 * ns, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.row_tt, row_tt.data(), 4 * tb.nrows, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaMemcpyAsync(tb.row_start, row_start.data(), 8 * (tb.nrows + 1), cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  return index_on_host() ? build_search_index(tb, tt.data(), cc.data(), off.data(), s) : build_search_index_dev(tb, s);
}

}  // namespace emu

using namespace emu;

extern "C" {

const char* emu_last_error(void) { return g_last_error.c_str(); }
int emu_version(void) { return 1; }

int emu_tables_create(const emu_table_view* decode, const emu_table_view* mixed, const emu_table_view* combined,
                      void* stream, emu_tables_t* out) {
  if (!out) return fail(EMU_ERR_INVALID, "out is NULL");
  *out = nullptr;
  cudaStream_t s = as_stream(stream);
  auto* t = new emu_tables_s();
  const emu_table_view* v[3] = {decode, mixed, combined};
  const char* names[3] = {"decode", "mixed", "combined"};
  for (int i = 0; i < 3; i++) {
    int rc = upload_table(v[i], names[i], s, t->tab[i]);
    if (rc) {
      for (int j = 0; j < 3; j++) t->tab[j].release();
      delete t;
      return rc;
    }
  }
  if (t->tab[2].ns != t->tab[0].ns + t->tab[1].ns) {
    std::string m = "combined table inconsistent: " + std::to_string(t->tab[2].ns) + " samples != decode+mixed " +
                    std::to_string(t->tab[0].ns + t->tab[1].ns);
    for (int j = 0; j < 3; j++) t->tab[j].release();
    delete t;
    return fail(EMU_ERR_INVALID, m);
  }
  *out = t;
  return EMU_OK;
}

int emu_tables_info(emu_tables_t t, int table_id, emu_table_info* out) {
  if (!t || !out || table_id < 0 || table_id > 2) return fail(EMU_ERR_INVALID, "bad emu_tables_info arguments");
  const TableBuf& b = t->tab[table_id];
  out->n_buckets = b.nb;
  out->n_samples = b.ns;
  out->tt_lo = b.tt_lo;
  out->tt_hi = b.tt_hi;
  out->conc_lo = b.c_lo;
  out->conc_hi = b.c_hi;
  return EMU_OK;
}

int emu_tables_device(emu_tables_t t, int table_id, emu_table_dev* out) {
  if (!t || !out || table_id < 0 || table_id > 2) return fail(EMU_ERR_INVALID, "bad emu_tables_device arguments");
  const TableBuf& b = t->tab[table_id];
  out->n_buckets = b.nb;
  out->n_samples = b.ns;
  out->n_rows = b.nrows;
  out->bkt_tt = b.bkt_tt;
  out->bkt_conc = b.bkt_conc;
  out->bkt_off = b.bkt_off;
  out->samples = b.samples;
  out->row_tt = b.row_tt;
  out->row_start = b.row_start;
  return EMU_OK;
}

void emu_tables_destroy(emu_tables_t t) {
  if (!t) return;
  for (int i = 0; i < 3; i++) t->tab[i].release();
  delete t;
}

}  // extern "C"
