// tables.h -- host-side table handle shared by the library's translation units.
#pragma once
#include "emu_internal.cuh"

namespace emu {

struct TableBuf {
  int32_t* bkt_tt = nullptr;
  int32_t* bkt_conc = nullptr;
  int64_t* bkt_off = nullptr;
  double* samples = nullptr;
  int32_t* row_tt = nullptr;
  int64_t* row_start = nullptr;
  int64_t nb = 0, ns = 0, nrows = 0;
  int32_t tt_lo = 0, tt_hi = 0, c_lo = 0, c_hi = 0;
  int32_t* bsat = nullptr;
  int32_t* ssat = nullptr;
  int64_t gnt = 0, gnc = 0;
  uint32_t* bmap = nullptr;
  int32_t* wpre = nullptr;
  int32_t* rowbase = nullptr;
  int32_t wpr = 0;
  int32_t* col_start = nullptr;  // [gnc+1]: buckets of conc index j are col_*[col_start[j] .. col_start[j+1])
  int32_t* col_tt = nullptr;     // [nb] tt of those buckets, ascending
  int32_t* col_b = nullptr;      // [nb] their bucket index
  double* sq_t = nullptr;
  double* sq_c = nullptr;
  int64_t lt = 0, lc = 0;
  void release();
  DevTable view() const;
};

// Every TableBuf array is allocated here (stream-ordered pool) and freed by release().
cudaError_t table_alloc(void** p, size_t bytes, cudaStream_t s);

// Build the search index (summed-area tables + squared-delta tables) from
// host copies of the bucket keys/offsets (construction time, not per query).
int build_search_index(TableBuf& tb, const int32_t* h_tt, const int32_t* h_cc, const int64_t* h_off, cudaStream_t s);
// The same index built on the device from tb's device bucket arrays (default);
// index_on_host() (EMU_INDEX_HOST=1) selects the host version instead.
int build_search_index_dev(TableBuf& tb, cudaStream_t s);
bool index_on_host();

}  // namespace emu

struct emu_tables_s {
  emu::TableBuf tab[3];  // decode, mixed, combined
};
