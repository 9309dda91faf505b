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
  void release();
  DevTable view() const;
};

}  // namespace emu

struct emu_tables_s {
  emu::TableBuf tab[3];  // decode, mixed, combined
};
