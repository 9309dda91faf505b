// prof.h -- launch counting + optional per-kernel CUDA-event timing.
#pragma once
#include <cuda_runtime.h>

namespace emu {
void prof_count();
bool prof_on();
void prof_begin(cudaStream_t s, cudaEvent_t* a);
void prof_end(const char* name, cudaStream_t s, cudaEvent_t a);
}  // namespace emu

// EMU_LAUNCH(name, stream, kernel<<<...>>>(...)) -- counts and (optionally) times one launch.
#define EMU_LAUNCH(name, stream, ...)             \
  do {                                            \
    ::emu::prof_count();                          \
    cudaEvent_t _emu_ev = nullptr;                \
    if (::emu::prof_on()) ::emu::prof_begin((stream), &_emu_ev); \
    __VA_ARGS__;                                  \
    if (_emu_ev) ::emu::prof_end((name), (stream), _emu_ev); \
  } while (0)
