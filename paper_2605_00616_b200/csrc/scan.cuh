// scan.cuh -- device-wide exclusive scan (reduce-then-scan, 3 kernels).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "prof.h"

namespace emu {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T& total, T* sm /* >= 33 */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[w] = x;
  __syncthreads();
  if (w == 0) {
    T s = lane < nw ? sm[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sm[lane] = s;
  }
  __syncthreads();
  T base = w ? sm[w - 1] : T(0);
  total = sm[nw - 1];
  __syncthreads();
  return base + x - v;
}

// in(i) is a functor giving element i (i < n).
template <typename T, typename In>
__global__ void k_scan_reduce(In in, int64_t n, T* partial) {
  __shared__ T sm[33];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  T acc = 0;
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + (int64_t)k * kScanThreads + threadIdx.x;
    if (i < n) acc += in(i);
  }
  T tot;
  block_excl_scan<T>(acc, tot, sm);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename T>
__global__ void k_scan_partials(T* partial, int64_t nb, T* total_out) {
  __shared__ T sm[33];
  T carry = 0;
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    T v = i < nb ? partial[i] : T(0);
    T tot;
    T ex = block_excl_scan<T>(v, tot, sm);
    if (i < nb) partial[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

// out(i, excl) receives each element's exclusive prefix.  Warp w of a tile
// owns 512 consecutive elements, read and emitted in 16 coalesced rounds of 32
// (loads and the out() stores stay coalesced); one block scan combines the
// warp totals.
template <typename T, typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(In in, Out out, int64_t n, const T* partial) {
  __shared__ T wsum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t wbase = (int64_t)blockIdx.x * kScanTile + (int64_t)w * (32 * kScanItems);
  T v[kScanItems];
  T acc = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    const int64_t i = wbase + k * 32 + lane;
    v[k] = i < n ? in(i) : T(0);
    acc += v[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) wsum[w] = acc;
  __syncthreads();
  T carry = partial[blockIdx.x];
  for (int q = 0; q < w; q++) carry += wsum[q];
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    T x = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const int64_t i = wbase + k * 32 + lane;
    if (i < n) out(i, carry + x - v[k]);
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
}

// Exclusive scan of in(0..n) into out(i, excl); *total_dev receives the sum.
// partial must hold ceil(n / kScanTile) elements.
template <typename T, typename In, typename Out>
cudaError_t device_excl_scan(In in, Out out, int64_t n, T* partial, T* total_dev, cudaStream_t s) {
  int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb < 1) nb = 1;
  EMU_LAUNCH("scan", s, k_scan_reduce<T, In><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, partial));
  EMU_LAUNCH("scan", s, k_scan_partials<T><<<1, 1024, 0, s>>>(partial, nb, total_dev));
  EMU_LAUNCH("scan", s, k_scan_down<T, In, Out><<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, partial));
  return cudaGetLastError();
}

}  // namespace emu
