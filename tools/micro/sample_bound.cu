// Micro-benchmark: what bounds k_sample?  Streams 21 B/query in, 12 B/query
// out, plus D dependent random 8-byte loads from an L2-resident table.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sb sample_bound.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int D, bool HINT>
__global__ void k(const int32_t* __restrict__ qt, const int32_t* __restrict__ qc, const uint8_t* __restrict__ qp,
                  const uint64_t* __restrict__ us, const uint32_t* __restrict__ ui, const uint64_t* __restrict__ tab,
                  uint64_t mask, int64_t Q, double* __restrict__ ol, int32_t* __restrict__ os) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Q; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t t, c; uint8_t p; uint64_t u; uint32_t w;
    if (HINT) { t = __ldcs(qt + i); c = __ldcs(qc + i); p = __ldcs(qp + i); u = __ldcs(us + i); w = __ldcs(ui + i); }
    else { t = qt[i]; c = qc[i]; p = qp[i]; u = us[i]; w = ui[i]; }
    uint64_t h = ((uint64_t)t * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)c << 17) ^ p;
#pragma unroll
    for (int d = 0; d < D; d++) h = tab[(h ^ (h >> 29)) & mask] + h;
    const double lat = (double)(h ^ u);
    if (HINT) { __stcs(ol + i, lat); __stcs(os + i, (int32_t)(w ^ (uint32_t)h)); }
    else { ol[i] = lat; os[i] = (int32_t)(w ^ (uint32_t)h); }
  }
}

template <int D, bool H>
float run(int grid, int block, int64_t Q, void** b, uint64_t* tab, uint64_t mask) {
  cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
  for (int r = 0; r < 3; r++) k<D, H><<<grid, block>>>((int32_t*)b[0], (int32_t*)b[1], (uint8_t*)b[2], (uint64_t*)b[3], (uint32_t*)b[4], tab, mask, Q, (double*)b[5], (int32_t*)b[6]);
  cudaEventRecord(a);
  for (int r = 0; r < 10; r++) k<D, H><<<grid, block>>>((int32_t*)b[0], (int32_t*)b[1], (uint8_t*)b[2], (uint64_t*)b[3], (uint32_t*)b[4], tab, mask, Q, (double*)b[5], (int32_t*)b[6]);
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, a, e); return ms / 10;
}

int main() {
  const int64_t Q = 10000000;
  void* b[7];
  size_t sz[7] = {4, 4, 1, 8, 4, 8, 4};
  for (int i = 0; i < 7; i++) { cudaMalloc(&b[i], sz[i] * Q); cudaMemset(b[i], i, sz[i] * Q); }
  const uint64_t n = 1 << 23;  // 64 MB table (L2-resident)
  uint64_t* tab; cudaMalloc(&tab, 8 * n); cudaMemset(tab, 1, 8 * n);
  const double bytes = 33.0 * Q;
  int grids[3] = {148 * 8, 148 * 16, 148 * 64};
  for (int g : grids) {
    float t0 = run<0, true>(g, 256, Q, b, tab, n - 1), t0n = run<0, false>(g, 256, Q, b, tab, n - 1);
    float t1 = run<1, true>(g, 256, Q, b, tab, n - 1), t2 = run<2, true>(g, 256, Q, b, tab, n - 1);
    float t4 = run<4, true>(g, 256, Q, b, tab, n - 1), t6 = run<6, true>(g, 256, Q, b, tab, n - 1);
    printf("grid %6d  D0 %.4f ms (%.0f GB/s)  D0-nohint %.4f  D1 %.4f  D2 %.4f  D4 %.4f  D6 %.4f\n", g, t0, bytes / t0 / 1e6, t0n, t1, t2, t4, t6);
  }
  return 0;
}
