// misc.cu -- normalized_distance over arrays and the synthetic token fill.
#include <cuda_runtime.h>

#include "emu_internal.cuh"
#include "prof.h"

namespace emu {

__global__ void k_distance(const int32_t* __restrict__ qt, const int32_t* __restrict__ qc,
                           const int32_t* __restrict__ bt, const int32_t* __restrict__ bc, int64_t n, int64_t tt_lo,
                           int64_t tt_hi, int64_t c_lo, int64_t c_hi, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = norm_dist((int64_t)qt[i] - bt[i], (int64_t)qc[i] - bc[i], tt_hi - tt_lo, c_hi - c_lo);
}

// Token part of EmulatorEngine._apply_outcome (engine.py:464-483): a prefill
// entry emits only when its chunk completes the prompt, a decode entry always
// emits; the emitted token's id is the request's generated count before the
// step (token k of request r has id k, engine.py:472-477).  Four entries per
// thread with 128-bit loads/stores when aligned.
__device__ __forceinline__ void fill_one(uint8_t pre, int32_t ch, int32_t prog, int32_t plen, int32_t gen, int32_t tgt,
                                         int32_t& id, uint8_t& fin) {
  const bool emit = !pre || (prog + ch == plen);
  id = emit ? gen : -1;
  fin = (uint8_t)(emit && gen + 1 >= tgt);
}

__global__ void k_token_fill(const uint8_t* __restrict__ pre, const int32_t* __restrict__ ch,
                             const int32_t* __restrict__ prog, const int32_t* __restrict__ plen,
                             const int32_t* __restrict__ gen, const int32_t* __restrict__ tgt, int64_t n,
                             int32_t* __restrict__ ids, uint8_t* __restrict__ fin) {
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n4; v += stride) {
    const uchar4 p = reinterpret_cast<const uchar4*>(pre)[v];
    const int4 c = reinterpret_cast<const int4*>(ch)[v];
    const int4 g = reinterpret_cast<const int4*>(prog)[v];
    const int4 l = reinterpret_cast<const int4*>(plen)[v];
    const int4 e = reinterpret_cast<const int4*>(gen)[v];
    const int4 t = reinterpret_cast<const int4*>(tgt)[v];
    int4 o;
    uchar4 f;
    fill_one(p.x, c.x, g.x, l.x, e.x, t.x, o.x, f.x);
    fill_one(p.y, c.y, g.y, l.y, e.y, t.y, o.y, f.y);
    fill_one(p.z, c.z, g.z, l.z, e.z, t.z, o.z, f.z);
    fill_one(p.w, c.w, g.w, l.w, e.w, t.w, o.w, f.w);
    reinterpret_cast<int4*>(ids)[v] = o;
    reinterpret_cast<uchar4*>(fin)[v] = f;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    fill_one(pre[i], ch[i], prog[i], plen[i], gen[i], tgt[i], ids[i], fin[i]);
}

__global__ void k_token_fill_scalar(const uint8_t* __restrict__ pre, const int32_t* __restrict__ ch,
                                    const int32_t* __restrict__ prog, const int32_t* __restrict__ plen,
                                    const int32_t* __restrict__ gen, const int32_t* __restrict__ tgt, int64_t n,
                                    int32_t* __restrict__ ids, uint8_t* __restrict__ fin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    fill_one(pre[i], ch[i], prog[i], plen[i], gen[i], tgt[i], ids[i], fin[i]);
}

static int grid_n(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > kNumSMs * 16) b = kNumSMs * 16;
  return (int)b;
}

}  // namespace emu

using namespace emu;

extern "C" {

int emu_distance(const int32_t* q_tt, const int32_t* q_conc, const int32_t* b_tt, const int32_t* b_conc, int64_t n,
                 int32_t tt_lo, int32_t tt_hi, int32_t conc_lo, int32_t conc_hi, double* out, void* stream) {
  if (n < 0) return fail(EMU_ERR_INVALID, "negative length");
  if (n == 0) return EMU_OK;
  EMU_LAUNCH("distance", as_stream(stream), k_distance<<<grid_n(n, 256), 256, 0, as_stream(stream)>>>(q_tt, q_conc, b_tt, b_conc, n, tt_lo, tt_hi, conc_lo, conc_hi,
                                                           out));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

int emu_token_fill(const uint8_t* is_prefill, const int32_t* chunk, const int32_t* prefill_progress,
                   const int32_t* prompt_len, const int32_t* generated, const int32_t* target_len, int64_t n,
                   int32_t* out_ids, uint8_t* out_finished, void* stream) {
  if (n < 0) return fail(EMU_ERR_INVALID, "negative length");
  if (n == 0) return EMU_OK;
  auto al = [](const void* p, int a) { return ((uintptr_t)p % a) == 0; };
  const bool vec = al(is_prefill, 4) && al(chunk, 16) && al(prefill_progress, 16) && al(prompt_len, 16) &&
                   al(generated, 16) && al(target_len, 16) && al(out_ids, 16) && al(out_finished, 4);
  cudaStream_t s = as_stream(stream);
  if (vec)
    EMU_LAUNCH("token_fill", s, k_token_fill<<<grid_n((n + 3) / 4, 256), 256, 0, s>>>(is_prefill, chunk, prefill_progress, prompt_len, generated,
                                                         target_len, n, out_ids, out_finished));
  else
    EMU_LAUNCH("token_fill", s, k_token_fill_scalar<<<grid_n(n, 256), 256, 0, s>>>(is_prefill, chunk, prefill_progress, prompt_len, generated,
                                                      target_len, n, out_ids, out_finished));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

}  // extern "C"
