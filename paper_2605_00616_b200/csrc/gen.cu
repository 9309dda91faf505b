// gen.cu -- batched capture stand-ins on the device.
//
//   k_ground_truth : ground_truth_latency (engine.py:128-147) for a batch of
//                    step keys: m * (base + per_token*tt + per_seq*conc) *
//                    (1 + g), g ~ N(0, cv) redrawn while the factor is
//                    nonpositive, m = prefill_multiplier for mixed steps.
//                    The deterministic part is the reference's expression in
//                    its evaluation order with IEEE rn ops (bit-identical);
//                    the deviates come from Box-Muller on Philox4x32-10 keyed
//                    by (seed, record index), not CPython's random.gauss
//                    stream (CPython parity is not required).
//   k_gen_keys     : step keys of the synthetic generator G:
//                    lognormal concurrency, a decode fraction, lognormal
//                    prefill chunks -- so 100M-record builds (config 4) start
//                    from device-resident records instead of a host sampler.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "emu_internal.cuh"
#include "prof.h"

namespace emu {

// Two standard normal deviates from one Philox block (Box-Muller).
__device__ __forceinline__ double2 philox_normal2(uint64_t idx, uint32_t round, uint2 key) {
  const uint4 r = philox4x32_10(make_uint4((uint32_t)idx, (uint32_t)(idx >> 32), round, 0x6e6f726du), key);
  // u1 in (0, 1], u2 in [0, 1): 53-bit uniforms
  const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
  const double u2 = (double)((((uint64_t)r.z << 32) | r.w) >> 11) * (1.0 / 9007199254740992.0);
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(rad * c, rad * s);
}

__global__ void k_ground_truth(const int32_t* __restrict__ tt, const int32_t* __restrict__ conc,
                               const uint8_t* __restrict__ phase, int64_t n, double base, double per_token,
                               double per_seq, double prefill_mult, double cv, uint2 key, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double mult = phase[i] ? prefill_mult : 1.0;
    // mult * (base + per_token * tt + per_seq * conc), Python's left-to-right order
    const double lat = __dmul_rn(mult, __dadd_rn(__dadd_rn(base, __dmul_rn(per_token, (double)tt[i])),
                                                 __dmul_rn(per_seq, (double)conc[i])));
    if (cv == 0.0) {  // no randomness consumed (engine.py:141-142)
      out[i] = lat;
      continue;
    }
    double factor = 0.0;
    for (uint32_t round = 0;; round++) {
      const double2 z = philox_normal2((uint64_t)i, round, key);
      factor = __dadd_rn(1.0, __dmul_rn(cv, z.x));
      if (factor > 0.0) break;
      factor = __dadd_rn(1.0, __dmul_rn(cv, z.y));
      if (factor > 0.0) break;
    }
    out[i] = __dmul_rn(lat, factor);
  }
}

__global__ void k_gen_keys(int64_t n, uint2 key, double conc_mu, double conc_sigma, int32_t conc_max, double p_decode,
                           double chunk_mu, double chunk_sigma, int32_t tt_max, int32_t* __restrict__ tt,
                           int32_t* __restrict__ conc, uint8_t* __restrict__ phase) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 z = philox_normal2((uint64_t)i, 0x4b455953u, key);
    const uint4 r = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0x64656364u, 1u), key);
    const double u = (double)((((uint64_t)r.x << 32) | r.y) >> 11) * (1.0 / 9007199254740992.0);
    double c = rint(exp(conc_mu + conc_sigma * z.x));
    c = fmin(fmax(c, 1.0), (double)conc_max);
    const int32_t ci = (int32_t)c;
    const bool decode = u < p_decode;
    int32_t t = ci;
    if (!decode) {
      double ch = rint(exp(chunk_mu + chunk_sigma * z.y));
      ch = fmin(fmax(ch, 1.0), (double)tt_max);
      t = (int32_t)min((int64_t)tt_max, (int64_t)ci - 1 + (int64_t)ch);
    }
    tt[i] = t;
    conc[i] = ci;
    phase[i] = decode ? 0 : 1;
  }
}

}  // namespace emu

using namespace emu;

extern "C" {

int emu_ground_truth(const int32_t* tt, const int32_t* conc, const uint8_t* phase, int64_t n, double base_s,
                     double per_token_s, double per_seq_s, double prefill_multiplier, double noise_cv, uint64_t seed,
                     double* out_lat, void* stream) {
  if (n < 0) return fail(EMU_ERR_INVALID, "negative record count");
  if (!(base_s > 0)) return fail(EMU_ERR_INVALID, "base_s must be > 0, got " + std::to_string(base_s));
  if (per_token_s < 0 || per_seq_s < 0) return fail(EMU_ERR_INVALID, "per_token_s and per_seq_s must be >= 0");
  if (prefill_multiplier < 1.0)
    return fail(EMU_ERR_INVALID, "prefill_multiplier must be >= 1, got " + std::to_string(prefill_multiplier));
  if (noise_cv < 0) return fail(EMU_ERR_INVALID, "noise_cv must be >= 0, got " + std::to_string(noise_cv));
  if (n == 0) return EMU_OK;
  if (!tt || !conc || !phase || !out_lat) return fail(EMU_ERR_INVALID, "NULL column");
  cudaStream_t s = as_stream(stream);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
  EMU_LAUNCH("ground_truth", s, k_ground_truth<<<grid, 256, 0, s>>>(tt, conc, phase, n, base_s, per_token_s, per_seq_s,
                                                                    prefill_multiplier, noise_cv,
                                                                    make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)),
                                                                    out_lat));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

int emu_gen_step_keys(int64_t n, uint64_t seed, double conc_mu, double conc_sigma, int32_t conc_max, double p_decode,
                      double chunk_mu, double chunk_sigma, int32_t tt_max, int32_t* tt, int32_t* conc, uint8_t* phase,
                      void* stream) {
  if (n < 0) return fail(EMU_ERR_INVALID, "negative key count");
  if (conc_max < 1 || tt_max < conc_max) return fail(EMU_ERR_INVALID, "need 1 <= conc_max <= tt_max");
  if (n == 0) return EMU_OK;
  if (!tt || !conc || !phase) return fail(EMU_ERR_INVALID, "NULL output column");
  cudaStream_t s = as_stream(stream);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 16);
  EMU_LAUNCH("gen_keys", s, k_gen_keys<<<grid, 256, 0, s>>>(n, make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)),
                                                            conc_mu, conc_sigma, conc_max, p_decode, chunk_mu,
                                                            chunk_sigma, tt_max, tt, conc, phase));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

}  // extern "C"
