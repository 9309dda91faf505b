/*
 * emu_abi.h -- C ABI of the B200 density-aware profile oracle (libemu_b200.so).
 *
 * This is the drop-in boundary for the hot path of LLM-Emu's `serve_emu`
 * package (reference: /root/reference/pkg/src/serve_emu).  Every entry point
 * takes plain pointers, sizes and a `void* stream` (a cudaStream_t; NULL means
 * the legacy default stream).  No torch or C++ types cross the boundary.
 *
 * Pointer residency: unless stated otherwise, array arguments may be host or
 * device pointers (the library copies with cudaMemcpyDefault); arrays marked
 * [dev] must be device pointers.  Output arrays marked [dev|host] may be either.
 *
 * Status codes (returned by every int function, mirrored to Python exceptions):
 *   EMU_OK             0
 *   EMU_ERR_NO_DATA    1  -> NoProfileDataError  (oracle.py:23-24, :138-144, :205-209)
 *   EMU_ERR_INVALID    2  -> ValueError / PackValidationError (oracle.py:33-35, :53-59,
 *                                                               profile.py:248-250)
 *   EMU_ERR_CUDA       3  -> RuntimeError (any CUDA failure; message from emu_last_error)
 *   EMU_ERR_CAPACITY   4  -> internal: pool arena / key map full; caller flushes and retries
 *   EMU_ERR_UNSUPPORTED 5 -> internal: a document outside the native codec's subset; the
 *                            Python mirror re-reads it with the reference's json path
 * emu_last_error() returns a thread-local, NUL-terminated message for the last
 * non-zero status on the calling thread.
 *
 * Phase encoding everywhere: 0 = StepPhase.DECODE_ONLY ("decode"),
 *                            1 = StepPhase.PREFILL_OR_MIXED ("mixed")
 *   (profile.py:20-25).  Table ids: 0 = decode, 1 = mixed, 2 = combined
 *   (TableKind, profile.py:28-32).
 */
#ifndef EMU_ABI_H
#define EMU_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMU_OK 0
#define EMU_ERR_NO_DATA 1
#define EMU_ERR_INVALID 2
#define EMU_ERR_CUDA 3
#define EMU_ERR_CAPACITY 4
#define EMU_ERR_UNSUPPORTED 5

/* RNG modes for emu_oracle_sample. */
#define EMU_RNG_EXPLICIT 0 /* caller supplies u_sel[Q] (u64) and u_idx[Q] (u32)           */
#define EMU_RNG_PHILOX 1   /* on-device Philox4x32-10 keyed by (seed, ctr_base + i)         */

typedef struct emu_tables_s* emu_tables_t;
typedef struct emu_oracle_s* emu_oracle_t;
typedef struct emu_pack_parsed_s* emu_pack_parsed_t;
typedef struct emu_sched_s* emu_sched_t;

/* One phase table in canonical SoA form: buckets sorted by (tt, conc),
 * bkt_off[n_buckets+1] are offsets into samples[n_samples] (bucket b owns
 * samples[bkt_off[b] .. bkt_off[b+1])), in the pack's own sample order.
 * Mirrors PhaseTable / _TableIndex (profile.py:113-129, oracle.py:168-178). */
typedef struct emu_table_view {
  int64_t n_buckets;
  int64_t n_samples;
  const int32_t* bkt_tt;   /* [n_buckets]   */
  const int32_t* bkt_conc; /* [n_buckets]   */
  const int64_t* bkt_off;  /* [n_buckets+1] */
  const double* samples;   /* [n_samples]   */
} emu_table_view;

/* Ranges/counts of one device table, for host-side mirrors. */
typedef struct emu_table_info {
  int64_t n_buckets;
  int64_t n_samples;
  int32_t tt_lo, tt_hi, conc_lo, conc_hi; /* valid iff n_buckets > 0 */
} emu_table_info;

/* Device views of a table handle's arrays (owned by the handle; [dev]). */
typedef struct emu_table_dev {
  int64_t n_buckets, n_samples, n_rows;
  int32_t* bkt_tt;
  int32_t* bkt_conc;
  int64_t* bkt_off;
  double* samples;
  int32_t* row_tt;    /* distinct tt values, ascending          [n_rows]   */
  int64_t* row_start; /* first bucket of each row               [n_rows+1] */
} emu_table_dev;

/* ---------------------------------------------------------------- tables --
 * emu_tables_create: upload three canonical tables (decode, mixed, combined)
 *   and build the per-table row index used by the neighbour search.
 *   Replaces LatencyOracle.__init__'s _TableIndex construction
 *   (oracle.py:187-198) and load_pack's PhaseTable.from_buckets (profile.py:122-129).
 *   Validates sortedness/uniqueness of (tt, conc), positive keys, nonempty buckets,
 *   positive samples and combined = decode + mixed sample counts
 *   (ProfilePack.validate, profile.py:178-194) -> EMU_ERR_INVALID with message.
 */
int emu_tables_create(const emu_table_view* decode, const emu_table_view* mixed,
                      const emu_table_view* combined, void* stream, emu_tables_t* out);

/* emu_tables_build: the offline profile-table build on the GPU.
 *   Replaces build_pack (profile.py:230-267) + PhaseTable.from_buckets
 *   (profile.py:122-129), and with canonical != 0 also save_pack's per-bucket
 *   ascending sample order (profile.py:281-282).
 *   Records are SoA: tt[n], conc[n], phase[n] (0/1), lat[n] (seconds),
 *   step[n] (may be NULL: not validated).  canonical == 0 keeps capture order
 *   inside each bucket, exactly like build_pack's dict appends.
 *   On an invalid record returns EMU_ERR_INVALID and writes the smallest
 *   offending index to *bad_index and the failed check to *bad_code:
 *     1 step_index < 0, 2 total_tokens < 1, 3 concurrency < 1,
 *     4 decode-only tt < conc, 5 latency_s !> 0    (StepTraceRecord.validate,
 *     profile.py:61-79, checked in that order). */
int emu_tables_build(const int32_t* tt, const int32_t* conc, const uint8_t* phase,
                     const double* lat, const int64_t* step, int64_t n, int canonical,
                     void* stream, emu_tables_t* out, int64_t* bad_index, int32_t* bad_code);
/* Builds run one at a time per process and bump-allocate their scratch (key
 * and sort buffers) from one persistent device buffer sized to the largest
 * build so far; this frees it. */
int emu_build_scratch_release(void);

int emu_tables_info(emu_tables_t t, int table_id, emu_table_info* out);
/* Device views of the handle-owned arrays (for copies out / NCCL broadcast). */
int emu_tables_device(emu_tables_t t, int table_id, emu_table_dev* out);
void emu_tables_destroy(emu_tables_t t);

/* ---------------------------------------------------------------- oracle --
 * emu_oracle_create: an oracle over a table handle with OracleConfig knobs
 *   (oracle.py:38-59).  Owns the device-side pool cache that mirrors
 *   LatencyOracle._cache (oracle.py:198-222): a dense (phase, tt, conc) key map
 *   over [1, dom_tt] x [1, dom_conc] (0 = derive from the tables), an
 *   open-addressing map for keys outside it, and a bump-allocated arena of
 *   pool slots {cdf f64, sample offset i32, count i32}.
 *   arena_slots / hash_slots = 0 pick defaults.  Returns EMU_ERR_INVALID for a
 *   config that fails OracleConfig.validate. */
int emu_oracle_create(emu_tables_t t, int32_t floor, double shepard_power, double epsilon,
                      int32_t dom_tt, int32_t dom_conc, int64_t arena_slots, int64_t hash_slots,
                      void* stream, emu_oracle_t* out);
void emu_oracle_destroy(emu_oracle_t o);
/* Drop every cached pool (the next batch rebuilds what it needs). */
int emu_oracle_flush(emu_oracle_t o, void* stream);

/* emu_oracle_pool: explicit pools for U keys (no caching), CSR output.
 *   Per key: table = phase table, or combined if it is empty (oracle.py:138-144);
 *   neighbours = shortest distance-sorted prefix reaching `floor`
 *   (_pool_order, oracle.py:80-105; ties by ascending (tt, conc));
 *   probs/cdf = _selection_probs (oracle.py:124-127) and Generator.choice's
 *   cumsum / cdf[-1] (oracle.py:133).
 *   Outputs ([dev]): pool_off[U+1] (int64, exclusive prefix of K_u; must hold
 *   U+1), pool_bkt/pool_dist/pool_prob/pool_cdf sized by `cap` entries,
 *   table_of_key[U] (int32 table id).  If sum K_u > cap returns
 *   EMU_ERR_CAPACITY with pool_off filled so the caller can size and retry. */
int emu_oracle_pool(emu_oracle_t o, const int32_t* key_tt, const int32_t* key_conc,
                    const uint8_t* key_phase, int64_t U, int64_t* pool_off, int32_t* pool_bkt,
                    double* pool_dist, double* pool_prob, double* pool_cdf, int64_t cap,
                    int32_t* table_of_key, void* stream);

/* emu_oracle_sample: Q independent draws (batched what-if sweeps / replay).
 *   Inputs [dev]: q_tt, q_conc, q_phase; u_sel/u_idx [dev] in EXPLICIT mode.
 *   Draw i: u = (u_sel>>11) * 2^-53, bucket slot = searchsorted(cdf, u, 'right'),
 *   index = 0 if n == 1 else Lemire32(u_idx word stream, n) -- exactly numpy's
 *   Generator.choice(p=...) then Generator.integers(n) (oracle.py:130-135).
 *   Outputs [dev]: out_lat[Q] (f64, a literal pack value), out_sidx[Q]
 *   (int32 index into the selected table's samples; bucket is implied).
 *   Pools missing from the cache are built first (lazy cache semantics). */
int emu_oracle_sample(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc,
                      const uint8_t* q_phase, int64_t Q, int rng_mode, const uint64_t* u_sel,
                      const uint32_t* u_idx, uint64_t seed, uint64_t ctr_base, double* out_lat,
                      int32_t* out_sidx, void* stream);

/* emu_oracle_sample_pcg64: Q draws that continue ONE numpy PCG64 stream in
 *   query order -- bit-identical to calling LatencyOracle.sample(tt, conc, phase)
 *   Q times on an oracle whose rng is np.random.default_rng(seed)
 *   (oracle.py:192, :224-226).  `pcg_state` [dev] is 6 x u64:
 *   {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}, read and
 *   advanced in place (numpy's PCG64.state dict, flattened). */
int emu_oracle_sample_pcg64(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc,
                            const uint8_t* q_phase, int64_t Q, uint64_t* pcg_state,
                            double* out_lat, int32_t* out_sidx, void* stream);

/* Same as emu_oracle_sample with HOST query and result buffers: chunks of 1M
 * queries are copied in on an internal stream, sampled on `stream` and copied
 * out on a second internal stream, so the copies overlap the pool build and
 * the draws (pinned buffers give full overlap).  Synchronizes before
 * returning.  `out_sidx` may be NULL (latencies only).  This is the call the
 * e2e measurement times. */
int emu_oracle_sample_host(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc,
                           const uint8_t* q_phase, int64_t Q, int rng_mode, const uint64_t* u_sel,
                           const uint32_t* u_idx, uint64_t seed, uint64_t ctr_base,
                           double* out_lat, int32_t* out_sidx, void* stream);

/* Single-step query for the engine's per-step backend call (engine.py:555-557):
 * one draw continuing the PCG64 stream held in device memory by the oracle
 * (seeded by emu_oracle_seed_pcg64), result returned by value through *out_lat.
 * Synchronous. */
int emu_oracle_seed_pcg64(emu_oracle_t o, const uint64_t* pcg_state6);
int emu_oracle_get_pcg64(emu_oracle_t o, uint64_t* pcg_state6);
int emu_oracle_step(emu_oracle_t o, int32_t tt, int32_t conc, int32_t phase, double* out_lat);
/* emu_oracle_step is served by a resident one-warp kernel that stays up for
 * EMU_STEP_SERVER_IDLE_US (default 100000) after the last step, so calls at the
 * engine's cadence (engine.py:565 sleeps the sampled latency) skip the kernel
 * launch.  A foreign device-wide synchronize waits for that timeout; park the
 * server first (it exits on its next poll; the next step relaunches it). */
int emu_oracle_park(emu_oracle_t o);

/* Build (without drawing) the pools of n keys [dev] not cached yet -- the
 * warm-up half of emu_oracle_sample (the lazy cache of _pooled, oracle.py:200-222). */
int emu_oracle_prefetch(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc,
                        const uint8_t* q_phase, int64_t n, void* stream);

/* Cache statistics: number of cached pools and arena slots in use. */
int emu_oracle_stats(emu_oracle_t o, int64_t* n_pools, int64_t* n_slots);

/* ------------------------------------------------------------- distances --
 * normalized_distance (oracle.py:62-77) over arrays: out[i] = distance of
 * (q_tt[i], q_conc[i]) to (b_tt[i], b_conc[i]) with the given ranges.  IEEE
 * round-to-nearest, no FMA contraction.  All arrays [dev]. */
int emu_distance(const int32_t* q_tt, const int32_t* q_conc, const int32_t* b_tt,
                 const int32_t* b_conc, int64_t n, int32_t tt_lo, int32_t tt_hi, int32_t conc_lo,
                 int32_t conc_hi, double* out, void* stream);

/* ------------------------------------------------------------ token fill --
 * Synthetic output-token fill for a batch of scheduled entries: the token part
 * of EmulatorEngine._apply_outcome (engine.py:464-483; ids per SPEC.md "token k
 * of request r has id k").  Per entry e (arrays [dev], length n):
 *   prefill entry: emits iff prefill_progress+chunk == prompt_len;
 *   decode entry : always emits;
 *   out_ids[e] = generated (the index of the emitted token) or -1;
 *   out_finished[e] = 1 iff the request is decoding and reaches target_len. */
int emu_token_fill(const uint8_t* is_prefill, const int32_t* chunk, const int32_t* prefill_progress,
                   const int32_t* prompt_len, const int32_t* generated, const int32_t* target_len,
                   int64_t n, int32_t* out_ids, uint8_t* out_finished, void* stream);

/* ------------------------------------------------------ capture stand-ins --
 * emu_ground_truth: ground_truth_latency (engine.py:128-147) for n step keys
 *   ([dev] columns): m * (base + per_token*tt + per_seq*conc) * (1 + g) with
 *   m = prefill_multiplier for mixed steps and g ~ N(0, noise_cv) redrawn while
 *   the factor is nonpositive; noise_cv == 0 consumes no randomness.  The
 *   deterministic part is bit-identical to the reference's expression; the
 *   deviates are Box-Muller on Philox4x32-10 keyed by (seed, i) (CPython's
 *   random.gauss stream is not reproduced).  GroundTruthParams.validate's
 *   checks and messages (engine.py:116-125) -> EMU_ERR_INVALID.
 * emu_gen_step_keys: n step keys ([dev] outputs) of the synthetic generator G
 *    from Philox(seed, i): conc = clip(rint(exp(conc_mu +
 *   conc_sigma z0)), 1, conc_max); decode with probability p_decode (tt = conc);
 *   else tt = min(tt_max, conc - 1 + clip(rint(exp(chunk_mu + chunk_sigma z1)), 1, tt_max)). */
int emu_ground_truth(const int32_t* tt, const int32_t* conc, const uint8_t* phase, int64_t n,
                     double base_s, double per_token_s, double per_seq_s, double prefill_multiplier,
                     double noise_cv, uint64_t seed, double* out_lat, void* stream);
int emu_gen_step_keys(int64_t n, uint64_t seed, double conc_mu, double conc_sigma, int32_t conc_max,
                      double p_decode, double chunk_mu, double chunk_sigma, int32_t tt_max, int32_t* tt,
                      int32_t* conc, uint8_t* phase, void* stream);

/* ------------------------------------------------------------ scheduler --
 * The reference scheduler in virtual time for S independent scenarios, one
 * GPU thread each (EmulatorEngine.admit / _schedule_step / _apply_outcome /
 * release_blocks, engine.py:323-483, driven like the reference's virtual-time
 * runs: admit arrivals <= t, schedule, latency, apply, t += latency).
 * emu_sched_create: scenario s owns requests [req_off[s], req_off[s+1]) of the
 *   concatenated host arrays prompt/target (int32) and arrival offsets (f64,
 *   ascending); one EngineConfig for all; at most max_steps steps each.
 *   EngineConfig.validate and admit's checks -> EMU_ERR_INVALID with the
 *   reference's messages.
 * emu_sched_run_replay      : step latencies from lat[S * max_steps] (parity replay);
 * emu_sched_run_ground_truth: ground_truth_latency with Philox(seed, s, step) noise;
 * emu_sched_run_oracle      : the oracle in the closed loop: scenario s draws from
 *   its own numpy PCG64 stream (pcg_states[6 s .. 6 s + 5], as in
 *   emu_oracle_sample_pcg64) exactly like LatencyOracle.sample; a step whose key
 *   has no pool pauses the scenario, the host builds the pools of all paused
 *   scenarios (emu_oracle_prefetch) and relaunches (*rounds = launches).
 * emu_sched_results: per scenario n_steps and status (1 done, 3 invariant
 *   error), per step [S * max_steps]: tt, conc, phase, latency, tokens emitted,
 *   requests finished, cumulative preemptions (host outputs; NULL skips). */
int emu_sched_create(int32_t S, const int64_t* req_off, const int32_t* prompt, const int32_t* target,
                     const double* arrival, int32_t num_gpu_blocks, int32_t block_size,
                     int32_t max_model_len, int32_t max_num_batched_tokens, int32_t max_num_seqs,
                     int64_t max_steps, emu_sched_t* out);
int emu_sched_run_replay(emu_sched_t sc, const double* lat, void* stream);
int emu_sched_run_ground_truth(emu_sched_t sc, double base_s, double per_token_s, double per_seq_s,
                               double prefill_multiplier, double noise_cv, uint64_t seed, void* stream);
int emu_sched_run_oracle(emu_sched_t sc, emu_oracle_t o, const uint64_t* pcg_states, int64_t* rounds,
                         void* stream);
int emu_sched_results(emu_sched_t sc, int64_t* n_steps, int32_t* status, int32_t* tt, int32_t* conc,
                      uint8_t* phase, double* lat, int32_t* tokens, int32_t* finished, int64_t* preempt);
/* Per-scenario totals [S x 4]: steps, tokens emitted, requests finished,
 * preemptions (accumulated by the kernel; valid with or without per-step outputs). */
int emu_sched_summary(emu_sched_t sc, int64_t* out4);
/* keep = 0 before a run: no per-step outputs (no S x max_steps x 33 B arrays; runs
 * of any length), totals only through emu_sched_summary.  Default 1. */
int emu_sched_keep_steps(emu_sched_t sc, int32_t keep);
void emu_sched_destroy(emu_sched_t sc);

/* --------------------------------------------------------------- codecs --
 * Native readers of the reference's on-disk formats (host-only; no CUDA).
 *
 * emu_pack_parse_json: a pack document as written by save_pack
 *   (profile.py:275-296) -> three tables in canonical SoA form, buckets stably
 *   sorted by (tt, conc) (PhaseTable.from_buckets, profile.py:122-129), samples
 *   in file order, numbers parsed correctly rounded (== Python float()).
 *   Replaces load_pack's json.loads + per-bucket objects (profile.py:299-347);
 *   validation stays with the caller (ProfilePack.validate).  Returns
 *   EMU_ERR_UNSUPPORTED for documents outside the subset the reference writes
 *   (syntax errors, escaped strings, non-integer keys, NaN, duplicate keys,
 *   schema_version != 1): the caller re-reads those with json.loads, which
 *   raises the reference's own PackFormatError / PackVersionError. */
int emu_pack_parse_json(const char* text, int64_t len, emu_pack_parsed_t* out);
/* sizes[6] = {B, N} of decode, mixed, combined; metadata_len = bytes of the
 * metadata object as canonical JSON (sorted keys, no spaces). */
int emu_pack_parsed_info(emu_pack_parsed_t p, int64_t* schema_version, int64_t* num_gpu_blocks,
                         int64_t* sizes, int64_t* metadata_len);
int emu_pack_parsed_copy(emu_pack_parsed_t p, int table, int32_t* tt, int32_t* conc, int64_t* off,
                         double* samples);
int emu_pack_parsed_metadata(emu_pack_parsed_t p, char* buf, int64_t cap);
void emu_pack_parsed_free(emu_pack_parsed_t p);

/* emu_trace_parse_jsonl: step-trace JSON lines (trace_record_to_line /
 *   parse_trace_line, profile.py:350-380) -> record columns in file order,
 *   blank lines skipped, parsed on n_threads host threads.  *n_out = records;
 *   EMU_ERR_CAPACITY if more than `cap`; EMU_ERR_UNSUPPORTED (with *bad_line =
 *   the record index) for a line outside the subset -- the caller re-reads
 *   the file with parse_trace_line for the reference's exact error.
 *   emu_trace_count_lines counts the non-blank lines. */
int64_t emu_trace_count_lines(const char* text, int64_t len);
int emu_trace_parse_jsonl(const char* text, int64_t len, int n_threads, int64_t cap, int64_t* step,
                          int32_t* tt, int32_t* conc, uint8_t* phase, double* lat, int64_t* n_out,
                          int64_t* bad_line);

/* ------------------------------------------------------------ profiling --
 * Every kernel the library launches goes through one launch macro that counts
 * it and, when profiling is on, brackets it with CUDA events recorded on the
 * launching stream.  emu_profile_read synchronizes the device, folds all
 * pending event pairs of `kernel` (e.g. "sample", "pool_warp", "mark") into
 * (*total_ms, *launches) and resets that kernel's accumulator. */
int64_t emu_launch_count(void);
/* Newline-separated names of the kernels with recorded launches (truncated to cap - 1 bytes). */
int emu_profile_names(char* buf, int64_t cap);
int emu_profile_enable(int on);
int emu_profile_read(const char* kernel, double* total_ms, int64_t* launches);

/* ---------------------------------------------------------------- misc --- */
const char* emu_last_error(void);
int emu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EMU_ABI_H */
