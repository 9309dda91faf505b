// sched.cu -- the reference scheduler in virtual time, one CTA per what-if
// scenario: a scheduling warp, plus a drawer warp in the oracle closed loop
// (the caller of the oracle that turns what-if scenarios
// into step-key streams).
//
// Restates EmulatorEngine._schedule_step / _apply_outcome / admit /
// release_blocks (engine.py:310-483) and the virtual-time driver of the
// reference's capture / acceptance runs: admit every request whose arrival
// offset is <= t, schedule a step, take its latency, apply the outcome,
// t += latency; an empty schedule jumps t to the next arrival.  Exact
// semantics kept: decode entries first over a snapshot of the running list,
// then prefills (running partial prefills, then the waiting queue in id order,
// both snapshotted before the pass), KV blocks reserved per step, make_room
// preempting the newest running request (which drops its entry and refunds its
// budget), FIFO admission that never preempts and stops at the first request
// that does not fit, and the completing prefill reserving its first output
// token.
//
// Latency sources: MODE 0 replays recorded latencies (parity with a recorded
// reference run); MODE 1 is ground_truth_latency with Philox noise (a capture
// stand-in); MODE 2 is the oracle itself in the closed loop -- each scenario
// owns a numpy PCG64 stream and draws exactly like LatencyOracle.sample; a step
// whose key has no pool yet pauses the scenario (the host builds the pools of
// all paused scenarios with the batched pool path and relaunches).
//
// The waiting queue is a bitmap over request ids (ids are arrival order, the
// queue is id-ordered); requests preempted after the candidate snapshot carry
// a later event stamp and are skipped, as the reference's list snapshot does.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <string>
#include <vector>

#include "emu_internal.cuh"
#include "prof.h"

namespace emu {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPf = 4;  // chunks of 32 requests whose loads are issued together
enum : uint8_t { RQ_WAITING = 0, RQ_PREFILLING = 1, RQ_DECODING = 2, RQ_PREEMPTED = 3, RQ_FINISHED = 4 };
enum : int32_t { SC_RUNNING = 0, SC_DONE = 1, SC_PAUSED = 2, SC_ERROR = 3 };

struct SchedArgs {
  int32_t num_blocks, block_size, max_batched, max_seqs;
  int32_t bs_shift;  // log2(block_size) when it is a power of two, else -1
  int64_t max_steps;
  int32_t S;
  // requests (per scenario slice [roff[s], roff[s+1]))
  const int64_t* roff;
  const int32_t* prompt;
  const int32_t* target;
  const double* arrival;
  int32_t* progress;
  int32_t* generated;
  int32_t* alloc;
  uint8_t* rphase;
  int32_t* eidx;
  int32_t* pevt;
  int32_t* running;  // slice of R_s
  int32_t* snap;     // slice of R_s
  uint32_t* wbits;   // slice [woff[s], woff[s+1])
  const int64_t* woff;
  // per-step entries [S * max_seqs]
  int32_t* ent_id;
  int32_t* ent_chunk;
  uint8_t* ent_pre;
  // scalar state [S]
  double* t;
  int32_t* next_arr;
  int32_t* nrun;
  int32_t* wfront;
  int32_t* free_blocks;
  int64_t* nsteps;
  int32_t* evt;
  int64_t* preempt;
  int32_t* status;
  int32_t* n_ent;
  int32_t* resume;
  int32_t* key;  // [S * 3] pending / current key (tt, conc, phase)
  uint64_t* pcg;  // [S * 6]
  // per-step outputs [S * max_steps], NULL when the run keeps totals only
  int32_t* o_tt;
  int32_t* o_conc;
  uint8_t* o_ph;
  double* o_lat;
  int32_t* o_tok;
  int32_t* o_fin;
  int64_t* o_pre;
  // latency sources
  int64_t* tot_tok;  // [S] tokens emitted / requests finished, summed over the run
  int64_t* tot_fin;
  const double* lat_in;  // MODE 0: [S * max_steps]
  double gt_base, gt_tok, gt_seq, gt_mult, gt_cv;
  uint64_t seed;
  MapView map;  // MODE 2
  const Slot* arena;
  const double* s0;
  const double* s1;
  // EMU_SCHED_PROF=1: per-scenario cycle / event counters [S * kProfN]
  long long* prof;
  int32_t smem;  // running list + entries in dynamic shared memory (17 B x max_seqs)
};
// prof slots: cycles in admit, decode pass, prefill pass, draw, apply+compact;
// then counts: steps, sequential-remainder iterations, waiting candidates,
// waiting-bitmap words scanned, preemptions' entry shifts
constexpr int kProfN = 10;

struct Scen {
  const SchedArgs& A;
  int32_t s;
  int64_t r0;  // first request (global index)
  int32_t R;
  int32_t* run;
  int32_t* snp;
  uint32_t* wb;
  int32_t* eid;
  int32_t* ech;
  uint8_t* epr;
  int32_t nrun, wfront, freeb, evt, ne, budget;
  int64_t npre;
  bool err;
  long long nseq = 0, ncand = 0, nwords = 0, nshift = 0;  // EMU_SCHED_PROF counters
  long long t_dec = 0;                                     // clock at the end of the decode pass
  int32_t lim = 0;  // requests admitted so far: every waiting id is below it
  int32_t cap = 0;  // capacity of run / snp (max_seqs when they live in shared memory)

  // token counts stay below max_model_len + max_num_batched_tokens: 32-bit division
  __device__ int32_t blocks_needed(int64_t tokens) const {
    const uint32_t n = (uint32_t)tokens + (uint32_t)A.block_size - 1u;
    return (int32_t)(A.bs_shift >= 0 ? n >> A.bs_shift : n / (uint32_t)A.block_size);
  }
  __device__ void wait_insert(int32_t r) {
    wb[r >> 5] |= 1u << (r & 31);
    if (r < wfront) wfront = r;
  }
  __device__ void wait_remove(int32_t r) { wb[r >> 5] &= ~(1u << (r & 31)); }
  // next waiting id >= r (or R); the scan stops at `lim`, so an empty queue
  // costs O(1) words instead of a pass over the not-yet-arrived tail
  __device__ int32_t wait_next(int32_t r) {
    int32_t w = r >> 5;
    const int32_t nw = (lim + 31) >> 5;
    if (w >= nw) return R;
    uint32_t m = wb[w] & (0xffffffffu << (r & 31));
    while (!m) {
      if (++w >= nw) return R;
      m = wb[w];
      nwords++;
    }
    return w * 32 + __ffs(m) - 1;
  }
  __device__ void release(int32_t r) {
    const int64_t g = r0 + r;
    if (A.alloc[g] == 0) err = true;  // EngineInvariantError: double free
    freeb += A.alloc[g];
    A.alloc[g] = 0;
  }
  __device__ void add_entry(int32_t r, int32_t chunk, bool pre) {
    eid[ne] = r;
    ech[ne] = chunk;
    epr[ne] = pre ? 1 : 0;
    A.eidx[r0 + r] = ne;
    ne++;
  }
  __device__ int32_t preempt_newest() {
    const int32_t v = run[--nrun];
    const int64_t g = r0 + v;
    A.rphase[g] = RQ_PREEMPTED;
    release(v);
    A.progress[g] = 0;
    wait_insert(v);
    A.pevt[g] = ++evt;
    npre++;
    const int32_t k = A.eidx[g];
    if (k >= 0) {  // drop its entry (order kept) and refund its budget
      budget += ech[k];
      nshift += ne - k - 1;
      for (int32_t q = k + 1; q < ne; q++) {
        eid[q - 1] = eid[q];
        ech[q - 1] = ech[q];
        epr[q - 1] = epr[q];
        A.eidx[r0 + eid[q - 1]] = q - 1;
      }
      ne--;
      A.eidx[g] = -1;
    }
    return v;
  }
  __device__ bool make_room(int32_t demand, int32_t requester) {
    while (freeb < demand)
      if (preempt_newest() == requester) return false;
    return true;
  }
  // one prefill candidate; returns false to stop the pass (reference `break`)
  __device__ bool prefill_candidate(int32_t r) {
    if (budget < 1 || ne >= A.max_seqs) return false;
    const int64_t g = r0 + r;
    const uint8_t ph = A.rphase[g];
    if (ph != RQ_PREFILLING && ph != RQ_WAITING && ph != RQ_PREEMPTED) return true;
    const int32_t prog = A.progress[g], pl = A.prompt[g];
    const int32_t chunk = min(pl - prog, budget);
    const bool completing = prog + chunk == pl;
    const int64_t new_total = (int64_t)prog + chunk + A.generated[g] + (completing ? 1 : 0);
    const int32_t demand = blocks_needed(new_total) - A.alloc[g];
    if (ph == RQ_PREFILLING) {
      if (demand > 0 && !make_room(demand, r)) return true;
    } else {
      if (demand > freeb) return false;
      wait_remove(r);
      if (nrun >= cap) {  // cannot happen: admissions need every running request to hold an entry
        err = true;
        return false;
      }
      run[nrun++] = r;
      A.rphase[g] = RQ_PREFILLING;
    }
    if (demand > 0) {
      freeb -= demand;
      A.alloc[g] += demand;
    }
    add_entry(r, chunk, true);
    budget -= chunk;
    return true;
  }
  // _schedule_step; returns the number of entries (0 = nothing to run).
  // Executed by the whole warp: sequential parts run identically on every
  // lane (uniform control flow, identical writes); the per-request loops are
  // lane-parallel where the reference's order cannot be observed.
  __device__ int32_t schedule() {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    budget = A.max_batched;
    ne = 0;
    const int32_t ns = nrun;
    for (int32_t k = lane; k < ns; k += 32) snp[k] = run[k];
    __syncwarp();
    // decoding requests first, one token each.  Per group of 32 x kPf
    // requests (lane-contiguous): decode ranks and the KV demand of the
    // admitted ones come from two warp scans; if every admitted entry's demand
    // fits in the free blocks, no make_room can fire and the group commits at
    // once (same order, same final state); otherwise commit up to the first
    // entry that would have to preempt and finish the pass sequentially.
    int32_t k_seq = ns;  // where the sequential remainder starts (ns = none)
    bool stop = false;
    for (int32_t base0 = 0; base0 < ns && !stop; base0 += 32 * kPf) {
      const int32_t kl = base0 + kPf * lane;
      int32_t rr[kPf], dmd[kPf], al[kPf];
      bool dc[kPf];
#pragma unroll
      for (int i = 0; i < kPf; i++) {
        rr[i] = -1;
        dmd[i] = 0;
        al[i] = 0;
        dc[i] = false;
        if (kl + i < ns) {
          const int32_t r = snp[kl + i];
          const int64_t g = r0 + r;
          rr[i] = r;
          const uint8_t ph = A.rphase[g];
          const int32_t pg = A.progress[g], gn = A.generated[g];
          al[i] = A.alloc[g];
          dc[i] = ph == RQ_DECODING;
          dmd[i] = blocks_needed((int64_t)pg + gn + 1) - al[i];
        }
      }
      int32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < kPf; i++) cnt += dc[i] ? 1 : 0;
      int32_t rk = cnt;  // inclusive scan of decode counts
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, rk, o);
        if (lane >= o) rk += y;
      }
      const int32_t ndec = __shfl_sync(kFull, rk, 31);
      rk -= cnt;  // decode rank of this lane's first request
      const int32_t allow = min(budget, A.max_seqs - ne);
      bool ok[kPf];
      int32_t lc[kPf], dsum = 0;
      {
        int32_t q = rk;
#pragma unroll
        for (int i = 0; i < kPf; i++) {
          ok[i] = dc[i] && q < allow;
          q += dc[i] ? 1 : 0;
          dsum += ok[i] && dmd[i] > 0 ? dmd[i] : 0;
          lc[i] = dsum;
        }
      }
      int32_t dx = dsum;  // inclusive scan of admitted demand
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(kFull, dx, o);
        if (lane >= o) dx += y;
      }
      const int32_t dtot = __shfl_sync(kFull, dx, 31);
      dx -= dsum;
      int32_t fi = kPf;
#pragma unroll
      for (int i = kPf - 1; i >= 0; i--)
        if (ok[i] && dx + lc[i] > freeb) fi = i;
      const unsigned fl = __ballot_sync(kFull, fi < kPf);
      int32_t fpos = ns, ncom, used;
      if (fl) {
        const int src = __ffs(fl) - 1;
        // the failing entry's rank = entries committed; demand before it
        int32_t frank = 0, fused = 0;
        if (lane == src) {
          int32_t q = rk, u = 0;
#pragma unroll
          for (int i = 0; i < kPf; i++)
            if (i < fi) {
              q += dc[i] ? 1 : 0;
              u += ok[i] && dmd[i] > 0 ? dmd[i] : 0;
            }
          frank = q;
          fused = dx + u;
        }
        fpos = base0 + kPf * src + __shfl_sync(kFull, fi, src);
        ncom = __shfl_sync(kFull, frank, src);
        used = __shfl_sync(kFull, fused, src);
      } else {
        ncom = min(ndec, allow);
        used = dtot;
      }
      {
        int32_t q = rk;
#pragma unroll
        for (int i = 0; i < kPf; i++) {
          if (ok[i] && kl + i < fpos) {
            const int64_t g = r0 + rr[i];
            if (dmd[i] > 0) A.alloc[g] = al[i] + dmd[i];
            const int32_t e = ne + q;
            eid[e] = rr[i];
            ech[e] = 1;
            epr[e] = 0;
            A.eidx[g] = e;
          }
          q += dc[i] ? 1 : 0;
        }
      }
      freeb -= used;
      ne += ncom;
      budget -= ncom;
      __syncwarp();
      if (fl) {
        k_seq = fpos;
        stop = true;
      } else if (ndec > allow) {
        stop = true;  // the reference breaks at the first decode request over the budget
      }
    }
    for (int32_t k = k_seq; k < ns; k++) {  // sequential remainder (preemption possible)
      nseq++;
      const int32_t r = snp[k];
      const int64_t g = r0 + r;
      if (A.rphase[g] != RQ_DECODING) continue;
      if (budget < 1 || ne >= A.max_seqs) break;
      const int32_t demand = blocks_needed((int64_t)A.progress[g] + A.generated[g] + 1) - A.alloc[g];
      if (demand > 0) {
        if (!make_room(demand, r)) continue;
        freeb -= demand;
        A.alloc[g] += demand;
      }
      add_entry(r, 1, false);
      budget -= 1;
      __syncwarp();
    }
    if (A.prof) t_dec = clock64();
    // prefills: running partial prefills, then the waiting queue (both as of now)
    int32_t nc = 0;
    __syncwarp();
    for (int32_t base0 = 0; base0 < nrun; base0 += 32 * kPf) {
      int32_t pr[kPf];
      bool pf[kPf];
#pragma unroll
      for (int j = 0; j < kPf; j++) {
        const int32_t k = base0 + 32 * j + lane;
        pr[j] = k < nrun ? run[k] : 0;
        pf[j] = k < nrun && A.rphase[r0 + pr[j]] == RQ_PREFILLING;
      }
#pragma unroll
      for (int j = 0; j < kPf; j++) {
        const unsigned m = __ballot_sync(kFull, pf[j]);
        if (pf[j]) snp[nc + __popc(m & lt)] = pr[j];
        nc += __popc(m);
      }
    }
    __syncwarp();
    const int32_t snap_evt = evt;
    const int32_t wstart = wfront;
    bool go = true;
    for (int32_t k = 0; k < nc && go; k++) {
      go = prefill_candidate(snp[k]);
      __syncwarp();
    }
    for (int32_t r = wait_next(wstart); go && r < R; r = wait_next(r + 1)) {
      ncand++;
      if (A.pevt[r0 + r] > snap_evt) continue;  // preempted after the snapshot
      go = prefill_candidate(r);
      __syncwarp();
    }
    // keep wfront a lower bound of the waiting ids
    wfront = wait_next(wfront);
    return ne;
  }
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ Pcg64 load_pcg(const uint64_t* p) {
  Pcg64 g;
  g.s_hi = p[0];
  g.s_lo = p[1];
  g.i_hi = p[2];
  g.i_lo = p[3];
  g.has_u32 = (uint32_t)p[4];
  g.u32 = (uint32_t)p[5];
  return g;
}

// The oracle draw of a step whose pool entry `e` exists (LatencyOracle._draw,
// oracle.py:130-135): choice over the pool CDF, then the sample index.
__device__ __forceinline__ double oracle_draw(const SchedArgs& A, long long e, int ph, Pcg64& g) {
  const PoolPick pk = pool_pick<true>(A.arena, e, unit_k53(pcg64_next64(g)));
  uint32_t j = 0;
  if (pk.n > 1) {
    const uint32_t w0 = pcg64_next32(g);
    j = lemire_index((uint32_t)pk.n, w0, [&]() { return pcg64_next32(g); });
  }
  return __ldcg((ph ? A.s1 : A.s0) + pk.soff + (int32_t)j);
}

// One scenario per CTA: scenarios diverge completely, so one warp each keeps S
// independent instruction streams spread over the SMs; the warp's lanes share
// the per-request loops of a step.  In the oracle closed loop (MODE 2) a
// second warp owns the scenario's PCG64 stream and draws the step's latency
// while the first applies the step's outcome (which does not need it).
template <int MODE>
__global__ void __launch_bounds__(64, 1) k_sched(SchedArgs A) {
  const int32_t s = blockIdx.x;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (s >= A.S) return;
  if (A.status[s] == SC_DONE || A.status[s] == SC_ERROR) return;
  __shared__ long long s_e;
  __shared__ double s_lat;
  __shared__ int s_ph, s_cmd;
  if (MODE == 2 && threadIdx.x >= 32) {  // the drawer warp
    uint64_t* p = A.pcg + 6 * (int64_t)s;
    Pcg64 g = load_pcg(p);
    for (;;) {
      named_bar(1, 64);
      if (!s_cmd) break;
      const double lat = oracle_draw(A, s_e, s_ph, g);
      if (lane == 0) s_lat = lat;
      named_bar(2, 64);
    }
    if (lane == 0) {
      p[0] = g.s_hi;
      p[1] = g.s_lo;
      p[2] = g.i_hi;
      p[3] = g.i_lo;
      p[4] = g.has_u32;
      p[5] = g.u32;
    }
    return;
  }
  const int64_t r0 = A.roff[s];
  Scen c{A, s, r0, (int32_t)(A.roff[s + 1] - r0), A.running + r0, A.snap + r0, A.wbits + A.woff[s],
         A.ent_id + (int64_t)s * A.max_seqs, A.ent_chunk + (int64_t)s * A.max_seqs, A.ent_pre + (int64_t)s * A.max_seqs,
         A.nrun[s], A.wfront[s], A.free_blocks[s], A.evt[s], A.n_ent[s], 0, A.preempt[s], false};
  c.cap = c.R;
  // running list, its snapshot and the step's entries live in shared memory
  // when max_seqs allows (running <= max_seqs: an admission needs every running
  // request to hold one of the <= max_seqs entries)
  extern __shared__ __align__(16) unsigned char dsm[];
  if (A.smem) {
    const int32_t q = A.max_seqs;
    int32_t* rs = reinterpret_cast<int32_t*>(dsm);
    for (int32_t k = lane; k < c.nrun; k += 32) rs[k] = c.run[k];
    for (int32_t k = lane; k < c.ne; k += 32) {
      rs[2 * q + k] = c.eid[k];
      rs[3 * q + k] = c.ech[k];
      reinterpret_cast<uint8_t*>(rs + 4 * q)[k] = c.epr[k];
    }
    c.run = rs;
    c.snp = rs + q;
    c.eid = rs + 2 * q;
    c.ech = rs + 3 * q;
    c.epr = reinterpret_cast<uint8_t*>(rs + 4 * q);
    c.cap = q;
    __syncwarp();
  }
  double t = A.t[s];
  int32_t nxt = A.next_arr[s];
  int64_t step = A.nsteps[s];
  int32_t st = SC_RUNNING;
  bool resume = A.resume[s] != 0;
  int32_t* key = A.key + 3 * (int64_t)s;
  const bool P = A.prof != nullptr;
  const int64_t step0 = step;
  long long tok_sum = 0, fin_sum = 0;
  long long pc0 = 0, pc1 = 0, pc2 = 0, pc3 = 0, pc4 = 0, tc = P ? clock64() : 0;
#define EMU_LAP(acc)                 \
  if (P) {                           \
    const long long n_ = clock64();  \
    acc += n_ - tc;                  \
    tc = n_;                         \
  }
  // arrival offsets of requests nxt .. nxt+3 in registers (+inf past the end)
  const double kNever = __longlong_as_double(0x7ff0000000000000LL);
  auto arrival_at = [&](int32_t i) { return i < c.R ? A.arrival[r0 + i] : kNever; };
  double a0 = arrival_at(nxt), a1 = arrival_at(nxt + 1), a2 = arrival_at(nxt + 2), a3 = arrival_at(nxt + 3);
  while (step < A.max_steps) {
    if (!resume) {
      while (a0 <= t) {  // admit (engine.py:323-340)
        const int64_t gi = r0 + nxt;
        A.rphase[gi] = RQ_WAITING;
        A.progress[gi] = 0;
        A.generated[gi] = 0;
        A.alloc[gi] = 0;
        A.eidx[gi] = -1;
        A.pevt[gi] = 0;
        c.wait_insert(nxt);
        nxt++;
        a0 = a1;  // the arrival window slides; its new tail load is not awaited here
        a1 = a2;
        a2 = a3;
        a3 = arrival_at(nxt + 3);
      }
      EMU_LAP(pc0);
      c.lim = nxt;
      const int32_t ne = c.schedule();
      if (P) {
        pc1 += c.t_dec - tc;
        tc = c.t_dec;
        EMU_LAP(pc2);
      }
      if (c.err) {
        st = SC_ERROR;
        break;
      }
      if (ne == 0) {
        if (nxt >= c.R) {
          st = SC_DONE;
          break;
        }
        t = a0;
        continue;
      }
      int32_t tt = 0;
      bool mixed = false;
      for (int32_t k = lane; k < ne; k += 32) {
        tt += c.ech[k];
        mixed |= c.epr[k] != 0;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(kFull, tt, o);
      const bool all_decode = !__any_sync(kFull, mixed);
      key[0] = tt;
      key[1] = ne;
      key[2] = all_decode ? 0 : 1;
    }
    resume = false;
    const int32_t tt = key[0], conc = key[1], ph = key[2];
    double lat;
    if (MODE == 0) {
      lat = A.lat_in[(int64_t)s * A.max_steps + step];
    } else if (MODE == 1) {
      const double m = ph ? A.gt_mult : 1.0;
      lat = __dmul_rn(m, __dadd_rn(__dadd_rn(A.gt_base, __dmul_rn(A.gt_tok, (double)tt)), __dmul_rn(A.gt_seq, (double)conc)));
      if (A.gt_cv > 0.0) {
        const uint2 k2 = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
        double f = 0.0;
        for (uint32_t round = 0;; round++) {
          const uint4 r = philox4x32_10(make_uint4((uint32_t)step, (uint32_t)((uint64_t)step >> 32), (uint32_t)s, round), k2);
          const double u1 = ((double)((((uint64_t)r.x << 32) | r.y) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
          const double u2 = (double)((((uint64_t)r.z << 32) | r.w) >> 11) * (1.0 / 9007199254740992.0);
          double sn, cs;
          sincospi(2.0 * u2, &sn, &cs);
          f = __dadd_rn(1.0, __dmul_rn(A.gt_cv, sqrt(-2.0 * log(u1)) * cs));
          if (f > 0.0) break;
        }
        lat = __dmul_rn(lat, f);
      }
    } else {
      const int64_t idx = map_find<false>(A.map, ph, tt, conc);
      const long long e = idx >= 0 ? __ldcg(map_entry_ptr(A.map, idx)) : 0;
      if (e <= 0) {  // no pool yet: pause; the host builds it and relaunches
        st = SC_PAUSED;
        A.resume[s] = 1;
        break;
      }
      if (lane == 0) {  // hand the draw to the drawer warp
        s_e = e;
        s_ph = ph;
        s_cmd = 1;
      }
      named_bar(1, 64);
      lat = 0.0;  // arrives after the outcome is applied
    }
    EMU_LAP(pc3);
    // _apply_outcome (engine.py:464-483): entries are distinct requests, so the
    // per-entry updates run lane-parallel; finished requests leave the running
    // list in one order-preserving compaction.
    int32_t tokens = 0, fin = 0, freed = 0;
    bool dfree = false;
    for (int32_t kb = 0; kb < c.ne; kb += 32 * kPf) {
      int32_t er[kPf], ech[kPf], epg[kPf], epl[kPf], egn[kPf], etg[kPf], eal[kPf];
      uint8_t eph[kPf], epr[kPf];
#pragma unroll
      for (int j = 0; j < kPf; j++) {
        const int32_t k = kb + 32 * j + lane;
        er[j] = -1;
        if (k < c.ne) {
          const int32_t r = c.eid[k];
          const int64_t gi = r0 + r;
          er[j] = r;
          ech[j] = c.ech[k];
          epr[j] = c.epr[k];
          epg[j] = A.progress[gi];
          epl[j] = A.prompt[gi];
          egn[j] = A.generated[gi];
          etg[j] = A.target[gi];
          eal[j] = A.alloc[gi];
          eph[j] = A.rphase[gi];
        }
      }
#pragma unroll
      for (int j = 0; j < kPf; j++) {
        if (er[j] < 0) continue;
        const int64_t gi = r0 + er[j];
        A.eidx[gi] = -1;
        uint8_t ph = eph[j];
        int32_t gn = egn[j];
        if (epr[j]) {
          const int32_t pg = epg[j] + ech[j];
          A.progress[gi] = pg;
          if (pg == epl[j]) {
            ph = RQ_DECODING;
            gn += 1;
            tokens++;
          }
        } else {
          gn += 1;
          tokens++;
        }
        if (ph == RQ_DECODING && gn >= etg[j]) {
          ph = RQ_FINISHED;
          dfree |= eal[j] == 0;
          freed += eal[j];
          A.alloc[gi] = 0;
          fin++;
        }
        if (gn != egn[j]) A.generated[gi] = gn;
        if (ph != eph[j]) A.rphase[gi] = ph;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tokens += __shfl_xor_sync(kFull, tokens, o);
      fin += __shfl_xor_sync(kFull, fin, o);
      freed += __shfl_xor_sync(kFull, freed, o);
    }
    if (__any_sync(kFull, dfree)) c.err = true;
    c.freeb += freed;
    __syncwarp();
    if (fin) {
      int32_t out = 0;
      for (int32_t base0 = 0; base0 < c.nrun; base0 += 32 * kPf) {
        int32_t pr[kPf];
        bool keep[kPf];
#pragma unroll
        for (int j = 0; j < kPf; j++) {
          const int32_t k = base0 + 32 * j + lane;
          pr[j] = k < c.nrun ? c.run[k] : 0;
          keep[j] = k < c.nrun && A.rphase[r0 + pr[j]] != RQ_FINISHED;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kPf; j++) {
          const unsigned m = __ballot_sync(kFull, keep[j]);
          if (keep[j]) c.run[out + __popc(m & lt)] = pr[j];
          out += __popc(m);
        }
        __syncwarp();
      }
      c.nrun = out;
    }
    if (MODE == 2) {
      named_bar(2, 64);
      lat = s_lat;
    }
    if (c.err) {
      st = SC_ERROR;
      break;
    }
    if (A.o_tt) {
      const int64_t o = (int64_t)s * A.max_steps + step;
      A.o_tt[o] = tt;
      A.o_conc[o] = conc;
      A.o_ph[o] = (uint8_t)ph;
      A.o_lat[o] = lat;
      A.o_tok[o] = tokens;
      A.o_fin[o] = fin;
      A.o_pre[o] = c.npre;
    }
    tok_sum += tokens;
    fin_sum += fin;
    c.ne = 0;
    t = __dadd_rn(t, lat);
    step++;
    EMU_LAP(pc4);
  }
  if (P && lane == 0) {
    long long* q = A.prof + (int64_t)s * kProfN;
    q[0] += pc0;
    q[1] += pc1;
    q[2] += pc2;
    q[3] += pc3;
    q[4] += pc4;
    q[5] += step - step0;
    q[6] += c.nseq;
    q[7] += c.ncand;
    q[8] += c.nwords;
    q[9] += c.nshift;
  }
  if (st == SC_RUNNING && step >= A.max_steps) st = SC_DONE;
  A.t[s] = t;
  A.next_arr[s] = nxt;
  A.nsteps[s] = step;
  A.nrun[s] = c.nrun;
  A.wfront[s] = c.wfront;
  A.free_blocks[s] = c.freeb;
  A.evt[s] = c.evt;
  A.preempt[s] = c.npre;
  A.n_ent[s] = c.ne;
  if (lane == 0) {
    A.tot_tok[s] += tok_sum;
    A.tot_fin[s] += fin_sum;
  }
  if (A.smem) {  // back to the scenario's global slices for the next launch
    __syncwarp();
    int32_t* gr = A.running + r0;
    const int64_t e0 = (int64_t)s * A.max_seqs;
    for (int32_t k = lane; k < c.nrun; k += 32) gr[k] = c.run[k];
    for (int32_t k = lane; k < c.ne; k += 32) {
      A.ent_id[e0 + k] = c.eid[k];
      A.ent_chunk[e0 + k] = c.ech[k];
      A.ent_pre[e0 + k] = c.epr[k];
    }
  }
  A.status[s] = st;
  if (st != SC_PAUSED) A.resume[s] = 0;
  if (MODE == 2) {  // release the drawer warp
    if (lane == 0) s_cmd = 0;
    named_bar(1, 64);
  }
#undef EMU_LAP
}

}  // namespace emu

using namespace emu;

namespace emu {
// oracle.cu: the cache views the closed loop reads, and the pool build for keys
int oracle_views(emu_oracle_t o, MapView* m, const Slot** arena, const double** s0, const double** s1);
}

struct emu_sched_s {
  SchedArgs a{};
  int32_t S = 0;
  int64_t R = 0, W = 0, max_steps = 0;
  bool keep = true;  // per-step outputs (allocated by the first run that keeps them)
  std::vector<void*> owned;
  std::vector<int64_t> roff_h;
  template <typename T>
  int alloc(T** p, int64_t n) {
    *p = nullptr;
    EMU_CUDA(cudaMalloc((void**)p, sizeof(T) * (size_t)std::max<int64_t>(1, n)));
    owned.push_back((void*)*p);
    return EMU_OK;
  }
  ~emu_sched_s() {
    if (a.prof) print_prof();
    for (void* p : owned) cudaFree(p);
  }
  void print_prof() {
    std::vector<long long> h((size_t)S * kProfN);
    if (cudaMemcpy(h.data(), a.prof, 8 * h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    static const char* names[kProfN] = {"admit_cyc", "decode_cyc", "prefill_cyc", "draw_cyc", "apply_cyc",
                                        "steps",     "seq_iters",  "wait_cands",  "wait_words", "entry_shifts"};
    std::vector<long long> sum(kProfN, 0);
    int32_t slow = 0;
    long long slow_c = -1;
    for (int32_t s = 0; s < S; s++) {
      long long c = 0;
      for (int i = 0; i < kProfN; i++) sum[i] += h[(size_t)s * kProfN + i];
      for (int i = 0; i < 5; i++) c += h[(size_t)s * kProfN + i];
      if (c > slow_c) slow_c = c, slow = s;
    }
    fprintf(stderr, "[sched prof] all scenarios:");
    for (int i = 0; i < kProfN; i++) fprintf(stderr, " %s=%lld", names[i], sum[i]);
    fprintf(stderr, "\n[sched prof] slowest scenario %d:", slow);
    for (int i = 0; i < kProfN; i++) fprintf(stderr, " %s=%lld", names[i], h[(size_t)slow * kProfN + i]);
    fprintf(stderr, "\n");
  }
};

static std::string fmt_i(int64_t v) { return std::to_string(v); }

static size_t sched_smem_bytes(int32_t max_seqs) { return ((size_t)17 * max_seqs + 15) & ~(size_t)15; }
constexpr size_t kSchedSmemMax = 160 * 1024;  // larger max_num_seqs keep the lists in global memory

static int sched_reset(emu_sched_t sc, cudaStream_t s) {
  SchedArgs& a = sc->a;
  const int32_t S = sc->S;
  EMU_CUDA(cudaMemsetAsync(a.wbits, 0, 4 * sc->W, s));
  EMU_CUDA(cudaMemsetAsync(a.t, 0, 8 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.next_arr, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.nrun, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.wfront, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.nsteps, 0, 8 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.tot_tok, 0, 8 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.tot_fin, 0, 8 * S, s));
  if (sc->keep && !a.o_tt) {  // per-step outputs, S x max_steps x 33 B
    const int64_t SM = (int64_t)S * sc->max_steps;
    int rc;
    if ((rc = sc->alloc(&a.o_tt, SM)) || (rc = sc->alloc(&a.o_conc, SM)) || (rc = sc->alloc(&a.o_ph, SM)) ||
        (rc = sc->alloc(&a.o_lat, SM)) || (rc = sc->alloc(&a.o_tok, SM)) || (rc = sc->alloc(&a.o_fin, SM)) ||
        (rc = sc->alloc(&a.o_pre, SM)))
      return rc;
  }
  EMU_CUDA(cudaMemsetAsync(a.evt, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.preempt, 0, 8 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.status, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.n_ent, 0, 4 * S, s));
  EMU_CUDA(cudaMemsetAsync(a.resume, 0, 4 * S, s));
  std::vector<int32_t> fb((size_t)S, a.num_blocks);
  EMU_CUDA(cudaMemcpyAsync(a.free_blocks, fb.data(), 4 * S, cudaMemcpyHostToDevice, s));
  EMU_CUDA(cudaStreamSynchronize(s));
  return EMU_OK;
}

extern "C" {

int emu_sched_create(int32_t S, const int64_t* req_off, const int32_t* prompt, const int32_t* target,
                     const double* arrival, int32_t num_gpu_blocks, int32_t block_size, int32_t max_model_len,
                     int32_t max_num_batched_tokens, int32_t max_num_seqs, int64_t max_steps, emu_sched_t* out) {
  if (!out) return fail(EMU_ERR_INVALID, "out is NULL");
  *out = nullptr;
  // EngineConfig.validate (engine.py:85-104)
  if (block_size < 1) return fail(EMU_ERR_INVALID, "block_size must be >= 1, got " + fmt_i(block_size));
  if (num_gpu_blocks < 1) return fail(EMU_ERR_INVALID, "num_gpu_blocks must be >= 1, got " + fmt_i(num_gpu_blocks));
  if (max_model_len < 1) return fail(EMU_ERR_INVALID, "max_model_len must be >= 1, got " + fmt_i(max_model_len));
  if (max_num_batched_tokens < block_size)
    return fail(EMU_ERR_INVALID, "max_num_batched_tokens " + fmt_i(max_num_batched_tokens) + " must be >= block_size " +
                                     fmt_i(block_size));
  if (max_num_seqs < 1) return fail(EMU_ERR_INVALID, "max_num_seqs must be >= 1, got " + fmt_i(max_num_seqs));
  if (max_num_batched_tokens < max_num_seqs)
    return fail(EMU_ERR_INVALID, "max_num_batched_tokens " + fmt_i(max_num_batched_tokens) +
                                     " must be >= max_num_seqs " + fmt_i(max_num_seqs));
  if (S < 1 || !req_off || max_steps < 1) return fail(EMU_ERR_INVALID, "need S >= 1 scenarios and max_steps >= 1");
  std::vector<int64_t> roff(req_off, req_off + S + 1);
  if (roff[0] != 0) return fail(EMU_ERR_INVALID, "req_off[0] must be 0");
  std::vector<int64_t> woff((size_t)S + 1, 0);
  for (int32_t s = 0; s < S; s++) {
    const int64_t n = roff[s + 1] - roff[s];
    if (n < 0 || n > (1LL << 30)) return fail(EMU_ERR_INVALID, "bad request offsets");
    woff[s + 1] = woff[s] + (n + 31) / 32;
  }
  const int64_t R = roff[S];
  // admission checks (engine.py:323-336) and ascending arrival offsets; the
  // request table is split over host threads, the first bad request reports
  std::atomic<int64_t> first_bad{R};
  auto check_range = [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi && i < first_bad.load(std::memory_order_relaxed); i++) {
      const int64_t total = (int64_t)prompt[i] + target[i];
      const bool bad = prompt[i] < 1 || target[i] < 1 || total > max_model_len ||
                       (total + block_size - 1) / block_size > num_gpu_blocks ||
                       (i > 0 && arrival[i] < arrival[i - 1] && !std::binary_search(roff.begin(), roff.end(), i));
      if (bad) {
        int64_t cur = first_bad.load();
        while (i < cur && !first_bad.compare_exchange_weak(cur, i)) {
        }
        return;
      }
    }
  };
  {
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), R / (1 << 20)));
    std::vector<std::thread> th;
    for (int k = 0; k < nt; k++) th.emplace_back(check_range, R * k / nt, R * (k + 1) / nt);
    for (auto& t : th) t.join();
  }
  if (first_bad.load() < R) {
    const int64_t i = first_bad.load();
    if (prompt[i] < 1) return fail(EMU_ERR_INVALID, "prompt_tokens must be >= 1, got " + fmt_i(prompt[i]));
    if (target[i] < 1) return fail(EMU_ERR_INVALID, "max_tokens must be >= 1, got " + fmt_i(target[i]));
    const int64_t total = (int64_t)prompt[i] + target[i];
    if (total > max_model_len)
      return fail(EMU_ERR_INVALID, "prompt_tokens + max_tokens = " + fmt_i(total) + " exceeds max_model_len " +
                                       fmt_i(max_model_len));
    const int64_t fb = (total + block_size - 1) / block_size;
    if (fb > num_gpu_blocks)
      return fail(EMU_ERR_INVALID, "request needs " + fmt_i(fb) + " KV blocks but the engine has only " +
                                       fmt_i(num_gpu_blocks));
    return fail(EMU_ERR_INVALID, "arrival offsets must ascend");
  }
  auto* sc = new emu_sched_s();
  sc->S = S;
  sc->R = R;
  sc->W = woff[S];
  sc->max_steps = max_steps;
  sc->roff_h = roff;
  SchedArgs& a = sc->a;
  a.num_blocks = num_gpu_blocks;
  a.block_size = block_size;
  a.bs_shift = -1;
  if ((block_size & (block_size - 1)) == 0)
    for (int b = 0; b < 31; b++)
      if ((1 << b) == block_size) a.bs_shift = b;
  a.max_batched = max_num_batched_tokens;
  a.max_seqs = max_num_seqs;
  a.max_steps = max_steps;
  a.S = S;
  int rc;
  int64_t *d_roff, *d_woff;
  int32_t *d_prompt, *d_target;
  double* d_arr;
  const int64_t SQ = (int64_t)S * max_num_seqs;
  if ((rc = sc->alloc(&d_roff, S + 1)) || (rc = sc->alloc(&d_woff, S + 1)) || (rc = sc->alloc(&d_prompt, R)) ||
      (rc = sc->alloc(&d_target, R)) || (rc = sc->alloc(&d_arr, R)) || (rc = sc->alloc(&a.progress, R)) ||
      (rc = sc->alloc(&a.generated, R)) || (rc = sc->alloc(&a.alloc, R)) || (rc = sc->alloc(&a.rphase, R)) ||
      (rc = sc->alloc(&a.eidx, R)) || (rc = sc->alloc(&a.pevt, R)) || (rc = sc->alloc(&a.running, R)) ||
      (rc = sc->alloc(&a.snap, R)) || (rc = sc->alloc(&a.wbits, sc->W)) || (rc = sc->alloc(&a.ent_id, SQ)) ||
      (rc = sc->alloc(&a.ent_chunk, SQ)) || (rc = sc->alloc(&a.ent_pre, SQ)) || (rc = sc->alloc(&a.t, S)) ||
      (rc = sc->alloc(&a.next_arr, S)) || (rc = sc->alloc(&a.nrun, S)) || (rc = sc->alloc(&a.wfront, S)) ||
      (rc = sc->alloc(&a.free_blocks, S)) || (rc = sc->alloc(&a.nsteps, S)) || (rc = sc->alloc(&a.evt, S)) ||
      (rc = sc->alloc(&a.preempt, S)) || (rc = sc->alloc(&a.status, S)) || (rc = sc->alloc(&a.n_ent, S)) ||
      (rc = sc->alloc(&a.resume, S)) || (rc = sc->alloc(&a.key, 3 * (int64_t)S)) ||
      (rc = sc->alloc(&a.pcg, 6 * (int64_t)S)) || (rc = sc->alloc(&a.tot_tok, S)) || (rc = sc->alloc(&a.tot_fin, S))) {
    delete sc;
    return rc;
  }
  const char* pe = getenv("EMU_SCHED_PROF");
  if (pe && pe[0] == '1') {
    if ((rc = sc->alloc(&a.prof, (int64_t)S * kProfN)) ||
        cudaMemset(a.prof, 0, 8 * (size_t)S * kProfN) != cudaSuccess) {
      delete sc;
      return rc ? rc : cuda_fail(cudaGetLastError(), "prof");
    }
  }
  a.roff = d_roff;
  a.woff = d_woff;
  a.prompt = d_prompt;
  a.target = d_target;
  a.arrival = d_arr;
  if (cudaMemcpy(d_roff, roff.data(), 8 * (S + 1), cudaMemcpyDefault) != cudaSuccess ||
      cudaMemcpy(d_woff, woff.data(), 8 * (S + 1), cudaMemcpyDefault) != cudaSuccess ||
      cudaMemcpy(d_prompt, prompt, 4 * R, cudaMemcpyDefault) != cudaSuccess ||
      cudaMemcpy(d_target, target, 4 * R, cudaMemcpyDefault) != cudaSuccess ||
      cudaMemcpy(d_arr, arrival, 8 * R, cudaMemcpyDefault) != cudaSuccess) {
    delete sc;
    return cuda_fail(cudaGetLastError(), "emu_sched_create copies");
  }
  *out = sc;
  return EMU_OK;
}

void emu_sched_destroy(emu_sched_t sc) { delete sc; }

static int launch_sched(emu_sched_t sc, int mode, cudaStream_t s) {
  const int grid = sc->S;
  const size_t sm = sched_smem_bytes(sc->a.max_seqs);
  sc->a.smem = sm <= kSchedSmemMax ? 1 : 0;
  if (const char* v = getenv("EMU_SCHED_SMEM"))  // 0: force the global-memory lists (tests)
    if (v[0] == '0') sc->a.smem = 0;
  const size_t dyn = sc->a.smem ? sm : 0;
  SchedArgs la = sc->a;
  if (!sc->keep) la.o_tt = nullptr;  // totals only
  if (dyn > 48 * 1024) {
    EMU_CUDA(cudaFuncSetAttribute(k_sched<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    EMU_CUDA(cudaFuncSetAttribute(k_sched<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    EMU_CUDA(cudaFuncSetAttribute(k_sched<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  }
  if (mode == 0) EMU_LAUNCH("sched", s, k_sched<0><<<grid, 32, dyn, s>>>(la));
  if (mode == 1) EMU_LAUNCH("sched", s, k_sched<1><<<grid, 32, dyn, s>>>(la));
  if (mode == 2) EMU_LAUNCH("sched", s, k_sched<2><<<grid, 64, dyn, s>>>(la));
  EMU_CUDA(cudaGetLastError());
  return EMU_OK;
}

int emu_sched_run_replay(emu_sched_t sc, const double* lat, void* stream) {
  if (!sc || !lat) return fail(EMU_ERR_INVALID, "NULL scheduler/latencies");
  cudaStream_t s = as_stream(stream);
  int rc = sched_reset(sc, s);
  if (rc) return rc;
  double* d = nullptr;
  EMU_CUDA(cudaMalloc(&d, 8 * (size_t)sc->S * sc->max_steps));
  EMU_CUDA(cudaMemcpyAsync(d, lat, 8 * (size_t)sc->S * sc->max_steps, cudaMemcpyDefault, s));
  sc->a.lat_in = d;
  rc = launch_sched(sc, 0, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(d);
  sc->a.lat_in = nullptr;
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "k_sched");
  return EMU_OK;
}

int emu_sched_run_ground_truth(emu_sched_t sc, double base_s, double per_token_s, double per_seq_s,
                               double prefill_multiplier, double noise_cv, uint64_t seed, void* stream) {
  if (!sc) return fail(EMU_ERR_INVALID, "NULL scheduler");
  if (!(base_s > 0)) return fail(EMU_ERR_INVALID, "base_s must be > 0");
  if (per_token_s < 0 || per_seq_s < 0) return fail(EMU_ERR_INVALID, "per_token_s and per_seq_s must be >= 0");
  if (prefill_multiplier < 1.0) return fail(EMU_ERR_INVALID, "prefill_multiplier must be >= 1");
  if (noise_cv < 0) return fail(EMU_ERR_INVALID, "noise_cv must be >= 0");
  cudaStream_t s = as_stream(stream);
  int rc = sched_reset(sc, s);
  if (rc) return rc;
  sc->a.gt_base = base_s;
  sc->a.gt_tok = per_token_s;
  sc->a.gt_seq = per_seq_s;
  sc->a.gt_mult = prefill_multiplier;
  sc->a.gt_cv = noise_cv;
  sc->a.seed = seed;
  if ((rc = launch_sched(sc, 1, s))) return rc;
  EMU_CUDA(cudaStreamSynchronize(s));
  return EMU_OK;
}

int emu_oracle_prefetch(emu_oracle_t o, const int32_t* q_tt, const int32_t* q_conc, const uint8_t* q_phase, int64_t n,
                        void* stream);

int emu_sched_run_oracle(emu_sched_t sc, emu_oracle_t o, const uint64_t* pcg_states, int64_t* rounds_out,
                         void* stream) {
  if (!sc || !o || !pcg_states) return fail(EMU_ERR_INVALID, "NULL scheduler/oracle/states");
  cudaStream_t s = as_stream(stream);
  int rc = sched_reset(sc, s);
  if (rc) return rc;
  const int32_t S = sc->S;
  EMU_CUDA(cudaMemcpyAsync(sc->a.pcg, pcg_states, 48 * (size_t)S, cudaMemcpyDefault, s));
  std::vector<int32_t> st((size_t)S), key((size_t)3 * S), ptt, pcc;
  std::vector<uint8_t> pph;
  int32_t *k_tt = nullptr, *k_cc = nullptr;
  uint8_t* k_ph = nullptr;
  EMU_CUDA(cudaMalloc(&k_tt, 4 * (size_t)S));
  EMU_CUDA(cudaMalloc(&k_cc, 4 * (size_t)S));
  EMU_CUDA(cudaMalloc(&k_ph, (size_t)S));
  int64_t rounds = 0;
  for (;;) {
    rounds++;
    if ((rc = oracle_views(o, &sc->a.map, &sc->a.arena, &sc->a.s0, &sc->a.s1))) break;
    if ((rc = launch_sched(sc, 2, s))) break;
    if (cudaMemcpyAsync(st.data(), sc->a.status, 4 * (size_t)S, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(key.data(), sc->a.key, 12 * (size_t)S, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "k_sched");
      break;
    }
    ptt.clear();
    pcc.clear();
    pph.clear();
    for (int32_t i = 0; i < S; i++)
      if (st[i] == SC_PAUSED) {
        ptt.push_back(key[3 * i]);
        pcc.push_back(key[3 * i + 1]);
        pph.push_back((uint8_t)key[3 * i + 2]);
      }
    if (ptt.empty()) break;
    const int64_t np = (int64_t)ptt.size();
    if (cudaMemcpyAsync(k_tt, ptt.data(), 4 * np, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(k_cc, pcc.data(), 4 * np, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(k_ph, pph.data(), np, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "pending keys");
      break;
    }
    if ((rc = emu_oracle_prefetch(o, k_tt, k_cc, k_ph, np, stream))) break;
  }
  cudaFree(k_tt);
  cudaFree(k_cc);
  cudaFree(k_ph);
  if (rounds_out) *rounds_out = rounds;
  return rc;
}

}  // extern "C"

extern "C" {

int emu_sched_keep_steps(emu_sched_t sc, int32_t keep) {
  if (!sc) return fail(EMU_ERR_INVALID, "NULL scheduler");
  sc->keep = keep != 0;
  return EMU_OK;
}

int emu_sched_summary(emu_sched_t sc, int64_t* out4) {
  if (!sc || !out4) return fail(EMU_ERR_INVALID, "NULL scheduler/output");
  const size_t S = (size_t)sc->S;
  std::vector<int64_t> v(4 * S);
  EMU_CUDA(cudaMemcpy(v.data(), sc->a.nsteps, 8 * S, cudaMemcpyDeviceToHost));
  EMU_CUDA(cudaMemcpy(v.data() + S, sc->a.tot_tok, 8 * S, cudaMemcpyDeviceToHost));
  EMU_CUDA(cudaMemcpy(v.data() + 2 * S, sc->a.tot_fin, 8 * S, cudaMemcpyDeviceToHost));
  EMU_CUDA(cudaMemcpy(v.data() + 3 * S, sc->a.preempt, 8 * S, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < S; s++)
    for (int k = 0; k < 4; k++) out4[4 * s + k] = v[k * S + s];
  return EMU_OK;
}

int emu_sched_results(emu_sched_t sc, int64_t* n_steps, int32_t* status, int32_t* tt, int32_t* conc, uint8_t* phase,
                      double* lat, int32_t* tokens, int32_t* finished, int64_t* preempt) {
  if (!sc) return fail(EMU_ERR_INVALID, "NULL scheduler");
  const size_t S = (size_t)sc->S, SM = S * (size_t)sc->max_steps;
  if ((tt || conc || phase || lat || tokens || finished || preempt) && !(sc->keep && sc->a.o_tt))
    return fail(EMU_ERR_INVALID, "per-step results were not kept (emu_sched_keep_steps(sc, 0) before the run)");
  if (n_steps) EMU_CUDA(cudaMemcpy(n_steps, sc->a.nsteps, 8 * S, cudaMemcpyDefault));
  if (status) EMU_CUDA(cudaMemcpy(status, sc->a.status, 4 * S, cudaMemcpyDefault));
  if (tt) EMU_CUDA(cudaMemcpy(tt, sc->a.o_tt, 4 * SM, cudaMemcpyDefault));
  if (conc) EMU_CUDA(cudaMemcpy(conc, sc->a.o_conc, 4 * SM, cudaMemcpyDefault));
  if (phase) EMU_CUDA(cudaMemcpy(phase, sc->a.o_ph, SM, cudaMemcpyDefault));
  if (lat) EMU_CUDA(cudaMemcpy(lat, sc->a.o_lat, 8 * SM, cudaMemcpyDefault));
  if (tokens) EMU_CUDA(cudaMemcpy(tokens, sc->a.o_tok, 4 * SM, cudaMemcpyDefault));
  if (finished) EMU_CUDA(cudaMemcpy(finished, sc->a.o_fin, 4 * SM, cudaMemcpyDefault));
  if (preempt) EMU_CUDA(cudaMemcpy(preempt, sc->a.o_pre, 8 * SM, cudaMemcpyDefault));
  return EMU_OK;
}

}  // extern "C"
