// cupso_spec.cuh -- speculative temporal blocking for the synchronous variant.
//
// In run_serial (engine_serial.hpp:26-39) iteration t moves every particle
// against the gbest snapshot taken at the start of t; the snapshot changes
// only when some particle's new fitness beats it (engine_queue.hpp:91). After
// the first few iterations that is rare (admission
// is ~0.002 % of particle-iterations; the BASELINE shapes see 0-7 gbest changes
// in hundreds of iterations). So for K consecutive iterations the particles
// are independent, and each thread can keep its particles in registers for
// all K of them: one HBM read and one write of the state per K iterations
// instead of per iteration, and no grid barrier at all.
//
// A pass speculates that the snapshot stays fixed over [t0, t0+K):
//   * state is read from buffer A and written to buffer B (A stays intact);
//   * a particle admitted at t < t0+K-1 falsifies the speculation: its thread
//     lowers spec.tmin to t with atomicMin; every thread re-reads tmin between
//     particles (and every 16 iterations) and stops at it, because iterations
//     past the earliest admission are computed against a stale snapshot;
//   * admissions at the last iteration t0+K-1 are legitimate: block winners go
//     to the grid queue exactly as in k_wave.
// The last block to finish resolves the pass:
//   * tmin < t0+K-1: discard B and re-run [t0, tmin] from A (K = tmin-t0+1).
//     That re-run is exact by construction -- nothing is admitted before tmin
//     -- and it resolves the admissions at tmin through the queue;
//   * otherwise: commit (swap A/B), trace[t0..t0+K-2] = the snapshot,
//     trace[t0+K-1] = the queue winner if any, and the next pass starts.
// Every particle still performs every iteration with its own (t, particle,
// axis) Philox draws in the reference's operation order, so the trajectory --
// trace, gbest index, final swarm state -- is bit-identical to run_serial.
// The pass schedule lives on the device (SpecCtl), so the host only launches
// passes and reads the control word back when its estimate runs out.
#pragma once

#include "cupso_kernels.cuh"

namespace cupso {

struct SpecCtl {
  uint32_t t0;      // first iteration of the next pass
  uint32_t K;       // its length
  uint32_t parity;  // 0: state in S0, 1: state in S1
  uint32_t kspec;   // speculation length (doubles after a quiet pass, halves on failure)
  uint32_t tmin;    // earliest admission seen in the running pass (~0u: none)
  uint32_t passes, fails, pad;
};

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// A shard's summary of one pass (multi-GPU: all-gathered between ranks):
// earliest admission seen, and the best candidate of the last iteration.
struct SpecRec {
  uint32_t tmin;      // ~0u: no admission before the last iteration
  uint32_t admitted;  // admissions at the last iteration
  double fit;         // best candidate of the last iteration (-inf / kNoParticle: none)
  uint32_t particle;
  uint32_t pad;
  // followed by pos[d]
};
__host__ __device__ constexpr size_t spec_rec_bytes(uint32_t d) { return sizeof(SpecRec) + 8ull * d; }

// The decision after a pass, identical on every rank (one block): the pass
// failed if any shard saw an admission before its last iteration -> re-run
// [t0, tmin] exactly; otherwise commit it: trace, snapshot (beats() among the
// shards' candidates, each of which already beat the snapshot), occupancy, and
// the next pass's schedule.
__device__ void spec_decide(const KParams& P, const KCtl& C, SpecCtl* sc, const unsigned char* recs, uint32_t nrec,
                            uint32_t t_end, uint32_t kmax) {
  __shared__ uint32_t s_t0, s_K, s_fail;
  __shared__ int s_w;
  __shared__ double s_of;
  __shared__ uint32_t s_oi;
  const uint32_t tid = threadIdx.x;
  const size_t rb = spec_rec_bytes(P.d);
  if (tid == 0) {
    const uint32_t t0 = ld_volatile_u32(&sc->t0), K = ld_volatile_u32(&sc->K);
    const uint32_t par = ld_volatile_u32(&sc->parity), ks0 = ld_volatile_u32(&sc->kspec);
    s_t0 = t0;
    s_K = K;
    s_fail = 0;
    s_w = -1;
    if (t0 < t_end) {
      const uint32_t tl = t0 + K - 1;
      uint32_t tm = ~0u;
      double bf = -INFINITY;
      uint32_t bi = kNoParticle;
      unsigned long long adm = 0;
      int w = -1;
      for (uint32_t r = 0; r < nrec; ++r) {
        const SpecRec* rec = reinterpret_cast<const SpecRec*>(recs + r * rb);
        tm = min(tm, rec->tmin);
        adm += rec->admitted;
        if (rec->particle != kNoParticle && beats(rec->fit, rec->particle, bf, bi)) {
          bf = rec->fit;
          bi = rec->particle;
          w = static_cast<int>(r);
        }
      }
      s_of = C.snap->fit;
      s_oi = C.snap->particle;
      if (tm < tl) {  // speculation failed at tm: re-run [t0, tm] exactly from A
        s_fail = 1;
        sc->K = tm - t0 + 1;
        sc->kspec = max(1u, ks0 / 2);
        sc->fails += 1;
      } else {
        s_w = w;  // every candidate passed fit > snapshot: the winner is adopted
        C.trace[tl] = w >= 0 ? bf : s_of;
        C.trace_idx[tl] = w >= 0 ? bi : s_oi;
        C.admitted[tl] = adm;
        if (w >= 0) {
          C.snap->fit = bf;
          C.snap->particle = bi;
        }
        // grow the speculation only after a pass whose last iteration left the
        // gbest alone: while it keeps moving every iteration (cfg5's first
        // iterations) a longer pass would just be falsified at its first one
        uint32_t ks = ks0;
        if (K >= ks && w < 0) ks = min(2 * ks, kmax);
        const uint32_t tn = t0 + K;
        sc->t0 = tn;
        sc->parity = K == 1 ? par : (par ^ 1u);
        sc->kspec = ks;
        sc->K = tn < t_end ? min(ks, t_end - tn) : 0u;
      }
      sc->tmin = ~0u;
      sc->passes += 1;
    } else {
      s_fail = 1;  // no pass ran: nothing to record
    }
  }
  __syncthreads();
  if (s_fail) return;
  const uint32_t t0 = s_t0, tl = s_t0 + s_K - 1;
  for (uint32_t t = t0 + tid; t < tl; t += blockDim.x) {
    C.trace[t] = s_of;
    C.trace_idx[t] = s_oi;
  }
  if (s_w >= 0) {
    const double* rpos = reinterpret_cast<const double*>(recs + s_w * rb + sizeof(SpecRec));
    for (uint32_t a = tid; a < P.d; a += blockDim.x) C.snap_pos[a] = rpos[a];
  }
}

// Sharded passes: the decision over the all-gathered records (one block).
__global__ void k_spec_commit(KParams P, KCtl C, SpecCtl* sc, const unsigned char* recs, uint32_t nrec,
                              uint32_t t_end, uint32_t kmax) {
  spec_decide(P, C, sc, recs, nrec, t_end, kmax);
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The pass-record all-gather over peer memory, run by the last block of every
// shard's k_spec (one block per rank): push this rank's record into slot
// p2p_rank of every rank's mailbox, publish exchange number e to each rank's
// flag[p2p_rank] (release, system scope: peers read it over NVLink), then wait
// until every rank's flag in the local array reached e. All ranks perform the
// same sequence of exchanges, so e (a local counter) agrees across ranks.
// Mailboxes are double-buffered by exchange parity: a rank can write its next
// record before a slower rank has read this one, but not the one after (that
// needs the slower rank's next flag).
__device__ const unsigned char* spec_exchange_p2p(const KParams& P, const KCtl& C, const unsigned char* rec) {
  __shared__ uint32_t s_e;
  const uint32_t tid = threadIdx.x, n = C.p2p_n, me = C.p2p_rank;
  const size_t rb = spec_rec_bytes(P.d);
  uint32_t* own = C.flag[me];
  if (tid == 0) {
    s_e = own[n] + 1u;  // this rank's exchange counter
    own[n] = s_e;
  }
  __syncthreads();
  const uint32_t e = s_e;
  const size_t half = (e & 1u) * n * rb;
  for (uint32_t r = 0; r < n; ++r)  // 8-byte words of the record to every rank (rb % 8 == 0)
    for (uint32_t w = tid; w < rb / 8; w += blockDim.x)
      reinterpret_cast<unsigned long long*>(C.mbox[r] + half + me * rb)[w] =
          reinterpret_cast<const unsigned long long*>(rec)[w];
  __threadfence_system();
  __syncthreads();
  if (tid < n) st_release_sys(C.flag[tid] + me, e);
  if (tid == 0) {
    const uint64_t ts = globaltimer_ns();
    for (uint32_t q = 0; q < n; ++q)
      while (ld_acquire_sys(own + q) < e)
        if (globaltimer_ns() - ts > kSpinTimeoutNs) __trap();
    __threadfence_system();
  }
  __syncthreads();
  return C.mbox[me] + half;
}

// End of a pass (every block): block winner of the last iteration to the grid
// queue; the last block to finish reduces the queue to this shard's SpecRec
// (rec_out) and -- unless the pass is sharded (the host all-gathers the
// records and runs k_spec_commit) -- takes the decision itself.
template <int D>
__device__ __forceinline__ void spec_finish(const KParams& P, const KState& So, const KCtl& C, SpecCtl* sc,
                                            const uint32_t* s_ctl, BlockCand& bc, ResolveSmem& rs, int& s_last,
                                            uint32_t t_end, uint32_t kmax, double snap_fit, double bf,
                                            uint32_t bi, uint32_t adm, unsigned char* rec_out, int sharded) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t t0 = s_ctl[0], K = s_ctl[1];
  const uint32_t tl = t0 + K - 1;
  const size_t ld = P.ld;
  warp_publish(bc, bf, bi, adm);
  __syncthreads();
  if (warp == 0) {
    const uint32_t nq = bc.n;
    if (nq) {  // block winner of iteration tl -> grid queue (position re-read from B)
      double f = lane < nq ? bc.f[lane] : -INFINITY;
      uint32_t i = lane < nq ? bc.i[lane] : kNoParticle;
      warp_argmax(f, i);
      uint32_t slot = 0;
      if (lane == 0) slot = queue_append(&C.q_count[0]);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (lane == 0) {
        C.q_fit[slot] = f;
        C.q_idx[slot] = i;
      }
      for (uint32_t a = lane; a < P.d; a += 32)
        C.q_pos[static_cast<size_t>(slot) * P.d + a] = So.pos[static_cast<size_t>(a) * ld + (i - P.base)];
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      if (bc.adm) atomicAdd(&C.admitted[tl], bc.adm);
      s_last = last_block_done(C);
    }
  }
  __syncthreads();
  if (!s_last) return;
  // ---- the last block: this shard's record of the pass
  __threadfence();
  const uint32_t nq = __ldcg(&C.q_count[0]);
  double wf = -INFINITY;
  uint32_t wi = kNoParticle, ws = 0;
  if (nq) resolve_queue(C, 0, nq, rs, wf, wi, ws);
  SpecRec* rec = reinterpret_cast<SpecRec*>(rec_out);
  double* rpos = reinterpret_cast<double*>(rec_out + sizeof(SpecRec));
  for (uint32_t a = tid; a < P.d; a += blockDim.x)
    rpos[a] = nq ? __ldcg(&C.q_pos[static_cast<size_t>(ws) * P.d + a]) : 0.0;
  if (tid == 0) {
    rec->tmin = ld_volatile_u32(&sc->tmin);
    rec->admitted = static_cast<uint32_t>(__ldcg(&C.admitted[tl]));
    rec->fit = wf;
    rec->particle = nq ? wi : kNoParticle;
    rec->pad = 0;
    C.admitted[tl] = 0;  // the decision writes the total over shards
    C.q_count[0] = 0;
    __threadfence();
  }
  __syncthreads();
  if (sharded && C.p2p_n) {  // the exchange itself, fused into the pass (peer memory)
    const unsigned char* all = spec_exchange_p2p(P, C, rec_out);
    spec_decide(P, C, sc, all, C.p2p_n, t_end, kmax);
  } else if (!sharded) {
    spec_decide(P, C, sc, rec_out, 1, t_end, kmax);
  }
}

// One thread unit of a pass: NP adjacent particles from li, K iterations in
// registers against the snapshot (the iteration loop of k_spec). Returns false
// when the pass has already failed at t0 (nothing left to compute).
template <int F, int D, int NP>
__device__ __forceinline__ bool spec_unit(const KParams& P, const KState& Si, const KState& So, const KCtl& C,
                                          SpecCtl* sc, uint32_t li, uint32_t t0, uint32_t K, bool inplace,
                                          double snap_fit, const double (&gp)[D], uint32_t& tstop, double& bf,
                                          uint32_t& bi, uint32_t& adm) {
  const uint32_t tl = t0 + K - 1;  // the only iteration whose admissions stand
  const size_t ld = P.ld;
  tstop = min(tstop, ld_relaxed_gpu(&sc->tmin));
  uint32_t te = min(t0 + K, tstop);  // iterations >= tstop cannot change the outcome
  if (te <= t0) return false;        // the pass already failed at t0
  const uint32_t g0 = P.base + li;
  double x[D][NP], v[D][NP], pb[D][NP], pbf[NP];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const size_t at = static_cast<size_t>(a) * ld + li;
    ldv<NP>(Si.pos + at, x[a]);
    ldv<NP>(Si.vel + at, v[a]);
    ldv<NP>(Si.pb + at, pb[a]);
  }
  ldv<NP>(Si.pbf + li, pbf);
  // a slot past the swarm's end (the last unit's padding) gets pbest_fit +inf:
  // it never improves, so the per-iteration fast-path test needs no validity
  // mask (the padding's pbest_fit is never read as a particle's)
#pragma unroll
  for (int k = 1; k < NP; ++k)
    if (li + k >= P.n) pbf[k] = INFINITY;
  uint32_t t = t0;
  bool bad = false;
  bool dirty = false;  // some pbest of this unit changed
  for (; t < te; ++t) {
    Fit<F> acc[NP];
#pragma unroll
    for (int a = 0; a < D; ++a) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double r1 = uniform53(P, t, g0 + k, a, 0);
        const double r2 = uniform53(P, t, g0 + k, a, 1);
        v[a][k] = vel_step53(P, v[a][k], x[a][k], pb[a][k], gp[a], r1, r2);
        x[a][k] = pos_step(P, x[a][k], v[a][k]);
        if (a == 0)
          acc[k].add_first(x[a][k]);  // unrolled: a is a constant
        else
          acc[k].add(x[a][k], a);
      }
    }
    // Fast path: no particle improved its pbest. The snapshot is the max of
    // the pbests when the pass starts and an admission before the last
    // iteration ends it, so f > snapshot implies f > pbest: one compare per
    // particle decides the common case (nothing to do) in a single branch.
    double fv[NP];
    bool any = false;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      fv[k] = acc[k].value();
      any |= fv[k] > pbf[k];
    }
    if (any) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double f = fv[k];
        if (k > 0 && li + k >= P.n) continue;  // padding slot
        if (f > pbf[k]) {  // update_pbest (swarm.hpp:100-108)
          dirty = true;
          pbf[k] = f;
#pragma unroll
          for (int a = 0; a < D; ++a) pb[a][k] = x[a][k];
        }
        if (f > snap_fit) {  // snapshot filter (engine_queue.hpp:91)
          if (t < tl) {
            bad = true;
          } else {
            ++adm;
            if (beats(f, g0 + k, bf, bi)) {
              bf = f;
              bi = g0 + k;
            }
          }
        }
      }
      if (bad) {
        spec_falsify(C, &sc->tmin, t);
        tstop = t;
        break;
      }
    }
    if (((t - t0) & 15u) == 15u) {
      tstop = min(tstop, ld_relaxed_gpu(&sc->tmin));
      te = min(te, tstop);
    }
  }
  if (!bad && t == t0 + K) {  // completed the pass: commit this unit to B
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const size_t at = static_cast<size_t>(a) * ld + li;
      stv<NP>(So.pos + at, x[a]);
      stv<NP>(So.vel + at, v[a]);
    }
    if (!inplace || dirty) {
#pragma unroll
      for (int a = 0; a < D; ++a) stv<NP>(So.pb + static_cast<size_t>(a) * ld + li, pb[a]);
      stv<NP>(So.pbf + li, pbf);
    }
  }
  return true;
}

// D: dims (compile time; the particle's whole state lives in registers).
// NP: adjacent particles per thread unit (2: LDG.128 / STG.128 on every row).
template <int F, int D, int NP, int MINB>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_spec(KParams P, KState S0, KState S1, KCtl C,
                                                            SpecCtl* sc, uint32_t t_end, uint32_t kmax,
                                                            unsigned char* rec_out, int sharded) {
  __shared__ double s_gpos[D];
  __shared__ BlockCand bc;
  __shared__ ResolveSmem rs;
  __shared__ uint32_t s_ctl[4];
  __shared__ int s_last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_ctl[0] = ld_volatile_u32(&sc->t0);
    s_ctl[1] = ld_volatile_u32(&sc->K);
    s_ctl[2] = ld_volatile_u32(&sc->parity);
    s_ctl[3] = ld_volatile_u32(&sc->kspec);
    bc.n = 0;
    bc.adm = 0;
  }
  if (tid < D) s_gpos[tid] = C.snap_pos[tid];
  __syncthreads();
  const uint32_t t0 = s_ctl[0], K = s_ctl[1], par = s_ctl[2];
  if (t0 >= t_end) return;  // the schedule finished in an earlier launch
  // A one-iteration pass cannot be falsified (its only iteration is the last),
  // so it updates A in place like k_wave: x and v stored, pbest only when it
  // changed -- (5d+1)*8 B per particle-update instead of (6d+2)*8.
  const bool inplace = K == 1;
  const KState Si = par ? S1 : S0;
  const KState So = inplace ? Si : (par ? S0 : S1);
  const double snap_fit = C.snap->fit;
  double gp[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gp[a] = s_gpos[a];
  double bf = -INFINITY;
  uint32_t bi = kNoParticle, adm = 0;
  uint32_t tstop = ld_relaxed_gpu(&sc->tmin);
  // Rounds of NP-particle units over the grid; when the last round would be
  // at most half full, its particles go to one round of NP/2-particle units
  // instead, so every thread finishes after the same work (2^20 d = 1 on 148
  // SMs x 512 threads: 3.46 rounds of 4 -> 3 rounds of 4 + 1 of 2).
  const uint32_t nthr = gridDim.x * blockDim.x, gt = blockIdx.x * blockDim.x + tid;
  constexpr bool kTail = NP >= 2 && (NP / 2 == 1 || (NP / 2) % 2 == 0);  // ldv: 1 or even
  uint32_t n_main = P.n;
  if constexpr (kTail) {
    const uint32_t per_round = NP * nthr;
    const uint32_t rem = P.n % per_round;
    if (rem && rem <= (NP / 2) * nthr) n_main = P.n - rem;
  }
  const uint32_t units = (n_main + NP - 1) / NP;
  bool live = true;
  for (uint32_t u = gt; u < units; u += nthr) {
    if (!(live = spec_unit<F, D, NP>(P, Si, So, C, sc, NP * u, t0, K, inplace, snap_fit, gp, tstop, bf, bi, adm)))
      break;
  }
  if constexpr (kTail) {
    const uint32_t li = n_main + (NP / 2) * gt;
    if (live && li < P.n)
      spec_unit<F, D, NP / 2>(P, Si, So, C, sc, li, t0, K, inplace, snap_fit, gp, tstop, bf, bi, adm);
  }
  spec_finish<D>(P, So, C, sc, s_ctl, bc, rs, s_last, t_end, kmax, snap_fit, bf, bi, adm, rec_out, sharded);
}

// ------------------------------------------------ k_spec for wide swarms
// tmin as one value for the whole warp (loop bounds of the split kernels must
// stay warp-uniform: their lanes meet in shuffles every iteration).
__device__ __forceinline__ uint32_t warp_tmin(const uint32_t* tmin) {
  uint32_t m = 0;
  if ((threadIdx.x & 31u) == 0) m = ld_relaxed_gpu(tmin);
  return __shfl_sync(0xffffffffu, m, 0);
}

// d = DL * G: a particle is owned by G consecutive lanes, lane s of the group
// holding axes [s*DL, s*DL + DL) in registers (cfg4: d = 32 = 8 x 4). Per
// iteration every lane computes its axes' Philox draws, kinematics and
// fitness terms (Fit<F>::term -- the cos of rastrigin/griewank included) in
// parallel; the accumulator then travels up the group (shfl_up) and each lane
// folds its terms in turn, so the sum keeps the reference's axis order bit for
// bit. The fitness is broadcast from the group's last lane and every lane
// makes the same pbest / snapshot decisions; lane 0 of the group speaks for
// the particle (admissions, candidates). Warps stay converged (partial groups
// at the swarm's end compute neutral state), so every shuffle is full-mask.
// SM: keep each lane's x / v / pbest columns and its fitness terms in shared
// memory (a private column per thread, stride blockDim: conflict-free) instead
// of registers -- fewer live registers, so more resident warps and no spills
// for the cos-heavy fitnesses; dynamic SMEM = (3 + term width) * DL * blockDim
// doubles.
// RAGGED: the swarm's d is below DL * G (any d up to 256): lane s holds axes
// [s*dl, s*dl + dl), dl = ceil(d / G) <= DL, and skips the slots past d
// (warp-uniform tests).
// PBSM = 1: only the pbest columns live in shared memory (DL * blockDim
// doubles): read once per axis-iteration (one LDS), written on the rare
// improvement. PBSM = 2: the velocity columns too (one LDS + one STS more).
template <int F, int DL, int G, int MINB, bool SM = false, bool RAGGED = false, int PBSM = 0>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_spec_split(KParams P, KState S0, KState S1, KCtl C,
                                                                  SpecCtl* sc, uint32_t t_end, uint32_t kmax,
                                                                  unsigned char* rec_out, int sharded) {
  constexpr int D = DL * G;
  static_assert(!(SM && RAGGED), "the SMEM-state split kernel needs d == DL * G");
  static_assert(!(SM && PBSM), "PBSM keeps only the pbest columns in SMEM");
  extern __shared__ double s_state[];
  static_assert(32 % G == 0, "G must divide the warp");
  __shared__ double s_gpos[D];
  __shared__ BlockCand bc;
  __shared__ ResolveSmem rs;
  __shared__ uint32_t s_ctl[4];
  __shared__ int s_last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t sub = lane % G;
  if (tid == 0) {
    s_ctl[0] = ld_volatile_u32(&sc->t0);
    s_ctl[1] = ld_volatile_u32(&sc->K);
    s_ctl[2] = ld_volatile_u32(&sc->parity);
    s_ctl[3] = ld_volatile_u32(&sc->kspec);
    bc.n = 0;
    bc.adm = 0;
  }
  for (uint32_t a = tid; a < D; a += blockDim.x) s_gpos[a] = a < P.d ? C.snap_pos[a] : 0.0;
  __syncthreads();
  const uint32_t t0 = s_ctl[0], K = s_ctl[1], par = s_ctl[2];
  if (t0 >= t_end) return;
  const bool inplace = K == 1;
  // RAGGED: the d axes spread evenly over the G lanes, ceil(d / G) <= DL each
  // (d = 12: 6 + 6 instead of 8 + 4 -- the slowest lane sets the pace)
  const uint32_t dl = RAGGED ? (P.d + G - 1) / G : DL;
  auto valid = [&](int a) { return !RAGGED || (static_cast<uint32_t>(a) < dl && sub * dl + a < P.d); };
  const KState Si = par ? S1 : S0;
  const KState So = inplace ? Si : (par ? S0 : S1);
  const double snap_fit = C.snap->fit;
  const uint32_t tl = t0 + K - 1;
  const uint32_t a0 = sub * dl;  // first axis of this lane
  // the gbest position is read from SMEM at each use (broadcast LDS): holding
  // its 8 doubles in registers cost spills (cfg4: 2.7 % slower)
  double bf = -INFINITY;
  uint32_t bi = kNoParticle, adm = 0;
  uint32_t tstop = warp_tmin(&sc->tmin);
  const uint32_t per_warp = 32 / G;
  const uint32_t stride = gridDim.x * (blockDim.x / G);
  const size_t ld = P.ld;
  // warp-uniform particle loop: particle = u0 + lane / G
  for (uint32_t u0 = (blockIdx.x * blockDim.x + (tid & ~31u)) / G; u0 < P.n; u0 += stride) {
    tstop = min(tstop, warp_tmin(&sc->tmin));
    uint32_t te = min(t0 + K, tstop);
    if (te <= t0) break;  // warp-uniform: one load serves the warp
    const uint32_t li = u0 + lane / G;
    const bool live = li < P.n;
    const uint32_t gi = P.base + li;
    double rx[SM ? 1 : DL], rv[SM || PBSM >= 2 ? 1 : DL], rpb[SM || PBSM ? 1 : DL], pbf = -INFINITY;
    const uint32_t bd = blockDim.x;
    auto X = [&](int a) -> double& {
      if constexpr (SM) return s_state[(0 * DL + a) * bd + tid]; else return rx[a];
    };
    auto V = [&](int a) -> double& {
      if constexpr (SM) return s_state[(1 * DL + a) * bd + tid];
      else if constexpr (PBSM >= 2) return s_state[(DL + a) * bd + tid];
      else return rv[a];
    };
    auto PB = [&](int a) -> double& {
      if constexpr (SM) return s_state[(2 * DL + a) * bd + tid];
      else if constexpr (PBSM) return s_state[a * bd + tid];
      else return rpb[a];
    };
    if (live) {
#pragma unroll
      for (int a = 0; a < DL; ++a) {
        if (!valid(a)) {
          X(a) = V(a) = PB(a) = 0.0;
          continue;
        }
        const size_t at = static_cast<size_t>(a0 + a) * ld + li;
        X(a) = Si.pos[at];
        V(a) = Si.vel[at];
        PB(a) = Si.pb[at];
      }
      pbf = Si.pbf[li];
    } else {
#pragma unroll
      for (int a = 0; a < DL; ++a) X(a) = V(a) = PB(a) = 0.0;
    }
    uint32_t t = t0;
    bool bad = false, dirty = false;
    for (; t < te; ++t) {
      Fit<F> acc;
      if constexpr (SM) {
        // axes one (two) at a time: x/v/pbest and the terms stay in SMEM, so
        // only ~2 axes' Philox chains are live -> no spills at 3-4 blocks/SM
        using Term = typename Fit<F>::Term;
        constexpr int TW = (sizeof(Term) + 7) / 8;
        double* tcol = s_state + (3 * DL) * bd + tid;  // TW * DL doubles, stride bd
#pragma unroll 2
        for (int a = 0; a < DL; ++a) {
          const double r1 = uniform53(P, t, gi, a0 + a, 0);
          const double r2 = uniform53(P, t, gi, a0 + a, 1);
          const double x0 = X(a);
          const double nv = vel_step53(P, V(a), x0, PB(a), s_gpos[a0 + a], r1, r2);
          const double nx = pos_step(P, x0, nv);
          V(a) = nv;
          X(a) = nx;
          if constexpr (sizeof(Term) >= 8) {
            const Term tv = Fit<F>::term(nx, a0 + a);
            double w[TW];
            memcpy(w, &tv, sizeof(Term));
#pragma unroll
            for (int q = 0; q < TW; ++q) tcol[(a * TW + q) * bd] = w[q];
          }
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {
          if (q > 0) acc.shfl_up(0xffffffffu, G);
          if (sub == static_cast<uint32_t>(q)) {
            for (int a = 0; a < DL; ++a) {
              Term tv{};
              if constexpr (sizeof(Term) >= 8) {
                double w[TW];
#pragma unroll
                for (int z = 0; z < TW; ++z) w[z] = tcol[(a * TW + z) * bd];
                memcpy(&tv, w, sizeof(Term));
              }
              acc.accum(tv, X(a), a0 + a);
            }
          }
        }
      } else {
        typename Fit<F>::Term tm[DL];
        double xs[F == kRosenbrock ? DL : 1];  // rosenbrock's fold needs the positions
#pragma unroll
        for (int a = 0; a < DL; ++a) {
          if (!valid(a)) continue;  // ragged tail: warp-uniform per lane group
          const double r1 = uniform53(P, t, gi, a0 + a, 0);
          const double r2 = uniform53(P, t, gi, a0 + a, 1);
          const double x0 = X(a);
          const double nv = vel_step53(P, V(a), x0, PB(a), s_gpos[a0 + a], r1, r2);
          const double nx = pos_step(P, x0, nv);
          V(a) = nv;
          X(a) = nx;
          tm[a] = Fit<F>::term(nx, a0 + a);
          if constexpr (F == kRosenbrock) xs[a] = nx;
        }
        // ordered fold across the group: lane s folds after lane s-1
#pragma unroll
        for (int q = 0; q < G; ++q) {
          if (q > 0) acc.shfl_up(0xffffffffu, G);
          if (sub == static_cast<uint32_t>(q)) {
#pragma unroll
            for (int a = 0; a < DL; ++a)
              if (valid(a)) acc.accum(tm[a], F == kRosenbrock ? xs[a] : 0.0, a0 + a);
          }
        }
      }
      const double f = __shfl_sync(0xffffffffu, acc.value(), G - 1, G);
      if (live && f > pbf) {  // update_pbest (swarm.hpp:100-108)
        dirty = true;
        pbf = f;
#pragma unroll
        for (int a = 0; a < DL; ++a) PB(a) = X(a);
      }
      bool early = false;
      if (live && f > snap_fit) {  // snapshot filter (engine_queue.hpp:91)
        if (t < tl) {
          early = true;
        } else if (sub == 0) {
          ++adm;
          if (beats(f, gi, bf, bi)) {
            bf = f;
            bi = gi;
          }
        }
      }
      if (__any_sync(0xffffffffu, early)) {  // the pass is falsified at t
        if (lane == 0) spec_falsify(C, &sc->tmin, t);
        tstop = t;
        bad = true;
        break;
      }
      if (((t - t0) & 15u) == 15u) {
        tstop = min(tstop, warp_tmin(&sc->tmin));
        te = min(te, tstop);
      }
    }
    if (!bad && t == t0 + K && live) {
#pragma unroll
      for (int a = 0; a < DL; ++a) {
        if (!valid(a)) continue;
        const size_t at = static_cast<size_t>(a0 + a) * ld + li;
        So.pos[at] = X(a);
        So.vel[at] = V(a);
        if (!inplace || dirty) So.pb[at] = PB(a);
      }
      if (sub == 0 && (!inplace || dirty)) So.pbf[li] = pbf;
    }
  }
  spec_finish<D>(P, So, C, sc, s_ctl, bc, rs, s_last, t_end, kmax, snap_fit, bf, bi, adm, rec_out, sharded);
}

}  // namespace cupso

namespace cupso {

// ------------------------------------------------ async, register-resident
// The asynchronous variant needs no speculation: a particle may move against
// whatever gbest was last published, so each thread keeps its particles in
// registers for K iterations at a time (the temporal blocking of
// k_async_tiled without SMEM tiles or block barriers). Per warp and unit:
//   * before the unit's K iterations the warp takes a consistent copy of the
//     live record (seqlock: even version, unchanged after the copy; skipped
//     when the version did not move);
//   * during them the thread counts admissions (f > its view) into admitted[t],
//     and an admitted particle becomes the thread's own view of the gbest (fit
//     and position);
//   * at an iteration where some lane of the warp made a find, the warp's best
//     new pbest (beats() order, warp ballot + shuffle argmax) is published by
//     its lane with the CAS(version even->odd) protocol of async_commit and
//     folded into trace_key[t];
//   * every iteration the warp compares the live record's version (a relaxed
//     load issued before the step, so its latency hides behind the arithmetic)
//     with the one it holds and re-reads the record when it moved, so particles
//     move against the latest published gbest, as in the paper's asynchronous
//     variant, while their state stays in registers for K iterations.
// Lanes past the end of the swarm run the loop with neutral state so every
// warp-collective sees all 32 lanes.
// Out-of-line slow paths of k_async_reg: keeping them out of the iteration
// loop keeps the loop body inside the instruction cache (inlined, they made
// the d=1 loop ~7x slower with no call ever taken after warm-up).
//
// Warp-collective: copy a consistent (even, unchanged) version of the live
// record into the warp's SMEM slot; returns the version read.
__device__ __noinline__ uint32_t areg_refresh(const KCtl& C, uint32_t d, uint32_t gver, double* slot,
                                             uint64_t ts) {
  const uint32_t lane = threadIdx.x & 31;
  (void)ts;
  uint64_t spin0 = 0;  // the timeout counts from the first wait, not from the kernel's start
  for (;;) {
    uint32_t v = 0;
    if (lane == 0) v = ld_acquire_gpu(C.seq);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v & 1u) {  // a writer holds the record: back off instead of hammering its L2 line
      const uint64_t now = globaltimer_ns();
      if (!spin0) spin0 = now;
      else if (now - spin0 > kSpinTimeoutNs) __trap();
      __nanosleep(200);
      continue;
    }
    if (v == gver) return v;
    __syncwarp();
    if (lane == 0) slot[0] = __ldcg(&C.live->fit);
    for (uint32_t a = lane; a < d; a += 32) slot[1 + a] = __ldcg(&C.live_pos[a]);
    __threadfence();
    uint32_t v2 = 0;
    if (lane == 0) v2 = ld_acquire_gpu(C.seq);
    v2 = __shfl_sync(0xffffffffu, v2, 0);
    __syncwarp();
    if (v2 == v) return v;
  }
}

// One lane: publish (wf, wi, pos[0..d)) into the live record if it still
// beats it (lock-free pre-check, CAS(version even->odd), re-check, write,
// release version+2). Returns the best fitness this lane knows afterwards.
__device__ __noinline__ double areg_publish(const KCtl& C, uint32_t d, double wf, uint32_t wi, const double* pos,
                                            double view) {
  const double lf0 = ld_acquire_gpu_f64(&C.live->fit);
  view = lf0 > view ? lf0 : view;
  if (!may_beat(C.live, wf, wi)) return view;
  const uint64_t tl = globaltimer_ns();
  uint32_t sv;
  for (;;) {
    sv = ld_acquire_gpu(C.seq);
    if (!(sv & 1u) && atomicCAS(C.seq, sv, sv + 1u) == sv) break;
    // lost the race: give up as soon as the record no longer loses to us
    // (after warm-up thousands of warps publish at once; re-checking turns
    // their CAS storm on one L2 line into reads)
    if (!may_beat(C.live, wf, wi)) return view;
    if (globaltimer_ns() - tl > kSpinTimeoutNs) __trap();
    __nanosleep(100);
  }
  __threadfence();
  const double lf = __ldcg(&C.live->fit);
  const uint32_t lp = __ldcg(&C.live->particle);
  if (beats(wf, wi, lf, lp)) {
    for (uint32_t a = 0; a < d; ++a) C.live_pos[a] = pos[a];
    write_rec(C.live, wf, wi);
    view = wf;
  } else {
    view = lf > view ? lf : view;
  }
  __threadfence();
  st_release_gpu(C.seq, sv + 2u);
  return view;
}

template <int F, int D, int NP, int MINB>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_async_reg(KParams P, KState S, KCtl C, uint32_t t0,
                                                                 uint32_t t1, uint32_t K) {
  __shared__ double s_slot[kSyncWarps][1 + D];  // per warp: copy of the live record
  __shared__ double s_pub[kSyncWarps][D];       // per warp: the publisher's position
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* slot = s_slot[warp];
  const uint64_t ts = globaltimer_ns();
  double gp[D];
  double gfit;
  uint32_t gver = 0xffffffffu;
  const uint32_t units = (P.n + NP - 1) / NP;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t wbase = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  const size_t ld = P.ld;
  for (uint32_t tb = t0; tb < t1; tb += K) {
    const uint32_t te = min(tb + K, t1);
    for (uint32_t u0 = wbase; u0 < units; u0 += stride) {  // warp-uniform trip count
      // the latest published gbest for this unit's K iterations
      gver = areg_refresh(C, D, gver, slot, ts);
      gfit = slot[0];
#pragma unroll
      for (int a = 0; a < D; ++a) gp[a] = slot[1 + a];
      const uint32_t u = u0 + lane;
      const bool live = u < units;
      const uint32_t li = NP * u, g0 = P.base + li;
      double x[D][NP], v[D][NP], pb[D][NP], pbf[NP];
      bool ok[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) ok[k] = live && (k == 0 || li + k < P.n);
      if (live) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const size_t at = static_cast<size_t>(a) * ld + li;
          ldv<NP>(S.pos + at, x[a]);
          ldv<NP>(S.vel + at, v[a]);
          ldv<NP>(S.pb + at, pb[a]);
        }
        ldv<NP>(S.pbf + li, pbf);
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          pbf[k] = -INFINITY;
#pragma unroll
          for (int a = 0; a < D; ++a) x[a][k] = v[a][k] = pb[a][k] = 0.0;
        }
      }
      bool dirty = false;
      for (uint32_t t = tb; t < te; ++t) {
        // the live record's version, read now and compared after the step: the
        // load's latency hides behind the iteration's arithmetic
        uint32_t vnow = 0;
        if (lane == 0) vnow = ld_relaxed_gpu(C.seq);
        Fit<F> acc[NP];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const double r1 = uniform53(P, t, g0 + k, a, 0);
            const double r2 = uniform53(P, t, g0 + k, a, 1);
            v[a][k] = vel_step53(P, v[a][k], x[a][k], pb[a][k], gp[a], r1, r2);
            x[a][k] = pos_step(P, x[a][k], v[a][k]);
            if (a == 0)
              acc[k].add_first(x[a][k]);  // unrolled: a is a constant
            else
              acc[k].add(x[a][k], a);
          }
        }
        uint32_t adm = 0;
        // fast path as in k_spec: the view is >= every pbest of this thread,
        // so "no pbest improved" covers "nothing admitted" too
        double fv[NP];
        bool any = false;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          fv[k] = acc[k].value();
          any |= ok[k] && fv[k] > pbf[k];
        }
        if (any) {
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const double f = fv[k];
            if (!ok[k]) continue;
            if (f > pbf[k]) {  // update_pbest (swarm.hpp:100-108)
              dirty = true;
              pbf[k] = f;
#pragma unroll
              for (int a = 0; a < D; ++a) pb[a][k] = x[a][k];
            }
            if (f > gfit) {  // beats this thread's view of the gbest: it becomes the view
              ++adm;
              gfit = f;
#pragma unroll
              for (int a = 0; a < D; ++a) gp[a] = x[a][k];
            }
          }
        }
        // Publish at the iteration of the find: the warp's best new pbest
        // (beats() order, ballot + shuffle argmax) goes to the live record by
        // the CAS(version even->odd) protocol of async_commit -- a block
        // publishes only when it improved the gbest (north_star), and rarely
        // after warm-up, so the common iteration pays one ballot.
        if (__any_sync(0xffffffffu, adm != 0)) {
          const unsigned m = __ballot_sync(0xffffffffu, adm != 0);
          const uint32_t wadm = __reduce_add_sync(0xffffffffu, adm);
          if (lane == static_cast<uint32_t>(__ffs(m) - 1))
            atomicAdd(&C.admitted[t], static_cast<unsigned long long>(wadm));
          double bf = -INFINITY;
          uint32_t bi = kNoParticle, bk = 0;
          const double view = slot[0];  // the last consistent copy of the live record
#pragma unroll
          for (int k = 0; k < NP; ++k)
            if (ok[k] && pbf[k] > view && beats(pbf[k], g0 + k, bf, bi)) {
              bf = pbf[k];
              bi = g0 + k;
              bk = k;
            }
          double wf = bf;
          uint32_t wi = bi;
          warp_argmax(wf, wi);
          __syncwarp();
          if (bi == wi && bi != kNoParticle) {  // the winning lane publishes
#pragma unroll
            for (int a = 0; a < D; ++a) {
              double pa = pb[a][0];
#pragma unroll
              for (int k = 1; k < NP; ++k)
                if (bk == static_cast<uint32_t>(k)) pa = pb[a][k];
              s_pub[warp][a] = pa;
            }
            const double seen = areg_publish(C, D, wf, wi, s_pub[warp], view);
            atomicMax(&C.trace_key[t], order_key(seen));
          }
          __syncwarp();
          vnow = ~gver;  // re-read the record below (ours, or the one that beat it)
        }
        // Re-read the live record when its version moved: every particle then
        // moves against the latest published gbest at the next iteration, while
        // its state stays in registers for the whole K-iteration unit.
        vnow = __shfl_sync(0xffffffffu, vnow, 0);
        if (vnow != gver) {
          gver = areg_refresh(C, D, gver, slot, ts);
          const double lf = slot[0];
          if (!(gfit > lf)) {  // never step back from this thread's own find
            gfit = lf;
#pragma unroll
            for (int a = 0; a < D; ++a) gp[a] = slot[1 + a];
          }
        }
      }
      if (live) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const size_t at = static_cast<size_t>(a) * ld + li;
          stv<NP>(S.pos + at, x[a]);
          stv<NP>(S.vel + at, v[a]);
        }
        if (dirty) {
#pragma unroll
          for (int a = 0; a < D; ++a) stv<NP>(S.pb + static_cast<size_t>(a) * ld + li, pb[a]);
          stv<NP>(S.pbf + li, pbf);
        }
      }
    }
  }
}


// ------------------------------------------- async, register-resident, wide
// cuda-async for d above 8 (up to 256): k_spec_split's lane layout (G lanes
// per particle, DL axes per lane, the ordered shfl_up fold) with k_async_reg's
// asynchronous protocol -- K iterations per unit with the state in registers,
// a find published at its iteration by the warp's best group (CAS-seqlock),
// the live record's version checked every iteration. Dynamic SMEM: two private
// columns per lane (pbest and this particle's view of the gbest), DL x
// blockDim doubles each; the warp's consistent copy of the live record and the
// publisher's position are static.
template <int F, int DL, int G, int MINB, bool RAGGED>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_async_split(KParams P, KState S, KCtl C, uint32_t t0,
                                                                   uint32_t t1, uint32_t K) {
  constexpr int D = DL * G;
  static_assert(32 % G == 0, "G must divide the warp");
  extern __shared__ double s_cols[];  // [0, DL): pbest columns, [DL, 2 DL): view columns
  __shared__ double s_slot[kSyncWarps][1 + D];
  __shared__ double s_pub[kSyncWarps][D];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, sub = lane % G;
  const uint32_t dl = RAGGED ? (P.d + G - 1) / G : DL;  // balanced ragged split, as k_spec_split
  const uint32_t bd = blockDim.x, a0 = sub * dl;
  double* slot = s_slot[warp];
  const uint64_t ts = globaltimer_ns();
  uint32_t gver = 0xffffffffu;
  auto valid = [&](int a) { return !RAGGED || (static_cast<uint32_t>(a) < dl && a0 + a < P.d); };
  auto PB = [&](int a) -> double& { return s_cols[a * bd + tid]; };
  auto GV = [&](int a) -> double& { return s_cols[(DL + a) * bd + tid]; };
  const uint32_t stride = gridDim.x * (blockDim.x / G);
  const size_t ld = P.ld;
  for (uint32_t tb = t0; tb < t1; tb += K) {
    const uint32_t te = min(tb + K, t1);
    for (uint32_t u0 = (blockIdx.x * blockDim.x + (tid & ~31u)) / G; u0 < P.n; u0 += stride) {
      gver = areg_refresh(C, P.d, gver, slot, ts);  // the latest published gbest for this unit
      double gfit = slot[0];
#pragma unroll
      for (int a = 0; a < DL; ++a) GV(a) = valid(a) ? slot[1 + a0 + a] : 0.0;
      const uint32_t li = u0 + lane / G;
      const bool live = li < P.n;
      const uint32_t gi = P.base + li;
      double rx[DL], rv[DL], pbf = -INFINITY;
#pragma unroll
      for (int a = 0; a < DL; ++a) {
        if (!live || !valid(a)) {
          rx[a] = rv[a] = PB(a) = 0.0;
          continue;
        }
        const size_t at = static_cast<size_t>(a0 + a) * ld + li;
        rx[a] = S.pos[at];
        rv[a] = S.vel[at];
        PB(a) = S.pb[at];
      }
      if (live) pbf = S.pbf[li];
      bool dirty = false;
      for (uint32_t t = tb; t < te; ++t) {
        uint32_t vnow = 0;
        if (lane == 0) vnow = ld_relaxed_gpu(C.seq);  // consumed after the step
        Fit<F> acc;
        typename Fit<F>::Term tm[DL];
        double xs[F == kRosenbrock ? DL : 1];
#pragma unroll
        for (int a = 0; a < DL; ++a) {
          if (!valid(a)) continue;
          const double r1 = uniform53(P, t, gi, a0 + a, 0);
          const double r2 = uniform53(P, t, gi, a0 + a, 1);
          const double x0 = rx[a];
          const double nv = vel_step53(P, rv[a], x0, PB(a), GV(a), r1, r2);
          const double nx = pos_step(P, x0, nv);
          rv[a] = nv;
          rx[a] = nx;
          tm[a] = Fit<F>::term(nx, a0 + a);
          if constexpr (F == kRosenbrock) xs[a] = nx;
        }
#pragma unroll
        for (int q = 0; q < G; ++q) {  // ordered fold across the group
          if (q > 0) acc.shfl_up(0xffffffffu, G);
          if (sub == static_cast<uint32_t>(q)) {
#pragma unroll
            for (int a = 0; a < DL; ++a)
              if (valid(a)) acc.accum(tm[a], F == kRosenbrock ? xs[a] : 0.0, a0 + a);
          }
        }
        const double f = __shfl_sync(0xffffffffu, acc.value(), G - 1, G);
        if (live && f > pbf) {  // update_pbest (swarm.hpp:100-108)
          dirty = true;
          pbf = f;
#pragma unroll
          for (int a = 0; a < DL; ++a) PB(a) = rx[a];
        }
        bool find = false;
        if (live && f > gfit) {  // beats this particle's view: it becomes the view
          find = true;
          gfit = f;
#pragma unroll
          for (int a = 0; a < DL; ++a) GV(a) = rx[a];
        }
        const unsigned fm = __ballot_sync(0xffffffffu, find && sub == 0);
        if (fm) {  // publish at the iteration of the find (rare after warm-up)
          if (lane == static_cast<uint32_t>(__ffs(fm) - 1))
            atomicAdd(&C.admitted[t], static_cast<unsigned long long>(__popc(fm)));
          const double view = slot[0];  // the last consistent copy of the live record
          const bool cand = sub == 0 && live && pbf > view;
          double wf = cand ? pbf : -INFINITY;
          uint32_t wi = cand ? gi : kNoParticle;
          warp_argmax(wf, wi);
          if (wi != kNoParticle) {
            if (gi == wi) {  // the winning group's lanes stage its pbest position
#pragma unroll
              for (int a = 0; a < DL; ++a)
                if (valid(a)) s_pub[warp][a0 + a] = PB(a);
            }
            __syncwarp();
            if (gi == wi && sub == 0) {
              const double seen = areg_publish(C, P.d, wf, wi, s_pub[warp], view);
              atomicMax(&C.trace_key[t], order_key(seen));
            }
            __syncwarp();
          }
          vnow = ~gver;  // re-read the record below
        }
        vnow = __shfl_sync(0xffffffffu, vnow, 0);
        if (vnow != gver) {
          gver = areg_refresh(C, P.d, gver, slot, ts);
          const double lf = slot[0];
          if (!(gfit > lf)) {  // never step back from this particle's own find
            gfit = lf;
#pragma unroll
            for (int a = 0; a < DL; ++a) GV(a) = valid(a) ? slot[1 + a0 + a] : 0.0;
          }
        }
      }
      if (live) {
#pragma unroll
        for (int a = 0; a < DL; ++a) {
          if (!valid(a)) continue;
          const size_t at = static_cast<size_t>(a0 + a) * ld + li;
          S.pos[at] = rx[a];
          S.vel[at] = rv[a];
          if (dirty) S.pb[at] = PB(a);
        }
        if (dirty && sub == 0) S.pbf[li] = pbf;
      }
    }
  }
}

}  // namespace cupso
