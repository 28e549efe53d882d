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
  uint32_t kspec;   // speculation length (doubles on success, halves on failure)
  uint32_t tmin;    // earliest admission seen in the running pass (~0u: none)
  uint32_t passes, fails, pad;
};

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// D: dims (compile time; the particle's whole state lives in registers).
// NP: adjacent particles per thread unit (2: LDG.128 / STG.128 on every row).
template <int F, int D, int NP, int MINB>
__global__ void __launch_bounds__(kSyncThreads, MINB) k_spec(KParams P, KState S0, KState S1, KCtl C,
                                                            SpecCtl* sc, uint32_t t_end, uint32_t kmax) {
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
  const uint32_t tl = t0 + K - 1;  // the only iteration whose admissions stand
  double gp[D];
#pragma unroll
  for (int a = 0; a < D; ++a) gp[a] = s_gpos[a];
  double bf = -INFINITY;
  uint32_t bi = kNoParticle, adm = 0;
  uint32_t tstop = ld_relaxed_gpu(&sc->tmin);
  const uint32_t units = (P.n + NP - 1) / NP;
  const size_t ld = P.ld;
  for (uint32_t u = blockIdx.x * blockDim.x + tid; u < units; u += gridDim.x * blockDim.x) {
    tstop = min(tstop, ld_relaxed_gpu(&sc->tmin));
    uint32_t te = min(t0 + K, tstop);  // iterations >= tstop cannot change the outcome
    if (te <= t0) break;               // the pass already failed at t0
    const uint32_t li = NP * u, g0 = P.base + li;
    double x[D][NP], v[D][NP], pb[D][NP], pbf[NP];
    bool ok[NP];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const size_t at = static_cast<size_t>(a) * ld + li;
      ldv<NP>(Si.pos + at, x[a]);
      ldv<NP>(Si.vel + at, v[a]);
      ldv<NP>(Si.pb + at, pb[a]);
    }
    ldv<NP>(Si.pbf + li, pbf);
#pragma unroll
    for (int k = 0; k < NP; ++k) ok[k] = k == 0 || li + k < P.n;
    uint32_t t = t0;
    bool bad = false;
    bool dirty = false;  // some pbest of this unit changed
    for (; t < te; ++t) {
      Fit<F> acc[NP];
#pragma unroll
      for (int a = 0; a < D; ++a) {
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const double r1 = uniform01(P, t, g0 + k, a, 0);
          const double r2 = uniform01(P, t, g0 + k, a, 1);
          v[a][k] = vel_step(P, v[a][k], x[a][k], pb[a][k], gp[a], r1, r2);
          x[a][k] = pos_step(P, x[a][k], v[a][k]);
          acc[k].add(x[a][k], a);
        }
      }
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double f = acc[k].value();
        if (!ok[k]) continue;
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
        atomicMin(&sc->tmin, t);
        tstop = t;
        break;
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
  }
  warp_publish(bc, bf, bi, adm);
  __syncthreads();
  if (warp == 0) {
    const uint32_t nq = bc.n;
    if (nq) {  // block winner of iteration tl -> grid queue (position re-read from B)
      double f = lane < nq ? bc.f[lane] : -INFINITY;
      uint32_t i = lane < nq ? bc.i[lane] : kNoParticle;
      warp_argmax(f, i);
      uint32_t slot = 0;
      if (lane == 0) slot = atomicAdd(&C.q_count[0], 1u);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (lane == 0) {
        C.q_fit[slot] = f;
        C.q_idx[slot] = i;
      }
      for (uint32_t a = lane; a < D; a += 32)
        C.q_pos[static_cast<size_t>(slot) * D + a] = So.pos[static_cast<size_t>(a) * ld + (i - P.base)];
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
  // ---- the last block resolves the pass and schedules the next one
  __threadfence();
  const uint32_t tm = ld_volatile_u32(&sc->tmin);
  if (tm < tl) {  // speculation failed at tm: re-run [t0, tm] exactly from A
    if (tid == 0) {
      C.admitted[tl] = 0;
      C.q_count[0] = 0;
      sc->K = tm - t0 + 1;
      sc->kspec = max(1u, s_ctl[3] / 2);
      sc->tmin = ~0u;
      sc->fails += 1;
      sc->passes += 1;
    }
    return;
  }
  const uint32_t nq = __ldcg(&C.q_count[0]);
  const double of = snap_fit;
  const uint32_t oi = C.snap->particle;
  double wf = of;
  uint32_t wi = oi, ws = 0;
  if (nq) {
    resolve_queue(C, 0, nq, rs, wf, wi, ws);
    for (uint32_t a = tid; a < D; a += blockDim.x)
      C.snap_pos[a] = __ldcg(&C.q_pos[static_cast<size_t>(ws) * D + a]);
  }
  for (uint32_t t = t0 + tid; t < tl; t += blockDim.x) {
    C.trace[t] = of;
    C.trace_idx[t] = oi;
  }
  if (tid == 0) {
    C.trace[tl] = wf;  // every queue entry passed fit > snapshot: the winner is adopted
    C.trace_idx[tl] = wi;
    if (nq) {
      C.snap->fit = wf;
      C.snap->particle = wi;
    }
    C.q_count[0] = 0;
    uint32_t ks = s_ctl[3];
    if (K >= ks) ks = min(2 * ks, kmax);
    const uint32_t tn = t0 + K;
    sc->t0 = tn;
    sc->parity = inplace ? par : (par ^ 1u);
    sc->kspec = ks;
    sc->K = tn < t_end ? min(ks, t_end - tn) : 0u;
    sc->tmin = ~0u;
    sc->passes += 1;
  }
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
//   * during them the thread only counts admissions (f > its view) into
//     admitted[t], and an admitted particle becomes the thread's own view of
//     the gbest (fit and position) -- no polling, no warp collectives in the
//     iteration loop;
//   * after them the warp's best pbest that beats the view (beats() order, warp
//     ballot + shuffle argmax) is published by its lane with the CAS(version
//     even->odd) protocol of async_commit, and folded into trace_key[t] at the
//     iteration it was found.
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
  for (;;) {
    uint32_t v = 0;
    if (lane == 0) v = ld_acquire_gpu(C.seq);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v & 1u) {  // a writer holds the record: back off instead of hammering its L2 line
      if (globaltimer_ns() - ts > kSpinTimeoutNs) __trap();
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
      uint32_t tfound = 0;  // iteration of this thread's latest admission
      for (uint32_t t = tb; t < te; ++t) {
        Fit<F> acc[NP];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const double r1 = uniform01(P, t, g0 + k, a, 0);
            const double r2 = uniform01(P, t, g0 + k, a, 1);
            v[a][k] = vel_step(P, v[a][k], x[a][k], pb[a][k], gp[a], r1, r2);
            x[a][k] = pos_step(P, x[a][k], v[a][k]);
            acc[k].add(x[a][k], a);
          }
        }
        uint32_t adm = 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          const double f = acc[k].value();
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
        if (adm) {  // rare after warm-up; one atomic per warp
          const unsigned m = __activemask();
          const uint32_t wadm = __reduce_add_sync(m, adm);
          if (lane == static_cast<uint32_t>(__ffs(m) - 1))
            atomicAdd(&C.admitted[t], static_cast<unsigned long long>(wadm));
          tfound = t;
        }
      }
      // Publish: the unit's pbests that beat the view are gbest candidates
      // (the gbest is the max of all pbests); the warp's best in beats()
      // order goes to the live record once per unit instead of per iteration.
      double bf = -INFINITY;
      uint32_t bi = kNoParticle, bk = 0;
      const double view = slot[0];  // the unit's starting view (gfit may hold own finds)
#pragma unroll
      for (int k = 0; k < NP; ++k)
        if (ok[k] && pbf[k] > view && beats(pbf[k], g0 + k, bf, bi)) {
          bf = pbf[k];
          bi = g0 + k;
          bk = k;
        }
      if (__any_sync(0xffffffffu, bi != kNoParticle)) {
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
          atomicMax(&C.trace_key[tfound], order_key(seen));
        }
        __syncwarp();
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

}  // namespace cupso
