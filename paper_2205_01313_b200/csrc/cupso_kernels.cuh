// cupso_kernels.cuh -- the PSO-step kernels for sm_100a.
//
// Classic per-iteration kernels (the paper's four GPU algorithms, one
// particle per thread, block = group_size, launched twice / once per
// iteration inside a CUDA graph):
//   k_classic_step<F, kTree|kTreeUnrolled>  + k_classic_fold   (reduction baseline)
//   k_classic_step<F, kQueue>               + k_classic_fold   (queue)
//   k_classic_step<F, kQueueLock>                              (queue-lock, fused)
// B200-native persistent kernels (two particles per thread, 128-bit accesses):
//   k_sync<F>   one cooperative launch for the whole run; per iteration a
//               warp-ballot filter, warp-shuffle argmax, block queue in smem,
//               a grid-level candidate queue and one grid barrier. Every block
//               resolves the (tiny) grid queue itself, so no second barrier.
//   k_async<F>  free-running blocks; the global best is a seqlock record
//               whose writers take it with a CAS on the version word.
//   k_propose<F> + k_commit: one iteration of a shard (multi-GPU exchange).
// The speculative register-resident passes that cuda-sync / cuda-async use for
// the BASELINE shapes live in cupso_spec.cuh, the FP32 engine in cupso_f32.cuh.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>

#include "cupso_device.cuh"

namespace cupso {

constexpr int kTree = 0, kTreeUnrolled = 1, kQueue = 2, kQueueLock = 3;
constexpr int kSyncThreads = 256;
constexpr int kSyncWarps = kSyncThreads / 32;

struct Rec {  // global-best record header; followed by pos[d] where stored as a record
  double fit;
  uint32_t particle;
  uint32_t admitted;
};

struct KCtl {
  Rec* snap;                      // iteration-start snapshot (read-only inside a step)
  double* snap_pos;               // [d]
  Rec* live;                      // queue-lock / async live record
  double* live_pos;               // [d]
  double* trace;                  // [T]
  uint32_t* trace_idx;            // [T]
  unsigned long long* admitted;   // [T] particles passing the snapshot filter
  unsigned long long* trace_key;  // [T] async: order-preserving max of the observed gbest
  double* aux_fit;                // [groups]
  uint32_t* aux_idx;              // [groups]
  uint32_t* lock;                 // queue-lock spin lock word
  uint32_t* ticket;               // last-block-done counter
  uint32_t* ticket_grp;           // [64] first-level counters of the hierarchical ticket
  unsigned long long* bar;        // grid barrier word (arrivals | appends << 32)
  uint32_t* seq;                  // async seqlock version
  uint32_t* q_count;              // [3] grid queue fill counters
  double* q_fit;                  // [3*cap]
  uint32_t* q_idx;                // [3*cap]
  double* q_pos;                  // [3*cap*d]
  uint32_t q_cap;
  // speculative passes of a sharded swarm: the other shards' SpecCtl.tmin
  // words (same process, or CUDA IPC over NVLink). A shard that falsifies a
  // pass lowers them too, so every shard stops early -- a hint only: the
  // decision always comes from the exchanged pass records.
  uint32_t npeers;
  uint32_t* peer_tmin[15];
  // In-kernel exchange of the pass records over peer memory (replaces the
  // all-gather + k_spec_commit when p2p_n > 0): rank r's record goes to slot r
  // of every rank's mailbox, then a release store of the exchange number to
  // that rank's flag[r]; each rank waits for all flags and decides locally.
  uint32_t p2p_n, p2p_rank;
  unsigned char* mbox[16];  // every rank's mailbox ([p2p_n] records)
  uint32_t* flag[16];       // every rank's flags ([p2p_n] exchange numbers + [1] own counter)
};

// Lower this shard's tmin and, when that was news, the peers' (rare path).
// The peer atomics execute at the owning GPU's L2 (NVLink P2P), so the
// owner's gpu-scope polls see them; polling at sys scope instead measured 2x
// slower passes (every poll leaves the GPU).
__device__ __forceinline__ void spec_falsify(const KCtl& C, uint32_t* tmin, uint32_t t) {
  if (atomicMin(tmin, t) > t)
    for (uint32_t p = 0; p < C.npeers; ++p) atomicMin_system(C.peer_tmin[p], t);
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// A spin that never returns means a co-residency bug; trap instead of hanging the GPU.
constexpr uint64_t kSpinTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_acquire_gpu_f64(const double* p) {
  double v;
  asm volatile("ld.acquire.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Lock-free pre-check of a (fit, particle) record that only grows in beats()
// order. Writers store particle, fence, then fit; reading fit with acquire and
// then particle yields a particle at least as new as the fit. If the
// candidate does not beat that pair it can never beat the live record, so
// the caller may skip the lock; otherwise it re-checks under the lock.
__device__ __forceinline__ bool may_beat(const Rec* r, double f, uint32_t i) {
  const double lf = ld_acquire_gpu_f64(&r->fit);
  const uint32_t lp = ld_relaxed_gpu(&r->particle);
  return beats(f, i, lf, lp);
}
__device__ __forceinline__ void write_rec(Rec* r, double f, uint32_t i) {
  *reinterpret_cast<volatile uint32_t*>(&r->particle) = i;
  __threadfence();
  *reinterpret_cast<volatile double*>(&r->fit) = f;
}

__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Order-preserving map double -> u64 (for the async trace max).
__device__ __forceinline__ unsigned long long order_key(double f) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(f));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// ------------------------------------------------------------------ init
// init_swarm (swarm.hpp:136-171): uniform_range draws in slots 2/3 at
// iteration 0, pbest = position, fitness evaluated. Padding lanes get a
// neutral state (zeros, pbest_fit = -inf).
template <int F>
__global__ void k_init(KParams P, KState S) {
  const double ninf = -INFINITY;
  for (uint64_t li = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; li < P.ld;
       li += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (li < P.n) {
      const uint32_t gi = P.base + static_cast<uint32_t>(li);
      Fit<F> fit;
      for (uint32_t a = 0; a < P.d; ++a) {
        const size_t at = static_cast<size_t>(a) * P.ld + li;
        const double ux = uniform01(P, 0, gi, a, 2);
        const double uv = uniform01(P, 0, gi, a, 3);
        const double x = __dadd_rn(P.min_pos, __dmul_rn(ux, __dsub_rn(P.max_pos, P.min_pos)));
        const double v = __dadd_rn(P.min_v, __dmul_rn(uv, __dsub_rn(P.max_v, P.min_v)));
        S.pos[at] = x;
        S.vel[at] = v;
        S.pb[at] = x;
        fit.add(x, a);
      }
      S.pbf[li] = fit.value();
    } else {
      for (uint32_t a = 0; a < P.d; ++a) {
        const size_t at = static_cast<size_t>(a) * P.ld + li;
        S.pos[at] = 0.0;
        S.vel[at] = 0.0;
        S.pb[at] = 0.0;
      }
      S.pbf[li] = ninf;
    }
  }
}

// Block argmax over pbest_fit (first strict max == beats order) -> aux.
__global__ void k_argmax_blocks(KParams P, const double* __restrict__ vals, double* aux_fit,
                                uint32_t* aux_idx) {
  __shared__ double sf[32];
  __shared__ uint32_t si[32];
  double f = -INFINITY;
  uint32_t i = kNoParticle;
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < P.n; li += gridDim.x * blockDim.x) {
    const double v = vals[li];
    if (beats(v, P.base + li, f, i)) {
      f = v;
      i = P.base + li;
    }
  }
  warp_argmax(f, i);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sf[warp] = f;
    si[warp] = i;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t nw = blockDim.x >> 5;
    f = lane < nw ? sf[lane] : -INFINITY;
    i = lane < nw ? si[lane] : kNoParticle;
    warp_argmax(f, i);
    if (lane == 0) {
      aux_fit[blockIdx.x] = f;
      aux_idx[blockIdx.x] = i;
    }
  }
}

// Fold aux -> initial gbest record (snapshot and live), gather position.
__global__ void k_argmax_final(KParams P, KState S, KCtl C, uint32_t nblocks) {
  __shared__ double sf[32];
  __shared__ uint32_t si[32];
  double f = -INFINITY;
  uint32_t i = kNoParticle;
  for (uint32_t k = threadIdx.x; k < nblocks; k += blockDim.x) {
    if (beats(C.aux_fit[k], C.aux_idx[k], f, i)) {
      f = C.aux_fit[k];
      i = C.aux_idx[k];
    }
  }
  warp_argmax(f, i);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sf[warp] = f;
    si[warp] = i;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t nw = blockDim.x >> 5;
    f = lane < nw ? sf[lane] : -INFINITY;
    i = lane < nw ? si[lane] : kNoParticle;
    warp_argmax(f, i);
    if (lane == 0) {
      sf[0] = f;
      si[0] = i;
    }
  }
  __syncthreads();
  f = sf[0];
  i = si[0];
  const bool adopt = f > -INFINITY;  // swarm.hpp:165 strict > against the -inf sentinel
  for (uint32_t a = threadIdx.x; a < P.d; a += blockDim.x) {
    const double x = adopt ? S.pb[static_cast<size_t>(a) * P.ld + (i - P.base)] : 0.0;
    C.snap_pos[a] = x;
    C.live_pos[a] = x;
  }
  if (threadIdx.x == 0) {
    const Rec r{adopt ? f : -INFINITY, adopt ? i : kNoParticle, 0u};
    *C.snap = r;
    *C.live = r;
  }
}

template <int F>
__global__ void k_eval(KParams P, const double* __restrict__ pos, double* out) {
  for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < P.n; li += gridDim.x * blockDim.x)
    out[li] = eval_position<F>(P, pos, li);
}

// ------------------------------------------------- classic tree helpers
// reduce_round (engine.hpp:45-55) over the padded smem arrays, looped tree.
__device__ __forceinline__ void tree_looped(double* wf, uint32_t* wi, uint32_t lane, uint32_t padded) {
  for (uint32_t stride = padded >> 1; stride >= 1; stride >>= 1) {
    if (lane < stride && beats(wf[lane + stride], wi[lane + stride], wf[lane], wi[lane])) {
      wf[lane] = wf[lane + stride];
      wi[lane] = wi[lane + stride];
    }
    __syncthreads();
  }
}

// Straight-line variant for padded in {32,64,128,256} (engine_reduction.hpp:48-76).
template <uint32_t S>
__device__ __forceinline__ void round_at(double* wf, uint32_t* wi, uint32_t lane) {
  if (lane < S && beats(wf[lane + S], wi[lane + S], wf[lane], wi[lane])) {
    wf[lane] = wf[lane + S];
    wi[lane] = wi[lane + S];
  }
  __syncthreads();
}
__device__ __forceinline__ void tree_unrolled(double* wf, uint32_t* wi, uint32_t lane, uint32_t padded) {
  switch (padded) {
    case 256: round_at<128>(wf, wi, lane); [[fallthrough]];
    case 128: round_at<64>(wf, wi, lane); [[fallthrough]];
    case 64: round_at<32>(wf, wi, lane); [[fallthrough]];
    case 32:
      round_at<16>(wf, wi, lane);
      round_at<8>(wf, wi, lane);
      round_at<4>(wf, wi, lane);
      round_at<2>(wf, wi, lane);
      round_at<1>(wf, wi, lane);
      break;
    default: tree_looped(wf, wi, lane, padded);
  }
}

// A unique slot in a block (smem) or grid (global) queue: Alg. 2 lines 1-4,
// atomic_append (group_runtime.hpp:182-187). Pinned by k_stress_append.
__device__ __forceinline__ uint32_t queue_append(uint32_t* count) { return atomicAdd(count, 1u); }

// Global spin lock (Alg. 3 atomicCAS(lock,0,1) / atomicExch(lock,0); group_runtime.hpp:190-205).
__device__ __forceinline__ void lock_acquire(uint32_t* lock) {
  const uint64_t t0 = globaltimer_ns();
  while (atomicCAS(lock, 0u, 1u) != 0u) {
    __nanosleep(32);
    if (globaltimer_ns() - t0 > kSpinTimeoutNs) __trap();
  }
  __threadfence();
}
__device__ __forceinline__ void lock_release(uint32_t* lock) {
  __threadfence();  // Alg. 3 line 5: publish the record before the release
  atomicExch(lock, 0u);
}

// ------------------------------------------------------ classic phase 1
// One particle per lane, block = group_size lanes (engine_reduction.hpp:33-36,
// engine_queue.hpp:39-58 / 86-104). Dynamic smem: padded doubles + padded u32.
template <int F, int MODE>
__global__ void k_classic_step(KParams P, KState S, KCtl C, uint32_t t, uint32_t padded) {
  extern __shared__ double smem_d[];
  double* wf = smem_d;
  uint32_t* wi = reinterpret_cast<uint32_t*>(wf + padded);
  __shared__ uint32_t s_n;
  const uint32_t lane = threadIdx.x;
  const uint32_t g = blockIdx.x;
  const uint32_t li = g * P.gs + lane;
  const bool active = li < P.n;
  if (MODE == kQueue || MODE == kQueueLock) {
    if (lane == 0) s_n = 0;
    __syncthreads();
  }
  double fit = -INFINITY;
  if (active) fit = advance_one<F>(P, S, t, li, C.snap_pos);

  if (MODE == kTree || MODE == kTreeUnrolled) {
    wf[lane] = active ? fit : -INFINITY;  // inactive lanes hold the sentinel
    wi[lane] = active ? P.base + li : kNoParticle;
    for (uint32_t pad = lane + P.gs; pad < padded; pad += P.gs) {
      wf[pad] = -INFINITY;
      wi[pad] = kNoParticle;
    }
    __syncthreads();
    if (MODE == kTreeUnrolled)
      tree_unrolled(wf, wi, lane, padded);
    else
      tree_looped(wf, wi, lane, padded);
    if (lane == 0) {
      C.aux_fit[g] = wf[0];
      C.aux_idx[g] = wi[0];
    }
  } else {
    const double snap_fit = C.snap->fit;
    if (active && fit > snap_fit) {  // Alg. 2 lines 1-4: conditional atomic append
      const uint32_t slot = queue_append(&s_n);
      wf[slot] = fit;
      wi[slot] = P.base + li;
    }
    __syncthreads();
    if (lane == 0) {
      const uint32_t n = s_n;
      double bf = -INFINITY;
      uint32_t bi = kNoParticle;
      if (n != 0) {  // scan_queue (engine_queue.hpp:28-35): sequential leader scan
        bf = wf[0];
        bi = wi[0];
        for (uint32_t j = 1; j < n; ++j)
          if (beats(wf[j], wi[j], bf, bi)) {
            bf = wf[j];
            bi = wi[j];
          }
        atomicAdd(&C.admitted[t], static_cast<unsigned long long>(n));
      }
      if (MODE == kQueue) {
        C.aux_fit[g] = bf;
        C.aux_idx[g] = bi;
      } else {  // queue-lock: lock-guarded beats() commit into the live record
        // Pre-check without the lock: the live record only grows in beats()
        // order, so a leader that cannot beat it now never will. Re-checked
        // under the lock, so the result is the reference's.
        if (n != 0 && may_beat(C.live, bf, bi)) {
          lock_acquire(C.lock);
          const double lf = *reinterpret_cast<volatile double*>(&C.live->fit);
          const uint32_t lp = *reinterpret_cast<volatile uint32_t*>(&C.live->particle);
          if (beats(bf, bi, lf, lp)) {
            for (uint32_t a = 0; a < P.d; ++a)
              C.live_pos[a] = S.pos[static_cast<size_t>(a) * P.ld + (bi - P.base)];
            write_rec(C.live, bf, bi);
          }
          lock_release(C.lock);
        }
        // last block to finish publishes live -> snapshot and the trace entry
        __threadfence();
        if (atomicAdd(C.ticket, 1u) == gridDim.x - 1) {
          __threadfence();
          const double lf = *reinterpret_cast<volatile double*>(&C.live->fit);
          const uint32_t lp = *reinterpret_cast<volatile uint32_t*>(&C.live->particle);
          if (lp != C.snap->particle || lf != C.snap->fit) {
            for (uint32_t a = 0; a < P.d; ++a)
              C.snap_pos[a] = *reinterpret_cast<volatile double*>(&C.live_pos[a]);
            C.snap->fit = lf;
            C.snap->particle = lp;
          }
          C.trace[t] = lf;
          C.trace_idx[t] = lp;
          *C.ticket = 0;
        }
      }
    }
  }
}

// ------------------------------------------------------ classic phase 2
// One group folds the aux slots (engine_reduction.hpp:29-32, engine_queue.hpp:63-78)
// and adopts the winner under a strict > against the record, gathering the
// position by index (adopt_record, engine.hpp:57-62).
template <int MODE>
__global__ void k_classic_fold(KParams P, KState S, KCtl C, uint32_t t, uint32_t groups,
                               uint32_t padded) {
  extern __shared__ double smem_d[];
  double* wf = smem_d;
  uint32_t* wi = reinterpret_cast<uint32_t*>(wf + padded);
  __shared__ uint32_t s_n;
  __shared__ double s_wf;
  __shared__ uint32_t s_wi;
  __shared__ int s_adopt;
  const uint32_t lane = threadIdx.x;
  double mf = -INFINITY;
  uint32_t mi = kNoParticle;
  // strided fold (engine_reduction.hpp:29-32); 8 independent loads in flight per lane
  constexpr uint32_t kBatch = 8;
  for (uint32_t k0 = lane; k0 < groups; k0 += kBatch * P.gs) {
    double ef[kBatch];
    uint32_t ei[kBatch];
#pragma unroll
    for (uint32_t j = 0; j < kBatch; ++j) {
      const uint32_t k = k0 + j * P.gs;
      ef[j] = k < groups ? C.aux_fit[k] : -INFINITY;
      ei[j] = k < groups ? C.aux_idx[k] : kNoParticle;
    }
#pragma unroll
    for (uint32_t j = 0; j < kBatch; ++j)
      if (beats(ef[j], ei[j], mf, mi)) {
        mf = ef[j];
        mi = ei[j];
      }
  }
  const double snap_fit = C.snap->fit;
  if (MODE == kTree || MODE == kTreeUnrolled) {
    wf[lane] = mf;
    wi[lane] = mi;
    for (uint32_t pad = lane + P.gs; pad < padded; pad += P.gs) {
      wf[pad] = -INFINITY;
      wi[pad] = kNoParticle;
    }
    __syncthreads();
    if (MODE == kTreeUnrolled)
      tree_unrolled(wf, wi, lane, padded);
    else
      tree_looped(wf, wi, lane, padded);
    if (lane == 0) {
      s_wf = wf[0];
      s_wi = wi[0];
      s_adopt = wf[0] > snap_fit;
    }
  } else {
    if (lane == 0) s_n = 0;
    __syncthreads();
    if (mf > snap_fit) {
      const uint32_t slot = queue_append(&s_n);
      wf[slot] = mf;
      wi[slot] = mi;
    }
    __syncthreads();
    if (lane == 0) {
      const uint32_t n = s_n;
      s_adopt = 0;
      if (n != 0) {
        double bf = wf[0];
        uint32_t bi = wi[0];
        for (uint32_t j = 1; j < n; ++j)
          if (beats(wf[j], wi[j], bf, bi)) {
            bf = wf[j];
            bi = wi[j];
          }
        s_wf = bf;
        s_wi = bi;
        s_adopt = bf > snap_fit;
      }
    }
  }
  __syncthreads();
  if (s_adopt) {
    const uint32_t w = s_wi;
    for (uint32_t a = lane; a < P.d; a += blockDim.x)
      C.snap_pos[a] = S.pos[static_cast<size_t>(a) * P.ld + (w - P.base)];
    if (lane == 0) {
      C.snap->fit = s_wf;
      C.snap->particle = w;
    }
  }
  if (lane == 0) {
    C.trace[t] = s_adopt ? s_wf : snap_fit;
    C.trace_idx[t] = s_adopt ? s_wi : C.snap->particle;
  }
}

// ---------------------------------------------------- shared block logic
// Per-thread candidate over the thread's pairs -> block queue in smem via
// warp ballot + shuffle argmax (one append per warp with a candidate).
constexpr int kMaxWarps = 32;
struct BlockCand {
  double f[kMaxWarps];
  uint32_t i[kMaxWarps];
  uint32_t n;
  unsigned long long adm;
};

__device__ __forceinline__ void warp_publish(BlockCand& bc, double bf, uint32_t bi, uint32_t adm) {
  const uint32_t lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, bi != kNoParticle);
  const uint32_t wadm = __reduce_add_sync(0xffffffffu, adm);
  if (m) {
    warp_argmax(bf, bi);
    if (lane == 0) {
      const uint32_t slot = atomicAdd(&bc.n, 1u);
      bc.f[slot] = bf;
      bc.i[slot] = bi;
    }
  }
  if (lane == 0 && wadm) atomicAdd(&bc.adm, static_cast<unsigned long long>(wadm));
}

// Tunings of the fused step: particles per thread-item (1: scalar LDG.64,
// 2: LDG.128 over two adjacent particles), software prefetch of the next
// item's loads, and the occupancy target handed to __launch_bounds__.
template <int NP_, int PF_, int MINB_, int KD_ = 1>
struct StepCfg {
  static constexpr int kNP = NP_;
  static constexpr int kPF = PF_;
  static constexpr int kMinBlocks = MINB_;
  static constexpr int kKD = KD_;  // axes whose loads are issued together (memory-level parallelism)
};

// NP adjacent particles of one axis row: scalar for NP = 1, 128-bit
// accesses (NP/2 of them) for even NP; rows are 512-B aligned and units start
// at multiples of NP, so every access is naturally aligned.
template <int NP>
__device__ __forceinline__ void ldv(const double* p, double (&o)[NP]) {
  static_assert(NP == 1 || NP % 2 == 0, "NP must be 1 or even");
  if constexpr (NP == 1) {
    o[0] = *p;
  } else {
#pragma unroll
    for (int k = 0; k < NP; k += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + k);
      o[k] = t.x;
      o[k + 1] = t.y;
    }
  }
}
template <int NP>
__device__ __forceinline__ void stv(double* p, const double (&o)[NP]) {
  static_assert(NP == 1 || NP % 2 == 0, "NP must be 1 or even");
  if constexpr (NP == 1) {
    *p = o[0];
  } else {
#pragma unroll
    for (int k = 0; k < NP; k += 2) *reinterpret_cast<double2*>(p + k) = make_double2(o[k], o[k + 1]);
  }
}

// Thread's share of the fused step (a unit = NP adjacent particles; thread
// (b, tid) takes units (b + k*gridDim)*blockDim + tid).
// The thread walks its (unit, axis) items; with PF the loads of item k+1 (and
// the next unit's pbest_fit) are issued before item k's Philox / kinematics /
// fitness chain so the long-scoreboard wait hides behind ~115 instructions of
// compute per particle-axis.
template <int F, class CFG>
__device__ __forceinline__ void step_items(const KParams& P, const KState& S, uint32_t t,
                                           const double* gpos, double snap_fit, double& bf,
                                           uint32_t& bi, uint32_t& adm) {
  constexpr int NP = CFG::kNP;
  bf = -INFINITY;
  bi = kNoParticle;
  adm = 0;
  // grid-stride over units: at any moment the whole grid streams one
  // contiguous window of every axis row (TLB / DRAM-page friendly)
  const uint32_t u_end = (P.n + NP - 1) / NP;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= u_end) return;
  if constexpr (!CFG::kPF) {
    // lean nested loops (unit, axis): minimal live state -> 32 registers,
    // full occupancy; latency is hidden by 64 resident warps per SM
    for (; u < u_end; u += stride) {
      const uint32_t li = NP * u;
      const uint32_t g0 = P.base + li;
      Fit<F> acc[NP];
      constexpr int KD = CFG::kKD;
      for (uint32_t a0 = 0; a0 < P.d; a0 += KD) {
        // issue the loads of KD axes before any of their compute
        double x[KD][NP], v[KD][NP], pb[KD][NP];
#pragma unroll
        for (int q = 0; q < KD; ++q) {
          if (KD == 1 || a0 + q < P.d) {
            const size_t at = static_cast<size_t>(a0 + q) * P.ld + li;
            ldv<NP>(S.pos + at, x[q]);
            ldv<NP>(S.vel + at, v[q]);
            ldv<NP>(S.pb + at, pb[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < KD; ++q) {
          if (KD > 1 && a0 + q >= P.d) break;
          const uint32_t a = a0 + q;
          const size_t at = static_cast<size_t>(a) * P.ld + li;
          const double g = gpos[a];
          double nx[NP], nv[NP];
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const double r1 = uniform01(P, t, g0 + k, a, 0);
            const double r2 = uniform01(P, t, g0 + k, a, 1);
            nv[k] = vel_step(P, v[q][k], x[q][k], pb[q][k], g, r1, r2);
            nx[k] = pos_step(P, x[q][k], nv[k]);
            acc[k].add(nx[k], a);
          }
          stv<NP>(S.vel + at, nv);
          stv<NP>(S.pos + at, nx);
        }
      }
      double pbf[NP];
      ldv<NP>(S.pbf + li, pbf);
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double f = acc[k].value();
        if (k > 0 && li + k >= P.n) break;
        if (f > pbf[k]) {  // update_pbest (swarm.hpp:100-108), rare after warm-up
          S.pbf[li + k] = f;
          for (uint32_t j = 0; j < P.d; ++j) {
            const size_t aj = static_cast<size_t>(j) * P.ld + li + k;
            S.pb[aj] = S.pos[aj];
          }
        }
        if (f > snap_fit) {  // snapshot filter (engine_queue.hpp:91)
          ++adm;
          if (beats(f, g0 + k, bf, bi)) {
            bf = f;
            bi = g0 + k;
          }
        }
      }
    }
    return;
  }
  const uint32_t d = P.d;
  const size_t ld = P.ld;
  uint32_t a = 0;
  size_t at = static_cast<size_t>(NP) * u;
  double x[NP], v[NP], pb[NP], pbf[NP];
  ldv<NP>(S.pos + at, x);
  ldv<NP>(S.vel + at, v);
  ldv<NP>(S.pb + at, pb);
  ldv<NP>(S.pbf + at, pbf);
  Fit<F> acc[NP];
  for (;;) {
    uint32_t un = u, an = a + 1;
    size_t atn = at + ld;
    bool next = true;
    if (an == d) {
      an = 0;
      un = u + stride;
      atn = static_cast<size_t>(NP) * un;
      next = un < u_end;
    }
    double xn[NP], vn[NP], pbn[NP], pbfn[NP];
    if constexpr (CFG::kPF) {
      if (next) {
        ldv<NP>(S.pos + atn, xn);
        ldv<NP>(S.vel + atn, vn);
        ldv<NP>(S.pb + atn, pbn);
        if (an == 0) ldv<NP>(S.pbf + atn, pbfn);
      }
    }
    const uint32_t li = NP * u;
    const uint32_t g0 = P.base + li;
    const double g = gpos[a];
    double nx[NP], nv[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double r1 = uniform01(P, t, g0 + k, a, 0);
      const double r2 = uniform01(P, t, g0 + k, a, 1);
      nv[k] = vel_step(P, v[k], x[k], pb[k], g, r1, r2);
      nx[k] = pos_step(P, x[k], nv[k]);
    }
    stv<NP>(S.vel + at, nv);
    stv<NP>(S.pos + at, nx);
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k].add(nx[k], a);
    if (a + 1 == d) {  // unit complete: pbest (swarm.hpp:100-108) + snapshot filter
      bool upd[NP];
      bool any = false;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        const double f = acc[k].value();
        acc[k] = Fit<F>();
        const bool ok = k == 0 || li + k < P.n;
        upd[k] = ok && f > pbf[k];
        any |= upd[k];
        if (upd[k]) S.pbf[li + k] = f;
        if (ok && f > snap_fit) {  // snapshot filter (engine_queue.hpp:91)
          ++adm;
          if (beats(f, g0 + k, bf, bi)) {
            bf = f;
            bi = g0 + k;
          }
        }
      }
      if (any) {  // rare after warm-up: re-read the just-written positions
        for (uint32_t j = 0; j < d; ++j) {
          const size_t aj = static_cast<size_t>(j) * ld + li;
#pragma unroll
          for (int k = 0; k < NP; ++k)
            if (upd[k]) S.pb[aj + k] = S.pos[aj + k];
        }
      }
    }
    if (!next) break;
    u = un;
    a = an;
    at = atn;
    if constexpr (CFG::kPF) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        x[k] = xn[k];
        v[k] = vn[k];
        pb[k] = pbn[k];
        if (an == 0) pbf[k] = pbfn[k];
      }
    } else {
      ldv<NP>(S.pos + at, x);
      ldv<NP>(S.vel + at, v);
      ldv<NP>(S.pb + at, pb);
      if (an == 0) ldv<NP>(S.pbf + at, pbf);
    }
  }
}

template <int NP>
__device__ __forceinline__ void block_unit_range(const KParams& P, uint32_t& b, uint32_t& e) {
  const uint64_t units = (P.n + NP - 1ull) / NP;
  b = static_cast<uint32_t>(units * blockIdx.x / gridDim.x);
  e = static_cast<uint32_t>(units * (blockIdx.x + 1) / gridDim.x);
}

// Block-wide argmax over grid-queue entries [0, nq) of buffer qb (all threads
// call; result broadcast through smem). Entries are deterministic, so every
// block (or the single resolving block) picks the same winner.
struct ResolveSmem {
  double f[kMaxWarps];
  uint32_t i[kMaxWarps], s[kMaxWarps];
};
__device__ __forceinline__ void resolve_queue(const KCtl& C, size_t base, uint32_t nq, ResolveSmem& rs,
                                              double& wf, uint32_t& wi, uint32_t& ws) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double f = -INFINITY;
  uint32_t i = kNoParticle, s = 0;
  for (uint32_t k = tid; k < nq; k += blockDim.x) {
    const double ef = __ldcg(&C.q_fit[base + k]);
    const uint32_t ei = __ldcg(&C.q_idx[base + k]);
    if (beats(ef, ei, f, i)) {
      f = ef;
      i = ei;
      s = k;
    }
  }
  warp_argmax3(f, i, s);
  if (lane == 0) {
    rs.f[warp] = f;
    rs.i[warp] = i;
    rs.s[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t nw = blockDim.x >> 5;
    f = lane < nw ? rs.f[lane] : -INFINITY;
    i = lane < nw ? rs.i[lane] : kNoParticle;
    s = lane < nw ? rs.s[lane] : 0;
    warp_argmax3(f, i, s);
    if (lane == 0) {
      rs.f[0] = f;
      rs.i[0] = i;
      rs.s[0] = s;
    }
  }
  __syncthreads();
  wf = rs.f[0];
  wi = rs.i[0];
  ws = rs.s[0];
}

// Shared tail of the persistent synchronous kernels, called by all threads
// once the block's candidates are in sh.bc (after a __syncthreads): warp 0
// appends the block winner {fit, idx, pos[d]} to the grid queue (pos_of(a, i)
// reads the winner's freshly written axis a), arrives at / waits on the grid
// barrier, then every block resolves the (usually empty) queue itself into the
// iteration-end snapshot. Deterministic whatever the arrival order.
struct SyncShared {
  BlockCand bc;
  ResolveSmem rs;
  uint32_t need;  // grid queue of this iteration may be non-empty
};

// Grid barrier word: low 32 bits count arrivals, high 32 bits count blocks
// that appended a candidate. A spinner that sees the high half unchanged
// knows the iteration admitted nothing (the common case after warm-up) and
// skips the queue entirely -- no extra L2 round trip on the critical path.
struct BarState {
  uint32_t target = 0;   // arrivals expected so far in this launch
  uint32_t appends = 0;  // exact appends counted through the end of the last iteration
};

__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// First half of sync_tail: warp 0 publishes the block winner and arrives at
// the grid barrier (release). The caller may do gbest-independent work (the
// next iteration's Philox draws) before sync_wait() blocks on the barrier.
template <class PosFn>
__device__ __forceinline__ void sync_arrive(const KParams& P, const KCtl& C, uint32_t t, SyncShared& sh,
                                            BarState& bs, uint32_t& nq_out, PosFn pos_of) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cap = C.q_cap, qb = t % 3;
  if (warp != 0) return;
  const uint32_t nq = sh.bc.n;
  nq_out = nq;
  if (nq) {
    double f = lane < nq ? sh.bc.f[lane] : -INFINITY;
    uint32_t i = lane < nq ? sh.bc.i[lane] : kNoParticle;
    warp_argmax(f, i);
    uint32_t slot = 0;
    if (lane == 0) slot = queue_append(&C.q_count[qb]);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    const size_t e = static_cast<size_t>(qb) * cap + slot;
    if (lane == 0) {
      C.q_fit[e] = f;
      C.q_idx[e] = i;
    }
    for (uint32_t a = lane; a < P.d; a += 32) C.q_pos[e * P.d + a] = pos_of(a, i);
    __threadfence();
  }
  __syncwarp();
  if (lane == 0) {
    if (sh.bc.adm) atomicAdd(&C.admitted[t], sh.bc.adm);
    sh.bc.n = 0;
    sh.bc.adm = 0;
    if (blockIdx.x == 0) C.q_count[(t + 1) % 3] = 0;
    bs.target += gridDim.x;
    red_release_gpu_add_u64(C.bar, 1ull | (nq ? (1ull << 32) : 0ull));
  }
}

// Second half: lane 0 of warp 0 spins until every block arrived, then the
// block resolves the grid queue when it may be non-empty.
__device__ __forceinline__ void sync_wait(const KParams& P, const KCtl& C, uint32_t t, SyncShared& sh,
                                          double* s_gpos, double& snap_fit, uint32_t& snap_idx,
                                          BarState& bs) {
  const uint32_t tid = threadIdx.x;
  const uint32_t cap = C.q_cap, qb = t % 3;
  if (tid == 0) {
    const uint64_t ts = globaltimer_ns();
    unsigned long long v;
    while (static_cast<uint32_t>(v = ld_acquire_gpu_u64(C.bar)) < bs.target) {
      if (globaltimer_ns() - ts > kSpinTimeoutNs) __trap();
    }
    sh.need = static_cast<uint32_t>(v >> 32) != bs.appends;
  }
  __syncthreads();
  if (sh.need) {  // block-uniform
    __threadfence();
    const uint32_t nq = __ldcg(&C.q_count[qb]);
    if (tid == 0) bs.appends += nq;
    if (nq) {
      double wf;
      uint32_t wi, ws;
      resolve_queue(C, static_cast<size_t>(qb) * cap, nq, sh.rs, wf, wi, ws);
      snap_fit = wf;
      snap_idx = wi;
      const size_t e = static_cast<size_t>(qb) * cap + ws;
      for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = __ldcg(&C.q_pos[e * P.d + a]);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    C.trace[t] = snap_fit;
    C.trace_idx[t] = snap_idx;
  }
}

template <class PosFn>
__device__ __forceinline__ void sync_tail(const KParams& P, const KCtl& C, uint32_t t, SyncShared& sh,
                                          double* s_gpos, double& snap_fit, uint32_t& snap_idx,
                                          BarState& bs, PosFn pos_of) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cap = C.q_cap, qb = t % 3;
  if (warp == 0) {  // block winner -> grid queue; then the grid barrier
    const uint32_t nq = sh.bc.n;
    if (nq) {
      double f = lane < nq ? sh.bc.f[lane] : -INFINITY;
      uint32_t i = lane < nq ? sh.bc.i[lane] : kNoParticle;
      warp_argmax(f, i);
      uint32_t slot = 0;
      if (lane == 0) slot = queue_append(&C.q_count[qb]);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      const size_t e = static_cast<size_t>(qb) * cap + slot;
      if (lane == 0) {
        C.q_fit[e] = f;
        C.q_idx[e] = i;
      }
      for (uint32_t a = lane; a < P.d; a += 32) C.q_pos[e * P.d + a] = pos_of(a, i);
      __threadfence();  // entry visible before the release below
    }
    __syncwarp();
    if (lane == 0) {
      if (sh.bc.adm) atomicAdd(&C.admitted[t], sh.bc.adm);
      sh.bc.n = 0;  // the other warps are parked at the __syncthreads below
      sh.bc.adm = 0;
      if (blockIdx.x == 0) C.q_count[(t + 1) % 3] = 0;  // last read two barriers ago
      bs.target += gridDim.x;
      red_release_gpu_add_u64(C.bar, 1ull | (nq ? (1ull << 32) : 0ull));
      const uint64_t ts = globaltimer_ns();
      unsigned long long v;
      while (static_cast<uint32_t>(v = ld_acquire_gpu_u64(C.bar)) < bs.target) {
        if (globaltimer_ns() - ts > kSpinTimeoutNs) __trap();
      }
      // a faster block may already have arrived at the next barrier; any
      // change of the high half only means "look at the queue"
      sh.need = static_cast<uint32_t>(v >> 32) != bs.appends;
    }
  }
  __syncthreads();
  if (sh.need) {  // block-uniform
    __threadfence();
    const uint32_t nq = __ldcg(&C.q_count[qb]);
    if (tid == 0) bs.appends += nq;  // exact appends of iteration t
    if (nq) {
      double wf;
      uint32_t wi, ws;
      resolve_queue(C, static_cast<size_t>(qb) * cap, nq, sh.rs, wf, wi, ws);
      snap_fit = wf;  // every entry passed fit > snap_fit, so the winner is adopted
      snap_idx = wi;
      const size_t e = static_cast<size_t>(qb) * cap + ws;
      for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = __ldcg(&C.q_pos[e * P.d + a]);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    C.trace[t] = snap_fit;
    C.trace_idx[t] = snap_idx;
  }
}

__device__ __forceinline__ void write_final_record(const KParams& P, const KCtl& C, const double* s_gpos,
                                                   double snap_fit, uint32_t snap_idx) {
  if (blockIdx.x != 0) return;
  for (uint32_t a = threadIdx.x; a < P.d; a += blockDim.x) {
    C.snap_pos[a] = s_gpos[a];
    C.live_pos[a] = s_gpos[a];
  }
  if (threadIdx.x == 0) {
    const Rec r{snap_fit, snap_idx, 0u};
    *C.snap = r;
    *C.live = r;
  }
}

// --------------------------------------------------------- sync (fused)
template <int F, class CFG>
__global__ void __launch_bounds__(kSyncThreads, CFG::kMinBlocks) k_sync(KParams P, KState S, KCtl C, uint32_t t0,
                                                       uint32_t t1) {
  extern __shared__ double s_gpos[];  // [d] iteration-start gbest position
  __shared__ SyncShared sh;
  const uint32_t tid = threadIdx.x;
  for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = C.snap_pos[a];
  if (tid == 0) {
    sh.bc.n = 0;
    sh.bc.adm = 0;
  }
  double snap_fit = C.snap->fit;
  uint32_t snap_idx = C.snap->particle;
  __syncthreads();
  BarState bs;
  auto pos_of = [&](uint32_t a, uint32_t i) { return S.pos[static_cast<size_t>(a) * P.ld + (i - P.base)]; };
  for (uint32_t t = t0; t < t1; ++t) {
    double bf;
    uint32_t bi, adm;
    step_items<F, CFG>(P, S, t, s_gpos, snap_fit, bf, bi, adm);
    warp_publish(sh.bc, bf, bi, adm);
    __syncthreads();
    sync_tail(P, C, t, sh, s_gpos, snap_fit, snap_idx, bs, pos_of);
  }
  write_final_record(P, C, s_gpos, snap_fit, snap_idx);
}

// ------------------------------------------------ sync, SMEM-resident
// The whole swarm lives in shared memory for the duration of the launch
// when its FP64 state fits: one 1024-thread block per SM owns a contiguous
// chunk of particles, stored axis-major in SMEM as x|v|pbest|pbest_fit.
// Per iteration there is no global-memory traffic for the state at all --
// only Philox/FP64 issue plus the grid barrier (cfg2: 2^20 x d=1 = 32 MB
// over 148 x 227 KB). State is loaded at launch start and written back at
// the end, so every launch boundary leaves HBM exact.
constexpr int kResThreads = 1024;

// D > 0 fixes the dimension at compile time (D = 1 is the BASELINE cfg2/cfg3
// shape): the axis counter then constant-folds into the first Philox rounds
// and the per-axis index arithmetic disappears.
template <int F, int D = 0>
__global__ void __launch_bounds__(kResThreads, 1) k_sync_res(KParams P, KState S, KCtl C, uint32_t t0,
                                                              uint32_t t1, uint32_t chunk_cap) {
  extern __shared__ double smem[];
  __shared__ SyncShared sh;
  const uint32_t tid = threadIdx.x;
  const uint32_t d = D > 0 ? static_cast<uint32_t>(D) : P.d;
  const uint32_t c0 = static_cast<uint32_t>(static_cast<uint64_t>(P.n) * blockIdx.x / gridDim.x);
  const uint32_t c1 = static_cast<uint32_t>(static_cast<uint64_t>(P.n) * (blockIdx.x + 1) / gridDim.x);
  const uint32_t m = c1 - c0;
  const uint32_t dpad = (d + 1u) & ~1u;
  double* s_gpos = smem;
  double* sx = smem + dpad;
  double* sv = sx + static_cast<size_t>(d) * chunk_cap;
  double* spb = sv + static_cast<size_t>(d) * chunk_cap;
  double* spbf = spb + static_cast<size_t>(d) * chunk_cap;
  for (uint32_t a = 0; a < d; ++a) {
    const size_t g = static_cast<size_t>(a) * P.ld + c0;
    const size_t l = static_cast<size_t>(a) * chunk_cap;
    for (uint32_t j = tid; j < m; j += blockDim.x) {
      sx[l + j] = S.pos[g + j];
      sv[l + j] = S.vel[g + j];
      spb[l + j] = S.pb[g + j];
    }
  }
  for (uint32_t j = tid; j < m; j += blockDim.x) spbf[j] = S.pbf[c0 + j];
  for (uint32_t a = tid; a < d; a += blockDim.x) s_gpos[a] = C.snap_pos[a];
  if (tid == 0) {
    sh.bc.n = 0;
    sh.bc.adm = 0;
  }
  double snap_fit = C.snap->fit;
  uint32_t snap_idx = C.snap->particle;
  __syncthreads();
  BarState bs;
  const uint32_t gbase = P.base + c0;
  auto pos_of = [&](uint32_t a, uint32_t i) { return sx[static_cast<size_t>(a) * chunk_cap + (i - gbase)]; };
  // d = 1: the r1/r2 draws of a thread's first kPre particles for iteration
  // t+1 depend on (t+1, particle) only, so they are computed while warp 0
  // waits on the grid barrier of iteration t (the barrier latency hides
  // behind ~60 Philox instructions per particle instead of idling).
  constexpr int kPre = D == 1 ? 2 : 0;
  double pre1[kPre > 0 ? kPre : 1], pre2[kPre > 0 ? kPre : 1];
  bool have_pre = false;
  for (uint32_t t = t0; t < t1; ++t) {
    double bf = -INFINITY;
    uint32_t bi = kNoParticle, adm = 0;
    auto finish = [&](uint32_t j, uint32_t gi, double f) {
      if (f > spbf[j]) {  // update_pbest (swarm.hpp:100-108)
        spbf[j] = f;
        for (uint32_t a = 0; a < d; ++a) {
          const size_t l = static_cast<size_t>(a) * chunk_cap + j;
          spb[l] = sx[l];
        }
      }
      if (f > snap_fit) {  // snapshot filter (engine_queue.hpp:91)
        ++adm;
        if (beats(f, gi, bf, bi)) {
          bf = f;
          bi = gi;
        }
      }
    };
    uint32_t j = tid;
    if constexpr (D == 1) {
      auto one = [&](uint32_t jj, double r1, double r2) {
        const double x = sx[jj];
        const double nv = vel_step(P, sv[jj], x, spb[jj], s_gpos[0], r1, r2);
        const double nx = pos_step(P, x, nv);
        sv[jj] = nv;
        sx[jj] = nx;
        Fit<F> acc;
        acc.add(nx, 0);
        finish(jj, gbase + jj, acc.value());
      };
#pragma unroll
      for (int k = 0; k < kPre; ++k, j += blockDim.x) {
        if (j < m) {
          const double r1 = have_pre ? pre1[k] : uniform01(P, t, gbase + j, 0, 0);
          const double r2 = have_pre ? pre2[k] : uniform01(P, t, gbase + j, 0, 1);
          one(j, r1, r2);
        }
      }
      for (; j < m; j += blockDim.x) one(j, uniform01(P, t, gbase + j, 0, 0), uniform01(P, t, gbase + j, 0, 1));
    } else {
      for (; j < m; j += blockDim.x) {
        const uint32_t gi = gbase + j;
        Fit<F> acc;
        for (uint32_t a = 0; a < d; ++a) {
          const size_t l = static_cast<size_t>(a) * chunk_cap + j;
          const double r1 = uniform01(P, t, gi, a, 0);
          const double r2 = uniform01(P, t, gi, a, 1);
          const double x = sx[l];
          const double nv = vel_step(P, sv[l], x, spb[l], s_gpos[a], r1, r2);
          const double nx = pos_step(P, x, nv);
          sv[l] = nv;
          sx[l] = nx;
          acc.add(nx, a);
        }
        finish(j, gi, acc.value());
      }
    }
    warp_publish(sh.bc, bf, bi, adm);
    __syncthreads();
    uint32_t nq_block = 0;
    sync_arrive(P, C, t, sh, bs, nq_block, pos_of);
    if constexpr (kPre > 0) {
      have_pre = t + 1 < t1;
      if (have_pre) {
        uint32_t jj = tid;
#pragma unroll
        for (int k = 0; k < kPre; ++k, jj += blockDim.x) {
          if (jj < m) {
            pre1[k] = uniform01(P, t + 1, gbase + jj, 0, 0);
            pre2[k] = uniform01(P, t + 1, gbase + jj, 0, 1);
          }
        }
      }
    }
    sync_wait(P, C, t, sh, s_gpos, snap_fit, snap_idx, bs);
  }
  for (uint32_t a = 0; a < d; ++a) {
    const size_t g = static_cast<size_t>(a) * P.ld + c0;
    const size_t l = static_cast<size_t>(a) * chunk_cap;
    for (uint32_t j = tid; j < m; j += blockDim.x) {
      S.pos[g + j] = sx[l + j];
      S.vel[g + j] = sv[l + j];
      S.pb[g + j] = spb[l + j];
    }
  }
  for (uint32_t j = tid; j < m; j += blockDim.x) S.pbf[c0 + j] = spbf[j];
  write_final_record(P, C, s_gpos, snap_fit, snap_idx);
}

// Hierarchical "last block done": blocks first count on one of 64 counters
// (blockIdx % 64) and only each group's last block touches the global
// ticket, so a 131072-block launch puts ~2048 atomics on each of 64 L2
// addresses instead of 131072 on one. Call from one thread after a fence.
__device__ __forceinline__ bool last_block_done(const KCtl& C) {
  const uint32_t G = gridDim.x;
  const uint32_t grp = blockIdx.x & 63u;
  const uint32_t ngrp = G < 64u ? G : 64u;
  const uint32_t grp_size = (G - grp + 63u) / 64u;
  if (atomicAdd(&C.ticket_grp[grp], 1u) != grp_size - 1u) return false;
  C.ticket_grp[grp] = 0u;  // every block of the group has arrived
  __threadfence();
  if (atomicAdd(C.ticket, 1u) != ngrp - 1u) return false;
  *C.ticket = 0u;
  __threadfence();
  return true;
}

// --------------------------------------------------------------- wave
// One launch per iteration (captured in a CUDA graph): one unit per thread,
// full occupancy, hardware block scheduling -- the HBM-bound shape of the
// synchronous variant. Blocks append their winner to the grid queue (rare);
// the last block resolves it into the snapshot record and trace[t]. No grid
// barrier, no lock, and no atomics on the common path except the ticket.
template <int F, class CFG>
__global__ void __launch_bounds__(kSyncThreads, CFG::kMinBlocks) k_wave(KParams P, KState S, KCtl C,
                                                                        uint32_t t) {
  extern __shared__ double s_gpos[];
  __shared__ BlockCand bc;
  __shared__ ResolveSmem rs;
  __shared__ int s_last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = C.snap_pos[a];
  if (tid == 0) {
    bc.n = 0;
    bc.adm = 0;
  }
  __syncthreads();
  const double snap_fit = C.snap->fit;
  double bf;
  uint32_t bi, adm;
  step_items<F, CFG>(P, S, t, s_gpos, snap_fit, bf, bi, adm);
  warp_publish(bc, bf, bi, adm);
  __syncthreads();
  if (warp == 0) {
    const uint32_t nq = bc.n;
    if (nq) {
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
        C.q_pos[static_cast<size_t>(slot) * P.d + a] = S.pos[static_cast<size_t>(a) * P.ld + (i - P.base)];
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      if (bc.adm) atomicAdd(&C.admitted[t], bc.adm);
      s_last = last_block_done(C);
    }
  }
  __syncthreads();
  if (!s_last) return;
  const uint32_t nq = __ldcg(&C.q_count[0]);
  if (nq) {
    double wf;
    uint32_t wi, ws;
    resolve_queue(C, 0, nq, rs, wf, wi, ws);
    for (uint32_t a = tid; a < P.d; a += blockDim.x)
      C.snap_pos[a] = __ldcg(&C.q_pos[static_cast<size_t>(ws) * P.d + a]);
    if (tid == 0) {  // every entry passed fit > snap_fit: adopt
      C.snap->fit = wf;
      C.snap->particle = wi;
    }
  }
  if (tid == 0) {
    C.trace[t] = nq ? rs.f[0] : snap_fit;
    C.trace_idx[t] = nq ? rs.i[0] : C.snap->particle;
    C.q_count[0] = 0;
  }
}

// ------------------------------------------------------- shard propose
// One iteration of the fused step on a shard; the last block to finish
// reduces the grid queue to the shard's candidate record
// {fit, particle, admitted, pos[d]} (sentinel when nothing was admitted).
template <int F, class CFG>
__global__ void __launch_bounds__(kSyncThreads, CFG::kMinBlocks) k_propose(KParams P, KState S, KCtl C, uint32_t t,
                                                          unsigned char* record) {
  extern __shared__ double s_gpos[];
  __shared__ BlockCand bc;
  __shared__ double s_rf[kSyncWarps];
  __shared__ uint32_t s_ri[kSyncWarps], s_rs[kSyncWarps];
  __shared__ int s_last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = C.snap_pos[a];
  if (tid == 0) {
    bc.n = 0;
    bc.adm = 0;
  }
  __syncthreads();
  const double snap_fit = C.snap->fit;
  double bf;
  uint32_t bi, adm;
  step_items<F, CFG>(P, S, t, s_gpos, snap_fit, bf, bi, adm);
  warp_publish(bc, bf, bi, adm);
  __syncthreads();
  if (warp == 0) {
    const uint32_t nq = bc.n;
    if (nq) {
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
        C.q_pos[static_cast<size_t>(slot) * P.d + a] = S.pos[static_cast<size_t>(a) * P.ld + (i - P.base)];
    }
    if (lane == 0 && bc.adm) atomicAdd(&C.admitted[t], bc.adm);
    __threadfence();
    __syncwarp();
    if (lane == 0) s_last = atomicAdd(C.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint32_t nq = __ldcg(&C.q_count[0]);
  double f = -INFINITY;
  uint32_t i = kNoParticle, s = 0;
  for (uint32_t k = tid; k < nq; k += blockDim.x) {
    const double ef = __ldcg(&C.q_fit[k]);
    const uint32_t ei = __ldcg(&C.q_idx[k]);
    if (beats(ef, ei, f, i)) {
      f = ef;
      i = ei;
      s = k;
    }
  }
  warp_argmax3(f, i, s);
  if (lane == 0) {
    s_rf[warp] = f;
    s_ri[warp] = i;
    s_rs[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    f = lane < kSyncWarps ? s_rf[lane] : -INFINITY;
    i = lane < kSyncWarps ? s_ri[lane] : kNoParticle;
    s = lane < kSyncWarps ? s_rs[lane] : 0;
    warp_argmax3(f, i, s);
    if (lane == 0) {
      s_rf[0] = f;
      s_ri[0] = i;
      s_rs[0] = s;
    }
  }
  __syncthreads();
  Rec* rec = reinterpret_cast<Rec*>(record);
  double* rpos = reinterpret_cast<double*>(record + sizeof(Rec));
  for (uint32_t a = tid; a < P.d; a += blockDim.x)
    rpos[a] = nq ? __ldcg(&C.q_pos[static_cast<size_t>(s_rs[0]) * P.d + a]) : 0.0;
  if (tid == 0) {
    const unsigned long long am = *reinterpret_cast<volatile unsigned long long*>(&C.admitted[t]);
    rec->fit = nq ? s_rf[0] : -INFINITY;
    rec->particle = nq ? s_ri[0] : kNoParticle;
    rec->admitted = static_cast<uint32_t>(am);
    C.q_count[0] = 0;
    *C.ticket = 0;
  }
}

// All shards apply the same selection: beats() among records, strict > vs snapshot.
__global__ void k_commit(KParams P, KCtl C, uint32_t t, const unsigned char* records, uint32_t nrec,
                         size_t rec_bytes, int count_admitted) {
  __shared__ int s_w;
  if (threadIdx.x == 0) {
    double bf = -INFINITY;
    uint32_t bi = kNoParticle;
    int w = -1;
    unsigned long long adm = 0;
    for (uint32_t r = 0; r < nrec; ++r) {
      const Rec* rec = reinterpret_cast<const Rec*>(records + r * rec_bytes);
      adm += rec->admitted;
      if (rec->particle != kNoParticle && beats(rec->fit, rec->particle, bf, bi)) {
        bf = rec->fit;
        bi = rec->particle;
        w = static_cast<int>(r);
      }
    }
    if (!(w >= 0 && bf > C.snap->fit)) w = -1;
    s_w = w;
    if (w >= 0) {
      C.snap->fit = bf;
      C.snap->particle = bi;
    }
    if (count_admitted) C.admitted[t] = adm;
    C.trace[t] = C.snap->fit;
    C.trace_idx[t] = C.snap->particle;
  }
  __syncthreads();
  if (s_w >= 0) {
    const double* rpos = reinterpret_cast<const double*>(records + s_w * rec_bytes + sizeof(Rec));
    for (uint32_t a = threadIdx.x; a < P.d; a += blockDim.x) C.snap_pos[a] = rpos[a];
  }
}

// Initial gbest of a sharded swarm: every shard adopts the beats()-max of the
// shards' local initial records (init_swarm's first strict max, swarm.hpp:164-170,
// taken over the whole swarm).
__global__ void k_adopt(KParams P, KCtl C, const unsigned char* records, uint32_t nrec,
                        size_t rec_bytes) {
  __shared__ int s_w;
  if (threadIdx.x == 0) {
    double bf = -INFINITY;
    uint32_t bi = kNoParticle;
    int w = -1;
    for (uint32_t r = 0; r < nrec; ++r) {
      const Rec* rec = reinterpret_cast<const Rec*>(records + r * rec_bytes);
      if (rec->particle != kNoParticle && beats(rec->fit, rec->particle, bf, bi)) {
        bf = rec->fit;
        bi = rec->particle;
        w = static_cast<int>(r);
      }
    }
    s_w = w;
    const Rec out{w >= 0 ? bf : -INFINITY, w >= 0 ? bi : kNoParticle, 0u};
    *C.snap = out;
    *C.live = out;
  }
  __syncthreads();
  for (uint32_t a = threadIdx.x; a < P.d; a += blockDim.x) {
    const double x = s_w >= 0
        ? reinterpret_cast<const double*>(records + s_w * rec_bytes + sizeof(Rec))[a] : 0.0;
    C.snap_pos[a] = x;
    C.live_pos[a] = x;
  }
}

// ---------------------------------------------------------------- async
// Free-running blocks. The live record {fit, particle, pos[d]} is guarded by
// a seqlock: readers retry on an odd or changed version; a writer takes the
// record with CAS(version: even -> odd), re-checks beats() under it, writes,
// and releases with version+2. No grid barrier anywhere.
constexpr int kTileThreads = 512;

struct AsyncShared {
  double fit;
  uint32_t idx, ver, have, ok;
};

// Consistent (torn-read-free) copy of the live record into s_gpos / as.fit;
// the position copy is skipped while the version is unchanged. All threads call.
__device__ __forceinline__ void async_read_gbest(const KParams& P, const KCtl& C, double* s_gpos,
                                                 AsyncShared& as) {
  const uint32_t tid = threadIdx.x;
  const uint64_t ts = globaltimer_ns();
  for (;;) {
    __syncthreads();  // previous round's readers are done with as.ok / as.have
    if (tid == 0) {
      const uint32_t v = ld_acquire_gpu(C.seq);
      as.ok = (v & 1u) == 0u;
      as.have = 1;  // unchanged since our last copy
      if (as.ok && v != as.ver) {
        as.have = 2;  // needs a copy
        as.ver = v;
      }
      if (!as.ok && globaltimer_ns() - ts > kSpinTimeoutNs) __trap();
    }
    __syncthreads();
    if (!as.ok) continue;
    if (as.have == 1) break;
    for (uint32_t a = tid; a < P.d; a += blockDim.x) s_gpos[a] = __ldcg(&C.live_pos[a]);
    if (tid == 0) {
      as.fit = __ldcg(&C.live->fit);
      as.idx = __ldcg(&C.live->particle);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const uint32_t v2 = ld_acquire_gpu(C.seq);
      as.ok = v2 == as.ver;
      if (!as.ok) as.ver = 0xffffffffu;
    }
    __syncthreads();
    if (as.ok) break;
  }
}

// Warp 0 publishes the block winner into the live record when it beats it
// (lock-free pre-check, then CAS(version even->odd), re-check, write, release
// version+2) and folds its view of the gbest into trace_key[t].
template <class PosFn>
__device__ __forceinline__ void async_commit(const KParams& P, const KCtl& C, uint32_t t, BlockCand& bc,
                                             double snap_fit, PosFn pos_of) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp != 0) return;
  const uint32_t nq = bc.n;
  double view = snap_fit;
  if (nq) {
    double f = lane < nq ? bc.f[lane] : -INFINITY;
    uint32_t i = lane < nq ? bc.i[lane] : kNoParticle;
    warp_argmax(f, i);
    // lane 0 decides for the whole warp: per-lane loads of a record that other
    // blocks are writing may disagree, and the warp must take one branch
    double lf0 = 0.0;
    int try_lock = 0;
    if (lane == 0) {
      lf0 = ld_acquire_gpu_f64(&C.live->fit);
      try_lock = may_beat(C.live, f, i);
    }
    lf0 = __shfl_sync(0xffffffffu, lf0, 0);
    try_lock = __shfl_sync(0xffffffffu, try_lock, 0);
    if (try_lock) {
      uint32_t v = 0;
      double lf = 0.0;
      uint32_t lp = 0;
      if (lane == 0) {
        const uint64_t tl = globaltimer_ns();
        for (;;) {
          v = ld_acquire_gpu(C.seq);
          if (!(v & 1u) && atomicCAS(C.seq, v, v + 1u) == v) break;
          if (globaltimer_ns() - tl > kSpinTimeoutNs) __trap();
        }
        __threadfence();
        lf = __ldcg(&C.live->fit);
        lp = __ldcg(&C.live->particle);
      }
      v = __shfl_sync(0xffffffffu, v, 0);
      lf = __shfl_sync(0xffffffffu, lf, 0);
      lp = __shfl_sync(0xffffffffu, lp, 0);
      if (beats(f, i, lf, lp)) {
        for (uint32_t a = lane; a < P.d; a += 32) C.live_pos[a] = pos_of(a, i);
        __syncwarp();
        if (lane == 0) write_rec(C.live, f, i);
        view = f;
      } else {
        view = lf;
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_gpu(C.seq, v + 2u);
    } else {
      view = lf0 > view ? lf0 : view;
    }
  }
  if (lane == 0) {
    if (bc.adm) atomicAdd(&C.admitted[t], bc.adm);
    atomicMax(&C.trace_key[t], order_key(view));
    bc.n = 0;
    bc.adm = 0;
  }
}

template <int F, class CFG>
__global__ void __launch_bounds__(kSyncThreads, CFG::kMinBlocks) k_async(KParams P, KState S, KCtl C, uint32_t t0,
                                                        uint32_t t1) {
  extern __shared__ double s_gpos[];
  __shared__ BlockCand bc;
  __shared__ AsyncShared as;
  if (threadIdx.x == 0) {
    as.have = 0;
    as.ver = 0xffffffffu;
    bc.n = 0;
    bc.adm = 0;
  }
  __syncthreads();
  auto pos_of = [&](uint32_t a, uint32_t i) { return S.pos[static_cast<size_t>(a) * P.ld + (i - P.base)]; };
  for (uint32_t t = t0; t < t1; ++t) {
    async_read_gbest(P, C, s_gpos, as);
    const double snap_fit = as.fit;
    double bf;
    uint32_t bi, adm;
    step_items<F, CFG>(P, S, t, s_gpos, snap_fit, bf, bi, adm);
    warp_publish(bc, bf, bi, adm);
    __syncthreads();
    async_commit(P, C, t, bc, snap_fit, pos_of);
    __syncthreads();
  }
}

// ------------------------------------------------------- async, tiled
// Temporal blocking for the asynchronous variant. Asynchronous PSO lets each
// particle advance at its own pace against the latest published gbest, so a
// block may keep a tile of its particles in SMEM and run K iterations on it
// before writing it back and loading the next tile. Every particle still does
// exactly T iterations with draws keyed by its own (t, particle, axis); HBM
// traffic drops from (5d+1)*8 B per particle-update to ~(8d+2)*8/K B and the
// kernel becomes issue-bound. Each tile-iteration re-reads the live record
// through the seqlock (skipping the copy when unchanged) and publishes
// improvements with the same CAS protocol as k_async.
template <int F, int D = 0>
__global__ void __launch_bounds__(kTileThreads, 2) k_async_tiled(KParams P, KState S, KCtl C, uint32_t t0,
                                                                 uint32_t t1, uint32_t tile_cap, uint32_t K) {
  extern __shared__ double smem[];
  __shared__ BlockCand bc;
  __shared__ AsyncShared as;
  const uint32_t tid = threadIdx.x;
  const uint32_t d = D > 0 ? static_cast<uint32_t>(D) : P.d;
  const uint32_t c0 = static_cast<uint32_t>(static_cast<uint64_t>(P.n) * blockIdx.x / gridDim.x);
  const uint32_t c1 = static_cast<uint32_t>(static_cast<uint64_t>(P.n) * (blockIdx.x + 1) / gridDim.x);
  const uint32_t dpad = (d + 1u) & ~1u;
  double* s_gpos = smem;
  double* sx = smem + dpad;
  double* sv = sx + static_cast<size_t>(d) * tile_cap;
  double* spb = sv + static_cast<size_t>(d) * tile_cap;
  double* spbf = spb + static_cast<size_t>(d) * tile_cap;
  if (tid == 0) {
    as.have = 0;
    as.ver = 0xffffffffu;
    bc.n = 0;
    bc.adm = 0;
  }
  __syncthreads();
  for (uint32_t tb = t0; tb < t1; tb += K) {
    const uint32_t te = tb + K < t1 ? tb + K : t1;
    for (uint32_t s0 = c0; s0 < c1; s0 += tile_cap) {
      const uint32_t m = (c1 - s0) < tile_cap ? (c1 - s0) : tile_cap;
      for (uint32_t a = 0; a < d; ++a) {
        const size_t g = static_cast<size_t>(a) * P.ld + s0;
        const size_t l = static_cast<size_t>(a) * tile_cap;
        for (uint32_t j = tid; j < m; j += blockDim.x) {
          sx[l + j] = S.pos[g + j];
          sv[l + j] = S.vel[g + j];
          spb[l + j] = S.pb[g + j];
        }
      }
      for (uint32_t j = tid; j < m; j += blockDim.x) spbf[j] = S.pbf[s0 + j];
      const uint32_t gbase = P.base + s0;
      auto pos_of = [&](uint32_t a, uint32_t i) { return sx[static_cast<size_t>(a) * tile_cap + (i - gbase)]; };
      async_read_gbest(P, C, s_gpos, as);  // also orders the tile load before use
      for (uint32_t t = tb; t < te; ++t) {
        // The version check for the *next* tile-iteration is issued now and
        // consumed after the compute, so its L2 latency overlaps the work; the
        // gbest used here may be one tile-iteration stale (asynchronous PSO).
        uint32_t ver_now = 0;
        if (tid == 0) ver_now = ld_acquire_gpu(C.seq);
        const double snap_fit = as.fit;
        double bf = -INFINITY;
        uint32_t bi = kNoParticle, adm = 0;
        for (uint32_t j = tid; j < m; j += blockDim.x) {
          const uint32_t gi = gbase + j;
          Fit<F> acc;
          for (uint32_t a = 0; a < d; ++a) {
            const size_t l = static_cast<size_t>(a) * tile_cap + j;
            const double r1 = uniform01(P, t, gi, a, 0);
            const double r2 = uniform01(P, t, gi, a, 1);
            const double x = sx[l];
            const double nv = vel_step(P, sv[l], x, spb[l], s_gpos[a], r1, r2);
            const double nx = pos_step(P, x, nv);
            sv[l] = nv;
            sx[l] = nx;
            acc.add(nx, a);
          }
          const double f = acc.value();
          if (f > spbf[j]) {
            spbf[j] = f;
            for (uint32_t a = 0; a < d; ++a) {
              const size_t l = static_cast<size_t>(a) * tile_cap + j;
              spb[l] = sx[l];
            }
          }
          if (f > snap_fit) {
            ++adm;
            if (beats(f, gi, bf, bi)) {
              bf = f;
              bi = gi;
            }
          }
        }
        warp_publish(bc, bf, bi, adm);
        if (tid == 0) as.have = ver_now != as.ver ? 2u : 1u;  // 2: the live record moved
        __syncthreads();
        if (tid == 0 && bc.n) as.have = 2u;  // publishing: re-read the record afterwards
        async_commit(P, C, t, bc, snap_fit, pos_of);
        __syncthreads();
        if (as.have == 2) async_read_gbest(P, C, s_gpos, as);  // block-uniform
      }
      for (uint32_t a = 0; a < d; ++a) {
        const size_t g = static_cast<size_t>(a) * P.ld + s0;
        const size_t l = static_cast<size_t>(a) * tile_cap;
        for (uint32_t j = tid; j < m; j += blockDim.x) {
          S.pos[g + j] = sx[l + j];
          S.vel[g + j] = sv[l + j];
          S.pb[g + j] = spb[l + j];
        }
      }
      for (uint32_t j = tid; j < m; j += blockDim.x) S.pbf[s0 + j] = spbf[j];
      __syncthreads();  // the next tile overwrites SMEM
    }
  }
}


// ------------------------------------------------ concurrency self-tests
// Device analogue of the reference's acceptance criterion 4
// (acceptance.cpp:126-200), run through cupso_selftest_*.
// (a) append uniqueness: every round, the lanes selected by
// ((lane ^ salt) + round) % 4 != 0 append to the block queue with
// queue_append; the claimed slots must be exactly 0..count-1, each once, and
// the counter must equal the number of appenders. Lane 0 of every block also
// appends once per round to a grid queue (unique over the whole grid,
// checked on the host).
__global__ void k_stress_append(uint32_t rounds, uint32_t salt, uint32_t* gq_count, uint32_t* gq_seen,
                                uint32_t gq_cap, unsigned long long* violations) {
  extern __shared__ uint32_t seen[];
  __shared__ uint32_t s_n;
  const uint32_t tid = threadIdx.x;
  uint32_t bad = 0;
  for (uint32_t round = 0; round < rounds; ++round) {
    seen[tid] = 0;
    if (tid == 0) s_n = 0;
    __syncthreads();
    const bool app = ((tid ^ salt) + round) % 4u != 0u;
    const uint32_t slot = app ? queue_append(&s_n) : kNoParticle;
    if (app) {
      if (slot < blockDim.x) atomicAdd(&seen[slot], 1u);
      else ++bad;
    }
    const uint32_t want = static_cast<uint32_t>(__syncthreads_count(app));
    if (tid == 0 && s_n != want) ++bad;
    if (seen[tid] != (tid < want ? 1u : 0u)) ++bad;
    if (tid == 0) {
      const uint32_t g = queue_append(gq_count);
      if (g < gq_cap) atomicAdd(&gq_seen[g], 1u);
    }
    __syncthreads();
  }
  if (bad) atomicAdd(violations, static_cast<unsigned long long>(bad));
}

// (b) lock exclusion: lane 0 of every warp increments a plain (non-atomic,
// volatile) counter `iters` times under lock_acquire / lock_release; any lost
// update shows as a counter below warps * iters.
__global__ void k_stress_lock(uint32_t iters, uint32_t* lock, unsigned long long* counter) {
  if ((threadIdx.x & 31u) != 0) return;
  volatile unsigned long long* c = counter;
  for (uint32_t i = 0; i < iters; ++i) {
    lock_acquire(lock);
    *c = *c + 1ull;
    lock_release(lock);
  }
}

}  // namespace cupso
