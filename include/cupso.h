/*
 * cupso.h -- C-ABI of the B200-native cuPSO engine (libcupso.so).
 *
 * Drop-in boundary for the reference's per-iteration PSO step. The reference
 * (psokit, header-only C++20) exposes the path as an engine plugin:
 *
 *   using engine_fn = std::function<run_result(const pso_params&, const fitness_fn&,
 *                                              rng_key, const exec_options&,
 *                                              const iteration_observer&)>;   engines.hpp:12-13
 *   struct engine_entry { std::string name; bool parallel; engine_fn run; };  engines.hpp:15-19
 *
 * The entry points below are what an engine_fn (or any FFI) binds; the C++
 * adapter include/psokit_cuda/engines.hpp builds psokit engine_entry objects
 * on top of them, and paper_2205_01313_b200/ mirrors the same API in Python.
 * Plain pointers and sizes only; every host buffer is caller-owned.
 *
 * Error convention: every call returns a cupso_status; the message of the
 * last failure on the calling thread is cupso_last_error(). The statuses map
 * one-to-one onto the reference's exception types (see cupso_status).
 */
#ifndef CUPSO_H
#define CUPSO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CUPSO_ABI_VERSION 1

/* Status codes. Reference exception each one maps to. */
typedef enum cupso_status {
  CUPSO_OK = 0,
  CUPSO_EINVAL = 1,   /* std::invalid_argument  (params.hpp:33-47, engines.hpp:47, fitness.hpp:102) */
  CUPSO_ERUNTIME = 2, /* std::runtime_error     (group_runtime.hpp:298-308) */
  CUPSO_ELOGIC = 3,   /* std::logic_error       (group_runtime.hpp:201-205) */
  CUPSO_EDOMAIN = 4,  /* std::domain_error      (fitness.hpp:35-42) */
  CUPSO_ECUDA = 5     /* CUDA runtime / device failure (no reference analogue) */
} cupso_status;

/* Mirrors psokit::pso_params (params.hpp:14-25), same field order. */
typedef struct cupso_params {
  double inertia;   /* w  */
  double cognitive; /* c1 */
  double social;    /* c2 */
  double min_pos, max_pos;
  double min_v, max_v;
  uint32_t particle_cnt;
  uint32_t dims;
  uint32_t max_iter;
  uint32_t group_size;
} cupso_params;

/* Aggregation variants ("engines"). The first four restate the reference's
 * parallel engines (engines.hpp:26-37) as classic per-iteration CUDA launches;
 * SYNC, ASYNC and SYNC_F32 are the B200-native engines (register-resident
 * speculative passes / free-running register kernels; see cupso_sync_mode). */
typedef enum cupso_variant {
  CUPSO_REDUCTION = 0,  /* "cuda-reduction": step+block tree, fold kernel  (engine_reduction.hpp:26-93) */
  CUPSO_UNROLLED = 1,   /* "cuda-unrolled" : same, straight-line tree      (engine_reduction.hpp:48-76) */
  CUPSO_QUEUE = 2,      /* "cuda-queue"    : filtered smem queue + fold     (engine_queue.hpp:39-78) */
  CUPSO_QUEUE_LOCK = 3, /* "cuda-queue-lock": fused, lock-guarded commit   (engine_queue.hpp:86-104) */
  CUPSO_SYNC = 4,       /* "cuda-sync"     : speculative passes of K iterations in registers, exact
                           re-run when falsified; grid queue per pass (bitwise == run_serial) */
  CUPSO_ASYNC = 5,      /* "cuda-async"    : free-running register kernel, CAS/seqlock gbest */
  CUPSO_SYNC_F32 = 6    /* "cuda-sync-f32" : FP32 state, packed 64-bit (fitness, index) atomicMax
                           aggregation; statistical (not bitwise) vs the FP64 reference */
} cupso_variant;

/* Read-only view handed to an observer (engine.hpp:29-30 iteration_observer).
 * Arrays are unpadded, axis-major (swarm.hpp:21-24), valid during the call. */
typedef struct cupso_state_view {
  uint32_t particle_cnt, dims;
  const double* positions;  /* particle_cnt*dims */
  const double* velocities; /* particle_cnt*dims */
  const double* fitness;    /* particle_cnt */
  const double* pbest_pos;  /* particle_cnt*dims */
  const double* pbest_fit;  /* particle_cnt */
  double gbest_fit;
  uint32_t gbest_particle;
  const double* gbest_pos;  /* dims */
} cupso_state_view;

typedef void (*cupso_observer_fn)(uint32_t iteration, const cupso_state_view* state, void* user);

/* Mirrors psokit::run_result (engine.hpp:16-26). Pointers are caller-owned
 * buffers of the stated length; any may be NULL to skip that output. */
typedef struct cupso_result {
  double gbest_fit;
  uint32_t gbest_particle;
  double initial_gbest_fit;
  double compute_seconds;    /* device time of the iteration loop (CUDA events) */
  double* gbest_pos;         /* [dims] */
  double* trace;             /* [max_iter] gbest_fit after every iteration */
  uint32_t* trace_particle;  /* [max_iter] gbest particle after every iteration */
  double* queue_occupancy;   /* [max_iter] admitted/particle_cnt; queue variants only */
  uint32_t has_occupancy;    /* out: 1 when queue_occupancy was written (reference: non-empty) */
} cupso_result;

typedef struct cupso_swarm cupso_swarm; /* opaque device-resident swarm */

/* ---- metadata / registry (fitness.hpp:87-103, engines.hpp:21-48) ---- */
int cupso_abi_version(void);
const char* cupso_last_error(void);
int cupso_fitness_id(const char* name);                     /* -1 if unknown (last_error lists known) */
const char* cupso_fitness_name(int fitness_id);
cupso_status cupso_fitness_box(int fitness_id, double* lo, double* hi);
int cupso_variant_id(const char* name);                     /* accepts "cuda-sync" or "sync" */
const char* cupso_variant_name(int variant);
int cupso_variant_count(void);
int cupso_variant_deterministic(int variant);               /* 1: bitwise-equal to serial */
cupso_status cupso_validate_params(const cupso_params* p);  /* params.hpp:33-47 */
cupso_status cupso_make_params(int fitness_id, uint32_t particle_cnt, uint32_t dims,
                               uint32_t max_iter, uint32_t group_size, cupso_params* out);
int cupso_device_count(void);

/* ---- one-shot run: the engine_fn body ---- */
cupso_status cupso_run(const cupso_params* p, int fitness_id, uint64_t seed, int variant,
                       int device, cupso_observer_fn observer, void* user, cupso_result* out);

/* ---- device-resident swarm handle (per-iteration drop-in) ----
 * Not thread-safe; separate handles run independently on their own streams. */
cupso_status cupso_create(const cupso_params* p, int fitness_id, uint64_t seed, int device,
                          cupso_swarm** out);
/* Shard of a larger swarm: local particle k is global particle first+k; RNG
 * counters and tie-breaks use the global index (multi-GPU partition). */
cupso_status cupso_create_shard(const cupso_params* global_params, int fitness_id, uint64_t seed,
                                int device, uint32_t first, uint32_t count, cupso_swarm** out);
cupso_status cupso_destroy(cupso_swarm* h);
cupso_status cupso_init(cupso_swarm* h);            /* init_swarm (swarm.hpp:136-171) on device */
/* Advance `iters` iterations with `variant`; device_seconds (may be NULL)
 * receives the CUDA-event time of exactly those iterations. */
cupso_status cupso_step(cupso_swarm* h, int variant, uint32_t iters, double* device_seconds);
cupso_status cupso_synchronize(cupso_swarm* h);
uint32_t cupso_iteration(const cupso_swarm* h);     /* iterations completed */
cupso_status cupso_get_gbest(cupso_swarm* h, double* fit, uint32_t* particle, double* pos);
cupso_status cupso_get_initial_gbest(cupso_swarm* h, double* fit, uint32_t* particle);
/* Trace entries [first, first+count); any pointer may be NULL. */
cupso_status cupso_get_trace(cupso_swarm* h, uint32_t first, uint32_t count, double* trace,
                             uint32_t* trace_particle, double* occupancy);
/* Unpadded axis-major state; NULL skips an array. fitness is f(positions). */
cupso_status cupso_download_state(cupso_swarm* h, double* positions, double* velocities,
                                  double* fitness, double* pbest_pos, double* pbest_fit);
/* Replace the state (checkpoint resume / external init); gbest given explicitly. */
cupso_status cupso_upload_state(cupso_swarm* h, uint32_t iteration, const double* positions,
                                const double* velocities, const double* pbest_pos,
                                const double* pbest_fit, double gbest_fit, uint32_t gbest_particle,
                                const double* gbest_pos);
/* Device pointers of the padded state (row stride = *ld elements). Valid until
 * the next cupso_step / cupso_upload_state / cupso_destroy on this handle: a
 * speculative cuda-sync step (sync mode 5/6) alternates between two state
 * buffers and may leave the state in the other one -- call again after each
 * step. */
cupso_status cupso_device_state(cupso_swarm* h, double** pos, double** vel, double** pbest_pos,
                                double** pbest_fit, uint64_t* ld);
size_t cupso_device_bytes(const cupso_swarm* h);
int cupso_sync_grid_blocks(const cupso_swarm* h);    /* persistent grid size (after a SYNC step) */
/* How cuda-sync runs on this handle: 0 not yet decided, 1 persistent
 * (k_sync), 2 graph of waves (k_wave), 3 SMEM-resident persistent
 * (k_sync_res), 4 NCCL-sharded per iteration (k_propose/k_commit), 5
 * speculative temporally-blocked passes (k_spec / k_spec_split; dims
 * 1/2/4/8/16/32/64), 6 NCCL-sharded speculative passes (k_spec + one
 * all-gather of a SpecRec per pass + k_spec_commit). */
int cupso_sync_mode(const cupso_swarm* h);
/* Speculative mode bookkeeping since the handle was created: passes that did
 * work, how many of them were falsified by an early admission (each such pass
 * is followed by an exact re-run), and kernel launches issued (passes plus the
 * no-op launches left over when the host's estimate overshoots). */
cupso_status cupso_spec_stats(const cupso_swarm* h, uint64_t* passes, uint64_t* fails, uint64_t* launches);
/* How cuda-async runs on this handle: 0 not yet decided, 1 free-running
 * blocks (k_async), 2 SMEM tiles (k_async_tiled), 3 registers (k_async_reg). */
int cupso_async_mode(const cupso_swarm* h);

/* ---- multi-GPU shard exchange (one exchange step per iteration) ----
 * A candidate record is cupso_record_bytes(dims) bytes:
 *   double fit; uint32_t particle; uint32_t admitted; double pos[dims]
 * (particle = 0xffffffff and fit = -inf when the shard admitted nothing).
 * Per iteration: cupso_shard_propose(t) runs the fused step on this shard and
 * writes the shard's best admitted candidate (or the sentinel) to `record`;
 * the caller all-gathers records across shards (NCCL or host); then
 * cupso_shard_commit applies the same deterministic selection on every
 * shard (beats() among records, strict > against the snapshot). */
size_t cupso_record_bytes(uint32_t dims);
/* Initial exchange after cupso_init on every shard: export the shard's local
 * initial gbest record, then adopt the beats()-max of all shards' records
 * (the whole swarm's init_swarm argmax). NCCL-attached shards do this inside
 * cupso_init. */
cupso_status cupso_shard_snapshot(cupso_swarm* h, void* record_host);
cupso_status cupso_shard_adopt(cupso_swarm* h, const void* records_host, uint32_t nrecords);
cupso_status cupso_shard_propose(cupso_swarm* h, void* record_host);
cupso_status cupso_shard_propose_device(cupso_swarm* h, void* record_dev);  /* stays on stream */
cupso_status cupso_shard_commit(cupso_swarm* h, const void* records_host, uint32_t nrecords);
cupso_status cupso_shard_commit_device(cupso_swarm* h, const void* records_dev, uint32_t nrecords);
/* Host-driven exchange (any transport: MPI, sockets, threads): like a
 * cupso_step(h, CUPSO_SYNC, iters) of an NCCL-initialised shard, but every
 * exchange calls fn(local, all, bytes, user), which must all-gather `bytes`
 * from each of the nranks shards into `all` in rank order and return 0. The
 * record is a speculative pass's SpecRec when the shard runs speculative passes,
 * else the per-iteration candidate record. Every shard of the swarm must call
 * it with the same iters. */
typedef int (*cupso_exchange_fn)(const void* local, void* all, size_t bytes, void* user);
/* Shards of one swarm driven from one process: let a shard that falsifies a
 * speculative pass stop the others early (each sees the others' pass-control
 * word). An optimisation only -- results never depend on it. NCCL shards do the
 * same through CUDA IPC at their first speculative step. */
cupso_status cupso_shard_link(cupso_swarm** shards, uint32_t n);
/* In-process shards (same GPU or peer-accessible GPUs): exchange the pass
 * records inside the pass kernel over peer memory -- the last block of each
 * shard's k_spec pushes its record into every shard's mailbox and waits for
 * theirs, then decides; no all-gather, no commit launch. Each shard must then be
 * stepped (cupso_step, CUPSO_SYNC) from its own host thread, all with the same
 * iteration counts. Also links the early-stop hints (cupso_shard_link). NCCL
 * ranks opt in with CUPSO_SPEC_EXCHANGE=p2p (CUDA IPC). */
cupso_status cupso_shard_p2p(cupso_swarm** shards, uint32_t n);
/* The same across processes through any host channel (what NCCL shards do
 * internally): every rank exports a 192-byte record of CUDA IPC handles
 * (cupso_ipc_handles), the caller all-gathers them in rank order, and every rank
 * opens its peers' (cupso_ipc_link): early-stop hints always, and with p2p the
 * pass-record exchange fused into the pass kernel -- then each rank steps with
 * plain cupso_step (p2p) or cupso_step_exchange (host all-gather). */
cupso_status cupso_ipc_handles(cupso_swarm* h, uint32_t nranks, int p2p, void* out192);
cupso_status cupso_ipc_link(cupso_swarm* h, const void* all_handles, uint32_t nranks, uint32_t rank, int p2p);
cupso_status cupso_step_exchange(cupso_swarm* h, uint32_t iters, uint32_t nranks, cupso_exchange_fn fn,
                                 void* user, double* device_seconds);

/* NCCL-backed exchange: after cupso_nccl_init every cupso_step(h, CUPSO_SYNC, k)
 * on a shard runs propose -> ncclAllGather -> commit per iteration, all on the
 * shard's stream (no host round trip). unique_id = 128-byte ncclUniqueId. */
cupso_status cupso_nccl_init(cupso_swarm* h, const void* unique_id, int nranks, int rank);
cupso_status cupso_nccl_unique_id(void* out128);
void* cupso_stream(cupso_swarm* h);                  /* cudaStream_t of the handle */

/* ---- device self-test hooks (pin the device primitives to the KATs) ---- */
cupso_status cupso_philox_batch(int device, const uint32_t* ctr4, const uint32_t* key2,
                                uint32_t* out4, size_t n);
cupso_status cupso_uniform01_batch(int device, uint64_t seed, const uint32_t* draw4, double* out,
                                   size_t n);
/* Evaluate a fitness on device for n points given axis-major (x[a*n + i]). */
cupso_status cupso_eval_fitness(int device, int fitness_id, const double* x, uint32_t n,
                                uint32_t dims, double* out);
/* Concurrency self-tests, the device analogue of the reference's acceptance
 * criterion 4 (acceptance.cpp:126-200). append: `launches` launches of
 * 2 x SMs blocks at random group sizes 2..1024, 200 rounds each; every round
 * a seeded subset of each block's lanes appends to the block queue and lane 0
 * to a grid queue (queue_append, the product's append); *violations counts
 * duplicate / missing slots and counter mismatches over *trials block-rounds.
 * lock: lane 0 of every warp of 4 x SMs blocks increments a plain counter
 * `iters` times under the product's spin lock (Alg. 3); *counter must equal
 * *expected and *lock_after 0. */
cupso_status cupso_selftest_append(int device, uint32_t launches, uint64_t seed, uint64_t* trials,
                                   uint64_t* violations);
cupso_status cupso_selftest_lock(int device, uint32_t iters, uint64_t* counter, uint64_t* expected,
                                 uint32_t* lock_after);
/* velocity_step/position_step on device for n scalar cases. */
cupso_status cupso_eval_kinematics(int device, const cupso_params* p, const double* v,
                                   const double* x, const double* pbest_x, const double* gbest_x,
                                   const double* r1, const double* r2, double* v_out,
                                   double* x_out, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* CUPSO_H */
