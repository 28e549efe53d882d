// cupso.cu -- host engine and C-ABI of libcupso.so (see include/cupso.h).
//
// The host side owns a device-resident swarm (axis-major SoA, rows padded to
// a multiple of 64 particles so every row is 512-byte aligned and the
// two-particle double2 path never straddles a row), a small control block
// (gbest snapshot/live records, trace arrays, counters) and a stream. A
// "step" launches one of the seven engines for a range of iterations and
// times exactly that range with CUDA events. cuda-sync normally runs the
// speculative register-resident passes of cupso_spec.cuh (second state
// buffer, device-side pass schedule), cuda-async the register-resident
// k_async_reg, cuda-sync-f32 the FP32 passes of cupso_f32.cuh; the classic
// kernels of cupso_kernels.cuh cover the paper's engines and other shapes.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cupso.h"
#include "cupso_kernels.cuh"
#include "cupso_spec.cuh"
#include "cupso_f32.cuh"

using namespace cupso;

namespace {

thread_local std::string g_err;

cupso_status fail(cupso_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(CUPSO_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define TRY(call)                        \
  do {                                   \
    cupso_status s_ = (call);            \
    if (s_ != CUPSO_OK) return s_;       \
  } while (0)

// fitness.hpp:87-95 registry order, plus the harness Rastrigin.
const char* const kFitNames[] = {"cubic", "sphere", "rosenbrock", "griewank", "rastrigin"};
const double kFitLo[] = {-100.0, -100.0, -2.048, -600.0, -5.12};
const double kFitHi[] = {100.0, 100.0, 2.048, 600.0, 5.12};
constexpr int kNumFit = 5;

const char* const kVarNames[] = {"cuda-reduction", "cuda-unrolled", "cuda-queue", "cuda-queue-lock",
                                 "cuda-sync",      "cuda-async",    "cuda-sync-f32"};
constexpr int kNumVar = 7;

// std::to_string(double) == "%f" (params.hpp:38-42 message text)
std::string fstr(double v) {
  char b[64];
  snprintf(b, sizeof b, "%f", v);
  return b;
}

cupso_status validate(const cupso_params* p) {
  if (!p) return fail(CUPSO_EINVAL, "pso_params: null");
  if (!(p->min_pos < p->max_pos))
    return fail(CUPSO_EINVAL, "pso_params: min_pos (%s) must be < max_pos (%s)",
                fstr(p->min_pos).c_str(), fstr(p->max_pos).c_str());
  if (!(p->min_v <= p->max_v))
    return fail(CUPSO_EINVAL, "pso_params: min_v (%s) must be <= max_v (%s)",
                fstr(p->min_v).c_str(), fstr(p->max_v).c_str());
  if (p->particle_cnt < 1) return fail(CUPSO_EINVAL, "pso_params: particle_cnt must be >= 1");
  if (p->dims < 1) return fail(CUPSO_EINVAL, "pso_params: dims must be >= 1");
  if (p->max_iter < 1) return fail(CUPSO_EINVAL, "pso_params: max_iter must be >= 1");
  if (p->group_size < 1) return fail(CUPSO_EINVAL, "pso_params: group_size must be >= 1");
  return CUPSO_OK;
}

uint32_t bit_ceil(uint32_t v) {
  uint32_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// ---------------------------------------------------------- NCCL (dlopen)
// Loaded lazily so the library has no link-time NCCL dependency and shares
// whatever libnccl.so.2 the process (e.g. torch) already mapped.
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void*) = nullptr;
  int (*commInitRank)(void**, int, const void*, int) = nullptr;  // ncclUniqueId by value (128 B)
  int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  bool ok = false;
};
struct NcclUid {
  char internal[128];
};
using CommInitRankFn = int (*)(void**, int, NcclUid, int);

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return a;
    a.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(a.h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<int (*)(void**, int, const void*, int)>(dlsym(a.h, "ncclCommInitRank"));
    a.allGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
        dlsym(a.h, "ncclAllGather"));
    a.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(a.h, "ncclCommDestroy"));
    a.getErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(a.h, "ncclGetErrorString"));
    a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.commDestroy;
    return a;
  }();
  return api;
}

}  // namespace

// ------------------------------------------------------------------ swarm
struct cupso_swarm {
  int device = 0;
  int fid = 0;
  uint64_t seed = 0;
  cupso_params gp{};          // global params (shards: the whole swarm)
  KParams P{};
  KState S{};
  KCtl C{};
  uint32_t T = 0;             // trace capacity = max_iter
  uint32_t t = 0;             // iterations completed
  bool initialized = false;
  double initial_fit = -INFINITY;
  uint32_t initial_particle = kNoParticle;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> allocs;
  unsigned char* ctl_block = nullptr;   // records + counters
  size_t rec_bytes = 0;
  double* eval_buf = nullptr;           // fitness export scratch
  uint32_t groups = 0;
  int sync_grid = 0;
  int step_cfg = 0;
  bool wave = false;
  int wave_cfg = 0;
  bool tile_checked = false;   // tiled cuda-async probed
  uint32_t tile_cap = 0;       // > 0: tiled async available (particles per SMEM tile)
  size_t tile_smem = 0;
  int tile_grid = 0, tile_k = 8;
  bool res_checked = false;    // SMEM-resident cuda-sync probed
  int res_grid = 0;            // > 0: resident mode available (one block per SM)
  uint32_t res_cap = 0;        // particles per block chunk (SMEM rows)
  size_t res_smem = 0;
  uint32_t q_alloc = 0;
  bool spec_checked = false;   // speculative temporally-blocked cuda-sync probed
  int spec_grid = 0;           // > 0: spec mode available
  KState S_alt{};              // the pass's write buffer (ping-pong with S)
  SpecCtl* spec_ctl = nullptr; // device pass schedule
  SpecCtl* spec_host = nullptr;  // pinned mirror
  // pinned staging for the per-run read-backs (trace, trace_idx, admitted,
  // trace_key, gbest record): pageable copies cost ~10 us each
  unsigned char* pin = nullptr;
  size_t pin_bytes = 0;
  uint32_t spec_kmax = 64;
  size_t spec_smem = 0;        // dynamic SMEM of the chosen spec kernel
  // host-driven exchange (cupso_step_exchange): the caller's all-gather
  cupso_exchange_fn xfn = nullptr;
  void* xuser = nullptr;
  uint32_t xranks = 0;
  std::vector<unsigned char> xlocal, xall;
  std::vector<void*> ipc_opened;      // peer SpecCtl mappings (CUDA IPC)
  bool p2p = false;                   // pass records exchanged in-kernel over peer memory
  unsigned char* p2p_buf = nullptr;   // mailbox [2][n] records + flags [n+1]
  uint32_t p2p_buf_n = 0;             // the shard count p2p_buf was sized for
  unsigned char* xrec_dev = nullptr;  // [xranks] gathered records on the device
  size_t xrec_cap = 0;
  unsigned char* spec_rec_local = nullptr;  // this shard's SpecRec of the running pass
  unsigned char* spec_rec_all = nullptr;    // [nranks] all-gathered records (sharded)
  uint64_t spec_passes = 0, spec_fails = 0, spec_launches = 0;
  // FP32 engine (cuda-sync-f32): its own double-buffered FP32 state; the
  // FP64 state stays authoritative for every other entry point (f32_active:
  // the FP32 copy is newer and must be converted back before FP64 use)
  bool f32_ready = false, f32_active = false;
  KState32 S32{}, S32_alt{};
  KParams32 Q{};
  SpecCtl32* spec32_ctl = nullptr;
  const void* f32_kfn = nullptr;
  int f32_grid = 0;
  bool areg_checked = false;   // register-resident cuda-async probed
  int areg_grid = 0, areg_k = 32;
  std::vector<int> async_iters;         // iterations produced by the async variant (trace decode)
  std::vector<uint8_t> is_async;
  std::map<std::tuple<int, uint32_t, uint32_t>, cudaGraphExec_t> graphs;
  // multi-GPU exchange
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  unsigned char* rec_local = nullptr;   // [rec_bytes]
  unsigned char* rec_all = nullptr;     // [nranks * rec_bytes]
};

namespace {

cupso_status dmalloc(cupso_swarm* h, void** p, size_t bytes) {
  CK(cudaMalloc(p, bytes));
  h->allocs.push_back(*p);
  return CUPSO_OK;
}

template <typename Fn>
cupso_status dispatch_fit(int fid, Fn&& fn) {
  switch (fid) {
    case kCubic: fn(std::integral_constant<int, kCubic>{}); break;
    case kSphere: fn(std::integral_constant<int, kSphere>{}); break;
    case kRosenbrock: fn(std::integral_constant<int, kRosenbrock>{}); break;
    case kGriewank: fn(std::integral_constant<int, kGriewank>{}); break;
    case kRastrigin: fn(std::integral_constant<int, kRastrigin>{}); break;
    default: return fail(CUPSO_EINVAL, "unknown fitness id %d", fid);
  }
  return CUPSO_OK;
}

// Fused-step tunings (particles per thread, prefetch, min blocks per SM).
using Cfg0 = StepCfg<2, 0, 5>;
using Cfg1 = StepCfg<2, 1, 3>;
using Cfg2 = StepCfg<1, 0, 8>;
using Cfg3 = StepCfg<1, 1, 6>;
using Cfg4 = StepCfg<2, 0, 6>;
using Cfg5 = StepCfg<1, 0, 6>;
constexpr int kNumCfg = 6;
// Wave-mode tunings: particles per thread, min blocks/SM, axes loaded together.
using WaveCfg0 = StepCfg<1, 0, 8, 1>;  // one particle per thread, 32 registers, 64 warps/SM
using WaveCfg1 = StepCfg<1, 0, 6, 2>;
using WaveCfg2 = StepCfg<1, 0, 5, 4>;
using WaveCfg3 = StepCfg<1, 0, 4, 4>;
using WaveCfg4 = StepCfg<2, 0, 4, 2>;
template <typename Fn>
void dispatch_wave(int c, Fn&& fn) {
  switch (c) {
    case 1: fn(WaveCfg1{}); break;
    case 2: fn(WaveCfg2{}); break;
    case 3: fn(WaveCfg3{}); break;
    case 4: fn(WaveCfg4{}); break;
    default: fn(WaveCfg0{}); break;
  }
}
int default_wave_cfg() {
  if (const char* e = getenv("CUPSO_WAVE_CFG")) return atoi(e);
  return 0;
}

template <typename Fn>
void dispatch_cfg(int c, Fn&& fn) {
  switch (c) {
    case 0: fn(Cfg0{}); break;
    case 1: fn(Cfg1{}); break;
    case 2: fn(Cfg2{}); break;
    case 3: fn(Cfg3{}); break;
    case 4: fn(Cfg4{}); break;
    default: fn(Cfg5{}); break;
  }
}

// cuda-sync runs as one persistent cooperative kernel when the swarm is
// L2-resident (latency/issue-bound: the grid barrier is cheaper than a launch)
// and as a CUDA graph of one-wave-per-iteration launches when it streams
// from HBM (occupancy-bound). Both are bit-identical; CUPSO_SYNC_MODE=
// persistent|wave overrides.
bool use_wave(const KParams& P) {
  if (const char* e = getenv("CUPSO_SYNC_MODE")) {
    if (!strcmp(e, "wave")) return true;
    if (!strcmp(e, "persistent")) return false;
  }
  // measured on B200 (profiles/r01_sync_modes.txt): d=1 streams best as the
  // persistent two-particles-per-thread kernel (LDG.128), d>=2 as waves
  const double state_bytes = static_cast<double>(P.ld) * (3.0 * P.d + 1.0) * 8.0;
  return P.d >= 2 && state_bytes > 64.0 * (1 << 20);
}

int default_step_cfg(const KParams& P) {
  if (const char* e = getenv("CUPSO_STEP_CFG")) {
    const int c = atoi(e);
    if (c >= 0 && c < kNumCfg) return c;
  }
  (void)P;
  return 0;
}

void key_schedule(uint64_t seed, KParams& P) {
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    P.k0[r] = k0;
    P.k1[r] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// c1 / c2 pre-scaled by 2^-53 for vel_step53; exact unless the scaling
// underflows (|c| < 2^-969), in which case the register-resident kernels
// (which rely on it) are not used.
void scale_draws(KParams& P) {
  P.c1s = std::ldexp(P.c1, -53);
  P.c2s = std::ldexp(P.c2, -53);
  auto exact = [](double c) { return c == 0.0 || !std::isfinite(c) || std::fabs(c) >= std::ldexp(1.0, -969); };
  P.scaled_ok = exact(P.c1) && exact(P.c2);
}

int num_sms(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v > 0 ? v : 1;
}

size_t sync_smem(const cupso_swarm* h) { return static_cast<size_t>(h->P.d) * sizeof(double); }
constexpr uint32_t kMaxSyncDims = 12288;  // 96 KiB of dynamic smem for the gbest snapshot

cupso_status ensure_queue(cupso_swarm* h, uint64_t cap);

// Persistent grid: every block co-resident (required by the grid barrier).
cupso_status ensure_sync_grid(cupso_swarm* h) {
  if (h->sync_grid > 0) return CUPSO_OK;
  if (h->P.d > kMaxSyncDims)
    return fail(CUPSO_EINVAL, "cuda-sync/async: dims (%u) above %u", h->P.d, kMaxSyncDims);
  const size_t smem = sync_smem(h);
  int per_sm = 0;
  int np = 1;
  cudaError_t e = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    dispatch_cfg(h->step_cfg, [&](auto CF) {
      using Cfg = decltype(CF);
      np = Cfg::kNP;
      if (smem > 48 * 1024) {
        cudaFuncSetAttribute(k_sync<f, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_async<f, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_propose<f, Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      }
      int a = 0, b = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_sync<f, Cfg>, kSyncThreads, smem);
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_async<f, Cfg>, kSyncThreads, smem);
      per_sm = std::min(a, b);
    });
  });
  CK(e);
  if (per_sm < 1) return fail(CUPSO_ECUDA, "cuda-sync: kernel cannot be resident (occupancy 0)");
  const uint64_t units = (h->P.n + np - 1ull) / np;
  uint64_t grid = static_cast<uint64_t>(per_sm) * num_sms(h->device);
  // keep at least ~2 units per thread of work per block when the swarm is small
  const uint64_t min_work = std::max<uint64_t>(1, units / (2 * kSyncThreads));
  grid = std::max<uint64_t>(1, std::min(grid, min_work));
  h->sync_grid = static_cast<int>(grid);
  TRY(ensure_queue(h, grid));
  return CUPSO_OK;
}

cupso_status ensure_queue(cupso_swarm* h, uint64_t cap) {
  if (h->q_alloc >= cap) return CUPSO_OK;
  void *qf, *qi, *qp;
  TRY(dmalloc(h, &qf, 3 * cap * sizeof(double)));
  TRY(dmalloc(h, &qi, 3 * cap * sizeof(uint32_t)));
  TRY(dmalloc(h, &qp, 3 * cap * h->P.d * sizeof(double)));
  h->C.q_fit = static_cast<double*>(qf);
  h->C.q_idx = static_cast<uint32_t*>(qi);
  h->C.q_pos = static_cast<double*>(qp);
  h->C.q_cap = static_cast<uint32_t>(cap);
  h->q_alloc = static_cast<uint32_t>(cap);
  h->graphs.clear();  // captured graphs hold the old queue pointers
  return CUPSO_OK;
}

// Wave mode of cuda-sync: [t0, t0+iters) as one CUDA graph of k_wave launches.
cupso_status wave_graph(cupso_swarm* h, uint32_t t0, uint32_t iters, cudaGraphExec_t* out) {
  int np = 1;
  dispatch_wave(h->wave_cfg, [&](auto WC) { np = decltype(WC)::kNP; });
  const uint32_t units = static_cast<uint32_t>((h->P.n + np - 1) / np);
  const uint32_t blocks = (units + kSyncThreads - 1) / kSyncThreads;
  TRY(ensure_queue(h, blocks));
  const auto key = std::make_tuple(100 + CUPSO_SYNC, t0, iters);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    *out = it->second;
    return CUPSO_OK;
  }
  if (h->P.d > kMaxSyncDims)
    return fail(CUPSO_EINVAL, "cuda-sync: dims (%u) above %u", h->P.d, kMaxSyncDims);
  const size_t smem = sync_smem(h);
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t le = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    dispatch_wave(h->wave_cfg, [&](auto WC) {
      using W = decltype(WC);
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_wave<f, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (uint32_t t = t0; t < t0 + iters && le == cudaSuccess; ++t) {
        k_wave<f, W><<<blocks, kSyncThreads, smem, h->stream>>>(h->P, h->S, h->C, t);
        le = cudaGetLastError();
      }
    });
  });
  cudaError_t ee = cudaStreamEndCapture(h->stream, &g);
  CK(le);
  CK(ee);
  cudaGraphExec_t ge;
  cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  CK(ie);
  h->graphs[key] = ge;
  *out = ge;
  return CUPSO_OK;
}

cupso_status copy_record(cupso_swarm* h, Rec* dst, const Rec* src) {
  CK(cudaMemcpyAsync(dst, src, h->rec_bytes, cudaMemcpyDeviceToDevice, h->stream));
  return CUPSO_OK;
}

// Classic variants: capture [t0, t0+iters) as one CUDA graph (2 or 1 launches per iteration).
cupso_status classic_graph(cupso_swarm* h, int variant, uint32_t t0, uint32_t iters,
                           cudaGraphExec_t* out) {
  const auto key = std::make_tuple(variant, t0, iters);
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    *out = it->second;
    return CUPSO_OK;
  }
  const uint32_t gs = h->P.gs;
  if (gs > 1024)
    return fail(CUPSO_EINVAL, "%s: group_size (%u) must be <= 1024 (CUDA block limit)",
                kVarNames[variant], gs);
  const uint32_t padded = bit_ceil(gs);
  const size_t smem = padded * (sizeof(double) + sizeof(uint32_t));
  const uint32_t groups = h->groups;
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t le = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    for (uint32_t t = t0; t < t0 + iters && le == cudaSuccess; ++t) {
      switch (variant) {
        case CUPSO_REDUCTION:
          k_classic_step<f, kTree><<<groups, gs, smem, h->stream>>>(h->P, h->S, h->C, t, padded);
          k_classic_fold<kTree><<<1, gs, smem, h->stream>>>(h->P, h->S, h->C, t, groups, padded);
          break;
        case CUPSO_UNROLLED:
          k_classic_step<f, kTreeUnrolled><<<groups, gs, smem, h->stream>>>(h->P, h->S, h->C, t, padded);
          k_classic_fold<kTreeUnrolled><<<1, gs, smem, h->stream>>>(h->P, h->S, h->C, t, groups, padded);
          break;
        case CUPSO_QUEUE:
          k_classic_step<f, kQueue><<<groups, gs, smem, h->stream>>>(h->P, h->S, h->C, t, padded);
          k_classic_fold<kQueue><<<1, gs, smem, h->stream>>>(h->P, h->S, h->C, t, groups, padded);
          break;
        case CUPSO_QUEUE_LOCK:
          k_classic_step<f, kQueueLock><<<groups, gs, smem, h->stream>>>(h->P, h->S, h->C, t, padded);
          break;
      }
      le = cudaGetLastError();
    }
  });
  cudaError_t ee = cudaStreamEndCapture(h->stream, &g);
  CK(le);
  CK(ee);
  cudaGraphExec_t ge;
  cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  CK(ie);
  h->graphs[key] = ge;
  *out = ge;
  return CUPSO_OK;
}

template <int F>
const void* resident_kernel(uint32_t d) {
  return d == 1 ? reinterpret_cast<const void*>(k_sync_res<F, 1>)
                : reinterpret_cast<const void*>(k_sync_res<F, 0>);
}

// SMEM-resident mode of cuda-sync: one 1024-thread block per SM holding its
// chunk of the swarm in shared memory for the whole launch. Possible when the
// chunk's FP64 state (3d+1 doubles per particle) fits the opt-in SMEM limit.
// Returns false (no error) when it does not fit; CUPSO_SYNC_MODE=persistent|wave
// disables it.
bool resident_fits(cupso_swarm* h) {
  if (h->res_checked) return h->res_grid > 0;
  h->res_checked = true;
  if (const char* e = getenv("CUPSO_SYNC_MODE"))
    if (strcmp(e, "resident") != 0 && strcmp(e, "auto") != 0) return false;
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device) != cudaSuccess)
    return false;
  const int nsm = num_sms(h->device);
  const uint64_t cap = (static_cast<uint64_t>(h->P.n) + nsm - 1) / nsm;
  const uint64_t dpad = (h->P.d + 1ull) & ~1ull;
  const uint64_t dyn = (dpad + (3ull * h->P.d + 1ull) * cap) * sizeof(double);
  bool ok = false;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    const void* kfn = resident_kernel<f>(h->P.d);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kfn) != cudaSuccess) return;
    if (dyn + fa.sharedSizeBytes > static_cast<uint64_t>(optin)) return;
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)) !=
        cudaSuccess)
      return;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kResThreads, dyn) != cudaSuccess) return;
    ok = per_sm >= 1;
  });
  cudaGetLastError();  // clear anything the probes left behind
  if (!ok) return false;
  if (ensure_queue(h, nsm) != CUPSO_OK) return false;
  h->res_grid = nsm;
  h->res_cap = static_cast<uint32_t>(cap);
  h->res_smem = static_cast<size_t>(dyn);
  return true;
}

cupso_status launch_resident(cupso_swarm* h, uint32_t t0, uint32_t t1) {
  cudaError_t e = cudaSuccess;
  CK(cudaMemsetAsync(h->C.bar, 0, sizeof(unsigned long long), h->stream));
  CK(cudaMemsetAsync(h->C.q_count, 0, 3 * sizeof(uint32_t), h->stream));
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    uint32_t cap = h->res_cap;
    void* args[] = {&h->P, &h->S, &h->C, &t0, &t1, &cap};
    e = cudaLaunchCooperativeKernel(resident_kernel<f>(h->P.d), dim3(h->res_grid), dim3(kResThreads), args,
                                    h->res_smem, h->stream);
  });
  CK(e);
  return CUPSO_OK;
}

// Tiled (temporally blocked) mode of cuda-async: two 512-thread blocks per SM,
// each cycling SMEM tiles of its particle chunk through K iterations at a
// time. Used when the swarm is larger than what SMEM holds at once (otherwise
// plain k_async is already L2/SMEM friendly). CUPSO_ASYNC_MODE=plain|tiled and
// CUPSO_ASYNC_K override.
template <int F>
const void* tiled_kernel(uint32_t d) {
  return d == 1 ? reinterpret_cast<const void*>(k_async_tiled<F, 1>)
                : reinterpret_cast<const void*>(k_async_tiled<F, 0>);
}

bool tiled_fits(cupso_swarm* h) {
  if (h->tile_checked) return h->tile_cap > 0;
  h->tile_checked = true;
  const char* mode = getenv("CUPSO_ASYNC_MODE");
  if (mode && !strcmp(mode, "plain")) return false;
  const double state_bytes = static_cast<double>(h->P.ld) * (3.0 * h->P.d + 1.0) * 8.0;
  if (!(mode && !strcmp(mode, "tiled")) && state_bytes <= 64.0 * (1 << 20)) return false;
  int per_sm_smem = 0;
  if (cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device) != cudaSuccess)
    return false;
  const uint64_t dpad = (h->P.d + 1ull) & ~1ull;
  bool ok = false;
  uint64_t cap = 0, dyn = 0;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    const void* kfn = tiled_kernel<f>(h->P.d);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kfn) != cudaSuccess) return;
    const int64_t budget = per_sm_smem / 2 - static_cast<int64_t>(fa.sharedSizeBytes) - 1024;
    if (budget <= 0) return;
    cap = (static_cast<uint64_t>(budget) / sizeof(double) - dpad) / (3ull * h->P.d + 1ull);
    cap = cap / 32 * 32;
    if (cap < static_cast<uint64_t>(kTileThreads)) return;
    dyn = (dpad + (3ull * h->P.d + 1ull) * cap) * sizeof(double);
    if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)) != cudaSuccess)
      return;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kTileThreads, dyn) != cudaSuccess) return;
    ok = per_sm >= 2;
  });
  cudaGetLastError();
  if (!ok) return false;
  h->tile_cap = static_cast<uint32_t>(cap);
  h->tile_smem = static_cast<size_t>(dyn);
  h->tile_grid = 2 * num_sms(h->device);
  const char* k = getenv("CUPSO_ASYNC_K");
  // K = 32: tile load/store amortised to ~2 B per particle-update (2^24 x d=1:
  // 121 us/iteration vs 157 at K = 8 and 141 for plain k_async; B200, round 1)
  h->tile_k = k ? std::max(1, atoi(k)) : 32;
  return true;
}

cupso_status launch_tiled(cupso_swarm* h, uint32_t t0, uint32_t t1) {
  CK(cudaMemsetAsync(h->C.seq, 0, sizeof(uint32_t), h->stream));
  cudaError_t e = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    uint32_t cap = h->tile_cap, K = static_cast<uint32_t>(h->tile_k);
    void* args[] = {&h->P, &h->S, &h->C, &t0, &t1, &cap, &K};
    e = cudaLaunchKernel(tiled_kernel<f>(h->P.d), dim3(h->tile_grid), dim3(kTileThreads), args, h->tile_smem,
                         h->stream);
  });
  CK(e);
  return CUPSO_OK;
}

#include "cupso_spec_host.inc"

cupso_status launch_persistent(cupso_swarm* h, int variant, uint32_t t0, uint32_t t1) {
  if (variant == CUPSO_SYNC && resident_fits(h)) return launch_resident(h, t0, t1);
  if (variant == CUPSO_ASYNC && async_reg_fits(h)) return launch_async_reg(h, t0, t1);
  if (variant == CUPSO_ASYNC && tiled_fits(h)) return launch_tiled(h, t0, t1);
  TRY(ensure_sync_grid(h));
  const size_t smem = sync_smem(h);
  cudaError_t e = cudaSuccess;
  // counters: bar (sync), seq (async), q_count[3]
  CK(cudaMemsetAsync(h->C.bar, 0, sizeof(unsigned long long), h->stream));
  CK(cudaMemsetAsync(h->C.seq, 0, sizeof(uint32_t), h->stream));
  CK(cudaMemsetAsync(h->C.q_count, 0, 3 * sizeof(uint32_t), h->stream));
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    dispatch_cfg(h->step_cfg, [&](auto CF) {
      using Cfg = decltype(CF);
      void* args[] = {&h->P, &h->S, &h->C, &t0, &t1};
      if (variant == CUPSO_SYNC)
        e = cudaLaunchCooperativeKernel((void*)k_sync<f, Cfg>, dim3(h->sync_grid), dim3(kSyncThreads),
                                        args, smem, h->stream);
      else
        e = cudaLaunchCooperativeKernel((void*)k_async<f, Cfg>, dim3(h->sync_grid), dim3(kSyncThreads),
                                        args, smem, h->stream);
    });
  });
  CK(e);
  return CUPSO_OK;
}

cupso_status propose_launch(cupso_swarm* h, uint32_t t, unsigned char* record_dev) {
  TRY(ensure_sync_grid(h));
  const size_t smem = sync_smem(h);
  cudaError_t e = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    dispatch_cfg(h->step_cfg, [&](auto CF) {
      using Cfg = decltype(CF);
      k_propose<f, Cfg><<<h->sync_grid, kSyncThreads, smem, h->stream>>>(h->P, h->S, h->C, t, record_dev);
    });
    e = cudaGetLastError();
  });
  CK(e);
  return CUPSO_OK;
}

cupso_status commit_launch(cupso_swarm* h, uint32_t t, const unsigned char* recs, uint32_t n) {
  k_commit<<<1, 256, 0, h->stream>>>(h->P, h->C, t, recs, n, h->rec_bytes, 1);
  CK(cudaGetLastError());
  return CUPSO_OK;
}

// NCCL-backed sharded sync step: propose -> allgather -> commit per iteration.
cupso_status sharded_steps(cupso_swarm* h, uint32_t t0, uint32_t t1) {
  NcclApi& api = nccl();
  for (uint32_t t = t0; t < t1; ++t) {
    TRY(propose_launch(h, t, h->rec_local));
    if (h->comm) {
      const int r = api.allGather(h->rec_local, h->rec_all, h->rec_bytes, /*ncclInt8*/ 0, h->comm,
                                  h->stream);
      if (r != 0)
        return fail(CUPSO_ERUNTIME, "ncclAllGather failed: %s",
                    api.getErrorString ? api.getErrorString(r) : "?");
      TRY(commit_launch(h, t, h->rec_all, static_cast<uint32_t>(h->nranks)));
    } else {  // host callback exchange
      unsigned char* all = nullptr;
      TRY(exchange(h, h->rec_local, h->rec_bytes, &all));
      TRY(commit_launch(h, t, all, h->xranks));
    }
  }
  return CUPSO_OK;
}

#include "cupso_f32_host.inc"

cupso_status do_step(cupso_swarm* h, int variant, uint32_t iters, double* seconds) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  if (variant < 0 || variant >= kNumVar) return fail(CUPSO_EINVAL, "unknown variant %d", variant);
  // The fused kernels stage the gbest position in SMEM (<= kMaxSyncDims axes).
  // Wider swarms run the same synchronous algorithm as the classic fused
  // queue-lock launches, which read it from global memory -- bit-identical.
  // A shard exchanging with others (NCCL, the cupso_step_exchange callback, the
  // peer-memory mailbox, or linked early-stop hints) steps with cuda-sync only:
  // any other variant would run its own slice and let the shards' gbest records
  // diverge while returning OK.
  const bool linked = h->comm || h->xfn || h->p2p || h->C.npeers > 0 || h->nranks > 1;
  if ((variant == CUPSO_SYNC || variant == CUPSO_ASYNC) && h->P.d > kMaxSyncDims) {
    if (linked) return fail(CUPSO_EINVAL, "sharded cuda-sync: dims (%u) above %u", h->P.d, kMaxSyncDims);
    variant = CUPSO_QUEUE_LOCK;
  }
  if (!h->initialized) return fail(CUPSO_ELOGIC, "cupso_step before cupso_init");
  if (static_cast<uint64_t>(h->t) + iters > h->T)
    return fail(CUPSO_EINVAL, "cupso_step: %u + %u iterations exceed max_iter (%u)", h->t, iters, h->T);
  if (linked && variant != CUPSO_SYNC) return fail(CUPSO_EINVAL, "sharded swarms step with cuda-sync only");
  CK(cudaSetDevice(h->device));
  const uint32_t t0 = h->t, t1 = h->t + iters;
  if (variant == CUPSO_SYNC_F32) {
    TRY(ensure_f32(h));
    if (!h->spec_host) {
      void* host = nullptr;
      CK(cudaMallocHost(&host, sizeof(SpecCtl)));
      h->spec_host = static_cast<SpecCtl*>(host);
    }
    if (!h->f32_active && iters) {  // FP64 state -> FP32 copy (outside the timed region)
      k_to_f32<<<conv_blocks(h), 256, 0, h->stream>>>(h->P, h->S, h->S32);
      CK(cudaGetLastError());
      h->f32_active = true;
    }
    CK(cudaMemsetAsync(&h->spec32_ctl->key, 0, sizeof(unsigned long long), h->stream));
    CK(cudaEventRecord(h->ev0, h->stream));
    if (iters) TRY(f32_steps(h, t0, t1));
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaEventSynchronize(h->ev1));
    CK(cudaGetLastError());
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (seconds) *seconds = ms * 1e-3;
    for (uint32_t t = t0; t < t1; ++t) h->is_async[t] = 0;
    h->t = t1;
    return CUPSO_OK;
  }
  TRY(sync_f64(h));
  cudaGraphExec_t ge = nullptr;
  if (iters && variant <= CUPSO_QUEUE_LOCK) TRY(classic_graph(h, variant, t0, iters, &ge));
  // probe outside the timed region (allocates the second state buffer once)
  const bool spec = iters && variant == CUPSO_SYNC && spec_fits(h);
  const bool shard_x = h->comm || h->xfn || h->p2p;  // exchanged with other shards
  if (h->p2p && variant == CUPSO_SYNC && iters && !spec_fits(h))
    return fail(CUPSO_ELOGIC, "peer-memory shards step with speculative passes only");
  const bool wave = variant == CUPSO_SYNC && h->wave && !shard_x && !spec;
  if (iters && wave) {
    TRY(wave_graph(h, t0, iters, &ge));
    CK(cudaMemsetAsync(h->C.q_count, 0, 3 * sizeof(uint32_t), h->stream));
  }
  if (iters && variant == CUPSO_QUEUE_LOCK) TRY(copy_record(h, h->C.live, h->C.snap));
  if (iters && variant == CUPSO_ASYNC) {
    TRY(copy_record(h, h->C.live, h->C.snap));
    CK(cudaMemsetAsync(h->C.trace_key + t0, 0, iters * sizeof(unsigned long long), h->stream));
  }
  if (iters && variant == CUPSO_SYNC && !wave && !spec && !shard_x) resident_fits(h);  // probe outside the timed region
  if (iters && variant == CUPSO_ASYNC && !async_reg_fits(h)) tiled_fits(h);
  if (iters && ((variant == CUPSO_SYNC && !wave && !spec) || variant == CUPSO_ASYNC)) TRY(ensure_sync_grid(h));
  CK(cudaEventRecord(h->ev0, h->stream));
  if (iters) {
    if (ge) {
      CK(cudaGraphLaunch(ge, h->stream));
    } else if (spec) {
      TRY(spec_steps(h, t0, t1));
    } else if (variant == CUPSO_SYNC && (h->comm || h->xfn)) {
      TRY(sharded_steps(h, t0, t1));
    } else {
      constexpr uint32_t kChunk = 1u << 20;  // keeps the barrier counter far from wrap
      for (uint32_t a = t0; a < t1; a += std::min(kChunk, t1 - a))
        TRY(launch_persistent(h, variant, a, a + std::min(kChunk, t1 - a)));
    }
  }
  CK(cudaEventRecord(h->ev1, h->stream));
  CK(cudaEventSynchronize(h->ev1));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  if (seconds) *seconds = ms * 1e-3;
  if (iters && variant == CUPSO_ASYNC) {
    TRY(copy_record(h, h->C.snap, h->C.live));
    CK(cudaStreamSynchronize(h->stream));
  }
  for (uint32_t t = t0; t < t1; ++t) h->is_async[t] = variant == CUPSO_ASYNC;
  h->t = t1;
  return CUPSO_OK;
}

// aux slots serve the classic engines' per-group winners and init_swarm's
// block argmax (at most kInitArgmaxBlocks blocks)
constexpr uint32_t kInitArgmaxBlocks = 1024;
uint64_t aux_entries(const cupso_swarm* h) { return std::max<uint64_t>(h->groups, kInitArgmaxBlocks) + 1; }

cupso_status create_impl(const cupso_params* p, int fid, uint64_t seed, int device, uint32_t first,
                         uint32_t count, cupso_swarm** out) {
  if (!out) return fail(CUPSO_EINVAL, "null output handle");
  *out = nullptr;
  TRY(validate(p));
  if (fid < 0 || fid >= kNumFit) {
    std::string known;
    for (auto n : kFitNames) known += std::string(" ") + n;
    return fail(CUPSO_EINVAL, "unknown fitness id %d; known:%s", fid, known.c_str());
  }
  if (count < 1 || static_cast<uint64_t>(first) + count > p->particle_cnt)
    return fail(CUPSO_EINVAL, "shard [%u, %u) outside the swarm of %u particles", first,
                first + count, p->particle_cnt);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(CUPSO_ECUDA, "no CUDA device available (cuda engines have no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(CUPSO_EINVAL, "device %d out of range [0, %d)", device, ndev);
  CK(cudaSetDevice(device));
  auto* h = new cupso_swarm();
  h->device = device;
  h->fid = fid;
  h->seed = seed;
  h->gp = *p;
  h->T = p->max_iter;
  KParams& P = h->P;
  P.w = p->inertia;
  P.c1 = p->cognitive;
  P.c2 = p->social;
  P.min_pos = p->min_pos;
  P.max_pos = p->max_pos;
  P.min_v = p->min_v;
  P.max_v = p->max_v;
  P.n = count;
  P.d = p->dims;
  P.base = first;
  P.gs = p->group_size;
  P.ld = (static_cast<uint64_t>(count) + 63) / 64 * 64;
  key_schedule(seed, P);
  scale_draws(P);
  h->step_cfg = default_step_cfg(P);
  h->wave = use_wave(P);
  h->wave_cfg = default_wave_cfg();
  h->groups = (count + p->group_size - 1) / p->group_size;
  h->rec_bytes = sizeof(Rec) + sizeof(double) * p->dims;
  h->is_async.assign(h->T, 0);
  auto bail = [&](cupso_status st) {
    cupso_destroy(h);
    return st;
  };
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&h->ev0) != cudaSuccess || cudaEventCreate(&h->ev1) != cudaSuccess)
    return bail(fail(CUPSO_ECUDA, "stream/event creation failed"));
  const size_t cells = P.ld * P.d;
  void *pos, *vel, *pb, *pbf, *ev;
  cupso_status st;
  if ((st = dmalloc(h, &pos, cells * 8)) || (st = dmalloc(h, &vel, cells * 8)) ||
      (st = dmalloc(h, &pb, cells * 8)) || (st = dmalloc(h, &pbf, P.ld * 8)) ||
      (st = dmalloc(h, &ev, P.ld * 8)))
    return bail(st);
  h->S = KState{static_cast<double*>(pos), static_cast<double*>(vel), static_cast<double*>(pb),
                static_cast<double*>(pbf)};
  h->eval_buf = static_cast<double*>(ev);
  // control block: snap rec, live rec, 2 shard records, counters
  const size_t rb = (h->rec_bytes + 15) / 16 * 16;
  const size_t ctl = 4 * rb + 64 + 64 * sizeof(uint32_t);
  void *c, *tr, *ti, *adm, *tk, *af, *ai, *rall;
  if ((st = dmalloc(h, &c, ctl)) || (st = dmalloc(h, &tr, h->T * 8ull)) ||
      (st = dmalloc(h, &ti, h->T * 4ull)) || (st = dmalloc(h, &adm, h->T * 8ull)) ||
      (st = dmalloc(h, &tk, h->T * 8ull)) || (st = dmalloc(h, &af, aux_entries(h) * 8ull)) ||
      (st = dmalloc(h, &ai, aux_entries(h) * 4ull)))
    return bail(st);
  (void)rall;
  h->ctl_block = static_cast<unsigned char*>(c);
  if (cudaMemset(c, 0, ctl) != cudaSuccess) return bail(fail(CUPSO_ECUDA, "memset failed"));
  KCtl& C = h->C;
  C.snap = reinterpret_cast<Rec*>(h->ctl_block);
  C.snap_pos = reinterpret_cast<double*>(h->ctl_block + sizeof(Rec));
  C.live = reinterpret_cast<Rec*>(h->ctl_block + rb);
  C.live_pos = reinterpret_cast<double*>(h->ctl_block + rb + sizeof(Rec));
  h->rec_local = h->ctl_block + 2 * rb;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(h->ctl_block + 4 * rb);
  C.lock = ctr + 0;
  C.ticket = ctr + 1;
  C.bar = reinterpret_cast<unsigned long long*>(ctr + 8);  // 8-byte aligned
  C.seq = ctr + 3;
  C.q_count = ctr + 4;  // [3]
  C.ticket_grp = ctr + 16;  // [64]
  C.trace = static_cast<double*>(tr);
  C.trace_idx = static_cast<uint32_t*>(ti);
  C.admitted = static_cast<unsigned long long*>(adm);
  C.trace_key = static_cast<unsigned long long*>(tk);
  C.aux_fit = static_cast<double*>(af);
  C.aux_idx = static_cast<uint32_t*>(ai);
  *out = h;
  return CUPSO_OK;
}

__global__ void k_clear_trace(KCtl C, uint32_t T) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    C.admitted[t] = 0;
    C.trace_key[t] = 0;
    C.trace[t] = 0.0;
    C.trace_idx[t] = kNoParticle;
  }
}

// The handle's pinned staging area, grown to at least `bytes` (16-byte aligned slices).
cupso_status pinned(cupso_swarm* h, size_t bytes, unsigned char** out) {
  if (h->pin_bytes < bytes) {
    if (h->pin) cudaFreeHost(h->pin);
    h->pin = nullptr;
    h->pin_bytes = 0;
    void* p = nullptr;
    CK(cudaMallocHost(&p, bytes));
    h->pin = static_cast<unsigned char*>(p);
    h->pin_bytes = bytes;
  }
  *out = h->pin;
  return CUPSO_OK;
}
size_t align16(size_t x) { return (x + 15) / 16 * 16; }

cupso_status init_impl(cupso_swarm* h) {
  CK(cudaSetDevice(h->device));
  h->f32_active = false;  // a fresh FP64 swarm
  const int blocks = static_cast<int>(std::min<uint64_t>((h->P.ld + 255) / 256, 148ull * 16));
  cudaError_t e = cudaSuccess;
  dispatch_fit(h->fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    k_init<f><<<blocks, 256, 0, h->stream>>>(h->P, h->S);
    e = cudaGetLastError();
  });
  CK(e);
  const uint32_t nb = static_cast<uint32_t>(std::min<uint64_t>((h->P.n + 255) / 256, kInitArgmaxBlocks));
  k_argmax_blocks<<<nb, 256, 0, h->stream>>>(h->P, h->S.pbf, h->C.aux_fit, h->C.aux_idx);
  k_argmax_final<<<1, 1024, 0, h->stream>>>(h->P, h->S, h->C, nb);
  CK(cudaGetLastError());
  // the per-iteration records, cleared in one launch instead of four memsets
  k_clear_trace<<<static_cast<int>(std::min<uint64_t>((h->T + 255) / 256, 1024)), 256, 0, h->stream>>>(h->C, h->T);
  CK(cudaGetLastError());
  if (h->comm) {  // sharded: the initial gbest is the argmax over all shards
    CK(cudaMemcpyAsync(h->rec_local, h->C.snap, h->rec_bytes, cudaMemcpyDeviceToDevice, h->stream));
    const int rc = nccl().allGather(h->rec_local, h->rec_all, h->rec_bytes, /*ncclInt8*/ 0, h->comm,
                                    h->stream);
    if (rc != 0) return fail(CUPSO_ERUNTIME, "ncclAllGather (init) failed (%d)", rc);
    k_adopt<<<1, 256, 0, h->stream>>>(h->P, h->C, h->rec_all, static_cast<uint32_t>(h->nranks),
                                      h->rec_bytes);
    CK(cudaGetLastError());
  }
  unsigned char* pin = nullptr;
  TRY(pinned(h, align16(sizeof(Rec)), &pin));
  CK(cudaMemcpyAsync(pin, h->C.snap, sizeof(Rec), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  Rec r;
  std::memcpy(&r, pin, sizeof r);
  h->initial_fit = r.fit;
  h->initial_particle = r.particle;
  h->t = 0;
  std::fill(h->is_async.begin(), h->is_async.end(), 0);
  h->initialized = true;
  return CUPSO_OK;
}

cupso_status download_impl(cupso_swarm* h, double* positions, double* velocities, double* fitness,
                           double* pbest_pos, double* pbest_fit) {
  CK(cudaSetDevice(h->device));
  TRY(sync_f64(h));
  const size_t n = h->P.n, d = h->P.d, ld = h->P.ld;
  auto rows = [&](double* dst, const double* src, size_t nrows) -> cupso_status {
    if (!dst) return CUPSO_OK;
    CK(cudaMemcpy2DAsync(dst, n * 8, src, ld * 8, n * 8, nrows, cudaMemcpyDeviceToHost, h->stream));
    return CUPSO_OK;
  };
  TRY(rows(positions, h->S.pos, d));
  TRY(rows(velocities, h->S.vel, d));
  TRY(rows(pbest_pos, h->S.pb, d));
  TRY(rows(pbest_fit, h->S.pbf, 1));
  if (fitness) {
    cudaError_t e = cudaSuccess;
    dispatch_fit(h->fid, [&](auto F) {
      constexpr int f = decltype(F)::value;
      const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148 * 16));
      k_eval<f><<<blocks, 256, 0, h->stream>>>(h->P, h->S.pos, h->eval_buf);
      e = cudaGetLastError();
    });
    CK(e);
    CK(cudaMemcpyAsync(fitness, h->eval_buf, n * 8, cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  return CUPSO_OK;
}

cupso_status gbest_impl(cupso_swarm* h, double* fit, uint32_t* particle, double* pos) {
  CK(cudaSetDevice(h->device));
  unsigned char* buf = nullptr;
  TRY(pinned(h, align16(h->rec_bytes), &buf));
  CK(cudaMemcpyAsync(buf, h->C.snap, h->rec_bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  const Rec* r = reinterpret_cast<const Rec*>(buf);
  if (fit) *fit = r->fit;
  if (particle) *particle = r->particle;
  if (pos) std::memcpy(pos, buf + sizeof(Rec), sizeof(double) * h->P.d);
  return CUPSO_OK;
}

uint64_t decode_key(unsigned long long k) {
  return (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
}

// The trace over [first, first+count); with gfit/gpart/gpos also the gbest
// record, read back under the same synchronisation (cupso_run's result).
cupso_status trace_impl(cupso_swarm* h, uint32_t first, uint32_t count, double* trace,
                        uint32_t* trace_particle, double* occupancy, double* gfit = nullptr,
                        uint32_t* gpart = nullptr, double* gpos = nullptr) {
  if (static_cast<uint64_t>(first) + count > h->t)
    return fail(CUPSO_EINVAL, "trace range [%u, %u) beyond completed iterations (%u)", first,
                first + count, h->t);
  if (!count && !(gfit || gpart || gpos)) return CUPSO_OK;
  CK(cudaSetDevice(h->device));
  // the async cummax needs the prefix; fetch [0, first+count)
  const uint32_t end = first + count;
  const size_t o_ti = align16(end * 8ull), o_adm = o_ti + align16(end * 4ull), o_tk = o_adm + align16(end * 8ull);
  const size_t o_rec = o_tk + align16(end * 8ull);
  unsigned char* buf = nullptr;
  TRY(pinned(h, o_rec + align16(h->rec_bytes), &buf));
  const bool with_gbest = gfit || gpart || gpos;
  if (with_gbest)
    CK(cudaMemcpyAsync(buf + o_rec, h->C.snap, h->rec_bytes, cudaMemcpyDeviceToHost, h->stream));
  double* tr = reinterpret_cast<double*>(buf);
  uint32_t* ti = reinterpret_cast<uint32_t*>(buf + o_ti);
  const unsigned long long* adm = reinterpret_cast<const unsigned long long*>(buf + o_adm);
  const unsigned long long* tk = reinterpret_cast<const unsigned long long*>(buf + o_tk);
  CK(cudaMemcpyAsync(tr, h->C.trace, end * 8ull, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(ti, h->C.trace_idx, end * 4ull, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(buf + o_adm, h->C.admitted, end * 8ull, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(buf + o_tk, h->C.trace_key, end * 8ull, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (with_gbest) {
    const Rec* r = reinterpret_cast<const Rec*>(buf + o_rec);
    if (gfit) *gfit = r->fit;
    if (gpart) *gpart = r->particle;
    if (gpos) std::memcpy(gpos, buf + o_rec + sizeof(Rec), sizeof(double) * h->P.d);
  }
  double prev = h->initial_fit;
  for (uint32_t t = 0; t < end; ++t) {
    if (h->is_async[t]) {
      double v = -INFINITY;
      if (tk[t]) {
        const uint64_t b = decode_key(tk[t]);
        std::memcpy(&v, &b, 8);
      }
      tr[t] = std::max(v, prev);  // gbest is monotone; blocks report the record they saw
      ti[t] = kNoParticle;
    }
    prev = tr[t];
  }
  const double nrm = static_cast<double>(h->gp.particle_cnt);
  for (uint32_t k = 0; k < count; ++k) {
    if (trace) trace[k] = tr[first + k];
    if (trace_particle) trace_particle[k] = ti[first + k];
    if (occupancy) occupancy[k] = static_cast<double>(adm[first + k]) / nrm;
  }
  return CUPSO_OK;
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int cupso_abi_version(void) { return CUPSO_ABI_VERSION; }
const char* cupso_last_error(void) { return g_err.c_str(); }

int cupso_fitness_id(const char* name) {
  if (name)
    for (int i = 0; i < kNumFit; ++i)
      if (std::strcmp(name, kFitNames[i]) == 0) return i;
  std::string known;
  for (auto n : kFitNames) known += std::string(" ") + n;
  fail(CUPSO_EINVAL, "unknown fitness '%s'; known:%s", name ? name : "(null)", known.c_str());
  return -1;
}

const char* cupso_fitness_name(int id) { return (id >= 0 && id < kNumFit) ? kFitNames[id] : nullptr; }

cupso_status cupso_fitness_box(int id, double* lo, double* hi) {
  if (id < 0 || id >= kNumFit) return fail(CUPSO_EINVAL, "unknown fitness id %d", id);
  if (lo) *lo = kFitLo[id];
  if (hi) *hi = kFitHi[id];
  return CUPSO_OK;
}

int cupso_variant_id(const char* name) {
  if (name)
    for (int i = 0; i < kNumVar; ++i)
      if (std::strcmp(name, kVarNames[i]) == 0 || std::strcmp(name, kVarNames[i] + 5) == 0) return i;
  std::string known;
  for (auto n : kVarNames) known += std::string(" ") + n;
  fail(CUPSO_EINVAL, "unknown engine '%s'; known:%s", name ? name : "(null)", known.c_str());
  return -1;
}

const char* cupso_variant_name(int v) { return (v >= 0 && v < kNumVar) ? kVarNames[v] : nullptr; }
int cupso_variant_count(void) { return kNumVar; }
int cupso_variant_deterministic(int v) { return v >= 0 && v < CUPSO_ASYNC; }  // FP32 is statistical

cupso_status cupso_validate_params(const cupso_params* p) { return validate(p); }

cupso_status cupso_make_params(int fid, uint32_t particle_cnt, uint32_t dims, uint32_t max_iter,
                               uint32_t group_size, cupso_params* out) {
  if (fid < 0 || fid >= kNumFit) return fail(CUPSO_EINVAL, "unknown fitness id %d", fid);
  if (!out) return fail(CUPSO_EINVAL, "null output");
  cupso_params p{};  // params.hpp:52-66
  p.inertia = 1.0;
  p.cognitive = 2.0;
  p.social = 2.0;
  p.min_pos = kFitLo[fid];
  p.max_pos = kFitHi[fid];
  p.max_v = (kFitHi[fid] - kFitLo[fid]) / 2.0;
  p.min_v = -p.max_v;
  p.particle_cnt = particle_cnt;
  p.dims = dims;
  p.max_iter = max_iter;
  p.group_size = group_size;
  *out = p;
  return validate(&p);
}

int cupso_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

cupso_status cupso_create(const cupso_params* p, int fid, uint64_t seed, int device, cupso_swarm** out) {
  if (!p) return fail(CUPSO_EINVAL, "pso_params: null");
  return create_impl(p, fid, seed, device, 0, p->particle_cnt, out);
}

cupso_status cupso_create_shard(const cupso_params* p, int fid, uint64_t seed, int device,
                                uint32_t first, uint32_t count, cupso_swarm** out) {
  if (!p) return fail(CUPSO_EINVAL, "pso_params: null");
  return create_impl(p, fid, seed, device, first, count, out);
}

cupso_status cupso_destroy(cupso_swarm* h) {
  if (!h) return CUPSO_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  if (h->comm && nccl().ok) nccl().commDestroy(h->comm);
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : h->allocs) cudaFree(p);
  if (h->spec_host) cudaFreeHost(h->spec_host);
  if (h->pin) cudaFreeHost(h->pin);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return CUPSO_OK;
}

cupso_status cupso_init(cupso_swarm* h) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  return init_impl(h);
}

cupso_status cupso_step(cupso_swarm* h, int variant, uint32_t iters, double* device_seconds) {
  return do_step(h, variant, iters, device_seconds);
}

cupso_status cupso_step_exchange(cupso_swarm* h, uint32_t iters, uint32_t nranks, cupso_exchange_fn fn,
                                 void* user, double* device_seconds) {
  if (!h || !fn) return fail(CUPSO_EINVAL, "null argument");
  if (nranks < 1) return fail(CUPSO_EINVAL, "cupso_step_exchange: nranks must be >= 1");
  if (h->comm) return fail(CUPSO_EINVAL, "cupso_step_exchange: the handle exchanges over NCCL");
  h->xfn = fn;
  h->xuser = user;
  h->xranks = nranks;
  const cupso_status st = do_step(h, CUPSO_SYNC, iters, device_seconds);
  h->xfn = nullptr;
  h->xuser = nullptr;
  return st;
}

cupso_status cupso_ipc_handles(cupso_swarm* h, uint32_t nranks, int p2p, void* out) {
  if (!h || !out) return fail(CUPSO_EINVAL, "null argument");
  if (nranks < 1 || nranks > 16) return fail(CUPSO_EINVAL, "cupso_ipc_handles: 1..16 ranks");
  CK(cudaSetDevice(h->device));
  if (!spec_fits(h)) return fail(CUPSO_EINVAL, "cupso_ipc_handles: no speculative kernel for this shape");
  IpcSlot s;
  ipc_export(h, nranks, p2p != 0, &s);
  std::memcpy(out, &s, sizeof s);
  return CUPSO_OK;
}

cupso_status cupso_ipc_link(cupso_swarm* h, const void* all, uint32_t nranks, uint32_t rank, int p2p) {
  if (!h || !all) return fail(CUPSO_EINVAL, "null argument");
  if (nranks < 1 || nranks > 16 || rank >= nranks) return fail(CUPSO_EINVAL, "cupso_ipc_link: bad rank");
  CK(cudaSetDevice(h->device));
  std::vector<IpcSlot> slots(nranks);
  std::memcpy(slots.data(), all, sizeof(IpcSlot) * nranks);
  std::vector<unsigned char*> boxes;
  const bool box_ok = ipc_open(h, slots.data(), nranks, rank, boxes);
  if (p2p) {
    if (!box_ok) return fail(CUPSO_ERUNTIME, "cupso_ipc_link: a peer mailbox could not be mapped");
    p2p_enable(h, boxes, nranks, rank);
  }
  return CUPSO_OK;
}

cupso_status cupso_shard_p2p(cupso_swarm** shards, uint32_t n) {
  if (!shards || n < 1 || n > 16) return fail(CUPSO_EINVAL, "cupso_shard_p2p: 1..16 shards");
  for (uint32_t i = 0; i < n; ++i) {
    cupso_swarm* h = shards[i];
    if (!h) return fail(CUPSO_EINVAL, "null shard handle");
    if (h->comm) return fail(CUPSO_EINVAL, "cupso_shard_p2p: NCCL shards use CUPSO_SPEC_EXCHANGE=p2p");
    CK(cudaSetDevice(h->device));
    if (!spec_fits(h))
      return fail(CUPSO_EINVAL, "cupso_shard_p2p: no speculative kernel for this shape (dims %u)", h->P.d);
    if (h->p2p_buf && h->p2p_buf_n != n)  // slots and the exchange counter are laid out for p2p_buf_n
      return fail(CUPSO_EINVAL, "cupso_shard_p2p: shard already linked with %u shards, not %u", h->p2p_buf_n, n);
    if (!h->p2p_buf) {
      void* b;
      TRY(dmalloc(h, &b, p2p_bytes(h, n)));
      CK(cudaMemset(b, 0, p2p_bytes(h, n)));
      h->p2p_buf = static_cast<unsigned char*>(b);
      h->p2p_buf_n = n;
    }
  }
  TRY(cupso_shard_link(shards, n));  // early-stop hints too
  for (uint32_t i = 0; i < n; ++i) {
    KCtl& C = shards[i]->C;
    for (uint32_t r = 0; r < n; ++r) {
      C.mbox[r] = shards[r]->p2p_buf;
      C.flag[r] = p2p_flags(shards[r], shards[r]->p2p_buf, n);
    }
    C.p2p_n = n;
    C.p2p_rank = i;
    shards[i]->p2p = true;
  }
  return CUPSO_OK;
}

cupso_status cupso_shard_link(cupso_swarm** shards, uint32_t n) {
  if (!shards || n < 1 || n > 16) return fail(CUPSO_EINVAL, "cupso_shard_link: 1..16 shards");
  for (uint32_t i = 0; i < n; ++i) {
    if (!shards[i]) return fail(CUPSO_EINVAL, "null shard handle");
    if (shards[i]->comm)
      return fail(CUPSO_EINVAL, "cupso_shard_link: NCCL shards link their peers themselves (CUDA IPC)");
    CK(cudaSetDevice(shards[i]->device));
    if (!spec_fits(shards[i])) return CUPSO_OK;  // no speculative passes on this shape: nothing to link
  }
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t np = 0;
    for (uint32_t j = 0; j < n; ++j) {
      if (j == i) continue;
      if (shards[j]->device != shards[i]->device) {
        CK(cudaSetDevice(shards[i]->device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(shards[j]->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
      shards[i]->C.peer_tmin[np++] = &shards[j]->spec_ctl->tmin;
    }
    shards[i]->C.npeers = np;
  }
  return CUPSO_OK;
}

cupso_status cupso_synchronize(cupso_swarm* h) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  return CUPSO_OK;
}

uint32_t cupso_iteration(const cupso_swarm* h) { return h ? h->t : 0; }

cupso_status cupso_get_gbest(cupso_swarm* h, double* fit, uint32_t* particle, double* pos) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  return gbest_impl(h, fit, particle, pos);
}

cupso_status cupso_get_initial_gbest(cupso_swarm* h, double* fit, uint32_t* particle) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  if (fit) *fit = h->initial_fit;
  if (particle) *particle = h->initial_particle;
  return CUPSO_OK;
}

cupso_status cupso_get_trace(cupso_swarm* h, uint32_t first, uint32_t count, double* trace,
                             uint32_t* trace_particle, double* occupancy) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  return trace_impl(h, first, count, trace, trace_particle, occupancy);
}

cupso_status cupso_download_state(cupso_swarm* h, double* positions, double* velocities,
                                  double* fitness, double* pbest_pos, double* pbest_fit) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  return download_impl(h, positions, velocities, fitness, pbest_pos, pbest_fit);
}

cupso_status cupso_upload_state(cupso_swarm* h, uint32_t iteration, const double* positions,
                                const double* velocities, const double* pbest_pos,
                                const double* pbest_fit, double gbest_fit, uint32_t gbest_particle,
                                const double* gbest_pos) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  if (!positions || !velocities || !pbest_pos || !pbest_fit || !gbest_pos)
    return fail(CUPSO_EINVAL, "cupso_upload_state: all state arrays are required");
  if (iteration > h->T) return fail(CUPSO_EINVAL, "iteration %u beyond max_iter %u", iteration, h->T);
  CK(cudaSetDevice(h->device));
  const size_t n = h->P.n, d = h->P.d, ld = h->P.ld;
  h->f32_active = false;  // the uploaded FP64 state is authoritative
  // neutral padding, then the rows
  if (!h->initialized) TRY(init_impl(h));
  auto rows = [&](double* dst, const double* src, size_t nrows) -> cupso_status {
    CK(cudaMemcpy2DAsync(dst, ld * 8, src, n * 8, n * 8, nrows, cudaMemcpyHostToDevice, h->stream));
    return CUPSO_OK;
  };
  TRY(rows(h->S.pos, positions, d));
  TRY(rows(h->S.vel, velocities, d));
  TRY(rows(h->S.pb, pbest_pos, d));
  TRY(rows(h->S.pbf, pbest_fit, 1));
  std::vector<unsigned char> rec(h->rec_bytes);
  Rec r{gbest_fit, gbest_particle, 0u};
  std::memcpy(rec.data(), &r, sizeof r);
  std::memcpy(rec.data() + sizeof(Rec), gbest_pos, d * 8);
  CK(cudaMemcpyAsync(h->C.snap, rec.data(), h->rec_bytes, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(h->C.live, rec.data(), h->rec_bytes, cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->t = iteration;
  h->initialized = true;
  return CUPSO_OK;
}

cupso_status cupso_device_state(cupso_swarm* h, double** pos, double** vel, double** pbest_pos,
                                double** pbest_fit, uint64_t* ld) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  TRY(sync_f64(h));
  CK(cudaStreamSynchronize(h->stream));
  if (pos) *pos = h->S.pos;
  if (vel) *vel = h->S.vel;
  if (pbest_pos) *pbest_pos = h->S.pb;
  if (pbest_fit) *pbest_fit = h->S.pbf;
  if (ld) *ld = h->P.ld;
  return CUPSO_OK;
}

size_t cupso_device_bytes(const cupso_swarm* h) {
  if (!h) return 0;
  return h->P.ld * (3ull * h->P.d + 2) * 8;
}

int cupso_sync_grid_blocks(const cupso_swarm* h) {
  if (!h) return 0;
  if (h->spec_grid > 0) return h->spec_grid;
  return h->res_grid > 0 ? h->res_grid : h->sync_grid;
}

int cupso_async_mode(const cupso_swarm* h) {
  if (!h) return 0;
  if (h->areg_grid > 0) return 3;
  if (h->tile_cap > 0) return 2;
  return h->sync_grid > 0 ? 1 : 0;
}

cupso_status cupso_spec_stats(const cupso_swarm* h, uint64_t* passes, uint64_t* fails, uint64_t* launches) {
  if (!h) return fail(CUPSO_EINVAL, "null swarm handle");
  if (passes) *passes = h->spec_passes;
  if (fails) *fails = h->spec_fails;
  if (launches) *launches = h->spec_launches;
  return CUPSO_OK;
}

int cupso_sync_mode(const cupso_swarm* h) {
  if (!h) return 0;
  if (h->comm) return h->spec_grid > 0 ? 6 : 4;
  if (h->spec_grid > 0) return 5;
  if (h->wave) return 2;
  if (h->res_grid > 0) return 3;
  return h->sync_grid > 0 ? 1 : 0;
}

size_t cupso_record_bytes(uint32_t dims) { return sizeof(Rec) + sizeof(double) * dims; }

cupso_status cupso_shard_propose_device(cupso_swarm* h, void* record_dev) {
  if (!h || !record_dev) return fail(CUPSO_EINVAL, "null argument");
  if (!h->initialized) return fail(CUPSO_ELOGIC, "propose before cupso_init");
  if (h->t >= h->T) return fail(CUPSO_EINVAL, "swarm already ran max_iter (%u) iterations", h->T);
  CK(cudaSetDevice(h->device));
  TRY(sync_f64(h));
  return propose_launch(h, h->t, static_cast<unsigned char*>(record_dev));
}

cupso_status cupso_shard_propose(cupso_swarm* h, void* record_host) {
  if (!h || !record_host) return fail(CUPSO_EINVAL, "null argument");
  TRY(cupso_shard_propose_device(h, h->rec_local));
  CK(cudaMemcpyAsync(record_host, h->rec_local, h->rec_bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return CUPSO_OK;
}

cupso_status cupso_shard_commit_device(cupso_swarm* h, const void* records_dev, uint32_t nrecords) {
  if (!h || !records_dev) return fail(CUPSO_EINVAL, "null argument");
  if (h->t >= h->T) return fail(CUPSO_EINVAL, "swarm already ran max_iter (%u) iterations", h->T);
  CK(cudaSetDevice(h->device));
  TRY(commit_launch(h, h->t, static_cast<const unsigned char*>(records_dev), nrecords));
  h->is_async[h->t] = 0;
  h->t += 1;
  return CUPSO_OK;
}

cupso_status cupso_shard_snapshot(cupso_swarm* h, void* record_host) {
  if (!h || !record_host) return fail(CUPSO_EINVAL, "null argument");
  if (!h->initialized) return fail(CUPSO_ELOGIC, "snapshot before cupso_init");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(record_host, h->C.snap, h->rec_bytes, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return CUPSO_OK;
}

cupso_status cupso_shard_adopt(cupso_swarm* h, const void* records_host, uint32_t nrecords) {
  if (!h || !records_host) return fail(CUPSO_EINVAL, "null argument");
  if (!h->initialized) return fail(CUPSO_ELOGIC, "adopt before cupso_init");
  CK(cudaSetDevice(h->device));
  void* d = nullptr;
  CK(cudaMallocAsync(&d, h->rec_bytes * nrecords, h->stream));
  CK(cudaMemcpyAsync(d, records_host, h->rec_bytes * nrecords, cudaMemcpyHostToDevice, h->stream));
  k_adopt<<<1, 256, 0, h->stream>>>(h->P, h->C, static_cast<const unsigned char*>(d), nrecords, h->rec_bytes);
  CK(cudaGetLastError());
  cudaFreeAsync(d, h->stream);
  Rec r;
  CK(cudaMemcpyAsync(&r, h->C.snap, sizeof r, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (h->t == 0) {
    h->initial_fit = r.fit;
    h->initial_particle = r.particle;
  }
  return CUPSO_OK;
}

cupso_status cupso_shard_commit(cupso_swarm* h, const void* records_host, uint32_t nrecords) {
  if (!h || !records_host) return fail(CUPSO_EINVAL, "null argument");
  CK(cudaSetDevice(h->device));
  void* d = nullptr;
  CK(cudaMallocAsync(&d, h->rec_bytes * nrecords, h->stream));
  CK(cudaMemcpyAsync(d, records_host, h->rec_bytes * nrecords, cudaMemcpyHostToDevice, h->stream));
  cupso_status st = cupso_shard_commit_device(h, d, nrecords);
  cudaFreeAsync(d, h->stream);
  CK(cudaStreamSynchronize(h->stream));
  return st;
}

cupso_status cupso_nccl_unique_id(void* out128) {
  NcclApi& api = nccl();
  if (!api.ok) return fail(CUPSO_ERUNTIME, "libnccl.so.2 not loadable");
  const int r = api.getUniqueId(out128);
  if (r != 0) return fail(CUPSO_ERUNTIME, "ncclGetUniqueId failed (%d)", r);
  return CUPSO_OK;
}

cupso_status cupso_nccl_init(cupso_swarm* h, const void* unique_id, int nranks, int rank) {
  if (!h || !unique_id) return fail(CUPSO_EINVAL, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CUPSO_EINVAL, "bad rank %d of %d", rank, nranks);
  NcclApi& api = nccl();
  if (!api.ok) return fail(CUPSO_ERUNTIME, "libnccl.so.2 not loadable");
  CK(cudaSetDevice(h->device));
  NcclUid uid;
  std::memcpy(uid.internal, unique_id, 128);
  void* comm = nullptr;
  const int r = reinterpret_cast<CommInitRankFn>(api.commInitRank)(&comm, nranks, uid, rank);
  if (r != 0)
    return fail(CUPSO_ERUNTIME, "ncclCommInitRank failed: %s", api.getErrorString ? api.getErrorString(r) : "?");
  void* all = nullptr;
  TRY(dmalloc(h, &all, h->rec_bytes * nranks));
  h->rec_all = static_cast<unsigned char*>(all);
  h->comm = comm;
  h->nranks = nranks;
  if (h->spec_rec_all) {  // spec buffers set up before the exchange existed: size them for nranks
    void* ra = nullptr;
    TRY(dmalloc(h, &ra, spec_rec_bytes(h->P.d) * nranks));
    h->spec_rec_all = static_cast<unsigned char*>(ra);
  }
  h->rank = rank;
  return CUPSO_OK;
}

void* cupso_stream(cupso_swarm* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

}  // extern "C"

// ------------------------------------------------------------- one-shot run
namespace {
// One cached swarm per thread (handles are not thread-safe; separate threads
// keep separate swarms). Deliberately never destroyed at exit: freeing CUDA
// memory during static destruction is unsafe, and the process is ending.
struct RunCache {
  cupso_swarm* h = nullptr;
  cupso_params p{};
  int fid = -1, device = -1;
  cupso_swarm* take(const cupso_params* q, int f, int dev) {
    if (h && fid == f && device == dev && std::memcmp(&p, q, sizeof p) == 0) {
      cupso_swarm* r = h;
      h = nullptr;
      return r;
    }
    return nullptr;
  }
  void put(cupso_swarm* s) {
    if (h && h != s) cupso_destroy(h);
    h = s;
    p = s->gp;
    fid = s->fid;
    device = s->device;
  }
};
RunCache& run_cache() {
  static thread_local RunCache* c = new RunCache();
  return *c;
}
}  // namespace

extern "C" {
cupso_status cupso_run(const cupso_params* p, int fid, uint64_t seed, int variant, int device,
                       cupso_observer_fn observer, void* user, cupso_result* out) {
  if (!out) return fail(CUPSO_EINVAL, "null result");
  TRY(validate(p));
  if (variant < 0 || variant >= kNumVar) return fail(CUPSO_EINVAL, "unknown variant %d", variant);
  // Repeated runs of the same shape on a thread reuse the device swarm
  // (allocation, stream, events, probes) instead of re-creating it; only the
  // Philox key schedule changes with the seed. Graphs bake kernel parameters
  // in at capture, so they are dropped when the seed changes.
  cupso_swarm* h = run_cache().take(p, fid, device);
  if (h) {
    if (h->seed != seed) {
      for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
      h->graphs.clear();
      h->seed = seed;
      key_schedule(seed, h->P);
    }
  } else {
    TRY(cupso_create(p, fid, seed, device, &h));
  }
  struct Guard {
    cupso_swarm* h;
    ~Guard() { run_cache().put(h); }
  } guard{h};
  TRY(init_impl(h));
  out->initial_gbest_fit = h->initial_fit;
  double total = 0.0;
  if (!observer) {
    TRY(do_step(h, variant, p->max_iter, &total));
  } else {
    const size_t n = p->particle_cnt, d = p->dims;
    std::vector<double> pos(n * d), vel(n * d), fit(n), pb(n * d), pbf(n), gpos(d);
    for (uint32_t t = 0; t < p->max_iter; ++t) {
      double s = 0.0;
      TRY(do_step(h, variant, 1, &s));
      total += s;
      TRY(download_impl(h, pos.data(), vel.data(), fit.data(), pb.data(), pbf.data()));
      cupso_state_view v{};
      v.particle_cnt = p->particle_cnt;
      v.dims = p->dims;
      v.positions = pos.data();
      v.velocities = vel.data();
      v.fitness = fit.data();
      v.pbest_pos = pb.data();
      v.pbest_fit = pbf.data();
      TRY(gbest_impl(h, &v.gbest_fit, &v.gbest_particle, gpos.data()));
      v.gbest_pos = gpos.data();
      observer(t, &v, user);
    }
  }
  out->compute_seconds = total;
  TRY(trace_impl(h, 0, p->max_iter, out->trace, out->trace_particle,
                 (variant == CUPSO_REDUCTION || variant == CUPSO_UNROLLED) ? nullptr : out->queue_occupancy,
                 &out->gbest_fit, &out->gbest_particle, out->gbest_pos));
  out->has_occupancy = !(variant == CUPSO_REDUCTION || variant == CUPSO_UNROLLED);
  return CUPSO_OK;
}

// ------------------------------------------------------ self-test hooks
}  // extern "C"

namespace {
__global__ void k_philox_batch(const uint32_t* ctr4, const uint32_t* key2, uint32_t* out4, size_t n) {
  for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    KParams P{};
    uint32_t k0 = key2[2 * k], k1 = key2[2 * k + 1];
    for (int r = 0; r < 10; ++r) {
      P.k0[r] = k0;
      P.k1[r] = k1;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t c0 = ctr4[4 * k], c1 = ctr4[4 * k + 1], c2 = ctr4[4 * k + 2], c3 = ctr4[4 * k + 3];
    philox10(c0, c1, c2, c3, P);
    out4[4 * k] = c0;
    out4[4 * k + 1] = c1;
    out4[4 * k + 2] = c2;
    out4[4 * k + 3] = c3;
  }
}
__global__ void k_uniform_batch(KParams P, const uint32_t* draw4, double* out, size_t n) {
  for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    out[k] = uniform01(P, draw4[4 * k], draw4[4 * k + 1], draw4[4 * k + 2], draw4[4 * k + 3]);
}
__global__ void k_kin_batch(KParams P, const double* v, const double* x, const double* pb,
                            const double* g, const double* r1, const double* r2, double* vo,
                            double* xo, size_t n) {
  for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const double nv = vel_step(P, v[k], x[k], pb[k], g[k], r1[k], r2[k]);
    vo[k] = nv;
    xo[k] = pos_step(P, x[k], nv);
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n * sizeof(T) + 16); }
};
}  // namespace

extern "C" {

cupso_status cupso_philox_batch(int device, const uint32_t* ctr4, const uint32_t* key2, uint32_t* out4,
                                size_t n) {
  if (!n) return CUPSO_OK;
  CK(cudaSetDevice(device));
  DevBuf<uint32_t> c, k, o;
  CK(c.alloc(4 * n));
  CK(k.alloc(2 * n));
  CK(o.alloc(4 * n));
  CK(cudaMemcpy(c.p, ctr4, 16 * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(k.p, key2, 8 * n, cudaMemcpyHostToDevice));
  k_philox_batch<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256>>>(c.p, k.p, o.p, n);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out4, o.p, 16 * n, cudaMemcpyDeviceToHost));
  return CUPSO_OK;
}

cupso_status cupso_uniform01_batch(int device, uint64_t seed, const uint32_t* draw4, double* out, size_t n) {
  if (!n) return CUPSO_OK;
  CK(cudaSetDevice(device));
  KParams P{};
  key_schedule(seed, P);
  DevBuf<uint32_t> dr;
  DevBuf<double> o;
  CK(dr.alloc(4 * n));
  CK(o.alloc(n));
  CK(cudaMemcpy(dr.p, draw4, 16 * n, cudaMemcpyHostToDevice));
  k_uniform_batch<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256>>>(P, dr.p, o.p, n);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, o.p, 8 * n, cudaMemcpyDeviceToHost));
  return CUPSO_OK;
}

cupso_status cupso_selftest_append(int device, uint32_t launches, uint64_t seed, uint64_t* trials,
                                   uint64_t* violations) {
  if (!trials || !violations) return fail(CUPSO_EINVAL, "cupso_selftest_append: null output");
  CK(cudaSetDevice(device));
  const uint32_t grid = 2u * static_cast<uint32_t>(num_sms(device)), rounds = 200;
  const uint32_t cap = grid * rounds;
  DevBuf<uint32_t> gq;
  DevBuf<unsigned long long> bad;
  CK(gq.alloc(1 + cap));
  CK(bad.alloc(1));
  std::vector<uint32_t> seen(1 + cap);
  uint64_t x = seed, tr = 0, vio = 0;
  auto next = [&x] {  // splitmix64
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  for (uint32_t l = 0; l < launches; ++l) {
    const uint32_t gs = 2 + static_cast<uint32_t>(next() % 1023);  // group sizes 2..1024
    const uint32_t salt = static_cast<uint32_t>(next());
    CK(cudaMemset(gq.p, 0, 4ull * (1 + cap)));
    CK(cudaMemset(bad.p, 0, 8));
    k_stress_append<<<grid, gs, gs * sizeof(uint32_t)>>>(rounds, salt, gq.p, gq.p + 1, cap, bad.p);
    CK(cudaGetLastError());
    unsigned long long b = 0;
    CK(cudaMemcpy(&b, bad.p, 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(seen.data(), gq.p, 4ull * (1 + cap), cudaMemcpyDeviceToHost));
    vio += b + (seen[0] != cap);
    for (uint32_t i = 0; i < cap; ++i) vio += seen[1 + i] != 1u;
    tr += static_cast<uint64_t>(grid) * rounds;
  }
  *trials = tr;
  *violations = vio;
  return CUPSO_OK;
}

cupso_status cupso_selftest_lock(int device, uint32_t iters, uint64_t* counter, uint64_t* expected,
                                 uint32_t* lock_after) {
  if (!counter || !expected || !lock_after) return fail(CUPSO_EINVAL, "cupso_selftest_lock: null output");
  CK(cudaSetDevice(device));
  const uint32_t grid = 4u * static_cast<uint32_t>(num_sms(device)), threads = 256;
  DevBuf<uint32_t> lk;
  DevBuf<unsigned long long> c;
  CK(lk.alloc(1));
  CK(c.alloc(1));
  CK(cudaMemset(lk.p, 0, 4));
  CK(cudaMemset(c.p, 0, 8));
  k_stress_lock<<<grid, threads>>>(iters, lk.p, c.p);
  CK(cudaGetLastError());
  unsigned long long v = 0;
  CK(cudaMemcpy(&v, c.p, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lock_after, lk.p, 4, cudaMemcpyDeviceToHost));
  *counter = v;
  *expected = static_cast<uint64_t>(grid) * (threads / 32) * iters;
  return CUPSO_OK;
}

cupso_status cupso_eval_fitness(int device, int fid, const double* x, uint32_t n, uint32_t dims,
                                double* out) {
  if (fid < 0 || fid >= kNumFit) return fail(CUPSO_EINVAL, "unknown fitness id %d", fid);
  if (!n) return CUPSO_OK;
  CK(cudaSetDevice(device));
  KParams P{};
  P.n = n;
  P.d = dims;
  P.ld = n;
  DevBuf<double> dx, o;
  CK(dx.alloc(static_cast<size_t>(n) * dims));
  CK(o.alloc(n));
  CK(cudaMemcpy(dx.p, x, 8ull * n * dims, cudaMemcpyHostToDevice));
  cudaError_t e = cudaSuccess;
  dispatch_fit(fid, [&](auto F) {
    constexpr int f = decltype(F)::value;
    k_eval<f><<<(n + 255) / 256, 256>>>(P, dx.p, o.p);
    e = cudaGetLastError();
  });
  CK(e);
  CK(cudaMemcpy(out, o.p, 8ull * n, cudaMemcpyDeviceToHost));
  return CUPSO_OK;
}

cupso_status cupso_eval_kinematics(int device, const cupso_params* p, const double* v, const double* x,
                                   const double* pbest_x, const double* gbest_x, const double* r1,
                                   const double* r2, double* v_out, double* x_out, size_t n) {
  if (!p) return fail(CUPSO_EINVAL, "pso_params: null");
  if (!n) return CUPSO_OK;
  CK(cudaSetDevice(device));
  KParams P{};
  P.w = p->inertia;
  P.c1 = p->cognitive;
  P.c2 = p->social;
  P.min_pos = p->min_pos;
  P.max_pos = p->max_pos;
  P.min_v = p->min_v;
  P.max_v = p->max_v;
  DevBuf<double> b;
  CK(b.alloc(8 * n));
  const double* srcs[6] = {v, x, pbest_x, gbest_x, r1, r2};
  for (int i = 0; i < 6; ++i) CK(cudaMemcpy(b.p + i * n, srcs[i], 8 * n, cudaMemcpyHostToDevice));
  k_kin_batch<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256>>>(
      P, b.p, b.p + n, b.p + 2 * n, b.p + 3 * n, b.p + 4 * n, b.p + 5 * n, b.p + 6 * n, b.p + 7 * n, n);
  CK(cudaGetLastError());
  CK(cudaMemcpy(v_out, b.p + 6 * n, 8 * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(x_out, b.p + 7 * n, 8 * n, cudaMemcpyDeviceToHost));
  return CUPSO_OK;
}

}  // extern "C"
