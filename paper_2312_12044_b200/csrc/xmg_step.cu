// xmg_step.cu — B200 (sm_100a) batched XLand-MiniGrid environment step.
//
// Implements the C ABI declared in include/xmg.h; the reference is the NumPy
// VecEnv.step of /root/reference/pkg/src/rulegrid/vecenv.py:295-364 (cited as
// ref:<file>:<line>):
//   action (:306-342) -> rules (:368-433) -> goal (:435-477) -> reward /
//   discount / step type (:351-357) -> auto-reset of finished trials
//   (:359-361 -> :224-291) -> egocentric observation (:481-500).
//
// Kernels:
//  * step_main — one thread per env, 64 envs per CTA: one 16-byte state word
//    per env, the grid bytes of the view window staged global->shared with
//    16-byte cp.async, the action, MOVE / PICK_UP rules and goals per lane
//    (select-based), counters and reward, the observation assembled in shared
//    memory and stored with one TMA bulk copy per warp; PUT_DOWN events and
//    finished trials are appended to work queues;
//  * step_rare — one warp per queued env: PUT_DOWN rule passes (speculative
//    per-slot evaluation) and trial rebuilds (Philox draws spread over lanes,
//    the reference's stable argsort replaced by a warp radix-select), launched
//    so that the next step's step_main overlaps it (programmatic dependent
//    launch, per-chunk release);
//  * rollout_kernel (xmg_rollout.cuh) — T steps fused, state on chip;
//  * sprite_kernel / image_kernel* (xmg_render.cuh) — 224x224 observation images.
// Files: xmg_common.cuh (Philox, codes, views, rules / goals, observation),
// xmg_build.cuh (trial builds), xmg_main.cuh (step_main, queue layout),
// xmg_rare.cuh (step_rare), xmg_rollout.cuh, xmg_render.cuh; this file holds
// the small helper kernels, the launchers and the C ABI.
// Nothing here is a dense contraction, so no tensor cores are used; the step
// is bounded by HBM bytes per env-step (roofline).

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <array>
#include <vector>

#include "../../include/xmg.h"

namespace {

#include "xmg_common.cuh"
#include "xmg_build.cuh"
#include "xmg_main.cuh"
#include "xmg_rare.cuh"

// ------------------------------------------------------- helper kernels
__global__ void philox_kernel(const uint64_t* ctr, const uint64_t* key, uint64_t* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Words4 w = philox(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], key[2 * i], key[2 * i + 1]);
  out[4 * i] = w.w0; out[4 * i + 1] = w.w1; out[4 * i + 2] = w.w2; out[4 * i + 3] = w.w3;
}

// keys[i] = fold_in(root, offset+i, SPLIT)  (ref:rng.py:142-145)
__global__ void split_batch_kernel(uint64_t hi, uint64_t lo, int64_t offset, int64_t n, uint64_t* keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Words4 w = philox((uint64_t)(offset + i), 0, kDomSplit, 0, hi, lo);
  keys[2 * i] = w.w0;
  keys[2 * i + 1] = w.w1;
}

// one thread per (env, 4-word block): actions[t][i] = word(t0+t) % 6
__global__ void random_actions_kernel(const uint64_t* keys, int64_t n, int64_t t0, int64_t steps, int64_t b0,
                                      int64_t nblocks, uint8_t* actions) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * nblocks) return;
  const int64_t i = idx % n, b = b0 + idx / n;
  const Words4 w = philox((uint64_t)b, 0, kDomDraw, 0, keys[2 * i], keys[2 * i + 1]);
  const uint64_t wv[4] = {w.w0, w.w1, w.w2, w.w3};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t t = 4 * b + k - t0;
    if (t >= 0 && t < steps) actions[t * n + i] = (uint8_t)(wv[k] % 6);
  }
}

// One small grid (it runs beside the previous step's step_rare): 16-byte
// loads, every byte / word checked against [0, 6).
__device__ __forceinline__ bool bad_action(const uint8_t* a, int dtype, int64_t i) {
  int64_t v;
  switch (dtype) {
    case XMG_ACT_U8: v = a[i]; break;
    case XMG_ACT_I32: v = reinterpret_cast<const int32_t*>(a)[i]; break;
    default: v = reinterpret_cast<const int64_t*>(a)[i];
  }
  return v < 0 || v >= 6;
}

__global__ void validate_kernel(const void* a, int dtype, int64_t n, uint32_t epoch, uint32_t* flag) {
  griddep_launch();  // the step's step_main may launch; it waits for this grid to finish
  const uint8_t* p = reinterpret_cast<const uint8_t*>(a);
  const int es = dtype == XMG_ACT_U8 ? 1 : dtype == XMG_ACT_I32 ? 4 : 8;
  const int64_t bytes = n * es;
  // elements before the first 16-byte boundary, and the 16-byte body
  const int64_t head = (int64_t)((16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15) / es;
  const int64_t nvec = head * es < bytes ? (bytes - head * es) / 16 : 0;
  const uint4* body = reinterpret_cast<const uint4*>(p + head * es);
  const int64_t tail0 = head + nvec * 16 / es;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t i = tid; i < nvec; i += nt) {
    const uint4 v = body[i];
    if (dtype == XMG_ACT_U8) {  // bytes >= 6 (unsigned: negative int8 can't occur in uint8)
      const uint32_t six = 0x06060606u;
      bad |= (__vcmpgeu4(v.x, six) | __vcmpgeu4(v.y, six) | __vcmpgeu4(v.z, six) | __vcmpgeu4(v.w, six)) != 0;
    } else if (dtype == XMG_ACT_I32) {
      bad |= v.x >= 6u || v.y >= 6u || v.z >= 6u || v.w >= 6u;  // unsigned compare catches negatives
    } else {
      bad |= (v.y != 0u || v.x >= 6u) || (v.w != 0u || v.z >= 6u);
    }
  }
  for (int64_t i = tid; i < head && i < n; i += nt) bad |= bad_action(p, dtype, i);
  for (int64_t i = tail0 + tid; i < n; i += nt) bad |= bad_action(p, dtype, i);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMax(flag, epoch);
  // the last CTA to finish publishes flag[1] = epoch (and re-arms the counter)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(flag + 2, 1u) == gridDim.x - 1) {
      flag[2] = 0;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag + 1), "r"(epoch) : "memory");
    }
  }
}

#include "xmg_rollout.cuh"
#include "xmg_render.cuh"

// ------------------------------------------------------- host side
thread_local std::string g_err;

int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

int check_launch(const char* what) {
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(std::string(what) + ": " + cudaGetErrorString(err));
  return 0;
}

// Profiling hook (xmg_profile): CUDA events around each step's two kernels.
// Recording them serialises the kernels (no overlap), so the durations are
// per-kernel standalone times, for rooflines; never used in timed runs.
struct Prof {
  std::mutex mu;
  bool on = false;
  std::vector<std::array<cudaEvent_t, 3>> events;
};
Prof g_prof;

bool prof_events(cudaEvent_t* ev) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  std::array<cudaEvent_t, 3> e;
  for (int k = 0; k < 3; ++k)
    if (cudaEventCreate(&e[k]) != cudaSuccess) return false;
  g_prof.events.push_back(e);
  for (int k = 0; k < 3; ++k) ev[k] = e[k];
  return true;
}

int pick_maxch(const xmg_env_desc* d) {
  const int need = needed_chunks(d->width, d->view_size);
  if (need <= 6) return 6;
  if (need <= 8) return 8;
  if (need <= 12) return 12;
  if (need <= 16) return 16;
  if (need <= 32) return 32;
  return 0;
}

template <typename K>
cudaError_t allow_smem(K kernel, int64_t dyn) {
  cudaFuncAttributes fa;
  cudaError_t err = cudaFuncGetAttributes(&fa, kernel);
  if (err != cudaSuccess) return err;
  (void)dyn;  // the opt-in covers any size up to the per-block limit left beside the static shared memory
  if ((int64_t)fa.sharedSizeBytes >= kMaxDynSmem) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem - (int)fa.sharedSizeBytes);
}

// Per-device facts and kernel attributes (SM count, the >48 KB dynamic
// shared-memory opt-in of the step / rare / pre-build / rollout kernels):
// attributes belong to the device context, so they are set once per device,
// not once per process (a process may drive several GPUs).
struct DevInfo {
  bool done = false;
  int sms = 0;
  cudaError_t err = cudaSuccess;
  const char* what = "";
  int64_t rare_smem = -1;  // occupancy cache of step_rare for this scratch size
  int rare_per_sm = 0;
  uint64_t pol[2] = {0, 0};  // L2 policies (evict_last, evict_first), policy_kernel
};
constexpr int kMaxDevices = 64;
DevInfo g_dev[kMaxDevices];
std::mutex g_dev_mu;

template <typename K>
bool set_attr(DevInfo& di, K kernel, const char* what) {
  if (di.err != cudaSuccess) return false;
  di.err = allow_smem(kernel, kMaxDynSmem - 1024);
  di.what = what;
  return di.err == cudaSuccess;
}

int device_attrs(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return fail("device index out of range");
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DevInfo& di = g_dev[dev];
  if (!di.done) {
    cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev);
    set_attr(di, step_main<6>, "step_main") && set_attr(di, step_main<8>, "step_main") &&
        set_attr(di, step_main<12>, "step_main") && set_attr(di, step_main<16>, "step_main") &&
        set_attr(di, step_main<32>, "step_main") &&
        set_attr(di, step_rare, "step_rare") && set_attr(di, prebuild_kernel, "prebuild_kernel") &&
        set_attr(di, rollout_kernel, "rollout_kernel");
    if (di.err == cudaSuccess) {
      uint64_t* dp = nullptr;
      di.what = "policy_kernel";
      di.err = cudaMalloc(&dp, 2 * sizeof(uint64_t));
      if (di.err == cudaSuccess) {
        policy_kernel<<<1, 1>>>(dp);
        di.err = cudaMemcpy(di.pol, dp, sizeof(di.pol), cudaMemcpyDeviceToHost);
        cudaFree(dp);
      }
    }
    di.done = true;
  }
  if (di.err != cudaSuccess) return fail(std::string(di.what) + " attributes: " + cudaGetErrorString(di.err));
  if (di.sms < 1) return fail("no SM count for this device");
  return 0;
}

// The current device's entry (after device_attrs); nullptr on failure.
DevInfo* cur_dev() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    fail("cudaGetDevice failed");
    return nullptr;
  }
  if (device_attrs(dev)) return nullptr;
  return &g_dev[dev];
}

// XMG_RARE_PDL=0: step_rare as a plain launch after step_main
bool rare_pdl();

// XMG_PDL=0 turns the programmatic (overlapped) launches off
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("XMG_PDL");
    on = (v && !strcmp(v, "0")) ? 0 : 1;
  }
  return on == 1;
}

// words per compact agent-rule row step_main fetches (0: whole task rows)
inline int agent_words(const xmg_env_desc* d) { return d->agent_rows != nullptr ? d->agent_row_words : 0; }

bool rare_pdl() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("XMG_RARE_PDL");
    on = (v && !strcmp(v, "0")) ? 0 : 1;
  }
  return on == 1 && pdl_enabled();
}

template <int MAXCH>
int launch_main(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const void* actions, int dtype,
                const uint32_t* flag, uint32_t epoch, int64_t n, cudaStream_t st, bool pdl) {
  const MainGeo geo = make_main_geo(d->view_size, MAXCH, d->rule_width, agent_words(d));
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const int64_t blocks = (n + kThreads - 1) / kThreads;
  // programmatic dependent of the previous kernel on the stream (the previous
  // step's step_rare, or this step's validation)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)geo.total;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err =
      cudaLaunchKernelEx(&cfg, step_main<MAXCH>, *d, *s, *o, actions, dtype, flag, epoch, n, di->pol[0], di->pol[1],
                         geo);
  if (err != cudaSuccess) return fail(std::string("step_main: ") + cudaGetErrorString(err));
  return check_launch("step_main");
}

// grids up to 1024 cells: the PUT_DOWN candidate lists and the radix select
// of the trial builds assume it
bool grid_fits(const xmg_env_desc* d) { return d->height * d->width <= 1024; }

int launch_rare(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const uint64_t* keys,
                const uint32_t* flag, uint32_t epoch, int64_t n, int track, cudaStream_t st) {
  const RareGeo geo = make_rare_geo(d->height, d->width, d->rule_width);
  DevInfo* di = cur_dev();
  if (!di) return -1;
  const int sms = di->sms;
  // resident CTAs per SM for this scratch size (cached per device: the query
  // costs microseconds of host time per launch, which small batches feel)
  if (di->rare_smem != geo.total) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&di->rare_per_sm, step_rare, kRareWarps * 32,
                                                      (size_t)geo.total) != cudaSuccess)
      di->rare_per_sm = 0;
    di->rare_smem = geo.total;
  }
  int per_sm = di->rare_per_sm;
  if (per_sm < 1) return fail("step_rare does not fit on an SM");
  // At most ~20 resident step_rare warps per SM: the kernel overlaps the next
  // step's step_main, and beyond that it crowds step_main's CTAs out
  // (measured at C3 / DoorKey: 20 warps 80 us/step, 21-24 warps 89-96 us).
  // XMG_RARE_CTAS overrides the CTA count per SM (tuning).
  static int cap = -1;
  if (cap < 0) {
    const char* v = getenv("XMG_RARE_CTAS");
    cap = v ? atoi(v) : kRareWarpsPerSM / kRareWarps;
  }
  if (cap > 0 && per_sm > cap) per_sm = cap;
  // a multiple of kQueues warps, so every sub-queue gets the same number of warps
  constexpr int64_t unit = kQueues / kRareWarps;
  int64_t blocks = (int64_t)per_sm * sms / unit * unit;
  const int64_t need = ((n + kRareWarps * 64 - 1) / (kRareWarps * 64) + unit - 1) / unit * unit;  // <= a warp / 64 envs
  if (blocks > need) blocks = need;
  if (blocks < unit) blocks = unit;
  // the step's drain: a programmatic dependent of its step_main (which
  // triggers as its CTAs finish; step_rare waits for that grid before reading
  // the queues), so its launch overlaps step_main's last CTAs
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = keys == nullptr && rare_pdl() ? 1 : 0;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kRareWarps * 32);
  cfg.dynamicSmemBytes = (size_t)geo.total;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, step_rare, *d, *s, *o, keys, flag, epoch, n, track);
  if (err != cudaSuccess) return fail(std::string("step_rare: ") + cudaGetErrorString(err));
  return check_launch("step_rare");
}


int validate_desc(const xmg_env_desc* d, const xmg_state* s, int64_t n) {
  if (!d) return fail("null env description");
  if (!s || !s->grids || !s->agent || !s->rng || !s->work) return fail("null state buffer");
  if ((s->next_grids == nullptr) != (s->next_state == nullptr) || (s->next_grids == nullptr) != (s->next_obs == nullptr))
    return fail("reset-ahead buffers next_grids / next_state / next_obs: all or none");
  if ((reinterpret_cast<uintptr_t>(s->next_grids) | reinterpret_cast<uintptr_t>(s->next_state) |
       reinterpret_cast<uintptr_t>(s->next_obs)) & 15)
    return fail("reset-ahead buffers must be 16-byte aligned");
  if (n < 1) return fail("n must be >= 1");
  if (n > (int64_t)kQEnv) return fail("n too large for one launch (< 2^30)");
  if (d->height < 1 || d->height > 255 || d->width < 1 || d->width > 255) return fail("grid size outside [1, 255]");
  if (d->view_size < 3 || !(d->view_size & 1)) return fail("view_size must be odd and >= 3");
  if (d->scenario < 0 || d->scenario > 6) return fail("unknown scenario");
  if (d->num_segments > 12) return fail("too many door segments");
  if (d->rule_width < 0 || d->rule_width > 255 || d->obj_width < 0 || d->obj_width > 255) return fail("bad widths");
  if (d->row_words < 4 || (d->row_words & 3)) return fail("row_words must be a positive multiple of 4");
  if (d->agent_rows != nullptr &&
      (d->agent_row_words < 4 || d->agent_row_words > 16 || (d->agent_row_words & 3)))
    return fail("agent_row_words must be 4, 8, 12 or 16 (<= 12 compact rules)");
  if (d->num_tasks < 1) return fail("empty task table");
  if (!d->base_cells || !d->task_rows) return fail("null base_cells / task_rows");
  if (pick_maxch(d) == 0) return fail("view window too wide for this build (v*W + v > 482)");
  if (!grid_fits(d)) return fail("grid too large for this build (H*W <= 1024)");
  if (make_main_geo(d->view_size, pick_maxch(d), d->rule_width, agent_words(d)).total > kMaxDynSmem - 1024 ||
      make_rare_geo(d->height, d->width, d->rule_width).total > kMaxDynSmem - 1024)
    return fail("grid too large for the shared-memory scratch of this build (H*W <= ~3000)");
  return 0;
}

int dispatch_main(const xmg_env_desc* d, const xmg_state* s, const xmg_out* o, const void* actions, int dtype,
                  const uint32_t* flag, uint32_t epoch, int64_t n, cudaStream_t st, bool pdl = true) {
  switch (pick_maxch(d)) {
    case 6: return launch_main<6>(d, s, o, actions, dtype, flag, epoch, n, st, pdl);
    case 8: return launch_main<8>(d, s, o, actions, dtype, flag, epoch, n, st, pdl);
    case 12: return launch_main<12>(d, s, o, actions, dtype, flag, epoch, n, st, pdl);
    case 16: return launch_main<16>(d, s, o, actions, dtype, flag, epoch, n, st, pdl);
    default: return launch_main<32>(d, s, o, actions, dtype, flag, epoch, n, st, pdl);
  }
}

// Reset-ahead batches (xmg_main.cuh): every `every`-th epoch, the class
// (epoch / every) mod B of envs gets its next trial pre-built, B = the number
// of classes whose cycle fits in budget - 2 steps (so every trial that runs
// to the budget meets its class once).  `every` is the smallest power of two
// >= 16 that gives a batch about four builds per resident warp (a build is
// latency-bound: small batches pay a whole build chain for a few envs; C4's
// 25x25 builds take ~25 us each), capped by budget - 2.  XMG_AHEAD_EVERY
// overrides it.
struct AheadPlan {
  int64_t every, classes;
};
AheadPlan ahead_plan(const xmg_env_desc* d, int64_t n, int sms) {
  static int every_env = -1;
  if (every_env < 0) {
    const char* v = getenv("XMG_AHEAD_EVERY");
    every_env = v ? std::max(1, atoi(v)) : 0;
  }
  const int64_t span = std::max<int64_t>(1, (int64_t)d->budget - 2);
  int64_t every = every_env;
  if (every <= 0) {
    const int64_t target = 4LL * 24 * std::max(sms, 1);  // builds per batch: ~4 per resident warp
    every = 16;
    while (every < span && n * every < target * span) every *= 2;
  }
  every = std::min<int64_t>(every, span);
  return {every, std::max<int64_t>(1, span / every)};
}

int launch_prebuild(const xmg_env_desc* d, const xmg_state* s, int64_t cls, int64_t classes, int64_t n,
                    cudaStream_t st, uint32_t epoch = 0) {
  const int64_t smem = (int64_t)kPreWarps * pre_warp_bytes(d->height, d->width);
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prebuild_kernel, kPreWarps * 32, (size_t)smem) !=
          cudaSuccess ||
      per_sm < 1)
    return fail("prebuild_kernel does not fit on an SM");
  const int64_t count = (n - cls + classes - 1) / classes;
  const int64_t need = (count + (int64_t)kPreWarps * kPreGroup - 1) / ((int64_t)kPreWarps * kPreGroup);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * di->sms, need));
  // a step's batch (epoch != 0) may overlap the previous step's step_rare
  // (programmatic dependent; prebuild_kernel waits per chunk)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = epoch != 0 && pdl_enabled() ? 1 : 0;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kPreWarps * 32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, prebuild_kernel, *d, *s, cls, classes, n,
                                             s->work + prebuild_ctr_base(n), epoch);
  if (err != cudaSuccess) return fail(std::string("prebuild_kernel: ") + cudaGetErrorString(err));
  return check_launch("prebuild_kernel");
}

// The reset-ahead batch of this epoch, if any; returns 1 when one was
// launched (the step's first kernel then waits for it: no programmatic
// overlap with it), 0 when not, <0 on error.
int maybe_prebuild(const xmg_env_desc* d, const xmg_state* s, uint32_t epoch, int64_t n, cudaStream_t st) {
  if (s->next_grids == nullptr) return 0;
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const AheadPlan p = ahead_plan(d, n, di->sms);
  if (epoch % (uint64_t)p.every != 0) return 0;
  const int64_t cls = (int64_t)((epoch / (uint64_t)p.every) % (uint64_t)p.classes);
  if (cls >= n) return 0;
  return launch_prebuild(d, s, cls, p.classes, n, st, epoch == 0 ? 0u : epoch) ? -1 : 1;
}

// envs per warp of the one-kernel step (xmg_step_fused): 32; XMG_FUSED_EPW
// (1..32, a power of two) for experiments — fewer envs per warp measured
// slower at C2 (17.4 -> 22.8 / 36.5 / 61 us per step at 16 / 8 / 4) and flat
// at C1: the step is throughput-, not chain-bound
int fused_epw(int64_t) {
  static int e = -1;
  if (e < 0) {
    const char* v = getenv("XMG_FUSED_EPW");
    e = v ? atoi(v) : 32;
    if (e != 1 && e != 2 && e != 4 && e != 8 && e != 16) e = 32;
  }
  return e;
}

int launch_rollout(const xmg_env_desc* d, const xmg_state* s, const uint64_t* pkeys, const uint8_t* actions,
                   int64_t t0, int64_t steps, int64_t n, const xmg_out* o, cudaStream_t st, uint32_t* gflag = nullptr,
                   int epw = 32) {
  const RollGeo geo = make_roll_geo(d->height, d->width, d->view_size, d->rule_width);
  if (!cur_dev()) return -1;
  if (geo.total > kMaxDynSmem - 1024) return fail("grid too large for the rollout kernel's shared-memory state");
  const int64_t chunks = (n + epw - 1) / epw;
  const int64_t blocks = (chunks + kRollWarps - 1) / kRollWarps;
  rollout_kernel<<<(unsigned)blocks, kRollWarps * 32, (size_t)geo.total, st>>>(*d, *s, pkeys, actions, t0, steps, n,
                                                                             *o, gflag, epw);
  return check_launch("rollout_kernel");
}

}  // namespace

// ================================================================ C ABI
extern "C" {

int32_t xmg_abi_version(void) { return XMG_ABI_VERSION; }

const char* xmg_last_error(void) { return g_err.c_str(); }

void xmg_philox_host(const uint64_t ctr[4], uint64_t k0, uint64_t k1, uint64_t out[4]) {
  philox_host(ctr, k0, k1, out);
}

void xmg_key_from_seed(uint64_t seed_lo, uint64_t seed_hi, uint64_t* out2) {
  const uint64_t ctr[4] = {seed_lo, seed_hi, kDomSeed, 0};
  uint64_t w[4];
  philox_host(ctr, 0, 0, w);
  out2[0] = w[0];
  out2[1] = w[1];
}

void xmg_fold_in(uint64_t hi, uint64_t lo, uint64_t data_lo, uint64_t data_hi, int32_t domain, uint64_t* out2) {
  const uint64_t ctr[4] = {data_lo, data_hi, (uint64_t)domain, 0};
  uint64_t w[4];
  philox_host(ctr, hi, lo, w);
  out2[0] = w[0];
  out2[1] = w[1];
}

int32_t xmg_philox(const uint64_t* ctr, const uint64_t* key, uint64_t* out, int64_t n, void* stream) {
  if (n <= 0) return 0;
  philox_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(ctr, key, out, n);
  return check_launch("philox_kernel");
}

int32_t xmg_split_batch(uint64_t root_hi, uint64_t root_lo, int64_t offset, int64_t n, uint64_t* keys,
                        void* stream) {
  if (n <= 0) return 0;
  split_batch_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(root_hi, root_lo, offset, n,
                                                                                     keys);
  return check_launch("split_batch_kernel");
}

int32_t xmg_random_actions(const uint64_t* keys, int64_t n, int64_t t0, int64_t steps, uint8_t* actions,
                           void* stream) {
  if (n <= 0 || steps <= 0) return 0;
  if (t0 < 0) return fail("t0 must be >= 0");
  const int64_t b0 = t0 / 4, b1 = (t0 + steps - 1) / 4;
  const int64_t nb = b1 - b0 + 1, total = n * nb;
  random_actions_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(keys, n, t0, steps, b0,
                                                                                          nb, actions);
  return check_launch("random_actions_kernel");
}

int32_t xmg_validate_actions(const void* actions, int32_t dtype, int64_t n, uint32_t epoch, uint32_t* flag,
                             void* stream) {
  if (n <= 0) return 0;
  if (dtype < 0 || dtype > 2) return fail("unknown action dtype");
  if (!flag) return fail("null flag");
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const int sms = di->sms;
#ifndef XMG_VAL_SMS
#define XMG_VAL_SMS 1  // validation CTAs per SM (at most)
#endif
#ifndef XMG_VAL_ELEMS
#define XMG_VAL_ELEMS 4096  // elements per validation CTA (at least)
#endif
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((n + XMG_VAL_ELEMS - 1) / XMG_VAL_ELEMS, (int64_t)sms * XMG_VAL_SMS));
  // may overlap the previous step's step_rare (it only reads the actions)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, validate_kernel, actions, (int)dtype, n, epoch, flag);
  if (err != cudaSuccess) return fail(std::string("validate_kernel: ") + cudaGetErrorString(err));
  return check_launch("validate_kernel");
}

int32_t xmg_reset(const xmg_env_desc* desc, const xmg_state* state, const uint64_t* keys, int64_t n,
                  const xmg_out* out, void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!out || !keys) return fail("null out/keys");
  return launch_rare(desc, state, out, keys, nullptr, 0, n, 0, (cudaStream_t)stream);
}

int32_t xmg_step(const xmg_env_desc* desc, const xmg_state* state, const void* actions, int32_t action_dtype,
                 int64_t n, const xmg_out* out, const uint32_t* abort_flag, uint32_t epoch, void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!out || !actions) return fail("null out/actions");
  if (action_dtype < 0 || action_dtype > 2) return fail("unknown action dtype");
  if ((reinterpret_cast<uintptr_t>(state->grids) & 15) ||
      (reinterpret_cast<uintptr_t>(state->agent) & 15) || (out->obs && (reinterpret_cast<uintptr_t>(out->obs) & 15)))
    return fail("actions / grids / agent / obs buffers must be 16-byte aligned");
  cudaEvent_t ev[3];
  const bool prof = g_prof.on && prof_events(ev);
  const int pre = maybe_prebuild(desc, state, epoch, n, (cudaStream_t)stream);
  if (pre < 0) return -1;
  if (prof) cudaEventRecord(ev[0], (cudaStream_t)stream);
  if (dispatch_main(desc, state, out, actions, action_dtype, abort_flag, epoch, n, (cudaStream_t)stream, pre == 0))
    return -1;
  if (prof) cudaEventRecord(ev[1], (cudaStream_t)stream);
  // step_main (window mode) records the tiles step_rare must release
  const int track = 1;
  const int rc = launch_rare(desc, state, out, nullptr, abort_flag, epoch, n, track, (cudaStream_t)stream);
  if (prof) cudaEventRecord(ev[2], (cudaStream_t)stream);
  return rc;
}

int32_t xmg_step_validated(const xmg_env_desc* desc, const xmg_state* state, const void* actions,
                           int32_t action_dtype, int64_t n, const xmg_out* out, uint32_t* flag, uint32_t epoch,
                           void* stream) {
  if (!flag) return fail("null flag");
  if (xmg_validate_actions(actions, action_dtype, n, epoch, flag, stream)) return -1;
  return xmg_step(desc, state, actions, action_dtype, n, out, flag, epoch, stream);
}

int32_t xmg_steps(const xmg_env_desc* desc, const xmg_state* state, const void* actions, int32_t action_dtype,
                  int64_t steps, int64_t n, const xmg_out* traj, uint32_t epoch0, void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!traj || !actions) return fail("null traj/actions");
  if (!traj->reward || !traj->discount || !traj->step_type) return fail("reward / discount / step_type are required");
  if (action_dtype < 0 || action_dtype > 2) return fail("unknown action dtype");
  if (steps < 0) return fail("steps must be >= 0");
  const int64_t ob = 2LL * desc->view_size * desc->view_size;
  if ((reinterpret_cast<uintptr_t>(state->grids) & 15) || (reinterpret_cast<uintptr_t>(state->agent) & 15) ||
      (traj->obs && (((reinterpret_cast<uintptr_t>(traj->obs)) & 15) || ((n * ob) & 15))))
    return fail("grids / agent / obs buffers must be 16-byte aligned (and n*2*v*v a multiple of 16 with obs)");
  const int asz = action_dtype == XMG_ACT_U8 ? 1 : action_dtype == XMG_ACT_I32 ? 4 : 8;
  const int track = 1;
  for (int64_t k = 0; k < steps; ++k) {
    xmg_out o = *traj;
    if (o.obs) o.obs += k * n * ob;
    if (o.reward) o.reward += k * n;
    if (o.discount) o.discount += k * n;
    if (o.step_type) o.step_type += k * n;
    const uint32_t ep = epoch0 + (uint32_t)k + 1u;
    const void* a = reinterpret_cast<const uint8_t*>(actions) + k * n * asz;
    const int pre = maybe_prebuild(desc, state, ep, n, (cudaStream_t)stream);
    if (pre < 0) return -1;
    if (dispatch_main(desc, state, &o, a, action_dtype, nullptr, ep, n, (cudaStream_t)stream, pre == 0)) return -1;
    if (launch_rare(desc, state, &o, nullptr, nullptr, ep, n, track, (cudaStream_t)stream)) return -1;
  }
  return 0;
}

int32_t xmg_profile(int32_t enable) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = enable != 0;
  return 0;
}

int32_t xmg_profile_read(double* main_ms, double* rare_ms, int64_t* steps) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  double a = 0, b = 0;
  for (auto& e : g_prof.events) {
    if (cudaEventSynchronize(e[2]) != cudaSuccess) return fail("xmg_profile_read: event sync failed");
    float x = 0, y = 0;
    cudaEventElapsedTime(&x, e[0], e[1]);
    cudaEventElapsedTime(&y, e[1], e[2]);
    a += x;
    b += y;
    for (int k = 0; k < 3; ++k) cudaEventDestroy(e[k]);
  }
  if (main_ms) *main_ms = a;
  if (rare_ms) *rare_ms = b;
  if (steps) *steps = (int64_t)g_prof.events.size();
  g_prof.events.clear();
  return 0;
}

int64_t xmg_step_smem_bytes(const xmg_env_desc* desc) {
  if (!desc) return -1;
  const int64_t a = make_main_geo(desc->view_size, pick_maxch(desc), desc->rule_width, agent_words(desc)).total;
  const int64_t b = make_rare_geo(desc->height, desc->width, desc->rule_width).total;
  return a > b ? a : b;
}

int64_t xmg_work_words(int64_t n) { return n < 0 || n > (int64_t)kQEnv ? -1 : work_words(n); }

int32_t xmg_prebuild(const xmg_env_desc* desc, const xmg_state* state, int64_t cls, int64_t classes, int64_t n,
                     void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!state->next_grids) return fail("xmg_prebuild needs the reset-ahead buffers");
  if (classes < 1 || cls < 0 || cls >= classes) return fail("need 0 <= cls < classes");
  if (cls >= n) return 0;
  return launch_prebuild(desc, state, cls, classes, n, (cudaStream_t)stream);
}

int32_t xmg_ahead_plan(const xmg_env_desc* desc, int64_t n, int64_t* every, int64_t* classes) {
  if (!desc) return fail("null env description");
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const AheadPlan p = ahead_plan(desc, n, di->sms);
  if (every) *every = p.every;
  if (classes) *classes = p.classes;
  return 0;
}

int32_t xmg_rollout(const xmg_env_desc* desc, const xmg_state* state, const uint64_t* policy_keys,
                    const uint8_t* actions, int64_t t0, int64_t steps, int64_t n, const xmg_out* traj,
                    void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!traj) return fail("null trajectory record");
  if ((policy_keys == nullptr) == (actions == nullptr)) return fail("exactly one of policy_keys / actions");
  if (t0 < 0 || steps < 0) return fail("t0 and steps must be >= 0");
  if (steps == 0) return 0;
  if ((reinterpret_cast<uintptr_t>(state->agent) & 15) || (reinterpret_cast<uintptr_t>(state->rng) & 15) ||
      (policy_keys && (reinterpret_cast<uintptr_t>(policy_keys) & 15)))
    return fail("agent / rng / policy key buffers must be 16-byte aligned");
  return launch_rollout(desc, state, policy_keys, actions, t0, steps, n, traj, (cudaStream_t)stream);
}

int32_t xmg_step_fused(const xmg_env_desc* desc, const xmg_state* state, const uint8_t* actions, int64_t n,
                       const xmg_out* out, uint32_t* gflag, void* stream) {
  if (validate_desc(desc, state, n)) return -1;
  if (!out || !actions || !gflag) return fail("null out / actions / gflag");
  if (!out->reward || !out->discount || !out->step_type) return fail("reward / discount / step_type are required");
  if ((reinterpret_cast<uintptr_t>(state->agent) & 15) || (reinterpret_cast<uintptr_t>(state->rng) & 15))
    return fail("agent / rng buffers must be 16-byte aligned");
  return launch_rollout(desc, state, nullptr, actions, 0, 1, n, out, (cudaStream_t)stream, gflag, fused_epw(n));
}

// One fused step as a one-node executable CUDA graph (built from explicit
// kernel-node parameters, not a stream capture, so the actions pointer of
// the node can be re-pointed at each launch: no staging copy).
struct GraphStep {
  cudaGraph_t graph = nullptr;  // kept: the node handle belongs to it
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t node = nullptr;
  cudaKernelNodeParams params = {};
  // the kernel's arguments (rollout_kernel), pointed to by params.kernelParams
  xmg_env_desc d;
  xmg_state s;
  const uint64_t* pkeys = nullptr;
  const uint8_t* actions = nullptr;
  int64_t t0 = 0, T = 1, n = 0;
  xmg_out o;
  uint32_t* gflag = nullptr;
  int epw = 32;
  void* args[10];
};

int32_t xmg_graph_create(const xmg_env_desc* desc, const xmg_state* state, const uint8_t* actions, int64_t n,
                         const xmg_out* out, uint32_t* gflag, void** graph_exec) {
  if (!graph_exec) return fail("null graph handle");
  *graph_exec = nullptr;
  if (validate_desc(desc, state, n)) return -1;
  if (!out || !actions || !gflag) return fail("null out / actions / gflag");
  if (!out->reward || !out->discount || !out->step_type) return fail("reward / discount / step_type are required");
  if (!cur_dev()) return -1;  // kernel attributes are set before the node is built
  const RollGeo geo = make_roll_geo(desc->height, desc->width, desc->view_size, desc->rule_width);
  if (geo.total > kMaxDynSmem - 1024) return fail("grid too large for the rollout kernel's shared-memory state");
  GraphStep* g = new GraphStep();
  g->d = *desc;
  g->s = *state;
  g->actions = actions;
  g->n = n;
  g->o = *out;
  g->gflag = gflag;
  g->epw = fused_epw(n);
  void* args[10] = {&g->d, &g->s, &g->pkeys, &g->actions, &g->t0, &g->T, &g->n, &g->o, &g->gflag, &g->epw};
  for (int i = 0; i < 10; ++i) g->args[i] = args[i];
  const int64_t blocks = ((n + g->epw - 1) / g->epw + kRollWarps - 1) / kRollWarps;
  g->params.func = reinterpret_cast<void*>(rollout_kernel);
  g->params.gridDim = dim3((unsigned)blocks);
  g->params.blockDim = dim3(kRollWarps * 32);
  g->params.sharedMemBytes = (unsigned)geo.total;
  g->params.kernelParams = g->args;
  g->params.extra = nullptr;
  int rc = 0;
  if (cudaGraphCreate(&g->graph, 0) != cudaSuccess) rc = fail("cudaGraphCreate failed");
  if (!rc) {
    const cudaError_t e = cudaGraphAddKernelNode(&g->node, g->graph, nullptr, 0, &g->params);
    if (e != cudaSuccess) rc = fail(std::string("cudaGraphAddKernelNode: ") + cudaGetErrorString(e));
  }
  if (!rc) {
    const cudaError_t e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) rc = fail(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  }
  if (rc) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return rc;
  }
  *graph_exec = g;
  return 0;
}

int32_t xmg_graph_launch(void* handle, void* stream) {
  if (!handle) return fail("null graph handle");
  GraphStep* g = static_cast<GraphStep*>(handle);
  const cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
  return e == cudaSuccess ? 0 : fail(std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
}

int32_t xmg_graph_step(void* handle, const uint8_t* src, uint8_t* staging, int64_t n, void* stream) {
  if (!handle) return fail("null graph handle");
  GraphStep* g = static_cast<GraphStep*>(handle);
  const uint8_t* want = src ? src : staging;
  if (n != g->n) return fail("xmg_graph_step: n differs from the graph's");
  if (want != g->actions) {  // re-point the node at this step's actions (host-side update, no copy)
    g->actions = want;
    const cudaError_t e = cudaGraphExecKernelNodeSetParams(g->exec, g->node, &g->params);
    if (e != cudaSuccess) return fail(std::string("cudaGraphExecKernelNodeSetParams: ") + cudaGetErrorString(e));
  }
  return xmg_graph_launch(handle, stream);
}

int32_t xmg_graph_destroy(void* handle) {
  if (handle) {
    GraphStep* g = static_cast<GraphStep*>(handle);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
  }
  return 0;
}

int32_t xmg_sprites(int32_t px, uint8_t* atlas, void* stream) {
  if (px < 4 || px > kImageSide) return fail("tile_px must be in [4, 224]");
  if (!atlas) return fail("null atlas");
  const int64_t total = 210LL * px * px;
  sprite_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(px, atlas);
  return check_launch("sprite_kernel");
}

int32_t xmg_image_obs(const uint8_t* obs, int64_t n, int32_t view, const uint8_t* atlas, uint8_t* out,
                      void* stream) {
  if (view < 1 || kImageSide / view < 4) return fail("view size leaves tiles under 4px");
  if (!obs || !atlas || !out) return fail("null buffer");
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail("image buffer must be 16-byte aligned");
  if (n <= 0) return 0;
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const int sms = di->sms;
  const int64_t blocks = std::min<int64_t>(n, (int64_t)sms * 12);
  image_kernel<<<(unsigned)blocks, kImageWords, 0, (cudaStream_t)stream>>>(obs, n, view, kImageSide / view, atlas,
                                                                          out);
  return check_launch("image_kernel");
}

int64_t xmg_image_atlas_bytes(int32_t view) {
  if (view < 1 || view > 37 || kImageSide / view < 6) return -1;
  return aligned_atlas_bytes(view);
}

int32_t xmg_image_atlas(int32_t view, const uint8_t* atlas, uint8_t* aligned, void* stream) {
  if (xmg_image_atlas_bytes(view) < 0) return fail("aligned image atlas needs view in [1, 37]");
  if (!atlas || !aligned) return fail("null buffer");
  if (reinterpret_cast<uintptr_t>(aligned) & 15) return fail("aligned atlas must be 16-byte aligned");
  const int64_t total = aligned_atlas_bytes(view);
  aligned_atlas_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(view, atlas, aligned);
  return check_launch("aligned_atlas_kernel");
}

int32_t xmg_image_obs_aligned(const uint8_t* obs, int64_t n, int32_t view, const uint8_t* aligned, uint8_t* out,
                              void* stream) {
  if (xmg_image_atlas_bytes(view) < 0) return fail("aligned image path needs view in [1, 37]");
  if (!obs || !aligned || !out) return fail("null buffer");
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail("image buffer must be 16-byte aligned");
  if (n <= 0) return 0;
  const DevInfo* di = cur_dev();
  if (!di) return -1;
  const int sms = di->sms;
  const int64_t blocks = std::min<int64_t>(n, (int64_t)sms * 12);
  image_kernel_aligned<<<(unsigned)blocks, kImgThreads, 0, (cudaStream_t)stream>>>(obs, n, view, aligned, out);
  return check_launch("image_kernel_aligned");
}

int64_t xmg_rollout_smem_bytes(const xmg_env_desc* desc) {
  if (!desc) return -1;
  return make_roll_geo(desc->height, desc->width, desc->view_size, desc->rule_width).total;
}

#ifdef XMG_TRACE
int32_t xmg_debug_trace(unsigned long long* host_out, int64_t rows) {
  return cudaMemcpyFromSymbol(host_out, g_trace, (size_t)rows * 24 * sizeof(unsigned long long)) == cudaSuccess ? 0
                                                                                                              : -1;
}
int32_t xmg_debug_trace_clear(void) {
  void* ptr = nullptr;
  if (cudaGetSymbolAddress(&ptr, g_trace) != cudaSuccess) return -1;
  return cudaMemset(ptr, 0, sizeof(g_trace)) == cudaSuccess ? 0 : -1;
}
#endif

}  // extern "C"
