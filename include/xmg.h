/*
 * xmg.h — C ABI of libxmg.so, the B200 (sm_100a) batched XLand-MiniGrid step.
 *
 * This is the drop-in boundary for the reference's batched operator API
 * (`rulegrid.VecEnv`, /root/reference/pkg/src/rulegrid/vecenv.py).  The
 * reference is a pure-Python package with no FFI; the entry points below are
 * what its VecEnv would bind if its NumPy body were replaced by native code
 * (see INTEGRATION.md for the ctypes stub).  Each entry point cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - All buffer pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors) unless stated; the library never allocates or frees them.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on that stream.
 *  - Return value: 0 on success, < 0 on error; xmg_last_error() returns a
 *    thread-local message for the last failing call on this thread.
 *  - Scalar key helpers (xmg_key_*) run on the host.
 *
 * Device state layout (structure of arrays, one row per env):
 *   grids  u8  [n][H*W]   row-major entity codes tile*16+color
 *                          (allocation must extend >= 64 bytes past n*H*W:
 *                          the step kernel reads 16-byte aligned chunks)
 *   agent  u64 [n][2]     word 0: r | c<<8 | dir<<16 | pocket<<24 | step_count<<32,
 *                         bits 18-19 = the reset-ahead stage (scheduling metadata,
 *                         not env state: 0 none, 1 next trial queued for pre-build
 *                         this step, 2 pre-built; see next_* below),
 *                         bit 20 = the grid buffer holding the env's grid
 *                         (0: grids, 1: next_grids; always 0 without reset-ahead)
 *                         word 1: goal | task<<32, where goal = encoding bytes
 *                         (kind, a1, a2, a3) little-endian and task = the row
 *                         of the task table this env runs (one 16-byte load)
 *   rng    u64 [n][2]     state key (hi, lo) = ref EnvState.rng
 * Task table (read-only), u32 [num_tasks][row_words]:
 *   word 0 = goal, word 1 = rule_count | obj_count<<8,
 *   word 2 = bitmask of rule slots gated on MOVE, word 3 = on PICK_UP
 *   (AGENT_NEAR family / + AGENT_HOLD, ref rules.py:60-72; all ones if R > 32),
 *   words 4..4+R-1 = active rules (kind, in_a, in_b, out) left-packed
 *   (AGENT_NEAR-family rules, whose in_b is 0, carry instead the neighbour
 *   slots they try: bit k = NEAR_OFFSETS[k], up / left / right / down),
 *   then ceil(O/4) words of active object codes, left-packed; rows are
 *   padded to a multiple of 4 words (16-byte aligned 128-bit loads).
 */
#ifndef XMG_H_
#define XMG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XMG_ABI_VERSION 3

/* scenario ids: ref scenarios.py:177-185 (SCENARIOS) */
enum {
    XMG_SCENARIO_XLAND = 0,
    XMG_SCENARIO_EMPTY = 1,
    XMG_SCENARIO_EMPTY_RANDOM = 2,
    XMG_SCENARIO_DOOR_KEY = 3,
    XMG_SCENARIO_FOUR_ROOMS = 4,
    XMG_SCENARIO_UNLOCK = 5,
    XMG_SCENARIO_UNLOCK_PICKUP = 6
};

/* action dtypes accepted by xmg_step / xmg_validate_actions */
enum { XMG_ACT_U8 = 0, XMG_ACT_I32 = 1, XMG_ACT_I64 = 2 };

/* Static environment description: ref EnvParams (env.py:50-73) plus the
 * layout plan (layouts.py:51-106) and the task table, all pre-resolved on
 * the host.  Pointers are device pointers. */
typedef struct xmg_env_desc {
    int32_t height, width, view_size, budget;
    int32_t scenario;            /* XMG_SCENARIO_* */
    int32_t see_through_walls;   /* 0: exact-integer line of sight, observation.py:46-87 */
    int32_t num_segments;        /* door segments, layouts.py:86-97 */
    int32_t fixed_doors;         /* R6: doors at segment midpoints */
    int32_t rule_width;          /* R (max active rules over the table) */
    int32_t obj_width;           /* O (max active objects over the table) */
    int32_t row_words;           /* u32 words per task row: 4 + R + ceil(O/4), rounded up to 4 */
    int32_t num_tasks;           /* M rows in task_rows */
    int32_t resample_tasks;      /* 0: a trial keeps its env's task (reference semantics,
                                  * vecenv.py:224-233); 1 (extension): every reset draws
                                  * task = rows[word0(split(ek, 2)) % M] (benchio.py:57-58) */
    const uint8_t* base_cells;   /* [H*W] grid before doors/objects for this scenario
                                  * (allocation padded to a multiple of 16 bytes) */
    const int16_t* seg_off;      /* [num_segments+1] offsets into seg_cells */
    const int16_t* seg_cells;    /* flat cell indices of each door segment */
    const uint32_t* task_rows;   /* [num_tasks][row_words] */
    /* ABI 3: optional compact rows of the rules a MOVE / PICK_UP can fire
     * (AGENT_HOLD, the AGENT_NEAR family), [num_tasks][agent_row_words]:
     * word 0 = count | MOVE slot mask << 8 | PICK_UP slot mask << 20 (12-bit
     * masks over these slots), then the rule words in stored order, padded
     * to 16 bytes.  NULL / 0: the step reads the whole task row. */
    int32_t agent_row_words;
    const uint32_t* agent_rows;
} xmg_env_desc;

typedef struct xmg_state {
    uint8_t* grids;
    uint64_t* agent;   /* [n][2] */
    uint64_t* rng;     /* [n][2] */
    uint32_t* work;    /* [xmg_work_words(n)], zero-initialised once: the queues of
                        * rare work (PUT_DOWN events, trial resets) handed from
                        * the streaming kernel to the warp-per-env kernel */
    /* Reset-ahead buffers (all NULL: off).  A trial's successor depends only
     * on the env's rng key and task (ref vecenv.py:224-233, 359-361), both
     * fixed while the trial runs, so xmg_step pre-builds it during the trial
     * (one env in (budget - 2) per step) and the auto-reset that ends the
     * trial takes these records over instead of building.  The grids are
     * double-buffered: a pre-build writes the buffer the env's state word
     * does not name, and the take-over flips bit 20 (no grid copy).  16-byte
     * aligned; next_state / next_obs are scratch owned by the library. */
    uint8_t* next_grids;   /* [n][H*W] (+64 B pad, like grids) the second grid buffer */
    uint64_t* next_state;  /* [n][4]: next state word 0, word 1, next rng (hi, lo) */
    uint8_t* next_obs;     /* [n][v][v][2] the next trial's first observation */
} xmg_state;

/* VecTimeStep (vecenv.py:95-105): observations may be NULL (compute_obs=False) */
typedef struct xmg_out {
    uint8_t* obs;       /* [n][v][v][2] (tile, color) */
    float* reward;      /* [n]  float32(1.0 - 0.9*(sc/budget)) evaluated in fp64 */
    float* discount;    /* [n] */
    int8_t* step_type;  /* [n]  FIRST 0 / MID 1 / LAST 2 */
    /* nullable episode statistics, one slot per 128 envs (little atomics
     * contention): stats[3*(e/128) + 0] += sum of rewards, [+1] += finished
     * trials, [+2] += their lengths (ref RolloutStats, harness.py:103-143) */
    double* stats;
} xmg_out;

int32_t xmg_abi_version(void);
const char* xmg_last_error(void);

/* ---- counter-based RNG (ref rng.py) -------------------------------------- */

/* One Philox4x64-10 block per row: out[i] = philox4(ctr[i], key[i]).
 * Known-answer hook for ref rng.py:42-57 / philox4_array :74-93. */
int32_t xmg_philox(const uint64_t* ctr /*[n][4]*/, const uint64_t* key /*[n][2]*/, uint64_t* out /*[n][4]*/,
                   int64_t n, void* stream);

/* keys[i] = fold_in(root, offset + i, SPLIT): ref split_batch rng.py:142-145
 * (offset lets a GPU shard derive the keys of its global env range). */
int32_t xmg_split_batch(uint64_t root_hi, uint64_t root_lo, int64_t offset, int64_t n, uint64_t* keys /*[n][2]*/,
                        void* stream);

/* Random policy: actions[t][i] = word (t0+t) of keys[i]'s draw stream mod 6,
 * ref harness.py:58-64 (random_policy) with per-env keys. */
int32_t xmg_random_actions(const uint64_t* keys /*[n][2]*/, int64_t n, int64_t t0, int64_t steps,
                           uint8_t* actions /*[steps][n]*/, void* stream);

/* Host-side scalar helpers: ref key_from_seed rng.py:96-99 and
 * fold_in rng.py:107-110 (domain: 1 draw, 2 split, 3 fold, 4 seed); data is
 * the 128-bit counter value (data & 2^64-1, data >> 64 & 2^64-1), so a
 * negative or >= 2^64 Python integer folds in exactly as in the reference. */
void xmg_key_from_seed(uint64_t seed_lo, uint64_t seed_hi, uint64_t* out2);
void xmg_fold_in(uint64_t hi, uint64_t lo, uint64_t data_lo, uint64_t data_hi, int32_t domain, uint64_t* out2);
void xmg_philox_host(const uint64_t ctr[4], uint64_t k0, uint64_t k1, uint64_t out[4]);

/* ---- the batched environment (ref vecenv.py) ----------------------------- */

/* ref VecEnv.reset_with_keys (vecenv.py:205-222): reset env i from keys[i];
 * writes the FIRST VecTimeStep (obs, reward 0, discount 1, step type 0). */
int32_t xmg_reset(const xmg_env_desc* desc, const xmg_state* state, const uint64_t* keys /*[n][2]*/, int64_t n,
                  const xmg_out* out, void* stream);

/* Validation flag block: XMG_FLAG_WORDS device u32, zero-initialised once.
 * [0] epoch of the last rejected batch, [1] epoch of the last finished
 * validation, [2] internal CTA counter. */
#define XMG_FLAG_WORDS 4

/* Raises flag[0] to `epoch` when any action lies outside [0, 6): the device
 * half of ref vecenv.py:297-301 (InvalidAction), then publishes flag[1] =
 * epoch.  The step with the same epoch then touches nothing.  May run
 * concurrently with the previous step's second kernel (it only reads
 * `actions`). */
int32_t xmg_validate_actions(const void* actions, int32_t action_dtype, int64_t n, uint32_t epoch, uint32_t* flag,
                             void* stream);

/* ref VecEnv.step (vecenv.py:295-364): action, rules, goal, reward, auto-reset
 * from each env's own rng, observation of the next playable state.  Two
 * kernels on `stream`: a streaming one-thread-per-env pass and a
 * one-warp-per-env pass over the envs it queued (PUT_DOWN events, resets).
 * `epoch` numbers the caller's steps (consecutive calls on one state must use
 * consecutive epochs: its parity selects the queue buffers).  abort_flag
 * (device flag block, nullable): the step waits for flag[1] == epoch (the
 * validation of this epoch), and when flag[0] == epoch no env is touched
 * (pairs with xmg_validate_actions so an invalid batch mutates nothing).
 * The first kernel of a step may start while the previous step's second
 * kernel still runs: envs that kernel has not released yet are waited for
 * individually (state.work bookkeeping). */
int32_t xmg_step(const xmg_env_desc* desc, const xmg_state* state, const void* actions, int32_t action_dtype,
                 int64_t n, const xmg_out* out, const uint32_t* abort_flag, uint32_t epoch, void* stream);

/* Reset-ahead (state.next_* non-NULL): xmg_step / xmg_steps of every epoch
 * that is a multiple of `every` first launch one batch that pre-builds the
 * next trial of the env class (epoch / every) mod `classes` (envs e with
 * e mod classes == class) whose running trial has none yet; a trial that
 * ends with its successor pre-built is reset by a copy.  xmg_ahead_plan
 * returns (every, classes) for a description and batch size (every *
 * classes <= budget - 2, so a trial that runs to the budget always meets its
 * class; every >= 16, larger for small batches of expensive builds);
 * xmg_prebuild runs one batch explicitly (e.g. right after xmg_reset). */
int32_t xmg_ahead_plan(const xmg_env_desc* desc, int64_t n, int64_t* every, int64_t* classes);
int32_t xmg_prebuild(const xmg_env_desc* desc, const xmg_state* state, int64_t cls, int64_t classes, int64_t n,
                     void* stream);

/* xmg_validate_actions then xmg_step for the same epoch, from one host call
 * (the per-call path of VecEnv.step with device actions). */
int32_t xmg_step_validated(const xmg_env_desc* desc, const xmg_state* state, const void* actions,
                           int32_t action_dtype, int64_t n, const xmg_out* out, uint32_t* flag, uint32_t epoch,
                           void* stream);

/* `steps` consecutive xmg_step calls issued from one host call (no per-step
 * host round trip: the path for batches too small to hide ~20-30 us of
 * Python + launch overhead per step).  actions [steps][n] must already be
 * valid (no device validation: the caller checks the block once); step k
 * uses epoch epoch0 + k + 1 and writes record k of traj: obs (nullable)
 * [steps][n][v][v][2] (n*2*v*v a multiple of 16), reward / discount /
 * step_type [steps][n] (required), stats as in xmg_out. */
int32_t xmg_steps(const xmg_env_desc* desc, const xmg_state* state, const void* actions, int32_t action_dtype,
                  int64_t steps, int64_t n, const xmg_out* traj, uint32_t epoch0, void* stream);

/* Profiling hook: while enabled, every xmg_step records CUDA events around
 * its two kernels (this serialises them: standalone per-kernel times, for
 * rooflines only).  xmg_profile_read synchronises, returns the summed
 * milliseconds of each kernel and the step count, and clears the record. */
int32_t xmg_profile(int32_t enable);
int32_t xmg_profile_read(double* main_ms, double* rare_ms, int64_t* steps);

/* Fused rollout: `steps` consecutive xmg_step calls in
 * one kernel, bit-identical to them, with each env's state on chip for the
 * whole rollout (ref harness.py:103-143 `rollout`, batched: the random-policy
 * loop of ref harness.py:149-158 around VecEnv.step, vecenv.py:295-364).
 * Actions: exactly one of
 *   policy_keys [n][2]   the random policy, action of step t = word (t0 + t)
 *                        of key i's draw stream mod 6 (ref harness.py:58-64,
 *                        == xmg_random_actions), or
 *   actions [steps][n]   u8 in [0, 6) (NOT validated here: the caller checks).
 * traj: every pointer nullable; obs [steps][n][v][v][2], reward / discount /
 * step_type [steps][n] (record t = what xmg_step t would return), stats as
 * in xmg_out, one slot per 128 envs.  state.work is not used: a rollout may sit
 * between xmg_step calls on the same state (same stream) without consuming
 * an epoch. */
int32_t xmg_rollout(const xmg_env_desc* desc, const xmg_state* state, const uint64_t* policy_keys,
                    const uint8_t* actions, int64_t t0, int64_t steps, int64_t n, const xmg_out* traj,
                    void* stream);

/* One xmg_step as ONE kernel (the fused rollout kernel for a single step),
 * for small batches where launches dominate, and capturable in a CUDA graph:
 * every CTA first checks all n u8 actions against [0, 6) (ref
 * vecenv.py:297-301) and an invalid batch changes nothing; the step number is
 * a device counter, so a replayed graph needs no host epoch.
 * gflag: XMG_FLAG_WORDS device u32, zero-initialised once, used only by this
 * entry point: [0] the number of the last rejected step, [2] CTA counter,
 * [3] steps issued (read it after a sync to match [0]).  Same records as
 * xmg_step (obs nullable; reward / discount / step type required); does not
 * consume an epoch of the two-kernel path (state.work unused). */
int32_t xmg_step_fused(const xmg_env_desc* desc, const xmg_state* state, const uint8_t* actions /*[n] u8*/, int64_t n,
                       const xmg_out* out, uint32_t* gflag, void* stream);

/* xmg_step_fused as a one-node executable CUDA graph bound to these buffers
 * (handle = opaque library object); xmg_graph_launch replays one step with
 * the actions buffer it was given (host cost: one graph launch). */
int32_t xmg_graph_create(const xmg_env_desc* desc, const xmg_state* state, const uint8_t* actions, int64_t n,
                         const xmg_out* out, uint32_t* gflag, void** graph_exec);
int32_t xmg_graph_launch(void* graph_exec, void* stream);
/* One step on the actions src [n] u8 (device; NULL = staging): the graph's
 * node is re-pointed at src when it changed (no copy), then one launch. */
int32_t xmg_graph_step(void* graph_exec, const uint8_t* src, uint8_t* staging, int64_t n, void* stream);
int32_t xmg_graph_destroy(void* graph_exec);

/* Dynamic shared memory per CTA (4 warps) of the rollout kernel (<0: unsupported). */
int64_t xmg_rollout_smem_bytes(const xmg_env_desc* desc);

/* ---- observation images (ref render.py) ---------------- */

/* Sprite atlas for one pixel size: atlas[tile][color] = (px, px, 3) u8 RGB,
 * 15 x 14 sprites, each equal to ref render.py:158-169 sprite(tile, color, px)
 * (masks of :107-155 in IEEE double, no contraction).  px in [4, 224]. */
int32_t xmg_sprites(int32_t px, uint8_t* atlas /*[15][14][px][px][3]*/, void* stream);

/* ref render.py:225-243 image_observation for n observations (v, v, 2):
 * out[i] = (224, 224, 3) u8, px = 224 / v (>= 4), the v*px square centred
 * with an UNSEEN-shade margin.  `atlas` from xmg_sprites(224 / v).  Codes
 * outside the enums (tile > 14, color > 13) draw as END_OF_MAP (the host
 * wrapper rejects them first, like the reference).  out 16-byte aligned; the
 * atlas allocation must extend >= 8 bytes before and after its 210*px*px*3
 * bytes (unaligned word reads). */
int32_t xmg_image_obs(const uint8_t* obs /*[n][v][v][2]*/, int64_t n, int32_t view, const uint8_t* atlas,
                      uint8_t* out /*[n][224][224][3]*/, void* stream);

/* Faster image path for views 1..37 (tiles >= 6 px): an "aligned atlas" with
 * every sprite row stored once per 16-byte phase the view's columns start
 * at, so an image is written in aligned 16-byte chunks.
 * xmg_image_atlas_bytes(view): its size (-1 if the view is outside the path);
 * xmg_image_atlas: builds it (16-byte aligned buffer) from xmg_sprites(224 /
 * view); xmg_image_obs_aligned: as xmg_image_obs, byte-identical output. */
int64_t xmg_image_atlas_bytes(int32_t view);
int32_t xmg_image_atlas(int32_t view, const uint8_t* atlas, uint8_t* aligned, void* stream);
int32_t xmg_image_obs_aligned(const uint8_t* obs /*[n][v][v][2]*/, int64_t n, int32_t view, const uint8_t* aligned,
                              uint8_t* out /*[n][224][224][3]*/, void* stream);

/* Size in u32 words of xmg_state.work for n envs (-1 unless 0 <= n < 2^30). */
int64_t xmg_work_words(int64_t n);

/* Bytes of dynamic shared memory per CTA the step/reset kernels use
 * for this description (host query, for capacity checks). <0 if unsupported. */
int64_t xmg_step_smem_bytes(const xmg_env_desc* desc);

#ifdef __cplusplus
}
#endif

#endif /* XMG_H_ */
