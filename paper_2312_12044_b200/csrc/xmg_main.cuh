// xmg_main.cuh — the streaming step kernel step_main and the work-queue
// layout it shares with step_rare (included by xmg_step.cu inside its
// anonymous namespace).

// ------------------------------------------------------- the step: two kernels
// step_main (one thread per env, streaming) applies the action, the
// agent-relative rules / goals of MOVE and PICK_UP, the counters, reward and
// observation of every env, and defers the two rare cases into a work queue:
//   * PUT_DOWN events (grid-wide TILE_NEAR rules / goals, ref:rules.py:60-72),
//   * finished trials (auto-reset, ref:vecenv.py:359-361).
// step_rare (one warp per queued env) drains the queue: the PUT_DOWN rule
// pass + goal + reward, the trial rebuild, and the observation of every env
// it touched.  Both run back to back on the caller's stream.
//
// Work queues (state.work, xmg_work_words(n) u32): a PUT_DOWN queue and a
// reset queue, each split in kQueues sub-queues fed by the CTAs with
// blockIdx % kQueues == k (spreads the atomics).  Counts are double-buffered
// by step parity: step t appends to counts[t & 1] while its CTA 0 clears
// counts[(t + 1) & 1] (consumed by the previous step), so no kernel ever
// waits for another.  Layout: counts [2 parities][2 kinds][kQueues], then the
// PUT entries (kQueues x queue_cap) and the reset entries (kQueues x queue_cap).
#ifndef XMG_QUEUES
#define XMG_QUEUES 64  // sub-queues per kind (C3 76.9 vs 77.0 us at 128, C4 66.5 vs 67.4; 32 and 256 slower)
#endif
constexpr int kQueues = XMG_QUEUES;
constexpr int kWorkHeader = 4 * kQueues;
__host__ __device__ inline int count_index(uint32_t parity, int kind, int q) {
  return (int)((parity & 1) * 2 * kQueues + kind * kQueues + q);
}
constexpr uint32_t kQPut = 1u << 31, kQReset = 1u << 30, kQEnv = (1u << 30) - 1;

// ------------------------------------------------------- reset-ahead
// A trial's successor is a function of the env's rng key and task only
// (ref:vecenv.py:224-233 via :359-361), both fixed while the trial runs.  So
// every K-th step (host side, xmg_step) a plain launch of prebuild_kernel
// builds the next trial of one class of envs (e mod B == class, B = the
// classes that fit in budget - 2 steps) into state.next_state / next_obs and
// the env's other grid buffer, and marks them stage 2 (state word 0 bits
// 18-19); the kernels after it see the records.  When a trial ends at stage
// 2, step_main (or step_rare, for a PUT_DOWN) takes the record over (state
// word with the buffer bit flipped, rng, first observation) instead of
// rebuilding; otherwise (a goal reached before the env's class came up) the
// in-place rebuild runs.  Every trial that runs to the budget passes one batch
// of its class, so the synchronized budget resets are all take-overs; the
// build work moves out of the burst and is done at full-GPU efficiency once
// per K steps, without touching the step_rare / step_main overlap.
constexpr uint64_t kStageReady = 2ull << 18, kStageMask = 3ull << 18;
// Double-buffered grids: bit 20 of state word 0 says which of the two grid
// buffers (state.grids = 0, state.next_grids = 1) holds the running trial;
// a pre-build writes the other one, so the auto-reset that consumes it only
// flips the bit (no grid copy).  Queue entries carry the bit in bit 30 (env
// indices are < 2^30), so step_rare addresses the grid without the state word.
constexpr uint64_t kBufBit = 1ull << 20;
constexpr uint32_t kEntBuf = 1u << 30;
__device__ __forceinline__ uint8_t* grid_ptr(const xmg_state& s, int64_t e, int HW, uint32_t buf) {
  return (buf ? s.next_grids : s.grids) + e * (int64_t)HW;
}
__device__ __forceinline__ bool ahead_on(const xmg_state& s) { return s.next_grids != nullptr; }

// capacity of one sub-queue: every env of the step_main CTAs (kThreads envs each)
// feeding it.  Unsigned arithmetic: n < 2^30 (validate_desc), and signed
// 64-bit divisions cost a sign fix-up in every kernel prologue.
__host__ __device__ inline int64_t queue_cap(int64_t n) {
  const uint32_t blocks = ((uint32_t)n + kThreads - 1) / kThreads;
  return (int64_t)((blocks + kQueues - 1) / kQueues * kThreads);
}

// Entry slots of sub-queue (parity, kind, q): double-buffered like the counts,
// so step t + 1's step_main appends while step t's step_rare still drains.
__host__ __device__ inline int64_t queue_base(int64_t n, uint32_t parity, int kind, int q) {
  return (int64_t)kWorkHeader + (int64_t)((parity & 1) * 2 * kQueues + (uint32_t)(kind * kQueues + q)) *
                                    queue_cap(n);
}

// Chunk bookkeeping after the queues (chunk = the 32 envs of one step_main warp):
//   pending[nchunks]  queued envs of the chunk step_rare has not finished yet
//   dirty[nchunks]    epoch of the last step that queued envs of the chunk
// Only the chunk's own warp reads and writes its dirty word, so the tag needs
// no clearing.  (32-bit arithmetic below: n < 2^30, validate_desc.)
__host__ __device__ inline int64_t num_chunks(int64_t n) {
  return (int64_t)(((uint32_t)n + kThreads - 1) / kThreads * kWarps);
}
__host__ __device__ inline int64_t pending_base(int64_t n) { return kWorkHeader + 4 * kQueues * queue_cap(n); }
__host__ __device__ inline int64_t dirty_base(int64_t n) { return pending_base(n) + num_chunks(n); }
// then the two counter words of the reset-ahead batches (prebuild_kernel)
__host__ __device__ inline int64_t prebuild_ctr_base(int64_t n) { return dirty_base(n) + num_chunks(n); }
__host__ __device__ inline int64_t work_words(int64_t n) { return prebuild_ctr_base(n) + 2; }

__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ ulonglong2 ld_cg_u64x2(const ulonglong2* p) {  // fresh from L2, not CSE'd
  ulonglong2 v;
  asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}
// L2 eviction-priority hints (XMG_L2HINT=1): the state words (16 B per env,
// read again next step) are kept with evict_last; the view-window reads and
// the write-once records (observations, reward, discount, step type) go with
// evict_first (C3: step_main 59.8 -> 57.8 us, the step 81.3 -> 78.8 us)
#ifndef XMG_L2HINT
#define XMG_L2HINT 1
#endif
#ifndef XMG_VAL_SLEEP
#define XMG_VAL_SLEEP 64  // ns between polls of the validation verdict
#endif
#ifndef XMG_L2HINT_GRID
#define XMG_L2HINT_GRID XMG_L2HINT
#endif
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ ulonglong2 ld_hint_u64x2(const ulonglong2* p, uint64_t pol) {
  ulonglong2 v;
  asm volatile("ld.global.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(v.x), "=l"(v.y) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint_u64(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint_f32(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint_s8(int8_t* p, int v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b8 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int load_action(const void* a, int dtype, int64_t e) {
  switch (dtype) {
    case XMG_ACT_U8: return reinterpret_cast<const uint8_t*>(a)[e];
    case XMG_ACT_I32: return reinterpret_cast<const int32_t*>(a)[e];
    default: return (int)reinterpret_cast<const int64_t*>(a)[e];
  }
}

__device__ __forceinline__ uint64_t pack_agent(int r, int c, int d, int pocket, uint32_t sc) {
  return (uint64_t)(uint32_t)r | ((uint64_t)(uint32_t)c << 8) | ((uint64_t)(uint32_t)d << 16) |
         ((uint64_t)(uint32_t)pocket << 24) | ((uint64_t)sc << 32);
}

// float32(1.0 - 0.9 * (sc / budget)) in IEEE double without contraction
// (ref:env.py:204, ref:vecenv.py:355)
__device__ __forceinline__ float goal_reward(uint32_t sc, int budget) {
  const double frac = __ddiv_rn((double)sc, (double)budget);
  return __double2float_rn(__dsub_rn(1.0, __dmul_rn(0.9, frac)));
}

// Per-CTA episode statistics slot (ref RolloutStats, harness.py:103-143).
__device__ __forceinline__ void warp_stats(double* stats, int slot, double rs, double trl, double ln) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    rs += __shfl_down_sync(0xffffffffu, rs, off);
    trl += __shfl_down_sync(0xffffffffu, trl, off);
    ln += __shfl_down_sync(0xffffffffu, ln, off);
  }
  if ((threadIdx.x & 31) == 0 && trl + rs > 0.0) {
    atomicAdd(stats + 3 * slot, rs);
    atomicAdd(stats + 3 * slot + 1, trl);
    atomicAdd(stats + 3 * slot + 2, ln);
  }
}

// The same slot update for one step of a warp's 32 envs: a reward is only
// paid on a step that ends the trial, so a warp with no trial ending (the
// common case, ~94% of warps per step at C3) does two votes and nothing
// else; trials and lengths are integer warp reductions (popc / redux.sync).
// Called converged (all 32 lanes).
__device__ __forceinline__ void warp_stats_step(double* stats, int slot, float rew, bool last, uint32_t sc) {
  const uint32_t lm = __ballot_sync(0xffffffffu, last);
  if (!lm) return;
  const uint32_t len = __reduce_add_sync(0xffffffffu, last ? sc : 0u);
  double rs = 0.0;
  if (__any_sync(0xffffffffu, rew != 0.f)) {
    rs = (double)rew;
#pragma unroll
    for (int off = 16; off; off >>= 1) rs += __shfl_down_sync(0xffffffffu, rs, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (rs != 0.0) atomicAdd(stats + 3 * slot, rs);
    atomicAdd(stats + 3 * slot + 1, (double)__popc(lm));
    atomicAdd(stats + 3 * slot + 2, (double)len);
  }
}

// Warp copy of nbytes from src to dst, the body in 16-byte chunks when both
// share their alignment mod 16 (else byte by byte); the source is read through L2 (.cg: records written by an
// earlier kernel, never cached in this SM's L1).
__device__ __forceinline__ void warp_copy_cg(uint8_t* dst, const uint8_t* src, int nbytes, int lane) {
  if ((reinterpret_cast<uintptr_t>(dst) ^ reinterpret_cast<uintptr_t>(src)) & 15) {  // different alignment: bytes
    for (int t = lane; t < nbytes; t += 32) dst[t] = __ldcg(src + t);
    return;
  }
  const int head = min((int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15), nbytes);
  if (lane < head) dst[lane] = __ldcg(src + lane);
  const int body = (nbytes - head) >> 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
  uint4* d4 = reinterpret_cast<uint4*>(dst + head);
  int i = lane;
  for (; i + 96 < body; i += 128) {  // four chunks in flight per lane
    const uint4 a = __ldcg(s4 + i), b = __ldcg(s4 + i + 32), c = __ldcg(s4 + i + 64), d = __ldcg(s4 + i + 96);
    d4[i] = a;
    d4[i + 32] = b;
    d4[i + 64] = c;
    d4[i + 96] = d;
  }
  for (; i < body; i += 32) d4[i] = __ldcg(s4 + i);
  for (int t = head + 16 * body + lane; t < nbytes; t += 32) dst[t] = __ldcg(src + t);
}

#ifndef XMG_CONSUME_INLINE
#define XMG_CONSUME_INLINE __forceinline__  // inlined: fewer spills in step_main than a call
#endif
// The auto-resets of the envs in `cm` (lanes of the warp's 32-env chunk
// starting at w0) from their pre-built records: state word (whose buffer bit
// now names the other grid buffer, where the pre-build put the new grid: no
// grid copy) and rng per lane, then the first observations copied into the
// warp's observation stage by the whole warp, one contiguous run of envs at a
// time (a burst of budget ends is one run of 32).
__device__ XMG_CONSUME_INLINE void consume_next(const xmg_state s, uint32_t cm, int64_t w0, int HW, int ob,
                                          uint8_t* obs_stage, int lane) {
  __syncwarp();  // every lane is done with its rule row (the observation stage aliases it)
  if ((cm >> lane) & 1) {
    const ulonglong2* ns = reinterpret_cast<const ulonglong2*>(s.next_state) + 2 * (w0 + lane);
    const ulonglong2 a = __ldcg(ns), b = __ldcg(ns + 1);
    reinterpret_cast<ulonglong2*>(s.agent)[w0 + lane] = a;
    reinterpret_cast<ulonglong2*>(s.rng)[w0 + lane] = b;
  }
  for (uint32_t m = cm; m;) {
    const int a = __ffs(m) - 1;
    const uint32_t gap = ~m & ~((1u << a) - 1u);
    const int b = gap ? __ffs(gap) - 1 : 32;
    m = b < 32 ? m & (~0u << b) : 0u;
    if (obs_stage != nullptr) warp_copy_cg(obs_stage + a * ob, s.next_obs + (w0 + a) * ob, (b - a) * ob, lane);
  }
  __syncwarp();
}

struct MainGeo {
  int ob, stg, rb;
  int64_t total;
};

// arw: words of the compact agent-rule rows (xmg_env_desc.agent_rows), 0
// when the step fetches whole task rows
__host__ __device__ inline MainGeo make_main_geo(int V, int maxch, int R, int arw) {
  MainGeo g;
  g.ob = 2 * V * V;
  g.stg = 16 * maxch + 16;
  // per-lane rule row; after the rule pass the warp's 32 rule rows hold its
  // 32 observation records (the staging area of the bulk store)
  g.rb = max(arw > 0 ? 4 * arw : 16 * ((kRowHeader + R + 3) / 4), round16(g.ob));
  g.total = (int64_t)kThreads * (g.stg + g.rb);
  return g;
}

// abort iff *flag == epoch: xmg_validate_actions tags a rejected batch with
// the epoch of its step (atomicMax), so the flag never needs clearing.
__device__ __forceinline__ bool batch_rejected(const uint32_t* flag, uint32_t epoch) {
  return flag != nullptr && *reinterpret_cast<volatile const uint32_t*>(flag) == epoch;
}

// The step of one kThreads-env tile after its loads (state word `ag` of this
// thread's env, its action, the chunk wait done): window staging, action,
// rules, goal, counters, queues, reset-ahead take-overs, statistics and the
// observation.
template <int MAXCH>
__device__ __forceinline__ void main_tile_body(const xmg_env_desc& d, const xmg_state& s, const xmg_out& o,
                                               uint32_t epoch, int64_t n, int64_t tile, int tid, int lane, int warp,
                                               const MainGeo& geo, WView& vw, uint32_t* rbuf, uint8_t* obs_stage,
                                               ulonglong2 ag, int act, uint64_t pol_keep, uint64_t pol_stream,
                                               const uint32_t* abort_flag) {
  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, R = d.rule_width;
  const int64_t e0 = tile * kThreads;
  const int64_t chunk = tile * kWarps + warp;
  uint32_t* pending = s.work + pending_base(n) + chunk;
  uint32_t* dirty = s.work + dirty_base(n) + chunk;
  const int64_t e = e0 + tid;
  const bool valid = e < n;
  (void)pol_keep;
  (void)pol_stream;
  int r = (int)(ag.x & 0xff), c = (int)((ag.x >> 8) & 0xff), dir = (int)((ag.x >> 16) & 3);
  int pocket = (int)((ag.x >> 24) & 0xff);
  uint32_t sc = (uint32_t)(ag.x >> 32);
  const uint32_t goal_word = (uint32_t)ag.y;
  const int task = (int)(ag.y >> 32);
  const uint32_t buf = (uint32_t)(ag.x >> 20) & 1u;  // which grid buffer holds the running trial
  vw.g = grid_ptr(s, valid ? e : 0, HW, buf);

  uint32_t qflags = 0;
  float rew = 0.f;
  bool last = false, consume = false;
  const bool ahead = ahead_on(s);  // (the consume path costs ~1 us/step of steady state at C3: measured)
  const int nd = act == 1 ? ((dir + 3) & 3) : (act == 2 ? ((dir + 1) & 3) : dir);
  if (valid) {
    // ---- stage the post-action window (MOVE: both candidate poses) and,
    // for actions that can raise an event, the env's rule row
    {
      int lo, hi;
      window_span(r, c, nd, act == 0 ? 1 : 0, act == 3 ? 1 : 0, H, W, V, lo, hi);
#if XMG_L2HINT_GRID
      stage_issue<MAXCH>(vw, lo, hi, HW, &pol_stream);
#else
      stage_issue<MAXCH>(vw, lo, hi, HW);
#endif
    }
    const bool rules_needed = R > 0 && (act == 0 || act == 3);
    if (rules_needed) {
      // the compact agent-rule row when the table has one (MOVE / PICK_UP
      // fire nothing else), else the whole task row
      const bool compact = d.agent_rows != nullptr;
      const uint32_t* src = compact ? d.agent_rows + (int64_t)task * d.agent_row_words
                                    : d.task_rows + (int64_t)task * d.row_words;
      const int nq = compact ? d.agent_row_words >> 2 : (kRowHeader + R + 3) >> 2;
      const uint32_t rs = smem_u32(rbuf);
      if (nq <= 8) {  // rows of up to 28 rules: straight-line, predicated
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < nq) cp_async16_s(rs + 16 * q, src + 4 * q);
      } else {
        for (int q = 0; q < nq; ++q) cp_async16_s(rs + 16 * q, src + 4 * q);
      }
    }
  }
  // this epoch's validation verdict (published by the last validation CTA),
  // awaited while the window is in flight: nothing is written before it
  if (abort_flag != nullptr) {
    if (lane == 0)
      for (uint32_t spins = 0; ld_acquire(abort_flag + 1) != epoch; ++spins) {
        if (spins > (1u << 25)) __trap();
        __nanosleep(XMG_VAL_SLEEP);
      }
    __syncwarp();
    if (batch_rejected(abort_flag, epoch)) {
      cp_async_wait_all();  // (no copy outlives the CTA)
      return;
    }
  }
  if (valid) {
    cp_async_wait_all();

    // ---- action, ref:vecenv.py:306-342 / ref:env.py:148-191
    const int tr = r + dir_dr(dir), tc = c + dir_dc(dir);
    const bool inside = tr >= 0 && tr < H && tc >= 0 && tc < W;
    const int tflat = tr * W + tc;
    // (turns stage the new facing's window, which need not hold the old target)
    const int tcode = (inside && act != 1 && act != 2) ? vw.rd(tflat) : 0, tt = tcode >> 4;
    // select-based: lanes with different actions stay converged
    const bool mv = act == 0 && inside && ((kWalkable >> tt) & 1);
    const bool pk = act == 3 && inside && pocket == 0 && ((kPickable >> tt) & 1);
    const bool pt = act == 4 && inside && pocket != 0 && tt == kFloor;
    const bool tg = act == 5 && inside && (tt == kClosed || (tt == kLocked && pocket == kKey * 16 + (tcode & 15)));
    const int ev = mv ? 0 : pk ? 1 : pt ? 2 : tg ? 3 : -1;
    const int wval = pk ? kFloorCode : pt ? pocket : kOpen * 16 + (tcode & 15);
    r = mv ? tr : r;
    c = mv ? tc : c;
    dir = nd;  // nd == dir unless turning
    pocket = pk ? tcode : pt ? 0 : pocket;
    if (pk || pt || tg) vw.wr(tflat, (uint8_t)wval);
    // ---- MOVE / PICK_UP: agent-relative rules (only the slots their event
    // gates, in stored order) and goal; TOGGLE gates no rule and no goal.
    bool goal = false;
    if (ev == 0 || ev == 1) {
      Nbrs nb = load_nbrs(vw, H, W, r, c);
      if (d.agent_rows != nullptr) {  // compact row: count | MOVE mask << 8 | PICK_UP mask << 20
        const uint32_t slots = R > 0 ? (rbuf[0] >> (8 + 12 * ev)) & 0xFFFu : 0u;
        if (slots) pocket = agent_rules(vw, nb, rbuf + 1, slots, pocket);
      } else if (const int nr = R > 0 ? (int)(rbuf[1] & 0xff) : 0) {
        if (R <= 32) {
          const uint32_t slots = rbuf[2 + ev];
          if (slots) pocket = agent_rules(vw, nb, rbuf + kRowHeader, slots, pocket);
        } else {  // wide tables: gate every slot here
          for (int s0 = 0; s0 < nr; ++s0) {
            const int kind = rbuf[kRowHeader + s0] & 0xff;
            if (kind >= 1 && kind <= 11 && ((cRuleGate[kind] >> ev) & 1))
              pocket = agent_rules(vw, nb, rbuf + kRowHeader + s0, 1u, pocket);
          }
        }
      }
      goal = agent_goal(nb, vw.rd(r * W + c), goal_word, ev, r, c, pocket);
    }
    // ---- counters and reward, ref:vecenv.py:351-357
    sc += 1;
    const int stage = (int)(ag.x >> 18) & 3;  // reset-ahead: 2 = next trial pre-built
    if (ev == 2) {
      qflags = kQPut;  // rules, goal and reward resolved by step_rare
    } else {
      last = goal || sc >= (uint32_t)d.budget;
      if (goal) rew = goal_reward(sc, d.budget);
#if XMG_L2HINT
      st_hint_f32(o.reward + e, rew, pol_stream);
      st_hint_f32(o.discount + e, last ? 0.f : 1.f, pol_stream);
      st_hint_s8(o.step_type + e, last ? 2 : 1, pol_stream);
#else
      o.reward[e] = rew;
      o.discount[e] = last ? 0.f : 1.f;
      o.step_type[e] = last ? 2 : 1;
#endif
      // auto-reset: the pre-built next trial when it is ready, else a rebuild
      if (last) {
        if (ahead && stage == 2) consume = true;
        else qflags = kQReset;
      }
    }
    if (!consume) {
#if XMG_L2HINT
      st_hint_u64(s.agent + 2 * e, pack_agent(r, c, dir | (stage << 2) | (int)(buf << 4), pocket, sc), pol_keep);
#else
      s.agent[2 * e] = pack_agent(r, c, dir | (stage << 2) | (int)(buf << 4), pocket, sc);
#endif
    }
  }

  // ---- defer the rare work: warp-aggregated append to this CTA's sub-queue
  const uint32_t qm = __ballot_sync(0xffffffffu, qflags != 0);
  if (qm) {
    const int k = (int)(tile % kQueues);
    if (lane == 0) {
      atomicAdd(pending, (uint32_t)__popc(qm));
      *dirty = epoch;
    }
    // PUT_DOWN and reset entries go to their own queues
#pragma unroll
    for (int kind = 0; kind < 2; ++kind) {
      const uint32_t want = kind ? kQReset : kQPut;
      const uint32_t km = __ballot_sync(0xffffffffu, qflags == want);
      if (!km) continue;
      const int leader = __ffs(km) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(s.work + count_index(epoch, kind, k), (uint32_t)__popc(km));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (qflags == want) {
        XMG_ASSERT(base + __popc(km & ((1u << lane) - 1)) < queue_cap(n));
        s.work[queue_base(n, epoch, kind, k) + base + __popc(km & ((1u << lane) - 1))] =
            (uint32_t)e | (buf << 30);
      }
    }
  }

  // ---- auto-resets from the pre-built records (reset-ahead)
  const uint32_t cm = __ballot_sync(0xffffffffu, consume);
  if (cm) consume_next(s, cm, e0 + warp * 32, HW, 2 * V * V, o.obs != nullptr ? obs_stage : nullptr, lane);

  // ---- episode statistics of the trials decided here
  if (o.stats != nullptr) warp_stats_step(o.stats, (int)(e0 / kStatEnvs), rew, last, sc);


  // ---- observation: assembled in smem, one TMA bulk store per warp
  // (envs queued for step_rare get theirs rewritten there)
  if (o.obs != nullptr) {
    __syncwarp();  // every lane is done with its rule row
    if (valid && !consume) {  // (consumed envs: copied from next_obs above)
      uint8_t* dst = obs_stage + lane * geo.ob;
      if (d.see_through_walls) {
        if (V == 5) obs_see<5>(vw.stage, vw.sbase, dst, r, c, dir, H, W, V);
        else obs_see<0>(vw.stage, vw.sbase, dst, r, c, dir, H, W, V);
      } else {
        obs_occluded(vw, dst, r, c, dir, H, W, V);
      }
    }
    const int64_t w0 = e0 + warp * 32;
    const int nvalid = (int)max((int64_t)0, min((int64_t)32, n - w0));
    const uint32_t bytes = (uint32_t)(nvalid * geo.ob);
    const uint32_t bulk = bytes & ~15u;
    uint8_t* gdst = o.obs + w0 * geo.ob;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && bulk) {
      const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(obs_stage);
#if XMG_L2HINT
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                   ::"l"(gdst), "r"(saddr), "r"(bulk), "l"(pol_stream) : "memory");
#else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(gdst), "r"(saddr), "r"(bulk) : "memory");
#endif
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (uint32_t k = bulk + lane; k < bytes; k += 32) gdst[k] = obs_stage[k];
    if (lane == 0 && bulk) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// The two L2 policies as values (createpolicy once per device, policy_kernel):
// kernel parameters live in the constant bank, so the step does not
// rematerialise them (six uniform-datapath instructions per use).
__global__ void policy_kernel(uint64_t* out) {
  out[0] = l2_policy_last();
  out[1] = l2_policy_first();
}

template <int MAXCH>
__global__ void __launch_bounds__(kThreads, XMG_MINB) step_main(const xmg_env_desc d, const xmg_state s,
                                                                const xmg_out o, const void* actions, int act_dtype,
                                                                const uint32_t* abort_flag, uint32_t epoch,
                                                                int64_t n, uint64_t pol_keep_in,
                                                                uint64_t pol_stream_in, const MainGeo geo) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Launched as a programmatic dependent of the previous kernel (the previous
  // step's step_rare, or this step's validation), so it runs concurrently with
  // the previous step_rare: with a validation it waits for the verdict, and
  // per 32-env chunk it waits only where the previous step queued envs (below).
  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, R = d.rule_width;
  // geo: make_main_geo(V, MAXCH, R), computed by the launcher (a kernel parameter)
  const int64_t tile = blockIdx.x;
  const int64_t e0 = tile * kThreads;
  const int64_t chunk = tile * kWarps + warp;
  uint32_t* pending = s.work + pending_base(n) + chunk;
  uint32_t* dirty = s.work + dirty_base(n) + chunk;
  const int64_t e = e0 + tid;
  const bool valid = e < n;

  uint8_t* rb_base = smem + kThreads * geo.stg;
  uint8_t* obs_stage = rb_base + warp * 32 * geo.rb;  // aliases the warp's rule rows
  WView vw;  // (its grid pointer is set from the state word: the env's current buffer)
  vw.stage = smem + tid * geo.stg;
  vw.sbase = vw.slo = vw.shi = 0;
  uint32_t* rbuf = reinterpret_cast<uint32_t*>(rb_base + tid * geo.rb);

  // ---- load: the 16-byte state word and the action
  ulonglong2 ag = make_ulonglong2(0, 0);
  int act = 1;
  const uint32_t was_dirty = e0 + warp * 32 < n ? *dirty : 0u;  // issued together with the state loads
#if XMG_L2HINT
  const uint64_t pol_keep = pol_keep_in, pol_stream = pol_stream_in;
#else
  (void)pol_keep_in;
  (void)pol_stream_in;
#endif
  if (valid) {
#if XMG_L2HINT
    ag = ld_hint_u64x2(reinterpret_cast<const ulonglong2*>(s.agent) + e, pol_keep);
#else
    ag = reinterpret_cast<const ulonglong2*>(s.agent)[e];
#endif
    act = load_action(actions, act_dtype, e);
  }
  // the previous step_rare has read these counts (it reads them before it
  // lets this grid launch); this step appends to the other parity
  if (blockIdx.x == 0)
    for (int i = tid; i < 2 * kQueues; i += blockDim.x) s.work[count_index(epoch + 1, 0, 0) + i] = 0;
  // (a rejected batch returns in main_tile_body, before its first write)
  if (was_dirty == epoch - 1 && e0 + warp * 32 < n) {
    // the previous step queued envs of this chunk: wait until its step_rare has
    // released them all, then reload the state word it may have rewritten
    if (lane == 0) {
      // bounded: a lost release is a bug, trap (launch error) rather than hang
      for (uint32_t spins = 0; ld_acquire(pending) != 0; ++spins) {
        if (spins > (1u << 25)) __trap();
        __nanosleep(128);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncwarp();
    if (valid) ag = ld_cg_u64x2(reinterpret_cast<const ulonglong2*>(s.agent) + e);
  }
  main_tile_body<MAXCH>(d, s, o, epoch, n, tile, tid, lane, warp, geo, vw, rbuf, obs_stage, ag, act,
#if XMG_L2HINT
                              pol_keep, pol_stream,
#else
                              0, 0,
#endif
                              abort_flag);
  // this CTA is done: the step's step_rare (a programmatic dependent that
  // waits for this grid's completion before it reads the queues) may be
  // scheduled as the last CTAs drain, instead of after the grid boundary
  griddep_launch();
}
