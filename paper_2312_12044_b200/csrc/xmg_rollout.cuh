// xmg_rollout.cuh — the fused multi-step rollout (included by xmg_step.cu,
// inside its anonymous namespace).
//
// T consecutive VecEnv.step calls (ref:vecenv.py:295-364) in ONE kernel, each
// env's state resident on chip for the whole rollout: a warp owns 32
// consecutive envs, their grids live in the warp's shared memory and their
// pose / pocket / step count / goal / task / rng key in the lanes' registers.
// Per step a lane applies its env's action, the agent-relative rules and goal
// of MOVE / PICK_UP (the same select-based code as step_main), and the warp
// resolves PUT_DOWN events (warp_put_env, speculative rule slots) and trial
// resets (warp_build, radix-select) in place, so nothing is queued and no
// state word crosses HBM between steps.  What leaves the SM per env-step is
// the trajectory record the caller asked for: the observation (one TMA bulk
// store of the warp's 32 records, double-buffered), reward, discount and step
// type; with all of them NULL only the episode statistics are produced.
//
// Actions: the random policy of ref harness.py:58-64 evaluated in the kernel
// (word t0 + t of the env's policy key mod 6, one Philox block per 4 steps),
// or a caller-supplied [T][n] u8 tensor.  The result is bit-identical to T
// calls of xmg_step with the same actions (tests/test_rollout_gpu.py).

#ifndef XMG_ROLL_WARPS
#define XMG_ROLL_WARPS 4  // warps per CTA (each owns 32 envs and its own scratch)
#endif
#ifndef XMG_ROLL_MINB
#define XMG_ROLL_MINB 4  // resident CTAs per SM the register allocation targets (4 x 4 warps: <= 128 registers)
#endif
constexpr int kRollWarps = XMG_ROLL_WARPS;
constexpr int kRollKeySlots = 16;  // trial keys derived in parallel (resets go in half-warp groups)

struct RollGeo {
  int hw, grids, rbw, rules, ob, obs, hwp, scratch, desc, warp_bytes;
  int64_t total;
};

__host__ __device__ inline RollGeo make_roll_geo(int H, int W, int V, int R) {
  RollGeo g;
  g.hw = H * W;
  g.grids = round16(32 * g.hw);                 // the 32 env grids
  g.rbw = 16 * ((kRowHeader + R + 3) / 4);      // one lane's task row header + rules
  g.rules = R > 0 ? 32 * g.rbw : 0;
  g.ob = 2 * V * V;
  // double-buffered observation records (waiting for the previous step's bulk
  // store to drain costs ~25% with one buffer); between the bulk stores of two
  // steps the same bytes hold the trial keys of the resets
  g.obs = max(2 * round16(32 * g.ob), round16(kRollKeySlots * (int)sizeof(TrialKeys)));
  g.hwp = round16(g.hw + 16);
  // WarpScratch of warp_build: wd u64[hwp] | fc u16[hwp] | slot u16[hwp] | bk | grid u8[hwp] | misc 64 u64;
  // the PUT_DOWN candidate list (u32[hw]) reuses wd (never live at once)
  g.scratch = warp_scratch_bytes(g.hwp);
  g.desc = round16((int)sizeof(xmg_env_desc));  // one copy per CTA
  g.warp_bytes = g.grids + g.rules + g.obs + g.scratch;
  g.total = (int64_t)kRollWarps * g.warp_bytes + g.desc;
  return g;
}

// action of step t: four words of one Philox block, mod 6, packed in a u32
#ifndef XMG_ROLL_POLICY_INLINE
#define XMG_ROLL_POLICY_INLINE __noinline__  // out of line: smaller hot loop, no spills (measured -5%)
#endif
__device__ XMG_ROLL_POLICY_INLINE uint32_t policy_block(uint64_t kh, uint64_t kl, uint64_t blk) {
  const Words4 w = philox<10>(blk, 0, kDomDraw, 0, kh, kl);
  return (uint32_t)(w.w0 % 6) | ((uint32_t)(w.w1 % 6) << 8) | ((uint32_t)(w.w2 % 6) << 16) |
         ((uint32_t)(w.w3 % 6) << 24);
}

// A warp-wide copy with plain loads (either side may be shared memory).
__device__ __forceinline__ void roll_copy(uint8_t* dst, const uint8_t* src, int nbytes, int lane) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    for (int i = lane; i < (nbytes >> 4); i += 32)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (int i = (nbytes & ~15) + lane; i < nbytes; i += 32) dst[i] = src[i];
  } else {
    for (int i = lane; i < nbytes; i += 32) dst[i] = src[i];
  }
}

// The warp's grids between HBM and shared memory.  Each env's grid lives in
// the buffer its state word's bit 20 names (bm: the lanes in buffer 1); runs
// of consecutive lanes in one buffer are contiguous on both sides, so a warp
// whose envs share a buffer moves its grids in one run.
__device__ __forceinline__ void roll_grids_io(const xmg_state& s, int64_t e0, uint32_t vm, uint32_t bm, int HW,
                                              uint8_t* grids, bool to_hbm, int lane) {
  for (uint32_t pass = 0; pass < 2; ++pass) {
    for (uint32_t m = (pass ? bm : ~bm) & vm; m;) {
      const int a = __ffs(m) - 1;
      const uint32_t gap = ~m & ~((1u << a) - 1u);
      const int b = gap ? __ffs(gap) - 1 : 32;
      m = b < 32 ? m & (~0u << b) : 0u;
      uint8_t* g = grid_ptr(s, e0 + a, HW, pass);
      if (to_hbm) roll_copy(g, grids + a * HW, (b - a) * HW, lane);
      else roll_copy(grids + a * HW, g, (b - a) * HW, lane);
    }
  }
}

// The auto-resets of the lanes in cm from their pre-built records: the grid
// bytes (in the other buffer, bm: the lanes whose current grid is in buffer 1)
// into the warp's shared grids, and each lane's next state words returned.
// The lane's buffer bit flips with it (the caller's write-back goes there).
__device__ __noinline__ ulonglong4 roll_consume(const xmg_state s, uint32_t cm, uint32_t bm, int64_t e0, int HW,
                                                uint8_t* grids, int lane) {
  ulonglong4 out = make_ulonglong4(0, 0, 0, 0);
  if ((cm >> lane) & 1) {
    const ulonglong2* ns = reinterpret_cast<const ulonglong2*>(s.next_state) + 2 * (e0 + lane);
    const ulonglong2 w = __ldcg(ns), k = __ldcg(ns + 1);
    out = make_ulonglong4(w.x, w.y, k.x, k.y);
  }
  for (uint32_t pass = 0; pass < 2; ++pass) {  // records of buffer-0 envs are in buffer 1, and back
    for (uint32_t m = cm & (pass ? bm : ~bm); m;) {
      const int a = __ffs(m) - 1;
      const uint32_t gap = ~m & ~((1u << a) - 1u);
      const int b = gap ? __ffs(gap) - 1 : 32;
      m = b < 32 ? m & (~0u << b) : 0u;
      warp_copy_cg(grids + a * HW, grid_ptr(s, e0 + a, HW, pass ^ 1u), (b - a) * HW, lane);
    }
  }
  __syncwarp();
  return out;
}

// gflag (xmg_step_fused, the one-kernel step for small batches and CUDA-graph
// replay): before anything changes, every CTA checks the whole batch of
// actions (u8, [n]) against [0, 6) (ref vecenv.py:297-301); an invalid batch
// is skipped by all CTAs and CTA 0 tags gflag[0] with the step's number.
// gflag[3] counts the steps (advanced by the last CTA to finish, so a
// replayed graph needs no host-side epoch); gflag[2] is the CTA counter.
__device__ __forceinline__ bool fused_batch_rejected(const uint8_t* actions, int64_t n, uint32_t* gflag) {
  const uint32_t clk = *reinterpret_cast<volatile uint32_t*>(gflag + 3);
  bool bad = false;
  const int64_t head = (int64_t)((16 - (reinterpret_cast<uintptr_t>(actions) & 15)) & 15);
  const int64_t h = head < n ? head : n;
  const int64_t nvec = (n - h) >> 4;
  const uint4* body = reinterpret_cast<const uint4*>(actions + h);
  const uint32_t six = 0x06060606u;
  for (int64_t i = threadIdx.x; i < nvec; i += blockDim.x) {
    const uint4 v = body[i];
    bad |= (__vcmpgeu4(v.x, six) | __vcmpgeu4(v.y, six) | __vcmpgeu4(v.z, six) | __vcmpgeu4(v.w, six)) != 0;
  }
  for (int64_t i = threadIdx.x; i < h; i += blockDim.x) bad |= actions[i] >= 6;
  for (int64_t i = h + 16 * nvec + threadIdx.x; i < n; i += blockDim.x) bad |= actions[i] >= 6;
  bad = __syncthreads_or(bad) != 0;
  if (threadIdx.x == 0) {
    if (bad && blockIdx.x == 0) atomicMax(gflag, clk + 1);
    __threadfence();
    if (atomicAdd(gflag + 2, 1u) == gridDim.x - 1) {  // every CTA has read the clock
      gflag[2] = 0;
      __threadfence();
      gflag[3] = clk + 1;
    }
  }
  return bad;
}

__global__ void __launch_bounds__(kRollWarps * 32, XMG_ROLL_MINB) rollout_kernel(const xmg_env_desc d, const xmg_state s,
                                                                 const uint64_t* pkeys, const uint8_t* actions,
                                                                 int64_t t0, int64_t T, int64_t n, const xmg_out o,
                                                                 uint32_t* gflag, int epw) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (gflag != nullptr && fused_batch_rejected(actions, n, gflag)) return;
  const int64_t chunk = (int64_t)blockIdx.x * kRollWarps + warp;
  // epw envs per warp (lanes >= epw idle): 32 for throughput; fewer for the
  // one-kernel step of small batches, where a warp's serial PUT_DOWN / reset
  // work (not occupancy) sets the latency
  const int64_t e0 = (int64_t)epw * chunk;
  if (e0 >= n) return;  // warp-uniform
  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, R = d.rule_width;
  const RollGeo geo = make_roll_geo(H, W, V, R);
  uint8_t* wb = smem + warp * geo.warp_bytes;
  uint8_t* grids = wb;
  uint32_t* rules_s = reinterpret_cast<uint32_t*>(wb + geo.grids);
  uint8_t* obs_s = wb + geo.grids + geo.rules;
  uint8_t* scratch = obs_s + geo.obs;
  uint32_t* cand = reinterpret_cast<uint32_t*>(scratch);      // aliases wd
  TrialKeys* keys = reinterpret_cast<TrialKeys*>(obs_s);      // aliases the observation buffers
  xmg_env_desc* sdesc = reinterpret_cast<xmg_env_desc*>(smem + kRollWarps * geo.warp_bytes);
  ResetOut* rout = reinterpret_cast<ResetOut*>(make_scratch(scratch, geo.hwp).misc + 40);

  const int nvalid = (int)min((int64_t)epw, n - e0);
  const int64_t e = e0 + lane;
  const bool valid = lane < nvalid;
  const bool xland = d.scenario == XMG_SCENARIO_XLAND;
  const bool resample = d.resample_tasks && xland;
  const bool see = d.see_through_walls != 0;
  if (lane == 0) *sdesc = d;

  // ---- state in: state words and rng keys, then the grids (in the buffers the words name)
  ulonglong2 ag = make_ulonglong2(0, 0), rk = make_ulonglong2(0, 0), pk = make_ulonglong2(0, 0);
  if (valid) {
    ag = reinterpret_cast<const ulonglong2*>(s.agent)[e];
    rk = reinterpret_cast<const ulonglong2*>(s.rng)[e];
    if (pkeys) pk = reinterpret_cast<const ulonglong2*>(pkeys)[e];
  }
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  uint32_t buf = (uint32_t)(ag.x >> 20) & 1u;
  roll_grids_io(s, e0, vmask, __ballot_sync(0xffffffffu, buf != 0), HW, grids, false, lane);
  int r = (int)(ag.x & 0xff), c = (int)((ag.x >> 8) & 0xff), dir = (int)((ag.x >> 16) & 3);
  int pocket = (int)((ag.x >> 24) & 0xff);
  uint32_t sc = (uint32_t)(ag.x >> 32);
  // reset-ahead (xmg_main.cuh): stage 2 = the next trial's records are in
  // next_* (pre-built by the batches VecEnv.rollout launches before this
  // kernel, or by earlier steps); a trial ending at stage 2 is reset by
  // copying them into the warp's grid (roll_consume)
  int stage = (int)((ag.x >> 18) & 3);
  uint32_t goal_word = (uint32_t)ag.y;
  int task = (int)(ag.y >> 32);
  uint32_t* rbuf = rules_s + lane * (geo.rbw / 4);
  auto load_row = [&](int who, int tk) {  // whole warp: task row header + rules of lane `who`
    if (R == 0) return;
    // rows and the shared row slots are 16-byte aligned and rbw bytes long
    const uint4* src = reinterpret_cast<const uint4*>(d.task_rows + (int64_t)tk * d.row_words);
    uint4* dst = reinterpret_cast<uint4*>(rules_s + who * (geo.rbw / 4));
    for (int i = lane; i < geo.rbw / 16; i += 32) dst[i] = src[i];
  };
  if (R > 0 && valid) {
    const uint4* src = reinterpret_cast<const uint4*>(d.task_rows + (int64_t)task * d.row_words);
    for (int i = 0; i < geo.rbw / 16; ++i) reinterpret_cast<uint4*>(rbuf)[i] = src[i];
  }
  __syncwarp();

  SView vw;
  vw.stage = grids + lane * HW;
#ifdef XMG_CHECKS
  vw.hw = HW;
#endif
  double st_ret = 0.0, st_trials = 0.0, st_len = 0.0;
  uint32_t acts4 = 0;

  for (int64_t t = 0; t < T; ++t) {
    // ---- action of this step
    int act = 1;
    const int64_t tt = t0 + t;
    if (actions != nullptr) {
      if (valid) act = actions[t * n + e];
    } else {
      if (t == 0 || (tt & 3) == 0) acts4 = valid ? policy_block(pk.x, pk.y, (uint64_t)(tt >> 2)) : 0x01010101u;
      act = (int)((acts4 >> (8 * (tt & 3))) & 0xff);
    }
    int ev = -1;
    bool goal = false;
    if (valid) {
      // ---- action, ref:vecenv.py:306-342 / ref:env.py:148-191 (select-based)
      const int tr = r + dir_dr(dir), tc = c + dir_dc(dir);
      const bool inside = tr >= 0 && tr < H && tc >= 0 && tc < W;
      const int tflat = tr * W + tc;
      const int tcode = inside ? vw.stage[tflat] : 0, ttile = tcode >> 4;
      const bool mv = act == 0 && inside && ((kWalkable >> ttile) & 1);
      const bool pkup = act == 3 && inside && pocket == 0 && ((kPickable >> ttile) & 1);
      const bool pt = act == 4 && inside && pocket != 0 && ttile == kFloor;
      const bool tg = act == 5 && inside && (ttile == kClosed || (ttile == kLocked && pocket == kKey * 16 + (tcode & 15)));
      ev = mv ? 0 : pkup ? 1 : pt ? 2 : tg ? 3 : -1;
      const int wval = pkup ? kFloorCode : pt ? pocket : kOpen * 16 + (tcode & 15);
      r = mv ? tr : r;
      c = mv ? tc : c;
      dir = act == 1 ? ((dir + 3) & 3) : act == 2 ? ((dir + 1) & 3) : dir;
      pocket = pkup ? tcode : pt ? 0 : pocket;
      if (pkup || pt || tg) vw.stage[tflat] = (uint8_t)wval;
      // ---- MOVE / PICK_UP: agent-relative rules (gated slots, stored order) and goal
      if (ev == 0 || ev == 1) {
        Nbrs nb = load_nbrs(vw, H, W, r, c);
        const int nr = R > 0 ? (int)(rbuf[1] & 0xff) : 0;
        if (nr) {
          if (R <= 32) {
            const uint32_t slots = rbuf[2 + ev];
            if (slots) pocket = agent_rules(vw, nb, rbuf + kRowHeader, slots, pocket);
          } else {
            for (int s0 = 0; s0 < nr; ++s0) {
              const int kind = rbuf[kRowHeader + s0] & 0xff;
              if (kind >= 1 && kind <= 11 && ((cRuleGate[kind] >> ev) & 1))
                pocket = agent_rules(vw, nb, rbuf + kRowHeader + s0, 1u, pocket);
            }
          }
        }
        goal = agent_goal(nb, vw.stage[r * W + c], goal_word, ev, r, c, pocket);
      }
    }
    // ---- PUT_DOWN: grid-wide rules and goal, one env at a time by the warp
    for (uint32_t pm = __ballot_sync(0xffffffffu, ev == 2); pm; pm &= pm - 1) {
      const int src = __ffs(pm) - 1;
      uint8_t* G = grids + src * HW;
      const int ar = __shfl_sync(0xffffffffu, r, src), ac = __shfl_sync(0xffffffffu, c, src);
      const uint32_t gw_src = __shfl_sync(0xffffffffu, goal_word, src);
      const uint32_t* rt = rules_s + src * (geo.rbw / 4);
      const int nr = R > 0 ? (int)(rt[1] & 0xff) : 0;
      const int res = warp_put_env(G, G, cand, lane, H, W, ar, ac, rt + kRowHeader, nr, gw_src);
      if (lane == src) goal = res & 1;
    }
    // ---- counters, reward, record, ref:vecenv.py:351-357
    float rew = 0.f;
    bool last = false;
    if (valid) {
      sc += 1;
      last = goal || sc >= (uint32_t)d.budget;
      if (goal) rew = goal_reward(sc, d.budget);
      const int64_t oi = t * n + e;
      if (o.reward) o.reward[oi] = rew;
      if (o.discount) o.discount[oi] = last ? 0.f : 1.f;
      if (o.step_type) o.step_type[oi] = last ? 2 : 1;
      st_ret += (double)rew;
      if (last) {
        st_trials += 1.0;
        st_len += (double)sc;
      }
    }
    // ---- auto-reset of finished trials (ref:vecenv.py:359-361 -> :224-291)
    uint32_t lm = __ballot_sync(0xffffffffu, last);
    if (lm) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // obs buffers free
      __syncwarp();
      // pre-built successors: the records in (out of line: keeps the step
      // loop's code small), state into the lane's registers
      const uint32_t cm = __ballot_sync(0xffffffffu, last && stage == 2);
      if (cm) {
        const ulonglong4 w = roll_consume(s, cm, __ballot_sync(0xffffffffu, buf != 0), e0, HW, grids, lane);
        if ((cm >> lane) & 1) {
          buf ^= 1u;
          r = (int)(w.x & 0xff);
          c = (int)((w.x >> 8) & 0xff);
          dir = (int)((w.x >> 16) & 3);
          pocket = 0;
          sc = 0;
          stage = 0;
          goal_word = (uint32_t)w.y;
          task = (int)(w.y >> 32);
          rk = make_ulonglong2(w.z, w.w);
        }
        if (resample)
          for (uint32_t m = cm; m; m &= m - 1) load_row(__ffs(m) - 1, __shfl_sync(0xffffffffu, task, __ffs(m) - 1));
        __syncwarp();
        lm &= ~cm;
      }
      for (int half = 0; half < 32; half += kRollKeySlots) {
      uint32_t hm = lm & (kRollKeySlots == 32 ? 0xffffffffu : (((1u << kRollKeySlots) - 1u) << half));
      if (!hm) continue;
      derive_keys_group(hm, half, rk.x, rk.y, resample, keys, lane);
      for (; hm; hm &= hm - 1) {
        const int src = __ffs(hm) - 1;
        const int tk = __shfl_sync(0xffffffffu, task, src);
        const uint32_t g_in = xland ? d.task_rows[(int64_t)tk * d.row_words] : 0u;
        warp_build(sdesc, scratch, geo.hwp, lane, keys + (src - half), tk, g_in, grids + src * HW, rout);
        const ResetOut ro = *rout;
        if (lane == src) {
          r = ro.r;
          c = ro.c;
          dir = ro.d;
          pocket = 0;
          sc = 0;
          stage = 0;
          goal_word = ro.goal;
          task = ro.task;
          rk = make_ulonglong2(ro.st_hi, ro.st_lo);
        }
        if (resample) load_row(src, ro.task);
        __syncwarp();
      }
      }
    }
    // ---- observation of the next playable state: staged, one bulk store per warp
    if (o.obs != nullptr) {
      uint8_t* ob = obs_s + (int)(t & 1) * (geo.obs / 2);
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // this buffer's last store
      __syncwarp();
      if (valid) {
        uint8_t* dst = ob + lane * geo.ob;
        if (see) {
          if (V == 5) obs_see<5>(vw.stage, 0, dst, r, c, dir, H, W, V);
          else obs_see<0>(vw.stage, 0, dst, r, c, dir, H, W, V);
        } else {
          View ov;
          ov.g = ov.stage = vw.stage;
          ov.sbase = ov.slo = 0;
          ov.shi = HW;
          obs_occluded(ov, dst, r, c, dir, H, W, V);
        }
      }
      const uint32_t bytes = (uint32_t)(nvalid * geo.ob);
      uint8_t* gdst = o.obs + (t * n + e0) * geo.ob;
      const bool aligned = (reinterpret_cast<uintptr_t>(gdst) & 15) == 0;
      const uint32_t bulk = aligned ? (bytes & ~15u) : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0 && bulk) {
        const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(ob);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(saddr),
                     "r"(bulk) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      for (uint32_t q = bulk + lane; q < bytes; q += 32) gdst[q] = ob[q];
    }
  }

  // ---- state out
  __syncwarp();
  roll_grids_io(s, e0, vmask, __ballot_sync(0xffffffffu, buf != 0), HW, grids, true, lane);
  if (valid) {
    reinterpret_cast<ulonglong2*>(s.agent)[e] =
        make_ulonglong2(pack_agent(r, c, dir | (stage << 2) | (int)(buf << 4), pocket, sc),
                        (uint64_t)goal_word | ((uint64_t)(uint32_t)task << 32));
    reinterpret_cast<ulonglong2*>(s.rng)[e] = rk;
  }
  if (o.stats != nullptr) warp_stats(o.stats, (int)(e0 / kStatEnvs), st_ret, st_trials, st_len);
  if (lane == 0 && o.obs != nullptr) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
