// xmg_rare.cuh — step_rare: the warp-per-env drain of the PUT_DOWN and
// reset queues, with the warp-level PUT_DOWN rule pass (included by
// xmg_step.cu inside its anonymous namespace).

// ------------------------------------------------------- step_rare
// Observation of pose (r, c, d) on a shared-memory grid copy G, by one lane
// (lane_obs) or one view cell per lane (warp_obs), written straight to the
// env's (v, v, 2) record.
__device__ __forceinline__ uint16_t obs_cell(const uint8_t* G, int r, int c, int d, int H, int W, int V, int cell,
                                             bool see) {
  const int h = V / 2;
  const int fr = dir_dr(d), fc = dir_dc(d), rr = fc, rc = -fr;
  const int i = V == 5 ? cell / 5 : cell / V, j = cell - i * V;  // (the registered views are 5)
  const int ahead = V - 1 - i, lat = j - h;
  const int wr = r + ahead * fr + lat * rr, wc = c + ahead * fc + lat * rc;
  if (wr < 0 || wr >= H || wc < 0 || wc >= W) return 0;
  if (!see) {
    View vw;  // grid fully staged: stage == G, range [0, HW)
    vw.g = nullptr;
    vw.stage = const_cast<uint8_t*>(G);
    vw.sbase = 0;
    vw.slo = 0;
    vw.shi = H * W;
    if (!cell_visible(vw, W, r, c, wr, wc)) return 1 | (1 << 8);  // (UNSEEN, UNSEEN)
  }
  const int code = G[wr * W + wc];
  return (uint16_t)((code >> 4) | ((code & 15) << 8));
}

__device__ __noinline__ void warp_obs(const uint8_t* G, uint8_t* gobs, int lane, int r, int c, int d, int H, int W,
                                      int V, bool see) {
  for (int cell = lane; cell < V * V; cell += 32)
    reinterpret_cast<uint16_t*>(gobs)[cell] = obs_cell(G, r, c, d, H, W, V, cell, see);
}

// ------------------------------------------------------- warp-level PUT_DOWN
// One PUT_DOWN event is resolved by a whole warp on a shared-memory copy G of
// the env's grid.  Rules are evaluated speculatively in parallel, lane s on
// rule slot s0 + s against the current grid: the first slot that fires is the
// one the sequential pass (ref:rules.py:162-213) would apply first, since no
// earlier slot changed anything; it is applied and evaluation restarts after
// it.  Events fire at most a few rules, so this is one or two rounds.  TILE
// rules scan a candidate list (every cell that is neither floor nor wall, in
// row-major order, built with ballots); generated rule inputs are objects, so
// only a scan for a floor / wall code falls back to the full grid.

// `b` at the neighbour of cell pos in the direction the variant tries
// (dir -1: first of NEAR_OFFSETS up, left, right, down; 0 up 1 right 2 down 3 left)
__device__ __forceinline__ int nb_match(const uint8_t* G, int H, int W, int pos, int b, int dir) {
  const int r = pos / W, c = pos - r * W;
  const bool up = r > 0 && G[pos - W] == b, left = c > 0 && G[pos - 1] == b;
  const bool right = c + 1 < W && G[pos + 1] == b, down = r + 1 < H && G[pos + W] == b;
  if (dir < 0) return up ? pos - W : left ? pos - 1 : right ? pos + 1 : down ? pos + W : -1;
  if (dir == 0) return up ? pos - W : -1;
  if (dir == 1) return right ? pos + 1 : -1;
  if (dir == 2) return down ? pos + W : -1;
  return left ? pos - 1 : -1;
}

__device__ __forceinline__ bool is_cand(int code) { return code != kFloorCode && code != kWallCode; }

// candidate list of G into cand[] (pos << 8 | code); returns the count
__device__ __forceinline__ int warp_cands(const uint8_t* G, int HW, uint32_t* cand, int lane) {
  int nc = 0;
  for (int base = 0; base < HW; base += 32) {
    const int p = base + lane;
    const int code = p < HW ? G[p] : kFloorCode;
    const uint32_t m = __ballot_sync(0xffffffffu, is_cand(code));
    if (is_cand(code)) cand[nc + __popc(m & ((1u << lane) - 1u))] = ((uint32_t)p << 8) | (uint32_t)code;
    nc += __popc(m);
  }
  __syncwarp();
  return nc;
}

// First cell (row-major) holding `a` with `b` at the neighbour of `dir`
// (ref:rules.py:192-213), by the whole warp: a ballot per 32 candidates (or
// cells, when `a` is floor / wall and so not in the candidate list).  Returns
// the cell and its neighbour `q` on every lane, or -1.
__device__ __forceinline__ int warp_tile_find(const uint8_t* G, const uint32_t* cand, int nc, int H, int W, int a,
                                              int b, int dir, int lane, int& q) {
  const bool in_list = is_cand(a);
  const int total = in_list ? nc : H * W;
  for (int base = 0; base < total; base += 32) {
    const int i = base + lane;
    int pos = -1, nb = -1;
    if (i < total) {
      int code;
      if (in_list) {
        const uint32_t en = cand[i];
        pos = (int)(en >> 8);
        code = (int)(en & 0xff);
      } else {
        pos = i;
        code = G[i];
      }
      if (code == a) nb = nb_match(G, H, W, pos, b, dir);
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, nb >= 0);
    if (hit) {
      const int w = __ffs(hit) - 1;
      q = __shfl_sync(0xffffffffu, nb, w);
      return __shfl_sync(0xffffffffu, pos, w);
    }
  }
  q = -1;
  return -1;
}

// The PUT_DOWN rule pass then the goal (ref:goals.py:130-177) of one env,
// whole warp; rewritten cells go to G and through to `genv` in global
// memory.  Returns goal | dirty << 1 on every lane.
__device__ __noinline__ int warp_put_env(uint8_t* G, uint8_t* genv, uint32_t* cand, int lane, int H, int W, int ar,
                                         int ac, const uint32_t* rules, int nr, uint32_t goal) {
  const int HW = H * W;
  int nc = warp_cands(G, HW, cand, lane);
  bool dirty = false;
  // Slots in stored order, restarting after every slot that fires (it changed
  // the grid).  AGENT_NEAR-family slots are cheap: lane s evaluates slot s0 + s
  // speculatively on the current grid.  TILE_NEAR-family slots are evaluated
  // only when they come first in order, by the whole warp (a ballot over the
  // candidate list: the lowest hit is the first in row-major order).
  for (int s0 = 0; s0 < nr;) {
    const int sl = s0 + lane;
    int p = -1, q = -1, out = 0;
    bool tile = false;
    if (sl < nr) {
      const uint32_t rw = rules[sl];
      const int kind = rw & 0xff, a = (rw >> 8) & 0xff;
      out = (int)(rw >> 24);
      if (kind == 2 || (kind >= 8 && kind <= 11)) {  // AGENT_NEAR family
        for (int k = 0; k < 4; ++k) {
          const int kk = kind == 2 ? k : dir_slot(kind - 8);
          const int r = ar + near_dr(kk), c = ac + near_dc(kk);
          if (r >= 0 && r < H && c >= 0 && c < W && G[r * W + c] == a) { p = r * W + c; break; }
          if (kind != 2) break;
        }
      } else if (kind >= 3 && kind <= 7) {  // TILE_NEAR family: resolved below, in order
        tile = true;
      }
    }
    const uint32_t fired = __ballot_sync(0xffffffffu, p >= 0);
    uint32_t pend = fired | __ballot_sync(0xffffffffu, tile);
    int w = -1;
    while (pend) {
      const int t = __ffs(pend) - 1;
      if ((fired >> t) & 1) {
        p = __shfl_sync(0xffffffffu, p, t);
        q = __shfl_sync(0xffffffffu, q, t);
        out = __shfl_sync(0xffffffffu, out, t);
        w = t;
        break;
      }
      const uint32_t rw = rules[s0 + t];
      const int kind = rw & 0xff, a = (rw >> 8) & 0xff, b = (rw >> 16) & 0xff;
      const int pt = warp_tile_find(G, cand, nc, H, W, a, b, kind == 3 ? -1 : kind - 4, lane, q);
      if (pt >= 0) {
        p = pt;
        out = (int)(rw >> 24);
        w = t;
        break;
      }
      pend &= pend - 1;
    }
    if (w < 0) {
      s0 += 32;
      continue;
    }
    XMG_ASSERT(p >= 0 && p < HW && q < HW);
    const int old = G[p];
    __syncwarp();
    if (lane == 0) {
      G[p] = (uint8_t)out;
      genv[p] = (uint8_t)out;
      if (q >= 0) {
        G[q] = kFloorCode;
        genv[q] = kFloorCode;
      }
    }
    __syncwarp();
    if (!is_cand(old) && is_cand(out)) {
      nc = warp_cands(G, HW, cand, lane);  // a new candidate cell: rebuild (rare)
    } else {
      for (int i = lane; i < nc; i += 32) {  // keep the list in step with G (positions unchanged)
        const int pos = (int)(cand[i] >> 8);
        if (pos == p) cand[i] = ((uint32_t)p << 8) | (uint32_t)out;
        else if (pos == q) cand[i] = ((uint32_t)q << 8) | kFloorCode;
      }
      __syncwarp();
    }
    dirty = true;
    s0 += w + 1;
  }
  bool hit = false;
  const int kind = goal & 0xff, a1 = (goal >> 8) & 0xff, a2 = (goal >> 16) & 0xff, a3 = goal >> 24;
  if (kind != 0 && kind <= 14 && ((cGoalGate[kind] >> 2) & 1)) {
    switch (kind) {
      case 2: hit = G[ar * W + ac] == a1; break;
      case 5: hit = ar == a1 && ac == a2; break;
      case 6: hit = a2 < H && a3 < W && G[a2 * W + a3] == a1; break;
      case 3:
        for (int k = 0; k < 4; ++k) {
          const int r = ar + near_dr(k), c = ac + near_dc(k);
          hit |= r >= 0 && r < H && c >= 0 && c < W && G[r * W + c] == a1;
        }
        break;
      case 11: case 12: case 13: case 14: {
        const int r = ar + dir_dr(kind - 11), c = ac + dir_dc(kind - 11);
        hit = r >= 0 && r < H && c >= 0 && c < W && G[r * W + c] == a1;
        break;
      }
      default: {  // TILE_NEAR goals: any matching cell, lanes over candidates / cells
        const int dir = kind == 4 ? -1 : kind - 7;
        bool any = false;
        if (is_cand(a1)) {
          for (int i = lane; i < nc; i += 32) {
            const uint32_t en = cand[i];
            any |= (int)(en & 0xff) == a1 && nb_match(G, H, W, (int)(en >> 8), a2, dir) >= 0;
          }
        } else {
          for (int p = lane; p < HW; p += 32) any |= G[p] == a1 && nb_match(G, H, W, p, a2, dir) >= 0;
        }
        hit = __any_sync(0xffffffffu, any);
      }
    }
  }
  return (int)hit | ((int)dirty << 1);
}


// Every lane's writes for the envs the warp just finished are made visible,
// then each `mine` lane releases its env's chunk for the next step_main.
__device__ __forceinline__ void release_envs(uint32_t* pending, bool mine, int64_t e) {
  __threadfence();
  __syncwarp();
  if (mine) atomicSub(pending + e / 32, 1u);
}

#ifndef XMG_PUT_BATCH
#define XMG_PUT_BATCH 6  // C3 76.7 -> 76.4 us, DoorKey-8x8 68.5 -> 68.3 vs 8 (4: 76.4 / 68.6)
#endif
#ifndef XMG_BUILD_COST
#define XMG_BUILD_COST 4.0  // a trial build's cost in PUT_DOWN events (the warp split below)
#endif
constexpr int kPutBatch = XMG_PUT_BATCH;  // PUT_DOWN envs a step_rare warp prefetches together
#ifndef XMG_RARE_WARPS
#define XMG_RARE_WARPS 4
#endif
constexpr int kRareWarps = XMG_RARE_WARPS;  // warps per step_rare CTA (each warp owns its scratch)
constexpr int kRareWarpsPerSM = 20;         // resident step_rare warps per SM (see launch_rare)
constexpr int kKeySlots = 16;  // trial keys derived in parallel per warp (resets go in half-warp groups)
static_assert(kPutBatch <= kKeySlots, "a PUT_DOWN batch derives its finished trials' keys at once");

struct RareGeo {
  int hwp, ws, rbw, keys, pgb, put;
  int64_t total;
};


__host__ __device__ inline RareGeo make_rare_geo(int H, int W, int R) {
  RareGeo g;
  g.hwp = round16(H * W + 16);
  g.rbw = round16(4 * (kRowHeader + R));
  g.keys = kKeySlots * (int)sizeof(TrialKeys);
  g.pgb = round16(H * W + 32);                      // one prefetched grid (16-byte chunks, unaligned start)
  g.put = kPutBatch * (g.pgb + g.rbw + 16) + 4 * g.hwp;  // grids | rule rows | state words | candidates
  // per warp: wd: u64[hwp] | fc: u16[hwp] | slot: u16[hwp] | bk: u32[2^lg] | grid: u8[hwp] | misc: 64 u64
  //           | rules | 32 trial keys | env description
  g.ws = warp_scratch_bytes(g.hwp) + g.rbw + g.keys +
         round16((int)sizeof(xmg_env_desc)) + g.put;
  g.total = (int64_t)kRareWarps * g.ws;
  return g;
}

// Rebuild env e's trial (ref:vecenv.py:359-361 -> :224-291), whole warp.
// The grid goes to the env's current buffer `buf` (xmg_main.cuh kBufBit),
// which the new state word keeps.  pre (reset-ahead): the same build from the
// same keys, written to the OTHER buffer and to the env's next_* records
// (state word naming that buffer, rng, first observation) for the auto-reset
// that will end the running trial; nothing of the running trial is touched.
__device__ __forceinline__ void warp_reset_env(const xmg_env_desc& d, const xmg_env_desc* sd, const xmg_state& s,
                                               const xmg_out& o, uint8_t* wbase, const RareGeo& geo, int lane,
                                               int64_t e, const TrialKeys* key, int task, bool reset_mode,
                                               ResetOut* rs, bool pre = false, uint32_t buf = 0) {
  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, ob = 2 * V * V;
  const WarpScratch ws = make_scratch(wbase, geo.hwp);
  const uint32_t g_in = d.scenario == XMG_SCENARIO_XLAND ? d.task_rows[(int64_t)task * d.row_words] : 0u;
  const uint32_t dst_buf = pre ? buf ^ 1u : buf;
  warp_build(sd, wbase, geo.hwp, lane, key, task, g_in, grid_ptr(s, e, HW, dst_buf), rs);
  const ResetOut ro = *rs;
  const ulonglong2 word = make_ulonglong2(pack_agent(ro.r, ro.c, ro.d | (int)(dst_buf << 4), 0, 0),
                                          (uint64_t)ro.goal | ((uint64_t)(uint32_t)ro.task << 32));
  if (lane == 0) {
    if (pre) {
      ulonglong2* ns = reinterpret_cast<ulonglong2*>(s.next_state) + 2 * e;
      ns[0] = word;
      ns[1] = make_ulonglong2(ro.st_hi, ro.st_lo);
    } else {
      reinterpret_cast<ulonglong2*>(s.rng)[e] = make_ulonglong2(ro.st_hi, ro.st_lo);
      reinterpret_cast<ulonglong2*>(s.agent)[e] = word;
    }
    if (reset_mode) {
      o.reward[e] = 0.f;
      o.discount[e] = 1.f;
      o.step_type[e] = 0;
    }
  }
  uint8_t* obs = pre ? s.next_obs : o.obs;
  if (obs != nullptr) warp_obs(ws.grid, obs + e * ob, lane, ro.r, ro.c, ro.d, H, W, V, d.see_through_walls != 0);
  __syncwarp();
  XMG_TRB(6);
}

// The auto-resets of the PUT_DOWN envs in cm (lanes of a step_rare batch,
// env e_l per lane) from their pre-built records: state word (its buffer bit
// names the other grid buffer, where the record's grid is) and rng per lane,
// then each env's first observation copied by the whole warp.
__device__ __noinline__ void put_consume(const xmg_state s, const xmg_out o, uint32_t cm, int64_t e_l, int ob,
                                         int lane) {
  if ((cm >> lane) & 1) {
    const ulonglong2* ns = reinterpret_cast<const ulonglong2*>(s.next_state) + 2 * e_l;
    const ulonglong2 a = __ldcg(ns), b = __ldcg(ns + 1);
    reinterpret_cast<ulonglong2*>(s.agent)[e_l] = a;
    reinterpret_cast<ulonglong2*>(s.rng)[e_l] = b;
  }
  if (o.obs != nullptr)
    for (uint32_t m = cm; m; m &= m - 1) {
      const int64_t e = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e_l, __ffs(m) - 1);
      warp_copy_cg(o.obs + e * ob, s.next_obs + e * ob, ob, lane);
    }
  __syncwarp();
}

// Resets of a group of up to 32 envs (one per lane, `mine`): each lane
// derives its env's trial keys, then the warp rebuilds the envs one by one.
__device__ __forceinline__ void warp_reset_group(const xmg_env_desc& d, const xmg_env_desc* sd, const xmg_state& s,
                                                 const xmg_out& o, uint8_t* wbase, const RareGeo& geo,
                                                 TrialKeys* keys, int lane, bool mine, int64_t e,
                                                 const uint64_t* reset_keys, int gw = 0, bool pre = false,
                                                 uint32_t buf = 0) {
  const bool resample = d.resample_tasks && d.scenario == XMG_SCENARIO_XLAND;
  int task = 0;
  ulonglong2 ek = make_ulonglong2(0, 0);
  if (mine) {
    ek = reinterpret_cast<const ulonglong2*>(reset_keys ? reset_keys : s.rng)[e];
    task = (int)(reinterpret_cast<const ulonglong2*>(s.agent)[e].y >> 32);
  }
#ifdef XMG_TRACE
  XMG_TR(gw, 7, gtime());
#endif
  // kKeySlots lanes at a time derive their keys in parallel, then the warp
  // rebuilds those envs one by one
  for (int half = 0; half < 32; half += kKeySlots) {
    const bool in = mine && lane >= half && lane < half + kKeySlots;
    uint32_t m = __ballot_sync(0xffffffffu, in);
    derive_keys_group(m, half, ek.x, ek.y, resample, keys, lane);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int64_t es = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e, src);
      const int ts = __shfl_sync(0xffffffffu, task, src);
      const bool ps = __shfl_sync(0xffffffffu, (int)pre, src) != 0;
      const uint32_t bs = __shfl_sync(0xffffffffu, buf, src);
      warp_reset_env(d, sd, s, o, wbase, geo, lane, es, keys + (src - half), ts, reset_keys != nullptr,
                     reinterpret_cast<ResetOut*>(make_scratch(wbase, geo.hwp).misc + 40), ps, bs);
    }
  }
}

// step_rare drains the two queues step_main filled, one env per warp:
//  * PUT_DOWN queue: the grid-wide rule pass, goal, reward (warp_put_env);
//  * reset queue: the trial rebuild (warp_build), 32 envs' keys at a time.
// Sub-queue q of each kind is served by the warps gw with gw % kQueues == q,
// striding over its entries; warps without entries exit at once.
// reset_keys != nullptr: reset mode (ref VecEnv.reset_with_keys,
// vecenv.py:205-222), every env [0, n) rebuilt from keys[e] with a FIRST
// record.
__global__ void __launch_bounds__(kRareWarps * 32, XMG_MINB_RARE * 4 / kRareWarps) step_rare(const xmg_env_desc d, const xmg_state s,
                                                                     const xmg_out o, const uint64_t* reset_keys,
                                                                     const uint32_t* abort_flag, uint32_t epoch,
                                                                     int64_t n, int track) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = blockIdx.x * kRareWarps + warp, tw = gridDim.x * kRareWarps;
#ifdef XMG_TRACE
  const unsigned long long t_start = gtime();
  XMG_TR(gw, 0, t_start);
#endif
  const bool reset_mode = reset_keys != nullptr;
  const int q = gw % kQueues, j = gw / kQueues, per_q = tw / kQueues;
  int64_t cnt_put = 0, cnt_reset = 0;
  // the sub-queue's warps split into PUT_DOWN warps [0, put_w) and reset
  // warps [put_w, per_q), in proportion to the work (a trial build costs
  // about four PUT_DOWN events), so a warp's chain is PUT_DOWN envs or builds,
  // not both
  int put_w = per_q, jp = j, jr = -1, rs_w = 0;
  if (!reset_mode) {
    // launched as a programmatic dependent of this step's step_main: the
    // queues are complete once that grid has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    cnt_put = s.work[count_index(epoch, 0, q)];
    cnt_reset = s.work[count_index(epoch, 1, q)];
    if (cnt_reset > 0 && per_q < 2) {  // a single warp per sub-queue does both
      rs_w = per_q;
      jr = j;
    } else if (cnt_reset > 0) {
      if (cnt_put == 0) {
        rs_w = per_q;
      } else {
        const double wr = XMG_BUILD_COST * (double)cnt_reset, wp = (double)cnt_put;
        rs_w = (int)(per_q * wr / (wr + wp) + 0.5);
        rs_w = rs_w < 1 ? 1 : rs_w > per_q - 1 ? per_q - 1 : rs_w;
      }
      put_w = per_q - rs_w;
      if (j >= put_w) {
        jp = -1;
        jr = j - put_w;
      }
    }
    const bool idle = (jp < 0 || jp >= cnt_put) && (jr < 0 || jr >= cnt_reset);
    // the counts are read (and used): the next step's step_main may launch
    // (it clears them), and waits per tile on `pending` for the envs below
    if (track) griddep_launch();
    if (idle) return;  // nothing queued for this warp
  } else if (gw >= n) {
    return;
  }
  if (batch_rejected(abort_flag, epoch)) return;

  const int H = d.height, W = d.width, HW = H * W, V = d.view_size, ob = 2 * V * V, R = d.rule_width;
  const RareGeo geo = make_rare_geo(H, W, R);
  uint8_t* wbase = smem + warp * geo.ws;
  const WarpScratch ws = make_scratch(wbase, geo.hwp);
  uint8_t* tail = wbase + geo.ws - geo.put;  // PUT_DOWN prefetch area
  uint32_t* rules_s = reinterpret_cast<uint32_t*>(tail - geo.rbw - geo.keys - round16((int)sizeof(xmg_env_desc)));
  TrialKeys* keys = reinterpret_cast<TrialKeys*>(tail - geo.keys - round16((int)sizeof(xmg_env_desc)));
  // this warp's copy of the description, for the out-of-line paths
  xmg_env_desc* sdesc = reinterpret_cast<xmg_env_desc*>(tail - round16((int)sizeof(xmg_env_desc)));
  (void)rules_s;
  if (lane == 0) *sdesc = d;
  __syncwarp();
  const bool see = d.see_through_walls != 0;
  const int64_t qcap = queue_cap(n);

  if (reset_mode) {
    for (int64_t g0 = gw; g0 < n; g0 += 32 * (int64_t)tw) {
      const int64_t e = g0 + (int64_t)lane * tw;
      warp_reset_group(d, sdesc, s, o, wbase, geo, keys, lane, e < n, e, reset_keys);
    }
    return;
  }

  // ---- PUT_DOWN events: entries j, j + per_q, ... of sub-queue q, kPutBatch
  // at a time prefetched into shared memory (one env per lane), then
  // resolved one by one by the whole warp
  if (jp >= 0 && jp < cnt_put) {
    const uint32_t* qp = s.work + queue_base(n, epoch, 0, q);
    uint8_t* pg = tail;                                                  // kPutBatch grids
    uint32_t* pr = reinterpret_cast<uint32_t*>(tail + kPutBatch * geo.pgb);  // kPutBatch rule rows
    ulonglong2* pa = reinterpret_cast<ulonglong2*>(tail + kPutBatch * (geo.pgb + geo.rbw));  // state words
    uint32_t* pc = reinterpret_cast<uint32_t*>(tail + kPutBatch * (geo.pgb + geo.rbw + 16));  // candidates
    const bool resample = d.resample_tasks && d.scenario == XMG_SCENARIO_XLAND;
    for (int64_t i0 = jp; i0 < cnt_put; i0 += (int64_t)kPutBatch * put_w) {
      const int64_t it = i0 + (int64_t)lane * put_w;
      const bool mine = lane < kPutBatch && it < cnt_put;
      int64_t e_l = 0;
      uint32_t buf_l = 0;
      int off_l = 0;
      if (mine) {
        const uint32_t ent = qp[it];
        e_l = (int64_t)(ent & kQEnv);
        buf_l = (ent >> 30) & 1u;
        const uintptr_t g0 = reinterpret_cast<uintptr_t>(grid_ptr(s, e_l, HW, buf_l));
        const uintptr_t a0 = g0 & ~uintptr_t(15);
        off_l = (int)(g0 - a0);
        const int nch = (off_l + HW + 15) >> 4;
        for (int k = 0; k < nch; ++k) cp_async16(pg + lane * geo.pgb + 16 * k, reinterpret_cast<const void*>(a0 + 16 * k));
        const ulonglong2 ag = reinterpret_cast<const ulonglong2*>(s.agent)[e_l];
        pa[lane] = ag;
        if (R > 0) {
          const uint32_t* row = d.task_rows + (int64_t)(ag.y >> 32) * d.row_words;
          for (int k = 0; k < (kRowHeader + R + 3) >> 2; ++k) cp_async16(pr + lane * (geo.rbw / 4) + 4 * k, row + 4 * k);
        }
        cp_async_wait_all();
      }
      __syncwarp();
#ifdef XMG_TRACE
      if (i0 == j) XMG_TR(gw, 4, gtime());
#endif
      uint32_t m = __ballot_sync(0xffffffffu, mine), lastm = 0;
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int64_t e = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e_l, src);
        const int off = __shfl_sync(0xffffffffu, off_l, src);
        const ulonglong2 ag = pa[src];
        const int r = (int)(ag.x & 0xff), c = (int)((ag.x >> 8) & 0xff), dir = (int)((ag.x >> 16) & 3);
        const uint32_t sc = (uint32_t)(ag.x >> 32);
        const uint32_t* rt = pr + src * (geo.rbw / 4);
        const int nr = R > 0 ? (int)(rt[1] & 0xff) : 0;
        uint8_t* G = pg + src * geo.pgb + off;
        const uint32_t bs = __shfl_sync(0xffffffffu, buf_l, src);
        const int res = warp_put_env(G, grid_ptr(s, e, HW, bs), pc, lane, H, W, r, c, rt + kRowHeader, nr,
                                     (uint32_t)ag.y);
        const bool last = (res & 1) || sc >= (uint32_t)d.budget;
#ifdef XMG_TRACE
        if (i0 == j && src == 0) XMG_TR(gw, 5, gtime());
#endif
        if (lane == 0) {
          const float rew = (res & 1) ? goal_reward(sc, d.budget) : 0.f;
          o.reward[e] = rew;
          o.discount[e] = last ? 0.f : 1.f;
          o.step_type[e] = last ? 2 : 1;
          if (o.stats != nullptr && (rew != 0.f || last)) {
            const int slot = (int)(e / kStatEnvs);
            atomicAdd(o.stats + 3 * slot, (double)rew);
            if (last) {
              atomicAdd(o.stats + 3 * slot + 1, 1.0);
              atomicAdd(o.stats + 3 * slot + 2, (double)sc);
            }
          }
        }
        // a rule changed the grid: the observation step_main wrote is stale
        if ((res & 2) && !last && o.obs != nullptr) warp_obs(G, o.obs + e * ob, lane, r, c, dir, H, W, V, see);
        if (last) lastm |= 1u << src;
      }
#ifdef XMG_TRACE
      if (i0 == j) XMG_TR(gw, 6, gtime());
#endif
      // ---- trials the PUT_DOWN finished: a pre-built successor taken over
      // (out of line: keeps step_rare's registers), else keys derived
      // lane-parallel and the envs rebuilt by the whole warp
      if (lastm && ahead_on(s)) {
        // trials with a pre-built successor (stage 2, e.g. every PUT_DOWN of a
        // synchronized budget end) take it over like step_main does
        const bool ready = ((lastm >> lane) & 1) && ((pa[lane].x & kStageMask) == kStageReady);
        const uint32_t cm = __ballot_sync(0xffffffffu, ready);
        if (cm) {
          put_consume(s, o, cm, e_l, ob, lane);
          lastm &= ~cm;
        }
      }
      if (lastm) {
        ulonglong2 ek = make_ulonglong2(0, 0);
        if ((lastm >> lane) & 1) ek = reinterpret_cast<const ulonglong2*>(s.rng)[e_l];
        derive_keys_group(lastm, 0, ek.x, ek.y, resample, keys, lane);
        while (lastm) {
          const int src = __ffs(lastm) - 1;
          lastm &= lastm - 1;
          const int64_t es = (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)e_l, src);
          const int ts = (int)(pa[src].y >> 32);
          const uint32_t bs = __shfl_sync(0xffffffffu, buf_l, src);
          warp_reset_env(d, sdesc, s, o, wbase, geo, lane, es, keys + src, ts, false,
                         reinterpret_cast<ResetOut*>(ws.misc + 40), false, bs);
        }
      }
      if (track) release_envs(s.work + pending_base(n), mine, e_l);
    }
  }
#ifdef XMG_TRACE
  XMG_TR(gw, 1, gtime());
  XMG_TR(gw, 3, (unsigned long long)cnt_put | ((unsigned long long)cnt_reset << 32));
#endif
  // ---- trial resets, 32 at a time (entries i0 + lane * per_q)
  if (jr >= 0 && jr < cnt_reset) {
    const uint32_t* qp = s.work + queue_base(n, epoch, 1, q);
    for (int64_t i0 = jr; i0 < cnt_reset; i0 += 32 * (int64_t)rs_w) {
      const int64_t i = i0 + (int64_t)lane * rs_w;
      const bool mine = i < cnt_reset;
      const uint32_t ent = mine ? qp[i] : 0u;
      const int64_t e = (int64_t)(ent & kQEnv);
      warp_reset_group(d, sdesc, s, o, wbase, geo, keys, lane, mine, e, nullptr, gw, false, (ent >> 30) & 1u);
      if (track) release_envs(s.work + pending_base(n), mine, e);
    }
  }
#ifdef XMG_TRACE
  XMG_TR(gw, 2, gtime());
#endif
}

// ------------------------------------------------------- reset-ahead batch
// prebuild_kernel (xmg_main.cuh "reset-ahead"): the next trial of every env
// e = cls + B * i whose running trial has none yet (stage 0), built by a warp
// per group of kPreGroup envs (keys derived lane-parallel) into state.next_*,
// then marked stage 2.  Warps take groups from a counter (ctr[0]; the last CTA
// to finish re-arms it), so no warp idles while groups remain.  A plain
// launch between two steps: nothing else runs on the state meanwhile.
#ifndef XMG_PRE_GROUP
#define XMG_PRE_GROUP 4  // C3 batch: 3.66 ns/build (8: 4.12, 2: 3.84)
#endif
#ifndef XMG_PRE_MINB
#define XMG_PRE_MINB 6  // resident 4-warp CTAs per SM the register allocation targets
#endif
#ifndef XMG_PRE_WARPS
#define XMG_PRE_WARPS 1  // one-warp CTAs: a finished warp frees its slot at once
#endif
constexpr int kPreWarps = XMG_PRE_WARPS;  // warps per prebuild_kernel CTA
constexpr int kPreGroup = XMG_PRE_GROUP;  // envs per warp group (<= kKeySlots)
static_assert(kPreGroup <= kKeySlots, "a group derives its keys at once");

// per-warp scratch of prebuild_kernel: the build scratch, the trial keys and
// the description (no PUT_DOWN prefetch area)
__host__ __device__ inline int pre_warp_bytes(int H, int W) {
  const int hwp = round16(H * W + 16);
  return warp_scratch_bytes(hwp) + kKeySlots * (int)sizeof(TrialKeys) + round16((int)sizeof(xmg_env_desc));
}

// epoch != 0 (the batch of xmg_step / xmg_steps epoch `epoch`): launched as a
// programmatic dependent, so it may run while the previous step's step_rare
// still drains; an env of a chunk that step queued is read only after that
// step_rare has released the chunk (the protocol of step_main).
__global__ void __launch_bounds__(kPreWarps * 32, XMG_PRE_MINB * 4 / kPreWarps)
    prebuild_kernel(const xmg_env_desc d, const xmg_state s, int64_t cls, int64_t B, int64_t n, uint32_t* ctr,
                    uint32_t epoch) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t count = cls < n ? (n - cls + B - 1) / B : 0;
  const int64_t groups = (count + kPreGroup - 1) / kPreGroup;
  const int ws_bytes = pre_warp_bytes(d.height, d.width);
  const int hwp = round16(d.height * d.width + 16);
  uint8_t* wbase = smem + warp * ws_bytes;
  TrialKeys* keys = reinterpret_cast<TrialKeys*>(wbase + warp_scratch_bytes(hwp));
  xmg_env_desc* sdesc = reinterpret_cast<xmg_env_desc*>(wbase + warp_scratch_bytes(hwp) +
                                                        kKeySlots * (int)sizeof(TrialKeys));
  if (lane == 0) *sdesc = d;
  __syncwarp();
  RareGeo geo;  // the fields warp_reset_env reads
  geo.hwp = hwp;
  const xmg_out none = {nullptr, nullptr, nullptr, nullptr, nullptr};
  for (;;) {
    int64_t g = 0;
    if (lane == 0) g = atomicAdd(ctr, 1u);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= groups) break;
    const int64_t i = g * kPreGroup + lane;
    const int64_t e = cls + B * i;
    uint64_t w0 = 0;
    bool need = false;
    if (lane < kPreGroup && i < count) {
      if (epoch != 0) {
        const int64_t chunk = e >> 5;
        if (s.work[dirty_base(n) + chunk] == epoch - 1) {
          const uint32_t* pending = s.work + pending_base(n) + chunk;
          for (uint32_t spins = 0; ld_acquire(pending) != 0; ++spins) {
            if (spins > (1u << 25)) __trap();
            __nanosleep(128);
          }
        }
        w0 = ld_cg_u64x2(reinterpret_cast<const ulonglong2*>(s.agent) + e).x;
      } else {
        w0 = s.agent[2 * e];
      }
      need = (w0 & kStageMask) == 0;
    }
    warp_reset_group(d, sdesc, s, none, wbase, geo, keys, lane, need, e, nullptr, 0, true,
                     (uint32_t)(w0 >> 20) & 1u);
    if (need) s.agent[2 * e] = w0 | kStageReady;
  }
  // the last CTA re-arms the counter for the next batch
  if (kPreWarps > 1) __syncthreads();
  else __syncwarp();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}
