// xmg_build.cuh — the warp-cooperative trial build (included by xmg_step.cu
// inside its anonymous namespace): ref:vecenv.py:224-291 and the scenario
// builders of ref:scenarios.py, with the stable argsort of the draws replaced
// by a warp radix-select.  Used by step_rare, xmg_reset and the rollout.

// ------------------------------------------------------- warp-cooperative reset
struct ResetOut {
  uint64_t st_hi, st_lo;  // next state key
  int r, c, d;
  uint32_t goal;
  int task;
};

// One warp's trial-build scratch (shared memory), hwp = round16(H*W + 16):
//   wd   u64[hwp]  draw words by free-cell index
//   fc   u16[hwp]  free cells (flat), row-major
//   slot u16[hwp]  the object cells' element indices (rank_place)
//   grid u8[hwp]   the trial grid under construction
//   misc u64[64]   door words [0, 24), agent words [24, 28), spawn [32], ResetOut at [40..)
constexpr int kScratchPad = 16;  // keeps `grid` 16-byte aligned
struct WarpScratch {
  uint64_t* wd;
  uint16_t* fc;
  uint16_t* slot;
  uint8_t* grid;
  uint64_t* misc;
};

__host__ __device__ inline int warp_scratch_bytes(int hwp) { return 12 * hwp + kScratchPad + hwp + 512; }

__device__ __forceinline__ WarpScratch make_scratch(uint8_t* wbase, int hwp) {
  WarpScratch ws;
  ws.wd = reinterpret_cast<uint64_t*>(wbase);
  ws.fc = reinterpret_cast<uint16_t*>(wbase + 8 * hwp);
  ws.slot = reinterpret_cast<uint16_t*>(wbase + 10 * hwp);
  ws.grid = wbase + 12 * hwp + kScratchPad;
  ws.misc = reinterpret_cast<uint64_t*>(ws.grid + hwp);
  return ws;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

// n bytes of the scratch grid (16-byte aligned shared memory, readable
// up to 4 bytes past n) to a grid in global memory at any alignment: a few
// head / tail bytes and 4-byte words, each assembled from two aligned shared
// words with a funnel shift.
__device__ __forceinline__ void warp_store_grid(uint8_t* dst, const uint8_t* src, int n, int lane) {
  const int head = min((int)((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3), n);
  if (lane < head) dst[lane] = src[lane];
  const int words = (n - head) >> 2;
  const int mis = head & 3;  // src offset of the body mod 4 (src is 16-byte aligned)
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src + head - mis);
  uint32_t* d32 = reinterpret_cast<uint32_t*>(dst + head);
  for (int w = lane; w < words; w += 32) {
    const uint32_t lo = s32[w], hi = s32[w + 1];
    d32[w] = mis ? __funnelshift_r(lo, hi, 8 * mis) : lo;
  }
  for (int i = head + 4 * words + lane; i < n; i += 32) dst[i] = src[i];
}

// x mod d for d < 2^16 with 32-bit arithmetic only (the 64-bit remainder is a
// long software sequence): x = hi * 2^32 + lo, so
// x mod d = ((hi mod d) * (2^32 mod d) + lo mod d) mod d, every term < 2^32.
// y mod d for y < 2^53 and 1 <= d < 2^16: the quotient from a double product
// (exact inputs; the estimate is within one of the quotient) then corrected.
__device__ __forceinline__ uint32_t mod_small(uint64_t y, uint32_t d, double rd) {
  const uint64_t q = (uint64_t)__dmul_rz((double)y, rd);
  int64_t r = (int64_t)(y - q * d);
  r += r < 0 ? (int64_t)d : 0;
  r -= r >= (int64_t)d ? (int64_t)d : 0;
  return (uint32_t)r;
}
__device__ __forceinline__ uint32_t mod64_small(uint64_t x, uint32_t d) {
  const double rd = __drcp_rn((double)d);
  const uint32_t a = mod_small(x >> 32, d, rd);  // hi mod d
  // x mod d = (a * 2^32 + lo) mod d, and a * 2^32 + lo < 2^48
  return mod_small(((uint64_t)a << 32) | (uint32_t)x, d, rd);
}

// Row-major floor cells of the scratch grid into fc[]; returns their count
// (the free list of ref:core.py:172-175, built with ballots).
__device__ int build_free_list(const WarpScratch& ws, int HW, int lane) {
  int count = 0;
  for (int base = 0; base < HW; base += 32) {
    const int i = base + lane;
    const bool fl = i < HW && (ws.grid[i] >> 4) == kFloor;
    const uint32_t m = __ballot_sync(0xffffffffu, fl);
    if (fl) ws.fc[count + __popc(m & ((1u << lane) - 1))] = (uint16_t)i;
    count += __popc(m);
  }
  __syncwarp();
  return count;
}

// Philox draw blocks for one env, spread over the lanes: words 0..F-1 of key
// kc into wd[], 2*nseg door words of kd into misc[0..], agent block of ka into
// misc[24..27].  ref:rng.py:113-118 (random_words), ref:vecenv.py:235-240.
__device__ void draw_all(const WarpScratch& ws, int lane, int F, uint64_t kc_hi, uint64_t kc_lo, int nseg,
                         uint64_t kd_hi, uint64_t kd_lo, uint64_t ka_hi, uint64_t ka_lo) {
  const int nO = (F + 3) >> 2, nD = (2 * nseg + 3) >> 2;
  const int jobs = nO + nD + 1;
  for (int j = lane; j < jobs; j += 32) {
    uint64_t* dst;
    uint64_t ctr, kh, kl;
    if (j < nO) {
      ctr = (uint64_t)j; kh = kc_hi; kl = kc_lo;
      dst = ws.wd + 4 * j;
    } else if (j < nO + nD) {
      ctr = (uint64_t)(j - nO); kh = kd_hi; kl = kd_lo;
      dst = ws.misc + 4 * (j - nO);
    } else {
      ctr = 0; kh = ka_hi; kl = ka_lo;
      dst = ws.misc + 24;
    }
    const Words4 w = philox<5>(ctr, 0, kDomDraw, 0, kh, kl);
    dst[0] = w.w0; dst[1] = w.w1; dst[2] = w.w2; dst[3] = w.w3;
  }
  __syncwarp();
}

// Column filter of the port builders: 0 none, 1 col < x, 2 col > x.
__device__ __forceinline__ bool col_ok(int mode, int cell, int W, int x) {
  if (mode == 0) return true;
  const int c = cell % W;
  return mode == 1 ? c < x : c > x;
}

// Warp radix-select over the draw words (ref:core.py:178-183,
// ref:vecenv.py:261-265: cells ordered by (word, index), a stable argsort).
// Element f (free-cell index) is owned by lane (f >> 2) & 31, bit
// 4 * (f >> 7) + (f & 3) of that lane's masks (the lane that drew its
// Philox block in draw_all).  Returns the element of rank t among the
// elements of `cand` (cnt of them, warp-uniform), on every lane.  Uniform
// 64-bit words leave one candidate after ~log2(cnt) bits; equal words fall
// back to index order.
__device__ int warp_select(const uint64_t* wd, int lane, int F, uint32_t cand, int cnt, int t) {
  const int K = (F + 127) >> 7;
  for (int b = 63; b >= 0 && cnt > 1; --b) {
    uint32_t z = 0;
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int bit = 4 * k + i;
        const int f = 128 * k + 4 * lane + i;
        if (((cand >> bit) & 1) && !((wd[f] >> b) & 1)) z |= 1u << bit;
      }
    }
    const int zeros = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(z));
    if (t < zeros) {
      cand = z;
      cnt = zeros;
    } else {
      cand &= ~z;
      t -= zeros;
      cnt -= zeros;
    }
  }
  // the survivors share one word: the t-th of them in index order
  for (int k = 0;; ++k) {
    const uint32_t nib = (cand >> (4 * k)) & 0xFu;
    const int c = __popc(nib);
    int inc = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, off);
      if (lane >= off) inc += v;
    }
    const int tot = __shfl_sync(0xffffffffu, inc, 31), pre = inc - c;
    if (t < tot) {
      int f = -1;
      if (t >= pre && t < inc) {
        uint32_t m = nib;
        for (int r = t - pre; r > 0; --r) m &= m - 1;
        f = 128 * k + 4 * lane + (__ffs(m) - 1);
      }
      const uint32_t who = __ballot_sync(0xffffffffu, f >= 0);
      return __shfl_sync(0xffffffffu, f, __ffs(who) - 1);
    }
    t -= tot;
  }
}

// warp_select with the lane's top-32-bit keys in registers (KR blocks of 4,
// F <= 128 * KR) and branch-free digit masks; two words sharing their top
// half (rare) fall back to the exact 64-bit select.
template <int KR>
__device__ __forceinline__ int warp_select_fast(const uint64_t* wd, int lane, int F, uint32_t cand, int cnt, int t) {
  uint32_t hi[4 * KR];
#pragma unroll
  for (int j = 0; j < 4 * KR; ++j) {
    const int f = 128 * (j >> 2) + 4 * lane + (j & 3);
    hi[j] = f < F ? (uint32_t)(wd[f] >> 32) : 0u;
  }
  uint32_t c = cand;
  int tt = t, cc = cnt;
  // two bits (one base-4 digit) per round: the three digit counts are
  // independent reductions, so a round costs about one reduction's latency
  for (int b = 31; b >= 1 && cc > 1; b -= 2) {
    uint32_t za = 0, zb = 0;  // bit b / bit b-1 of each element
#pragma unroll
    for (int j = 0; j < 4 * KR; ++j) {
      za |= ((hi[j] >> b) & 1u) << j;
      zb |= ((hi[j] >> (b - 1)) & 1u) << j;
    }
    const uint32_t d0 = c & ~(za | zb), d1 = c & ~za & zb, d2 = c & za & ~zb;
    const int n0 = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(d0));
    const int n1 = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(d1));
    const int n2 = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(d2));
    if (tt < n0) {
      c = d0;
      cc = n0;
    } else if (tt < n0 + n1) {
      c = d1;
      tt -= n0;
      cc = n1;
    } else if (tt < n0 + n1 + n2) {
      c = d2;
      tt -= n0 + n1;
      cc = n2;
    } else {
      c &= za & zb;
      tt -= n0 + n1 + n2;
      cc -= n0 + n1 + n2;
    }
  }
  if (cc > 1) return warp_select(wd, lane, F, cand, cnt, t);
  const uint32_t who = __ballot_sync(0xffffffffu, c != 0);
  const int src = __ffs(who) - 1;
  const int bit = __ffs(c) - 1;
  const int f = 128 * (bit >> 2) + 4 * lane + (bit & 3);
  return __shfl_sync(0xffffffffu, f, src);
}

__device__ __forceinline__ int select_rank(const uint64_t* wd, int lane, int F, uint32_t cand, int cnt, int t) {
  if (F <= 128) return warp_select_fast<1>(wd, lane, F, cand, cnt, t);
  if (F <= 256) return warp_select_fast<2>(wd, lane, F, cand, cnt, t);
  if (F <= 512) return warp_select_fast<4>(wd, lane, F, cand, cnt, t);
  return warp_select(wd, lane, F, cand, cnt, t);
}

// Places `nobj` objects on the (filtered) free cells of ranks 0..nobj-1 and
// records in misc[32] the cell of rank spawn_base + spawn_word % (count -
// spawn_base) (ref:scenarios.py:43-50), via warp_select: the element of
// rank nobj - 1 bounds the object cells, which are then ordered exactly
// among themselves.
__device__ void rank_place(const WarpScratch& ws, int lane, int F, int W, int mode, int x, int obj_lane,
                           int nobj, int spawn_base, uint64_t spawn_word) {
  const int K = (F + 127) >> 7;
  uint32_t valid = 0;
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int f = 128 * k + 4 * lane + i;
      if (f < F && col_ok(mode, ws.fc[f], W, x)) valid |= 1u << (4 * k + i);
    }
  const int total = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(valid));
  XMG_TRB(7);
  const int no = nobj < total ? nobj : total;
  uint32_t* list = reinterpret_cast<uint32_t*>(ws.slot);  // the object cells' element indices
  if (no > 0) {
    const int fb = select_rank(ws.wd, lane, F, valid, total, no - 1);
    XMG_TRB(8);
    const uint64_t wb = ws.wd[fb];
    int cnt = 0;
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int f = 128 * k + 4 * lane + i;
        bool in = false;
        if ((valid >> (4 * k + i)) & 1) {
          const uint64_t w = ws.wd[f];
          in = w < wb || (w == wb && f <= fb);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        if (in) list[cnt + __popc(m & ((1u << lane) - 1u))] = (uint32_t)f;
        cnt += __popc(m);
      }
    __syncwarp();
    XMG_TRB(9);
    // exact rank among the no (<= 32) smallest; object `rank` comes from
    // lane `rank` (objects were read into lanes before the draws)
    int f = 0, rank = 0;
    if (lane < no) {
      f = (int)list[lane];
      const uint64_t w = ws.wd[f];
      for (int m = 0; m < no; ++m) {
        const int g = (int)list[m];
        const uint64_t wg = ws.wd[g];
        rank += (wg < w) | ((wg == w) & (g < f));
      }
    }
    const int obj = __shfl_sync(0xffffffffu, obj_lane, rank & 31);
    if (lane < no) ws.grid[ws.fc[f]] = (uint8_t)obj;
  }
  XMG_TRB(10);
  const int tail = total - spawn_base;
  if (tail > 0) {
    const int fs = select_rank(ws.wd, lane, F, valid, total, spawn_base + (int)mod64_small(spawn_word, (uint32_t)tail));
    if (lane == 0) reinterpret_cast<int*>(ws.misc + 32)[0] = ws.fc[fs];
  }
  __syncwarp();
}

// Every key a trial reset consumes, derived from the episode key ek:
// ref:vecenv.py:224-227 (ks = split(ek, 0), next state key st = split(ek, 1))
// and ref:scenarios.py:55,106,125,138 (k0, k1, k2 = split(ks, 3)); and in
// resample mode (an extension, not in the reference) the task word
// draw0(split(ek, 2)) of Benchmark.sample_ruleset (ref:benchio.py:57-58).
struct TrialKeys {
  uint64_t st_hi, st_lo, k0h, k0l, k1h, k1l, k2h, k2l, task_word;
};

// The keys of up to 16 envs at once, spread over the lanes in two
// dependent rounds instead of five blocks in series per env: round 1 derives
// ks = split(ek, 0) and st = split(ek, 1) (+ split(ek, 2) for resample) of
// every env, round 2 the three children of ks (+ the resample draw).  Env
// slot k is lane `base + k` of `m` (its episode key in that lane's ek);
// results go to out[k].  Called by all 32 lanes.
__device__ __noinline__ void derive_keys_group(uint32_t m, int base, uint64_t ek_hi, uint64_t ek_lo, bool resample,
                                               TrialKeys* out, int lane) {
  const int nb1 = resample ? 3 : 2, nb2 = resample ? 4 : 3;
  const uint32_t slots = (m >> base) & 0xFFFFu;
  if (!slots) return;
  const int hi_slot = 32 - __clz(slots);  // slots 0 .. hi_slot-1 cover every env
  for (int j0 = 0; j0 < nb1 * hi_slot; j0 += 32) {
    const int j = j0 + lane, k = j / nb1, b = j - k * nb1;
    const uint64_t eh = shfl64(ek_hi, (base + k) & 31), el = shfl64(ek_lo, (base + k) & 31);
    if (j < nb1 * hi_slot && ((slots >> k) & 1)) {
      const Words4 w = philox<2>((uint64_t)b, 0, kDomSplit, 0, eh, el);
      TrialKeys& t = out[k];
      if (b == 0) { t.k2h = w.w0; t.k2l = w.w1; }        // ks, parked in k2 until round 2
      else if (b == 1) { t.st_hi = w.w0; t.st_lo = w.w1; }
      else { t.task_word = w.w0; t.k0h = w.w1; }        // split(ek, 2), parked
    }
  }
  __syncwarp();
  for (int j0 = 0; j0 < nb2 * hi_slot; j0 += 32) {
    const int j = j0 + lane, k = j / nb2, b = j - k * nb2;
    const bool act = j < nb2 * hi_slot && ((slots >> k) & 1);
    uint64_t kh = 0, kl = 0;
    if (act) {
      const TrialKeys& t = out[k];
      kh = b < 3 ? t.k2h : t.task_word;
      kl = b < 3 ? t.k2l : t.k0h;
    }
    __syncwarp();
    if (act) {
      const Words4 w = b < 3 ? philox<2>((uint64_t)b, 0, kDomSplit, 0, kh, kl) : philox<2>(0, 0, kDomDraw, 0, kh, kl);
      TrialKeys& t = out[k];
      if (b == 0) { t.k0h = w.w0; t.k0l = w.w1; }
      else if (b == 1) { t.k1h = w.w0; t.k1l = w.w1; }
      else if (b == 2) { t.k2h = w.w0; t.k2l = w.w1; }
      else t.task_word = w.w0;
    }
    __syncwarp();
  }
  if (!resample)
    for (int k = lane; k < hi_slot; k += 32) out[k].task_word = 0;
  __syncwarp();
}

// Rebuild one env's trial with the scenario builders ref:scenarios.py:53-174
// (batched: ref:vecenv.py:242-291).  Called by all 32 lanes with the same
// arguments; writes the new grid to `gdst` (and leaves it in ws.grid) and
// returns the new pose / goal / task on every lane.
__device__ __noinline__ void warp_build(const xmg_env_desc* dp, uint8_t* wbase, int hwp, int lane,
                                        const TrialKeys* keyp, int task_in, uint32_t goal_in, uint8_t* gdst,
                                        ResetOut* outp) {
  XMG_TRB(0);
  const TrialKeys key = *keyp;
  const xmg_env_desc& d = *dp;  // CTA copy in shared memory
  const WarpScratch ws = make_scratch(wbase, hwp);
  const int H = d.height, W = d.width, HW = H * W;
  const int sc = d.scenario;
  ResetOut res;
  res.st_hi = key.st_hi;
  res.st_lo = key.st_lo;
  res.goal = goal_in;
  res.task = task_in;
  if (d.resample_tasks && sc == XMG_SCENARIO_XLAND) {
    res.task = (int)(key.task_word % (uint64_t)d.num_tasks);
    res.goal = d.task_rows[(int64_t)res.task * d.row_words];
  }
  const uint32_t* row = d.task_rows + (int64_t)res.task * d.row_words;
  // the objects this trial places, one per lane, read now so the load is in
  // flight during the draws (ref:vecenv.py:261-270; FourRooms: the goal,
  // ref:scenarios.py:123-132; EmptyRandom: none)
  int nobj = 0, obj_lane = 0;
  if (sc == XMG_SCENARIO_XLAND) {
    nobj = (int)((row[1] >> 8) & 0xff);
    if (lane < nobj) obj_lane = reinterpret_cast<const uint8_t*>(row + kRowHeader + d.rule_width)[lane];
  } else if (sc == XMG_SCENARIO_FOUR_ROOMS) {
    nobj = 1;
    obj_lane = kGreenGoal;
  }
  // base cells of this scenario, 16 bytes per lane (base_cells and the
  // scratch grid are 16-byte aligned and padded)
  for (int i = lane; i < (HW + 15) >> 4; i += 32)
    reinterpret_cast<uint4*>(ws.grid)[i] = __ldg(reinterpret_cast<const uint4*>(d.base_cells) + i);
  if (sc == XMG_SCENARIO_EMPTY) {  // ref:scenarios.py:82-89
    __syncwarp();
    warp_store_grid(gdst, ws.grid, HW, lane);
    res.r = 1; res.c = 1; res.d = 1;
    res.goal = 2u | ((uint32_t)kGreenGoal << 8);
    if (lane == 0) *outp = res;
    __syncwarp();
    return;
  }
  const uint64_t k0h = key.k0h, k0l = key.k0l, k1h = key.k1h, k1l = key.k1l, k2h = key.k2h, k2l = key.k2l;

  int wall_col = -1, color = 0;
  const bool two_rooms = sc == XMG_SCENARIO_DOOR_KEY || sc == XMG_SCENARIO_UNLOCK || sc == XMG_SCENARIO_UNLOCK_PICKUP;
  if (two_rooms) {  // ref:scenarios.py:103-115, 135-147
    Words4 w = {0, 0, 0, 0};
    if (lane == 0) w = philox<2>(0, 0, kDomDraw, 0, k0h, k0l);
    const uint64_t w0 = shfl64(w.w0, 0), w1 = shfl64(w.w1, 0);
    int door_row;
    if (sc == XMG_SCENARIO_DOOR_KEY) {
      wall_col = 2 + (int)mod64_small(w0, (uint32_t)(W - 4));
      door_row = 1 + (int)mod64_small(w1, (uint32_t)(H - 2));
      color = 7;  // yellow
    } else {
      wall_col = (W - 1) / 2;
      door_row = 1 + (int)mod64_small(w0, (uint32_t)(H - 2));
      color = cGenColors[w1 % 10];
    }
    __syncwarp();
    for (int r = lane; r < H; r += 32) ws.grid[r * W + wall_col] = kWallCode;
    __syncwarp();
    if (lane == 0) ws.grid[door_row * W + wall_col] = (uint8_t)(kLocked * 16 + color);
  }
  __syncwarp();
  XMG_TRB(1);
  const int F = build_free_list(ws, HW, lane);
  XMG_TRB(2);
  const int nseg = (sc == XMG_SCENARIO_XLAND || sc == XMG_SCENARIO_FOUR_ROOMS) ? d.num_segments : 0;
  draw_all(ws, lane, F, k1h, k1l, nseg, k0h, k0l, k2h, k2l);
  XMG_TRB(3);
  // doors: ref:layouts.py:109-121 (segments never hold free cells)
  if (lane < nseg) {
    const int off = d.seg_off[lane], len = d.seg_off[lane + 1] - off;
    const int pos = d.fixed_doors ? len / 2 : (int)mod64_small(ws.misc[2 * lane], (uint32_t)len);
    ws.grid[d.seg_cells[off + pos]] = (uint8_t)(kClosed * 16 + cGenColors[ws.misc[2 * lane + 1] % 10]);
  }
  const uint64_t a0 = ws.misc[24], a1 = ws.misc[25];
  res.d = (int)(a1 & 3);  // a1 % 4
  if (sc == XMG_SCENARIO_XLAND || sc == XMG_SCENARIO_FOUR_ROOMS || sc == XMG_SCENARIO_EMPTY_RANDOM) {
    if (sc != XMG_SCENARIO_XLAND) res.goal = 2u | ((uint32_t)kGreenGoal << 8);  // ref:scenarios.py:92-132
    rank_place(ws, lane, F, W, 0, 0, obj_lane, nobj, nobj, a0);
  } else {  // two-room ports: shuffle all free cells, keep the left room
    rank_place(ws, lane, F, W, 1, wall_col, kKey * 16 + color, 1, 1, a0);
    if (sc == XMG_SCENARIO_DOOR_KEY) {
      res.goal = 2u | ((uint32_t)kGreenGoal << 8);
    } else if (sc == XMG_SCENARIO_UNLOCK) {  // ref:scenarios.py:155-159
      res.goal = 2u | ((uint32_t)(kOpen * 16 + color) << 8);
    } else {  // UNLOCK_PICKUP, ref:scenarios.py:162-174: reshuffle with the key placed
      const int ball = kBall * 16 + cGenColors[ws.wd[2] % 10];
      const int F2 = build_free_list(ws, HW, lane);  // draw words for indices < F2 are unchanged
      uint64_t bw = ~0ull;
      int bg = 0x7fffffff;
      for (int f = lane; f < F2; f += 32) {
        if (!col_ok(2, ws.fc[f], W, wall_col)) continue;
        const uint64_t w = ws.wd[f];
        if (w < bw || (w == bw && f < bg)) { bw = w; bg = f; }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        const uint64_t ow = shfl64(bw, (lane + off) & 31);
        const int og = __shfl_sync(0xffffffffu, bg, (lane + off) & 31);
        if (ow < bw || (ow == bw && og < bg)) { bw = ow; bg = og; }
      }
      if (lane == 0 && bg < F2) ws.grid[ws.fc[bg]] = (uint8_t)ball;
      res.goal = 1u | ((uint32_t)ball << 8);
      __syncwarp();
    }
  }
  XMG_TRB(4);
  const int spawn_cell = reinterpret_cast<const int*>(ws.misc + 32)[0];
  res.r = spawn_cell / W;
  res.c = spawn_cell - res.r * W;
  warp_store_grid(gdst, ws.grid, HW, lane);
  if (lane == 0) *outp = res;
  __syncwarp();
  XMG_TRB(5);
}
